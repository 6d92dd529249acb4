"""B200-native generalized sparse convolution (Choy et al., arXiv 1904.08755) — Python binding.

Thin marshalling layer over the C ABI in ``include/mk.h`` (libmk.so): every step of the
hot path runs in the library's sm_100a kernels; torch provides device memory, streams
and (in ``dist``) process groups.  Function names mirror the C entry points without the
``mk_`` prefix.  There is no CPU or eager fallback: without a CUDA device and libmk.so
the calls raise.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib
from ._lib import BF16, CUSTOM, F32, HYBRID, HYPERCROSS, HYPERCUBE, POOL_AVG, POOL_MAX, POOL_SUM

__all__ = [
    "MkError", "Coords", "KernelMap", "Region", "context",
    "coords_quantize", "coords_create", "coords_stride", "coords_lookup", "coords_export",
    "region_offsets", "kmap_build", "kmap_export",
    "conv_forward", "conv_backward", "conv_transpose_forward", "conv_transpose_backward",
    "kernel_launch_count", "HYPERCUBE", "HYPERCROSS", "HYBRID", "CUSTOM", "F32", "BF16",
]

_L = _lib.load()


class MkError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.name = _lib.STATUS.get(status, str(status))
        self.row = int(_L.mk_last_error_row())
        msg = _L.mk_last_error_message().decode(errors="replace")
        super().__init__(f"{where}: {self.name}: {msg}")


def _check(st: int, where: str):
    if st != 0:
        raise MkError(st, where)


_ctx = {}


def context(device: Optional[int] = None) -> ctypes.c_void_p:
    """The library context of a CUDA device (created once per device)."""
    if device is None:
        device = torch.cuda.current_device()
    if device not in _ctx:
        h = ctypes.c_void_p()
        _check(_L.mk_context_create(device, None, None, None, ctypes.byref(h)), "mk_context_create")
        _ctx[device] = h
    return _ctx[device]


def _stream(t: Optional[torch.Tensor] = None) -> int:
    """Raw handle of torch's current stream on the tensor's device (cheap accessor)."""
    idx = t.device.index if t is not None else torch.cuda.current_device()
    return torch._C._cuda_getCurrentRawStream(idx)


class _on_device:
    """Makes `device` current for the duration of a call, only when it is not already."""

    __slots__ = ("idx", "prev")

    def __init__(self, device):
        self.idx = device.index if isinstance(device, torch.device) else int(device)
        self.prev = None

    def __enter__(self):
        cur = torch.cuda.current_device()
        if cur != self.idx:
            self.prev = cur
            torch.cuda.set_device(self.idx)

    def __exit__(self, *exc):
        if self.prev is not None:
            torch.cuda.set_device(self.prev)


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _cuda(t: torch.Tensor, dtype: torch.dtype, what: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{what} must be a CUDA tensor (no CPU path)")
    return t.to(dtype).contiguous()


def kernel_launch_count() -> int:
    return int(_L.mk_kernel_launch_count())


# ------------------------------------------------------------------------------ coords
class Coords:
    """Immutable coordinate set C (Eq. 1) with its GPU hash table (``mk_coords``)."""

    def __init__(self, handle: ctypes.c_void_p, device: torch.device, deferred: bool = False):
        self._h = handle
        self.device = device
        n, D = ctypes.c_int64(), ctypes.c_int32()
        ts = (ctypes.c_int32 * 8)()  # >= MK_MAX_DIM
        _check(_L.mk_coords_info(handle, None if deferred else ctypes.byref(n), ctypes.byref(D), ts), "mk_coords_info")
        self.D = int(D.value)
        self.tensor_stride = [int(ts[d]) for d in range(self.D)]
        self._n = None if deferred else int(n.value)

    @property
    def n(self) -> int:
        """Row count N.  For a deferred quantize the first access waits for it (and raises
        the input error, if any)."""
        if self._n is None:
            n = ctypes.c_int64()
            _check(_L.mk_coords_info(self._h, ctypes.byref(n), None, None), "mk_coords_info")
            self._n = int(n.value)
        return self._n

    def __len__(self):
        return self.n

    def __del__(self):
        if getattr(self, "_h", None) and _L is not None:
            _L.mk_coords_destroy(self._h)
            self._h = None

    def export(self) -> torch.Tensor:
        return coords_export(self)

    def lookup(self, queries: torch.Tensor) -> torch.Tensor:
        return coords_lookup(self, queries)


def coords_quantize(points: torch.Tensor, voxel: float, batch: Optional[torch.Tensor] = None,
                    return_maps: bool = True, deferred: bool = False):
    """Alg. 1 -> (Coords, point_to_row int32 [N_p], first_point int32 [N]).
    deferred=True returns before the row count is known (mk_coords_quantize_deferred): the
    count is collected when first needed (Coords.n, a kernel-map build, ...), and first_point
    is returned with its full capacity N_p (rows >= N undefined)."""
    pts = _cuda(points, torch.float32, "points")
    n, D = pts.shape
    b = None if batch is None else _cuda(batch, torch.int32, "batch")
    p2r = torch.empty(n, dtype=torch.int32, device=pts.device) if return_maps else None
    first = torch.empty(max(n, 1), dtype=torch.int32, device=pts.device) if return_maps else None
    h = ctypes.c_void_p()
    fn = _L.mk_coords_quantize_deferred if deferred else _L.mk_coords_quantize
    with _on_device(pts.device):
        _check(fn(context(pts.device.index), _ptr(pts), _ptr(b), n, D, ctypes.c_float(voxel), _stream(pts),
                  ctypes.byref(h), _ptr(p2r), _ptr(first)), "mk_coords_quantize")
    c = Coords(h, pts.device, deferred=deferred)
    if not return_maps:
        return c
    if deferred:
        # capacity N_p, rows >= N undefined: coords_labels cuts it to c.n (collecting the count)
        first._mk_deferred_coords = c
        return c, p2r, first
    return c, p2r, first[:c.n]


def coords_labels(point_to_row: torch.Tensor, first_point: torch.Tensor, labels: torch.Tensor,
                  ignore_label: int = -1, coords: Optional["Coords"] = None) -> torch.Tensor:
    """Per-voxel labels of Alg. 1: the points' common label, else ignore_label.
    point_to_row / first_point are the maps returned by coords_quantize.  With a deferred
    quantize pass its Coords as `coords`: first_point then has capacity N_p and only its
    first c.n rows are defined, so it is cut to them (rows >= N would index out of bounds)."""
    coords = coords if coords is not None else getattr(first_point, "_mk_deferred_coords", None)
    if coords is not None:
        first_point = first_point[:coords.n]
    if first_point.shape[0] > point_to_row.shape[0]:
        raise ValueError("first_point has more rows than there are points")
    p2r = _cuda(point_to_row, torch.int32, "point_to_row")
    first = _cuda(first_point, torch.int32, "first_point")
    lab = _cuda(labels, torch.int32, "labels")
    if lab.shape[0] != p2r.shape[0]:
        raise ValueError("labels and point_to_row must have one entry per point")
    out = torch.empty(first.shape[0], dtype=torch.int32, device=p2r.device)
    with _on_device(p2r.device):
        _check(_L.mk_coords_labels(_ptr(p2r), _ptr(first), _ptr(lab), p2r.shape[0], first.shape[0], int(ignore_label),
                                   _ptr(out), _stream(p2r)), "mk_coords_labels")
    return out


def coords_create(coords: torch.Tensor, tensor_stride: Optional[Sequence[int]] = None, return_inverse: bool = False):
    """Coordinate set from integer rows [n][D+1] (batch last); first occurrence wins."""
    c = _cuda(coords, torch.int32, "coords")
    n, Dp1 = c.shape
    D = Dp1 - 1
    ts = None if tensor_stride is None else (ctypes.c_int32 * D)(*tensor_stride)
    inv = torch.empty(n, dtype=torch.int32, device=c.device) if return_inverse else None
    h = ctypes.c_void_p()
    with _on_device(c.device):
        _check(_L.mk_coords_create(context(c.device.index), _ptr(c), n, D, ts, _stream(c), ctypes.byref(h), _ptr(inv)),
               "mk_coords_create")
    out = Coords(h, c.device)
    return (out, inv) if return_inverse else out


def coords_stride(cin: Coords, conv_stride: Sequence[int]) -> Coords:
    """Strided output coordinates (R11)."""
    cs = (ctypes.c_int32 * cin.D)(*conv_stride)
    h = ctypes.c_void_p()
    with _on_device(cin.device):
        _check(_L.mk_coords_stride(context(cin.device.index), cin._h, cs, _stream(), ctypes.byref(h)),
               "mk_coords_stride")
    return Coords(h, cin.device)


def coords_expand(cin: Coords, region: "Region", tensor_stride: Optional[Sequence[int]] = None) -> Coords:
    """Generative transposed-conv output coordinates (f4): {u + i * s_out}."""
    r = region._struct()
    ts = None if tensor_stride is None else (ctypes.c_int32 * cin.D)(*tensor_stride)
    h = ctypes.c_void_p()
    with _on_device(cin.device):
        _check(_L.mk_coords_expand(context(cin.device.index), cin._h, ctypes.byref(r), ts, _stream(),
                                   ctypes.byref(h)), "mk_coords_expand")
    return Coords(h, cin.device)


def coords_export(c: Coords) -> torch.Tensor:
    out = torch.empty((c.n, c.D + 1), dtype=torch.int32, device=c.device)
    with _on_device(c.device):
        _check(_L.mk_coords_export(c._h, _ptr(out), _stream()), "mk_coords_export")
    return out


def coords_lookup(c: Coords, queries: torch.Tensor) -> torch.Tensor:
    q = _cuda(queries, torch.int32, "queries")
    rows = torch.empty(q.shape[0], dtype=torch.int32, device=q.device)
    with _on_device(c.device):
        _check(_L.mk_coords_lookup(c._h, _ptr(q), q.shape[0], _ptr(rows), _stream()), "mk_coords_lookup")
    return rows


# ------------------------------------------------------------------------------ regions
class Region:
    """Kernel offset set N^D description (``mk_region``)."""

    def __init__(self, kind: int, D: int, size=3, dilation=1, temporal_axis: int = -1, offsets=None):
        self.kind, self.D = kind, D
        self.size = list(size) if np.ndim(size) else [size] * D
        self.dilation = list(dilation) if np.ndim(dilation) else [dilation] * D
        self.temporal_axis = temporal_axis
        self.offsets = None if offsets is None else np.ascontiguousarray(offsets, np.int32).reshape(-1, D)

    def _struct(self) -> _lib.MkRegion:
        s = getattr(self, "_s", None)  # built once: a Region is not modified after construction
        if s is None:
            s = self._s = self._build_struct()
        return s

    def _build_struct(self) -> _lib.MkRegion:
        r = _lib.MkRegion()
        r.type, r.D, r.temporal_axis = self.kind, self.D, self.temporal_axis
        for d in range(self.D):
            r.size[d] = self.size[d]
            r.dilation[d] = self.dilation[d]
        if self.offsets is not None:
            r.offsets = self.offsets.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
            r.n_offsets = self.offsets.shape[0]
        return r


def region_offsets(region: Region) -> np.ndarray:
    r = region._struct()
    K = ctypes.c_int32()
    _check(_L.mk_region_offsets(ctypes.byref(r), ctypes.byref(K), None), "mk_region_offsets")
    out = np.zeros((K.value, region.D), np.int32)
    _check(_L.mk_region_offsets(ctypes.byref(r), ctypes.byref(K), out.ctypes.data_as(ctypes.c_void_p)),
           "mk_region_offsets")
    return out


# ------------------------------------------------------------------------------ kernel maps
class KernelMap:
    """Immutable kernel map M = {(I_i, O_i)} with its conv-side neighbour tables."""

    def __init__(self, handle, device, cin: Coords, cout: Coords, transposed: bool):
        self._h = handle
        self.device = device
        self.transposed = transposed
        self._keep = (cin, cout)  # a map never outlives the coordinate sets it indexes
        K, nin, nout = ctypes.c_int32(), ctypes.c_int64(), ctypes.c_int64()
        _check(_L.mk_kmap_info(handle, ctypes.byref(K), None, ctypes.byref(nin), ctypes.byref(nout)), "mk_kmap_info")
        self.K, self.n_in, self.n_out = K.value, nin.value, nout.value
        self._n_pairs = None

    @property
    def n_pairs(self) -> int:
        """|M|.  The build is asynchronous; the first access waits for it (event wait)."""
        if self._n_pairs is None:
            n = ctypes.c_int64()
            _check(_L.mk_kmap_info(self._h, None, ctypes.byref(n), None, None), "mk_kmap_info")
            self._n_pairs = n.value
        return self._n_pairs

    def __del__(self):
        if getattr(self, "_h", None) and _L is not None:
            _L.mk_kmap_destroy(self._h)
            self._h = None

    def export(self):
        return kmap_export(self)


def kmap_build(cin: Coords, cout: Coords, region: Region, transposed: bool = False) -> KernelMap:
    r = region._struct()
    h = ctypes.c_void_p()
    with _on_device(cin.device):
        _check(_L.mk_kmap_build(context(cin.device.index), cin._h, cout._h, ctypes.byref(r), int(transposed),
                                _stream(), ctypes.byref(h)), "mk_kmap_build")
    return KernelMap(h, cin.device, cin, cout, transposed)


def kmap_export(m: KernelMap):
    """CSR (ptr int64 [K+1], in int32 [|M|], out int32 [|M|]) on the device."""
    ptr = torch.empty(m.K + 1, dtype=torch.int64, device=m.device)
    ins = torch.empty(m.n_pairs, dtype=torch.int32, device=m.device)
    outs = torch.empty(m.n_pairs, dtype=torch.int32, device=m.device)
    with _on_device(m.device):
        _check(_L.mk_kmap_export(m._h, _ptr(ptr), _ptr(ins), _ptr(outs), _stream()), "mk_kmap_export")
    return ptr, ins, outs


# ------------------------------------------------------------------------------ convolution
_DT = {torch.float32: F32, torch.bfloat16: BF16}


def _dt(t: torch.Tensor) -> int:
    if t.dtype not in _DT:
        raise TypeError(f"features must be float32 or bfloat16, got {t.dtype}")
    return _DT[t.dtype]


def _out_buf(buf, shape, dtype, device, what):
    """A caller-supplied output buffer after validation, or a new one."""
    if buf is None:
        return torch.empty(shape, dtype=dtype, device=device)
    if tuple(buf.shape) != tuple(shape) or buf.dtype != dtype or buf.device != device or not buf.is_contiguous():
        raise ValueError(f"{what}: expected a contiguous {dtype} tensor of shape {tuple(shape)} on {device}, got "
                         f"{buf.dtype} {tuple(buf.shape)} on {buf.device} (contiguous={buf.is_contiguous()})")
    return buf


def _conv(fn, name, m: KernelMap, f_in, W, out_dtype, out=None):
    if not (f_in.is_cuda and W.is_cuda):
        raise ValueError("conv inputs must be CUDA tensors (no CPU path)")
    K, c_out, c_in = W.shape
    if K != m.K or f_in.shape[-1] != c_in or f_in.shape[0] != m.n_in or W.dtype != f_in.dtype:
        raise ValueError(f"{name}: shape/dtype mismatch (K={m.K}, n_in={m.n_in})")
    out_dtype = out_dtype or f_in.dtype
    y = _out_buf(out, (m.n_out, c_out), out_dtype, f_in.device, "out")
    # contiguous copies are bound to locals so they stay alive until the call returns (a
    # temporary freed early could be reused by the next argument's copy)
    x, w = f_in.contiguous(), W.contiguous()
    with _on_device(f_in.device):
        _check(fn(context(f_in.device.index), m._h, _ptr(x), c_in, _ptr(w), _ptr(y),
                  c_out, _dt(f_in), _DT[out_dtype], _stream(f_in)), name)
    return y


def conv_forward(m: KernelMap, f_in: torch.Tensor, W: torch.Tensor, out_dtype=None, out=None, scale=None,
                 shift=None, residual=None, relu: bool = False) -> torch.Tensor:
    """Alg. 2: F_out[o] = sum_k W_k F_in[I_k] scattered to O_k.  W [K][C_out][C_in].
    With scale / shift (fp32 [C_out], folded BatchNorm), residual ([n_out][C_out], output
    dtype) or relu, the row-wise epilogue act(conv * scale + shift + residual) runs fused in
    the conv kernel (mk_conv_forward_fused)."""
    if scale is None and shift is None and residual is None and not relu:
        return _conv(_L.mk_conv_forward, "mk_conv_forward", m, f_in, W, out_dtype, out)
    return _conv_fused(m, f_in, W, out_dtype, out, scale, shift, residual, relu)


def _conv_fused(m: KernelMap, f_in, W, out_dtype, out, scale, shift, residual, relu):
    if not (f_in.is_cuda and W.is_cuda):
        raise ValueError("conv inputs must be CUDA tensors (no CPU path)")
    K, c_out, c_in = W.shape
    if K != m.K or f_in.shape[-1] != c_in or f_in.shape[0] != m.n_in or W.dtype != f_in.dtype:
        raise ValueError(f"mk_conv_forward_fused: shape/dtype mismatch (K={m.K}, n_in={m.n_in})")
    out_dtype = out_dtype or f_in.dtype
    y = _out_buf(out, (m.n_out, c_out), out_dtype, f_in.device, "out")
    sc = None if scale is None else _cuda(scale, torch.float32, "scale")
    sh = None if shift is None else _cuda(shift, torch.float32, "shift")
    for t, nm in ((sc, "scale"), (sh, "shift")):
        if t is not None and t.numel() != c_out:
            raise ValueError(f"{nm} must have C_out = {c_out} entries")
    res = None
    if residual is not None:
        res = _cuda(residual, out_dtype, "residual")
        if tuple(res.shape) != (m.n_out, c_out):
            raise ValueError("residual must be [n_out][C_out]")
    x, w = f_in.contiguous(), W.contiguous()
    with _on_device(f_in.device):
        _check(_L.mk_conv_forward_fused(context(f_in.device.index), m._h, _ptr(x), c_in,
                                        _ptr(w), _ptr(y), c_out, _dt(f_in), _DT[out_dtype], _ptr(sc),
                                        _ptr(sh), _ptr(res), int(bool(relu)), _stream(f_in)), "mk_conv_forward_fused")
    return y


def conv_transpose_forward(m: KernelMap, f_in: torch.Tensor, W: torch.Tensor, out_dtype=None, out=None, scale=None,
                           shift=None, residual=None, relu: bool = False):
    """Transposed conv on a map built with transposed=True; the optional fused
    epilogue is that of conv_forward."""
    if scale is None and shift is None and residual is None and not relu:
        return _conv(_L.mk_conv_transpose_forward, "mk_conv_transpose_forward", m, f_in, W, out_dtype, out)
    if not m.transposed:
        raise ValueError("conv_transpose_forward: the map is not transposed")
    return _conv_fused(m, f_in, W, out_dtype, out, scale, shift, residual, relu)


def _backward(fn, name, m: KernelMap, g_out, f_in, W, need_gin=True, need_gw=True, gin=None, gw=None):
    K, c_out, c_in = W.shape
    if g_out.shape != (m.n_out, c_out) or f_in.shape != (m.n_in, c_in) or K != m.K:
        raise ValueError(f"{name}: shape mismatch")
    if not (g_out.dtype == f_in.dtype == W.dtype):
        raise TypeError(f"{name}: g_out, f_in and W must share a dtype")
    if need_gin:
        gin = _out_buf(gin, (m.n_in, c_in), f_in.dtype, f_in.device, "gin")
    if need_gw:
        gw = _out_buf(gw, (K, c_out, c_in), torch.float32, f_in.device, "gw")
    g, x, w = g_out.contiguous(), f_in.contiguous(), W.contiguous()  # alive until the call returns
    with _on_device(f_in.device):
        _check(fn(context(f_in.device.index), m._h, _ptr(g), _ptr(x),
                  _ptr(w), c_in, c_out, _dt(f_in), _ptr(gin if need_gin else None),
                  _ptr(gw if need_gw else None), _stream(f_in)), name)
    return (gin if need_gin else None), (gw if need_gw else None)


def conv_backward(m: KernelMap, g_out, f_in, W, need_gin=True, need_gw=True, gin=None, gw=None):
    """(G_in, dW) of conv_forward; dW is float32 [K][C_out][C_in]."""
    return _backward(_L.mk_conv_backward, "mk_conv_backward", m, g_out, f_in, W, need_gin, need_gw, gin, gw)


def conv_transpose_backward(m: KernelMap, g_out, f_in, W, need_gin=True, need_gw=True, gin=None, gw=None):
    return _backward(_L.mk_conv_transpose_backward, "mk_conv_transpose_backward", m, g_out, f_in, W, need_gin,
                     need_gw, gin, gw)


# ------------------------------------------------------------------------------ pooling
def pool_forward(m: KernelMap, f_in: torch.Tensor, mode: int = POOL_MAX, out=None, argmax=None):
    """Pooling over a kernel map: POOL_MAX (Alg. 3), POOL_AVG / POOL_SUM (Alg. 4).
    Returns (f_out [n_out][C], argmax [n_out][C] int32 for max pooling, else None)."""
    if not f_in.is_cuda:
        raise ValueError("pool inputs must be CUDA tensors (no CPU path)")
    if f_in.shape[0] != m.n_in:
        raise ValueError(f"pool_forward: f_in has {f_in.shape[0]} rows, the map has n_in={m.n_in}")
    x = f_in.contiguous()
    C = x.shape[1]
    y = _out_buf(out, (m.n_out, C), x.dtype, x.device, "out")
    am = None
    if mode == POOL_MAX:
        am = _out_buf(argmax, (m.n_out, C), torch.int32, x.device, "argmax")
    with _on_device(x.device):
        _check(_L.mk_pool_forward(context(x.device.index), m._h, int(mode), _ptr(x), C, _dt(x), _ptr(y), _ptr(am),
                                  _stream(x)), "mk_pool_forward")
    return y, am


def pool_backward(m: KernelMap, g_out: torch.Tensor, mode: int = POOL_MAX, argmax=None, out=None):
    """Reverse mode of pool_forward: G_in [n_in][C] (argmax required for POOL_MAX)."""
    if g_out.shape[0] != m.n_out:
        raise ValueError(f"pool_backward: g_out has {g_out.shape[0]} rows, the map has n_out={m.n_out}")
    g = g_out.contiguous()
    C = g.shape[1]
    gi = _out_buf(out, (m.n_in, C), g.dtype, g.device, "out")
    if mode == POOL_MAX:
        if argmax is None:
            raise ValueError("pool_backward: POOL_MAX needs the argmax of pool_forward")
        argmax = _out_buf(argmax, (m.n_out, C), torch.int32, g.device, "argmax")
    with _on_device(g.device):
        _check(_L.mk_pool_backward(context(g.device.index), m._h, int(mode), _ptr(g), C, _dt(g), _ptr(argmax),
                                   _ptr(gi), _stream(g)), "mk_pool_backward")
    return gi


def global_pool(c: Coords, f_in: torch.Tensor, n_batch: int, mode: int = POOL_AVG) -> torch.Tensor:
    """Global pooling: [n_batch][C] sum / mean of the rows of each batch index."""
    if f_in.shape[0] != c.n:
        raise ValueError("global_pool: f_in must have one row per coordinate")
    x = f_in.contiguous()
    y = torch.empty((n_batch, x.shape[1]), dtype=x.dtype, device=x.device)
    with _on_device(x.device):
        _check(_L.mk_global_pool(context(x.device.index), c._h, int(mode), _ptr(x), x.shape[1], _dt(x), int(n_batch),
                                 _ptr(y), _stream(x)), "mk_global_pool")
    return y


# ------------------------------------------------------------------------------ TS-CRF
def crf_infer(m: KernelMap, phi_u: torch.Tensor, W: torch.Tensor, n_iters: int = 3) -> torch.Tensor:
    """Mean-field TS-CRF inference (Alg. 5): Q^N over the map's node set; fp32."""
    phi = _cuda(phi_u, torch.float32, "phi_u")
    w = _cuda(W, torch.float32, "W")
    n, C = phi.shape
    if n != m.n_out or m.n_in != m.n_out or tuple(w.shape) != (m.K, C, C):
        raise ValueError("crf_infer: phi_u [n][C] over the map's nodes and W [K][C][C] expected")
    q = torch.empty_like(phi)
    with _on_device(phi.device):
        _check(_L.mk_crf_infer(context(phi.device.index), m._h, _ptr(phi), _ptr(w), C, int(n_iters), _ptr(q),
                               _stream(phi)), "mk_crf_infer")
    return q


def crf_backward(m: KernelMap, phi_u: torch.Tensor, W: torch.Tensor, n_iters: int, grad_q: torch.Tensor):
    """Eq. 5: (dL/dphi_u [n][C], dL/dW [K][C][C]) of crf_infer's Q^N given
    dL/dQ^N, by backpropagation through the n_iters mean-field steps; fp32."""
    phi = _cuda(phi_u, torch.float32, "phi_u")
    w = _cuda(W, torch.float32, "W")
    g = _cuda(grad_q, torch.float32, "grad_q")
    n, C = phi.shape
    if n != m.n_out or m.n_in != m.n_out or tuple(w.shape) != (m.K, C, C) or tuple(g.shape) != (n, C):
        raise ValueError("crf_backward: phi_u / grad_q [n][C] over the map's nodes and W [K][C][C] expected")
    gphi = torch.empty_like(phi)
    gw = torch.zeros_like(w)
    with _on_device(phi.device):
        _check(_L.mk_crf_backward(context(phi.device.index), m._h, _ptr(phi), _ptr(w), C, int(n_iters), _ptr(g),
                                  _ptr(gphi), _ptr(gw), _stream(phi)), "mk_crf_backward")
    return gphi, gw


def debug_sort_perm(keys: torch.Tensor, bits: int) -> torch.Tensor:
    """The map builder's stable radix sort (mk_debug_sort_perm): permutation sorting the low
    `bits` bits of uint32 keys (given as int32 / int64 tensors of non-negative values)."""
    k = _cuda(keys, torch.int32, "keys")
    perm = torch.empty(k.shape[0], dtype=torch.int32, device=k.device)
    with _on_device(k.device):
        _check(_L.mk_debug_sort_perm(context(k.device.index), _ptr(k), k.shape[0], int(bits), _ptr(perm),
                                     _stream(k)), "mk_debug_sort_perm")
    return perm
