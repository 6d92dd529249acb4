"""CPU oracle for the generalized sparse convolution hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` leg may import this package.  The product path
(``paper_1904_08755_b200``) never imports it and shares no code with it.

This module is argument marshalling over ``liboracle.so`` (oracle.cpp, plain C++17,
fp64, ``std::unordered_map``).  Each wrapper names the passage of the paper it follows
(``P:n`` = line n of PAPER.md).  Pins: tests/test_oracle_*.py.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SO = _HERE / "liboracle.so"

OK, INVALID_ARGUMENT, DIMENSION_MISMATCH, SHAPE_MISMATCH = 0, 1, 2, 3
NONFINITE_INPUT, COORD_RANGE, STRIDE, UNSUPPORTED = 4, 5, 6, 7
HYPERCUBE, HYPERCROSS, HYBRID, CUSTOM = 0, 1, 2, 3


class OracleError(RuntimeError):
    def __init__(self, status: int, row: int = -1):
        super().__init__(f"oracle status {status} (row {row})")
        self.status = status
        self.row = row


def build(force: bool = False) -> Path:
    """Compile oracle.cpp (no fast-math: reading R6 needs IEEE fp32 division)."""
    src = _HERE / "oracle.cpp"
    if force or not _SO.exists() or _SO.stat().st_mtime < max(src.stat().st_mtime, (_HERE / "oracle.h").stat().st_mtime):
        tmp = _SO.with_suffix(f".so.{os.getpid()}")
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fPIC", "-shared", "-fno-fast-math", "-fopenmp",
                               "-o", str(tmp), str(src)])
        os.replace(tmp, _SO)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_SO))
        P = ctypes.c_void_p
        i32, i64, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        L.orc_quantize.argtypes = [P, P, i64, i32, f32, P, P, P, P, P]
        L.orc_create.argtypes = [P, i64, i32, P, P, P, P, P]
        L.orc_stride.argtypes = [P, i64, i32, P, P, P, P, P]
        L.orc_region.argtypes = [i32, i32, P, P, i32, P, i32, P, P]
        L.orc_lookup.argtypes = [P, i64, i32, P, i64, P]
        L.orc_labels.argtypes = [P, P, i64, i64, i32, P]
        L.orc_expand.argtypes = [P, i64, i32, P, i32, P, P, P, P]
        L.orc_pool_forward.argtypes = [P, P, P, i32, P, i32, i64, i32, P, P]
        L.orc_pool_backward.argtypes = [P, P, P, i32, P, i32, i64, i32, P, P, i64]
        L.orc_global_pool.argtypes = [P, i64, P, i32, i32, i32, P]
        L.orc_crf_infer.argtypes = [P, P, P, i32, P, i64, i32, P, i32, P]
        L.orc_kmap.argtypes = [P, i64, P, i64, i32, P, i32, P, i32, P, P, P]
        L.orc_conv_forward.argtypes = [P, P, P, i32, P, i32, P, P, i64, i32]
        L.orc_conv_forward_rows.argtypes = [P, P, P, i32, P, i32, P, i32, P, i64, P]
        L.orc_conv_dgrad.argtypes = [P, P, P, i32, P, i32, P, P, i64, i32]
        L.orc_conv_wgrad.argtypes = [P, P, P, i32, P, i32, P, i32, P]
        L.orc_kmap_reverse.argtypes = [P, P, P, i32, P, P, P]
        L.orc_set_threads.argtypes = [i32]
        L.orc_set_threads.restype = ctypes.c_int
        for f in ("orc_quantize", "orc_create", "orc_stride", "orc_region", "orc_lookup", "orc_kmap"):
            getattr(L, f).restype = ctypes.c_int
        _lib = L
    return _lib


def set_threads(n: int = 0) -> int:
    """Threads of the oracle's OpenMP loops (0 = leave as is); returns the count in effect.
    Results are bit-identical for any count (only disjoint writes are split)."""
    return int(lib().orc_set_threads(int(n)))


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def quantize(points, voxel: float, batch=None):
    """Alg. 1: returns (coords[N][D+1], point_to_row[N_p], first_point[N])."""
    pts = _c(points, np.float32)
    n, D = pts.shape
    b = None if batch is None else _c(batch, np.int32)
    coords = np.zeros((max(n, 1), D + 1), np.int32)
    p2r = np.zeros(max(n, 1), np.int32)
    first = np.zeros(max(n, 1), np.int32)
    n_out, err = ctypes.c_int64(), ctypes.c_int64()
    st = lib().orc_quantize(_p(pts), _p(b), n, D, ctypes.c_float(voxel), _p(coords), _p(p2r), _p(first),
                            ctypes.byref(n_out), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    N = n_out.value
    return coords[:N].copy(), p2r[:n].copy(), first[:N].copy()


def create(coords, tensor_stride=None):
    """Unique coordinate set from integer rows (Eq. 1), first occurrence wins."""
    c = _c(coords, np.int32)
    n, Dp1 = c.shape
    D = Dp1 - 1
    ts = None if tensor_stride is None else _c(tensor_stride, np.int32)
    out = np.zeros((max(n, 1), Dp1), np.int32)
    inv = np.zeros(max(n, 1), np.int32)
    n_out, err = ctypes.c_int64(), ctypes.c_int64()
    st = lib().orc_create(_p(c), n, D, _p(ts), _p(out), _p(inv), ctypes.byref(n_out), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return out[:n_out.value].copy(), inv[:n].copy()


def stride(coords, conv_stride, tensor_stride=None):
    """Strided output coordinates (reading R11): floor_div(u, s_in*sigma)*(s_in*sigma)."""
    c = _c(coords, np.int32)
    n, Dp1 = c.shape
    D = Dp1 - 1
    ts = _c(tensor_stride if tensor_stride is not None else [1] * D, np.int32)
    cs = _c(conv_stride, np.int32)
    out = np.zeros((max(n, 1), Dp1), np.int32)
    n_out, err = ctypes.c_int64(), ctypes.c_int64()
    st = lib().orc_stride(_p(c), n, D, _p(ts), _p(cs), _p(out), ctypes.byref(n_out), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return out[:n_out.value].copy()


def region(kind: int, D: int, size=None, dilation=None, temporal_axis: int = -1, custom=None):
    """Kernel offset set N^D as int32[K][D]."""
    sz = None if size is None else _c(size if np.ndim(size) else [size] * D, np.int32)
    dl = None if dilation is None else _c(dilation if np.ndim(dilation) else [dilation] * D, np.int32)
    cu = None if custom is None else _c(custom, np.int32).reshape(-1, D)
    ncu = 0 if cu is None else cu.shape[0]
    K = ctypes.c_int32()
    st = lib().orc_region(kind, D, _p(sz), _p(dl), temporal_axis, _p(cu), ncu, None, ctypes.byref(K))
    if st:
        raise OracleError(st)
    offs = np.zeros((K.value, D), np.int32)
    lib().orc_region(kind, D, _p(sz), _p(dl), temporal_axis, _p(cu), ncu, _p(offs), ctypes.byref(K))
    return offs


def expand(coords, offsets, scale=None):
    """f4: output coordinates of a generative transposed conv, {u + i * scale}."""
    c = _c(coords, np.int32)
    offs = _c(offsets, np.int32)
    n, Dp1 = c.shape
    D = Dp1 - 1
    K = offs.shape[0]
    sc = None if scale is None else _c(scale, np.int32)
    out = np.zeros((max(n * K, 1), Dp1), np.int32)
    n_out, err = ctypes.c_int64(), ctypes.c_int64()
    st = lib().orc_expand(_p(c), n, D, _p(offs), K, _p(sc), _p(out), ctypes.byref(n_out), ctypes.byref(err))
    if st:
        raise OracleError(st, err.value)
    return out[:n_out.value].copy()


def labels(point_to_row, point_labels, n_rows: int, ignore_label: int = -1):
    """O1': per-voxel label, the points' common label or IGNORE_LABEL."""
    p2r = _c(point_to_row, np.int32)
    lab = _c(point_labels, np.int32)
    out = np.zeros(max(n_rows, 1), np.int32)
    st = lib().orc_labels(_p(p2r), _p(lab), p2r.shape[0], n_rows, ignore_label, _p(out))
    if st:
        raise OracleError(st)
    return out[:n_rows].copy()


def lookup(coords, queries):
    c = _c(coords, np.int32)
    q = _c(queries, np.int32)
    rows = np.zeros(max(q.shape[0], 1), np.int32)
    st = lib().orc_lookup(_p(c), c.shape[0], c.shape[1] - 1, _p(q), q.shape[0], _p(rows))
    if st:
        raise OracleError(st)
    return rows[:q.shape[0]].copy()


def kmap(c_in, c_out, offsets, scale=None, transposed: bool = False):
    """Kernel map M = {(I_i, O_i)} (Eq. 3) as CSR (ptr[K+1], in[|M|], out[|M|])."""
    ci = _c(c_in, np.int32)
    co = _c(c_out, np.int32)
    offs = _c(offsets, np.int32)
    K, D = offs.shape
    sc = _c(scale if scale is not None else [1] * D, np.int32)
    ptr = np.zeros(K + 1, np.int64)
    L = lib()
    st = L.orc_kmap(_p(ci), ci.shape[0], _p(co), co.shape[0], D, _p(offs), K, _p(sc), int(transposed),
                    _p(ptr), None, None)
    if st:
        raise OracleError(st)
    M = int(ptr[-1])
    ins = np.zeros(max(M, 1), np.int32)
    outs = np.zeros(max(M, 1), np.int32)
    L.orc_kmap(_p(ci), ci.shape[0], _p(co), co.shape[0], D, _p(offs), K, _p(sc), int(transposed),
               _p(ptr), _p(ins), _p(outs))
    return ptr, ins[:M].copy(), outs[:M].copy()


def kmap_reverse(kmap_csr, n_in: int | None = None):
    """The map with input and output roles exchanged, output-ascending per offset."""
    ptr, ins, outs = (np.ascontiguousarray(a) for a in kmap_csr)
    ptr = _c(ptr, np.int64)
    ins, outs = _c(ins, np.int32), _c(outs, np.int32)
    K = ptr.shape[0] - 1
    M = max(int(ptr[-1]), 1)
    rptr = np.zeros(K + 1, np.int64)
    rin = np.zeros(M, np.int32)
    rout = np.zeros(M, np.int32)
    lib().orc_kmap_reverse(_p(ptr), _p(ins), _p(outs), K, _p(rptr), _p(rin), _p(rout))
    return rptr, rin[:int(ptr[-1])].copy(), rout[:int(ptr[-1])].copy()


def conv_forward(kmap_csr, f_in, W, n_out: int):
    """Alg. 2 in fp64: F_out[o] += W_k F_in[a] for every pair (a, o) of offset k."""
    ptr, ins, outs = kmap_csr
    x = _c(f_in, np.float64)
    w = _c(W, np.float64)
    K, c_out, c_in = w.shape
    y = np.zeros((n_out, c_out), np.float64)
    lib().orc_conv_forward(_p(ptr), _p(ins), _p(outs), K, _p(x), c_in, _p(w), _p(y), n_out, c_out)
    return y


def conv_forward_rows(kmap_csr, f_in, W, rows):
    """Eq. 3 evaluated only at the selected output rows (fp64)."""
    ptr, ins, outs = kmap_csr
    x = _c(f_in, np.float64)
    w = _c(W, np.float64)
    K, c_out, c_in = w.shape
    r = _c(rows, np.int32)
    y = np.zeros((r.shape[0], c_out), np.float64)
    lib().orc_conv_forward_rows(_p(ptr), _p(ins), _p(outs), K, _p(x), c_in, _p(w), c_out, _p(r), r.shape[0], _p(y))
    return y


def conv_dgrad(kmap_csr, g_out, W, n_in: int):
    """Input gradient G_in[a] += W_k^T G_out[o] (reverse mode of Alg. 2), fp64."""
    ptr, ins, outs = kmap_csr
    g = _c(g_out, np.float64)
    w = _c(W, np.float64)
    K, c_out, c_in = w.shape
    gi = np.zeros((n_in, c_in), np.float64)
    lib().orc_conv_dgrad(_p(ptr), _p(ins), _p(outs), K, _p(g), c_out, _p(w), _p(gi), n_in, c_in)
    return gi


def conv_wgrad(kmap_csr, g_out, f_in, K: int):
    """Weight gradient dW_k = sum over pairs of offset k of G_out[o] F_in[a]^T, fp64."""
    ptr, ins, outs = kmap_csr
    g = _c(g_out, np.float64)
    x = _c(f_in, np.float64)
    c_out, c_in = g.shape[1], x.shape[1]
    dW = np.zeros((K, c_out, c_in), np.float64)
    lib().orc_conv_wgrad(_p(ptr), _p(ins), _p(outs), K, _p(g), c_out, _p(x), c_in, _p(dW))
    return dW


POOL_MAX, POOL_AVG, POOL_SUM = 0, 1, 2


def pool_forward(kmap_csr, f_in, n_out: int, mode: int):
    """f2: max (Alg. 3) / average / sum (Alg. 4) pooling over a kernel map, fp64.
    Returns (f_out [n_out][C], argmax [n_out][C] int32 for max, else None)."""
    ptr, ins, outs = kmap_csr
    x = _c(f_in, np.float64)
    C = x.shape[1]
    y = np.zeros((max(n_out, 1), C), np.float64)
    am = np.zeros((max(n_out, 1), C), np.int32) if mode == POOL_MAX else None
    lib().orc_pool_forward(_p(ptr), _p(ins), _p(outs), len(ptr) - 1, _p(x), C, n_out, mode, _p(y), _p(am))
    return y[:n_out].copy(), (am[:n_out].copy() if am is not None else None)


def pool_backward(kmap_csr, g_out, n_in: int, mode: int, argmax=None):
    ptr, ins, outs = kmap_csr
    g = _c(g_out, np.float64)
    C = g.shape[1]
    am = _c(argmax, np.int32) if argmax is not None else None
    gi = np.zeros((max(n_in, 1), C), np.float64)
    lib().orc_pool_backward(_p(ptr), _p(ins), _p(outs), len(ptr) - 1, _p(g), C, g.shape[0], mode, _p(am), _p(gi),
                            n_in)
    return gi[:n_in].copy()


def global_pool(batch, f_in, n_batch: int, mode: int):
    """Global pooling: one row per batch index, sum or average of its rows."""
    b = _c(batch, np.int32)
    x = _c(f_in, np.float64)
    y = np.zeros((max(n_batch, 1), x.shape[1]), np.float64)
    lib().orc_global_pool(_p(b), b.shape[0], _p(x), x.shape[1], n_batch, mode, _p(y))
    return y[:n_batch].copy()


def crf_infer(kmap_csr, phi_u, W, n_iters: int):
    """f3 (Alg. 5): mean-field TS-CRF inference over a (7D) kernel map, fp64."""
    ptr, ins, outs = kmap_csr
    phi = _c(phi_u, np.float64)
    w = _c(W, np.float64)
    n, C = phi.shape
    q = np.zeros((max(n, 1), C), np.float64)
    lib().orc_crf_infer(_p(ptr), _p(ins), _p(outs), len(ptr) - 1, _p(phi), n, C, _p(w), n_iters, _p(q))
    return q[:n].copy()


def epilogue(y, scale=None, shift=None, residual=None, relu: bool = False):
    """f4 block epilogue (ReLU and 1D batch normalisation act on the rows of F;
    P:303-306: residual blocks), reading R26: act(y * scale + shift + residual) per row,
    BatchNorm in its folded inference form, act = max(0, .) or identity.  fp64."""
    z = np.asarray(y, np.float64).copy()
    if scale is not None:
        z = z * np.asarray(scale, np.float64)[None, :]
    if shift is not None:
        z = z + np.asarray(shift, np.float64)[None, :]
    if residual is not None:
        z = z + np.asarray(residual, np.float64)
    return np.maximum(z, 0.0) if relu else z


def conv_forward_fused(kmap_csr, f_in, W, n_out: int, scale=None, shift=None, residual=None, relu: bool = False):
    """Alg. 2 followed by the block epilogue (R26), fp64: epilogue(conv_forward(...))."""
    return epilogue(conv_forward(kmap_csr, f_in, W, n_out), scale, shift, residual, relu)


def bn_fold(gamma, beta, mean, var, eps: float = 1e-5):
    """Inference BatchNorm as a per-channel affine map: y = gamma (x - mean) /
    sqrt(var + eps) + beta = x * scale + shift."""
    g, b, m, v = (np.asarray(a, np.float64) for a in (gamma, beta, mean, var))
    scale = g / np.sqrt(v + eps)
    return scale, b - m * scale


def crf_backward(kmap_csr, phi_u, W, n_iters: int, grad_q):
    """f3 learning (Eq. 5), fp64: dL/dphi_u and dL/dphi_p of Q^N (Alg. 5 with
    Q^0 = softmax(phi_u), reading R25) given dL/dQ^N, by backpropagation through the
    n_iters mean-field steps: for n = N..1, dA^n = Q^n (g - <Q^n, g>) (softmax reverse),
    dphi_u += dA^n, dphi_p += wgrad(dA^n, Q^(n-1)), g <- dgrad(dA^n, phi_p); finally
    dphi_u += the softmax reverse of Q^0."""
    phi = np.asarray(phi_u, np.float64)
    w = np.asarray(W, np.float64)
    n, C = phi.shape
    K = w.shape[0]

    def softmax(a):
        e = np.exp(a - a.max(axis=1, keepdims=True))
        return e / e.sum(axis=1, keepdims=True)

    def softmax_rev(q, g):
        return q * (g - (q * g).sum(axis=1, keepdims=True))

    Q = [softmax(phi)]
    for _ in range(n_iters):
        Q.append(softmax(phi + conv_forward(kmap_csr, Q[-1], w, n)))
    g = np.asarray(grad_q, np.float64)
    gphi = np.zeros_like(phi)
    gW = np.zeros_like(w)
    for it in range(n_iters, 0, -1):
        dA = softmax_rev(Q[it], g)
        gphi += dA
        gW += conv_wgrad(kmap_csr, dA, Q[it - 1], K)
        g = conv_dgrad(kmap_csr, dA, w, n)
    gphi += softmax_rev(Q[0], g)
    return gphi, gW
