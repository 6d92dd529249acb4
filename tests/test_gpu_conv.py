"""GPU <-> fp64 oracle parity of the feature path: forward, dgrad, wgrad, transposed conv,
in fp32 mode (tolerance 1e-5) and bf16 mode (2e-2), at oracle-sized cases spanning many
128-row tiles with ragged tails, and on sampled rows at full BASELINE sizes."""
import numpy as np
import pytest
import torch

import synthetic
from gpu_util import BF16_TOL, FP32_TOL, assert_close, csr_np, to_np

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    return m


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def _sparse(mk, orc, seed, n, span, D=3, ts=1, nb=2):
    g = np.random.default_rng(seed)
    rows = np.concatenate([g.integers(-span, span, (n, D)) * ts, g.integers(0, nb, (n, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows, [ts] * D)
    return mk.coords_create(dev(oc), [ts] * D), oc


def _check_all(mk, orc, m, km_np, X, W, G, dt, tol, transposed=False, what=""):
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    # bf16 mode: inputs rounded RNE from the same fp32 samples; compared to the fp64 oracle
    # on the ORIGINAL fp32 values (DESIGN.md §3 R21).
    Xd, Wd, Gd = dev(X).to(tdt), dev(W).to(tdt), dev(G).to(tdt)
    fwd = mk.conv_transpose_forward if transposed else mk.conv_forward
    bwd = mk.conv_transpose_backward if transposed else mk.conv_backward
    K, c_out, c_in = W.shape
    y = fwd(m, Xd, Wd, out_dtype=torch.float32)
    y64 = orc.conv_forward(km_np, X, W, m.n_out)
    assert_close(to_np(y), y64, orc.conv_forward(km_np, np.abs(X), np.abs(W), m.n_out), tol, what + " fwd")
    gin, gw = bwd(m, Gd, Xd, Wd)
    gin64 = orc.conv_dgrad(km_np, G, W, m.n_in)
    assert_close(to_np(gin), gin64, orc.conv_dgrad(km_np, np.abs(G), np.abs(W), m.n_in), tol, what + " dgrad")
    gw64 = orc.conv_wgrad(km_np, G, X, K)
    assert_close(to_np(gw), gw64, orc.conv_wgrad(km_np, np.abs(G), np.abs(X), K), tol, what + " wgrad")
    # determinism: bit-identical on repeat (fixed reduction order)
    y2 = fwd(m, Xd, Wd, out_dtype=torch.float32)
    gin2, gw2 = bwd(m, Gd, Xd, Wd)
    assert torch.equal(y, y2) and torch.equal(gin, gin2) and torch.equal(gw, gw2)


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("cin,cout,n,span", [(16, 16, 2000, 16), (64, 64, 20000, 30), (32, 64, 9000, 20),
                                             (96, 96, 5000, 15), (16, 32, 333, 6)])
def test_submanifold_conv(mk, orc, dt, tol, cin, cout, n, span):
    c, oc = _sparse(mk, orc, cin + n, n, span)
    r = mk.Region(mk.HYPERCUBE, 3, 3)
    m = mk.kmap_build(c, c, r)
    km = csr_np(m)
    g = np.random.default_rng(n)
    X = synthetic.features(1, c.n, cin)
    W = synthetic.weights(2, 27, cout, cin)
    G = g.uniform(-1, 1, (c.n, cout)).astype(np.float32)
    _check_all(mk, orc, m, km, X, W, G, dt, tol, what=f"{dt} {cin}->{cout}")


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_hybrid_4d_conv(mk, orc, dt, tol):
    c, oc = _sparse(mk, orc, 44, 12000, 14, D=4)
    m = mk.kmap_build(c, c, mk.Region(mk.HYBRID, 4, 3))
    km = csr_np(m)
    X = synthetic.features(3, c.n, 32)
    W = synthetic.weights(4, 29, 64, 32)
    G = synthetic.features(5, c.n, 64)
    _check_all(mk, orc, m, km, X, W, G, dt, tol, what="hybrid")


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("K", [2, 3])
def test_strided_conv_and_transpose(mk, orc, dt, tol, K):
    fine, ofine = _sparse(mk, orc, 70 + K, 15000, 24)
    coarse = mk.coords_stride(fine, [2, 2, 2])
    r = mk.Region(mk.HYPERCUBE, 3, K)
    m = mk.kmap_build(fine, coarse, r)
    km = csr_np(m)
    Kv = m.K
    cin, cout = 32, 48
    X = synthetic.features(6, fine.n, cin)
    W = synthetic.weights(7, Kv, cout, cin)
    G = synthetic.features(8, coarse.n, cout)
    _check_all(mk, orc, m, km, X, W, G, dt, tol, what=f"down K={K}")
    # transposed conv coarse -> fine
    mt = mk.kmap_build(coarse, fine, r, transposed=True)
    kmt = csr_np(mt)
    Y = synthetic.features(9, coarse.n, cout)
    WT = synthetic.weights(10, Kv, cin, cout)
    GT = synthetic.features(11, fine.n, cin)
    _check_all(mk, orc, mt, kmt, Y, WT, GT, dt, tol, transposed=True, what=f"up K={K}")


def test_adjoint_identity_fp32(mk, orc):
    # <conv_W x, y> = <x, convT_{W^T} y> holds for the GPU results to fp32 rounding.
    fine, _ = _sparse(mk, orc, 5, 20000, 25)
    coarse = mk.coords_stride(fine, [2, 2, 2])
    r = mk.Region(mk.HYPERCUBE, 3, 3)
    m = mk.kmap_build(fine, coarse, r)
    mt = mk.kmap_build(coarse, fine, r, transposed=True)
    X = dev(synthetic.features(1, fine.n, 32))
    W = dev(synthetic.weights(2, 27, 16, 32))
    Y = dev(synthetic.features(3, coarse.n, 16))
    lhs = (mk.conv_forward(m, X, W).double() * Y.double()).sum().item()
    rhs = (X.double() * mk.conv_transpose_forward(mt, Y, W.transpose(1, 2).contiguous()).double()).sum().item()
    assert abs(lhs - rhs) <= 1e-5 * (abs(lhs) + 1e-6)


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_room_full_size_sampled(mk, orc, dt, tol):
    # BASELINE configs[1] at full size in the bench launch configuration; the oracle
    # evaluates Eq. 3 on sampled output rows (O6 row by row).
    pts = synthetic.room_points(2003)
    c, _, _ = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL)
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 3, 3))
    km = csr_np(m)
    X = synthetic.features(1, c.n, 64)
    W = synthetic.weights(2, 27, 64, 64)
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    y = to_np(mk.conv_forward(m, dev(X).to(tdt), dev(W).to(tdt), out_dtype=torch.float32))
    rows = np.random.default_rng(0).choice(c.n, 2000, replace=False).astype(np.int32)
    rows = np.concatenate([rows, [0, c.n - 1]]).astype(np.int32)
    y64 = orc.conv_forward_rows(km, X, W, rows)
    s64 = orc.conv_forward_rows(km, np.abs(X), np.abs(W), rows)
    assert_close(y[rows], y64, s64, tol, f"room {dt}")


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_tesseract_4d_conv(mk, orc, dt, tol):
    # K = 3^4 = 81 offsets (the 4D hypercube of P:253): exercises the K > 32 kernel-map path
    # (k-major table, identity row order, exact pair lists) and the conv kernels' multi-word
    # offset masks.
    c, oc = _sparse(mk, orc, 81, 6000, 7, D=4)
    m = mk.kmap_build(c, c, mk.Region(mk.HYPERCUBE, 4, 3))
    assert m.K == 81
    km = csr_np(m)
    optr, oin, oout = orc.kmap(oc, oc, mk.region_offsets(mk.Region(mk.HYPERCUBE, 4, 3)))
    assert np.array_equal(km[0], optr) and np.array_equal(km[1], oin) and np.array_equal(km[2], oout)
    X = synthetic.features(12, c.n, 16)
    W = synthetic.weights(13, 81, 32, 16)
    G = synthetic.features(14, c.n, 32)
    _check_all(mk, orc, m, km, X, W, G, dt, tol, what="tesseract")
