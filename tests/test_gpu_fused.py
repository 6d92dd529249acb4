"""GPU <-> fp64 oracle parity of the fused block epilogue (f4, reading R26):
mk_conv_forward_fused = act(conv * scale + shift + residual) in the conv kernels' epilogue,
fp32 (FFMA) and bf16 (tcgen05) inputs, fp32 and bf16 outputs, on a submanifold map, on a
map between different coordinate sets (rows without pairs: act(shift + residual)) and on a
transposed map; plus a two-conv residual block chained on the GPU."""
import numpy as np
import pytest
import torch

import synthetic
from gpu_util import BF16_TOL, FP32_TOL, assert_close, to_np
from parity import Spec, map_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    return m


def dev(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def _coords(mk, orc, seed, n, span, D=3, ts=1):
    g = np.random.default_rng(seed)
    rows = np.concatenate([g.integers(-span, span, (n, D)) * ts, g.integers(0, 2, (n, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows, [ts] * D)
    c = mk.coords_create(dev(rows), [ts] * D)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    return c, oc


def _epi_params(seed, c_out, n_out):
    g = np.random.default_rng(seed)
    gamma, beta = g.uniform(0.5, 1.5, c_out), g.uniform(-0.5, 0.5, c_out)
    mean, var = g.uniform(-0.2, 0.2, c_out), g.uniform(0.5, 2.0, c_out)
    return gamma, beta, mean, var, g.uniform(-1, 1, (n_out, c_out)).astype(np.float32)


def _check(mk, orc, m, km, X, W, dt, out_dt, tol, opts, seed, transposed=False):
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    odt = torch.float32 if out_dt == "f32" else torch.bfloat16
    K, c_out, c_in = W.shape
    gamma, beta, mean, var, R = _epi_params(seed, c_out, m.n_out)
    scale, shift = orc.bn_fold(gamma, beta, mean, var)
    kw = {}
    if "bn" in opts:
        kw["scale"], kw["shift"] = dev(scale.astype(np.float32)), dev(shift.astype(np.float32))
    if "res" in opts:
        kw["residual"] = dev(R).to(odt)
    relu = "relu" in opts
    y = mk.conv_forward(m, dev(X).to(tdt), dev(W).to(tdt), out_dtype=odt, relu=relu, **kw)
    # the oracle sees the fp32-folded scale / shift and the residual as the GPU stores it
    sc = scale.astype(np.float32).astype(np.float64) if "bn" in opts else None
    sh = shift.astype(np.float32).astype(np.float64) if "bn" in opts else None
    res = to_np(kw["residual"]).astype(np.float64) if "res" in opts else None
    y64 = orc.conv_forward_fused(km, X, W, m.n_out, sc, sh, res, relu)
    # error scale: the epilogue of the conv of absolute values (act is 1-Lipschitz)
    s64 = orc.epilogue(orc.conv_forward(km, np.abs(X), np.abs(W), m.n_out), None if sc is None else np.abs(sc),
                       None if sh is None else np.abs(sh), None if res is None else np.abs(res))
    if out_dt == "bf16":  # bf16 output: the rounding (2^-9 of the value) sets the tolerance
        s64 = s64 + np.abs(y64)
        tol = max(tol, BF16_TOL)
    assert_close(to_np(y), y64, s64, tol, f"fused {dt}->{out_dt} {opts}")
    if relu:
        assert (to_np(y) >= 0).all()
    y2 = mk.conv_forward(m, dev(X).to(tdt), dev(W).to(tdt), out_dtype=odt, relu=relu, **kw)
    assert torch.equal(y, y2)  # deterministic


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
@pytest.mark.parametrize("opts", [("bn", "res", "relu"), ("relu",), ("bn",), ("res",)])
def test_fused_submanifold(mk, orc, dt, tol, out_dt, opts):
    c, oc = _coords(mk, orc, 5, 9000, 20)
    m, km = map_pair(mk, orc, c, c, oc, oc, Spec(0, 3, 3), [1] * 3)
    X = synthetic.features(11, c.n, 32)
    W = synthetic.weights(12, 27, 64, 32)
    _check(mk, orc, m, km, X, W, dt, out_dt, tol, opts, 13)


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_fused_rows_without_pairs(mk, orc, dt, tol):
    cin, ocin = _coords(mk, orc, 21, 3000, 25)
    cout, ocout = _coords(mk, orc, 22, 2500, 25)  # a different set: many output rows have no pair
    m, km = map_pair(mk, orc, cin, cout, ocin, ocout, Spec(0, 3, 3), [1] * 3)
    assert m.n_pairs > 0
    X = synthetic.features(23, cin.n, 16)
    W = synthetic.weights(24, 27, 48, 16)
    _check(mk, orc, m, km, X, W, dt, "f32", tol, ("bn", "res", "relu"), 25)


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_fused_transposed(mk, orc, dt, tol):
    c, oc = _coords(mk, orc, 31, 8000, 24)
    cs = mk.coords_stride(c, [2, 2, 2])
    ocs = orc.stride(oc, [2, 2, 2])
    m, km = map_pair(mk, orc, cs, c, ocs, oc, Spec(0, 3, 2), [1] * 3, transposed=True)
    X = synthetic.features(32, cs.n, 64)
    W = synthetic.weights(33, 8, 32, 64)
    _check(mk, orc, m, km, X, W, dt, "f32", tol, ("bn", "relu"), 34)


def test_residual_block_chain_fp32(mk, orc):
    """MinkowskiNet basic block: relu(bn2(conv2(relu(bn1(conv1 x)))) + x), both
    convs with fused epilogues, against the oracle chain in fp64."""
    c, oc = _coords(mk, orc, 41, 12000, 22)
    m, km = map_pair(mk, orc, c, c, oc, oc, Spec(0, 3, 3), [1] * 3)
    C = 32
    X = synthetic.features(42, c.n, C)
    W1, W2 = synthetic.weights(43, 27, C, C), synthetic.weights(44, 27, C, C)
    p1, p2 = _epi_params(45, C, 1)[:4], _epi_params(46, C, 1)[:4]
    s1, b1 = orc.bn_fold(*p1)
    s2, b2 = orc.bn_fold(*p2)
    f32 = lambda a: dev(np.asarray(a, np.float32))  # noqa: E731
    h = mk.conv_forward(m, dev(X), dev(W1), scale=f32(s1), shift=f32(b1), relu=True)
    y = mk.conv_forward(m, h, dev(W2), scale=f32(s2), shift=f32(b2), residual=dev(X), relu=True)
    s1, b1, s2, b2 = (np.asarray(a, np.float32).astype(np.float64) for a in (s1, b1, s2, b2))
    h64 = orc.conv_forward_fused(km, X, W1, c.n, s1, b1, None, True)
    y64 = orc.conv_forward_fused(km, h64, W2, c.n, s2, b2, X, True)
    err = np.abs(to_np(y) - y64).max() / np.abs(y64).max()
    assert err <= 1e-5, err
