"""GPU <-> fp64 oracle parity of pooling over kernel maps (Alg. 3/4):
max values and argmax bit-exact, average / sum within the fp32 tolerance, reverse modes,
for strided (2^3 and 3^3 onto the stride-2 set), submanifold and transposed (unpooling) maps,
fp32 and bf16 features."""
import numpy as np
import pytest
import torch

from gpu_util import FP32_TOL, assert_close
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


def _sets(mk, orc, seed, n=20000, span=30):
    g = np.random.default_rng(seed)
    rows = np.concatenate([g.integers(-span, span, (n, 3)), g.integers(0, 2, (n, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows)
    fine = mk.coords_create(dev(rows))
    assert np.array_equal(fine.export().cpu().numpy(), oc)
    coarse = mk.coords_stride(fine, [2, 2, 2])
    return fine, coarse, oc, orc.stride(oc, [2, 2, 2])


@pytest.mark.parametrize("dt", ["f32", "bf16"])
@pytest.mark.parametrize("K,kind", [(2, "strided"), (3, "strided"), (3, "submanifold"), (2, "transposed")])
def test_pool_matches_oracle(mk, orc, dt, K, kind):
    fine, coarse, ofine, ocoarse = _sets(mk, orc, 10 * K + len(kind))
    spec = Spec(0, 3, K)
    if kind == "strided":
        m, km = map_pair(mk, orc, fine, coarse, ofine, ocoarse, spec, [1] * 3)
    elif kind == "submanifold":
        m, km = map_pair(mk, orc, fine, fine, ofine, ofine, spec, [1] * 3)
    else:  # unpooling: coarse -> fine on the transposed map ("transposed pooling")
        m, km = map_pair(mk, orc, coarse, fine, ocoarse, ofine, spec, [1] * 3, transposed=True)
    g = np.random.default_rng(K)
    C = 40
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    # values rounded to the feature dtype first, so the fp64 oracle sees the same inputs
    X = dev(g.standard_normal((m.n_in, C)).astype(np.float32)).to(tdt)
    G = dev(g.standard_normal((m.n_out, C)).astype(np.float32)).to(tdt)
    Xn, Gn = X.float().cpu().numpy(), G.float().cpu().numpy()
    y, am = mk.pool_forward(m, X, mk.POOL_MAX)
    y64, am64 = orc.pool_forward(km, Xn, m.n_out, 0)
    assert np.array_equal(y.float().cpu().numpy(), y64.astype(np.float32))  # max is exact
    assert np.array_equal(am.cpu().numpy(), am64)
    gi = mk.pool_backward(m, G, mk.POOL_MAX, am)
    gi64 = orc.pool_backward(km, Gn, m.n_in, 0, am64)
    tol = FP32_TOL if dt == "f32" else 1e-2  # bf16 outputs: one RNE rounding of the result
    assert_close(gi.float().cpu().numpy(), gi64, orc.pool_backward(km, np.abs(Gn), m.n_in, 0, am64), tol, "max bwd")
    for mode in (1, 2):
        y, _ = mk.pool_forward(m, X, mode)
        y64, _ = orc.pool_forward(km, Xn, m.n_out, mode)
        s64, _ = orc.pool_forward(km, np.abs(Xn), m.n_out, mode)
        assert_close(y.float().cpu().numpy(), y64, s64, tol, f"mode {mode} fwd")
        gi = mk.pool_backward(m, G, mode)
        gi64 = orc.pool_backward(km, Gn, m.n_in, mode)
        si64 = orc.pool_backward(km, np.abs(Gn), m.n_in, mode)
        assert_close(gi.float().cpu().numpy(), gi64, si64, tol, f"mode {mode} bwd")
    # determinism
    y1, a1 = mk.pool_forward(m, X, mk.POOL_MAX)
    y2, a2 = mk.pool_forward(m, X, mk.POOL_MAX)
    assert torch.equal(y1, y2) and torch.equal(a1, a2)


@pytest.mark.parametrize("dt", ["f32", "bf16"])
def test_global_pool_matches_oracle(mk, orc, dt):
    # P:222 global pooling: one row per batch index (sum / mean), vs the oracle's group-by
    g = np.random.default_rng(21)
    n = 30000
    rows = np.concatenate([g.integers(-50, 50, (n, 3)), g.integers(0, 5, (n, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows)
    c = mk.coords_create(dev(oc))
    tdt = torch.float32 if dt == "f32" else torch.bfloat16
    X = dev(g.standard_normal((c.n, 48)).astype(np.float32)).to(tdt)
    Xn = X.float().cpu().numpy()
    tol = FP32_TOL if dt == "f32" else 1e-2
    for mode in (1, 2):
        y = mk.global_pool(c, X, 6, mode).float().cpu().numpy()  # batch 5 has no rows -> 0
        y64 = orc.global_pool(oc[:, 3], Xn, 6, mode)
        s64 = orc.global_pool(oc[:, 3], np.abs(Xn), 6, mode)
        assert_close(y, y64, s64, tol, f"global mode {mode}")
        assert np.all(y[5] == 0)
        y2 = mk.global_pool(c, X, 6, mode).float().cpu().numpy()
        assert np.array_equal(y, y2)  # deterministic
