"""GPU parity of the 7D space-time-chroma path: packed 7D coordinates
(byte-identical rows and lookups), the 7D hypercross kernel map (bit-exact CSR) and TS-CRF
mean-field inference (Alg. 5) against the fp64 oracle (fp32 tolerance)."""
import numpy as np
import pytest
import torch

from gpu_util import FP32_TOL, assert_close
from parity import Spec, map_pair

pytestmark = pytest.mark.gpu
D = 7


@pytest.fixture(scope="module")
def mk():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    return m


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _lattice7(seed, n=20000):
    # a colored 4D scan lifted to (x, y, z, r, g, b, t) (Alg. 5: C_crf = [C, F, T]): points on
    # a few planes, colour = patch colour + small noise (quantized), 3 frames
    g = np.random.default_rng(seed)
    xyz = g.integers(-60, 60, (n, 3))
    xyz[: n // 2, 2] = g.integers(-2, 2, n // 2)  # a floor
    rgb = (np.stack([xyz[:, 0] // 20, xyz[:, 1] // 20, xyz[:, 2] // 30], axis=1) * 3 + g.integers(-1, 2, (n, 3)))
    t = g.integers(0, 3, (n, 1))
    b = g.integers(0, 2, (n, 1))
    return np.concatenate([xyz, rgb, t, b], axis=1).astype(np.int32)


def test_coords7_create_lookup_and_ranges(mk, orc):
    rows = _lattice7(1)
    c, inv = mk.coords_create(dev(rows), return_inverse=True)
    oc, oinv = orc.create(rows)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    assert np.array_equal(inv.cpu().numpy(), oinv)
    q = np.concatenate([oc[:500], oc[:500] + np.array([0, 0, 0, 0, 0, 0, 7, 0], np.int32)])
    assert np.array_equal(c.lookup(dev(q)).cpu().numpy(), orc.lookup(oc, q))
    bad = rows[:10].copy()
    bad[3, 0] = 1 << 19  # axis 0 of a D = 7 key holds [-2^19, 2^19) (R19)
    with pytest.raises(mk.MkError) as e:
        mk.coords_create(dev(bad))
    assert e.value.name == "MK_ERR_COORD_RANGE" and e.value.row == 3


def test_kmap7_hypercross_matches_oracle(mk, orc):
    rows = _lattice7(2)
    oc, _ = orc.create(rows)
    c = mk.coords_create(dev(oc))
    m, _ = map_pair(mk, orc, c, c, oc, oc, Spec(1, D, 3), [1] * D, what="7D hypercross")
    assert m.K == 15


@pytest.mark.parametrize("C,n_iters", [(8, 3), (20, 1)])
def test_crf_infer_matches_oracle(mk, orc, C, n_iters):
    rows = _lattice7(3)
    oc, _ = orc.create(rows)
    c = mk.coords_create(dev(oc))
    m, km = map_pair(mk, orc, c, c, oc, oc, Spec(1, D, 3), [1] * D)
    g = np.random.default_rng(C)
    phi = g.standard_normal((c.n, C)).astype(np.float32)
    W = (g.standard_normal((15, C, C)) * 0.5).astype(np.float32)
    q = mk.crf_infer(m, dev(phi), dev(W), n_iters).cpu().numpy()
    q64 = orc.crf_infer(km, phi, W, n_iters)
    assert_close(q, q64, np.ones_like(q64), FP32_TOL, "crf")  # probabilities: absolute scale 1
    np.testing.assert_allclose(q.sum(axis=1), 1.0, rtol=1e-5)


# Eq. 5 learning: the fp32 tolerance of north_star, normwise (measured: <= 3.4e-6 for dW,
# <= 3.3e-7 for dphi_u at N = 3)
CRF_BWD_TOL = FP32_TOL


@pytest.mark.parametrize("C,n_iters", [(8, 3), (20, 1), (4, 0)])
def test_crf_backward_matches_oracle(mk, orc, C, n_iters):
    rows = _lattice7(5, n=12000)
    oc, _ = orc.create(rows)
    c = mk.coords_create(dev(oc))
    m, km = map_pair(mk, orc, c, c, oc, oc, Spec(1, D, 3), [1] * D)
    g = np.random.default_rng(100 + C)
    phi = g.standard_normal((c.n, C)).astype(np.float32)
    W = (g.standard_normal((15, C, C)) * 0.5).astype(np.float32)
    G = g.standard_normal((c.n, C)).astype(np.float32)
    gphi, gW = mk.crf_backward(m, dev(phi), dev(W), n_iters, dev(G))
    gphi64, gW64 = orc.crf_backward(km, phi, W, n_iters, G)
    e_phi = np.abs(gphi.cpu().numpy() - gphi64).max() / np.abs(gphi64).max()
    print(f"crf backward C={C} N={n_iters}: dphi normwise {e_phi:.2e}", end="")
    assert e_phi <= CRF_BWD_TOL
    if n_iters > 0:
        e_w = np.abs(gW.cpu().numpy() - gW64).max() / np.abs(gW64).max()
        print(f", dW normwise {e_w:.2e}")
        assert e_w <= CRF_BWD_TOL
    else:
        assert not gW.any()
    np.testing.assert_allclose(gphi.cpu().numpy().sum(axis=1), 0.0, atol=1e-5)  # logit shift invariance
    gphi2, gW2 = mk.crf_backward(m, dev(phi), dev(W), n_iters, dev(G))
    assert torch.equal(gphi, gphi2) and torch.equal(gW, gW2)  # deterministic
