"""Pins for the oracle's pooling (Alg. 3 / Alg. 4) against the
SPEC worked examples, the dense library routines (on a fully occupied grid a 2x2x2
stride-2 region IS torch max_pool3d / avg_pool3d), autograd, and the adjoint identity.
No GPU."""
import numpy as np
import pytest
import torch
import torch.nn.functional as F

from conftest import full_grid

MAX, AVG, SUM = 0, 1, 2


def _csr_one_output(values_per_offset):
    # one output row (0) fed by one input row per offset: input row k at offset k
    K = len(values_per_offset)
    ptr = np.arange(K + 1, dtype=np.int64)
    ins = np.arange(K, dtype=np.int32)
    outs = np.zeros(K, np.int32)
    return (ptr, ins, outs), np.array(values_per_offset, np.float64).reshape(K, 1)


def test_pool_worked_examples(orc):
    # S:229 inputs {1, 5, 3} mapping to one output, 1 channel -> max 5
    km, x = _csr_one_output([1.0, 5.0, 3.0])
    y, am = orc.pool_forward(km, x, 1, MAX)
    assert y.tolist() == [[5.0]] and am.tolist() == [[1]]
    # S:238 inputs {2, 4} -> avg 3, sum 6
    km, x = _csr_one_output([2.0, 4.0])
    assert orc.pool_forward(km, x, 1, AVG)[0].tolist() == [[3.0]]
    assert orc.pool_forward(km, x, 1, SUM)[0].tolist() == [[6.0]]
    # S:230 single input per output -> identity
    km, x = _csr_one_output([-7.5])
    for mode in (MAX, AVG, SUM):
        assert orc.pool_forward(km, x, 1, mode)[0].tolist() == [[-7.5]]
    # ties: the lowest concatenated index (offset order) wins
    km, x = _csr_one_output([2.0, 9.0, 9.0, 1.0])
    assert orc.pool_forward(km, x, 1, MAX)[1].tolist() == [[1]]


def _dense(rows, coords, G, C):
    d = torch.zeros(1, C, G, G, G, dtype=torch.float64)
    d[0][:, coords[:, 0], coords[:, 1], coords[:, 2]] = torch.from_numpy(rows.T)
    return d


@pytest.mark.parametrize("G,C", [(4, 3), (6, 5)])
def test_pool_equals_dense_pool3d(orc, G, C):
    # Fully occupied G^3 grid, K = 2 region {0,1}^3 (R3) from the fine set to its stride-2
    # set: max / average pooling = torch max_pool3d / avg_pool3d(kernel 2, stride 2); sum =
    # 8 x average.  Backward of max = autograd of max_pool3d (random values: no ties).
    g = np.random.default_rng(G)
    fine = full_grid(G, 3)
    coarse = orc.stride(fine, [2, 2, 2])
    km = orc.kmap(fine, coarse, orc.region(0, 3, [2, 2, 2]))
    X = g.standard_normal((fine.shape[0], C))
    xd = _dense(X, fine, G, C).requires_grad_(True)
    cc = coarse // 2
    ymax, am = orc.pool_forward(km, X, coarse.shape[0], MAX)
    yd = F.max_pool3d(xd, 2, 2)
    np.testing.assert_array_equal(ymax, yd[0].detach().numpy()[:, cc[:, 0], cc[:, 1], cc[:, 2]].T)
    yavg, _ = orc.pool_forward(km, X, coarse.shape[0], AVG)
    ya = F.avg_pool3d(xd.detach(), 2, 2)[0].numpy()[:, cc[:, 0], cc[:, 1], cc[:, 2]].T
    np.testing.assert_allclose(yavg, ya, rtol=1e-13, atol=1e-13)
    ysum, _ = orc.pool_forward(km, X, coarse.shape[0], SUM)
    np.testing.assert_allclose(ysum, 8 * ya, rtol=1e-13, atol=1e-13)
    Gout = g.standard_normal((coarse.shape[0], C))
    gd = torch.zeros_like(yd)
    gd[0][:, cc[:, 0], cc[:, 1], cc[:, 2]] = torch.from_numpy(Gout.T)
    (yd * gd).sum().backward()
    gin = orc.pool_backward(km, Gout, fine.shape[0], MAX, am)
    np.testing.assert_array_equal(gin, xd.grad[0].numpy()[:, fine[:, 0], fine[:, 1], fine[:, 2]].T)


@pytest.mark.parametrize("mode", [AVG, SUM])
def test_pool_adjoint_and_avg_identity(orc, mode):
    # sparse random set, 3x3x3 pooling onto its stride-2 set: <pool(x), g> = <x, pool^T(g)>
    # (linear modes), and avg = sum / counts elementwise
    g = np.random.default_rng(11 + mode)
    rows = np.concatenate([g.integers(-9, 9, (700, 3)), np.zeros((700, 1), np.int64)], axis=1).astype(np.int32)
    fine, _ = orc.create(rows)
    coarse = orc.stride(fine, [2, 2, 2])
    km = orc.kmap(fine, coarse, orc.region(0, 3, [3, 3, 3]))
    X = g.standard_normal((fine.shape[0], 4))
    Gout = g.standard_normal((coarse.shape[0], 4))
    y, _ = orc.pool_forward(km, X, coarse.shape[0], mode)
    gi = orc.pool_backward(km, Gout, fine.shape[0], mode)
    lhs, rhs = float((y * Gout).sum()), float((X * gi).sum())
    assert abs(lhs - rhs) <= 1e-12 * (abs(lhs) + 1.0)
    counts = np.bincount(km[2], minlength=coarse.shape[0]).astype(np.float64)
    ysum, _ = orc.pool_forward(km, X, coarse.shape[0], SUM)
    yavg, _ = orc.pool_forward(km, X, coarse.shape[0], AVG)
    np.testing.assert_allclose(yavg, ysum / counts[:, None], rtol=1e-14, atol=1e-14)


def test_global_pool(orc):
    g = np.random.default_rng(3)
    # single-row tensor -> that row (avg and sum)
    x = g.standard_normal((1, 5))
    for mode in (AVG, SUM):
        np.testing.assert_array_equal(orc.global_pool(np.zeros(1, np.int32), x, 1, mode), x)
    # numpy group-by reference
    b = g.integers(0, 4, 300).astype(np.int32)
    x = g.standard_normal((300, 6))
    ysum = orc.global_pool(b, x, 4, SUM)
    yavg = orc.global_pool(b, x, 4, AVG)
    for k in range(4):
        np.testing.assert_allclose(ysum[k], x[b == k].sum(0), rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(yavg[k], x[b == k].mean(0), rtol=1e-13, atol=1e-13)
