"""Pins for the oracle's feature operations (O6-O9) against textbook / library routines.

Eq. 2 special case: on a fully occupied grid with a hypercube region the
generalized sparse convolution IS the dense convolution, so torch.nn.functional.conv3d
(and its autograd, and conv_transpose3d) in fp64 on the CPU pin forward, dgrad, wgrad and
the transposed conv.  Adjoint identities pin the backward maps on random sparse sets.
No GPU."""
import itertools

import numpy as np
import pytest
import torch
import torch.nn.functional as F

from conftest import full_grid


def _dense_to_rows(dense, coords):
    # dense: [C][G][G][G] -> rows [n][C] at coords (x, y, z)
    return dense[:, coords[:, 0], coords[:, 1], coords[:, 2]].T


def _w_to_torch(W, offs, K):
    # W [Kvol][C_out][C_in] with offsets in [-(K-1)/2 ..] (odd) or [0..K-1] (even)
    Kv, co, ci = W.shape
    w = np.zeros((co, ci, K, K, K))
    base = (K - 1) // 2 if K % 2 == 1 else 0
    for k, (a, b, c) in enumerate(offs.tolist()):
        w[:, :, a + base, b + base, c + base] = W[k]
    return torch.from_numpy(w)


@pytest.mark.parametrize("G,cin,cout", [(5, 3, 4), (6, 8, 8)])
def test_forward_dgrad_wgrad_equal_dense_conv3d(orc, G, cin, cout):
    g = np.random.default_rng(G)
    c = full_grid(G, 3)
    offs = orc.region(0, 3, [3, 3, 3])
    km = orc.kmap(c, c, offs)
    X = g.standard_normal((c.shape[0], cin))
    W = g.standard_normal((27, cout, cin))
    Gout = g.standard_normal((c.shape[0], cout))
    y = orc.conv_forward(km, X, W, c.shape[0])
    xd = torch.zeros(1, cin, G, G, G, dtype=torch.float64)
    xd[0][:, c[:, 0], c[:, 1], c[:, 2]] = torch.from_numpy(X.T)
    xd.requires_grad_(True)
    wt = _w_to_torch(W, offs, 3).requires_grad_(True)
    yd = F.conv3d(xd, wt, padding=1)
    np.testing.assert_allclose(y, _dense_to_rows(yd[0].detach().numpy(), c), rtol=1e-12, atol=1e-12)
    gd = torch.zeros_like(yd)
    gd[0][:, c[:, 0], c[:, 1], c[:, 2]] = torch.from_numpy(Gout.T)
    (yd * gd).sum().backward()
    gin = orc.conv_dgrad(km, Gout, W, c.shape[0])
    np.testing.assert_allclose(gin, _dense_to_rows(xd.grad[0].numpy(), c), rtol=1e-12, atol=1e-12)
    dW = orc.conv_wgrad(km, Gout, X, 27)
    for k, (a, b, cc) in enumerate(offs.tolist()):
        np.testing.assert_allclose(dW[k], wt.grad[:, :, a + 1, b + 1, cc + 1].numpy(), rtol=1e-12, atol=1e-12)


def test_strided_k3_equals_conv3d_stride2(orc):
    G, cin, cout = 6, 4, 5
    g = np.random.default_rng(1)
    fine = full_grid(G, 3)
    coarse = orc.stride(fine, [2, 2, 2])
    offs = orc.region(0, 3, [3, 3, 3])
    km = orc.kmap(fine, coarse, offs)
    X = g.standard_normal((fine.shape[0], cin))
    W = g.standard_normal((27, cout, cin))
    y = orc.conv_forward(km, X, W, coarse.shape[0])
    xd = torch.zeros(1, cin, G, G, G, dtype=torch.float64)
    xd[0][:, fine[:, 0], fine[:, 1], fine[:, 2]] = torch.from_numpy(X.T)
    yd = F.conv3d(xd, _w_to_torch(W, offs, 3), stride=2, padding=1)[0].numpy()
    np.testing.assert_allclose(y, _dense_to_rows(yd, coarse // 2), rtol=1e-12, atol=1e-12)


def test_k2_stride2_and_transpose_equal_conv3d(orc):
    G, cin, cout = 6, 3, 4
    g = np.random.default_rng(2)
    fine = full_grid(G, 3)
    coarse = orc.stride(fine, [2, 2, 2])
    offs = orc.region(0, 3, [2, 2, 2])
    km = orc.kmap(fine, coarse, offs)
    X = g.standard_normal((fine.shape[0], cin))
    W = g.standard_normal((8, cout, cin))
    y = orc.conv_forward(km, X, W, coarse.shape[0])
    xd = torch.zeros(1, cin, G, G, G, dtype=torch.float64)
    xd[0][:, fine[:, 0], fine[:, 1], fine[:, 2]] = torch.from_numpy(X.T)
    wt = _w_to_torch(W, offs, 2)
    yd = F.conv3d(xd, wt, stride=2)[0].numpy()
    np.testing.assert_allclose(y, _dense_to_rows(yd, coarse // 2), rtol=1e-12, atol=1e-12)
    # transposed conv: coarse -> fine with W'_k = W_k^T equals conv_transpose3d
    kmT = orc.kmap(coarse, fine, offs, transposed=True)
    Y = g.standard_normal((coarse.shape[0], cout))
    WT = np.transpose(W, (0, 2, 1)).copy()
    z = orc.conv_forward(kmT, Y, WT, fine.shape[0])
    yd2 = torch.zeros(1, cout, G // 2, G // 2, G // 2, dtype=torch.float64)
    cc = coarse // 2
    yd2[0][:, cc[:, 0], cc[:, 1], cc[:, 2]] = torch.from_numpy(Y.T)
    zd = F.conv_transpose3d(yd2, wt, stride=2)[0].numpy()
    np.testing.assert_allclose(z, _dense_to_rows(zd, fine), rtol=1e-12, atol=1e-12)


def test_hybrid_4d_equals_dense_shift_and_add(orc):
    # 4D grid, hybrid region (reading R4): dense zero-padded shift-and-add (numpy) per offset.
    G, cin, cout = 4, 3, 2
    g = np.random.default_rng(3)
    c = full_grid(G, 4)
    offs = orc.region(2, 4, [3, 3, 3, 3])
    km = orc.kmap(c, c, offs)
    X = g.standard_normal((c.shape[0], cin))
    W = g.standard_normal((offs.shape[0], cout, cin))
    y = orc.conv_forward(km, X, W, c.shape[0])
    dense = np.zeros((G + 2,) * 4 + (cin,))
    dense[tuple((c[:, d] + 1) for d in range(4))] = X
    want = np.zeros((c.shape[0], cout))
    for k, off in enumerate(offs.tolist()):
        src = dense[tuple((c[:, d] + 1 + off[d]) for d in range(4))]
        want += src @ W[k].T
    np.testing.assert_allclose(y, want, rtol=1e-12, atol=1e-12)


def test_k1_is_matmul_and_identity(orc):
    g = np.random.default_rng(4)
    c, _ = orc.create(np.concatenate([g.integers(-9, 9, (100, 3)), np.zeros((100, 1), int)], axis=1))
    X = g.standard_normal((c.shape[0], 6))
    W = g.standard_normal((1, 5, 6))
    km = orc.kmap(c, c, orc.region(0, 3, [1, 1, 1]))
    np.testing.assert_allclose(orc.conv_forward(km, X, W, c.shape[0]), X @ W[0].T, rtol=1e-12, atol=1e-13)
    I = np.eye(6)[None]
    np.testing.assert_array_equal(orc.conv_forward(km, X, I, c.shape[0]), X)


def _random_sparse(orc, g, n, span, ts=1, D=3):
    c = np.concatenate([g.integers(-span, span, (n, D)) * ts, g.integers(0, 2, (n, 1))], axis=1)
    return orc.create(c.astype(np.int32), tensor_stride=[ts] * D)[0]


def test_adjoint_identities(orc):
    # <conv_W x, g> = <x, dgrad_W g> = <W, wgrad(x, g)>  (1e-10 in fp64)
    g = np.random.default_rng(5)
    c_in = _random_sparse(orc, g, 400, 5)
    c_out = orc.stride(c_in, [2, 2, 2])
    offs = orc.region(0, 3, [3, 3, 3])
    km = orc.kmap(c_in, c_out, offs)
    X = g.standard_normal((c_in.shape[0], 7))
    W = g.standard_normal((27, 5, 7))
    Gr = g.standard_normal((c_out.shape[0], 5))
    lhs = float(np.sum(orc.conv_forward(km, X, W, c_out.shape[0]) * Gr))
    mid = float(np.sum(X * orc.conv_dgrad(km, Gr, W, c_in.shape[0])))
    rhs = float(np.sum(W * orc.conv_wgrad(km, Gr, X, 27)))
    assert abs(lhs - mid) <= 1e-10 * abs(lhs) and abs(lhs - rhs) <= 1e-10 * abs(lhs)
    # convT adjoint: <conv_W x, y> = <x, convT_{W^T} y>  (BASELINE north_star)
    kmT = orc.kmap(c_out, c_in, offs, scale=[1, 1, 1], transposed=True)
    WT = np.transpose(W, (0, 2, 1)).copy()
    rhsT = float(np.sum(X * orc.conv_forward(kmT, Gr, WT, c_in.shape[0])))
    assert abs(lhs - rhsT) <= 1e-10 * abs(lhs)
    # zero gradient -> zero gradients
    assert not orc.conv_dgrad(km, np.zeros_like(Gr), W, c_in.shape[0]).any()
    assert not orc.conv_wgrad(km, np.zeros_like(Gr), X, 27).any()


def test_forward_rows_and_equivariance(orc):
    g = np.random.default_rng(6)
    c = _random_sparse(orc, g, 500, 6)
    offs = orc.region(0, 3, [3, 3, 3])
    km = orc.kmap(c, c, offs)
    X = g.standard_normal((c.shape[0], 4))
    W = g.standard_normal((27, 3, 4))
    y = orc.conv_forward(km, X, W, c.shape[0])
    rows = np.array([0, 5, c.shape[0] - 1, 17], np.int32)
    np.testing.assert_allclose(orc.conv_forward_rows(km, X, W, rows), y[rows], rtol=1e-13, atol=1e-13)
    # translation equivariance at stride 1
    ct = c.copy()
    ct[:, :3] += np.array([7, -3, 11], np.int32)
    yt = orc.conv_forward(orc.kmap(ct, ct, offs), X, W, c.shape[0])
    np.testing.assert_allclose(yt, y, rtol=1e-13, atol=1e-13)
    # row-permutation equivariance
    perm = g.permutation(c.shape[0])
    yp = orc.conv_forward(orc.kmap(c[perm], c[perm], offs), X[perm], W, c.shape[0])
    np.testing.assert_allclose(yp, y[perm], rtol=1e-13, atol=1e-13)
    # linearity
    X2 = g.standard_normal(X.shape)
    np.testing.assert_allclose(orc.conv_forward(km, 2 * X - 3 * X2, W, c.shape[0]),
                               2 * y - 3 * orc.conv_forward(km, X2, W, c.shape[0]), rtol=1e-11, atol=1e-11)


# ---------------------------------------------------------------- tensor stride > 1 (R14)
# "stride size of the input sparse tensor": a sparse tensor of tensor stride s has
# coordinates on the lattice sZ^D, and its neighbours at offset i are u + i*s.  A fully
# occupied stride-2 lattice is therefore the dense grid with every index doubled (P:159's
# dense special case on the compacted grid), so F.conv3d on the compacted grid pins the
# offset scaling of orc_kmap: a dropped scale (u + i) finds no neighbour on 2Z^3, a doubled
# one (u + 4i) skips the nearest ones — both change every output.
def _stride2_grid(G, base=-4):
    c = full_grid(G, 3)
    c[:, :3] = 2 * c[:, :3] + base  # the lattice 2Z^3 shifted to negative coordinates
    return c


def _compact(c, base=-4, s=2):
    return (c[:, :3] - base) // s


@pytest.mark.parametrize("G,cin,cout", [(5, 3, 4), (4, 5, 2)])
def test_tensor_stride2_submanifold_equals_conv3d(orc, G, cin, cout):
    g = np.random.default_rng(40 + G)
    c, _ = orc.create(_stride2_grid(G), tensor_stride=[2, 2, 2])
    offs = orc.region(0, 3, [3, 3, 3])
    km = orc.kmap(c, c, offs, scale=[2, 2, 2])
    X = g.standard_normal((c.shape[0], cin))
    W = g.standard_normal((27, cout, cin))
    Gout = g.standard_normal((c.shape[0], cout))
    cc = _compact(c)
    xd = torch.zeros(1, cin, G, G, G, dtype=torch.float64)
    xd[0][:, cc[:, 0], cc[:, 1], cc[:, 2]] = torch.from_numpy(X.T)
    xd.requires_grad_(True)
    wt = _w_to_torch(W, offs, 3).requires_grad_(True)
    yd = F.conv3d(xd, wt, padding=1)
    np.testing.assert_allclose(orc.conv_forward(km, X, W, c.shape[0]), _dense_to_rows(yd[0].detach().numpy(), cc),
                               rtol=1e-12, atol=1e-12)
    gd = torch.zeros_like(yd)
    gd[0][:, cc[:, 0], cc[:, 1], cc[:, 2]] = torch.from_numpy(Gout.T)
    (yd * gd).sum().backward()
    np.testing.assert_allclose(orc.conv_dgrad(km, Gout, W, c.shape[0]), _dense_to_rows(xd.grad[0].numpy(), cc),
                               rtol=1e-12, atol=1e-12)
    dW = orc.conv_wgrad(km, Gout, X, 27)
    for k, (a, b, e) in enumerate(offs.tolist()):
        np.testing.assert_allclose(dW[k], wt.grad[:, :, a + 1, b + 1, e + 1].numpy(), rtol=1e-12, atol=1e-12)
    # |M| on the full lattice is the closed form (3G - 2)^3 only with the scaled offsets
    assert km[0][-1] == (3 * G - 2) ** 3


@pytest.mark.parametrize("K", [2, 3])
def test_tensor_stride2_to_4_and_transpose_equal_conv3d(orc, K):
    # stride-2 input -> stride-4 output (s_out = s_in * sigma), offsets scaled by s_in = 2;
    # the transposed map probes the fine (stride 2) set at v - i*2 (R13/R14).
    G, cin, cout = 6, 3, 4
    g = np.random.default_rng(50 + K)
    fine, _ = orc.create(_stride2_grid(G), tensor_stride=[2, 2, 2])
    coarse = orc.stride(fine, [2, 2, 2], [2, 2, 2])
    assert np.all(coarse[:, :3] % 4 == 0)
    offs = orc.region(0, 3, [K] * 3)
    km = orc.kmap(fine, coarse, offs, scale=[2, 2, 2])
    X = g.standard_normal((fine.shape[0], cin))
    W = g.standard_normal((offs.shape[0], cout, cin))
    y = orc.conv_forward(km, X, W, coarse.shape[0])
    cf = _compact(fine)
    xd = torch.zeros(1, cin, G, G, G, dtype=torch.float64)
    xd[0][:, cf[:, 0], cf[:, 1], cf[:, 2]] = torch.from_numpy(X.T)
    wt = _w_to_torch(W, offs, K)
    # base -4 is a multiple of 4, so the coarse lattice point 4j + base sits at compact 2j
    yd = F.conv3d(xd, wt, stride=2, padding=1 if K == 3 else 0)[0].numpy()
    np.testing.assert_allclose(y, _dense_to_rows(yd, _compact(coarse) // 2), rtol=1e-12, atol=1e-12)
    if K == 2:
        kmT = orc.kmap(coarse, fine, offs, scale=[2, 2, 2], transposed=True)
        Y = g.standard_normal((coarse.shape[0], cout))
        WT = np.transpose(W, (0, 2, 1)).copy()
        z = orc.conv_forward(kmT, Y, WT, fine.shape[0])
        cc = _compact(coarse) // 2
        yd2 = torch.zeros(1, cout, G // 2, G // 2, G // 2, dtype=torch.float64)
        yd2[0][:, cc[:, 0], cc[:, 1], cc[:, 2]] = torch.from_numpy(Y.T)
        zd = F.conv_transpose3d(yd2, wt, stride=2)[0].numpy()
        np.testing.assert_allclose(z, _dense_to_rows(zd, cf), rtol=1e-12, atol=1e-12)
