"""Pins for the oracle's kernel regions (O4) and kernel maps (O5).  No GPU."""
import itertools

import numpy as np
import pytest

from conftest import full_grid, golden_lines

KIND = {"hypercube": 0, "hypercross": 1, "hybrid": 2}


def test_region_cardinalities(orc):
    # tests/golden/region_counts.txt: P:96.
    for line in golden_lines("region_counts.txt"):
        lhs, rhs = line.split("->")
        kind, D, size = lhs.split()
        offs = orc.region(KIND[kind], int(D), [int(x) for x in size.split(",")])
        assert offs.shape == (int(rhs), int(D))
        assert len({tuple(o) for o in offs.tolist()}) == offs.shape[0]


def test_region_v1_3_and_order(orc):
    assert orc.region(0, 1, [3]).ravel().tolist() == [-1, 0, 1]  # V^1(3)
    cube = orc.region(0, 3, [3, 3, 3]).tolist()
    assert cube == sorted(cube)  # lexicographic, axis 0 most significant (R2)
    assert cube[13] == [0, 0, 0]
    assert cube == [list(t) for t in itertools.product([-1, 0, 1], repeat=3)]


def test_region_even_and_dilation(orc):
    # Reading R3: even K -> {0..K-1}; dilation multiplies each component.
    assert orc.region(0, 3, [2, 2, 2]).tolist() == [list(t) for t in itertools.product([0, 1], repeat=3)]
    d = orc.region(0, 2, [3, 3], dilation=[2, 3])
    assert d.tolist() == [[a, b] for a in (-2, 0, 2) for b in (-3, 0, 3)]


def test_region_hybrid_composition(orc):
    # Reading R4: (3^3 cube at t=0) U {(0,0,0,+-1)}.
    h = {tuple(o) for o in orc.region(2, 4, [3, 3, 3, 3]).tolist()}
    cube = {t + (0,) for t in itertools.product([-1, 0, 1], repeat=3)}
    assert h == cube | {(0, 0, 0, -1), (0, 0, 0, 1)}


def test_region_custom(orc):
    offs = [[1, 0], [0, 0], [-1, 2]]
    assert orc.region(3, 2, custom=offs).tolist() == offs  # caller's order kept
    with pytest.raises(orc.OracleError):
        orc.region(3, 2, custom=[[0, 0], [0, 0]])


def test_kmap_worked_examples(orc):
    # tests/golden/kmap_grid.txt: S:160-161.
    for line in golden_lines("kmap_grid.txt"):
        lhs, rhs = line.split("->")
        G, D, K = [int(x) for x in lhs.split()]
        c = full_grid(G, D)
        offs = orc.region(0, D, [K] * D)
        ptr, ins, outs = orc.kmap(c, c, offs)
        assert ptr[-1] == int(rhs)
        if G == 1:
            center = offs.tolist().index([0] * D)
            assert ptr[center + 1] - ptr[center] == 1


@pytest.mark.parametrize("G,D", [(3, 1), (5, 2), (4, 3), (3, 4)])
def test_kmap_full_grid_closed_form(orc, G, D):
    # Fully occupied G^D grid, 3^D cube: every axis contributes 3G-2 pairs -> (3G-2)^D.
    c = full_grid(G, D)
    ptr, _, _ = orc.kmap(c, c, orc.region(0, D, [3] * D))
    assert ptr[-1] == (3 * G - 2) ** D


def _brute_pairs(c_in, c_out, offs, scale, sign=1):
    """O(N_in * N_out * K) brute force: compare every input against every shifted output."""
    D = offs.shape[1]
    pairs = []
    for k, off in enumerate(offs):
        shifted = c_out[:, :D].astype(np.int64) + sign * off.astype(np.int64) * np.asarray(scale)
        eq = np.all(shifted[:, None, :] == c_in[None, :, :D], axis=2) & (c_out[:, None, D] == c_in[None, :, D])
        o, a = np.nonzero(eq)
        order = np.argsort(o, kind="stable")
        pairs.append((a[order], o[order]))
    return pairs


def _csr_pairs(ptr, ins, outs):
    return [(ins[ptr[k]:ptr[k + 1]], outs[ptr[k]:ptr[k + 1]]) for k in range(len(ptr) - 1)]


@pytest.mark.parametrize("kind,D,size", [(0, 3, 3), (1, 3, 3), (2, 4, 3), (0, 2, 5)])
def test_kmap_brute_force_submanifold(orc, kind, D, size):
    g = np.random.default_rng(D * 10 + kind)
    c = g.integers(-4, 4, (300, D))
    rows = np.concatenate([c, g.integers(0, 2, (300, 1))], axis=1).astype(np.int32)
    rows, _ = orc.create(rows)
    offs = orc.region(kind, D, [size] * D)
    got = _csr_pairs(*orc.kmap(rows, rows, offs))
    want = _brute_pairs(rows, rows, offs, [1] * D)
    for (ga, go), (wa, wo) in zip(got, want):
        assert np.array_equal(ga, wa) and np.array_equal(go, wo)
    # submanifold: the centre offset pairs every row with itself
    if kind != 2 or True:
        center = offs.tolist().index([0] * D)
        ca, co = got[center]
        assert np.array_equal(ca, np.arange(rows.shape[0])) and np.array_equal(co, ca)


def test_kmap_strided_brute_force_and_partition(orc):
    # Strided conv ("multiples of a natural number"): fine stride 1 -> coarse stride 2.
    g = np.random.default_rng(7)
    fine = np.concatenate([g.integers(-6, 6, (400, 3)), np.zeros((400, 1), int)], axis=1).astype(np.int32)
    fine, _ = orc.create(fine)
    coarse = orc.stride(fine, [2, 2, 2])
    offs = orc.region(0, 3, [2, 2, 2])
    ptr, ins, outs = orc.kmap(fine, coarse, offs, scale=[1, 1, 1])
    want = _brute_pairs(fine, coarse, offs, [1, 1, 1])
    for (ga, go), (wa, wo) in zip(_csr_pairs(ptr, ins, outs), want):
        assert np.array_equal(ga, wa) and np.array_equal(go, wo)
    # Reading R3 pin: with K = sigma = 2 every input row is in exactly one pair.
    assert ptr[-1] == fine.shape[0]
    assert np.array_equal(np.sort(ins), np.arange(fine.shape[0]))
    # K=3, stride 2 also matches brute force
    offs3 = orc.region(0, 3, [3, 3, 3])
    ptr3, ins3, outs3 = orc.kmap(fine, coarse, offs3)
    for (ga, go), (wa, wo) in zip(_csr_pairs(ptr3, ins3, outs3), _brute_pairs(fine, coarse, offs3, [1] * 3)):
        assert np.array_equal(ga, wa) and np.array_equal(go, wo)


@pytest.mark.parametrize("K", [2, 3])
def test_kmap_transposed_duality(orc, K):
    # the transposed map is the forward map with the roles reversed.
    g = np.random.default_rng(11 + K)
    fine = np.concatenate([g.integers(-5, 5, (300, 3)) * 2, g.integers(0, 2, (300, 1))], axis=1).astype(np.int32)
    fine, _ = orc.create(fine, tensor_stride=[2, 2, 2])
    coarse = orc.stride(fine, [2, 2, 2], [2, 2, 2])
    offs = orc.region(0, 3, [K] * 3)
    fwd = _csr_pairs(*orc.kmap(fine, coarse, offs, scale=[2, 2, 2]))
    tr = _csr_pairs(*orc.kmap(coarse, fine, offs, scale=[2, 2, 2], transposed=True))
    for (fa, fo), (ta, to) in zip(fwd, tr):
        order = np.argsort(fa, kind="stable")
        assert np.array_equal(to, fa[order]) and np.array_equal(ta, fo[order])


def test_lookup(orc):
    g = np.random.default_rng(3)
    rows, _ = orc.create(np.concatenate([g.integers(-9, 9, (200, 3)), np.zeros((200, 1), int)], axis=1))
    assert np.array_equal(orc.lookup(rows, rows), np.arange(rows.shape[0]))
    miss = rows.copy()
    miss[:, 3] = 5
    assert np.all(orc.lookup(rows, miss) == -1)


@pytest.mark.parametrize("K", [2, 3])
def test_kmap_reverse_is_transposed_map_and_involution(orc, K):
    # P:202 (roles reversed): reverse(map fine -> coarse) is the transposed map coarse -> fine,
    # which is built by independent probing (v - i*s); reversing twice gives the map back.
    g = np.random.default_rng(21 + K)
    fine = np.concatenate([g.integers(-6, 6, (300, 3)) * 2, g.integers(0, 2, (300, 1))], axis=1).astype(np.int32)
    fine, _ = orc.create(fine, tensor_stride=[2, 2, 2])
    coarse = orc.stride(fine, [2, 2, 2], [2, 2, 2])
    offs = orc.region(0, 3, [K] * 3)
    fwd = orc.kmap(fine, coarse, offs, scale=[2, 2, 2])
    tr = orc.kmap(coarse, fine, offs, scale=[2, 2, 2], transposed=True)
    rev = orc.kmap_reverse(fwd)
    for a, b in zip(rev, tr):
        assert np.array_equal(a, b)
    for a, b in zip(orc.kmap_reverse(rev), fwd):
        assert np.array_equal(a, b)
    # O7 = O6 on the reverse map with W_k^T, element by element
    X = g.standard_normal((coarse.shape[0], 3))
    W = g.standard_normal((offs.shape[0], 3, 4))
    rows = np.arange(fine.shape[0], dtype=np.int32)
    np.testing.assert_allclose(orc.conv_forward_rows(rev, X, np.transpose(W, (0, 2, 1)).copy(), rows),
                               orc.conv_dgrad(fwd, X, W, fine.shape[0]), rtol=1e-13, atol=1e-13)
