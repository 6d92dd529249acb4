"""Pins for the oracle's TS-CRF mean-field inference (Alg. 5, Eq. 4,
P:316-352) on 7D space-time-chroma coordinates: closed forms (zero pairwise kernel; an
isolated node), a brute-force dict/numpy evaluation of Eq. 4 that shares nothing with the
oracle's kernel map, and stationarity (translation invariance).  No GPU."""
import numpy as np

D = 7


def _softmax(a):
    e = np.exp(a - a.max(axis=1, keepdims=True))
    return e / e.sum(axis=1, keepdims=True)


def _lattice(seed, n=300, span=3):
    g = np.random.default_rng(seed)
    rows = np.concatenate([g.integers(-span, span + 1, (n, D)), np.zeros((n, 1), np.int64)], axis=1)
    return np.unique(rows, axis=0).astype(np.int32)


def test_crf_zero_kernel_is_unary_softmax(orc):
    c = _lattice(0)
    offs = orc.region(1, D, [3] * D)  # 7D hypercross: 15 offsets
    km = orc.kmap(c, c, offs)
    phi = np.random.default_rng(1).standard_normal((c.shape[0], 5))
    for n_iters in (0, 1, 3):
        q = orc.crf_infer(km, phi, np.zeros((offs.shape[0], 5, 5)), n_iters)
        np.testing.assert_allclose(q, _softmax(phi), rtol=1e-14, atol=1e-15)


def test_crf_isolated_node_closed_form(orc):
    # one node: its only neighbour is itself (offset 0); Q^1 = softmax(phi + W_0 softmax(phi))
    c = np.zeros((1, D + 1), np.int32)
    offs = orc.region(1, D, [3] * D)
    km = orc.kmap(c, c, offs)
    g = np.random.default_rng(2)
    phi = g.standard_normal((1, 4))
    W = g.standard_normal((offs.shape[0], 4, 4))
    k0 = [i for i, o in enumerate(offs.tolist()) if not any(o)][0]
    q1 = _softmax(phi + _softmax(phi) @ W[k0].T)
    np.testing.assert_allclose(orc.crf_infer(km, phi, W, 1), q1, rtol=1e-13, atol=1e-15)


def test_crf_matches_brute_force_eq4(orc):
    # Eq. 4 evaluated directly: Q_i <- softmax(phi_i + sum_k W_k Q_{x_i + i_k}) with the
    # neighbours found by a python dict over the 7D rows (no kernel map)
    c = _lattice(3)
    offs = orc.region(1, D, [3] * D)
    g = np.random.default_rng(4)
    phi = g.standard_normal((c.shape[0], 3))
    W = g.standard_normal((offs.shape[0], 3, 3)) * 0.5
    index = {tuple(r): i for i, r in enumerate(c.tolist())}
    q = _softmax(phi)
    for _ in range(3):
        qt = np.zeros_like(q)
        for i, r in enumerate(c.tolist()):
            for k, o in enumerate(offs.tolist()):
                j = index.get(tuple(r[d] + o[d] for d in range(D)) + (r[D],))
                if j is not None:
                    qt[i] += W[k] @ q[j]
        q = _softmax(phi + qt)
    got = orc.crf_infer(orc.kmap(c, c, offs), phi, W, 3)
    np.testing.assert_allclose(got, q, rtol=1e-12, atol=1e-14)


def test_crf_stationarity(orc):
    # phi_p(u, v) = phi_p(u + tau, v + tau): translating every node leaves Q unchanged
    c = _lattice(5)
    offs = orc.region(1, D, [3] * D)
    g = np.random.default_rng(6)
    phi = g.standard_normal((c.shape[0], 4))
    W = g.standard_normal((offs.shape[0], 4, 4)) * 0.3
    q = orc.crf_infer(orc.kmap(c, c, offs), phi, W, 2)
    tau = np.array([5, -3, 2, 7, -1, 4, 9, 0], np.int32)
    c2 = c + tau
    np.testing.assert_allclose(orc.crf_infer(orc.kmap(c2, c2, offs), phi, W, 2), q, rtol=1e-13, atol=1e-15)


def _tiny(orc, seed, n=40, C=3):
    g = np.random.default_rng(seed)
    c = _lattice(seed, n=n, span=1)
    offs = orc.region(1, D, [3] * D)
    km = orc.kmap(c, c, offs)
    phi = g.standard_normal((c.shape[0], C))
    W = g.standard_normal((offs.shape[0], C, C)) * 0.5
    G = g.standard_normal((c.shape[0], C))
    return km, phi, W, G


def test_crf_backward_matches_finite_differences(orc):
    # Eq. 5 pinned by central differences of L = sum(G * Q^N) (fp64; no shared formula)
    km, phi, W, G = _tiny(orc, 11)
    n_iters = 2
    gphi, gW = orc.crf_backward(km, phi, W, n_iters, G)
    L = lambda p, w: float((G * orc.crf_infer(km, p, w, n_iters)).sum())  # noqa: E731
    h = 1e-6
    g = np.random.default_rng(12)
    for _ in range(12):
        i, c = g.integers(0, phi.shape[0]), g.integers(0, phi.shape[1])
        d = np.zeros_like(phi)
        d[i, c] = h
        fd = (L(phi + d, W) - L(phi - d, W)) / (2 * h)
        assert abs(fd - gphi[i, c]) <= 1e-7 + 1e-6 * abs(fd)
        k, a, b = g.integers(0, W.shape[0]), g.integers(0, W.shape[1]), g.integers(0, W.shape[2])
        e = np.zeros_like(W)
        e[k, a, b] = h
        fd = (L(phi, W + e) - L(phi, W - e)) / (2 * h)
        assert abs(fd - gW[k, a, b]) <= 1e-7 + 1e-6 * abs(fd)


def test_crf_backward_shift_invariance_and_zero_iterations(orc):
    # adding a constant to a node's logits leaves every Q^n unchanged, so each row of
    # dL/dphi_u sums to 0; with N = 0 the gradient is the softmax Jacobian applied to G
    km, phi, W, G = _tiny(orc, 13)
    for n_iters in (0, 1, 3):
        gphi, gW = orc.crf_backward(km, phi, W, n_iters, G)
        np.testing.assert_allclose(gphi.sum(axis=1), 0.0, atol=1e-12)
        if n_iters == 0:
            q = _softmax(phi)
            J = np.einsum("ic,cd->icd", q, np.eye(q.shape[1])) - np.einsum("ic,id->icd", q, q)
            np.testing.assert_allclose(gphi, np.einsum("icd,ic->id", J, G), atol=1e-14)
            assert not gW.any()
