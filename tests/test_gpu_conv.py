"""GPU <-> fp64 oracle parity of the feature path: forward, dgrad, wgrad and the transposed
conv, in fp32 mode (tolerance 1e-5) and bf16 mode (2e-2), with every expectation built by the
oracle alone (tests/parity.py): oracle coordinates, oracle offsets, oracle kernel map.

Sizes: oracle-sized cases spanning many 128-row tiles with ragged tails, a sweep of every
bf16 channel pair (C_in, C_out) in {16, 32, ..., 256}^2, and BASELINE.json configs[1]-[3] at
full size in the launch configuration bench.py times (configs[4] is in test_gpu_configs.py).
"""
import numpy as np
import pytest
import torch

import synthetic
from gpu_util import BF16_TOL, FP32_TOL
from parity import Spec, check_features, dev, map_pair, oracle_threads, sample

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mk(orc):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    oracle_threads(orc)
    return m


def _sparse(mk, orc, seed, n, span, D=3, ts=1, nb=2):
    g = np.random.default_rng(seed)
    rows = np.concatenate([g.integers(-span, span, (n, D)) * ts, g.integers(0, nb, (n, 1))], axis=1).astype(np.int32)
    oc, _ = orc.create(rows, [ts] * D)
    c = mk.coords_create(dev(rows), [ts] * D)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    return c, oc


CUBE3 = Spec(0, 3, 3)


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("cin,cout,n,span", [(16, 16, 2000, 16), (64, 64, 20000, 30), (32, 64, 9000, 20),
                                             (96, 96, 5000, 15), (16, 32, 333, 6)])
def test_submanifold_conv(mk, orc, dt, tol, cin, cout, n, span):
    c, oc = _sparse(mk, orc, cin + n, n, span)
    m, okm = map_pair(mk, orc, c, c, oc, oc, CUBE3, [1, 1, 1])
    g = np.random.default_rng(n)
    X = synthetic.features(1, c.n, cin)
    W = synthetic.weights(2, 27, cout, cin)
    G = g.uniform(-1, 1, (c.n, cout)).astype(np.float32)
    check_features(mk, orc, m, okm, X, W, G, dt, tol, what=f"{dt} {cin}->{cout}")


@pytest.mark.parametrize("cin,cout", [(12, 20), (3, 40), (64, 24), (40, 64)])
def test_fp32_channel_counts_off_the_tensor_core_grid(mk, orc, cin, cout):
    # fp32 with a channel count that is not a multiple of 16 (on either side) runs the
    # exact-FFMA kernels and must match the oracle at the fp32 tolerance, like the bf16x3
    # split path (R28) that the multiples-of-16 cases above take
    c, oc = _sparse(mk, orc, cin * 7 + cout, 4000, 14)
    m, okm = map_pair(mk, orc, c, c, oc, oc, CUBE3, [1, 1, 1])
    X = synthetic.features(21, c.n, cin)
    W = synthetic.weights(22, 27, cout, cin)
    G = synthetic.features(23, c.n, cout)
    check_features(mk, orc, m, okm, X, W, G, "f32", FP32_TOL, what=f"f32 {cin}->{cout}")


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
def test_hybrid_4d_conv(mk, orc, dt, tol):
    c, oc = _sparse(mk, orc, 44, 12000, 14, D=4)
    m, okm = map_pair(mk, orc, c, c, oc, oc, Spec(2, 4, 3), [1] * 4)
    X = synthetic.features(3, c.n, 32)
    W = synthetic.weights(4, 29, 64, 32)
    G = synthetic.features(5, c.n, 64)
    check_features(mk, orc, m, okm, X, W, G, dt, tol, what="hybrid")


@pytest.mark.parametrize("dt,tol", [("f32", FP32_TOL), ("bf16", BF16_TOL)])
@pytest.mark.parametrize("K,ts", [(2, 1), (3, 1), (2, 2), (3, 2)])
def test_strided_conv_and_transpose(mk, orc, dt, tol, K, ts):
    # input tensor stride ts: offsets are scaled by ts (R14); coarse stride 2 ts
    fine, ofine = _sparse(mk, orc, 70 + K + 10 * ts, 15000, 24, ts=ts)
    coarse = mk.coords_stride(fine, [2, 2, 2])
    ocoarse = orc.stride(ofine, [2, 2, 2], [ts] * 3)
    assert np.array_equal(coarse.export().cpu().numpy(), ocoarse)
    spec = Spec(0, 3, K)
    m, okm = map_pair(mk, orc, fine, coarse, ofine, ocoarse, spec, [ts] * 3, what=f"down K={K}")
    cin, cout = 32, 48
    X = synthetic.features(6, fine.n, cin)
    W = synthetic.weights(7, m.K, cout, cin)
    G = synthetic.features(8, coarse.n, cout)
    check_features(mk, orc, m, okm, X, W, G, dt, tol, what=f"down K={K} ts={ts}")
    # transposed conv coarse -> fine, probing v - i*ts in the coarse table
    mt, okmt = map_pair(mk, orc, coarse, fine, ocoarse, ofine, spec, [ts] * 3, transposed=True, what=f"up K={K}")
    Y = synthetic.features(9, coarse.n, cout)
    WT = synthetic.weights(10, m.K, cin, cout)
    GT = synthetic.features(11, fine.n, cin)
    check_features(mk, orc, mt, okmt, Y, WT, GT, dt, tol, transposed=True, what=f"up K={K} ts={ts}")


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
def test_tesseract_4d_conv(mk, orc, dt, tol):
    # K = 3^4 = 81 offsets (the 4D hypercube of P:253): the K > 32 kernel-map path (k-major
    # table, identity row order, host split-K plan) and multi-word offset masks.
    c, oc = _sparse(mk, orc, 81, 6000, 7, D=4)
    m, okm = map_pair(mk, orc, c, c, oc, oc, Spec(0, 4, 3), [1] * 4)
    assert m.K == 81
    X = synthetic.features(12, c.n, 16)
    W = synthetic.weights(13, 81, 32, 16)
    G = synthetic.features(14, c.n, 32)
    check_features(mk, orc, m, okm, X, W, G, dt, tol, what="tesseract")


# ------------------------------------------------------------------ channel contract
@pytest.fixture(scope="module")
def sweep_map(mk, orc):
    c, oc = _sparse(mk, orc, 777, 1500, 9)
    m, okm = map_pair(mk, orc, c, c, oc, oc, CUBE3, [1, 1, 1])
    return c, m, okm


@pytest.mark.parametrize("cin", list(range(16, 257, 16)))
def test_bf16_channel_sweep(mk, orc, sweep_map, cin):
    # mk.h's bf16 channel contract: every (C_in, C_out) in {16, ..., 256}^2 plans (no
    # MK_ERR_UNSUPPORTED) and matches the oracle in fwd, dgrad and wgrad.
    c, m, okm = sweep_map
    for cout in range(16, 257, 16):
        print(f"sweep {cin}->{cout}", flush=True)
        X = synthetic.features(cin, c.n, cin)
        W = synthetic.weights(cout, 27, cout, cin)
        G = synthetic.features(cin + cout, c.n, cout)
        check_features(mk, orc, m, okm, X, W, G, "bf16", BF16_TOL, what=f"sweep {cin}->{cout}", repeat=False)


# ------------------------------------------------------------------ BASELINE configs at full size
@pytest.fixture(scope="module")
def room(mk, orc):
    # configs[1]: the bench's ScanNet-shaped room (seed 2000), quantized on both sides
    pts = synthetic.room_points(2000)
    c, _, _ = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL)
    oc, _, _ = orc.quantize(pts, synthetic.ROOM_VOXEL)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    m, okm = map_pair(mk, orc, c, c, oc, oc, CUBE3, [1, 1, 1], what="room")
    return c, oc, m, okm


@pytest.mark.parametrize("dt,tol", [("bf16", BF16_TOL), ("f32", FP32_TOL)])
def test_config1_room_full_size_all_rows(mk, orc, room, dt, tol):
    # configs[1] at full size (150k voxels, 1.39M pairs, C 64 -> 64): every row of fwd and
    # dgrad and all of dW, element by element.  The weight-gradient split-K gives each of its
    # 444 CTAs ~49 stages of 64 pairs, so its 4-slot stage ring wraps ~12 times.
    c, oc, m, okm = room
    assert m.n_pairs > 444 * 64 * 8
    X = synthetic.features(1, c.n, 64)
    W = synthetic.weights(2, 27, 64, 64)
    G = synthetic.features(3, c.n, 64)
    check_features(mk, orc, m, okm, X, W, G, dt, tol, what=f"configs[1] {dt}")


def test_config2_video_hybrid_full_size(mk, orc):
    # configs[2]: 3-frame Synthia-like video, 4D (x, y, z, t), hybrid kernel (29 offsets),
    # C 32 -> 64, full size, all rows.
    pts, fr = synthetic.video_points(3000)
    c3, _, _ = mk.coords_quantize(dev(pts), synthetic.VIDEO_VOXEL, dev(fr))
    o3, _, _ = orc.quantize(pts, synthetic.VIDEO_VOXEL, fr)
    assert np.array_equal(c3.export().cpu().numpy(), o3)
    o4 = np.concatenate([o3, np.zeros((o3.shape[0], 1), np.int32)], axis=1)  # frame -> t, b = 0
    c4 = mk.coords_create(dev(o4))
    m, okm = map_pair(mk, orc, c4, c4, o4, o4, Spec(2, 4, 3), [1] * 4, what="video")
    assert m.K == 29 and c4.n > 200000
    X = synthetic.features(31, c4.n, 32)
    W = synthetic.weights(32, 29, 64, 32)
    G = synthetic.features(33, c4.n, 64)
    check_features(mk, orc, m, okm, X, W, G, "bf16", BF16_TOL, what="configs[2]")


def test_config3_unet_pair_full_size(mk, orc, room):
    # configs[3]: the encoder / decoder layer pair on the room: output coordinates of the
    # stride-2 conv, 2x2x2 conv 128 -> 256 (fwd, dgrad, wgrad), and the transposed
    # 2x2x2 conv 256 -> 128 back onto the cached fine set (fwd, dgrad, wgrad).
    c, oc, _, _ = room
    coarse = mk.coords_stride(c, [2, 2, 2])
    ocoarse = orc.stride(oc, [2, 2, 2])
    assert np.array_equal(coarse.export().cpu().numpy(), ocoarse)
    spec = Spec(0, 3, 2)
    md, okd = map_pair(mk, orc, c, coarse, oc, ocoarse, spec, [1, 1, 1], what="down")
    assert md.n_pairs == c.n  # R3: with K = sigma = 2 every fine row is in exactly one pair
    X = synthetic.features(41, c.n, 128)
    W = synthetic.weights(42, 8, 256, 128)
    G = synthetic.features(43, coarse.n, 256)
    check_features(mk, orc, md, okd, X, W, G, "bf16", BF16_TOL, what="configs[3] down 128->256")
    mu, oku = map_pair(mk, orc, coarse, c, ocoarse, oc, spec, [1, 1, 1], transposed=True, what="up")
    Y = synthetic.features(44, coarse.n, 256)
    WT = synthetic.weights(45, 8, 128, 256)
    GT = synthetic.features(46, c.n, 128)
    check_features(mk, orc, mu, oku, Y, WT, GT, "bf16", BF16_TOL, transposed=True, what="configs[3] up 256->128")


def test_wgrad_two_streams_share_the_scratch(mk, orc):
    # The bf16 weight gradient keeps its partial sums in one per-context scratch buffer; calls
    # on two streams alternate on it (the second waits for the first one's event).  Launch
    # interleaved weight gradients of two different maps / channel counts on two streams and
    # compare both with the oracle.
    cases = []
    for j, (cin, cout, n, span) in enumerate([(96, 96, 6000, 16), (64, 128, 9000, 20)]):
        c, oc = _sparse(mk, orc, 700 + j, n, span)
        m, okm = map_pair(mk, orc, c, c, oc, oc, CUBE3, [1, 1, 1])
        X = synthetic.features(31 + j, c.n, cin)
        G = synthetic.features(41 + j, c.n, cout)
        W = synthetic.weights(51 + j, 27, cout, cin)
        want = orc.conv_wgrad(okm, G, X, 27)
        cases.append((m, X, G, W, want))
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    outs = [[], []]
    dev_in = [(dev(X).bfloat16(), dev(G).bfloat16(), dev(W).bfloat16()) for (_, X, G, W, _) in cases]
    torch.cuda.synchronize()
    for rep in range(3):
        for j in (0, 1):
            with torch.cuda.stream(streams[j]):
                Xd, Gd, Wd = dev_in[j]
                _, gw = mk.conv_backward(cases[j][0], Gd, Xd, Wd, need_gin=False, need_gw=True)
                outs[j].append(gw)
    torch.cuda.synchronize()
    for j in (0, 1):
        want = cases[j][4]
        for gw in outs[j]:
            got = gw.cpu().numpy()
            err = np.abs(got - want).max() / np.abs(want).max()
            assert err <= BF16_TOL, f"stream {j}: normwise error {err:.3e}"
        assert all(torch.equal(outs[j][0], o) for o in outs[j][1:]), "not deterministic across streams"
