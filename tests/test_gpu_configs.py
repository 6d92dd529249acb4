"""BASELINE.json configs[4] on one GPU: a batch of 16 ScanNet-shaped scans (b = 0..15,
~2.4M voxels), 3x3x3, C 96 -> 96, against the fp64 oracle; and the batch-index sharded
execution of bench.py (each rank quantizes, maps and convolves only its own scans, LPT on
|M|) emulated rank by rank on the one device: the per-rank results
concatenated equal the batched oracle (batch isolation) and the per-rank weight
gradients sum to the batched one (the NCCL all-reduce's input)."""
import numpy as np
import pytest
import torch

import synthetic
from gpu_util import BF16_TOL, assert_close, to_np
from parity import Spec, assert_map_equal, check_features, dev, map_pair, oracle_threads, sample

pytestmark = pytest.mark.gpu

C = 96


@pytest.fixture(scope="module")
def mk(orc):
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    import paper_1904_08755_b200 as m
    oracle_threads(orc)
    return m


@pytest.fixture(scope="module")
def batch16(mk, orc):
    pts, bat = synthetic.rooms_batch(5000, 16)
    c, _, _ = mk.coords_quantize(dev(pts), synthetic.ROOM_VOXEL, dev(bat))
    oc, _, _ = orc.quantize(pts, synthetic.ROOM_VOXEL, bat)
    assert np.array_equal(c.export().cpu().numpy(), oc)
    m, okm = map_pair(mk, orc, c, c, oc, oc, Spec(0, 3, 3), [1, 1, 1], what="configs[4] batch")
    X = synthetic.features(51, c.n, C)
    W = synthetic.weights(52, 27, C, C)
    G = synthetic.features(53, c.n, C)
    return pts, bat, c, oc, m, okm, X, W, G


def test_config4_batch16_one_gpu(mk, orc, batch16):
    # 2.4M voxels, ~22M pairs: fwd / dgrad on 3,000 sampled rows each, dW in full
    pts, bat, c, oc, m, okm, X, W, G = batch16
    assert c.n > 2_000_000 and sorted(set(oc[:, 3].tolist())) == list(range(16))
    rows = sample(c.n, 3000, 54)
    check_features(mk, orc, m, okm, X, W, G, "bf16", BF16_TOL, what="configs[4]", sample_rows=(rows, rows),
                   repeat=False)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_config4_sharded_ranks_equal_batched(mk, orc, batch16, world):
    from paper_1904_08755_b200.dist import lpt_assign, rank_points
    pts, bat, c, oc, m, okm, X, W, G = batch16
    # |M| per scan from the oracle's batched map (the product computes it on the GPU at setup)
    o_of = okm[2]
    cost = np.bincount(oc[o_of, 3], minlength=16).astype(float)
    shards = lpt_assign(cost.tolist(), world)
    assert sorted(s for sh in shards for s in sh) == list(range(16))
    loads = [cost[sh].sum() for sh in shards]
    assert max(loads) <= 1.1 * sum(loads) / world  # LPT balance (scans are 150k +- 3%)
    Wd = dev(W).to(torch.bfloat16)
    dW = torch.zeros((27, C, C), dtype=torch.float32, device="cuda")
    y_all = np.zeros((c.n, C), np.float32)
    gin_all = np.zeros((c.n, C), np.float32)
    for r in range(world):
        p_r, b_r = rank_points(pts, bat, shards[r])
        cr, _, _ = mk.coords_quantize(dev(p_r), synthetic.ROOM_VOXEL, dev(b_r))
        sel = np.isin(oc[:, 3], shards[r])  # the batched rows of this rank's scans, in order
        assert np.array_equal(cr.export().cpu().numpy(), oc[sel])
        mr = mk.kmap_build(cr, cr, mk.Region(mk.HYPERCUBE, 3, 3))
        idx = np.nonzero(sel)[0]
        Xr, Gr = dev(X[idx]).to(torch.bfloat16), dev(G[idx]).to(torch.bfloat16)
        y_all[idx] = to_np(mk.conv_forward(mr, Xr, Wd, out_dtype=torch.float32))
        gin, gw = mk.conv_backward(mr, Gr, Xr, Wd)
        gin_all[idx] = to_np(gin)
        dW += gw  # the all-reduce's sum
    rows = sample(c.n, 2000, 55 + world)
    assert_close(y_all[rows], orc.conv_forward_rows(okm, X, W, rows),
                 orc.conv_forward_rows(okm, np.abs(X), np.abs(W), rows), BF16_TOL, f"sharded fwd ws={world}")
    rokm = orc.kmap_reverse(okm)
    WT = np.ascontiguousarray(np.transpose(W, (0, 2, 1)))
    assert_close(gin_all[rows], orc.conv_forward_rows(rokm, G, WT, rows),
                 orc.conv_forward_rows(rokm, np.abs(G), np.abs(WT), rows), BF16_TOL, f"sharded dgrad ws={world}")
    if world == 2:  # full dW once (0.4 TFLOP of fp64 oracle work per evaluation)
        assert_close(to_np(dW), orc.conv_wgrad(okm, G, X, 27), orc.conv_wgrad(okm, np.abs(G), np.abs(X), 27),
                     BF16_TOL, "sharded dW sum")
    else:  # the sum of the shards' dW is the batched GPU dW up to fp32 summation order
        _, gw_batched = mk.conv_backward(m, dev(G).to(torch.bfloat16), dev(X).to(torch.bfloat16), Wd, need_gin=False)
        np.testing.assert_allclose(to_np(dW), to_np(gw_batched), rtol=0, atol=1e-4 * float(gw_batched.abs().max()))
