"""Multi-process (gloo, world size 2, CPU) test of the batch-index sharding semantics
(SURVEY §8(e), O10): the per-rank results concatenated equal the batched result (batch
isolation) and the all-reduced weight gradient equals the batched dW.  The per-rank
compute is the CPU oracle (test infrastructure); the sharding / collectives are the
product's host logic (paper_1904_08755_b200/dist.py)."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parents[1]


def _scans(n_scans=5, seed=3):
    """Small float point clouds, one per batch index, concatenated in ascending scan order
    (as bench.py's configs[4] batch)."""
    g = np.random.default_rng(seed)
    pts, bat = [], []
    for b in range(n_scans):
        n = int(g.integers(300, 700))
        pts.append(g.uniform(-0.6, 0.6, (n, 3)).astype(np.float32))
        bat.append(np.full(n, b, np.int32))
    return np.concatenate(pts), np.concatenate(bat)


VOXEL = 0.1


def _features(n_rows):
    g = np.random.default_rng(9)
    X = g.standard_normal((n_rows, 4))
    W = g.standard_normal((27, 5, 4))
    G = g.standard_normal((n_rows, 5))
    return X, W, G


def _worker(rank, world, port, out_dir):
    # The host side of bench.py's multi-GPU step, driven with the oracle as the per-rank
    # compute: LPT shard plan on per-scan |M|, the rank's own points (rank_points), its own
    # coordinates and map, the dW all-reduce (allreduce_grad) and the output all-gather
    # (RowGather), over gloo instead of NCCL.
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1904_08755_b200.dist import RowGather, allreduce_grad, lpt_assign, rank_points
    pts, bat = _scans()
    offs = oracle.region(0, 3, [3, 3, 3])
    n_scans = int(bat.max()) + 1
    costs = []  # |M| per scan (setup, every rank the same)
    for b in range(n_scans):
        cb, _, _ = oracle.quantize(pts[bat == b], VOXEL, bat[bat == b])
        costs.append(float(oracle.kmap(cb, cb, offs)[0][-1]))
    mine = lpt_assign(costs, world)[rank]
    p_r, b_r = rank_points(pts, bat, mine)
    coords_r, _, _ = oracle.quantize(p_r, VOXEL, b_r)
    # features are indexed by the batched row (the rows of the rank's scans, in order)
    coords_all, _, _ = oracle.quantize(pts, VOXEL, bat)
    sel = np.nonzero(np.isin(coords_all[:, 3], mine))[0]
    assert np.array_equal(coords_all[sel], coords_r)
    X, W, G = _features(coords_all.shape[0])
    km = oracle.kmap(coords_r, coords_r, offs)
    y = oracle.conv_forward(km, X[sel], W, sel.size)
    dW = oracle.conv_wgrad(km, G[sel], X[sel], 27)
    dW_t = allreduce_grad(torch.from_numpy(dW.copy()))
    y_rows = torch.from_numpy(np.concatenate([sel[:, None].astype(np.float64), y], axis=1))
    gather = RowGather(y_rows.shape[0], y_rows.shape[1], y_rows.dtype, y_rows.device)
    gather(y_rows)
    if rank == 0:
        full = torch.cat(gather.views()).numpy()
        np.save(os.path.join(out_dir, "y.npy"), full)
        np.save(os.path.join(out_dir, "dW.npy"), dW_t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_lpt_assign_is_balanced_and_deterministic():
    from paper_1904_08755_b200.dist import lpt_assign
    costs = [150.0, 148.0, 152.0, 149.0, 151.0, 147.0, 153.0, 150.0]
    a = lpt_assign(costs, 4)
    assert a == lpt_assign(costs, 4)
    assert sorted(i for r in a for i in r) == list(range(8))
    loads = [sum(costs[i] for i in r) for r in a]
    assert max(loads) - min(loads) <= max(costs) - min(costs)


def test_sharded_equals_batched_gloo(tmp_path, orc):
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    mp.start_processes(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True, start_method="spawn")
    y = np.load(tmp_path / "y.npy")
    dW = np.load(tmp_path / "dW.npy")
    pts, bat = _scans()
    coords, _, _ = orc.quantize(pts, VOXEL, bat)  # the batched scans (all at once)
    offs = orc.region(0, 3, [3, 3, 3])
    X, W, G = _features(coords.shape[0])
    km = orc.kmap(coords, coords, offs)
    y_all = orc.conv_forward(km, X, W, coords.shape[0])
    dW_all = orc.conv_wgrad(km, G, X, 27)
    order = np.argsort(y[:, 0])
    assert np.array_equal(y[order, 0].astype(int), np.arange(coords.shape[0]))
    np.testing.assert_allclose(y[order, 1:], y_all, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dW, dW_all, rtol=1e-12, atol=1e-12)
