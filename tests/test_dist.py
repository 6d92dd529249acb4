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
    g = np.random.default_rng(seed)
    rows = []
    for b in range(n_scans):
        n = int(g.integers(150, 400))
        c = g.integers(-6, 6, (n, 3))
        rows.append(np.concatenate([c, np.full((n, 1), b)], axis=1))
    return np.concatenate(rows).astype(np.int32)


def _worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_1904_08755_b200.dist import allreduce_grad, gather_rows, lpt_assign
    rows = _scans()
    coords, _ = oracle.create(rows)
    offs = oracle.region(0, 3, [3, 3, 3])
    g = np.random.default_rng(9)
    X = g.standard_normal((coords.shape[0], 4))
    W = g.standard_normal((27, 5, 4))
    G = g.standard_normal((coords.shape[0], 5))
    scans = sorted(set(coords[:, 3].tolist()))
    costs = []
    for b in scans:
        sel = coords[:, 3] == b
        costs.append(float(oracle.kmap(coords[sel], coords[sel], offs)[0][-1]))
    mine = lpt_assign(costs, world)[rank]
    y_parts, dW = [], np.zeros_like(W)
    for b in mine:
        sel = np.nonzero(coords[:, 3] == b)[0]
        km = oracle.kmap(coords[sel], coords[sel], offs)
        y_parts.append(np.concatenate([sel[:, None], oracle.conv_forward(km, X[sel], W, sel.size)], axis=1))
        dW += oracle.conv_wgrad(km, G[sel], X[sel], 27)
    y_local = torch.from_numpy(np.concatenate(y_parts) if y_parts else np.zeros((0, 6)))
    dW_t = allreduce_grad(torch.from_numpy(dW.copy()))
    gathered = gather_rows(y_local)
    if rank == 0:
        full = torch.cat(gathered).numpy()
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
    rows = _scans()
    coords, _ = orc.create(rows)
    offs = orc.region(0, 3, [3, 3, 3])
    g = np.random.default_rng(9)
    X = g.standard_normal((coords.shape[0], 4))
    W = g.standard_normal((27, 5, 4))
    G = g.standard_normal((coords.shape[0], 5))
    km = orc.kmap(coords, coords, offs)  # the batched map (all scans at once)
    y_all = orc.conv_forward(km, X, W, coords.shape[0])
    dW_all = orc.conv_wgrad(km, G, X, 27)
    order = np.argsort(y[:, 0])
    assert np.array_equal(y[order, 0].astype(int), np.arange(coords.shape[0]))
    np.testing.assert_allclose(y[order, 1:], y_all, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(dW, dW_all, rtol=1e-12, atol=1e-12)
