"""Batch-index data parallelism for the sparse-conv hot path.

Scans with different batch indices never interact: kernel offsets never change the batch
index b (reading R18), so every rank owns whole scans — their coordinate tables,
kernel maps and conv rows — and the path has no exchange step.  The only collective of a
training step is the sum of the per-rank weight gradients (NCCL ``all_reduce`` over
NVLink); gathering output features on one rank is optional and done with padded
``all_gather`` (shards are uneven).

Host logic only: the compute stays in libmk's kernels.
"""
from __future__ import annotations

from typing import List, Sequence

import torch
import torch.distributed as dist


def lpt_assign(costs: Sequence[float], world: int) -> List[List[int]]:
    """Greedy longest-processing-time assignment of scans to ranks (deterministic:
    ties broken by scan index, then by rank).  Returns the scan indices of every rank in
    ascending order."""
    order = sorted(range(len(costs)), key=lambda i: (-costs[i], i))
    load = [0.0] * world
    out: List[List[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda j: (load[j], j))
        out[r].append(i)
        load[r] += costs[i]
    return [sorted(x) for x in out]


def allreduce_grad(dW: torch.Tensor, group=None) -> torch.Tensor:
    """Sum of the weight gradients of all ranks (in place)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(dW, op=dist.ReduceOp.SUM, group=group)
    return dW


def gather_rows(y: torch.Tensor, group=None) -> List[torch.Tensor]:
    """All-gather of uneven row shards: every rank receives every rank's [n_r][C] tensor."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return [y]
    world = dist.get_world_size(group)
    n = torch.tensor([y.shape[0]], dtype=torch.int64, device=y.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    nmax = int(max(int(s.item()) for s in sizes))
    pad = torch.zeros((nmax,) + tuple(y.shape[1:]), dtype=y.dtype, device=y.device)
    pad[: y.shape[0]] = y
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return [b[: int(s.item())] for b, s in zip(bufs, sizes)]
