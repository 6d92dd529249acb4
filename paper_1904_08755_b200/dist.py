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


def rank_points(points, batch, scans: Sequence[int]):
    """The raw points of a rank's scans (host arrays): every point whose batch index is in
    `scans`, in input order.  When the batched input lists its scans in ascending batch
    order (as a data loader concatenating scans does), the rank's quantized rows are exactly
    the batched rows of its scans, in the same order (first occurrence, reading R8)."""
    import numpy as np
    sel = np.isin(batch, np.asarray(sorted(scans), dtype=batch.dtype))
    return points[sel], batch[sel]


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


class RowGather:
    """All-gather of uneven row shards with a fixed layout: the shard sizes are exchanged once
    (at construction), every call copies the local rows into a padded [n_max][C] slot and
    runs one ``all_gather_into_tensor`` into a preallocated [world * n_max][C] buffer (one
    NCCL call over NVLink; padding <= the LPT imbalance).  ``views()`` are the ranks' rows."""

    def __init__(self, n_local: int, cols: int, dtype, device, group=None):
        self.group = group
        self.world = dist.get_world_size(group) if (dist.is_available() and dist.is_initialized()) else 1
        n = torch.tensor([n_local], dtype=torch.int64, device=device)
        sizes = [torch.zeros_like(n) for _ in range(self.world)]
        if self.world > 1:
            dist.all_gather(sizes, n, group=group)
        else:
            sizes = [n]
        self.sizes = [int(x.item()) for x in sizes]
        self.n_max = max(self.sizes) if self.sizes else 0
        self.pad = torch.zeros((self.n_max, cols), dtype=dtype, device=device)
        self.out = torch.empty((self.world * self.n_max, cols), dtype=dtype, device=device)

    @property
    def bytes_per_call(self) -> int:
        """Bytes each rank receives per call (the padded NCCL all-gather payload)."""
        return int(self.out.numel() * self.out.element_size())

    def __call__(self, y: torch.Tensor) -> torch.Tensor:
        if self.world == 1:
            self.out[: y.shape[0]].copy_(y)
            return self.out
        self.pad[: y.shape[0]].copy_(y)
        dist.all_gather_into_tensor(self.out, self.pad, group=self.group)
        return self.out

    def views(self):
        return [self.out[r * self.n_max: r * self.n_max + n] for r, n in enumerate(self.sizes)]

