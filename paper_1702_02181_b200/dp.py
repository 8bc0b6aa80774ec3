"""Data-parallel plumbing: input graphs are independent (a
batch is a *disconnected* graph), so ranks split the tree list and each schedules and
runs its own shard; the only exchange is one all_reduce(SUM) of the flat fp32 weight
gradient [dU | db | dE] per step (NCCL over NVLink on B200s; gloo in CPU tests).

Host logic only — no method arithmetic lives here.
"""
from __future__ import annotations

import numpy as np
import torch


def shard_bounds(tree_sizes, world: int) -> np.ndarray:
    """Contiguous prefix split of the tree list by node count: shard r gets trees
    [b[r], b[r+1]), where the cumulative node count first reaches ceil(r*N/world).
    Deterministic; every shard is within one tree of N/world nodes."""
    sizes = np.asarray(tree_sizes, dtype=np.int64)
    cum = np.concatenate([[0], np.cumsum(sizes)])
    total = int(cum[-1])
    bounds = [0]
    for r in range(1, world):
        target = (total * r + world - 1) // world
        bounds.append(int(np.searchsorted(cum, target, side="left")))
    bounds.append(len(sizes))
    return np.maximum.accumulate(np.asarray(bounds, dtype=np.int64))


def shard(graphs, rank: int, world: int):
    """This rank's sub-batch (trees renumbered from 0) of a foldgen.Graphs-like batch."""
    import foldgen  # input slicing helper (no method arithmetic)
    b = shard_bounds(graphs.tree_sizes, world)
    return foldgen.sub_batch(graphs, int(b[rank]), int(b[rank + 1]))


class FlatParams:
    """U, b, E (and their gradients) as views of one flat fp32 buffer each, so one
    all_reduce and one SGD launch cover all parameters."""

    def __init__(self, U: np.ndarray, b: np.ndarray, E: np.ndarray, device):
        self.shapes = (U.shape, b.shape, E.shape)
        self.sizes = (U.size, b.size, E.size)
        n = sum(self.sizes)
        self.flat = torch.empty(n, dtype=torch.float32, device=device)
        self.grad = torch.zeros(n, dtype=torch.float32, device=device)
        self.U, self.b, self.E = self._views(self.flat)
        self.dU, self.db, self.dE = self._views(self.grad)
        for dst, src in ((self.U, U), (self.b, b), (self.E, E)):
            dst.copy_(torch.from_numpy(np.ascontiguousarray(src, dtype=np.float32)))

    def _views(self, buf):
        out, off = [], 0
        for shp, sz in zip(self.shapes, self.sizes):
            out.append(buf[off:off + sz].view(shp))
            off += sz
        return out


def allreduce_grads(grad_flat: torch.Tensor, group=None):
    """Sum the flat gradient over ranks (one collective per step)."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(grad_flat, op=dist.ReduceOp.SUM, group=group)
    return grad_flat
