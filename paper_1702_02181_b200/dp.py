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


def exchange_plan(counts, S: int, V: int, world: int) -> tuple[str, int]:
    """Sparse or dense exchange of the embedding gradient dE [V][S].
    counts[r] = rows rank r touched (its batch's distinct tokens). Sparse: every rank
    all-gathers world x maxn rows of S floats plus their ids; dense: a ring all_reduce moves
    ~2 (world - 1) / world x V S floats per rank. Returns (mode, maxn)."""
    maxn = int(max(counts)) if len(counts) else 0
    sparse_bytes = world * maxn * (S + 1) * 4
    dense_bytes = 2 * (world - 1) / max(world, 1) * V * S * 4
    return ("sparse" if sparse_bytes < dense_bytes else "dense"), maxn


def exchange_grads(flat_g: torch.Tensor, n_dense: int, dE: torch.Tensor, rows: torch.Tensor, group=None,
                   mode: str = "auto", scratch: dict | None = None) -> str:
    """Data-parallel gradient exchange: all_reduce of the dense part flat_g[:n_dense] ([dU | db]),
    and the embedding gradient dE [V][S] (a view of flat_g) either all-reduced (dense) or
    exchanged as the touched rows only: all-gather each rank's packed rows (fold_gather_rows,
    padded with id -1 to the largest count), zero dE, then add rank 0's rows, rank 1's, ...
    (fold_scatter_add_rows, one call per rank: the same order on every rank, so every rank ends
    with bitwise the same dE). `rows` = this rank's distinct tokens (fold_touched_rows).
    Returns the mode used."""
    import torch.distributed as dist
    from . import fold
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return "local"
    world = dist.get_world_size(group)
    dist.all_reduce(flat_g[:n_dense], op=dist.ReduceOp.SUM, group=group)
    V, S = int(dE.shape[0]), int(dE.shape[1])
    cnt = torch.tensor([int(rows.numel())], dtype=torch.int64, device=flat_g.device)
    counts = [torch.zeros_like(cnt) for _ in range(world)]
    dist.all_gather(counts, cnt, group=group)
    plan, maxn = exchange_plan([int(c.item()) for c in counts], S, V, world)
    if mode != "auto":
        plan = mode
    if plan == "dense" or maxn == 0:
        dist.all_reduce(dE, op=dist.ReduceOp.SUM, group=group)
        return "dense"
    sc = scratch if scratch is not None else {}
    dev = flat_g.device
    if sc.get("maxn", -1) < maxn:
        sc["maxn"] = maxn
        sc["ids"] = torch.empty(maxn, dtype=torch.int32, device=dev)
        sc["rows"] = torch.empty((maxn, S), dtype=torch.float32, device=dev)
        sc["all_ids"] = [torch.empty(maxn, dtype=torch.int32, device=dev) for _ in range(world)]
        sc["all_rows"] = [torch.empty((maxn, S), dtype=torch.float32, device=dev) for _ in range(world)]
    ids, packed = sc["ids"][:maxn], sc["rows"][:maxn]
    ids.fill_(-1)
    ids[:rows.numel()].copy_(rows)
    fold.gather_rows(dE, ids, packed)
    all_ids = [x[:maxn] for x in sc["all_ids"]]
    all_rows = [x[:maxn] for x in sc["all_rows"]]
    dist.all_gather(all_ids, ids, group=group)
    dist.all_gather(all_rows, packed, group=group)
    dE.zero_()
    for r in range(world):
        fold.scatter_add_rows(all_rows[r], all_ids[r], dE)
    return "sparse"
