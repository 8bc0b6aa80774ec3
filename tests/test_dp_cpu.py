"""Multi-process (gloo, world size 2) checks of the data-parallel host logic on CPU:
node-balanced contiguous sharding and the summed gradient = full-batch gradient."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import foldgen
import oracle
from paper_1702_02181_b200 import dp


def test_shard_bounds_cover_and_balance():
    rng = np.random.default_rng(0)
    sizes = rng.integers(1, 200, 1000)
    for world in (1, 2, 3, 4, 8):
        b = dp.shard_bounds(sizes, world)
        assert b[0] == 0 and b[-1] == len(sizes) and np.all(np.diff(b) >= 0)
        per = [int(sizes[b[r]:b[r + 1]].sum()) for r in range(world)]
        assert sum(per) == int(sizes.sum())
        assert max(per) - min(per) <= 2 * int(sizes.max())


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    gr = foldgen.config_c3(12, vocab=20)
    S = 6
    p = foldgen.make_params("treelstm", S, gr.vocab)
    g = foldgen.make_upstream(gr.n_graphs, S)
    b = dp.shard_bounds(gr.tree_sizes, world)
    sub = dp.shard(gr, rank, world)
    gs = g[b[rank]:b[rank + 1]]
    dU, db, dE = oracle.backward("treelstm", sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E, gs)
    fp = dp.FlatParams(p.U, p.b, p.E, "cpu")
    fp.dU.copy_(torch.from_numpy(dU)); fp.db.copy_(torch.from_numpy(db)); fp.dE.copy_(torch.from_numpy(dE))
    dp.allreduce_grads(fp.grad)
    if rank == 0:
        out.put(fp.grad.numpy().copy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gradient_allreduce_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = q.get(timeout=120)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    gr = foldgen.config_c3(12, vocab=20)
    S = 6
    p = foldgen.make_params("treelstm", S, gr.vocab)
    g = foldgen.make_upstream(gr.n_graphs, S)
    dU, db, dE = oracle.backward("treelstm", gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    ref = np.concatenate([dU.ravel(), db.ravel(), dE.ravel()]).astype(np.float32)
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-6)


def test_exchange_plan():
    """Sparse dE exchange only when its all-gather moves fewer bytes than the dense ring
    all-reduce; maxn = the largest per-rank row count (the padding)."""
    from paper_1702_02181_b200 import dp
    assert dp.exchange_plan([3000, 5000], 300, 16384, 2) == ("sparse", 5000)
    # C2-like: every token touched -> dense
    assert dp.exchange_plan([16384] * 8, 1024, 16384, 8)[0] == "dense"
    assert dp.exchange_plan([0, 0], 8, 100, 2) == ("sparse", 0)
    # the crossover: world * maxn * (S + 1) vs 2 (world - 1) / world * V * S
    S, V, w = 64, 1000, 4
    lim = 2 * (w - 1) / w * V * S / (w * (S + 1))
    assert dp.exchange_plan([int(lim) - 1], S, V, w)[0] == "sparse"
    assert dp.exchange_plan([int(lim) + 1], S, V, w)[0] == "dense"
