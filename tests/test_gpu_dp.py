"""Data-parallel training step on the CUDA path: two ranks (gloo
process group; one GPU here, so both ranks share cuda:0), each scheduling and running
fold_forward / fold_backward on its node-balanced shard (dp.shard), then one all_reduce of
the flat device gradient [dU | db | dE] (dp.FlatParams / dp.allreduce_grads, the bench's
exchange). The summed gradient must equal the single-rank full-batch gradient of the same
library (fp32 mode: 1e-5, only the summation order differs; bf16: 1e-2) and the fp64 oracle."""
import os
import socket

import numpy as np
import pytest

import foldgen
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu

S = 64


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, prec, q):
    import torch
    import torch.distributed as dist
    from paper_1702_02181_b200 import dp, fold
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    full = foldgen.config_c3(96, vocab=200)
    gfull = foldgen.make_upstream(full.n_graphs, S)
    b = dp.shard_bounds(full.tree_sizes, world)
    sub = dp.shard(full, rank, world)
    p = foldgen.make_params("treelstm", S, full.vocab)
    fp = dp.FlatParams(p.U, p.b, p.E, "cuda")
    model = fold.Model(fp.U, fp.b, fp.E, prec=prec)
    s = fold.schedule(*fold.graphs_to_device(sub, "cuda"), sub.vocab)
    _, _, acts = fold.forward(s, model)
    g = torch.tensor(gfull[b[rank]:b[rank + 1]], device="cuda")
    fold.backward(s, model, acts, g, grads=(fp.dU, fp.db, fp.dE))
    torch.cuda.synchronize()
    dp.allreduce_grads(fp.grad)
    torch.cuda.synchronize()
    if rank == 0:
        q.put((fp.grad.cpu().numpy().copy(), [int(x) for x in b]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("prec,tol", [("fp32", 1e-5), ("bf16", 1e-2)])
def test_two_rank_cuda_step_matches_one_rank(prec, tol):
    import torch
    import torch.multiprocessing as mp
    from paper_1702_02181_b200 import dp, fold
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, prec, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got, bounds = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    assert 0 < bounds[1] < 96  # both ranks had trees
    # one rank, whole batch, same library
    full = foldgen.config_c3(96, vocab=200)
    g = foldgen.make_upstream(full.n_graphs, S)
    p = foldgen.make_params("treelstm", S, full.vocab)
    fp = dp.FlatParams(p.U, p.b, p.E, "cuda")
    model = fold.Model(fp.U, fp.b, fp.E, prec=prec)
    s = fold.schedule(*fold.graphs_to_device(full, "cuda"), full.vocab)
    _, _, acts = fold.forward(s, model)
    fold.backward(s, model, acts, torch.tensor(g, device="cuda"), grads=(fp.dU, fp.db, fp.dE))
    one = fp.grad.cpu().numpy()
    n1, n2 = p.U.size, p.U.size + p.b.size
    for name, sl in (("dU", slice(0, n1)), ("db", slice(n1, n2)), ("dE", slice(n2, None))):
        e = rel_err(got[sl], one[sl])
        assert e <= (1e-5 if prec == "fp32" else 2e-3), (name, e)
    dU, db, dE = oracle.backward("treelstm", full.op, full.child, full.token, full.root, p.U, p.b, p.E, g)
    for name, x, y in (("dU", got[:n1], dU.ravel()), ("db", got[n1:n2], db), ("dE", got[n2:], dE.ravel())):
        e = rel_err(x, y)
        assert e <= tol, (name, e)


def _worker_sparse(rank, world, port, q):
    """Each rank: its shard's backward, then dp.exchange_grads (sparse dE all-gather when it
    moves fewer bytes than the dense all-reduce, forced dense for the comparison)."""
    import torch
    import torch.distributed as dist
    from paper_1702_02181_b200 import dp, fold
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    full = foldgen.config_c3(64)            # Zipf tokens over V = 16384: few touched rows
    gfull = foldgen.make_upstream(full.n_graphs, S)
    b = dp.shard_bounds(full.tree_sizes, world)
    sub = dp.shard(full, rank, world)
    p = foldgen.make_params("treelstm", S, full.vocab)
    out = {}
    for mode in ("auto", "dense"):
        fp = dp.FlatParams(p.U, p.b, p.E, "cuda")
        model = fold.Model(fp.U, fp.b, fp.E, prec="fp32")
        s = fold.schedule(*fold.graphs_to_device(sub, "cuda"), sub.vocab)
        _, _, acts = fold.forward(s, model)
        g = torch.tensor(gfull[b[rank]:b[rank + 1]], device="cuda")
        fold.backward(s, model, acts, g, grads=(fp.dU, fp.db, fp.dE))
        rows = fold.touched_rows(s)
        used = dp.exchange_grads(fp.grad, p.U.size + p.b.size, fp.dE, rows, mode=mode)
        torch.cuda.synchronize()
        out[mode] = (used, fp.grad.cpu().numpy().copy(), int(rows.numel()))
    q.put((rank, out))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sparse_dE_exchange():
    """NEXT-4 sparse dE exchange: the touched rows all-gathered and added in rank order give
    the dense all-reduce's gradient (fp32 rounding order only), bitwise the same on both ranks,
    and the single-rank full-batch gradient within 1e-5; fold_touched_rows = the distinct
    tokens of the rank's leaves."""
    import torch
    import torch.multiprocessing as mp
    from paper_1702_02181_b200 import dp, fold
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sparse, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(2))
    for pr in procs:
        pr.join(timeout=120)
        assert pr.exitcode == 0
    full = foldgen.config_c3(64)
    b = dp.shard_bounds(full.tree_sizes, 2)
    for r in range(2):
        sub = dp.shard(full, r, 2)
        assert res[r]["auto"][2] == len(np.unique(sub.token[sub.op == 0]))
        assert res[r]["auto"][0] == "sparse" and res[r]["dense"][0] == "dense"
    assert np.array_equal(res[0]["auto"][1], res[1]["auto"][1])
    sparse, dense = res[0]["auto"][1], res[0]["dense"][1]
    n2 = None
    p = foldgen.make_params("treelstm", S, full.vocab)
    n2 = p.U.size + p.b.size
    assert rel_err(sparse[n2:], dense[n2:]) <= 1e-6
    assert np.array_equal(sparse[:n2], dense[:n2])
    fp = dp.FlatParams(p.U, p.b, p.E, "cuda")
    model = fold.Model(fp.U, fp.b, fp.E, prec="fp32")
    s = fold.schedule(*fold.graphs_to_device(full, "cuda"), full.vocab)
    _, _, acts = fold.forward(s, model)
    g = foldgen.make_upstream(full.n_graphs, S)
    fold.backward(s, model, acts, torch.tensor(g, device="cuda"), grads=(fp.dU, fp.db, fp.dE))
    one = fp.grad.cpu().numpy()
    assert rel_err(sparse, one) <= 1e-5
    assert 0 < b[1] < 64
