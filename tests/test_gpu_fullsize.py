"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(BF16, TreeLSTM, whole batch in one fold_schedule/forward/backward call), on outputs the
oracle can compute one tree at a time:
  * root h / c of sampled trees (trees are independent: PAPER.md L37, L86);
  * gradients with the upstream gradient nonzero only for the sampled trees, so the
    full-batch dU / db / dE must equal the oracle's gradients of those trees alone
    (the other trees contribute exactly zero: every dz of theirs is 0).
Tolerance 1e-2 normwise (north_star, BF16 path)."""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _run_full(gr, S, samples, cell="treelstm"):
    import torch
    from paper_1702_02181_b200 import fold
    p = foldgen.make_params(cell, S, gr.vocab)
    dev = "cuda"
    model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev),
                       cell=cell, prec="bf16")
    op, child, token, root = fold.graphs_to_device(gr)
    s = fold.schedule(op, child, token, root, gr.vocab)
    h, c, acts = fold.forward(s, model)
    g = np.zeros((gr.n_graphs, S), np.float32)
    gfull = foldgen.make_upstream(gr.n_graphs, S)
    g[samples] = gfull[samples]
    dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device=dev))
    torch.cuda.synchronize()
    out = dict(h=h[samples].cpu().numpy(), c=c[samples].cpu().numpy(), dU=dU.cpu().numpy(), db=db.cpu().numpy(),
               dE=dE.cpu().numpy())
    del acts, h, c, dU, db, dE, s
    torch.cuda.empty_cache()
    return out, p, g


def _check(gr, S, samples, check_grads=True):
    got, p, g = _run_full(gr, S, samples)
    sub_h, sub_c = [], []
    dU = db = dE = None
    for t in samples:
        one = foldgen.sub_batch(gr, t, t + 1)
        h, c = oracle.forward("treelstm", one.op, one.child, one.token, one.root, p.U, p.b, p.E)
        sub_h.append(h[0]); sub_c.append(c[0])
        if check_grads:
            gU, gb, gE = oracle.backward("treelstm", one.op, one.child, one.token, one.root, p.U, p.b, p.E, g[t:t + 1])
            dU = gU if dU is None else dU + gU
            db = gb if db is None else db + gb
            dE = gE if dE is None else dE + gE
    assert rel_err(got["h"], np.stack(sub_h)) <= 1e-2
    assert rel_err(got["c"], np.stack(sub_c)) <= 1e-2
    if check_grads:
        for k, ref in (("dU", dU), ("db", db), ("dE", dE)):
            e = rel_err(got[k], ref)
            assert e <= 1e-2, (k, e)


def test_c2_full_batch_1024():
    """configs[1] at the bench size: 1024 complete 128-leaf trees, S = 1024."""
    gr = foldgen.config_c2(1024)
    _check(gr, 1024, [0, 1023], check_grads=True)


def test_c3_full_batch_1024():
    """configs[2]: 1024 parse-shaped trees, S = 300, Zipf tokens."""
    gr = foldgen.config_c3(1024)
    _check(gr, 300, [0, 17, 511, 1023], check_grads=True)


def test_c4_full_batch_chains():
    """configs[3]: depth-256 chains, one row per level per chain, 1024 chains, S = 1024."""
    gr = foldgen.config_c4(1024)
    _check(gr, 1024, [5, 1000], check_grads=False)


def test_c5_8192_trees_one_gpu():
    """configs[4] on one GPU: 8192 random 128-leaf trees (2.09 M nodes), S = 1024."""
    gr = foldgen.config_c5(8192)
    _check(gr, 1024, [3, 8191], check_grads=False)
