"""Gradient parity with EVERY tree's upstream gradient live, at bench-like sizes (VERDICT r01
"what's weak" 2: the full-size tests zeroed the gradient of all but a few trees, so >99% of
the dZ rows entering the dU / db reductions were exact zeros).

  * C2 (complete 128-leaf trees, S = 1024) at B = 64, C3 (parse-shaped, S = 300, Zipf
    tokens) at B = 1024 and C4 (depth-256 chains, S = 1024) at B = 16: root h / c and dU, db,
    dE of the whole batch against the fp64 oracle summed over all trees (host thread pool,
    tests/oracle_pool.py), element-wise normwise error <= 1e-2 (BF16 path, north_star).
  * C5 (8192 random 128-leaf trees, S = 1024) and C2 at B = 1024, too large for the oracle:
    the gradient is linear in the upstream gradient g for a fixed forward (the
    backward of the unrolled loop), so the full-batch gradients with all of g live must equal
    the sum of two runs with g split between tree sets A and B (fixed-order fp32 sums of the
    same bf16 products: within 1e-4), and the run with only A live must match the oracle on
    the trees of A (1e-2).
"""
import numpy as np
import pytest

import foldgen
from tests.helpers import rel_err
from tests.oracle_pool import batch_reference

pytestmark = pytest.mark.gpu

TOL = 1e-2


def _gpu(gr, S, gs, prec="bf16", cell="treelstm"):
    """Forward once, then one backward per upstream gradient in `gs` (same activations)."""
    import torch
    from paper_1702_02181_b200 import fold
    p = foldgen.make_params(cell, S, gr.vocab)
    dev = "cuda"
    model = fold.Model(*(torch.tensor(x, device=dev) for x in (p.U, p.b, p.E)), cell=cell, prec=prec)
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    ws = fold.Workspace(dev)
    h, c, acts = fold.forward(s, model, ws=ws)
    outs = []
    for g in gs:
        dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device=dev), ws=ws)
        outs.append(tuple(t.cpu().numpy() for t in (dU, db, dE)))
    res = (h.cpu().numpy(), c.cpu().numpy(), outs, p)
    del acts, ws, s
    torch.cuda.empty_cache()
    return res


def _full_check(gr, S):
    g = foldgen.make_upstream(gr.n_graphs, S)
    h, c, outs, p = _gpu(gr, S, [g])
    rh, rc, rU, rb, rE = batch_reference(gr, p, g)
    errs = {"h": rel_err(h, rh), "c": rel_err(c, rc)}
    for k, x, y in zip(("dU", "db", "dE"), outs[0], (rU, rb, rE)):
        errs[k] = rel_err(x, y)
    for k, e in errs.items():
        assert e <= TOL, (k, e, errs)
    return errs


def test_c2_all_gradients_live_b64():
    """configs[1] shape, 64 complete 128-leaf trees (8128 cells: 32 row tiles at the widest
    level, the top levels in the narrow kernels), every tree's g nonzero."""
    _full_check(foldgen.config_c2(64), 1024)


def test_c3_all_gradients_live_b1024():
    """configs[2] at its full batch: 1024 parse-shaped trees, S = 300 (K and N not multiples
    of 64: TMA zero fill), Zipf tokens (long dE segments), every tree's g nonzero."""
    _full_check(foldgen.config_c3(1024), 300)


def test_c4_all_gradients_live_b16():
    """configs[3] shape: 16 chains of 256 leaves, 255 dependent cell levels (narrow and
    wide backward kernels, dCe carried through 255 levels), every chain's g nonzero."""
    _full_check(foldgen.config_c4(16), 1024)


@pytest.mark.parametrize("S", [33, 130])
def test_bf16_odd_state_split_k(S):
    """~5k cells at an odd / non-multiple-of-4 state size in BF16 (the split-K
    reduction of dU / db must not assume gates*S % 4 == 0 or aligned slabs)."""
    rng = np.random.default_rng(5000 + S)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(2, 60))) for _ in range(170)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 300), 300)
    assert 4000 < (gr.op == foldgen.CELL).sum() < 7000
    _full_check(gr, S)


def _linearity(gr, S, sample):
    G = gr.n_graphs
    g = foldgen.make_upstream(G, S)
    mask = np.zeros(G, bool)
    mask[sample] = True
    gA = np.where(mask[:, None], g, 0.0).astype(np.float32)
    gB = np.where(mask[:, None], 0.0, g).astype(np.float32)
    h, c, outs, p = _gpu(gr, S, [g, gA, gB])
    full, A, B = outs
    for k, x, a, b in zip(("dU", "db", "dE"), full, A, B):
        e = rel_err(x, a.astype(np.float64) + b)
        assert e <= 1e-4, (k, e)
    rh, rc, rU, rb, rE = batch_reference(gr, p, g, trees=sample)
    assert rel_err(h[sample], rh) <= TOL
    assert rel_err(c[sample], rc) <= TOL
    for k, x, y in zip(("dU", "db", "dE"), A, (rU, rb, rE)):
        e = rel_err(x, y)
        assert e <= TOL, (k, e)


def test_c2_b1024_linearity_all_live():
    """The bench configuration (C2, B = 1024, S = 1024): all 1024 trees' gradients live."""
    _linearity(foldgen.config_c2(1024), 1024, [0, 1, 511, 1023])


def test_c5_8192_linearity_all_live():
    """configs[4] on one GPU (2.09 M nodes): all 8192 trees' gradients live."""
    _linearity(foldgen.config_c5(8192), 1024, [3, 4096, 8191])
