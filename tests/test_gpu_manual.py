"""Manual batching (caller-fixed levels, PAPER.md L83 / Table 1) on the CUDA path:
schedules bit-exact with the oracle, status codes identical, forward/backward within the
north_star tolerances. The executor runs these schedules unchanged: one row per level for
a single tree (the unbatched, node-at-a-time baseline), B rows per level for B trees of
one shape, ragged levels and empty levels for mixed shapes."""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import random_dag, rel_err

pytestmark = pytest.mark.gpu

KEYS = ("depth", "perm", "rank", "gather", "level_off", "group_off", "cons_off", "cons_edge", "leaf_perm",
        "tok_seg", "root_row", "root_perm")
TOL = {"fp32": 1e-5, "bf16": 1e-2}


def _dev(gr, level):
    import torch
    from paper_1702_02181_b200 import fold
    op, child, token, root = fold.graphs_to_device(gr)
    lv = torch.tensor(np.asarray(level, np.int32), device="cuda")
    return op, child, token, root, lv


def _compare_sched(gr, level):
    import torch
    from paper_1702_02181_b200 import fold
    ref = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab, level=level)
    op, child, token, root, lv = _dev(gr, level)
    s = fold.schedule(op, child, token, root, gr.vocab, level=lv)
    torch.cuda.synchronize()
    got = s.to_numpy()
    for k in KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    for k in ("n_levels", "n_leaves", "n_cells", "n_tok_segs"):
        assert got[k] == ref[k], k
    return ref


@pytest.mark.parametrize("B,same", [(1, True), (3, True), (64, True), (9, False), (1024, True), (512, False)])
def test_manual_schedule_bit_exact(B, same):
    gr = foldgen.table1_batch(B, same)
    _compare_sched(gr, foldgen.manual_levels(gr))


def test_manual_schedule_shuffled_and_gaps():
    """Arbitrary node order, DAG sharing, and levels with gaps: level = 3 depth - k,
    k in {0, 1, 2} (still above every child's level, at most 3 depth)."""
    rng = np.random.default_rng(8)
    done = 0
    while done < 10:
        gr = random_dag(rng, int(rng.integers(20, 400)), 7)
        gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
        d = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)["depth"]
        level = np.where(gr.op == 0, 1, 3 * d - rng.integers(0, 3, gr.n_nodes)).astype(np.int32)
        if level.max() > gr.n_nodes:
            continue
        _compare_sched(gr, level)
        done += 1


@pytest.mark.parametrize("case,status,node", [
    (dict(level=[1, 1, 1], root=[2]), "LEVEL", 2),
    (dict(level=[2, 1, 3], root=[2]), "LEVEL", 0),
    (dict(level=[1, 1, 4], root=[2]), "LEVEL", 2),
    (dict(level=[1, 1, 0], root=[2]), "LEVEL", 2),
    (dict(level=[2, 1, 3], root=[5]), "ROOT_RANGE", 0),
])
def test_level_errors_match_oracle(case, status, node):
    from paper_1702_02181_b200 import fold
    op, child, token = [0, 0, 1], [[-1, -1], [-1, -1], [0, 1]], [0, 0, 0]
    with pytest.raises(oracle.OracleError) as eo:
        oracle.schedule(op, child, token, case["root"], 4, level=case["level"])
    gr = foldgen.Graphs(np.asarray(op, np.int32), np.asarray(child, np.int32), np.asarray(token, np.int32),
                        np.asarray(case["root"], np.int32), 4, np.asarray([3]))
    op_d, child_d, token_d, root_d, lv = _dev(gr, case["level"])
    with pytest.raises(fold.FoldError) as eg:
        fold.schedule(op_d, child_d, token_d, root_d, 4, level=lv)
    assert eg.value.status == eo.value.status == status
    assert eg.value.detail == eo.value.node == node


def _fwd_bwd(gr, level, cell, prec, S):
    import torch
    from paper_1702_02181_b200 import fold
    p = foldgen.make_params(cell, S, gr.vocab)
    g = foldgen.make_upstream(gr.n_graphs, S)
    model = fold.Model(torch.tensor(p.U, device="cuda"), torch.tensor(p.b, device="cuda"),
                       torch.tensor(p.E, device="cuda"), cell=cell, prec=prec)
    op, child, token, root, lv = _dev(gr, level)
    s = fold.schedule(op, child, token, root, gr.vocab, level=lv)
    h, c, acts = fold.forward(s, model)
    dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device="cuda"))
    torch.cuda.synchronize()
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    rU, rb, rE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    errs = {"h": rel_err(h.cpu().numpy(), hr), "dU": rel_err(dU.cpu().numpy(), rU),
            "db": rel_err(db.cpu().numpy(), rb), "dE": rel_err(dE.cpu().numpy(), rE)}
    if cell == "treelstm":
        errs["c"] = rel_err(c.cpu().numpy(), cr)
    for k, e in errs.items():
        assert e <= TOL[prec], (k, e)
    return errs


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("B,same", [(1, True), (5, True), (7, False)])
def test_manual_fwd_bwd_parity(prec, B, same):
    gr = foldgen.table1_batch(B, same, leaves=24, vocab=64)
    _fwd_bwd(gr, foldgen.manual_levels(gr), "treelstm", prec, 96)


def test_manual_treernn_and_gaps_bf16():
    gr = foldgen.table1_batch(4, False, leaves=17, vocab=32)
    lv = foldgen.manual_levels(gr)
    lv = np.where(lv > 1, 2 * lv, 1).astype(np.int32)  # every other level empty
    _fwd_bwd(gr, lv, "treernn", "bf16", 64)
    _fwd_bwd(gr, lv, "treelstm", "bf16", 64)


def test_manual_unbatched_full_state():
    """The bench's unbatched baseline: one complete 128-leaf tree at S = 1024, one cell
    per level (127 dependent levels), forward + backward."""
    gr = foldgen.config_c2(1)
    _fwd_bwd(gr, foldgen.manual_levels(gr), "treelstm", "bf16", 1024)


@pytest.mark.parametrize("B,same", [(3, False), (40, True)])
def test_narrow_paths_s512(B, same):
    """S = 512 (the stationary-U narrow kernels of both directions apply: GATES*S/8 is a
    multiple of 64): ragged chunks, random shapes, dynamic and manual schedules."""
    gr = foldgen.table1_batch(B, same, leaves=40, vocab=64)
    import oracle as _o
    d = _o.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)["depth"]
    _fwd_bwd(gr, d.astype(np.int32), "treelstm", "bf16", 512)   # levels = L40 depths
    _fwd_bwd(gr, foldgen.manual_levels(gr), "treelstm", "bf16", 512)
    _fwd_bwd(gr, foldgen.manual_levels(gr), "treernn", "bf16", 512)
