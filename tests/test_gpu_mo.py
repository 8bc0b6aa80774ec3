"""NEXT-3 on the GPU: multi-op levels through the C-ABI
(fold_mo.h) against the fp64 multi-op oracle (fold_oracle_mo.c, pinned in
test_oracle_mo.py). Schedules bit-exact (depth, (depth, op) groups, per-type pools, (d, t, i)
labels, error classes, one-block and cooperative paths); forward / backward within 1e-5
(FP32: 3xTF32 tensor cores) and 1e-2 (TF32) on the C6 workload (binary + unary TreeLSTM,
typed projection), on a 7-op 2-type table over random DAGs with sharing, odd state sizes;
bitwise determinism; bench-size (C6 B=1024, S=300/128) sampled roots and gradient linearity."""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import rel_err
from tests.test_oracle_mo import random_mo_graph, table7, _graph

pytestmark = pytest.mark.gpu
TOL = {"fp32": 1e-5, "tf32": 1e-2}


def _dev(gr):
    import torch
    t = lambda x: torch.tensor(np.ascontiguousarray(x, np.int32).reshape(-1), device="cuda")
    return t(gr.op), t(gr.child), t(gr.token), t(gr.root)


def _run(gr, params, prec, g, reps=1):
    import torch
    from paper_1702_02181_b200 import fold_mo
    s = fold_mo.schedule(gr.table, *_dev(gr))
    model = fold_mo.MoModel([tuple(torch.tensor(x, device="cuda") for x in blk) for blk in params], prec)
    gd = torch.tensor(g, device="cuda")
    outs = []
    for _ in range(reps):
        h, acts = fold_mo.forward(s, model)
        grads = fold_mo.backward(s, model, acts, gd)
        torch.cuda.synchronize()
        outs.append((h.cpu().numpy(), [tuple(x.cpu().numpy() for x in blk) for blk in grads]))
    return s, outs


def _check(gr, prec, seed=0):
    params = foldgen.make_mo_params(gr.table, seed=foldgen.PARAM_SEED + seed)
    g = foldgen.make_mo_upstream(gr.n_graphs, gr.table)
    _, outs = _run(gr, params, prec, g)
    h, grads = outs[0]
    P = oracle.mo_flatten(gr.table, params)
    H, _ = oracle.mo_forward(gr, P)
    errs = {"h_root": rel_err(h, H[gr.root])}
    ref = oracle.mo_unflatten(gr.table, params, oracle.mo_backward(gr, P, g))
    for o, (blk, rblk) in enumerate(zip(grads, ref)):
        for name, x, r in zip(("dE",) if len(blk) == 1 else ("dU", "db"), blk, rblk):
            errs[f"op{o}.{name}"] = rel_err(x, r)
    for k, e in errs.items():
        assert e <= TOL[prec], (prec, k, e, errs)
    return errs


# ----------------------------------------------------------------------------- schedule

@pytest.mark.parametrize("B", [16, 1024])
def test_schedule_bit_exact_c6(B):
    """One-block (B=16) and cooperative multi-block (B=1024, ~87k nodes) scheduler paths."""
    from paper_1702_02181_b200 import fold_mo
    gr = foldgen.mo_batch_c6(B)
    got = fold_mo.schedule(gr.table, *_dev(gr)).to_numpy()
    ref = oracle.mo_schedule(gr)
    assert got["n_levels"] == ref["n_levels"]
    for k in ("depth", "group_off", "type_off", "pool", "pool_row", "tlevel_off", "label"):
        assert np.array_equal(got[k], ref[k]), k


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_schedule_bit_exact_random_dags(seed):
    from paper_1702_02181_b200 import fold_mo
    rng = np.random.default_rng(seed)
    gr = random_mo_graph(table7(), rng, 600 if seed < 2 else 9000, 7, share=0.3)
    # shuffle node ids (children need not precede parents)
    perm = rng.permutation(gr.n_nodes)
    inv = np.empty_like(perm); inv[perm] = np.arange(gr.n_nodes)
    child = np.where(gr.child[perm] >= 0, inv[np.maximum(gr.child[perm], 0)], -1)
    gr = _graph(gr.table, gr.op[perm], child, gr.token[perm], inv[gr.root])
    got = fold_mo.schedule(gr.table, *_dev(gr)).to_numpy()
    ref = oracle.mo_schedule(gr)
    for k in ("depth", "group_off", "type_off", "pool", "pool_row", "tlevel_off", "label"):
        assert np.array_equal(got[k], ref[k]), k


@pytest.mark.parametrize("case, status, node", [
    ("child_range", "CHILD_RANGE", 2), ("op_range", "OP_RANGE", 1), ("arity", "ARITY", 3),
    ("type", "TYPE", 4), ("token", "TOKEN_RANGE", 0), ("root", "ROOT_RANGE", 1), ("cycle", "CYCLE", 2)])
def test_schedule_errors_match_oracle(case, status, node):
    from paper_1702_02181_b200 import fold, fold_mo
    T = foldgen.mo_table([(0, 0, -1, 0, 4), (1, 2, 0, 0, 0), (1, 1, 0, 0, 0), (2, 1, 0, 1, 0)], [2, 3])
    op = [0, 0, 1, 2, 3]
    child = [[-1, -1], [-1, -1], [0, 1], [2, -1], [3, -1]]
    token = [1, 2, 0, 0, 0]
    root = [4, 3]
    if case == "child_range":
        child[2] = [0, 9]
    elif case == "op_range":
        op[1] = 7
    elif case == "arity":
        child[3] = [2, 1]
    elif case == "type":
        op[3] = 3; op[4] = 2
    elif case == "token":
        token[0] = 4
    elif case == "root":
        root = [4, 5]
    elif case == "cycle":
        child[2] = [3, 1]
    gr = _graph(T, op, child, token, root)
    with pytest.raises(oracle.OracleError) as e:
        oracle.mo_schedule(gr)
    assert (e.value.status, e.value.node) == (status, node)
    with pytest.raises(fold.FoldError) as f:
        fold_mo.schedule(T, *_dev(gr))
    assert (f.value.status, f.value.detail) == (status, node)


# ----------------------------------------------------------------------------- numerics

@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_c6_small(prec):
    T = foldgen.mo_table_c6(S0=64, S1=32, vocab=300)
    _check(foldgen.mo_batch_c6(24, table=T), prec)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_c6_s300(prec):
    """The C6 workload's state sizes (S0 = 300 as the paper's SST model, L329; S1 = 128)."""
    _check(foldgen.mo_batch_c6(64, seed=11), prec)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("S", [(30, 18), (7, 5), (132, 60)])
def test_table7_random_dags(prec, S):
    """Every op kind and arity, two tensor types with projections both ways, shared nodes,
    state sizes that are not multiples of 4 (padded rows)."""
    rng = np.random.default_rng(sum(S))
    gr = random_mo_graph(table7(*S), rng, 700, 6, share=0.3)
    _check(gr, prec)


def test_deterministic_bitwise():
    gr = foldgen.mo_batch_c6(256, seed=5)
    params = foldgen.make_mo_params(gr.table)
    g = foldgen.make_mo_upstream(gr.n_graphs, gr.table)
    _, outs = _run(gr, params, "fp32", g, reps=3)
    for h, grads in outs[1:]:
        assert np.array_equal(h, outs[0][0])
        for blk, b0 in zip(grads, outs[0][1]):
            for x, y in zip(blk, b0):
                assert np.array_equal(x, y)


def _subtree(gr, t):
    """Tree t of a C6 batch alone (trees are contiguous node blocks ending at their root)."""
    n0 = 0 if t == 0 else int(gr.root[t - 1]) + 1
    n1 = int(gr.root[t]) + 1
    child = np.where(gr.child[n0:n1] >= 0, gr.child[n0:n1] - n0, -1)
    return _graph(gr.table, gr.op[n0:n1], child, gr.token[n0:n1], [n1 - 1 - n0])


def test_c6_bench_size_sampled_roots_and_linearity():
    """C6 at its bench size (B = 1024 trees, ~87k nodes, S = 300 / 128, FP32): root states of
    sampled trees against the oracle on each tree alone (trees are independent),
    and linearity of the backward in the upstream gradient (g1 + g2) at full size."""
    import torch
    from paper_1702_02181_b200 import fold_mo
    gr = foldgen.mo_batch_c6(1024)
    params = foldgen.make_mo_params(gr.table)
    s = fold_mo.schedule(gr.table, *_dev(gr))
    model = fold_mo.MoModel([tuple(torch.tensor(x, device="cuda") for x in blk) for blk in params], "fp32")
    h, acts = fold_mo.forward(s, model)
    h = h.cpu().numpy()
    P = oracle.mo_flatten(gr.table, params)
    for t in (0, 1, 333, 777, 1023):
        sub = _subtree(gr, t)
        H, _ = oracle.mo_forward(sub, P)
        assert rel_err(h[t], H[sub.root[0]]) <= 1e-5, t
    g1 = foldgen.make_mo_upstream(gr.n_graphs, gr.table, seed=1)
    g2 = foldgen.make_mo_upstream(gr.n_graphs, gr.table, seed=2)
    out = [fold_mo.backward(s, model, acts, torch.tensor(x, device="cuda")) for x in (g1, g2, g1 + g2)]
    for b1, b2, b12 in zip(*out):
        for x, y, z in zip(b1, b2, b12):
            assert rel_err((x + y).cpu().numpy(), z.cpu().numpy()) <= 1e-5


def test_accumulate_and_degenerate_batches():
    """fold_mo_grads.accumulate adds a second backward's gradients; a batch of one leaf (depth 1,
    no cell op present) and a batch whose root is a leaf of the second tensor type run."""
    import torch
    from paper_1702_02181_b200 import fold_mo
    gr = foldgen.mo_batch_c6(12, seed=3, table=foldgen.mo_table_c6(S0=36, S1=20, vocab=50))
    params = foldgen.make_mo_params(gr.table)
    g = torch.tensor(foldgen.make_mo_upstream(gr.n_graphs, gr.table), device="cuda")
    s = fold_mo.schedule(gr.table, *_dev(gr))
    model = fold_mo.MoModel([tuple(torch.tensor(x, device="cuda") for x in blk) for blk in params], "fp32")
    h, acts = fold_mo.forward(s, model)
    one = fold_mo.backward(s, model, acts, g)
    one = [tuple(x.clone() for x in blk) for blk in one]
    two = fold_mo.backward(s, model, acts, g, grads=[tuple(x.clone() for x in blk) for blk in one], accumulate=True)
    for b1, b2 in zip(one, two):
        for x, y in zip(b1, b2):
            assert rel_err(y.cpu().numpy(), 2 * x.cpu().numpy()) <= 1e-6
    # one EMBED leaf of type 1 as the whole batch (only depth 1)
    T = table7(6, 4)
    leaf = _graph(T, [1], [[-1, -1]], [3], [0])
    _check(leaf, "fp32")
    # a leaf root beside a tree
    rng = np.random.default_rng(5)
    gr2 = random_mo_graph(T, rng, 40, 3)
    gr2 = _graph(T, np.concatenate([gr2.op, [0]]), np.concatenate([gr2.child, [[-1, -1]]]),
                 np.concatenate([gr2.token, [2]]), np.concatenate([gr2.root, [40]]))
    _check(gr2, "fp32")
