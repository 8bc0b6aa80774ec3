"""Pins for the oracle's schedule (CPU only). Each test cites what fixes the expected
value independently of the oracle: the paper's worked example, closed forms, brute
force on tiny inputs, or invariants stated by the paper (§2)."""
import itertools
import json
import os

import numpy as np
import pytest

import foldgen
import oracle
from oracle import paper_form

HERE = os.path.dirname(os.path.abspath(__file__))


def _fig1():
    with open(os.path.join(HERE, "golden", "fig1.json")) as f:
        return json.load(f)


def test_fig1_executor_form():
    """PAPER.md L58-77 Fig. 1 worked example; values hand-derived from L40-44."""
    g = _fig1()
    s = oracle.schedule(g["op"], g["child"], g["token"], g["root"], g["vocab"])
    exp = g["executor_form"]
    for k in ("depth", "perm", "rank", "level_off", "group_off", "cons_off", "cons_edge",
              "leaf_perm", "tok_seg", "root_row"):
        assert s[k].tolist() == exp[k], k
    assert s["gather"].tolist() == exp["gather"]
    assert (s["n_levels"], s["n_leaves"], s["n_cells"]) == (exp["n_levels"], exp["n_leaves"], exp["n_cells"])


def test_fig1_paper_form():
    """Fig. 1 with pass-throughs: 'The long downward arrows are the pass-throughs' (L55);
    one pass-through for embed(w5) at depth 2; labels (d,t,i) per L44."""
    g = _fig1()
    ps = paper_form.schedule(g["op"], g["child"], g["token"], g["root"])
    assert paper_form.dump(ps).split("\n") == g["paper_form_dump"]
    assert ps["n_pass"] == g["n_pass"]


def test_four_leaf_complete():
    """4-leaf complete tree, post-order ids."""
    o, l, r = foldgen.complete_shape(4)
    child = np.stack([l, r], 1)
    s = oracle.schedule(o, child, np.zeros(7, np.int32), [6], 1)
    assert s["depth"].tolist() == [1, 1, 2, 1, 1, 2, 3]
    assert s["perm"].tolist() == [0, 1, 3, 4, 2, 5, 6]
    assert s["gather"][4:].tolist() == [[0, 1], [2, 3], [4, 5]]


@pytest.mark.parametrize("k", [0, 1, 2, 3, 5, 7])
@pytest.mark.parametrize("B", [1, 3])
def test_complete_tree_levels(k, B):
    """PAPER.md L123 'invokes it once for each depth, so the number of kernel invocations
    is log(n)': 2^k leaves -> k cell levels + 1 embed level; widths B*2^(k-j)."""
    gr = foldgen.replicate_shape(foldgen.complete_shape(2 ** k), B, lambda n: np.zeros(n), 1)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 1)
    assert s["n_levels"] == k + 1
    widths = np.diff(s["level_off"][1:]).tolist()
    assert widths == [B * 2 ** (k - j) for j in range(k + 1)]
    # one group per level (a single op per depth in these trees)
    go = s["group_off"]
    nonempty = sum(1 for i in range(len(go) - 1) if go[i + 1] > go[i])
    assert nonempty == k + 1


@pytest.mark.parametrize("L", [2, 3, 8, 40])
def test_chain_levels_and_passthroughs(L):
    """Fold chain: every depth >= 2 has exactly B rows; the paper form
    needs sum_{k=2}^{L-1} (k-1) = (L-1)(L-2)/2 pass-throughs per chain (L41)."""
    B = 3
    gr = foldgen.replicate_shape(foldgen.caterpillar_shape(L), B, lambda n: np.arange(n) % 5, 5)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 5)
    assert s["n_levels"] == L
    widths = np.diff(s["level_off"][1:]).tolist()
    assert widths[0] == B * L and all(w == B for w in widths[1:])
    one = foldgen.sub_batch(gr, 0, 1)
    ps = paper_form.schedule(one.op, one.child, one.token, one.root)
    assert ps["n_pass"] == (L - 1) * (L - 2) // 2


# ---------------------------------------------------------------- brute force

def _all_shapes(n):
    """All binary tree shapes with n leaves as nested tuples (Catalan(n-1) many)."""
    if n == 1:
        return ["x"]
    out = []
    for s in range(1, n):
        for a in _all_shapes(s):
            for b in _all_shapes(n - s):
                out.append((a, b))
    return out


def _emit(shape, op, child):
    if shape == "x":
        op.append(0); child.append([-1, -1]); return len(op) - 1
    a = _emit(shape[0], op, child)
    b = _emit(shape[1], op, child)
    op.append(1); child.append([a, b]); return len(op) - 1


def _brute_schedule(op, child, token, root, V):
    """Definition written out independently: depth by fixed-point iteration of
    PAPER.md L40, order by O(N^2) selection of the smallest (depth, op, id) (L42-43),
    gather by definition (L44)."""
    N = len(op)
    depth = [0] * N
    for _ in range(N + 1):
        for n in range(N):
            depth[n] = 1 if op[n] == 0 else 1 + max(depth[child[n][0]], depth[child[n][1]])
    remaining = list(range(N))
    perm = []
    while remaining:
        best = min(remaining, key=lambda n: (depth[n], op[n], n))
        perm.append(best); remaining.remove(best)
    rank = [0] * N
    for r, n in enumerate(perm):
        rank[n] = r
    gather = [[rank[child[n][0]], rank[child[n][1]]] if op[n] == 1 else [-1, -1] for n in perm]
    D = max(depth) if N else 0
    level_off = [sum(1 for n in range(N) if depth[n] < d) for d in range(D + 2)]
    return depth, perm, rank, gather, level_off


@pytest.mark.parametrize("leaves", [1, 2, 3, 4, 5, 6, 7])
def test_brute_force_all_shapes(leaves):
    shapes = _all_shapes(leaves)
    rng = np.random.default_rng(leaves)
    catalan = [1, 1, 2, 5, 14, 42, 132]
    assert len(shapes) == catalan[leaves - 1]
    for shape in shapes:
        op, child = [], []
        _emit(shape, op, child)
        N = len(op)
        token = [int(t) for t in rng.integers(0, 4, N)]
        for numbering in range(3):
            if numbering == 0:
                p = np.arange(N)
            elif numbering == 1:
                p = np.arange(N)[::-1].copy()
            else:
                p = rng.permutation(N)
            gr = foldgen.permute_nodes(foldgen.Graphs(np.asarray(op, np.int32), np.asarray(child, np.int32),
                                                      np.asarray(token, np.int32), np.asarray([N - 1], np.int32),
                                                      4, np.asarray([N], np.int32)), p)
            s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 4)
            depth, perm, rank, gather, lo = _brute_schedule(gr.op.tolist(), gr.child.tolist(),
                                                            gr.token.tolist(), gr.root.tolist(), 4)
            assert s["depth"].tolist() == depth
            assert s["perm"].tolist() == perm
            assert s["rank"].tolist() == rank
            assert s["gather"].tolist() == gather
            assert s["level_off"].tolist() == lo


def test_batch_of_small_shapes_brute_force():
    """Batches (disconnected graphs) of random small shapes, shuffled ids."""
    rng = np.random.default_rng(7)
    for trial in range(40):
        shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 8))) for _ in range(int(rng.integers(1, 6)))]
        gr = foldgen.batch_from_shapes(shapes, lambda n: rng.integers(0, 6, n), 6)
        gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
        s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 6)
        depth, perm, rank, gather, lo = _brute_schedule(gr.op.tolist(), gr.child.tolist(),
                                                        gr.token.tolist(), gr.root.tolist(), 6)
        assert s["perm"].tolist() == perm and s["gather"].tolist() == gather
        assert s["level_off"].tolist() == lo


def test_merged_identical_trees():
    """two identical trees merged -> each level's rows are the single-tree
    rows, then the second tree's rows offset by the first tree's level widths."""
    rng = np.random.default_rng(3)
    sh = foldgen.random_split_shape(rng, 9)
    one = foldgen.batch_from_shapes([sh], lambda n: np.arange(n) % 3, 3)
    two = foldgen.batch_from_shapes([sh, sh], lambda n: np.arange(n) % 3, 3)
    s1 = oracle.schedule(one.op, one.child, one.token, one.root, 3)
    s2 = oracle.schedule(two.op, two.child, two.token, two.root, 3)
    n = one.n_nodes
    lo1 = s1["level_off"]
    w = np.diff(lo1)
    assert (s2["level_off"] == 2 * lo1).all()
    for d in range(1, s1["n_levels"] + 1):
        rows1 = s1["perm"][lo1[d]:lo1[d + 1]]
        rows2 = s2["perm"][2 * lo1[d]:2 * lo1[d + 1]]
        assert rows2.tolist() == rows1.tolist() + (rows1 + n).tolist()
        # gathers of the second copy = first copy's, shifted by the child level's width
        g1 = s1["gather"][lo1[d]:lo1[d + 1]]
        g2 = s2["gather"][2 * lo1[d]:2 * lo1[d + 1]]
        if d >= 2:
            def shift(gather_rows, copy):
                out = []
                for row in gather_rows:
                    r2 = []
                    for x in row:
                        dd = int(np.searchsorted(lo1, x, side="right")) - 1  # depth of child
                        r2.append(2 * lo1[dd] + (x - lo1[dd]) + copy * w[dd])
                    out.append(r2)
                return out
            assert g2.tolist() == shift(g1, 0) + shift(g1, 1)


def _random_dag(rng, N, V, p_share=0.3):
    """Random DAG in id order (children have smaller ids), with sharing and L==R."""
    op = np.zeros(N, np.int32)
    child = np.full((N, 2), -1, np.int32)
    token = np.zeros(N, np.int32)
    for n in range(N):
        if n < 2 or rng.random() < 0.35:
            op[n] = 0; token[n] = rng.integers(0, V)
        else:
            op[n] = 1
            a = rng.integers(0, n)
            b = a if rng.random() < 0.1 else rng.integers(0, n)
            child[n] = (a, b)
    G = int(rng.integers(1, 4))
    root = rng.integers(0, N, G).astype(np.int32)
    return op, child, token, root


def test_invariants_random_dags():
    """SPEC S:L431-437 invariants on many random DAGs: every edge spans >= 1 depth,
    each node in exactly one group, 0 <= gather < level_off[depth(parent)], consumer
    CSR = transpose of gather (gather/scatter adjoint S:L81), leaves sorted by (token,row),
    determinism."""
    rng = np.random.default_rng(11)
    for _ in range(300):
        N = int(rng.integers(1, 40)); V = 5
        op, child, token, root = _random_dag(rng, N, V)
        p = rng.permutation(N)
        gr = foldgen.permute_nodes(foldgen.Graphs(op, child, token, root, V, np.asarray([N])), p)
        s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, V)
        s2 = oracle.schedule(gr.op, gr.child, gr.token, gr.root, V)
        for k in s:
            if isinstance(s[k], np.ndarray):
                assert (s[k] == s2[k]).all()
        depth, perm, rank = s["depth"], s["perm"], s["rank"]
        assert sorted(perm.tolist()) == list(range(N))
        lo = s["level_off"]
        nl = s["n_leaves"]
        for r in range(N):
            n = perm[r]
            assert lo[depth[n]] <= r < lo[depth[n] + 1]
            if gr.op[n] == 1:
                for k in range(2):
                    c = gr.child[n][k]
                    assert depth[c] < depth[n]
                    assert 0 <= s["gather"][r][k] < lo[depth[n]]
                    assert s["gather"][r][k] == rank[c]
        # CSR is the transpose of gather: adjoint identity with random vectors
        x = rng.standard_normal(N); y = rng.standard_normal(2 * s["n_cells"])
        lhs = sum(x[s["gather"][nl + c][k]] * y[2 * c + k] for c in range(s["n_cells"]) for k in range(2))
        co, ce = s["cons_off"], s["cons_edge"]
        rhs = sum(x[r] * sum(y[e] for e in ce[co[r]:co[r + 1]]) for r in range(N))
        assert abs(lhs - rhs) < 1e-9
        for r in range(N):
            assert list(ce[co[r]:co[r + 1]]) == sorted(ce[co[r]:co[r + 1]])
        # leaves by (token, row)
        lp = s["leaf_perm"]
        keys = [(gr.token[perm[r]], r) for r in lp]
        assert keys == sorted(keys) and sorted(lp.tolist()) == list(range(nl))
        ts = s["tok_seg"]
        for i in range(s["n_tok_segs"]):
            toks = {gr.token[perm[r]] for r in lp[ts[i]:ts[i + 1]]}
            assert len(toks) == 1
        assert (s["root_row"] == rank[gr.root]).all()
        rp = s["root_perm"]
        assert [(s["root_row"][g], g) for g in rp] == sorted((s["root_row"][g], g) for g in range(len(gr.root)))


def test_empty_and_single_leaf():
    s = oracle.schedule(np.zeros(0), np.zeros((0, 2)), np.zeros(0), np.zeros(0), 1)
    assert s["n_levels"] == 0 and s["level_off"].tolist() == [0, 0]
    s = oracle.schedule([0], [[-1, -1]], [2], [0], 3)
    assert s["n_levels"] == 1 and s["perm"].tolist() == [0] and s["level_off"].tolist() == [0, 0, 1]


@pytest.mark.parametrize("case,status,node", [
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, 5], [0, 1]], token=[0, 0, 0], root=[2]), "CHILD_RANGE", 1),
    (dict(op=[0, 2, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 0, 0], root=[2]), "OP_RANGE", 1),
    (dict(op=[0, 0, 1, 1], child=[[-1, -1], [-1, -1], [0, -1], [0, 1]], token=[0, 0, 0, 0], root=[3]), "ARITY", 2),
    (dict(op=[0, 1], child=[[0, -1], [0, 0]], token=[0, 0], root=[1]), "ARITY", 0),
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 9, 0], root=[2]), "TOKEN_RANGE", 1),
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 0, 0], root=[2, 3]), "ROOT_RANGE", 1),
    (dict(op=[0, 1, 1, 1], child=[[-1, -1], [0, 2], [1, 0], [0, 0]], token=[0, 0, 0, 0], root=[3]), "CYCLE", 1),
    (dict(op=[0, 1, 1], child=[[-1, -1], [0, 2], [0, 1]], token=[0, 0, 0], root=[0]), "CYCLE", 1),
    (dict(op=[0, 1], child=[[-1, -1], [1, 0]], token=[0, 0], root=[0]), "CYCLE", 1),
])
def test_errors(case, status, node):
    """Error classes in order CHILD_RANGE, OP_RANGE, ARITY, TOKEN_RANGE, ROOT_RANGE,
    CYCLE; smallest offending id (reading R21)."""
    with pytest.raises(oracle.OracleError) as ei:
        oracle.schedule(case["op"], case["child"], case["token"], case["root"], 4)
    assert ei.value.status == status and ei.value.node == node


def test_config_shapes():
    """Recipe sanity (DESIGN.md Inputs): C2 complete-128 has 255 nodes/tree, D=8; C4 has
    depth 256; C3 depth distribution is parse-skewed."""
    gr = foldgen.config_c2(2)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    assert gr.n_nodes == 510 and s["n_levels"] == 8
    gr = foldgen.config_c4(1)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    assert s["n_levels"] == 256
    gr = foldgen.config_c3(256)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    assert 20 <= s["n_levels"] <= 45
