"""Pins for the multi-op oracle (fold_oracle_mo.c):
a hand-computed (d, t, i) schedule (tests/golden/mo_schedule.json), schedule invariants on
random multi-op DAGs, error classes, reduction of the 2-op table to the pinned single-op
oracle (TreeLSTM and TreeRNN: schedule, forward, backward), closed forms (constant-gate
unary chains, a typed projection at U = 0 and its exact gradient), and central finite
differences on every parameter of a 7-op, 2-type table with shared nodes."""
import json
import os

import numpy as np
import pytest

import foldgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
EMB, LSTM, RNN = foldgen.MO_EMBED, foldgen.MO_LSTM, foldgen.MO_RNN


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


def _graph(table, op, child, token, root):
    return foldgen.MoGraphs(np.asarray(op, np.int32), np.asarray(child, np.int32).reshape(-1, 2),
                            np.asarray(token, np.int32), np.asarray(root, np.int32), table)


def random_mo_graph(table, rng, n_nodes, n_graphs, share=0.2):
    """Random multi-op DAG for any table: nodes are created bottom-up; an op is drawn among
    those whose input type has enough earlier nodes; children are recent nodes of the input
    type (with probability `share` an already-consumed node: a DAG with shared nodes).
    Roots: the last n_graphs nodes."""
    op, child, token = [], [], []
    by_type = {t: [] for t in range(table.n_types)}
    used = set()
    for n in range(n_nodes):
        cands = [o for o in range(table.n_ops) if table.kind[o] == EMB
                 or len(by_type[int(table.in_type[o])]) >= int(table.arity[o])]
        emb = [o for o in cands if table.kind[o] == EMB]
        inner = [o for o in cands if table.kind[o] != EMB]
        o = int(rng.choice(inner if inner and rng.random() < 0.6 else (emb or inner)))
        kids = [-1, -1]
        if table.kind[o] != EMB:
            pool = by_type[int(table.in_type[o])]
            fresh = [x for x in pool if x not in used]
            for k in range(int(table.arity[o])):
                src = pool if (rng.random() < share or not fresh) else fresh
                c = int(src[-1 - int(rng.integers(0, min(len(src), 6)))])
                kids[k] = c
                used.add(c)
                if c in fresh:
                    fresh.remove(c)
        op.append(o)
        child.append(kids)
        token.append(int(rng.integers(0, int(table.vocab[o]))) if table.kind[o] == EMB else 0)
        by_type[int(table.out_type[o])].append(n)
    root = list(range(n_nodes - n_graphs, n_nodes))
    return _graph(table, op, child, token, root)


def table7(S0=3, S1=2):
    """Every kind and arity, two tensor types, typed projections both ways."""
    return foldgen.mo_table([(EMB, 0, -1, 0, 9), (EMB, 0, -1, 1, 6), (LSTM, 2, 0, 0, 0), (LSTM, 1, 0, 0, 0),
                             (RNN, 2, 0, 1, 0), (LSTM, 1, 1, 1, 0), (RNN, 1, 1, 0, 0)], [S0, S1])


# ----------------------------------------------------------------------------- schedule

def test_golden_hand_computed_schedule():
    fx = json.load(open(os.path.join(HERE, "golden", "mo_schedule.json")))
    t = fx["table"]
    T = foldgen.mo_table(list(zip(t["kind"], t["arity"], t["in_type"], t["out_type"], t["vocab"])), t["S"])
    s = oracle.mo_schedule(_graph(T, fx["op"], fx["child"], fx["token"], fx["root"]))
    for k in ("depth", "group_off", "type_off", "pool", "pool_row"):
        assert s[k].tolist() == fx[k], k
    assert s["n_levels"] == fx["n_levels"]
    assert s["tlevel_off"].tolist() == fx["tlevel_off"]
    for n in range(len(fx["op"])):
        want = fx["label"].get(str(n), [[-1, -1, -1], [-1, -1, -1]])
        assert s["label"][n].tolist() == want, n


@pytest.mark.parametrize("seed", range(6))
def test_schedule_invariants_random(seed):
    """Depth = 1 + max child depth (L40); groups are the (depth, op) counts (L42); each type
    pool is ordered by (depth, op enumeration, id) (L43); labels decode to the child (L44)."""
    rng = np.random.default_rng(seed)
    T = table7()
    gr = random_mo_graph(T, rng, 80, 5)
    s = oracle.mo_schedule(gr)
    d = s["depth"]
    for n in range(gr.n_nodes):
        kids = [c for c in gr.child[n] if c >= 0]
        assert d[n] == 1 + (max(d[c] for c in kids) if kids else 0)
    D, K = s["n_levels"], T.n_ops
    cnt = np.bincount(d * K + gr.op, minlength=(D + 1) * K)
    assert np.array_equal(np.diff(s["group_off"]), cnt)
    for t in range(T.n_types):
        nodes = s["pool"][s["type_off"][t]:s["type_off"][t + 1]]
        assert all(T.out_type[gr.op[n]] == t for n in nodes)
        keys = [(d[n], gr.op[n], n) for n in nodes]
        assert keys == sorted(keys)
        assert len(nodes) == np.sum(T.out_type[gr.op] == t)
        for dd in range(D + 2):
            assert s["tlevel_off"][t, dd] == sum(1 for n in nodes if d[n] < dd)
        for r, n in enumerate(nodes):
            assert s["pool_row"][n] == r
    for n in range(gr.n_nodes):
        for k in range(2):
            c = gr.child[n, k]
            lab = s["label"][n, k]
            if c < 0:
                assert lab.tolist() == [-1, -1, -1]
                continue
            dd, t, i = lab
            assert dd == d[c] and t == T.out_type[gr.op[c]]
            assert s["pool"][s["type_off"][t] + s["tlevel_off"][t, dd] + i] == c


def test_two_op_table_matches_single_op_schedule():
    """EMBED + binary cell as a 2-op table: depths and (depth, op) groups equal the pinned
    single-op oracle's (its key is 2*depth + op)."""
    gr = foldgen.config_c3(24)
    T = foldgen.mo_table([(EMB, 0, -1, 0, gr.vocab), (LSTM, 2, 0, 0, 0)], [4])
    m = oracle.mo_schedule(_graph(T, gr.op, gr.child, gr.token, gr.root))
    r = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    assert np.array_equal(m["depth"], r["depth"])
    assert np.array_equal(m["group_off"], r["group_off"])
    assert np.array_equal(m["pool"], r["perm"])


@pytest.mark.parametrize("case, status, node", [
    ("child_range", "CHILD_RANGE", 2), ("op_range", "OP_RANGE", 1), ("arity", "ARITY", 3),
    ("type", "TYPE", 4), ("token", "TOKEN_RANGE", 0), ("root", "ROOT_RANGE", 1), ("cycle", "CYCLE", 2)])
def test_error_classes(case, status, node):
    T = foldgen.mo_table([(EMB, 0, -1, 0, 4), (LSTM, 2, 0, 0, 0), (LSTM, 1, 0, 0, 0), (RNN, 1, 0, 1, 0)], [2, 3])
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
        op[3] = 3                 # n3 = projection of n2 into type 1 ...
        op[4] = 2                 # ... consumed by n4, a type-0 unary LSTM: TYPE at node 4
    elif case == "token":
        token[0] = 4
    elif case == "root":
        root = [4, 5]
    elif case == "cycle":
        child[2] = [3, 1]    # n2 <- n3 <- n2
    gr = _graph(T, op, child, token, root)
    with pytest.raises(oracle.OracleError) as e:
        oracle.mo_schedule(gr)
    assert e.value.status == status
    assert e.value.node == node


# ----------------------------------------------------------------------------- reductions

@pytest.mark.parametrize("cell, kind", [("treelstm", LSTM), ("treernn", RNN)])
def test_two_op_table_equals_single_op_oracle(cell, kind):
    """A 2-op table (EMBED, binary cell) computes exactly what the pinned single-op oracle
    does (Fig. 1 / FD / closed-form pinned): root states and all gradients."""
    gr = foldgen.config_c1()
    S = 5
    p = foldgen.make_params(cell, S, gr.vocab)
    T = foldgen.mo_table([(EMB, 0, -1, 0, gr.vocab), (kind, 2, 0, 0, 0)], [S])
    mg = _graph(T, gr.op, gr.child, gr.token, gr.root)
    P = oracle.mo_flatten(T, [(p.E,), (p.U, p.b)])
    H, C = oracle.mo_forward(mg, P)
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    np.testing.assert_allclose(H[gr.root], hr, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(C[gr.root], cr, rtol=1e-13, atol=1e-15)
    g = foldgen.make_upstream(gr.n_graphs, S)
    dP = oracle.mo_backward(mg, P, g)
    (dE,), (dU, db) = oracle.mo_unflatten(T, [(p.E,), (p.U, p.b)], dP)
    rU, rb, rE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    for x, y in ((dU, rU), (db, rb), (dE, rE)):
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("k", [1, 2, 5, 17])
def test_unary_chain_constant_gates(k):
    """U = 0: a chain of k unary LSTM nodes above a leaf (c = 0):
    c_k = s(b_i) tanh(b_u) (1 - s(b_f)^k) / (1 - s(b_f)),  h_k = s(b_o) tanh(c_k)."""
    S = 4
    rng = np.random.default_rng(k)
    T = foldgen.mo_table([(EMB, 0, -1, 0, 3), (LSTM, 1, 0, 0, 0)], [S])
    b = rng.uniform(-1, 1, 4 * S)
    op = [0] + [1] * k
    child = [[-1, -1]] + [[n, -1] for n in range(k)]
    gr = _graph(T, op, child, [2] + [0] * k, [k])
    P = oracle.mo_flatten(T, [(rng.uniform(-1, 1, (3, S)),), (np.zeros((4 * S, S)), b)])
    H, C = oracle.mo_forward(gr, P)
    si, sf, so, tu = sig(b[:S]), sig(b[S:2 * S]), sig(b[2 * S:3 * S]), np.tanh(b[3 * S:])
    c = si * tu * (1 - sf ** k) / (1 - sf)
    np.testing.assert_allclose(C[k, :S], c, rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(H[k, :S], so * np.tanh(c), rtol=1e-13, atol=1e-15)


def test_typed_projection_closed_form():
    """RNN projection type 0 (S0=3) -> type 1 (S1=5) over one leaf x = E[t]: h = tanh(U x + b);
    L = <g, h>: dU = (g (1 - h^2)) x^T, db = g (1 - h^2), dE[t] = U^T (g (1 - h^2))."""
    rng = np.random.default_rng(7)
    T = foldgen.mo_table([(EMB, 0, -1, 0, 4), (RNN, 1, 0, 1, 0)], [3, 5])
    E = rng.uniform(-1, 1, (4, 3)); U = rng.uniform(-1, 1, (5, 3)); b = rng.uniform(-1, 1, 5)
    gr = _graph(T, [0, 1], [[-1, -1], [0, -1]], [2, 0], [1])
    P = oracle.mo_flatten(T, [(E,), (U, b)])
    H, _ = oracle.mo_forward(gr, P)
    x = E[2]
    h = np.tanh(U @ x + b)
    np.testing.assert_allclose(H[1, :5], h, rtol=1e-14)
    g = rng.uniform(-1, 1, (1, 5))
    dP = oracle.mo_backward(gr, P, g)
    (dE,), (dU, db) = oracle.mo_unflatten(T, [(E,), (U, b)], dP)
    dz = g[0] * (1 - h * h)
    np.testing.assert_allclose(dU, np.outer(dz, x), rtol=1e-13, atol=1e-15)
    np.testing.assert_allclose(db, dz, rtol=1e-13, atol=1e-15)
    want = np.zeros_like(E); want[2] = U.T @ dz
    np.testing.assert_allclose(dE, want, rtol=1e-13, atol=1e-15)


# ----------------------------------------------------------------------------- finite differences

@pytest.mark.parametrize("seed", [0, 1])
def test_finite_differences_all_params(seed):
    """Central differences of L = sum_g <g_g, h_root(g)> on every parameter of a 7-op,
    2-type table over a random DAG with shared nodes (relative error < 1e-6)."""
    rng = np.random.default_rng(100 + seed)
    T = table7()
    gr = random_mo_graph(T, rng, 40, 4, share=0.3)
    params = foldgen.make_mo_params(T, seed=seed)
    P = oracle.mo_flatten(T, params) * 1.5
    Sm = int(T.S.max())
    g = rng.uniform(-1, 1, (gr.n_graphs, Sm))

    def loss(P):
        H, _ = oracle.mo_forward(gr, P)
        tot = 0.0
        for gi, r in enumerate(gr.root):
            Sr = int(T.S[T.out_type[gr.op[r]]])
            tot += float(np.dot(g[gi, :Sr], H[r, :Sr]))
        return tot

    dP = oracle.mo_backward(gr, P, g)
    eps = 1e-6
    idx = np.arange(P.size)
    for i in idx:
        Pp, Pm = P.copy(), P.copy()
        Pp[i] += eps; Pm[i] -= eps
        fd = (loss(Pp) - loss(Pm)) / (2 * eps)
        assert abs(fd - dP[i]) <= 1e-6 * max(1.0, abs(fd)), (i, fd, dP[i])
