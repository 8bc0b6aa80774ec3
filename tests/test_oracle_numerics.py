"""Pins for the oracle's fp64 forward/backward (CPU only): closed forms derived from the
cell equations (Tai et al. eqs 9-14 via PAPER.md L301-304), bitwise
batched == unbatched, and central finite differences."""
import numpy as np
import pytest

import foldgen
import oracle


def sig(x):
    return 1.0 / (1.0 + np.exp(-x))


def _params(cell, S, V, rng, scale=1.0):
    g = foldgen.gates_of(cell)
    U = rng.uniform(-scale, scale, (g * S, 2 * S)) / np.sqrt(S)
    b = rng.uniform(-0.3, 0.3, g * S)
    E = rng.uniform(-0.5, 0.5, (V, S))
    return U, b, E


def test_zero_params_treelstm():
    """U=0, b=0: i=f=o=1/2, u=0 => c = (c_L+c_R)/2 = 0 with leaf c=0, h = 0 at every cell
    (SPEC S:L601)."""
    gr = foldgen.config_c1()
    S, V = 6, gr.vocab
    U = np.zeros((5 * S, 2 * S)); b = np.zeros(5 * S)
    E = np.random.default_rng(0).uniform(-1, 1, (V, S))
    hr, cr, H, C = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E, all_nodes=True)
    cells = gr.op == 1
    assert np.all(H[cells] == 0) and np.all(C[cells] == 0)
    leaves = gr.op == 0
    assert np.array_equal(H[leaves], E[gr.token[leaves]])


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_constant_gates_complete_tree(k):
    """U=0: c(n) = s(b_i)tanh(b_u) + s(b_fL)c(L) + s(b_fR)c(R). On a complete tree with k
    cell levels: c_k = s_i t_u (1 - beta^k)/(1 - beta), beta = s(b_fL)+s(b_fR);
    h = s(b_o) tanh(c)."""
    S = 4
    rng = np.random.default_rng(k)
    b = rng.uniform(-1, 1, 5 * S)
    U = np.zeros((5 * S, 2 * S)); E = rng.uniform(-1, 1, (3, S))
    gr = foldgen.replicate_shape(foldgen.complete_shape(2 ** k), 2, lambda n: np.arange(n) % 3, 3)
    hr, cr = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E)
    si, sfl, sfr, so, tu = sig(b[:S]), sig(b[S:2 * S]), sig(b[2 * S:3 * S]), sig(b[3 * S:4 * S]), np.tanh(b[4 * S:])
    beta = sfl + sfr
    c = si * tu * (1 - beta ** k) / (1 - beta)
    np.testing.assert_allclose(cr, np.tile(c, (2, 1)), rtol=1e-13, atol=1e-14)
    np.testing.assert_allclose(hr, np.tile(so * np.tanh(c), (2, 1)), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("L", [2, 3, 7, 30])
def test_constant_gates_caterpillar(L):
    """Caterpillar c_k = cell(c_{k-1}, leaf): c_k = s_i t_u (1 - s_fL^k)/(1 - s_fL) — pins
    the left/right wiring of both the h gather and the c gather (b_fL != b_fR)."""
    S = 3
    rng = np.random.default_rng(L)
    b = rng.uniform(-1, 1, 5 * S)
    U = np.zeros((5 * S, 2 * S)); E = rng.uniform(-1, 1, (2, S))
    gr = foldgen.replicate_shape(foldgen.caterpillar_shape(L), 1, lambda n: np.arange(n) % 2, 2)
    hr, cr = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E)
    si, sfl, tu = sig(b[:S]), sig(b[S:2 * S]), np.tanh(b[4 * S:])
    k = L - 1
    c = si * tu * (1 - sfl ** k) / (1 - sfl)
    np.testing.assert_allclose(cr[0], c, rtol=1e-13, atol=1e-14)
    # mirrored chain (right-leaning) uses the right forget gate
    o, l, r = foldgen.caterpillar_shape(L)
    gr2 = foldgen.replicate_shape((o, r, l), 1, lambda n: np.arange(n) % 2, 2)
    _, cr2 = oracle.forward("treelstm", gr2.op, gr2.child, gr2.token, gr2.root, U, b, E)
    sfr = sig(b[2 * S:3 * S])
    np.testing.assert_allclose(cr2[0], si * tu * (1 - sfr ** k) / (1 - sfr), rtol=1e-13, atol=1e-14)


@pytest.mark.parametrize("side", [0, 1])
def test_treernn_spine(side):
    """TreeRNN with W = [I 0] (side 0) or [0 I], b = 0: root h = tanh^k(E[leftmost/rightmost
    leaf]) with k = length of that spine — pins the gather wiring of both child slots."""
    S = 5
    rng = np.random.default_rng(5 + side)
    W = np.zeros((S, 2 * S)); W[:, side * S:(side + 1) * S] = np.eye(S)
    b = np.zeros(S); E = rng.uniform(-1, 1, (11, S))
    for _ in range(10):
        o, l, r = foldgen.random_split_shape(rng, int(rng.integers(1, 12)))
        gr = foldgen.batch_from_shapes([(o, l, r)], lambda n: rng.integers(0, 11, n), 11)
        hr, _ = oracle.forward("treernn", gr.op, gr.child, gr.token, gr.root, W, b, E)
        n, k = int(gr.root[0]), 0
        while gr.op[n] == 1:
            n = gr.child[n][side]; k += 1
        x = E[gr.token[n]].copy()
        for _ in range(k):
            x = np.tanh(x)
        np.testing.assert_allclose(hr[0], x, rtol=1e-14, atol=1e-15)


@pytest.mark.parametrize("cell", ["treernn", "treelstm"])
def test_batched_equals_unbatched_bitwise(cell):
    """PAPER.md L49/L86 + SPEC S:L437/S:L530: the level-batched evaluation (the loop of
    L47 driven by the oracle's schedule) equals node-at-a-time evaluation exactly, and a
    merged batch gives each tree's isolated result exactly."""
    rng = np.random.default_rng(17)
    S, V = 7, 9
    U, b, E = _params(cell, S, V, rng)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 14))) for _ in range(6)]
    gr = foldgen.batch_from_shapes(shapes, lambda n: rng.integers(0, V, n), V)
    gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
    hr, cr, H, C = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, U, b, E, all_nodes=True)
    H2, C2 = oracle.forward_levels(cell, gr.op, gr.child, gr.token, gr.root, U, b, E)
    assert np.array_equal(H, H2) and np.array_equal(C, C2)
    gr0 = foldgen.batch_from_shapes(shapes, lambda n: np.zeros(n), V)  # same shapes
    # isolated runs, one tree at a time, on the unpermuted batch
    rng2 = np.random.default_rng(3)
    toks = rng2.integers(0, V, gr0.n_nodes)
    gr0.token[:] = np.where(gr0.op == 0, toks, 0)
    hr0, cr0 = oracle.forward(cell, gr0.op, gr0.child, gr0.token, gr0.root, U, b, E)
    for t in range(len(shapes)):
        one = foldgen.sub_batch(gr0, t, t + 1)
        h1, c1 = oracle.forward(cell, one.op, one.child, one.token, one.root, U, b, E)
        assert np.array_equal(h1[0], hr0[t]) and np.array_equal(c1[0], cr0[t])


def test_bounds():
    """|h| < 1 at cells (h = o*tanh(c)); |c(n)| <= #cells in n's subtree
    (|i*u| < 1, f in (0,1), leaf c = 0)."""
    rng = np.random.default_rng(2)
    gr = foldgen.config_c3(20)
    S = 8
    U, b, E = _params("treelstm", S, gr.vocab, rng, scale=3.0)
    hr, cr, H, C = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E, all_nodes=True)
    cells = gr.op == 1
    assert np.abs(H[cells]).max() < 1
    ncell = np.zeros(gr.n_nodes)
    for n in range(gr.n_nodes):  # post-order: children first
        if gr.op[n] == 1:
            ncell[n] = 1 + ncell[gr.child[n][0]] + ncell[gr.child[n][1]]
    assert np.all(np.abs(C).max(axis=1) <= ncell + 1e-12)


# ---------------------------------------------------------------- backward

def _loss(cell, gr, U, b, E, g, gc):
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, U, b, E)
    L = float((hr * g).sum())
    if gc is not None:
        L += float((cr * gc).sum())
    return L


def _fd_check(cell, gr, S, V, rng, with_dc):
    U, b, E = _params(cell, S, V, rng, scale=2.0)
    G = gr.n_graphs
    g = rng.uniform(-1, 1, (G, S))
    gc = rng.uniform(-1, 1, (G, S)) if with_dc else None
    dU, db, dE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, U, b, E, g, gc)
    h = 1e-6
    for P, dP in ((U, dU), (b, db), (E, dE)):
        flat = P.reshape(-1); dflat = dP.reshape(-1)
        num = np.zeros_like(dflat)
        for i in range(flat.size):
            old = flat[i]
            flat[i] = old + h; lp = _loss(cell, gr, U, b, E, g, gc)
            flat[i] = old - h; lm = _loss(cell, gr, U, b, E, g, gc)
            flat[i] = old
            num[i] = (lp - lm) / (2 * h)
        err = np.abs(num - dflat).max() / max(np.abs(num).max(), 1e-30)
        assert err < 1e-6, (P.shape, err)


@pytest.mark.parametrize("cell", ["treernn", "treelstm"])
def test_finite_differences_trees(cell):
    """central FD at fp64, h=1e-6, rel < 1e-6, for every entry of U, b, E."""
    rng = np.random.default_rng(23)
    shapes = [foldgen.random_split_shape(rng, n) for n in (1, 3, 5)]
    gr = foldgen.batch_from_shapes(shapes, lambda n: rng.integers(0, 4, n), 4)
    _fd_check(cell, gr, 3, 4, rng, with_dc=(cell == "treelstm"))


@pytest.mark.parametrize("cell", ["treernn", "treelstm"])
def test_finite_differences_dag(cell):
    """DAG sharing (a node with several consumers, cell(x, x)) and a root that is also
    consumed: the gradient of a shared node is the sum over its consumers."""
    op = [0, 0, 1, 1, 1, 0, 1]
    child = [[-1, -1], [-1, -1], [0, 1], [2, 2], [3, 2], [-1, -1], [4, 5]]
    token = [0, 1, 0, 0, 0, 1, 0]
    root = [6, 2, 4]
    gr = foldgen.Graphs(np.asarray(op, np.int32), np.asarray(child, np.int32), np.asarray(token, np.int32),
                        np.asarray(root, np.int32), 3, np.asarray([7]))
    _fd_check(cell, gr, 3, 3, np.random.default_rng(29), with_dc=True)


def test_zero_params_backward_closed_form():
    """U=0, b=0 (every cell c=h=0, gates 1/2, u=0): at a cell at distance k from its root
    dc = g 2^-(k+1), dz = [0,0,0,0, g 2^-(k+2)], so dU[u-block] = sum_cells g 2^-(k+2) (x)
    [h_L; h_R] with leaf children contributing E[tok] and cell children 0,
    db[u] = sum_cells g 2^-(k+2), all other blocks 0, dE = 0 except single-leaf trees."""
    rng = np.random.default_rng(31)
    S, V = 4, 6
    shapes = [foldgen.random_split_shape(rng, n) for n in (1, 2, 5, 9)]
    gr = foldgen.batch_from_shapes(shapes, lambda n: rng.integers(0, V, n), V)
    U = np.zeros((5 * S, 2 * S)); b = np.zeros(5 * S); E = rng.uniform(-1, 1, (V, S))
    g = rng.uniform(-1, 1, (gr.n_graphs, S))
    dU, db, dE = oracle.backward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E, g)
    eU = np.zeros_like(dU); eb = np.zeros_like(db); eE = np.zeros_like(dE)
    for t, r in enumerate(gr.root):
        if gr.op[r] == 0:
            eE[gr.token[r]] += g[t]
            continue
        stack = [(int(r), 0)]
        while stack:
            n, k = stack.pop()
            if gr.op[n] == 0:
                continue
            dzu = g[t] * 2.0 ** -(k + 2)
            L, R = gr.child[n]
            hl = E[gr.token[L]] if gr.op[L] == 0 else np.zeros(S)
            hr = E[gr.token[R]] if gr.op[R] == 0 else np.zeros(S)
            eU[4 * S:, :] += np.outer(dzu, np.concatenate([hl, hr]))
            eb[4 * S:] += dzu
            stack += [(int(L), k + 1), (int(R), k + 1)]
    np.testing.assert_allclose(dU, eU, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(db, eb, rtol=1e-14, atol=1e-15)
    np.testing.assert_allclose(dE, eE, rtol=1e-14, atol=1e-15)


def test_backward_linearity_over_trees():
    """Gradients of a merged batch are the sum of the per-tree gradients (weights shared
    by all invocations accumulate)."""
    rng = np.random.default_rng(41)
    S, V = 5, 7
    U, b, E = _params("treelstm", S, V, rng)
    shapes = [foldgen.random_split_shape(rng, n) for n in (2, 6, 4)]
    gr = foldgen.batch_from_shapes(shapes, lambda n: rng.integers(0, V, n), V)
    g = rng.uniform(-1, 1, (3, S))
    dU, db, dE = oracle.backward("treelstm", gr.op, gr.child, gr.token, gr.root, U, b, E, g)
    acc = [np.zeros_like(dU), np.zeros_like(db), np.zeros_like(dE)]
    for t in range(3):
        one = foldgen.sub_batch(gr, t, t + 1)
        for a, x in zip(acc, oracle.backward("treelstm", one.op, one.child, one.token, one.root,
                                              U, b, E, g[t:t + 1])):
            a += x
    for x, y in zip((dU, db, dE), acc):
        np.testing.assert_allclose(x, y, rtol=1e-12, atol=1e-14)
