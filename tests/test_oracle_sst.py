"""Pins of the §3.5 oracle (oracle_sst_forward / oracle_sst_backward), each
against something other than the oracle's own formulas:

  * leaf = the R1 cell on (x, 0): TreeLSTM(E[w], 0, 0) (L300) equals the x = 0 TreeLSTM cell
    of oracle.forward (a different code path) applied to a left child h_L = x and a right
    child 0, both with c = 0, when U's left-half blocks i, o, u are W's blocks (Tai eqs 9-14:
    the input term W x enters exactly like U_L h_L) — pins the leaf gates and c = i u;
  * closed forms with Ws = 0: p = softmax(bs) at every node, so L = N lse(bs) - sum_n
    bs[y_n], dbs = N softmax(bs) - counts(y), dWs = sum_n (p - e_{y_n}) h_n^T, and no gradient
    reaches the tree (dU = db = dE = dW = 0);
  * central finite differences (h = 1e-6, rel < 1e-6) for entries of every parameter
    (U, b, E, W, Ws, bs) on trees with shared tokens;
  * linearity over trees: a merged batch's loss and gradients are the sums of the isolated
    trees' (a batch is one disconnected graph).
"""
import numpy as np

import foldgen
import oracle


def _tiny(seed=0, B=4, S=3, V=5):
    rng = np.random.default_rng(seed)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 6))) for _ in range(B)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, V), V)
    p = foldgen.make_params("treelstm", S, V, seed=seed + 10)
    q = foldgen.make_sst_params(S, seed=seed + 20)
    y = foldgen.make_labels(gr.n_nodes, seed=seed + 30)
    return gr, p, q, y


def test_leaf_is_the_cell_on_x_and_zero():
    S, V = 6, 7
    rng = np.random.default_rng(1)
    p = foldgen.make_params("treelstm", S, V)
    q = foldgen.make_sst_params(S)
    for tok in range(V):
        # SST model on a single leaf: h, c of that leaf
        op = np.array([0], np.int32); child = np.array([[-1, -1]], np.int32); token = np.array([tok], np.int32)
        _, H, C = oracle.sst_forward(op, child, token, np.zeros(1, np.int32), p.U, p.b, p.E, q.W, q.Ws, q.bs,
                                     all_nodes=True)
        # R1 oracle: cell(leaf x, leaf 0) with U_L blocks (i, *, *, o, u) = W blocks (i, o, u), U_R = 0
        U = np.zeros((5 * S, 2 * S))
        U[0:S, :S] = q.W[0:S]
        U[3 * S:4 * S, :S] = q.W[S:2 * S]
        U[4 * S:5 * S, :S] = q.W[2 * S:3 * S]
        U[S:3 * S, :S] = rng.standard_normal((2 * S, S))  # forget gates: irrelevant (c_k = 0)
        E2 = np.stack([p.E[tok], np.zeros(S)])
        op2 = np.array([0, 0, 1], np.int32)
        ch2 = np.array([[-1, -1], [-1, -1], [0, 1]], np.int32)
        hr, cr = oracle.forward("treelstm", op2, ch2, np.array([0, 1, 0], np.int32), np.array([2], np.int32), U,
                                p.b, E2)
        np.testing.assert_allclose(H[0], hr[0], rtol=1e-13, atol=1e-15)
        np.testing.assert_allclose(C[0], cr[0], rtol=1e-13, atol=1e-15)


def test_zero_classifier_closed_forms():
    gr, p, q, y = _tiny(3, B=6, S=4)
    C = foldgen.SST_CLASSES
    Ws0 = np.zeros_like(q.Ws)
    loss, dU, db, dE, dW, dWs, dbs = oracle.sst_backward(gr.op, gr.child, gr.token, y, p.U, p.b, p.E, q.W, Ws0, q.bs)
    bs = q.bs.astype(np.float64)
    lse = np.log(np.exp(bs).sum())
    N = gr.n_nodes
    assert abs(loss - (N * lse - bs[y].sum())) <= 1e-10 * abs(loss)
    sm = np.exp(bs - lse)
    counts = np.bincount(y, minlength=C)
    np.testing.assert_allclose(dbs, N * sm - counts, atol=1e-12)
    _, H, _ = oracle.sst_forward(gr.op, gr.child, gr.token, y, p.U, p.b, p.E, q.W, Ws0, q.bs, all_nodes=True)
    D = sm[None, :] - np.eye(C)[y]
    np.testing.assert_allclose(dWs, D.T @ H, atol=1e-12)
    for g in (dU, db, dE, dW):
        assert np.abs(g).max() == 0.0


def _loss(gr, y, P):
    return oracle.sst_forward(gr.op, gr.child, gr.token, y, *P)


def test_finite_differences_every_parameter():
    gr, p, q, y = _tiny(7, B=3, S=3, V=4)
    P = [p.U.astype(np.float64), p.b.astype(np.float64), p.E.astype(np.float64), q.W.astype(np.float64),
         q.Ws.astype(np.float64), q.bs.astype(np.float64)]
    loss, *grads = oracle.sst_backward(gr.op, gr.child, gr.token, y, *P)
    h = 1e-6
    rng = np.random.default_rng(0)
    for k, (x, gx) in enumerate(zip(P, grads)):
        flat = x.reshape(-1)
        idx = rng.choice(flat.size, size=min(flat.size, 12), replace=False)
        for i in idx:
            old = flat[i]
            flat[i] = old + h
            lp = _loss(gr, y, P)
            flat[i] = old - h
            lm = _loss(gr, y, P)
            flat[i] = old
            fd = (lp - lm) / (2 * h)
            an = gx.reshape(-1)[i]
            assert abs(fd - an) <= 1e-6 * max(1.0, abs(an)), (k, i, fd, an)


def test_merged_batch_is_sum_of_trees():
    gr, p, q, y = _tiny(11, B=5, S=4, V=6)
    P = (p.U, p.b, p.E, q.W, q.Ws, q.bs)
    full = oracle.sst_backward(gr.op, gr.child, gr.token, y, *P)
    acc = None
    off = 0
    for t in range(gr.n_graphs):
        sub = foldgen.sub_batch(gr, t, t + 1)
        n = sub.n_nodes
        r = oracle.sst_backward(sub.op, sub.child, sub.token, y[off:off + n], *P)
        acc = list(r) if acc is None else [a + b for a, b in zip(acc, r)]
        off += n
    for a, b in zip(full, acc):
        np.testing.assert_allclose(a, b, rtol=1e-12, atol=1e-14)
