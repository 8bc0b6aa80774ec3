"""Oracle evaluation over many trees on all host cores (test infrastructure).

Trees of a batch are independent (a batch is one disconnected graph; L86:
trees of different shapes carry no penalty), so the fp64 oracle runs tree by tree on a
thread pool (its C calls release the GIL) and the per-tree results are summed in tree
order (fixed order, so a test's reference does not depend on the thread count)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

import foldgen
import oracle


def cores() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def per_tree(gr, p, g, trees, cell="treelstm", grads=True):
    """For each tree t in `trees`: (h_root, c_root[, dU, db, dE]) of that tree alone with
    upstream gradient g[t]."""
    def one(t):
        sub = foldgen.sub_batch(gr, t, t + 1)
        h, c = oracle.forward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E)
        if not grads:
            return h[0], c[0]
        dU, db, dE = oracle.backward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E, g[t:t + 1])
        return h[0], c[0], dU, db, dE
    with ThreadPoolExecutor(max_workers=cores()) as ex:
        return list(ex.map(one, list(trees)))


def batch_reference(gr, p, g, trees=None, cell="treelstm"):
    """Root states of `trees` (default: all) and the gradients summed over them."""
    trees = range(gr.n_graphs) if trees is None else trees
    res = per_tree(gr, p, g, trees, cell)
    h = np.stack([r[0] for r in res])
    c = np.stack([r[1] for r in res])
    dU = np.zeros_like(res[0][2]); db = np.zeros_like(res[0][3]); dE = np.zeros_like(res[0][4])
    for r in res:
        dU += r[2]; db += r[3]; dE += r[4]
    return h, c, dU, db, dE
