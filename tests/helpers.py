"""Shared helpers for the parity tests (the CUDA path vs the fp64 oracle)."""
import numpy as np

import foldgen


def rel_err(x, y):
    """Normwise-inf relative error max|x - y| / max|y| (SURVEY §8(c.7) reading; DESIGN.md
    'Tolerances')."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    den = np.abs(y).max() if y.size else 0.0
    num = np.abs(x - y).max() if y.size else 0.0
    if den == 0.0:
        return num
    return num / den


def small_params(cell, S, V, seed=foldgen.PARAM_SEED, scale=1.0):
    p = foldgen.make_params(cell, S, V, seed)
    if scale != 1.0:
        p.U *= scale
    return p


def random_dag(rng, N, V, p_share=0.3, G=None):
    """Random DAG (children have smaller ids before the caller shuffles), with sharing
    and cell(x, x)."""
    op = np.zeros(N, np.int32)
    child = np.full((N, 2), -1, np.int32)
    token = np.zeros(N, np.int32)
    for n in range(N):
        if n < 2 or rng.random() < 0.35:
            op[n] = 0
            token[n] = rng.integers(0, V)
        else:
            op[n] = 1
            a = rng.integers(max(0, n - 12), n)
            b = a if rng.random() < 0.1 else rng.integers(0, n)
            child[n] = (a, b)
    G = G or int(rng.integers(1, 5))
    root = rng.integers(0, N, G).astype(np.int32)
    return foldgen.Graphs(op, child, token, root, V, np.asarray([N], np.int32))
