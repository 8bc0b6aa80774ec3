"""fp64 CPU oracle for dynamic batching (arXiv 1702.02181) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (its `cpu_baseline` leg and
`--impl reference`) may import this package. The product package
`paper_1702_02181_b200` never imports it, and this package imports nothing from
the product; the two share only the seeded input generators in `foldgen`.

Contents
  fold_oracle.c  plain C, fp64: schedule by definition, node-at-a-time forward,
                 level-ordered forward (self-check), hand-derived backward.
                 §3.5 model (leaf TreeLSTM(E[w],0,0) + per-node softmax CE).
  paper_form.py  the paper-form schedule with pass-through operations and (d,t,i)
                 edge labels, pure Python, for Fig. 1 parity.

Every function here is pinned by `-m "not gpu"` tests against values the paper
fixes (Fig. 1), closed forms, brute force on tiny inputs and finite differences
(see DESIGN.md "Oracle pins"). Throughput parity vs the paper is unpinned.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "fold_oracle.c")
_SRC_MO = os.path.join(_HERE, "fold_oracle_mo.c")
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lock = threading.Lock()
_lib = None

STATUS = {0: "OK", 1: "INVALID", 2: "CHILD_RANGE", 3: "ARITY", 4: "TOKEN_RANGE",
          5: "ROOT_RANGE", 6: "CYCLE", 10: "OP_RANGE", 11: "TYPE", 12: "LEVEL"}
CELLS = {"treernn": 0, "treelstm": 1}


def build(force: bool = False) -> str:
    """Compile fold_oracle.c + fold_oracle_mo.c with gcc (plain C11, -O2, no fast-math)."""
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    if (not force and os.path.exists(_LIB_PATH)
            and all(os.path.getmtime(_LIB_PATH) >= os.path.getmtime(f) for f in (_SRC, _SRC_MO))):
        return _LIB_PATH
    tmp = _LIB_PATH + f".{os.getpid()}.tmp"
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-fno-fast-math", "-fPIC", "-shared",
                           "-o", tmp, _SRC, _SRC_MO, "-lm"])
    os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            _lib = ctypes.CDLL(build())
    return _lib


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, status, node=-1):
        super().__init__(f"oracle status {STATUS.get(status, status)} (node {node})")
        self.status = STATUS.get(status, status)
        self.node = node


def schedule(op, child, token, root, vocab, level=None):
    """Executor-form schedule (see fold_oracle.c `oracle_schedule`); `level` = optional
    caller-fixed levels (manual batching). Returns a dict of
    int32 arrays sized to their logical lengths, plus n_levels/n_leaves/n_cells/n_tok_segs.
    Raises OracleError with the status name and offending node on invalid input."""
    lib = _load()
    op, child, token, root = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(root)
    level = _i32(level) if level is not None else None
    N, G = len(op), len(root)
    out = {k: np.zeros(n, np.int32) for k, n in [
        ("depth", N), ("perm", N), ("rank", N), ("gather", 2 * N), ("level_off", N + 2),
        ("group_off", 2 * N + 3), ("cons_off", N + 1), ("cons_edge", 2 * N),
        ("leaf_perm", N), ("tok_seg", N + 1), ("root_row", G), ("root_perm", G)]}
    info = np.zeros(5, np.int32)
    st = lib.oracle_schedule(ctypes.c_int(N), ctypes.c_int(G), ctypes.c_int(vocab),
                             _p(op), _p(child), _p(token), _p(root), _p(level),
                             *[_p(out[k]) for k in ("depth", "perm", "rank", "gather", "level_off",
                                                    "group_off", "cons_off", "cons_edge", "leaf_perm",
                                                    "tok_seg", "root_row", "root_perm")], _p(info))
    if st != 0:
        raise OracleError(st, int(info[4]))
    D, nl, nc, ns = (int(x) for x in info[:4])
    out["gather"] = out["gather"].reshape(N, 2)
    out["level_off"] = out["level_off"][:D + 2]
    out["group_off"] = out["group_off"][:2 * (D + 1) + 1]
    out["cons_edge"] = out["cons_edge"][:2 * nc]
    out["leaf_perm"] = out["leaf_perm"][:nl]
    out["tok_seg"] = out["tok_seg"][:ns + 1]
    out.update(n_levels=D, n_leaves=nl, n_cells=nc, n_tok_segs=ns)
    return out


def forward(cell, op, child, token, root, U, b, E, all_nodes=False):
    """Node-at-a-time fp64 forward. Returns (h_root[G,S], c_root[G,S]) and, with
    all_nodes=True, also (H[N,S], C[N,S]) in node-id order."""
    lib = _load()
    op, child, token, root = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(root)
    U, b, E = _f64(U), _f64(b), _f64(E)
    N, G = len(op), len(root)
    V, S = E.shape
    hr = np.zeros((G, S)); cr = np.zeros((G, S))
    H = np.zeros((N, S)) if all_nodes else None
    C = np.zeros((N, S)) if all_nodes else None
    st = lib.oracle_forward(CELLS[cell], S, N, G, V, _p(op), _p(child), _p(token), _p(root),
                            _p(U), _p(b), _p(E), _p(hr), _p(cr), _p(H), _p(C))
    if st != 0:
        raise OracleError(st)
    return (hr, cr, H, C) if all_nodes else (hr, cr)


def forward_levels(cell, op, child, token, root, U, b, E, level=None):
    """Level-ordered fp64 forward over this oracle's own schedule (optionally with
    caller-fixed levels); (H[N,S], C[N,S])."""
    lib = _load()
    op, child, token, root = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(root)
    level = _i32(level) if level is not None else None
    U, b, E = _f64(U), _f64(b), _f64(E)
    N, G = len(op), len(root)
    V, S = E.shape
    H = np.zeros((N, S)); C = np.zeros((N, S))
    st = lib.oracle_forward_levels(CELLS[cell], S, N, G, V, _p(op), _p(child), _p(token), _p(root),
                                   _p(level), _p(U), _p(b), _p(E), _p(H), _p(C))
    if st != 0:
        raise OracleError(st)
    return H, C


def backward(cell, op, child, token, root, U, b, E, dh_root, dc_root=None):
    """fp64 reverse mode of L = sum_g <dh_root[g], h_root(g)> + <dc_root[g], c_root(g)>.
    Returns (dU, db, dE) with the shapes of (U, b, E)."""
    lib = _load()
    op, child, token, root = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(root)
    U, b, E = _f64(U), _f64(b), _f64(E)
    dh = _f64(dh_root)
    dc = _f64(dc_root) if dc_root is not None else None
    N, G = len(op), len(root)
    V, S = E.shape
    dU = np.zeros_like(U); db = np.zeros_like(b); dE = np.zeros_like(E)
    st = lib.oracle_backward(CELLS[cell], S, N, G, V, _p(op), _p(child), _p(token), _p(root),
                             _p(U), _p(b), _p(E), _p(dh), _p(dc), _p(dU), _p(db), _p(dE))
    if st != 0:
        raise OracleError(st)
    return dU, db, dE


def sst_forward(op, child, token, label, U, b, E, W, Ws, bs, all_nodes=False):
    """§3.5 model (fold_oracle.c oracle_sst_forward): total per-node
    softmax cross-entropy over all nodes; with all_nodes=True also (H[N,S], C[N,S])."""
    lib = _load()
    op, child, token, label = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(label)
    U, b, E, W, Ws, bs = (_f64(x) for x in (U, b, E, W, Ws, bs))
    N = len(op)
    V, S = E.shape
    C = bs.shape[0]
    loss = np.zeros(1)
    H = np.zeros((N, S)) if all_nodes else None
    Cs = np.zeros((N, S)) if all_nodes else None
    st = lib.oracle_sst_forward(S, N, V, C, _p(op), _p(child), _p(token), _p(label), _p(U), _p(b), _p(E), _p(W),
                                _p(Ws), _p(bs), _p(loss), _p(H), _p(Cs))
    if st != 0:
        raise OracleError(st)
    return (float(loss[0]), H, Cs) if all_nodes else float(loss[0])


def sst_backward(op, child, token, label, U, b, E, W, Ws, bs):
    """Reverse mode of the §3.5 loss: (loss, dU, db, dE, dW, dWs, dbs)."""
    lib = _load()
    op, child, token, label = _i32(op), _i32(child).reshape(-1), _i32(token), _i32(label)
    U, b, E, W, Ws, bs = (_f64(x) for x in (U, b, E, W, Ws, bs))
    N = len(op)
    V, S = E.shape
    C = bs.shape[0]
    loss = np.zeros(1)
    out = [np.zeros_like(x) for x in (U, b, E, W, Ws, bs)]
    st = lib.oracle_sst_backward(S, N, V, C, _p(op), _p(child), _p(token), _p(label), _p(U), _p(b), _p(E), _p(W),
                                 _p(Ws), _p(bs), _p(loss), *[_p(x) for x in out])
    if st != 0:
        raise OracleError(st)
    return (float(loss[0]), *out)


# ----------------------------------------------------------------------------- multi-op (NEXT-3)
# fold_oracle_mo.c: several operations and tensor types per depth.
# Parameters travel as one flat fp64 array in the oracle's own layout (op o's block at
# mo_param_offsets(table)[o]: EMBED E_o; LSTM / RNN U_o then b_o).

def _table_args(table):
    return (ctypes.c_int(table.n_ops), ctypes.c_int(table.n_types), *[_p(_i32(x)) for x in (
        table.kind, table.arity, table.in_type, table.out_type, table.vocab, table.S)])


def _keep(table):
    return [_i32(x) for x in (table.kind, table.arity, table.in_type, table.out_type, table.vocab, table.S)]


def mo_param_offsets(table):
    lib = _load()
    lib.mo_param_offsets.restype = ctypes.c_int64
    poff = np.zeros(table.n_ops + 1, np.int64)
    ks = _keep(table)
    lib.mo_param_offsets(ctypes.c_int(table.n_ops), ctypes.c_int(table.n_types), *[_p(x) for x in ks], _p(poff))
    return poff


def mo_flatten(table, params):
    """Per-op parameter tuples (foldgen.make_mo_params) -> the oracle's flat fp64 array."""
    poff = mo_param_offsets(table)
    P = np.zeros(int(poff[-1]), np.float64)
    for o, blk in enumerate(params):
        flat = np.concatenate([np.asarray(x, np.float64).reshape(-1) for x in blk])
        assert flat.size == poff[o + 1] - poff[o]
        P[poff[o]:poff[o + 1]] = flat
    return P


def mo_unflatten(table, params, P):
    """Inverse of mo_flatten, shaped like `params` (gradients back per op)."""
    poff = mo_param_offsets(table)
    out = []
    for o, blk in enumerate(params):
        off, parts = int(poff[o]), []
        for x in blk:
            n = int(np.asarray(x).size)
            parts.append(P[off:off + n].reshape(np.asarray(x).shape))
            off += n
        out.append(tuple(parts))
    return out


def mo_schedule(gr):
    """fold_oracle_mo.c oracle_mo_schedule on a foldgen.MoGraphs: depth, group_off (per
    (depth, op) key), type_off / pool / pool_row (the per-type concatenation of PAPER.md L43),
    tlevel_off [n_types, D+2], label [N, 2, 3] = (d, t, i) per edge (L44)."""
    lib = _load()
    T = gr.table
    ks = _keep(T)
    op, child, token, root = _i32(gr.op), _i32(gr.child).reshape(-1), _i32(gr.token), _i32(gr.root)
    N, G = len(op), len(root)
    out = {k: np.zeros(n, np.int32) for k, n in [
        ("depth", N), ("group_off", (N + 1) * T.n_ops + 1), ("type_off", T.n_types + 1), ("pool", N),
        ("pool_row", N), ("tlevel_off", T.n_types * (N + 2)), ("label", N * 2 * 3)]}
    info = np.zeros(2, np.int32)
    st = lib.oracle_mo_schedule(ctypes.c_int(T.n_ops), ctypes.c_int(T.n_types), *[_p(x) for x in ks],
                                ctypes.c_int(N), ctypes.c_int(G), _p(op), _p(child), _p(token), _p(root),
                                *[_p(out[k]) for k in ("depth", "group_off", "type_off", "pool", "pool_row",
                                                       "tlevel_off", "label")], _p(info))
    if st != 0:
        raise OracleError(st, int(info[1]))
    D = int(info[0])
    out["group_off"] = out["group_off"][:(D + 1) * T.n_ops + 1]
    out["tlevel_off"] = out["tlevel_off"][:T.n_types * (D + 2)].reshape(T.n_types, D + 2)
    out["label"] = out["label"].reshape(N, 2, 3)
    out["n_levels"] = D
    return out


def mo_forward(gr, P):
    """Node-at-a-time fp64 forward: (H [N, S_max], C [N, S_max]) in node-id order."""
    lib = _load()
    T = gr.table
    ks = _keep(T)
    op, child, token, root = _i32(gr.op), _i32(gr.child).reshape(-1), _i32(gr.token), _i32(gr.root)
    N, G = len(op), len(root)
    Sm = int(np.max(T.S))
    H = np.zeros((N, Sm)); C = np.zeros((N, Sm))
    P = _f64(P)
    st = lib.oracle_mo_forward(ctypes.c_int(T.n_ops), ctypes.c_int(T.n_types), *[_p(x) for x in ks],
                               ctypes.c_int(N), ctypes.c_int(G), _p(op), _p(child), _p(token), _p(root), _p(P),
                               _p(H), _p(C))
    if st != 0:
        raise OracleError(st)
    return H, C


def mo_backward(gr, P, g):
    """fp64 reverse mode of L = sum_g <g[g, :S_root], h_root(g)>; dP in P's layout."""
    lib = _load()
    T = gr.table
    ks = _keep(T)
    op, child, token, root = _i32(gr.op), _i32(gr.child).reshape(-1), _i32(gr.token), _i32(gr.root)
    N, G = len(op), len(root)
    P, g = _f64(P), _f64(g)
    dP = np.zeros_like(P)
    st = lib.oracle_mo_backward(ctypes.c_int(T.n_ops), ctypes.c_int(T.n_types), *[_p(x) for x in ks],
                                ctypes.c_int(N), ctypes.c_int(G), _p(op), _p(child), _p(token), _p(root), _p(P),
                                _p(g), _p(dP))
    if st != 0:
        raise OracleError(st)
    return dP
