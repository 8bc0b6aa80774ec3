"""ctypes binding of include/fold_mo.h (multi-op dynamic batching).

Argument marshalling only: every step of the path runs in libfold.so's kernels; PyTorch
provides device memory and streams. There is no CPU fallback (a missing library raises).
"""
from __future__ import annotations

import ctypes
import dataclasses

import numpy as np
import torch

from . import fold

MAX_OPS, MAX_TYPES = 8, 4
EMBED, LSTM, RNN = 0, 1, 2
PREC = {"fp32": 0, "tf32": 1, "bf16": 2}
_A8 = ctypes.c_int32 * MAX_OPS


class _Table(ctypes.Structure):
    _fields_ = [("n_ops", ctypes.c_int32), ("n_types", ctypes.c_int32), ("kind", _A8), ("arity", _A8),
                ("in_type", _A8), ("out_type", _A8), ("vocab", _A8), ("S", ctypes.c_int32 * MAX_TYPES)]


class _Graphs(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int32), ("n_graphs", ctypes.c_int32), ("op", ctypes.c_void_p),
                ("child", ctypes.c_void_p), ("token", ctypes.c_void_p), ("root", ctypes.c_void_p)]


_ARRAYS = ("depth", "group_off", "type_off", "pool", "pool_row", "tlevel_off", "label", "order", "cons_off",
           "cons_edge", "root_off", "root_graph", "leaf_seg", "leaf_order")


class _Sched(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in _ARRAYS] + [
        ("group_off_host", ctypes.c_void_p), ("n_nodes", ctypes.c_int32), ("n_graphs", ctypes.c_int32),
        ("n_levels", ctypes.c_int32), ("n_leaf_segs", ctypes.c_int32), ("op", ctypes.c_void_p),
        ("child", ctypes.c_void_p), ("token", ctypes.c_void_p), ("root", ctypes.c_void_p)]


_P8 = ctypes.c_void_p * MAX_OPS


class _Model(ctypes.Structure):
    _fields_ = [("prec", ctypes.c_int32), ("U", _P8), ("b", _P8), ("E", _P8)]


class _Grads(ctypes.Structure):
    _fields_ = [("dU", _P8), ("db", _P8), ("dE", _P8), ("accumulate", ctypes.c_int32)]


EXPORTED = ("fold_mo_schedule_workspace", "fold_mo_schedule", "fold_mo_acts_bytes", "fold_mo_forward_workspace",
            "fold_mo_forward", "fold_mo_backward_workspace", "fold_mo_backward")

_bound = None


def load():
    global _bound
    L = fold.load()
    if _bound is None:
        vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
        T, S = ctypes.POINTER(_Table), ctypes.POINTER(_Sched)
        L.fold_mo_schedule_workspace.restype = sz
        L.fold_mo_schedule_workspace.argtypes = [T, i32, i32]
        L.fold_mo_schedule.restype = i32
        L.fold_mo_schedule.argtypes = [T, ctypes.POINTER(_Graphs), S, vp, sz, vp]
        L.fold_mo_acts_bytes.restype = sz
        L.fold_mo_acts_bytes.argtypes = [T, S]
        L.fold_mo_forward_workspace.restype = sz
        L.fold_mo_forward_workspace.argtypes = [T, S]
        L.fold_mo_backward_workspace.restype = sz
        L.fold_mo_backward_workspace.argtypes = [T, S]
        L.fold_mo_forward.restype = i32
        L.fold_mo_forward.argtypes = [T, S, ctypes.POINTER(_Model), vp, vp, vp, sz, vp]
        L.fold_mo_backward.restype = i32
        L.fold_mo_backward.argtypes = [T, S, ctypes.POINTER(_Model), vp, vp, ctypes.POINTER(_Grads), vp, sz, vp]
        _bound = True
    return L


def table_struct(table) -> _Table:
    """A foldgen.MoTable (or any object with kind/arity/in_type/out_type/vocab/S arrays)."""
    t = _Table()
    t.n_ops, t.n_types = int(len(table.kind)), int(len(table.S))
    for o in range(t.n_ops):
        t.kind[o], t.arity[o] = int(table.kind[o]), int(table.arity[o])
        t.in_type[o], t.out_type[o], t.vocab[o] = int(table.in_type[o]), int(table.out_type[o]), int(table.vocab[o])
    for i in range(t.n_types):
        t.S[i] = int(table.S[i])
    return t


@dataclasses.dataclass
class MoSchedule:
    table: _Table
    arrays: dict
    group_off_host: np.ndarray
    n_nodes: int
    n_graphs: int
    n_levels: int
    n_leaf_segs: int
    _struct: _Sched = None
    _keep: tuple = ()

    def struct(self) -> _Sched:
        return self._struct

    def to_numpy(self) -> dict:
        """Logical-length host copies, keyed like oracle.mo_schedule."""
        a = {k: v.cpu().numpy() for k, v in self.arrays.items()}
        N, D, K, T = self.n_nodes, self.n_levels, self.table.n_ops, self.table.n_types
        return {"depth": a["depth"][:N], "group_off": a["group_off"][:(D + 1) * K + 1],
                "type_off": a["type_off"][:T + 1], "pool": a["pool"][:N], "pool_row": a["pool_row"][:N],
                "tlevel_off": a["tlevel_off"][:T * (D + 2)].reshape(T, D + 2),
                "label": a["label"][:6 * N].reshape(N, 2, 3), "order": a["order"][:N],
                "cons_off": a["cons_off"][:N + 1], "cons_edge": a["cons_edge"][:2 * N],
                "root_off": a["root_off"][:N + 1], "root_graph": a["root_graph"][:self.n_graphs],
                "leaf_seg": a["leaf_seg"][:self.n_leaf_segs + 1], "n_levels": D}


def _sizes(N, G, K, T):
    return {"depth": N, "group_off": (N + 1) * K + 1, "type_off": T + 1, "pool": N, "pool_row": N,
            "tlevel_off": T * (N + 2), "label": 6 * N, "order": N, "cons_off": N + 1, "cons_edge": 2 * N,
            "root_off": N + 1, "root_graph": G, "leaf_seg": N + 1, "leaf_order": N}


def schedule(table, op, child, token, root, stream=None) -> MoSchedule:
    """fold_mo_schedule over int32 device tensors op[N], child[N,2], token[N], root[G]. The
    schedule keeps references to them (the executor reads the graph arrays)."""
    L = load()
    dev = op.device
    for x in (op, child, token, root):
        assert x.dtype == torch.int32 and x.is_cuda and x.is_contiguous()
    ts = table_struct(table)
    N, G = int(op.shape[0]), int(root.shape[0])
    sizes = _sizes(N, G, ts.n_ops, ts.n_types)
    offs, o = {}, 0
    for k, n in sizes.items():
        offs[k] = (o, max(n, 1))
        o += (max(n, 1) + 63) // 64 * 64
    buf = torch.empty(o, dtype=torch.int32, device=dev)
    arrays = {k: buf[a:a + n] for k, (a, n) in offs.items()}
    host = np.zeros((N + 1) * ts.n_ops + 1, np.int32)
    ws_bytes = int(L.fold_mo_schedule_workspace(ctypes.byref(ts), N, G))
    ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    g = _Graphs(N, G, op.data_ptr(), child.data_ptr(), token.data_ptr(), root.data_ptr())
    base = buf.data_ptr()
    s = _Sched(*[base + 4 * offs[k][0] for k in _ARRAYS], host.ctypes.data, 0, 0, 0, 0, None, None, None, None)
    fold._check(L.fold_mo_schedule(ctypes.byref(ts), ctypes.byref(g), ctypes.byref(s), ctypes.c_void_p(ws.data_ptr()),
                                   ws_bytes, fold._stream(stream)), "fold_mo_schedule")
    return MoSchedule(ts, arrays, host, s.n_nodes, s.n_graphs, s.n_levels, s.n_leaf_segs, _struct=s,
                      _keep=(buf, op, child, token, root, host))


@dataclasses.dataclass
class MoModel:
    """Per-op parameters (device fp32): EMBED ops (E,), cell ops (U, b) — the layout of
    fold_mo.h (and of foldgen.make_mo_params)."""
    params: list
    prec: str = "fp32"

    def struct(self) -> _Model:
        m = _Model()
        m.prec = PREC[self.prec]
        for o, blk in enumerate(self.params):
            for x in blk:
                assert x.dtype == torch.float32 and x.is_cuda and x.is_contiguous()
            if len(blk) == 1:
                m.E[o] = blk[0].data_ptr()
            else:
                m.U[o], m.b[o] = blk[0].data_ptr(), blk[1].data_ptr()
        return m


def forward(sched: MoSchedule, model: MoModel, stream=None):
    """fold_mo_forward: (h_root [G, S_max] fp32, acts buffer)."""
    L = load()
    ts, ss, ms = sched.table, sched.struct(), model.struct()
    dev = model.params[0][0].device
    nacts = int(L.fold_mo_acts_bytes(ctypes.byref(ts), ctypes.byref(ss)))
    acts = torch.empty(max(nacts, 16), dtype=torch.uint8, device=dev)
    nws = int(L.fold_mo_forward_workspace(ctypes.byref(ts), ctypes.byref(ss)))
    ws = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev)
    smax = max(int(ts.S[i]) for i in range(ts.n_types))
    h_root = torch.empty((sched.n_graphs, smax), dtype=torch.float32, device=dev)
    fold._check(L.fold_mo_forward(ctypes.byref(ts), ctypes.byref(ss), ctypes.byref(ms), ctypes.c_void_p(acts.data_ptr()),
                                  fold._ptr(h_root), ctypes.c_void_p(ws.data_ptr()), nws, fold._stream(stream)),
                "fold_mo_forward")
    return h_root, acts


def backward(sched: MoSchedule, model: MoModel, acts: torch.Tensor, dh_root: torch.Tensor, grads=None,
             accumulate: bool = False, stream=None):
    """fold_mo_backward: per-op gradients shaped like model.params ((dE,) or (dU, db))."""
    L = load()
    ts, ss, ms = sched.table, sched.struct(), model.struct()
    dev = model.params[0][0].device
    assert dh_root.dtype == torch.float32 and dh_root.is_cuda and dh_root.is_contiguous()
    if grads is None:
        grads = [tuple(torch.empty_like(x) for x in blk) for blk in model.params]
    g = _Grads()
    g.accumulate = 1 if accumulate else 0
    for o, blk in enumerate(grads):
        if len(blk) == 1:
            g.dE[o] = blk[0].data_ptr()
        else:
            g.dU[o], g.db[o] = blk[0].data_ptr(), blk[1].data_ptr()
    nws = int(L.fold_mo_backward_workspace(ctypes.byref(ts), ctypes.byref(ss)))
    ws = torch.empty(max(nws, 16), dtype=torch.uint8, device=dev)
    fold._check(L.fold_mo_backward(ctypes.byref(ts), ctypes.byref(ss), ctypes.byref(ms), ctypes.c_void_p(acts.data_ptr()),
                                   fold._ptr(dh_root), ctypes.byref(g), ctypes.c_void_p(ws.data_ptr()), nws,
                                   fold._stream(stream)), "fold_mo_backward")
    return grads
