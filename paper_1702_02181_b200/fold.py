"""Thin Python binding over libfold.so (include/fold.h) — argument marshalling only.

Every step of the hot path (schedule, forward, backward, SGD) runs in the library's
CUDA kernels; PyTorch supplies device memory (torch.empty on cuda) and the stream.
There is no CPU fallback: if libfold.so is missing or the device is not sm_100,
the calls raise.

    sched = schedule(op, child, token, root, vocab)            # fold_schedule
    h_root, c_root, acts = forward(sched, model)               # fold_forward
    dU, db, dE = backward(sched, model, acts, dh_root)         # fold_backward
    sgd_update(param, grad, lr)                                # fold_sgd_update
"""
from __future__ import annotations

import ctypes
import dataclasses
import os

import numpy as np
import torch

from . import build as _build

OK = 0
STATUS = {0: "OK", 1: "INVALID", 2: "CHILD_RANGE", 3: "ARITY", 4: "TOKEN_RANGE", 5: "ROOT_RANGE",
          6: "CYCLE", 7: "WORKSPACE", 8: "CUDA", 9: "MISMATCH", 10: "OP_RANGE", 11: "UNSUPPORTED",
          12: "LEVEL", 13: "TYPE"}
CELLS = {"treernn": 0, "treelstm": 1}
PRECS = {"fp32": 0, "tf32": 1, "bf16": 2}

_i32p = ctypes.POINTER(ctypes.c_int32)
_f32p = ctypes.POINTER(ctypes.c_float)


class _Graphs(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int32), ("n_graphs", ctypes.c_int32), ("vocab", ctypes.c_int32),
                ("op", ctypes.c_void_p), ("child", ctypes.c_void_p), ("token", ctypes.c_void_p),
                ("root", ctypes.c_void_p), ("level", ctypes.c_void_p)]


_SCHED_ARRAYS = ("depth", "perm", "rank", "gather", "level_off", "group_off", "cons_off", "cons_edge",
                 "leaf_perm", "tok_seg", "root_row", "root_perm", "leaf_token")


class _Sched(ctypes.Structure):
    _fields_ = [(k, ctypes.c_void_p) for k in _SCHED_ARRAYS] + [
        ("level_off_host", ctypes.c_void_p),
        ("n_nodes", ctypes.c_int32), ("n_graphs", ctypes.c_int32), ("n_levels", ctypes.c_int32),
        ("n_leaves", ctypes.c_int32), ("n_cells", ctypes.c_int32), ("n_tok_segs", ctypes.c_int32),
        ("tree_like", ctypes.c_int32)]


class _Model(ctypes.Structure):
    _fields_ = [("cell", ctypes.c_int32), ("prec", ctypes.c_int32), ("S", ctypes.c_int32),
                ("vocab", ctypes.c_int32), ("U", ctypes.c_void_p), ("b", ctypes.c_void_p),
                ("E", ctypes.c_void_p)]


class _ActsLayout(ctypes.Structure):
    _fields_ = [("bytes", ctypes.c_size_t), ("h_off", ctypes.c_size_t), ("c_off", ctypes.c_size_t),
                ("g_off", ctypes.c_size_t), ("ld", ctypes.c_int32), ("h_elem_bytes", ctypes.c_int32)]


class _Grads(ctypes.Structure):
    _fields_ = [("dU", ctypes.c_void_p), ("db", ctypes.c_void_p), ("dE", ctypes.c_void_p),
                ("accumulate", ctypes.c_int32), ("sweep_done_event", ctypes.c_void_p)]


class _Sst(ctypes.Structure):
    _fields_ = [("W", ctypes.c_void_p), ("Ws", ctypes.c_void_p), ("bs", ctypes.c_void_p), ("label", ctypes.c_void_p),
                ("n_classes", ctypes.c_int32)]


class _SstGrads(ctypes.Structure):
    _fields_ = [("dW", ctypes.c_void_p), ("dWs", ctypes.c_void_p), ("dbs", ctypes.c_void_p)]


_lib = None


def lib_path() -> str:
    return _build.LIB_PATH


def load() -> ctypes.CDLL:
    """Load libfold.so (built by __graft_entry__.build() / `python -m paper_1702_02181_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_build.LIB_PATH):
        raise ImportError(f"libfold.so not built at {_build.LIB_PATH}; run `python -m paper_1702_02181_b200.build`")
    L = ctypes.CDLL(_build.LIB_PATH)
    vp, sz, i32 = ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int32
    L.fold_schedule_workspace.restype = sz
    L.fold_schedule_workspace.argtypes = [i32, i32]
    L.fold_schedule.restype = i32
    L.fold_schedule.argtypes = [ctypes.POINTER(_Graphs), ctypes.POINTER(_Sched), vp, sz, vp]
    L.fold_set_reserved_sms.restype = i32
    L.fold_set_reserved_sms.argtypes = [i32]
    L.fold_schedule_ex.restype = i32
    L.fold_schedule_ex.argtypes = [ctypes.POINTER(_Graphs), ctypes.POINTER(_Sched), vp, sz, vp, i32]
    L.fold_acts_layout.restype = i32
    L.fold_acts_layout.argtypes = [ctypes.POINTER(_Sched), ctypes.POINTER(_Model), ctypes.POINTER(_ActsLayout)]
    L.fold_forward_workspace.restype = sz
    L.fold_forward_workspace.argtypes = [ctypes.POINTER(_Sched), ctypes.POINTER(_Model)]
    L.fold_forward.restype = i32
    L.fold_forward.argtypes = [ctypes.POINTER(_Sched), ctypes.POINTER(_Model), vp, vp, vp, vp, sz, vp]
    L.fold_backward_workspace.restype = sz
    L.fold_backward_workspace.argtypes = [ctypes.POINTER(_Sched), ctypes.POINTER(_Model)]
    L.fold_backward.restype = i32
    L.fold_backward.argtypes = [ctypes.POINTER(_Sched), ctypes.POINTER(_Model), vp, vp, vp,
                                ctypes.POINTER(_Grads), vp, sz, vp]
    L.fold_touched_rows.restype = i32
    L.fold_touched_rows.argtypes = [ctypes.POINTER(_Sched), vp, vp]
    L.fold_gather_rows.restype = i32
    L.fold_gather_rows.argtypes = [vp, ctypes.c_int64, vp, i32, i32, vp, vp]
    L.fold_scatter_add_rows.restype = i32
    L.fold_scatter_add_rows.argtypes = [vp, vp, i32, i32, vp, ctypes.c_int64, vp]
    L.fold_sgd_update.restype = i32
    L.fold_sgd_update.argtypes = [vp, vp, ctypes.c_int64, ctypes.c_float, vp]
    L.fold_status_string.restype = ctypes.c_char_p
    L.fold_status_string.argtypes = [i32]
    L.fold_last_error_detail.restype = i32
    L.fold_last_error_context.restype = i32
    L.fold_last_error_context.argtypes = [ctypes.POINTER(ctypes.c_int32)] * 3
    L.fold_abi_version.restype = i32
    L.fold_device_check.restype = i32
    L.fold_launch_count.restype = ctypes.c_int64
    L.fold_launch_count.argtypes = [i32]
    L.fold_profile_enable.restype = None
    L.fold_profile_enable.argtypes = [i32]
    L.fold_profile_enable_classes.restype = None
    L.fold_profile_enable_classes.argtypes = [ctypes.c_uint32]
    L.fold_profile_read.restype = i32
    L.fold_profile_read.argtypes = [i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int64)]
    L.fold_debug_fwd_trace.argtypes = [vp, i32]
    L.fold_debug_fwd_trace.restype = i32
    L.fold_debug_bwd_trace.argtypes = [vp, i32]
    L.fold_debug_bwd_trace.restype = i32
    L.fold_debug_sched_trace.argtypes = [vp]
    L.fold_debug_sched_trace.restype = i32
    SP, MP, SQ = ctypes.POINTER(_Sched), ctypes.POINTER(_Model), ctypes.POINTER(_Sst)
    L.fold_sst_acts_layout.restype = i32
    L.fold_sst_acts_layout.argtypes = [SP, MP, SQ, ctypes.POINTER(_ActsLayout)]
    L.fold_sst_forward_workspace.restype = sz
    L.fold_sst_forward_workspace.argtypes = [SP, MP, SQ]
    L.fold_sst_backward_workspace.restype = sz
    L.fold_sst_backward_workspace.argtypes = [SP, MP, SQ]
    L.fold_sst_forward.restype = i32
    L.fold_sst_forward.argtypes = [SP, MP, SQ, vp, vp, vp, sz, vp]
    L.fold_sst_backward.restype = i32
    L.fold_sst_backward.argtypes = [SP, MP, SQ, vp, ctypes.POINTER(_Grads), ctypes.POINTER(_SstGrads), vp, sz, vp]
    L.fold_debug_gemm_tf32.restype = i32
    L.fold_debug_gemm_tf32.argtypes = [vp, ctypes.c_int64, i32, vp, ctypes.c_int64, i32, i32, i32, i32, vp,
                                       ctypes.c_int64, i32, i32, vp, ctypes.c_int64, vp]
    L.fold_debug_gemm_tf32_ws.restype = ctypes.c_int64
    L.fold_debug_gemm_tf32_ws.argtypes = [i32, i32, i32]
    _lib = L
    return L


EXPORTED = ("fold_schedule_workspace", "fold_schedule", "fold_schedule_ex", "fold_set_reserved_sms", "fold_acts_layout", "fold_forward_workspace",
            "fold_forward", "fold_backward_workspace", "fold_backward", "fold_sgd_update",
            "fold_status_string", "fold_last_error_detail", "fold_last_error_context", "fold_abi_version", "fold_device_check",
            "fold_launch_count", "fold_profile_enable", "fold_profile_enable_classes", "fold_profile_read", "fold_debug_fwd_trace", "fold_debug_bwd_trace",
            "fold_debug_sched_trace", "fold_debug_gemm_tf32", "fold_debug_gemm_tf32_ws",
            "fold_sst_acts_layout", "fold_sst_forward_workspace", "fold_sst_forward", "fold_sst_backward_workspace",
            "fold_sst_backward", "fold_touched_rows", "fold_gather_rows", "fold_scatter_add_rows")

PROF_CLASSES = ("schedule", "embed_fwd", "cell_fwd", "bwd_pointwise", "gemm_dA", "gemm_dU", "embed_bwd",
                "db_colsum", "sgd", "weight_prep", "root_out")


def profile_enable(on: bool = True, classes=None):
    """classes: names from PROF_CLASSES to record (None: all)."""
    if on and classes is not None:
        load().fold_profile_enable_classes(sum(1 << PROF_CLASSES.index(c) for c in set(classes)))
    else:
        load().fold_profile_enable(1 if on else 0)


def profile_read() -> dict:
    """{class: (total_ms, launches)} for the launches bracketed since profile_enable()."""
    n = len(PROF_CLASSES)
    ms = (ctypes.c_double * n)()
    cnt = (ctypes.c_int64 * n)()
    _check(load().fold_profile_read(n, ms, cnt), "fold_profile_read")
    return {PROF_CLASSES[i]: (float(ms[i]), int(cnt[i])) for i in range(n)}


class FoldError(RuntimeError):
    def __init__(self, status: int, what: str, detail: int = -1, depth: int = -1, op: int = -1):
        super().__init__(f"{what}: FOLD_E_{STATUS.get(status, status)} (node {detail}, depth {depth}, op {op})")
        self.status = STATUS.get(status, status)
        self.detail = detail
        self.depth = depth
        self.op = op


def last_error_context() -> tuple[int, int, int]:
    """(node, depth, op) of the last data-dependent fold_schedule error (fold.h)."""
    v = [ctypes.c_int32(-1) for _ in range(3)]
    load().fold_last_error_context(*(ctypes.byref(x) for x in v))
    return tuple(int(x.value) for x in v)


def _check(st: int, what: str):
    if st != OK:
        node, depth, op = last_error_context()
        raise FoldError(st, what, load().fold_last_error_detail(), depth, op)


def _ptr(t: torch.Tensor | None):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def set_reserved_sms(n: int) -> int:
    """fold_set_reserved_sms: SMs the persistent level kernels leave free (returns the old value)."""
    return int(load().fold_set_reserved_sms(int(n)))


def device_check():
    _check(load().fold_device_check(), "fold_device_check")


def launch_count(reset: bool = False) -> int:
    return int(load().fold_launch_count(1 if reset else 0))


# ----------------------------------------------------------------------------- schedule

class _LazyArrays(dict):
    """Views of the schedule arrays inside one device buffer, created on first access
    (`.buffer` is the allocation, e.g. for record_stream)."""

    def __init__(self, buf: torch.Tensor, offs: dict):
        super().__init__()
        self.buffer = buf
        self._offs = offs

    def __missing__(self, k):
        o, n = self._offs[k]
        v = self.buffer[o:o + n]
        self[k] = v
        return v

    def _all(self):
        for k in self._offs:
            self[k]
        return self

    def items(self):
        return dict.items(self._all())

    def values(self):
        return dict.values(self._all())

    def keys(self):
        return self._offs.keys()


@dataclasses.dataclass
class Schedule:
    """Device arrays of the executor-form schedule (fold.h) + host scalars."""
    arrays: dict
    level_off_host: np.ndarray
    n_nodes: int
    n_graphs: int
    n_levels: int
    n_leaves: int
    n_cells: int
    n_tok_segs: int
    tree_like: bool = False
    _struct: _Sched = None
    _host_buf: np.ndarray = None

    def struct(self) -> _Sched:
        return self._struct

    def to_numpy(self) -> dict:
        """Logical-length host copies (for tests): same keys/lengths as oracle.schedule."""
        a = {k: v.cpu().numpy() for k, v in self.arrays.items()}
        N, D = self.n_nodes, self.n_levels
        out = {"depth": a["depth"][:N], "perm": a["perm"][:N], "rank": a["rank"][:N],
               "gather": a["gather"][:2 * N].reshape(N, 2), "level_off": a["level_off"][:D + 2],
               "group_off": a["group_off"][:2 * (D + 1) + 1], "cons_off": a["cons_off"][:N + 1],
               "cons_edge": a["cons_edge"][:2 * self.n_cells], "leaf_perm": a["leaf_perm"][:self.n_leaves],
               "tok_seg": a["tok_seg"][:self.n_tok_segs + 1], "root_row": a["root_row"][:self.n_graphs],
               "root_perm": a["root_perm"][:self.n_graphs], "leaf_token": a["leaf_token"][:self.n_leaves],
               "n_levels": D, "n_leaves": self.n_leaves, "n_cells": self.n_cells,
               "n_tok_segs": self.n_tok_segs}
        return out


def _schedule_layout(N: int, G: int):
    sizes = {"depth": N, "perm": N, "rank": N, "gather": 2 * N, "level_off": N + 2, "group_off": 2 * N + 3,
             "cons_off": N + 1, "cons_edge": 2 * N, "leaf_perm": N, "tok_seg": N + 1, "root_row": G,
             "root_perm": G, "leaf_token": N}
    offs, o = {}, 0
    for k, n in sizes.items():  # each array 256-byte aligned
        offs[k] = (o, max(n, 1))
        o += (max(n, 1) + 63) // 64 * 64
    return offs, o


def schedule_buffer_len(n_nodes: int, n_graphs: int) -> int:
    """int32 elements of the device buffer `schedule(..., out=)` needs."""
    return _schedule_layout(int(n_nodes), int(n_graphs))[1]


def schedule(op: torch.Tensor, child: torch.Tensor, token: torch.Tensor, root: torch.Tensor, vocab: int,
             stream=None, workspace: torch.Tensor | None = None, level: torch.Tensor | None = None,
             out: torch.Tensor | None = None, max_blocks: int = 0) -> Schedule:
    """fold_schedule over int32 device tensors op[N], child[N,2], token[N], root[G];
    `level` = optional caller-fixed levels [N] (manual batching, fold.h fold_graphs.level);
    `out` = optional int32 device buffer of schedule_buffer_len(N, G) elements for the
    schedule arrays (else one is allocated); `max_blocks` > 0 caps the scheduler's grid
    (fold_schedule_ex: a schedule running beside other kernels)."""
    L = load()
    dev = op.device
    N, G = int(op.shape[0]), int(root.shape[0])
    for t in (op, child, token, root) + ((level,) if level is not None else ()):
        assert t.dtype == torch.int32 and t.is_cuda and t.is_contiguous()
    # one device buffer for all schedule arrays: a dozen small torch allocations cost more host
    # time than a small batch's whole schedule kernel
    offs, o = _schedule_layout(N, G)
    if out is not None:
        assert out.dtype == torch.int32 and out.is_cuda and out.numel() >= o
        buf = out
    else:
        buf = torch.empty(o, dtype=torch.int32, device=dev)
    arrays = _LazyArrays(buf, offs)
    host = np.zeros(N + 2, np.int32)
    ws_bytes = int(L.fold_schedule_workspace(N, G))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=dev)
    g = _Graphs(N, G, int(vocab), op.data_ptr(), child.data_ptr(), token.data_ptr(), root.data_ptr(),
                level.data_ptr() if level is not None else None)
    base = buf.data_ptr()
    s = _Sched(*[base + 4 * offs[k][0] for k in _SCHED_ARRAYS], host.ctypes.data, 0, 0, 0, 0, 0, 0, 0)
    if max_blocks:
        _check(L.fold_schedule_ex(ctypes.byref(g), ctypes.byref(s), ctypes.c_void_p(workspace.data_ptr()),
                                  ws_bytes, _stream(stream), int(max_blocks)), "fold_schedule_ex")
    else:
        _check(L.fold_schedule(ctypes.byref(g), ctypes.byref(s), ctypes.c_void_p(workspace.data_ptr()),
                               ws_bytes, _stream(stream)), "fold_schedule")
    return Schedule(arrays, host, s.n_nodes, s.n_graphs, s.n_levels, s.n_leaves, s.n_cells, s.n_tok_segs,
                    bool(s.tree_like), _struct=s, _host_buf=host)


# ----------------------------------------------------------------------------- model / acts

@dataclasses.dataclass
class Model:
    U: torch.Tensor   # [gates*S, 2S] fp32
    b: torch.Tensor   # [gates*S] fp32
    E: torch.Tensor   # [V, S] fp32
    cell: str = "treelstm"
    prec: str = "bf16"

    @property
    def S(self) -> int:
        return int(self.E.shape[1])

    def struct(self) -> _Model:
        for t in (self.U, self.b, self.E):
            assert t.dtype == torch.float32 and t.is_cuda and t.is_contiguous()
        return _Model(CELLS[self.cell], PRECS[self.prec], self.S, int(self.E.shape[0]),
                      self.U.data_ptr(), self.b.data_ptr(), self.E.data_ptr())


@dataclasses.dataclass
class Acts:
    buf: torch.Tensor
    layout: _ActsLayout

    def views(self, sched: Schedule, model: Model):
        """(H [N, ld], C [N, ld]) views into the activation buffer (pool-row order)."""
        N = sched.n_nodes
        lay = self.layout
        hdt = torch.bfloat16 if lay.h_elem_bytes == 2 else torch.float32
        H = self.buf[lay.h_off: lay.h_off + N * lay.ld * lay.h_elem_bytes].view(hdt).view(N, lay.ld)
        C = self.buf[lay.c_off: lay.c_off + N * lay.ld * 4].view(torch.float32).view(N, lay.ld)
        return H, C


class Workspace:
    """Reusable device scratch (grown on demand) so repeated steps do not re-allocate."""

    def __init__(self, device):
        self.device = device
        self.bufs = {}

    def get(self, name: str, nbytes: int) -> torch.Tensor:
        t = self.bufs.get(name)
        if t is None or t.numel() < nbytes:
            t = torch.empty(max(int(nbytes), 1), dtype=torch.uint8, device=self.device)
            self.bufs[name] = t
        return t


def forward(sched: Schedule, model: Model, stream=None, ws: Workspace | None = None,
            want_c: bool = True, h_root: torch.Tensor | None = None):
    L = load()
    dev = model.E.device
    ms = model.struct()
    lay = _ActsLayout()
    _check(L.fold_acts_layout(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(lay)), "fold_acts_layout")
    ws = ws or Workspace(dev)
    acts_buf = ws.get("acts", lay.bytes)
    fws = int(L.fold_forward_workspace(ctypes.byref(sched.struct()), ctypes.byref(ms)))
    fbuf = ws.get("fwd", fws)
    S, G = model.S, sched.n_graphs
    if h_root is None:
        h_root = torch.empty((G, S), dtype=torch.float32, device=dev)
    assert h_root.dtype == torch.float32 and h_root.is_contiguous() and h_root.numel() >= G * S
    c_root = torch.empty((G, S), dtype=torch.float32, device=dev) if want_c else None
    _check(L.fold_forward(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.c_void_p(acts_buf.data_ptr()),
                          _ptr(h_root), _ptr(c_root), ctypes.c_void_p(fbuf.data_ptr()), fws, _stream(stream)),
           "fold_forward")
    return h_root, c_root, Acts(acts_buf, lay)


def backward(sched: Schedule, model: Model, acts: Acts, dh_root: torch.Tensor, dc_root: torch.Tensor | None = None,
             grads=None, accumulate: bool = False, stream=None, ws: Workspace | None = None,
             sweep_done: torch.cuda.Event | None = None):
    """fold_backward; `sweep_done` (optional torch.cuda.Event) is recorded once the level sweep
    is enqueued, before the weight-gradient GEMM (fold.h fold_grads.sweep_done_event)."""
    L = load()
    dev = model.E.device
    ms = model.struct()
    if grads is None:
        grads = (torch.empty_like(model.U), torch.empty_like(model.b), torch.empty_like(model.E))
    dU, db, dE = grads
    ev = None
    if sweep_done is not None:
        sweep_done.record(torch.cuda.current_stream() if stream is None else stream)  # materialise the event
        ev = sweep_done.cuda_event
    gs = _Grads(dU.data_ptr(), db.data_ptr(), dE.data_ptr(), 1 if accumulate else 0, ev)
    ws = ws or Workspace(dev)
    bws = int(L.fold_backward_workspace(ctypes.byref(sched.struct()), ctypes.byref(ms)))
    bbuf = ws.get("bwd", bws)
    assert dh_root.dtype == torch.float32 and dh_root.is_contiguous()
    _check(L.fold_backward(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.c_void_p(acts.buf.data_ptr()),
                           _ptr(dh_root), _ptr(dc_root), ctypes.byref(gs), ctypes.c_void_p(bbuf.data_ptr()), bws,
                           _stream(stream)), "fold_backward")
    return dU, db, dE


# ----------------------------------------------------------------------------- §3.5 model (NEXT-2)

@dataclasses.dataclass
class SstHead:
    """The §3.5 model's extra parameters (fold.h fold_sst): leaf input weights W [3S][S]
    (row blocks i, o, u), per-node classifier Ws [C][S], bs [C]; labels [n_nodes] int32 in
    node-id order."""
    W: torch.Tensor
    Ws: torch.Tensor
    bs: torch.Tensor
    label: torch.Tensor

    def struct(self) -> _Sst:
        for t in (self.W, self.Ws, self.bs):
            assert t.dtype == torch.float32 and t.is_cuda and t.is_contiguous()
        assert self.label.dtype == torch.int32 and self.label.is_cuda and self.label.is_contiguous()
        return _Sst(self.W.data_ptr(), self.Ws.data_ptr(), self.bs.data_ptr(), self.label.data_ptr(),
                    int(self.bs.shape[0]))


def sst_forward(sched: Schedule, model: Model, head: SstHead, stream=None, ws: Workspace | None = None):
    """fold_sst_forward: (loss [1] device tensor, Acts) of the §3.5 model."""
    L = load()
    ms, qs = model.struct(), head.struct()
    lay = _ActsLayout()
    _check(L.fold_sst_acts_layout(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(qs), ctypes.byref(lay)),
           "fold_sst_acts_layout")
    ws = ws or Workspace(model.E.device)
    acts = ws.get("sst_acts", lay.bytes)
    n = int(L.fold_sst_forward_workspace(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(qs)))
    fbuf = ws.get("sst_fwd", n)
    loss = torch.empty(1, dtype=torch.float32, device=model.E.device)
    _check(L.fold_sst_forward(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(qs),
                              ctypes.c_void_p(acts.data_ptr()), _ptr(loss), ctypes.c_void_p(fbuf.data_ptr()), n,
                              _stream(stream)), "fold_sst_forward")
    return loss, Acts(acts, lay)


def sst_backward(sched: Schedule, model: Model, head: SstHead, acts: Acts, grads=None, accumulate: bool = False,
                 stream=None, ws: Workspace | None = None):
    """fold_sst_backward: (dU, db, dE, dW, dWs, dbs) of the summed per-node cross-entropy."""
    L = load()
    ms, qs = model.struct(), head.struct()
    if grads is None:
        grads = tuple(torch.empty_like(t) for t in (model.U, model.b, model.E, head.W, head.Ws, head.bs))
    dU, db, dE, dW, dWs, dbs = grads
    gs = _Grads(dU.data_ptr(), db.data_ptr(), dE.data_ptr(), 1 if accumulate else 0, None)
    sg = _SstGrads(dW.data_ptr(), dWs.data_ptr(), dbs.data_ptr())
    ws = ws or Workspace(model.E.device)
    n = int(L.fold_sst_backward_workspace(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(qs)))
    bbuf = ws.get("sst_bwd", n)
    _check(L.fold_sst_backward(ctypes.byref(sched.struct()), ctypes.byref(ms), ctypes.byref(qs),
                               ctypes.c_void_p(acts.buf.data_ptr()), ctypes.byref(gs), ctypes.byref(sg),
                               ctypes.c_void_p(bbuf.data_ptr()), n, _stream(stream)), "fold_sst_backward")
    return grads


def debug_gemm_tf32(A: torch.Tensor, B: torch.Tensor, M: int, N: int, K: int, a_mn: bool, b_mn: bool,
                    npass: int, C: torch.Tensor | None = None, accumulate: bool = False, stream=None):
    """fold_debug_gemm_tf32 (test hook): C = A * B on the tcgen05 TF32 GEMM of the FP32 /
    TF32 modes. A: [M][K] (or [K][M] if a_mn), B: [N][K] (or [K][N] if b_mn), fp32 2-D."""
    L = load()
    if C is None:
        C = torch.empty((M, N), dtype=torch.float32, device=A.device)
    nws = int(L.fold_debug_gemm_tf32_ws(M, N, K))
    ws = torch.empty(max(nws, 1), dtype=torch.float32, device=A.device)
    _check(L.fold_debug_gemm_tf32(_ptr(A), A.stride(0), int(a_mn), _ptr(B), B.stride(0), int(b_mn), M, N, K,
                                  _ptr(C), C.stride(0), int(accumulate), npass, _ptr(ws), nws, _stream(stream)),
           "fold_debug_gemm_tf32")
    return C


def sgd_update(param: torch.Tensor, grad: torch.Tensor, lr: float, stream=None):
    assert param.dtype == torch.float32 and grad.dtype == torch.float32
    _check(load().fold_sgd_update(_ptr(param), _ptr(grad), param.numel(), ctypes.c_float(lr), _stream(stream)),
           "fold_sgd_update")


def touched_rows(sched: Schedule, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """fold_touched_rows: int32 device tensor of the batch's distinct tokens (ascending)."""
    n = sched.n_tok_segs
    dev = sched.arrays.buffer.device if hasattr(sched.arrays, "buffer") else None
    if out is None:
        out = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _check(load().fold_touched_rows(ctypes.byref(sched.struct()), _ptr(out), _stream(stream)), "fold_touched_rows")
    return out[:n]


def gather_rows(src: torch.Tensor, rows: torch.Tensor, out: torch.Tensor, stream=None):
    """fold_gather_rows: out[i] = src[rows[i]] (zero rows where rows[i] < 0)."""
    n, S = int(rows.numel()), int(src.shape[1])
    _check(load().fold_gather_rows(_ptr(src), src.stride(0), _ptr(rows), n, S, _ptr(out), _stream(stream)),
           "fold_gather_rows")
    return out


def scatter_add_rows(src: torch.Tensor, rows: torch.Tensor, dst: torch.Tensor, stream=None):
    """fold_scatter_add_rows: dst[rows[i]] += src[i] (distinct rows; rows[i] < 0 skipped)."""
    n, S = int(rows.numel()), int(dst.shape[1])
    _check(load().fold_scatter_add_rows(_ptr(src), _ptr(rows), n, S, _ptr(dst), dst.stride(0), _stream(stream)),
           "fold_scatter_add_rows")
    return dst


def graphs_to_device(gr, device="cuda", non_blocking=False):
    """int32 device tensors (op, child, token, root) from a foldgen.Graphs-like object."""
    conv = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.int32)).to(device, non_blocking=non_blocking)
    return conv(gr.op), conv(gr.child.reshape(-1, 2)), conv(gr.token), conv(gr.root)
