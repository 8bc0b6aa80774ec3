#!/usr/bin/env python
"""bench.py — TreeLSTM tree nodes/s, forward + backward (BASELINE.json metric), B200.

One step = the whole hot path of SURVEY.md §8(a) over one batch of synthetic trees:
fold_schedule (validate, depths, (depth, op) grouping, gather vectors, consumer CSR) ->
fold_forward (embedding level + one fused tcgen05 cell kernel per depth) ->
fold_backward (reverse level sweep + weight-gradient GEMM) -> NCCL all_reduce of the
flat [dU | db | dE] gradient (N > 1) -> fold_sgd_update.

Default workload (N = 1): BASELINE configs[1] — complete 128-leaf binary trees
("tree size is 128"), B = 1024 trees, state S = 1024, vocab 16384,
TreeLSTM, BF16 operands / fp32 accumulation. With N > 1 (torchrun) every rank runs
its own B-tree batch (weak scaling) and the gradients are all-reduced.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import foldgen  # noqa: E402

METRIC = "TreeLSTM tree nodes/sec fwd+bwd"
UNIT = "nodes/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["fold", "reference"], default="fold")
    ap.add_argument("--model", choices=["r1", "sst", "mo"], default="r1",
                    help="r1: the headline TreeLSTM (leaf = embedding lookup, root gradient); sst: the §3.5 "
                         "sentiment model (NEXT-2)")
    ap.add_argument("--config", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--batch", type=int, default=None, help="trees per GPU (default: config's full size)")
    ap.add_argument("--prec", default="bf16", choices=["bf16", "tf32", "fp32"])
    ap.add_argument("--cell", default=None, choices=["treelstm", "treernn"])
    ap.add_argument("--lr", type=float, default=1e-4)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--prof", default="roofline", choices=["roofline", "all"],
                    help="kernel classes bracketed by CUDA events inside the timed region: only the "
                         "roofline's tensor classes (default; the per-class breakdown then comes from "
                         "a separate profiled pass after it) or all classes")
    ap.add_argument("--reserve-sms", type=int, default=24,
                    help="SMs the level kernels leave to a small batch's pipelined schedule")
    ap.add_argument("--reserve-max-work", type=float, default=2e10,
                    help="largest nodes x S^2 whose pipelined schedule gets --reserve-sms SMs")
    ap.add_argument("--sched-bg-blocks", type=int, default=32,
                    help="scheduler CTAs of a pipelined schedule that overlaps the weight-gradient GEMM")
    ap.add_argument("--no-c5-strong", action="store_true", help="N > 1: skip the C5 strong-scaling record")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-batch1", action="store_true")
    ap.add_argument("--no-clocks", action="store_true")
    ap.add_argument("--ref-trees", type=int, default=1, help="trees per oracle step (--impl reference)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the nodes/s vs batch-size sweep")
    ap.add_argument("--pipeline", default="on", choices=["on", "off"],
                    help="run the next batch's fold_schedule on a side stream while the current batch executes "
                         "(batches of more than 131072 nodes or 64 levels: after its level sweep)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: testing the multi-rank path on one GPU)")
    ap.add_argument("--exchange", default="auto", choices=["auto", "sparse", "dense"],
                    help="N > 1: dE exchange (auto: sparse all-gather of the touched rows when cheaper)")
    ap.add_argument("--no-table1", action="store_true",
                    help="skip the unbatched baseline and the PAPER.md Table 1 reproduction")
    return ap.parse_args()


DEFAULT_B = {"c1": None, "c2": 1024, "c3": 1024, "c4": 1024, "c5": 8192}


def workload(args, rank=0, world=1):
    """C2/C3/C4: every rank runs its own B-tree batch (weak scaling, seed + rank). C5: ONE
    global batch of B trees sharded across the ranks by node count (strong scaling,
    SURVEY §8(e)); returns (graphs of this rank, cell, S, description, global node count)."""
    cfg = args.config
    B = args.batch or DEFAULT_B[cfg]
    cell = args.cell or ("treernn" if cfg == "c1" else "treelstm")
    S = foldgen.CONFIG_STATE[cfg]
    if cfg == "c5":
        from paper_1702_02181_b200 import dp
        full = foldgen.make_config(cfg, B)
        gr = dp.shard(full, rank, world)
        desc = (f"C5 random-split 128-leaf trees, global batch {full.n_graphs} sharded by node count over "
                f"{world} GPU(s), TreeLSTM S=1024, V=16384")
        return gr, cell, S, desc, full.n_nodes
    gr = foldgen.make_config(cfg, B, seed=foldgen.GRAPH_SEED + rank)
    desc = {
        "c1": "C1 TreeRNN, 8 random-split trees (<=16 leaves), S=16, V=32",
        "c2": f"C2 complete-128-leaf binary trees, B={gr.n_graphs}/GPU, TreeLSTM S=1024, V=16384",
        "c3": f"C3 parse-shaped trees (1-60 leaves), B={gr.n_graphs}/GPU, TreeLSTM S=300, V=16384 Zipf",
        "c4": f"C4 chain-256 (depth 256), B={gr.n_graphs}/GPU, TreeLSTM S=1024",
    }[cfg]
    return gr, cell, S, desc, world * gr.n_nodes


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """SM clock, power and clock-event (throttle) reasons sampled DURING the timed region:
    NVML polled every ~5 ms from a thread (the timed region is ~0.1 s, shorter than
    nvidia-smi's sampling period); nvidia-smi -lms 200 as a fallback."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_slowdown"}

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.stop_flag = False
        self.t = None
        self.nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nvml = None

    def _poll(self):
        nv = self.nvml
        while not self.stop_flag:
            try:
                self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            except Exception:
                pass
            time.sleep(0.005)

    def start(self):
        if self.nvml is None:
            return
        self.t = threading.Thread(target=self._poll, daemon=True)
        self.t.start()

    def stop(self):
        if self.t is None:
            return None
        self.stop_flag = True
        self.t.join(timeout=1)
        if not self.rows:
            return None
        reasons = set()
        for _, r in self.rows:
            for bit, name in self.REASONS.items():
                if r & bit:
                    reasons.add(name)
        sm = [c for c, _ in self.rows]
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "sm_min_mhz": min(sm),
                "reasons": sorted(reasons), "samples": len(sm), "source": "nvml, ~5 ms polling"}


# ============================================================================ fold arm

def run_fold(args):
    import torch
    import torch.distributed as dist

    from paper_1702_02181_b200 import dp, fold

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    local = local % max(torch.cuda.device_count(), 1)  # (gloo test runs: several ranks per GPU)
    if world > 1:
        if args.backend == "nccl":
            # communicator setup (ranks, NVLink / NVLS transport) in the log, on stderr
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    fold.device_check()

    gr, cell, S, desc, global_nodes = workload(args, rank, world)
    strong = args.config == "c5"
    V = gr.vocab
    gates = foldgen.gates_of(cell)
    N_nodes = gr.n_nodes
    n_cells = int((gr.op == 1).sum())
    p = foldgen.make_params(cell, S, V)
    # flat parameter / gradient buffers: one all_reduce and one SGD launch per step
    nU, nb, nE = p.U.size, p.b.size, p.E.size
    flat_p = torch.empty(nU + nb + nE, dtype=torch.float32, device=dev)
    flat_g = torch.zeros_like(flat_p)
    U = flat_p[:nU].view(p.U.shape); b = flat_p[nU:nU + nb]; E = flat_p[nU + nb:].view(p.E.shape)
    U.copy_(torch.from_numpy(p.U)); b.copy_(torch.from_numpy(p.b)); E.copy_(torch.from_numpy(p.E))
    dU = flat_g[:nU].view(p.U.shape); db = flat_g[nU:nU + nb]; dE = flat_g[nU + nb:].view(p.E.shape)
    model = fold.Model(U, b, E, cell=cell, prec=args.prec)
    g_host = foldgen.make_upstream(gr.n_graphs, S)
    g_dev = torch.from_numpy(g_host).to(dev)
    op, child, token, root = fold.graphs_to_device(gr, dev)
    ws = fold.Workspace(dev)
    sched_ws = torch.empty(1, dtype=torch.uint8, device=dev)

    # the data-parallel exchange (N > 1): all_reduce of [dU | db]; dE as the all-gathered
    # touched rows when that moves fewer bytes than its dense all_reduce (dp.exchange_plan,
    # SURVEY §8(f) NEXT-4), else dense. The mode of the last step is reported.
    xrows = torch.empty(max(N_nodes, 1), dtype=torch.int32, device=dev)
    xscratch = {}
    xmode = ["none"]

    def exchange(sc):
        rows = fold.touched_rows(sc, out=xrows)
        xmode[0] = dp.exchange_grads(flat_g, nU + nb, dE, rows, mode=args.exchange, scratch=xscratch)

    def step(op, child, token, root, g, level=None, train=True):
        nonlocal sched_ws
        s = fold.schedule(op, child, token, root, V, workspace=sched_ws, level=level)
        h, c, acts = fold.forward(s, model, ws=ws, want_c=False)
        if not train:
            return h
        fold.backward(s, model, acts, g, grads=(dU, db, dE), ws=ws)
        if world > 1:
            exchange(s)
        fold.sgd_update(flat_p, flat_g, args.lr)
        return h

    # Pipelined steps ("overlap fold_schedule(k+1) with execution of
    # batch k"): the next batch's schedule is computed on a side stream right after batch k's
    # forward / backward / SGD are enqueued, so its kernel fills the gaps of batch k's tail
    # and its one host sync no longer idles the GPU; batch k+1's forward waits on its event.
    # Every step still schedules its own batch (K schedules in K timed steps).
    side_stream = torch.cuda.Stream(device=dev) if args.pipeline != "off" else None
    pipe_max_nodes = 131072
    side = None  # set per timed workload by use_pipeline()

    gate = [None]  # event the next schedule waits for (None: start right away)

    def use_pipeline(n_nodes, n_levels):
        # measured: small batches gain most when the next schedule starts right
        # away; with a few hundred thousand nodes or hundreds of levels its cooperative kernel
        # must not take SMs from the persistent level kernels (which own every SM), so it is
        # gated on the previous batch's level sweep and overlaps only its weight-gradient GEMM
        nonlocal side
        side = side_stream if args.pipeline != "off" else None
        small = n_nodes <= pipe_max_nodes and n_levels <= 64
        gate[0] = None if small else sweep_done
        # a small batch's next schedule starts right away: when the level kernels have little
        # GEMM work (~ nodes x S^2 <= args.reserve_max_work; they are latency-bound there) they
        # leave it SMs so it runs beside them (fold_set_reserved_sms; measured with 24 SMs:
        # C3 B=1024 1.135 -> 1.077 ms, C2 B=64 0.924 -> 0.91 ms; C2 B=256 (6.8e10) +7%, so
        # larger work reserves none; 16 SMs: C2 B=64 0.83 ms but C3 1.15 ms)
        fold.set_reserved_sms(args.reserve_sms if (small and side is not None
                                                   and n_nodes * S * S <= args.reserve_max_work) else 0)
        return side is not None

    sweep_done = torch.cuda.Event()  # re-recorded by every fold_backward after its level sweep
    # no allocation inside the timed loops: three rotating schedule buffers (a buffer is
    # rewritten only after the step that read it has finished on the compute stream) and one
    # root-state output
    sbuf = [torch.empty(fold.schedule_buffer_len(N_nodes, gr.n_graphs), dtype=torch.int32, device=dev)
            for _ in range(3)]
    sbuf_free = [torch.cuda.Event() for _ in range(3)]
    sbuf_used = [False] * 3
    slot = [0]
    h_root_buf = torch.empty((gr.n_graphs, S), dtype=torch.float32, device=dev)

    def schedule_async(op, child, token, root, copies=(), level=None, after=None):
        nonlocal h_root_buf
        need = fold.schedule_buffer_len(op.shape[0], root.shape[0])
        if sbuf[0].numel() < need:  # a larger workload (Table 1 / sweeps, outside timed loops)
            torch.cuda.synchronize()
            for k in range(3):
                sbuf[k] = torch.empty(need, dtype=torch.int32, device=dev)
        if h_root_buf.shape[0] < root.shape[0]:
            torch.cuda.synchronize()
            h_root_buf = torch.empty((root.shape[0], S), dtype=torch.float32, device=dev)
        i = slot[0]
        slot[0] = (i + 1) % 3
        if side is None:
            for d, h in copies:
                d.copy_(h, non_blocking=True)
            return fold.schedule(op, child, token, root, V, workspace=sched_ws, level=level, out=sbuf[i]), None, i
        with torch.cuda.stream(side):
            if sbuf_used[i]:
                side.wait_event(sbuf_free[i])
            if after is not None:  # start once the previous batch's level sweep is done, so the
                side.wait_event(after)  # scheduler overlaps its weight-gradient GEMM, not the
                # persistent level kernels (which own every SM)
            for d, h in copies:
                d.copy_(h, non_blocking=True)
            # gated (it overlaps the weight-gradient GEMM): a few scheduler CTAs leave the GEMM
            # its SMs (fold_schedule_ex)
            sc = fold.schedule(op, child, token, root, V, workspace=sched_ws, stream=side, level=level, out=sbuf[i],
                               max_blocks=args.sched_bg_blocks if after is not None else 0)
            ev = torch.cuda.Event()
            ev.record(side)
        return sc, ev, i

    def run_step(sc, ev, i, g, train=True, collective=True, hbuf=None):
        main = torch.cuda.current_stream()
        if ev is not None:
            main.wait_event(ev)
        hb = h_root_buf if hbuf is None else hbuf
        h, c, acts = fold.forward(sc, model, ws=ws, want_c=False, h_root=hb[:sc.n_graphs])
        if train:
            fold.backward(sc, model, acts, g, grads=(dU, db, dE), ws=ws, sweep_done=sweep_done)
            if world > 1 and collective:
                exchange(sc)
            fold.sgd_update(flat_p, flat_g, args.lr)
        sbuf_free[i].record(main)
        sbuf_used[i] = True
        return h

    def time_steps(o, g, nrep, level=None, train=True, warm=3):
        """ms per step of nrep steps over the device graphs o (same step and pipelining
        policy as the headline: schedule + forward [+ backward + SGD]). Rank 0 only (the
        single-GPU context numbers): no collective, the other ranks wait at a barrier."""
        nlev = fold.schedule(*o, V, workspace=sched_ws, level=level).n_levels
        use_pipeline(int(o[0].shape[0]), nlev)
        sp = schedule_async(*o, level=level)
        aft = gate[0] if train else None
        for _ in range(warm):
            run_step(*sp, g, train, collective=False)
            sp = schedule_async(*o, level=level, after=aft)
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(nrep):
            run_step(*sp, g, train, collective=False)
            sp = schedule_async(*o, level=level, after=aft)
        if sp[1] is not None:
            torch.cuda.current_stream().wait_event(sp[1])
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / nrep

    # size the schedule workspace once (fold_schedule_workspace)
    sched_ws = torch.empty(int(fold.load().fold_schedule_workspace(N_nodes, gr.n_graphs)), dtype=torch.uint8,
                           device=dev)
    for _ in range(args.warmup):
        step(op, child, token, root, g_dev)
    n_levels = fold.schedule(op, child, token, root, V, workspace=sched_ws).n_levels
    torch.cuda.synchronize()
    # the host enqueues every kernel of a step: keep the Python cyclic GC out of the timed
    # regions (a collection pause idles the GPU for tens of ms; nothing here builds cycles)
    import gc
    gc.collect()
    gc.disable()
    # pipelined warm-up (the allocator reaches its steady rotation of schedule arrays), then
    # batch 1's schedule, both before the timed region
    pipelined = use_pipeline(N_nodes, n_levels)
    sp = schedule_async(op, child, token, root)
    for _ in range(max(args.warmup, 3)):
        run_step(*sp, g_dev)
        sp = schedule_async(op, child, token, root, after=gate[0])
    torch.cuda.synchronize()

    clocks = ClockSampler(local) if not args.no_clocks else None
    # ---------------- timed region (device-resident inputs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if clocks:
        clocks.start()
    fold.launch_count(reset=True)
    fold.profile_enable(True, classes=timed_prof_classes(args))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    # per-step boundaries (median and p10/p90 of the steps)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record()
    marks[0].record()
    for i in range(args.steps):
        run_step(*sp, g_dev)
        sp = schedule_async(op, child, token, root, after=gate[0])  # the next batch's schedule (side stream)
        marks[i + 1].record()
    if sp[1] is not None:
        torch.cuda.current_stream().wait_event(sp[1])  # the K-th schedule inside the region
    e1.record()
    torch.cuda.synchronize()
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    launches = fold.launch_count()
    prof = fold.profile_read()
    fold.profile_enable(False)
    if world > 1:
        dist.barrier()
    clk = clocks.stop() if clocks else None
    if sp[1] is not None:
        torch.cuda.current_stream().wait_event(sp[1])
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    value = global_nodes / (ms_per_step / 1e3)

    # ---------------- e2e: host buffers, H2D + D2H inside the timed region
    e2e = None
    if not args.no_e2e:
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
        h_op, h_child, h_tok, h_root = pin(gr.op.astype(np.int32)), pin(gr.child.astype(np.int32)), \
            pin(gr.token.astype(np.int32)), pin(gr.root.astype(np.int32))
        h_g = pin(g_host)
        h_out = torch.empty((gr.n_graphs, S), dtype=torch.float32).pin_memory()
        d_op, d_child, d_tok, d_root = (torch.empty_like(x, device=dev) for x in (h_op, h_child, h_tok, h_root))
        d_g = torch.empty_like(h_g, device=dev)
        h2d = sum(x.numel() * x.element_size() for x in (h_op, h_child, h_tok, h_root, h_g))
        d2h = h_out.numel() * 4

        graph_copies = ((d_op, h_op), (d_child, h_child), (d_tok, h_tok), (d_root, h_root))
        # pipelined: the root states go D2H on a copy stream from the other of two root buffers
        # and the next step's upstream gradient H2D on another, so neither copy sits between two
        # steps' kernels on the compute stream (both still run every step inside the timed
        # region, which ends after the last of them). On the pipeline's side stream the gradient
        # copy measured no better (it queues behind the next schedule there)
        hbufs = [torch.empty((gr.n_graphs, S), dtype=torch.float32, device=dev) for _ in range(2)]
        out_done = [torch.cuda.Event(), torch.cuda.Event()]
        out_used = [False, False]
        copy_stream = torch.cuda.Stream(device=dev)
        # the upstream gradient: the next step's H2D on its own stream into the other of two
        # device buffers, once the step before has finished reading it
        h2d_stream = torch.cuda.Stream(device=dev)
        d_gs = [d_g, torch.empty_like(d_g)]
        g_ready = [torch.cuda.Event(), torch.cuda.Event()]
        g_free = [torch.cuda.Event(), torch.cuda.Event()]
        ke = [0]

        def e2e_step(sp):
            # this batch's upstream gradient H2D on the compute stream; the next batch's graph
            # arrays H2D + schedule on the side stream (pipelined); the result D2H on the copy
            # stream (pipelined) or the compute stream (--pipeline off)
            main = torch.cuda.current_stream()
            if side is None:
                d_g.copy_(h_g, non_blocking=True)
                hr = run_step(*sp, d_g)
                nxt = schedule_async(d_op, d_child, d_tok, d_root, copies=graph_copies, after=gate[0])
                h_out.copy_(hr, non_blocking=True)
                return nxt
            j = ke[0] % 2
            ke[0] += 1
            main.wait_event(g_ready[j])
            if out_used[j]:
                main.wait_event(out_done[j])
            hr = run_step(*sp, d_gs[j], hbuf=hbufs[j])
            g_free[j].record(main)
            with torch.cuda.stream(h2d_stream):  # the next step's gradient
                h2d_stream.wait_event(g_free[1 - j])
                d_gs[1 - j].copy_(h_g, non_blocking=True)
                g_ready[1 - j].record(h2d_stream)
            done = torch.cuda.Event()
            done.record(main)
            nxt = schedule_async(d_op, d_child, d_tok, d_root, copies=graph_copies, after=gate[0])
            copy_stream.wait_event(done)
            with torch.cuda.stream(copy_stream):
                h_out.copy_(hr, non_blocking=True)
                out_done[j].record(copy_stream)
            out_used[j] = True
            return nxt

        use_pipeline(N_nodes, n_levels)
        sp = schedule_async(d_op, d_child, d_tok, d_root, copies=graph_copies)
        for j in range(2):  # both gradient buffers filled once; each step refills the other
            d_gs[j].copy_(h_g, non_blocking=True)
            g_ready[j].record(torch.cuda.current_stream())
            g_free[j].record(torch.cuda.current_stream())
        for _ in range(max(args.warmup, 3)):
            sp = e2e_step(sp)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(args.steps):
            sp = e2e_step(sp)
        if sp[1] is not None:
            torch.cuda.current_stream().wait_event(sp[1])
        torch.cuda.current_stream().wait_stream(copy_stream)  # the last root-state D2H
        torch.cuda.current_stream().wait_stream(h2d_stream)   # and the last gradient H2D
        a1.record()
        torch.cuda.synchronize()
        t2 = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t2, op=dist.ReduceOp.MAX)
        e_ms = float(t2.item()) / args.steps
        e2e = {"value": global_nodes / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---------------- per-class breakdown: a separate profiled pass, after the device-timed
    # region and the e2e measurement (which run back to back, so both see the same clocks)
    use_pipeline(N_nodes, n_levels)
    sp_box = [schedule_async(op, child, token, root)]

    def _bd_step():
        run_step(*sp_box[0], g_dev)
        sp_box[0] = schedule_async(op, child, token, root, after=gate[0])
    per_class = breakdown_pass(args, fold, _bd_step, prof)
    if sp_box[0][1] is not None:
        torch.cuda.current_stream().wait_event(sp_box[0][1])
    torch.cuda.synchronize()

    # ---------------- N > 1: BASELINE configs[4] strong scaling beside the weak-scaled headline:
    # ONE global batch of 8192 random 128-leaf trees sharded by node count (dp.shard), the
    # same step (schedule + fwd + bwd + all_reduce + SGD), max over ranks
    c5 = None
    if world > 1 and args.config == "c2" and not args.no_c5_strong:
        from paper_1702_02181_b200 import dp
        full5 = foldgen.config_c5(8192)
        gr5 = dp.shard(full5, rank, world)
        o5 = fold.graphs_to_device(gr5, dev)
        g5 = torch.from_numpy(foldgen.make_upstream(gr5.n_graphs, S)).to(dev)
        for _ in range(max(args.warmup, 3)):
            step(*o5, g5)
        torch.cuda.synchronize()
        dist.barrier()
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        for _ in range(args.steps):
            step(*o5, g5)
        c1.record()
        torch.cuda.synchronize()
        t5 = torch.tensor([c0.elapsed_time(c1)], dtype=torch.float64, device=dev)
        dist.all_reduce(t5, op=dist.ReduceOp.MAX)
        ms5 = float(t5.item()) / args.steps
        c5 = {"value": full5.n_nodes / (ms5 / 1e3), "unit": UNIT, "ms_per_step": ms5, "scaling": "strong",
              "trees": full5.n_graphs, "nodes": full5.n_nodes, "nodes_rank0": gr5.n_nodes,
              "shard": "contiguous tree ranges balanced by node count (dp.shard)",
              "step": "schedule+fwd+bwd+exchange(all_reduce [dU|db] %.0f MB + dE %s)+sgd"
                      % ((nU + nb) * 4 / 1e6, xmode[0])}

    # ---------------- batch-1 (within-tree batching only) for the speedup-vs-batch-size context
    batch1 = None
    if not args.no_batch1 and rank == 0 and args.config in ("c2", "c3", "c4", "c5"):
        one = foldgen.sub_batch(gr, 0, 1)
        o1 = fold.graphs_to_device(one, dev)
        g1 = g_dev[:1].contiguous()
        ms1 = time_steps(o1, g1, 20)
        batch1 = {"nodes_per_s": one.n_nodes / (ms1 / 1e3), "ms_per_tree": ms1}

    # ---------------- nodes/s vs batch size (BASELINE metric "... vs batch size"), rank 0
    sweep = None
    if not args.no_sweep and rank == 0 and args.config in ("c2", "c3", "c4", "c5"):
        sweep = {}
        for Bs in (1, 4, 16, 64, 256):
            if Bs >= gr.n_graphs:
                break
            sub = foldgen.sub_batch(gr, 0, Bs)
            o = fold.graphs_to_device(sub, dev)
            gs = g_dev[:Bs].contiguous()
            msb = time_steps(o, gs, 10)
            sweep[str(Bs)] = {"nodes_per_s": sub.n_nodes / (msb / 1e3), "ms_per_step": msb}
        sweep[str(gr.n_graphs)] = {"nodes_per_s": value / world, "ms_per_step": ms_per_step}

    # ---------------- unbatched baseline + PAPER.md Table 1 on B200 (rank 0)
    t1 = None
    if not args.no_table1 and rank == 0 and args.config in ("c2", "c5"):
        t1 = table1(time_steps, fold, gr, g_dev, V, S, dev)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---------------- roofline of the dominant kernel class (tensor-bound GEMM kernels)
    roofline = roofline_record(prof, args.steps, ms_per_step, gates, S, n_cells, clk,
                               cfg_key=f"{args.config}/{gr.n_graphs}/{S}/{args.prec}", prec=args.prec)

    # ---------------- CPU baseline: the fp64 oracle as it stands, bounded sample, 1 thread
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        cpu = cpu_baseline(gr, cell, p, g_host, n_trees=2 if args.config in ("c2", "c4", "c5") else 64)

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None, "dtype": args.prec, "data": "synthetic",
        "config": {"workload": desc, "trees_per_gpu": gr.n_graphs, "nodes_per_gpu": N_nodes,
                   "cells_per_gpu": n_cells, "state": S, "cell": cell, "levels": n_levels,
                   "step": "schedule+fwd+bwd+allreduce+sgd" if world > 1 else "schedule+fwd+bwd+sgd",
                   "l2": "working set > L2 (pool+saved gates+grads ~%.1f GB); no flush" % (
                       (N_nodes * S * 6 + n_cells * gates * S * 4 + n_cells * S * 16) / 1e9),
                   "parallelism": f"dp{world}",
                   "exchange": (xmode[0] if world > 1 else None),
                   "pipeline": ("next batch's fold_schedule on a side stream during this batch's step" +
                                ("" if gate[0] is None else ", started after this batch's level sweep"))
                   if pipelined else "off"},
        "gpu_launches": int(launches),
        "step_ms": {"median": float(np.median(step_ms)), "p10": float(np.percentile(step_ms, 10)),
                    "p90": float(np.percentile(step_ms, 90)), "rank0": [round(x, 4) for x in step_ms]},
        "kernels": per_class, "kernels_source": kernels_source(args),
        "us_per_level": {  # the latency-bound view (n_levels - 1 cell levels)
            "fwd": 1e3 * sum(per_class.get(k, {}).get("ms_per_step", 0.0) for k in ("cell_fwd",)) / max(n_levels - 1, 1),
            "bwd": 1e3 * sum(per_class.get(k, {}).get("ms_per_step", 0.0) for k in ("gemm_dA", "bwd_pointwise"))
                   / max(n_levels - 1, 1),
            # one cross-SM dependency hop with the executor's publication pattern, measured
            # (tools/micro/hop_latency.cu, profiles/r01/hop_latency.json)
            "hop_floor_us": 0.40},
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clk,
    }
    if c5:
        out["c5_strong"] = c5
    if sweep:
        out["sweep_nodes_per_s_vs_batch"] = sweep
    if batch1:
        out["batch1"] = batch1
        out["speedup_vs_batch1"] = (value / world) / batch1["nodes_per_s"]
    if t1:
        ub = t1.pop("unbatched")
        out["unbatched"] = ub
        out["speedup_vs_unbatched"] = (value / world) / ub["nodes_per_s"]
        out["table1"] = t1
    print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


# algorithmic DRAM bytes per cell of each tensor kernel (SURVEY §8(d.4), BF16 path; fp32 c and
# gradients): forward reads 2S h (bf16) + 2S child c (fp32), writes S h + S c + 5S gates
# (28 S); the dA sweep reads the edge gradients dh, dc (2 S fp32), gates (5S bf16), c, c_L,
# c_R (3 S fp32), writes dZ (5S bf16) + dA / dCe (4 S fp32) (56 S); dU re-reads the 2S h
# operand row and the 5S dZ row (14 S)
ALGO_BYTES_PER_CELL_PER_S = {"k_fwd_levels": 28, "k_bwd_levels": 56, "k_gemm_dU_tc": 14}


ROOF_CLASSES = ("cell_fwd", "gemm_dA", "gemm_dU")


def timed_prof_classes(args, extra=()):
    """Classes recorded inside the timed region: each bracket is a pair of event records on
    the stream, which costs host enqueue time in the many-level configs (SST, C6)."""
    return None if args.prof == "all" else ROOF_CLASSES + tuple(extra)


def kernels_source(args):
    return ("CUDA events inside the timed region" if args.prof == "all" else
            f"CUDA events over a profiled pass of {min(args.steps, 5)} steps after the timed region "
            f"(the timed region brackets only the roofline classes)")


def breakdown_pass(args, fold, run, prof):
    """Per-class kernel times (ms/step, launches/step): from the timed region when every
    class was recorded there, else from a profiled pass of min(steps, 5) more steps."""
    import torch
    n = args.steps
    if args.prof != "all":
        n = min(args.steps, 5)
        fold.profile_enable(True)
        for _ in range(n):
            run()
        torch.cuda.synchronize()
        prof = fold.profile_read()
        fold.profile_enable(False)
    return {k: {"ms_per_step": v[0] / n, "launches_per_step": v[1] / n} for k, v in prof.items() if v[1] > 0}


def roofline_record(prof, steps, ms_per_step, gates, S, n_cells, clk, cfg_key=None, prec="bf16"):
    """Roofline of the three tcgen05 GEMM kernel classes (each = one persistent launch per
    step), the dominant one as the headline object. achieved = 2 * gates*S * 2S FLOP per cell
    x cells per launch / the class's CUDA-event time per step (on its launch stream, inside
    the timed region). Peak: MEASURED_PEAKS.json's burst bf16 figure when the timed region's
    median SM clock is within 5% of max (the GPU ran at full clock), else the sustained one
    (power-capped clocks); both fractions are printed. traffic = ncu DRAM bytes of one launch
    (profiles/ncu_traffic.json), beside the algorithmic bytes of SURVEY §8(d.4)."""
    pk, pk_src = peaks()
    burst = pk.get("bf16_tflops")
    sustained = pk.get("bf16_tflops_sustained", burst)
    # TF32 / FP32 (3xTF32) modes: the TF32 peak = the measured bf16 peak x the nominal dense
    # ratio 1.125 / 2.25 PF (B200_PROFILING.md); 3xTF32 issues three MMAs per algorithmic
    # product, so its ceiling in algorithmic FLOP/s is a third of that
    scale = {"bf16": 1.0, "tf32": 0.5, "fp32": 0.5 / 3}[prec]
    burst, sustained = burst * scale, sustained * scale
    dtype_note = {"bf16": "bf16", "tf32": "tf32 (= bf16 x 0.5 nominal ratio)",
                  "fp32": "3xTF32 (= bf16 x 0.5 / 3 MMA passes)"}[prec]
    full_clock = bool(clk and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"])
    peak, which = (burst, "burst") if (full_clock or clk is None) else (sustained, "sustained")
    flops_per_cell = 2.0 * gates * S * 2 * S  # one GEMM pass (fwd Z, bwd dA, or dU) per cell
    tensor_classes = {"cell_fwd": "k_fwd_levels", "gemm_dA": "k_bwd_levels", "gemm_dU": "k_gemm_dU_tc"}
    if prec != "bf16":  # per-level gather + k_gemm_tf32 + pointwise; dA and dU on k_gemm_tf32
        tensor_classes = {"cell_fwd": "k_gemm_tf32 (fwd levels, + gather/pointwise)",
                          "gemm_dA": "k_gemm_tf32 (dA levels)", "gemm_dU": "k_gemm_tf32 (dU)"}
    ncu = {}
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            ncu = json.load(open(tpath))
        except Exception:
            ncu = {}
        if ncu.get("_config") != cfg_key:  # captured on another workload: no traffic figure
            ncu = {}
    per = {}
    for cls, kern in tensor_classes.items():
        ms_total, launches = prof.get(cls, (0.0, 0))
        if launches <= 0 or ms_total <= 0:
            continue
        ms = ms_total / steps
        ach = flops_per_cell * n_cells / (ms / 1e3) / 1e12
        algo = ALGO_BYTES_PER_CELL_PER_S.get(kern, 0) * S * n_cells
        tr = ncu.get(kern, {}).get("dram_bytes_per_launch")
        per[kern] = {"ms_per_step": ms, "achieved": ach, "frac": ach / peak, "frac_burst": ach / burst,
                     "frac_sustained": ach / sustained, "share_of_step": ms / ms_per_step,
                     "algorithmic_bytes": algo, "traffic": tr,
                     "traffic_over_algorithmic": (tr / algo) if tr else None}
    dom = max(per, key=lambda k: per[k]["ms_per_step"])
    d = per[dom]
    return {"bound": "tensor", "kernel": dom, "achieved": d["achieved"], "peak": peak, "unit": "TFLOP/s",
            "frac": d["frac"], "traffic": d["traffic"],
            "peak_kind": which, "frac_burst": d["frac_burst"], "frac_sustained": d["frac_sustained"],
            "peak_source": f"{pk_src} bf16_tflops ({which}) for {dtype_note}; burst {burst:.1f}, sustained "
                           f"{sustained:.1f} TF/s (MEASURED_PEAKS.json); "
                           f"burst when the timed region's median SM clock >= 0.95 x max",
            "algorithmic": f"{flops_per_cell:.4g} FLOP/cell x {n_cells} cells per launch (one launch per step)",
            "share_of_step": d["share_of_step"],
            "traffic_source": "ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum of one launch "
                              "(profiles/ncu_traffic.json)" if d["traffic"] else None,
            "kernels": per}


def _time(fn, nrep, warm=2):
    import torch
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(nrep):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / nrep


def table1(time_steps, fold, gr, g_dev, V, S, dev):
    """PAPER.md L83-L127 / Table 1 with our kernels on B200, training (fwd+bwd+SGD, the
    bench step) and inference (schedule + forward) per-tree times.
      unbatched:   ONE tree of the headline workload, manual levels (one cell per level:
                   the node-at-a-time, batch-size-1 evaluation), the speedup denominator
                   of BASELINE.json's "speedup vs unbatched".
      manual:      B copies of one random 128-leaf shape, every tree position its own op
                   (foldgen.manual_levels), batched across trees only (L83).
      dynamic:     the same batch under the dynamic-batching schedule (L40-44).
      full_dynamic: B random 128-leaf shapes, dynamic batching (L86 "full dynamic").
    cost_ratio = dynamic / manual per-tree time (L114 column); speedup_ratio = manual
    B=1 per-tree time / full-dynamic per-tree time at B (L127 column)."""
    import torch

    def dev_graphs(g, manual):
        t = fold.graphs_to_device(g, dev)
        lv = torch.from_numpy(foldgen.manual_levels(g)).to(dev) if manual else None
        return t, lv

    def per_tree(g, manual, train, nrep):
        t, lv = dev_graphs(g, manual)
        gg = g_dev[:g.n_graphs].contiguous() if g.n_graphs <= g_dev.shape[0] else \
            torch.ones((g.n_graphs, S), device=dev) * 0.01
        ms = time_steps(t, gg, nrep, level=lv, train=train, warm=2)
        return ms / g.n_graphs

    one = foldgen.sub_batch(gr, 0, 1)
    ms_ub = per_tree(one, True, True, 10)
    out = {"unbatched": {"nodes_per_s": one.n_nodes / (ms_ub / 1e3), "ms_per_tree": ms_ub,
                         "levels": 1 + int((one.op == 1).sum()),
                         "how": "one tree of the headline workload, manual levels (one cell per level), "
                                "schedule+fwd+bwd+sgd"}}
    rows = {}
    for B in (1, 32, 64, 128, 256, 512, 1024):
        same = foldgen.table1_batch(B, True, vocab=V)
        full = foldgen.table1_batch(B, False, vocab=V)
        nrep = 10 if B >= 256 else 20
        row = {}
        for mode, train in (("train", True), ("infer", False)):
            m = per_tree(same, True, train, nrep)
            d = per_tree(same, False, train, nrep)
            f = per_tree(full, False, train, nrep)
            row[mode] = {"manual_ms_per_tree": m, "dynamic_ms_per_tree": d, "full_dynamic_ms_per_tree": f,
                         "cost_ratio": d / m}
        rows[str(B)] = row
    for mode in ("train", "infer"):
        m1 = rows["1"][mode]["manual_ms_per_tree"]
        for B, row in rows.items():
            row[mode]["speedup_ratio"] = m1 / row[mode]["full_dynamic_ms_per_tree"]
    out["rows"] = rows
    out["workload"] = "random-split 128-leaf trees (Table 1: 'tree size is 128'), TreeLSTM S=1024, bf16"
    return out


def cpu_baseline(gr, cell, p, g_host, n_trees):
    """Time the fp64 oracle (forward + backward, node at a time, 1 thread) on the first
    n_trees trees of the same workload."""
    import oracle
    sub = foldgen.sub_batch(gr, 0, min(n_trees, gr.n_graphs))
    g = g_host[:sub.n_graphs]
    t0 = time.perf_counter()
    oracle.forward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E)
    oracle.backward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E, g)
    dt = time.perf_counter() - t0
    out = {"value": sub.n_nodes / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
           "sample": f"first {sub.n_graphs} trees ({sub.n_nodes} nodes) of the same batch, fp64 "
                     f"forward + backward, single thread, {dt:.1f} s"}
    # all host cores: one tree per task on a thread pool (the oracle's C
    # calls release the GIL), as many trees as cores, same workload
    import concurrent.futures
    cores = len(os.sched_getaffinity(0))
    per = max(1, sub.n_graphs // 2)  # trees per task (same per-call overhead as the 1-thread run)
    ntr = min(cores * per, gr.n_graphs)
    tasks = [(i, min(i + per, ntr)) for i in range(0, ntr, per)]
    trees = [foldgen.sub_batch(gr, a, b) for a, b in tasks]
    U64, b64, E64 = (np.ascontiguousarray(x, dtype=np.float64) for x in (p.U, p.b, p.E))

    def one(i):
        t = trees[i]
        a = tasks[i][0]
        oracle.forward(cell, t.op, t.child, t.token, t.root, U64, b64, E64)
        oracle.backward(cell, t.op, t.child, t.token, t.root, U64, b64, E64, g_host[a:a + t.n_graphs])
    t0 = time.perf_counter()
    with concurrent.futures.ThreadPoolExecutor(max_workers=cores) as ex:
        list(ex.map(one, range(len(tasks))))
    dta = time.perf_counter() - t0
    nn = sum(t.n_nodes for t in trees)
    out["all_cores"] = {"value": nn / dta, "unit": UNIT, "cores": cores,
                        "sample": f"first {ntr} trees ({nn} nodes), {per} tree(s) per task on {cores} threads, "
                                  f"{dta:.1f} s"}
    return out


# ============================================================================ reference arm

def run_reference(args):
    """--impl reference: the fp64 oracle (the only reference this paper-only task has),
    timed as it stands on host cores; each step = forward + backward over a bounded
    sample (args.ref_trees trees) of the same workload. Rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    gr, cell, S, desc, _ = workload(args, 0, 1)
    p = foldgen.make_params(cell, S, gr.vocab)
    g_host = foldgen.make_upstream(gr.n_graphs, S)
    sub = foldgen.sub_batch(gr, 0, min(args.ref_trees, gr.n_graphs))
    g = g_host[:sub.n_graphs]

    def step():
        oracle.forward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E)
        oracle.backward(cell, sub.op, sub.child, sub.token, sub.root, p.U, p.b, p.E, g)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    value = sub.n_nodes / dt
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": desc, "trees_per_step": sub.n_graphs, "nodes_per_step": sub.n_nodes,
                      "state": S, "cell": cell},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": "oracle",
                            "sample": f"{sub.n_graphs} tree(s) ({sub.n_nodes} nodes) per step, fp64 fwd+bwd, "
                                      f"single thread"},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ============================================================================ §3.5 model (NEXT-2)

def run_sst(args):
    """--model sst: the §3.5 sentiment model (leaf TreeLSTM(E[w],0,0),
    internal TreeLSTM(0,h_L,h_R), 5-way softmax cross-entropy at every node) training step
    = fold_schedule + fold_sst_forward + fold_sst_backward + SGD over all parameters, on
    parse-shaped trees (C3 shapes, S = 300, synthetic uniform labels); FP32 (3xTF32) or TF32
    tensor-core GEMMs. One GPU (rank 0 prints)."""
    import torch
    from paper_1702_02181_b200 import fold
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    fold.device_check()
    prec = args.prec if args.prec != "bf16" else "fp32"
    cfg = args.config if args.config in ("c2", "c3", "c5") else "c3"
    gr = foldgen.make_config(cfg, args.batch or DEFAULT_B[cfg])
    S = foldgen.CONFIG_STATE[cfg]
    V = gr.vocab
    p = foldgen.make_params("treelstm", S, V)
    q = foldgen.make_sst_params(S)
    y = foldgen.make_labels(gr.n_nodes)
    sizes = [p.U.size, p.b.size, p.E.size, q.W.size, q.Ws.size, q.bs.size]
    flat_p = torch.empty(sum(sizes), dtype=torch.float32, device=dev)
    flat_g = torch.zeros_like(flat_p)

    def views(buf):
        out, o = [], 0
        for a, n in zip((p.U, p.b, p.E, q.W, q.Ws, q.bs), sizes):
            out.append(buf[o:o + n].view(a.shape))
            o += n
        return out
    P, Gr = views(flat_p), views(flat_g)
    for d, a in zip(P, (p.U, p.b, p.E, q.W, q.Ws, q.bs)):
        d.copy_(torch.from_numpy(a))
    model = fold.Model(P[0], P[1], P[2], prec=prec)
    head = fold.SstHead(P[3], P[4], P[5], torch.from_numpy(y).to(dev))
    op, child, token, root = fold.graphs_to_device(gr, dev)
    ws = fold.Workspace(dev)
    n_cells = int((gr.op == 1).sum())

    # pipelined steps as in the headline bench: the next batch's fold_schedule on a side stream
    # during this batch's step (K schedules in K timed steps)
    side = torch.cuda.Stream(device=dev) if args.pipeline != "off" else None
    pend = [None]

    def sched(o, stream=None):
        return fold.schedule(*o, V, stream=stream, workspace=ws.get("sched", int(fold.load().fold_schedule_workspace(
            o[0].shape[0], o[3].shape[0]))))

    def step(o, copies=(), o_next=None, copies_next=(), done_prev=None, label=None, label_next=None):
        main = torch.cuda.current_stream()
        if pend[0] is None:
            for d, hsrc in copies:
                d.copy_(hsrc, non_blocking=True)
            s = sched(o)
        else:
            s, ev = pend[0]
            main.wait_event(ev)
            s.arrays.buffer.record_stream(main)
            pend[0] = None
        if label is not None:
            head.label = label
        loss, acts = fold.sst_forward(s, model, head, ws=ws)
        fold.sst_backward(s, model, head, acts, grads=tuple(Gr), ws=ws)
        fold.sgd_update(flat_p, flat_g, args.lr)
        if side is not None:
            with torch.cuda.stream(side):
                if done_prev is not None:
                    side.wait_event(done_prev)
                for d, hsrc in copies_next:
                    d.copy_(hsrc, non_blocking=True)
                sn = sched(o_next or o, stream=side)
                ev = torch.cuda.Event()
                ev.record(side)
            pend[0] = (sn, ev)
        return loss
    for _ in range(max(args.warmup, 3)):
        step((op, child, token, root))
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.disable()
    clocks = ClockSampler(0) if not args.no_clocks else None
    if clocks:
        clocks.start()
    fold.launch_count(reset=True)
    fold.profile_enable(True, classes=timed_prof_classes(args, ("embed_fwd", "embed_bwd")))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record()
    marks[0].record()
    for i_step in range(args.steps):
        step((op, child, token, root))
        marks[i_step + 1].record()
    e1.record()
    torch.cuda.synchronize()
    launches = fold.launch_count()
    prof = fold.profile_read()
    fold.profile_enable(False)
    clk = clocks.stop() if clocks else None
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    per_class = breakdown_pass(args, fold, lambda: step((op, child, token, root)), prof)
    timed = {k: v[0] / args.steps for k, v in prof.items() if v[1] > 0}
    ms = e0.elapsed_time(e1) / args.steps
    value = gr.n_nodes / (ms / 1e3)
    # e2e: graph arrays + labels H2D from pinned memory, the loss D2H, every step
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    hs = [pin(a.astype(np.int32)) for a in (gr.op, gr.child, gr.token, gr.root, y)]
    # two device buffer sets (the next batch's copies never overwrite arrays a running step reads)
    dsets = [[torch.empty_like(h, device=dev) for h in hs] for _ in range(2)]
    dev_done = [None, None]
    hloss = torch.empty(1, dtype=torch.float32).pin_memory()
    h2d = sum(h.numel() * 4 for h in hs)
    pend[0] = None
    k_e2e = [0]

    def e2e_step():
        i = k_e2e[0] % 2
        cur, nxt = dsets[i], dsets[1 - i]
        loss = step(tuple(cur[:4]), copies=list(zip(cur, hs)), o_next=tuple(nxt[:4]),
                    copies_next=list(zip(nxt, hs)), done_prev=dev_done[1 - i], label=cur[4])
        hloss.copy_(loss, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        dev_done[i] = ev
        k_e2e[0] += 1
    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(args.steps):
        e2e_step()
    a1.record()
    torch.cuda.synchronize()
    e_ms = a0.elapsed_time(a1) / args.steps
    # roofline: the three cell GEMM passes + the leaf level's (K = S, N = 5S padded: 10 S^2 per
    # leaf forward, 2 x 10 S^2 backward) on the TF32 peak (3xTF32: a third of it)
    pk, pk_src = peaks()
    scale = 0.5 if prec == "tf32" else 0.5 / 3
    full_clock = bool(clk and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"])
    peak = pk["bf16_tflops"] * scale if (full_clock or clk is None) else pk["bf16_tflops_sustained"] * scale
    n_leaves = gr.n_nodes - n_cells
    flops = 3 * 20.0 * S * S * n_cells + 3 * 10.0 * S * S * n_leaves
    gemm_ms = sum(timed.get(k, 0.0) for k in ("cell_fwd", "gemm_dA", "gemm_dU",
                                                                          "embed_fwd", "embed_bwd"))
    achieved = flops / (gemm_ms / 1e3) / 1e12 if gemm_ms > 0 else 0.0
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        sub = foldgen.sub_batch(gr, 0, min(16, gr.n_graphs))
        t0 = time.perf_counter()
        oracle.sst_backward(sub.op, sub.child, sub.token, y[:sub.n_nodes], p.U, p.b, p.E, q.W, q.Ws, q.bs)
        dt = time.perf_counter() - t0
        cpu = {"value": sub.n_nodes / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {sub.n_graphs} trees ({sub.n_nodes} nodes), fp64 §3.5 forward+backward "
                         f"(oracle_sst_backward), single thread, {dt:.1f} s"}
    out = {"metric": "§3.5 TreeLSTM sentiment model tree nodes/sec fwd+bwd (NEXT-2)", "value": value, "unit": UNIT,
           "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
           "config": {"workload": f"{cfg.upper()} tree shapes, B={gr.n_graphs}, S={S}, V={V}, 5 classes, "
                                  f"labels at every node (PAPER.md L297), leaf TreeLSTM(E[w],0,0)",
                      "nodes": gr.n_nodes, "cells": n_cells, "leaves": n_leaves,
                      "step": "schedule+sst_fwd+sst_bwd+sgd", "l2": "no flush (working set > L2 at B=1024)",
                      "pipeline": "next batch's fold_schedule on a side stream during this batch's step"
                      if side is not None else "off"},
           "gpu_launches": int(launches), "step_ms": {"median": float(np.median(step_ms)), "p10": float(np.percentile(step_ms, 10)),
                       "p90": float(np.percentile(step_ms, 90)), "all": [round(x, 4) for x in step_ms]},
           "kernels": per_class, "kernels_source": kernels_source(args),
           "roofline": {"bound": "tensor", "kernel": "k_gemm_tf32 (all GEMM passes)", "achieved": achieved,
                        "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak if peak else None, "traffic": None,
                        "peak_source": f"{pk_src} bf16 x {scale:.4f} ({prec}: TF32 = bf16/2 nominal"
                                       f"{', 3 MMA passes' if prec == 'fp32' else ''})",
                        "algorithmic": "60 S^2 FLOP per cell + 30 S^2 per leaf (padded 5-gate leaf GEMMs)"},
           "cpu_baseline": cpu,
           "e2e": {"value": gr.n_nodes / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": 4},
           "clocks": clk}
    print(json.dumps(out), flush=True)


# ============================================================================ multi-op levels (NEXT-3)

def run_mo(args):
    """--model mo: multi-op dynamic batching (fold_mo.h) on the C6 workload
    (foldgen.mo_batch_c6: parse-shaped trees with binary TreeLSTM, unary TreeLSTM chains and a
    typed projection RNN at the root; S0 = 300, S1 = 128, V = 16384 Zipf). Training step =
    fold_mo_schedule + fold_mo_forward + fold_mo_backward + SGD over all parameters; FP32
    (3xTF32) or TF32 tensor-core GEMMs. One GPU (rank 0 prints)."""
    import torch
    from paper_1702_02181_b200 import fold, fold_mo
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    fold.device_check()
    prec = args.prec if args.prec != "bf16" else "fp32"
    B = args.batch or 1024
    gr = foldgen.mo_batch_c6(B)
    T = gr.table
    params = foldgen.make_mo_params(T)
    arrs = [x for blk in params for x in blk]
    sizes = [a.size for a in arrs]
    # 16-byte aligned parameter blocks: pad each block's offset to 4 floats
    offs, o = [], 0
    for n in sizes:
        offs.append(o)
        o += (n + 3) // 4 * 4
    flat_p = torch.zeros(o, dtype=torch.float32, device=dev)
    flat_g = torch.zeros_like(flat_p)

    def views(buf):
        out, k = [], 0
        for blk in params:
            v = []
            for x in blk:
                v.append(buf[offs[k]:offs[k] + x.size].view(x.shape))
                k += 1
            out.append(tuple(v))
        return out
    P, Gr = views(flat_p), views(flat_g)
    for blk, src in zip(P, params):
        for d, a in zip(blk, src):
            d.copy_(torch.from_numpy(a))
    model = fold_mo.MoModel(P, prec)
    t = lambda x: torch.tensor(np.ascontiguousarray(x, np.int32).reshape(-1), device=dev)
    dvs = (t(gr.op), t(gr.child), t(gr.token), t(gr.root))
    g = torch.tensor(foldgen.make_mo_upstream(gr.n_graphs, T), device=dev)

    # pipelined steps (as in the headline bench): right after batch k's
    # forward / backward / SGD are enqueued, batch k+1's fold_mo_schedule runs on a side stream
    # (its one host sync then overlaps batch k's execution); batch k+1's forward waits on it.
    # Every timed step still schedules a batch (K schedules in K timed steps).
    side = torch.cuda.Stream(device=dev) if args.pipeline != "off" else None
    pend = [None]

    def step(o, copies=(), o_next=None, copies_next=(), done_prev=None):
        """o: this batch's device graph arrays (copies: its H2D copies if not yet scheduled);
        o_next / copies_next: the next batch's (default: the same arrays), whose schedule
        starts on the side stream once `done_prev` (the event of the step that last read
        o_next's buffers) has passed."""
        main = torch.cuda.current_stream()
        if pend[0] is None:
            for d, hsrc in copies:
                d.copy_(hsrc, non_blocking=True)
            s = fold_mo.schedule(T, *o)
        else:
            s, ev = pend[0]
            main.wait_event(ev)
            s._keep[0].record_stream(main)
            pend[0] = None
        h, acts = fold_mo.forward(s, model)
        fold_mo.backward(s, model, acts, g, grads=Gr)
        fold.sgd_update(flat_p, flat_g, args.lr)
        if side is not None:
            with torch.cuda.stream(side):
                if done_prev is not None:
                    side.wait_event(done_prev)
                for d, hsrc in copies_next:
                    d.copy_(hsrc, non_blocking=True)
                sn = fold_mo.schedule(T, *(o_next or o), stream=side)
                ev = torch.cuda.Event()
                ev.record(side)
            pend[0] = (sn, ev)
        return h
    for _ in range(max(args.warmup, 3)):
        step(dvs)
    torch.cuda.synchronize()
    import gc
    gc.collect()
    gc.disable()
    clocks = ClockSampler(0) if not args.no_clocks else None
    if clocks:
        clocks.start()
    fold.launch_count(reset=True)
    fold.profile_enable(True, classes=timed_prof_classes(args))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record()
    marks[0].record()
    for i_step in range(args.steps):
        step(dvs)
        marks[i_step + 1].record()
    e1.record()
    torch.cuda.synchronize()
    launches = fold.launch_count()
    prof = fold.profile_read()
    fold.profile_enable(False)
    clk = clocks.stop() if clocks else None
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    per_class = breakdown_pass(args, fold, lambda: step(dvs), prof)
    timed = {k: v[0] / args.steps for k, v in prof.items() if v[1] > 0}
    ms = e0.elapsed_time(e1) / args.steps
    value = gr.n_nodes / (ms / 1e3)
    # e2e: graph arrays H2D from pinned memory, the root states D2H, every step
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.int32).reshape(-1)).pin_memory()
    hs = [pin(a) for a in (gr.op, gr.child, gr.token, gr.root)]
    # two device buffer sets: the next batch's copies never overwrite arrays a running step reads
    dsets = [[torch.empty_like(h, device=dev) for h in hs] for _ in range(2)]
    dev_done = [None, None]
    hout = torch.empty((gr.n_graphs, int(T.S.max())), dtype=torch.float32).pin_memory()
    h2d = sum(h.numel() * 4 for h in hs)

    pend[0] = None  # (the device-resident batch's pending schedule is not the e2e batch's)
    k_e2e = [0]

    def e2e_step():
        i = k_e2e[0] % 2
        cur, nxt = dsets[i], dsets[1 - i]
        hout.copy_(step(tuple(cur), copies=list(zip(cur, hs)), o_next=tuple(nxt), copies_next=list(zip(nxt, hs)),
                        done_prev=dev_done[1 - i]), non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream())
        dev_done[i] = ev
        k_e2e[0] += 1
    for _ in range(3):
        e2e_step()
    torch.cuda.synchronize()
    a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a0.record()
    for _ in range(args.steps):
        e2e_step()
    a1.record()
    torch.cuda.synchronize()
    e_ms = a0.elapsed_time(a1) / args.steps
    # roofline: three GEMM passes (forward Z, backward dA, weight dU) of 2 * nout * kin FLOP per
    # cell node, on the TF32 peak (3xTF32: a third of it); the schedule is excluded
    pk, pk_src = peaks()
    scale = 0.5 if prec == "tf32" else 0.5 / 3
    full_clock = bool(clk and clk.get("sm_max_mhz") and clk["sm_mhz"] >= 0.95 * clk["sm_max_mhz"])
    peak = pk["bf16_tflops"] * scale if (full_clock or clk is None) else pk["bf16_tflops_sustained"] * scale
    cnt = np.bincount(gr.op, minlength=T.n_ops)
    flops = 0.0
    for o in range(T.n_ops):
        if T.kind[o] == foldgen.MO_EMBED:
            continue
        So, Si, a = int(T.S[T.out_type[o]]), int(T.S[T.in_type[o]]), int(T.arity[o])
        nout = (3 + a) * So if T.kind[o] == foldgen.MO_LSTM else So
        flops += 6.0 * nout * a * Si * cnt[o]
    exec_ms = sum(timed.get(k, 0.0) for k in ("cell_fwd", "gemm_dA"))
    achieved = flops / (exec_ms / 1e3) / 1e12 if exec_ms > 0 else 0.0
    cpu = None
    if not args.no_cpu_baseline:
        import oracle
        n1 = int(gr.root[min(16, gr.n_graphs) - 1]) + 1
        sub = foldgen.MoGraphs(gr.op[:n1], gr.child[:n1], gr.token[:n1], gr.root[:min(16, gr.n_graphs)], T)
        Pf = oracle.mo_flatten(T, params)
        t0 = time.perf_counter()
        oracle.mo_backward(sub, Pf, foldgen.make_mo_upstream(sub.n_graphs, T))
        dt = time.perf_counter() - t0
        cpu = {"value": sub.n_nodes / dt, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": f"first {sub.n_graphs} trees ({sub.n_nodes} nodes), fp64 multi-op forward+backward "
                         f"(oracle_mo_backward), single thread, {dt:.1f} s"}
    out = {"metric": "multi-op TreeLSTM tree nodes/sec fwd+bwd (NEXT-3: binary + unary cells, typed projection)",
           "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": prec, "data": "synthetic",
           "config": {"workload": f"C6 multi-op: B={gr.n_graphs} parse-shaped trees + unary LSTM chains "
                                  f"(p=0.3) + root projection; ops EMBED/LSTM2/LSTM1/RNN1, S0={int(T.S[0])}, "
                                  f"S1={int(T.S[1])}, V={int(T.vocab[0])} Zipf",
                      "nodes": gr.n_nodes, "nodes_per_op": cnt.tolist(),
                      "step": "mo_schedule+mo_fwd+mo_bwd+sgd", "l2": "no flush (working set > L2 at B=1024)",
                      "pipeline": "next batch's fold_mo_schedule on a side stream during this batch's step"
                      if side is not None else "off"},
           "gpu_launches": int(launches), "step_ms": {"median": float(np.median(step_ms)), "p10": float(np.percentile(step_ms, 10)),
                       "p90": float(np.percentile(step_ms, 90)), "all": [round(x, 4) for x in step_ms]},
           "kernels": per_class, "kernels_source": kernels_source(args),
           "roofline": {"bound": "tensor", "kernel": "k_gemm_tf32_grouped (+ gather / pointwise per level)",
                        "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                        "frac": achieved / peak if peak else None, "traffic": None,
                        "peak_source": f"{pk_src} bf16 x {scale:.4f} ({prec}: TF32 = bf16/2 nominal"
                                       f"{', 3 MMA passes' if prec == 'fp32' else ''})",
                        "algorithmic": "6 * nout * kin FLOP per cell node (forward Z, dA, dU)"},
           "cpu_baseline": cpu,
           "e2e": {"value": gr.n_nodes / (e_ms / 1e3), "unit": UNIT, "ms_per_step": e_ms, "h2d_bytes_per_step": h2d,
                   "d2h_bytes_per_step": int(hout.numel() * 4)},
           "clocks": clk}
    print(json.dumps(out), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    elif args.model == "sst":
        run_sst(args)
    elif args.model == "mo":
        run_mo(args)
    else:
        run_fold(args)


if __name__ == "__main__":
    main()
