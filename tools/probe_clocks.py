"""Probe: SM clock / power while the C2 step loops (pynvml, ~2 ms sampling).

    python tools/probe_clocks.py [--steps 300] [--batch 1024]
Prints median/min SM clock and power under load and the per-class kernel times.
"""
import argparse, os, sys, threading, time, statistics, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import pynvml
import foldgen
from paper_1702_02181_b200 import fold

ap = argparse.ArgumentParser()
ap.add_argument("--steps", type=int, default=300)
ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--S", type=int, default=1024)
a = ap.parse_args()
dev = torch.device("cuda", 0)
gr = foldgen.config_c2(a.batch)
S, V = a.S, gr.vocab
p = foldgen.make_params("treelstm", S, V)
U = torch.tensor(p.U, device=dev); b = torch.tensor(p.b, device=dev); E = torch.tensor(p.E, device=dev)
model = fold.Model(U, b, E, cell="treelstm", prec="bf16")
g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
op, child, token, root = fold.graphs_to_device(gr, dev)
ws = fold.Workspace(dev)
dU = torch.zeros_like(U); db = torch.zeros_like(b); dE = torch.zeros_like(E)
def step():
    s = fold.schedule(op, child, token, root, V)
    h, c, acts = fold.forward(s, model, ws=ws, want_c=False)
    fold.backward(s, model, acts, g, grads=(dU, db, dE), ws=ws)
for _ in range(5): step()
torch.cuda.synchronize()
pynvml.nvmlInit(); hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
rows = []; stop = False
def samp():
    while not stop:
        rows.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                     pynvml.nvmlDeviceGetPowerUsage(hdl) / 1000.0,
                     pynvml.nvmlDeviceGetCurrentClocksEventReasons(hdl)))
        time.sleep(0.002)
th = threading.Thread(target=samp, daemon=True); th.start()
fold.profile_enable(True)
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.steps): step()
e1.record(); torch.cuda.synchronize()
stop = True; th.join()
prof = fold.profile_read(); fold.profile_enable(False)
ms = e0.elapsed_time(e1) / a.steps
clk = [r[0] for r in rows]; pw = [r[1] for r in rows]
print(json.dumps({"ms_per_step": ms, "nodes_per_s": gr.n_nodes / ms * 1e3, "samples": len(rows),
                  "sm_mhz_median": statistics.median(clk), "sm_mhz_min": min(clk), "sm_mhz_p10": sorted(clk)[len(clk)//10],
                  "power_median": statistics.median(pw), "power_max": max(pw),
                  "reasons_seen": sorted({hex(r[2]) for r in rows}),
                  "kernels": {k: v[0] / a.steps for k, v in prof.items() if v[1]}}, indent=1))
