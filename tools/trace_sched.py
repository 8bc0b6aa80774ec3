"""Scheduler phase timeline (FOLD_DBG_SCHED=1): FOLD_DBG_SCHED=1 python tools/trace_sched.py c2:1024 c2:16"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, foldgen
from paper_1702_02181_b200 import fold
names = ["P0 init", "P1 validate", "P2 parent offs", "P3 parent lists", "P4 depths", "P5 keys", "P6 sort",
         "P7 perm/offs", "P8 gather", "P9 cons CSR", "P10 leaves/tokens", "P11 roots"]
for cb in sys.argv[1:]:
    cfg, B = cb.split(":")
    gr = foldgen.make_config(cfg, int(B))
    op, child, token, root = fold.graphs_to_device(gr)
    for _ in range(3):
        fold.schedule(op, child, token, root, gr.vocab)
    torch.cuda.synchronize()
    buf = np.zeros(13, np.uint64)
    fold.load().fold_debug_sched_trace(buf.ctypes.data)
    t = buf.astype(np.int64)
    d = np.diff(t) / 1e3
    print(cb, "N=%d total %.1f us: " % (gr.n_nodes, (t[12] - t[0]) / 1e3) + ", ".join(f"{n.split()[0]} {x:.1f}" for n, x in zip(names, d)))
