"""Time fold_schedule alone on a config/batch (CUDA events, median of reps)."""
import argparse, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, foldgen
from paper_1702_02181_b200 import fold
ap = argparse.ArgumentParser(); ap.add_argument("cfgs", nargs="+")
a = ap.parse_args()
for cb in a.cfgs:
    cfg, B = cb.split(":")
    gr = foldgen.make_config(cfg, int(B))
    op, child, token, root = fold.graphs_to_device(gr)
    ws = torch.empty(int(fold.load().fold_schedule_workspace(gr.n_nodes, gr.n_graphs)), dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fold.schedule(op, child, token, root, gr.vocab, workspace=ws)
    ts = []
    for _ in range(20):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); s = fold.schedule(op, child, token, root, gr.vocab, workspace=ws); e1.record()
        torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    print(f"{cb:10s} N={gr.n_nodes:7d} D={s.n_levels:4d} sched {statistics.median(ts)*1e3:8.1f} us  "
          f"smallN={os.environ.get('FOLD_SCHED_SMALLN')} perblock={os.environ.get('FOLD_SCHED_PER_BLOCK')}")
