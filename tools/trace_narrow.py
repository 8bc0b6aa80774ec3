"""Per-chunk timeline of k_fwd_narrow (CTA 0), FOLD_DBG_FWD=2:
    FOLD_DBG_FWD=2 python tools/trace_narrow.py --config c4 --batch 1"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import foldgen
from paper_1702_02181_b200 import fold

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4"); ap.add_argument("--batch", type=int, default=1)
a = ap.parse_args()
gr = foldgen.make_config(a.config, a.batch)
S = foldgen.CONFIG_STATE[a.config]
p = foldgen.make_params("treelstm", S, gr.vocab)
model = fold.Model(torch.tensor(p.U, device="cuda"), torch.tensor(p.b, device="cuda"), torch.tensor(p.E, device="cuda"))
op, child, token, root = fold.graphs_to_device(gr)
s = fold.schedule(op, child, token, root, gr.vocab)
ws = fold.Workspace("cuda")
for _ in range(3):
    fold.forward(s, model, ws=ws)
torch.cuda.synchronize()
n = 65536
buf = np.zeros((9, n), np.uint64)
fold.load().fold_debug_fwd_trace(buf.ctypes.data, n)
t = buf.astype(np.int64)
m = int((t[4] > 0).sum())
t = t[:, :m]
d = (t - t[0].min()) / 1e3
names = {0: "p_start", 1: "p_inputs", 2: "mma_done_issue", 5: "e_start", 3: "e_acc", 6: "e_stored", 4: "e_pub",
         7: "mma_b_full"}
print("chunks", m, "span %.1f us, per chunk %.2f us" % (d[4].max(), d[4].max() / max(m, 1)))
pairs = [(0, 1), (1, 7), (7, 2), (2, 3), (5, 3), (3, 6), (6, 4), (4, 1)]
for i, j in pairs:
    if j == 1 and i == 4:
        x = d[1][1:] - d[4][:-1]
    else:
        x = d[j] - d[i]
    print(f"{names[i]:>15} -> {names[j]:<15} median {np.median(x):7.2f} us  p90 {np.percentile(x, 90):7.2f}")
