"""Per-level forward timeline from the FOLD_DBG_FWD=1 tile stamps (fold_debug_fwd_trace).
    FOLD_DBG_FWD=1 python tools/trace_fwd.py --config c4 --batch 1"""
import argparse, ctypes, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import foldgen
from paper_1702_02181_b200 import fold

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4"); ap.add_argument("--batch", type=int, default=1)
ap.add_argument("--levels", type=int, default=16)
a = ap.parse_args()
assert os.environ.get("FOLD_DBG_FWD") == "1"
gr = foldgen.make_config(a.config, a.batch)
print("nodes", gr.n_nodes)
S = foldgen.CONFIG_STATE[a.config]
p = foldgen.make_params("treelstm", S, gr.vocab)
dev = "cuda"
model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev))
op, child, token, root = fold.graphs_to_device(gr)
s = fold.schedule(op, child, token, root, gr.vocab)
ws = fold.Workspace(dev)
for _ in range(3):
    fold.forward(s, model, ws=ws)
torch.cuda.synchronize()
L = fold.load()
n = 65536
buf = np.zeros((9, n), np.uint64)
got = L.fold_debug_fwd_trace(buf.ctypes.data, n)
lo = s.level_off_host[: s.n_levels + 2]
npairs = 74
tiles = []
for d in range(2, s.n_levels + 1):
    M = int(lo[d + 1] - lo[d]); mt = math.ceil(M / 256)
    W = 48 if mt * math.ceil(S / 48) >= npairs // 2 else 16
    if W == 48:  # the kernel's wave model (fwd_level_W): mid width 32 when it fills the waves better
        cost = lambda w: math.ceil(mt * math.ceil(S / w) / npairs) * max(32 * 5 * w, 4096 + 16 * 5 * w)
        W = 32 if cost(32) < cost(48) else 48
    tiles.append((d, M, W, mt * math.ceil(S / W)))
t = buf[:, :got].astype(np.int64)
t0 = t[0][t[0] > 0].min()
d_ = (t - t0) / 1e3
names = ["start", "inputs", "mma_iss", "acc", "pub", "stg_ok", "epi_done", "st_read", "st_done"]
print("tiles", got, "span us %.1f" % (d_[4].max()))
ntot = min(got, sum(x[3] for x in tiles))
dd = d_[:, :ntot]
print("medians over %d tiles (us): " % ntot + " ".join(f"{names[i]}-{names[j]}={np.median(dd[j]-dd[i]):.2f}"
      for i, j in ((0, 1), (1, 2), (2, 3), (3, 5), (5, 6), (6, 7), (7, 8), (8, 4))))
# per-pair cadence in the first level: start of tile T + npairs minus start of tile T
n1 = tiles[0][3]
if n1 > 2 * npairs:
    cad = dd[0][npairs:n1] - dd[0][:n1 - npairs]
    print("level-2 per-pair tile cadence (us): median %.2f p10 %.2f p90 %.2f" % (
        np.median(cad), np.percentile(cad, 10), np.percentile(cad, 90)))
    for i, j in ((1, 3), (3, 5), (5, 6), (6, 8), (8, 4)):
        x = dd[j][:n1] - dd[i][:n1]
        print(f"  level-2 {names[i]}->{names[j]}: median {np.median(x):.2f} p90 {np.percentile(x, 90):.2f}")
T0 = 0
prev = 0.0
print("level  M  W tiles | first_start max_inputs max_acc max_epi_done max_pub | period")
for (d, M, W, nt) in tiles[: a.levels] + tiles[-3:]:
    pass
T0 = 0
rows = []
for (d, M, W, nt) in tiles:
    sl = slice(T0, T0 + nt)
    rows.append((d, M, W, nt, d_[0][sl].min(), d_[1][sl].max(), d_[3][sl].max(), d_[6][sl].max(), d_[4][sl].max()))
    T0 += nt
prev = 0.0
for r in rows[: a.levels] + rows[-3:]:
    print("%3d %6d %2d %4d | %8.2f %8.2f %8.2f %8.2f %8.2f | %6.2f" % (r + (r[8] - prev,)))
    prev = r[8]
