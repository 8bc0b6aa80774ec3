"""Per-level timeline of the wide backward kernel from the FOLD_DBG_BWD=1 tile stamps
(fold_debug_bwd_trace).   FOLD_DBG_BWD=1 python tools/trace_bwd.py --config c4 --batch 1024"""
import argparse, math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import foldgen
from paper_1702_02181_b200 import fold

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c4"); ap.add_argument("--batch", type=int, default=1024)
ap.add_argument("--levels", type=int, default=12)
ap.add_argument("--narrow-max", type=int, default=int(os.environ.get("FOLD_BWD_NARROW_MAX", "32")))
a = ap.parse_args()
assert os.environ.get("FOLD_DBG_BWD") == "1"
gr = foldgen.make_config(a.config, a.batch)
S = foldgen.CONFIG_STATE[a.config]
p = foldgen.make_params("treelstm", S, gr.vocab)
dev = "cuda"
model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev))
op, child, token, root = fold.graphs_to_device(gr)
s = fold.schedule(op, child, token, root, gr.vocab)
ws = fold.Workspace(dev)
g = torch.rand((gr.n_graphs, S), device=dev) * 2 - 1
for _ in range(3):
    _, _, acts = fold.forward(s, model, ws=ws)
    fold.backward(s, model, acts, g, ws=ws)
torch.cuda.synchronize()
n = 65536
buf = np.zeros((12, n), np.uint64)
got = fold.load().fold_debug_bwd_trace(buf.ctypes.data, n)
lo = [int(x) for x in s.level_off_host[: s.n_levels + 2]]
D = s.n_levels
npairs = 74
ld_u = 2 * math.ceil(S / 64) * 64
d = D
while d >= 2 and lo[d + 1] - lo[d] <= a.narrow_max:
    d -= 1
KB = math.ceil(5 * S / 64)
ks_on = os.environ.get("FOLD_BWD_KSPLIT", "1") != "0"
ks256 = os.environ.get("FOLD_BWD_KSPLIT", "1") != "2"
defer = os.environ.get("FOLD_BWD_DEFER", "1") != "0"
Sp = math.ceil(S / 64) * 64
sn = s.to_numpy()
gat = np.asarray(sn["gather"]).reshape(-1, 2)
nl = s.n_leaves


def mask_of(dd):  # bit k: some cell of level dd has a cell child in slot k (k_bwd_prelude)
    g = gat[lo[dd]:lo[dd + 1]]
    return int((g[:, 0] >= nl).any()) | (int((g[:, 1] >= nl).any()) << 1) if defer else 3


def rng(N, mask, crit):  # k_bwd_tiles' column-tile ranges
    NT = math.ceil(ld_u / N)
    lc, rc0 = math.ceil(Sp / N), Sp // N
    a_, b_ = (0, NT) if mask & 3 == 3 else (0, lc) if mask & 1 else (rc0, NT) if mask & 2 else (0, 0)
    if crit:
        return b_ - a_
    return NT if b_ == a_ else (NT - b_ if a_ == 0 else a_)


tiles = []   # (level, M, N*10+KS, units) in unit order: per level its critical units (level),
end = []     # its inline deferred tiles (1000 + level); then the end section (-level)
for dd in range(d, 1, -1):
    M = lo[dd + 1] - lo[dd]
    mt = math.ceil(M / 256)
    mk = mask_of(dd)
    n128, n256 = rng(128, mk, True), rng(256, mk, True)
    if ks_on and KB >= 8 and n128 > 0 and 2 * mt * n128 <= npairs:
        N, KS, n = 128, 2, n128
    elif ks_on and ks256 and KB >= 8 and n256 > 0 and 2 * mt * n256 <= npairs:
        N, KS, n = 256, 2, n256
    elif mt * n256 < npairs:
        N, KS, n = 128, 1, n128
    else:
        N, KS, n = 256, 1, n256
    c = mt * n * KS
    e = 0 if mk == 3 else mt * rng(256, mk, False)
    ni = min(e, (npairs - c % npairs) % npairs) if c > 0 else 0
    tiles.append((dd, M, N * 10 + KS, c))
    tiles.append((1000 + dd, M, 2561, ni))
    end.append((-dd, M, 2561, e - ni))
tiles += end
tiles = [t_ for t_ in tiles if t_[3] > 0]
ntot = min(got, sum(x[3] for x in tiles))
t = buf[:, :ntot].astype(np.int64)
t0 = t[0][t[0] > 0].min()
x = (t - t0) / 1e3
names = ["start", "inputs", "acc_free", "mma_done", "acc_ready", "published", "slab0_in_smem", "slab0_rows_done", "first_stage", "group0_done"]
print(f"{a.config} B={a.batch}: wide levels {len(tiles)} (from d={d}), tiles {ntot}, span {x[5].max():.1f} us")
print("medians (us): " + " ".join(f"{names[i]}->{names[j]}={np.median(x[j] - x[i]):.2f}"
                                   for i, j in ((0, 1), (1, 8), (8, 3), (1, 3), (3, 4), (4, 5), (4, 6), (6, 9), (9, 7), (6, 7), (7, 5), (0, 5))))
cyc = (buf[11, :ntot].astype(np.int64) - buf[10, :ntot].astype(np.int64))
ns = (buf[3, :ntot].astype(np.int64) - buf[8, :ntot].astype(np.int64))
okc = (ns > 0) & (cyc > 0)
print(f"first_stage->mma_done: median {np.median(cyc[okc]):.0f} SM cycles, {np.median(ns[okc]) / 1e3:.2f} us, "
      f"implied SM clock {np.median(cyc[okc] / ns[okc]) * 1e3:.0f} MHz")
print("level     M N*10+KS tiles |  first_start  max_inputs  max_mma_done  max_acc_ready  max_pub | period")
T0, prev = 0, 0.0
rows = []
for (dd, M, N, nt) in tiles:
    if T0 + nt > ntot:
        break
    sl = slice(T0, T0 + nt)
    r = (dd, M, N, nt, x[0][sl].min(), x[1][sl].max(), x[3][sl].max(), x[4][sl].max(), x[5][sl].max())
    rows.append(r)
    T0 += nt
for i, r in enumerate(rows):
    if i < a.levels or i >= len(rows) - 3:
        print(f"{r[0]:5d} {r[1]:6d} {r[2]:4d} {r[3]:5d} | {r[4]:11.1f} {r[5]:11.1f} {r[6]:13.1f} {r[7]:14.1f} {r[8]:8.1f} | "
              f"{r[8] - (rows[i - 1][8] if i else 0):6.1f}")
# per-level phase medians (us): MMA (first stage -> accumulator committed), the MMA warp's wait
# for a free accumulator (start -> acc_free), the epilogue (accumulator ready -> published) and
# the epilogue's wait on the accumulator of the tile (previous tile published -> acc ready)
print("level tiles | mma(first_stage->mma_done) acc_wait(start->acc_free) epi(acc_ready->published) "
      "slab_rows(slab0_in_smem->rows_done) inputs_wait(start->inputs) acc_ready->slab0_in_smem acc_ready->pt9")
T0 = 0
for (dd, M, N, nt) in tiles:
    if T0 + nt > ntot:
        break
    sl = slice(T0, T0 + nt)
    med = lambda i, j: float(np.median(x[j][sl] - x[i][sl]))
    print(f"{dd:5d} {nt:5d} | {med(8, 3):8.2f} {med(0, 2):8.2f} {med(4, 5):8.2f} {med(6, 7):8.2f} {med(0, 1):8.2f} {med(4, 6):8.2f} {med(4, 9):8.2f}")
    T0 += nt
