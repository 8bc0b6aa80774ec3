"""Hunt the BF16 backward nondeterminism: repeat fold_backward on one
forward's activations and compare dU / db / dE / dZ bitwise with the first call; db is also
recomputed from the workspace dZ rows (torch fp64 column sum) to tell a dZ race from a race
in the fused db summation.

    python tools/db_race.py [--config c2] [--batch 256] [--reps 40]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import foldgen  # noqa: E402
from paper_1702_02181_b200 import fold  # noqa: E402


def a256(x):
    return (x + 255) & ~255


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--reps", type=int, default=40)
    args = ap.parse_args()
    gr = foldgen.make_config(args.config, args.batch)
    S = {"c2": 1024, "c3": 300, "c4": 1024, "c5": 1024}[args.config]
    p = foldgen.make_params("treelstm", S, gr.vocab)
    dev = "cuda"
    model = fold.Model(*(torch.tensor(x, device=dev) for x in (p.U, p.b, p.E)), prec="bf16")
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
    ws = fold.Workspace(dev)
    _, _, acts = fold.forward(s, model, ws=ws)
    nc = s.n_cells
    ldz = (5 * S + 7) // 8 * 8
    o_dz = a256((2 * nc + 1) * S * 4)
    o_dz += a256((2 * nc + 1) * S * 4)
    first = None
    bad = {"dU": 0, "db": 0, "dE": 0, "dZ": 0, "db_vs_dZ": 0}
    for r in range(args.reps):
        dU, db, dE = fold.backward(s, model, acts, g, ws=ws)
        torch.cuda.synchronize()
        dZ = ws.bufs["bwd"][o_dz:o_dz + nc * ldz * 2].view(torch.bfloat16).view(nc, ldz)[:, :5 * S]
        db_ref = dZ.double().sum(0)
        cur = {"dU": dU.clone(), "db": db.clone(), "dE": dE.clone(), "dZ": dZ.clone()}
        e = (db.double() - db_ref).abs().max().item() / db_ref.abs().max().item()
        if e > 1e-5:
            bad["db_vs_dZ"] += 1
            d = (db.double() - db_ref).abs()
            idx = torch.nonzero(d > 1e-5 * db_ref.abs().max()).flatten().cpu().numpy()
            print(f"rep {r}: db vs colsum(dZ) rel {e:.3e}; {idx.size} rows differ, first {idx[:16]}", flush=True)
        if first is None:
            first = cur
            continue
        for k in cur:
            if not torch.equal(cur[k], first[k]):
                bad[k] += 1
                dd = (cur[k].double() - first[k].double()).abs()
                nz = torch.nonzero(dd.flatten()).flatten()
                print(f"rep {r}: {k} differs from rep 0 at {nz.numel()} elements, max {dd.max().item():.3e}, "
                      f"first idx {nz[:8].cpu().numpy()}", flush=True)
    print("summary", args.config, args.batch, bad, flush=True)


if __name__ == "__main__":
    main()
