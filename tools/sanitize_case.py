"""One small schedule + forward + backward through the C-ABI, for compute-sanitizer
(SURVEY §4 test layer T5: memcheck / racecheck / synccheck on C1 and small C2 / C3 / C4).

    compute-sanitizer --tool racecheck python tools/sanitize_case.py c2 16 bf16

Arguments: config (c1..c5 | sst), batch, precision (bf16 | tf32 | fp32). Prints the
max |x - y| between two identical backward calls (a race that flips bits shows here too).
The oracle is not used: this is a sanitizer harness, not a parity test.
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import foldgen  # noqa: E402
from paper_1702_02181_b200 import fold  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    prec = sys.argv[3] if len(sys.argv) > 3 else "bf16"
    S_override = int(sys.argv[4]) if len(sys.argv) > 4 else None
    dev = "cuda:0"
    torch.cuda.set_device(0)
    sst = cfg == "sst"
    gr = foldgen.make_config("c3" if sst else cfg, B)
    cell = "treernn" if cfg == "c1" else "treelstm"
    S = S_override or {"c1": 16, "c3": 300, "sst": 300}.get(cfg, 1024)
    p = foldgen.make_params(cell, S, gr.vocab)
    op, child, token, root = fold.graphs_to_device(gr, dev)
    sched = fold.schedule(op, child, token, root, gr.vocab)
    model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev),
                       cell=cell, prec=prec)
    if sst:
        sp = foldgen.make_sst_params(S)
        n = int(gr.op.shape[0])
        head = fold.SstHead(torch.tensor(sp.W, device=dev), torch.tensor(sp.Ws, device=dev),
                            torch.tensor(sp.bs, device=dev),
                            torch.tensor(foldgen.make_labels(n), device=dev))
        loss, acts = fold.sst_forward(sched, model, head)
        g1 = fold.sst_backward(sched, model, head, acts)
        g2 = fold.sst_backward(sched, model, head, acts)
    else:
        h, c, acts = fold.forward(sched, model)
        g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
        g1 = fold.backward(sched, model, acts, g)
        g2 = fold.backward(sched, model, acts, g)
    torch.cuda.synchronize()
    diff = max(float((a - b).abs().max()) for a, b in zip(g1, g2) if torch.is_tensor(a) and a.numel())
    print(f"sanitize_case {cfg} B={B} {prec} S={S}: repeat max|diff| = {diff:.3g}")


if __name__ == "__main__":
    main()
