"""Localise narrow-kernel parity problems: prints per-tensor errors for a few cases."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import foldgen, oracle
from paper_1702_02181_b200 import fold
from tests.helpers import rel_err


def run(gr, level, S, cell="treelstm"):
    p = foldgen.make_params(cell, S, gr.vocab)
    g = foldgen.make_upstream(gr.n_graphs, S)
    model = fold.Model(torch.tensor(p.U, device="cuda"), torch.tensor(p.b, device="cuda"),
                       torch.tensor(p.E, device="cuda"), cell=cell, prec="bf16")
    op, child, token, root = fold.graphs_to_device(gr)
    lv = torch.tensor(level, device="cuda") if level is not None else None
    s = fold.schedule(op, child, token, root, gr.vocab, level=lv)
    h, c, acts = fold.forward(s, model)
    dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device="cuda"))
    torch.cuda.synchronize()
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    rU, rb, rE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    dUn, dbn, dEn = dU.cpu().numpy(), db.cpu().numpy(), dE.cpu().numpy()
    out = {"h": rel_err(h.cpu().numpy(), hr), "dU": rel_err(dUn, rU), "db": rel_err(dbn, rb), "dE": rel_err(dEn, rE)}
    # per gate block of db, nan counts
    out["db_blocks"] = [round(rel_err(dbn[k * S:(k + 1) * S], rb[k * S:(k + 1) * S]), 4) for k in range(len(rb) // S)]
    out["nan_dU"] = int(np.isnan(dUn).sum()); out["nan_dE"] = int(np.isnan(dEn).sum())
    bad_tok = np.nonzero(np.abs(dEn - rE).max(1) > 1e-2 * np.abs(rE).max())[0]
    out["bad_tokens"] = len(bad_tok)
    return out


print("mode", os.environ.get("FOLD_BWD_NARROW_MAX"))
gr = foldgen.config_c2(1)
print("C2 B=1 dyn", run(gr, None, 1024))
print("C2 B=1 manual", run(gr, foldgen.manual_levels(gr), 1024))
gr = foldgen.table1_batch(3, False, leaves=40, vocab=64)
print("S512 random B=3 dyn", run(gr, None, 512))
gr = foldgen.config_c4(1)
print("C4 B=1", run(gr, None, 1024))
gr = foldgen.config_c3(64)
print("C3 B=64 S=300", run(gr, None, 300))
print("C3 B=64 S=300 manual", run(gr, foldgen.manual_levels(gr), 300))
print("C3 B=64 S=300 rnn", run(gr, None, 300, cell="treernn"))
