"""Parity with every level forced into the weight-stationary narrow kernels (and with them
disabled), each in a fresh process: the thresholds are read once per process
(FOLD_FWD_NARROW_MAX / FOLD_BWD_NARROW_MAX; fold.h documents no env knob, these are test
hooks). The default-threshold runs of the other GPU tests cover the mixed case."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, %r)
import numpy as np, torch, foldgen, oracle
from paper_1702_02181_b200 import fold
from tests.helpers import rel_err
TOL = 1e-2
def check(gr, S, cell, level=None):
    p = foldgen.make_params(cell, S, gr.vocab)
    g = foldgen.make_upstream(gr.n_graphs, S)
    m = fold.Model(torch.tensor(p.U, device="cuda"), torch.tensor(p.b, device="cuda"),
                   torch.tensor(p.E, device="cuda"), cell=cell, prec="bf16")
    op, child, token, root = fold.graphs_to_device(gr)
    lv = torch.tensor(level, device="cuda") if level is not None else None
    s = fold.schedule(op, child, token, root, gr.vocab, level=lv)
    h, c, acts = fold.forward(s, m)
    dU, db, dE = fold.backward(s, m, acts, torch.tensor(g, device="cuda"))
    torch.cuda.synchronize()
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    rU, rb, rE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    errs = [rel_err(h.cpu().numpy(), hr), rel_err(dU.cpu().numpy(), rU), rel_err(db.cpu().numpy(), rb),
            rel_err(dE.cpu().numpy(), rE)]
    assert max(errs) <= TOL, (S, cell, errs)
check(foldgen.config_c2(3), 1024, "treelstm")
check(foldgen.config_c3(40), 300, "treelstm")
check(foldgen.config_c3(40), 300, "treernn")
gr = foldgen.table1_batch(6, True, leaves=30, vocab=64)
check(gr, 512, "treelstm", foldgen.manual_levels(gr))
gr = foldgen.config_c4(5, leaves=40)
check(gr, 1024, "treelstm")
# chains at S where the child slots' column halves do not align with the column tiles
# (deferred leaf-child tiles of the wide backward, k_bwd_tiles), and mirrored chains (the
# LEFT child is the leaf: the left half's tiles are deferred)
check(foldgen.config_c4(5, leaves=40), 300, "treelstm")
check(foldgen.config_c4(3, leaves=24), 130, "treelstm")
gm = foldgen.config_c4(4, leaves=30)
ch = gm.child.copy()
cells = gm.op == 1
ch[cells] = ch[cells][:, ::-1]
import dataclasses
gm = dataclasses.replace(gm, child=ch)
check(gm, 1024, "treelstm")
check(gm, 300, "treelstm")
print("ok")
""" % ROOT


@pytest.mark.parametrize("mode", ["all_narrow", "no_narrow", "no_narrow_nodefer"])
def test_forced_narrow_modes(mode):
    env = dict(os.environ)
    big = "100000000" if mode == "all_narrow" else "0"
    env.update(FOLD_FWD_NARROW_MAX=big, FOLD_BWD_NARROW_MAX=big)
    if mode == "no_narrow_nodefer":  # every backward tile in the dependent sweep
        env.update(FOLD_BWD_DEFER="0")
    r = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout[-2000:] + r.stderr[-4000:]
