"""Bitwise determinism at the bench shapes (include/fold.h: "bitwise-identical results for
identical inputs (no floating-point atomics)"). VERDICT r01: the fused db
summation of the BF16 dU GEMM raced under load (db differed between identical calls at
C2 B = 256 / 1024 while dZ and dU matched), which a one-shot small test did not catch. Each
case repeats the forward and the backward on the same inputs and compares every output
and gradient bit for bit with the first run."""
import pytest

import foldgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("config,B,reps", [("c2", 1024, 10), ("c2", 256, 20), ("c3", 1024, 20), ("c4", 256, 4),
                                           ("c5", 8192, 3)])
def test_repeated_steps_bitwise(config, B, reps):
    import torch
    from paper_1702_02181_b200 import fold
    gr = foldgen.make_config(config, B)
    S = foldgen.CONFIG_STATE[config]
    p = foldgen.make_params("treelstm", S, gr.vocab)
    dev = "cuda"
    model = fold.Model(*(torch.tensor(x, device=dev) for x in (p.U, p.b, p.E)), prec="bf16")
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
    ws = fold.Workspace(dev)
    first = None
    for r in range(reps):
        h, c, acts = fold.forward(s, model, ws=ws)
        grads = fold.backward(s, model, acts, g, ws=ws)
        cur = [t.clone() for t in (h, c) + tuple(grads)]
        if first is None:
            first = cur
            continue
        for name, x, y in zip(("h", "c", "dU", "db", "dE"), cur, first):
            assert torch.equal(x, y), f"{config} B={B}: {name} differs in repetition {r}"
    del acts, ws, s
    torch.cuda.empty_cache()
