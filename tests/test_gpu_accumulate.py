"""fold_grads.accumulate (fold.h): a second fold_backward with accumulate = 1 adds its
gradients to dU, db, dE. The kernels are deterministic, so two identical calls give
twice one call's gradients up to the rounding of the final additions (the accumulated
value joins the fixed-order sums first) — through every output path: dU / db written
directly (one split-K slab) and through the split-K partials, the embedding gradient, FP32
and BF16 modes."""
import numpy as np
import pytest
import torch

import foldgen

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec,B", [("bf16", 2), ("fp32", 2), ("bf16", 256)])
def test_accumulate_doubles(prec, B):
    from paper_1702_02181_b200 import fold
    gr = foldgen.make_config("c2", B)
    S = 1024
    p = foldgen.make_params("treelstm", S, gr.vocab)
    dev = "cuda"
    model = fold.Model(*(torch.tensor(x, device=dev) for x in (p.U, p.b, p.E)), prec=prec)
    o = fold.graphs_to_device(gr, dev)
    s = fold.schedule(*o, gr.vocab)
    g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
    ws = fold.Workspace(dev)
    _, _, acts = fold.forward(s, model, ws=ws)
    one = [t.clone() for t in fold.backward(s, model, acts, g, ws=ws)]
    grads = tuple(t.clone() for t in one)
    fold.backward(s, model, acts, g, grads=grads, accumulate=True, ws=ws)
    torch.cuda.synchronize()
    for name, x, y in zip(("dU", "db", "dE"), grads, one):
        x, y = x.double().cpu().numpy(), y.double().cpu().numpy()
        scale = np.abs(y).max()
        assert scale > 0
        # a handful of fp32 roundings of the running sums (split-K / token pieces)
        assert np.abs(x - 2 * y).max() <= 1e-5 * 2 * scale, f"{prec} B={B}: {name} is not twice one backward"


def test_misaligned_gradients_rejected():
    """fold.h fold_grads: dU / db / dE must be 16-byte aligned (vectorised stores and
    read-modify-writes); a misaligned view is FOLD_E_INVALID, not a device fault."""
    from paper_1702_02181_b200 import fold
    gr = foldgen.make_config("c2", 2)
    S = 64
    p = foldgen.make_params("treelstm", S, gr.vocab)
    dev = "cuda"
    model = fold.Model(*(torch.tensor(x, device=dev) for x in (p.U, p.b, p.E)), prec="bf16")
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)
    _, _, acts = fold.forward(s, model)
    ok = [torch.empty_like(t) for t in (model.U, model.b, model.E)]
    for i in range(3):
        bad = list(ok)
        raw = torch.empty(ok[i].numel() + 1, dtype=torch.float32, device=dev)
        bad[i] = raw[1:].view_as(ok[i])
        with pytest.raises(fold.FoldError) as ei:
            fold.backward(s, model, acts, g, grads=tuple(bad))
        assert ei.value.status == "INVALID"
    fold.backward(s, model, acts, g, grads=tuple(ok))
    torch.cuda.synchronize()
