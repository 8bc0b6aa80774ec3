"""The pipelined training step that bench.py times (the next batch's
fold_schedule runs on a side stream while this batch's forward / backward / SGD run; three
rotating schedule buffers; the schedule optionally gated on fold_backward's sweep_done
event) gives bit-identical parameters to the same steps run one after another on one
stream. Every kernel is deterministic, so a missing stream or event dependency (a schedule
buffer rewritten while a step still reads it, a step starting before its schedule is
complete) shows up as a difference."""
import numpy as np
import pytest
import torch

import foldgen

pytestmark = pytest.mark.gpu

LR = 0.05


def _run(gr, S, steps, mode):
    from paper_1702_02181_b200 import fold
    dev = "cuda"
    p = foldgen.make_params("treelstm", S, gr.vocab)
    U, b, E = (torch.tensor(x, device=dev) for x in (p.U, p.b, p.E))
    model = fold.Model(U, b, E)
    dU, db, dE = torch.empty_like(U), torch.empty_like(b), torch.empty_like(E)
    ws = fold.Workspace(dev)
    o = fold.graphs_to_device(gr, dev)
    g = torch.tensor(foldgen.make_upstream(gr.n_graphs, S), device=dev)

    def train(sc, sweep=None):
        _, _, acts = fold.forward(sc, model, ws=ws, want_c=False)
        fold.backward(sc, model, acts, g, grads=(dU, db, dE), ws=ws, sweep_done=sweep)
        for prm, grd in ((U, dU), (b, db), (E, dE)):
            fold.sgd_update(prm, grd, LR)

    if mode == "serial":
        for _ in range(steps):
            train(fold.schedule(*o, gr.vocab))
    else:
        side = torch.cuda.Stream()
        main = torch.cuda.current_stream()
        n = fold.schedule_buffer_len(int(o[0].shape[0]), int(o[3].shape[0]))
        sbuf = [torch.empty(n, dtype=torch.int32, device=dev) for _ in range(3)]
        free = [torch.cuda.Event() for _ in range(3)]
        used = [False] * 3
        sweep = torch.cuda.Event()

        def schedule_async(i, after):
            with torch.cuda.stream(side):
                if used[i]:
                    side.wait_event(free[i])
                if after is not None:
                    side.wait_event(after)
                sc = fold.schedule(*o, gr.vocab, stream=side, out=sbuf[i])
                ev = torch.cuda.Event()
                ev.record(side)
            return sc, ev

        sc, ev = schedule_async(0, None)
        for k in range(steps):
            main.wait_event(ev)
            train(sc, sweep)
            free[k % 3].record(main)
            used[k % 3] = True
            if k + 1 < steps:
                sc, ev = schedule_async((k + 1) % 3, sweep if mode == "gated" else None)
    torch.cuda.synchronize()
    return U.cpu().numpy(), b.cpu().numpy(), E.cpu().numpy()


@pytest.mark.parametrize("cfg,B", [("c2", 16), ("c3", 64), ("c4", 4)])
def test_pipelined_steps_match_serial(cfg, B):
    gr = foldgen.make_config(cfg, B)
    S = foldgen.CONFIG_STATE[cfg]
    ref = _run(gr, S, 4, "serial")
    for mode in ("pipelined", "gated"):
        got = _run(gr, S, 4, mode)
        for name, x, y in zip(("U", "b", "E"), got, ref):
            assert np.array_equal(x, y), f"{cfg} B={B} {mode}: {name} differs from the serial steps"
    # the steps did train: the parameters moved
    p0 = foldgen.make_params("treelstm", S, gr.vocab)
    assert not np.array_equal(ref[0], p0.U)
