"""NEXT-2: the §3.5 sentiment model on the GPU path against the fp64
oracle (oracle_sst_forward / oracle_sst_backward, pinned in test_oracle_sst.py): leaves
h = TreeLSTM(E[w], 0, 0), internal TreeLSTM(0, h_L, h_R), 5-way softmax cross-entropy at
every node. FP32 mode (3xTF32 tensor-core GEMMs) at the north_star's 1e-5, TF32 at 1e-2,
on the loss and all six gradients; parse-shaped SST-like trees (C3 shapes, S = 300 like the
paper's "increased the LSTM state size ... to 300", L329), complete trees, a DAG with
sharing, odd S, determinism."""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import random_dag, rel_err

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "tf32": 1e-2}


def _gpu(gr, S, prec, y, p, q, reps=1):
    import torch
    from paper_1702_02181_b200 import fold
    dev = "cuda"
    t = lambda x: torch.tensor(x, device=dev)
    model = fold.Model(t(p.U), t(p.b), t(p.E), prec=prec)
    head = fold.SstHead(t(q.W), t(q.Ws), t(q.bs), torch.tensor(y, dtype=torch.int32, device=dev))
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    outs = []
    for _ in range(reps):
        loss, acts = fold.sst_forward(s, model, head)
        grads = fold.sst_backward(s, model, head, acts)
        torch.cuda.synchronize()
        outs.append([float(loss.item())] + [g.cpu().numpy() for g in grads])
    return outs


def _check(gr, S, prec, seed=0):
    p = foldgen.make_params("treelstm", S, gr.vocab, seed=foldgen.PARAM_SEED + seed)
    q = foldgen.make_sst_params(S)
    y = foldgen.make_labels(gr.n_nodes)
    got = _gpu(gr, S, prec, y, p, q)[0]
    ref = oracle.sst_backward(gr.op, gr.child, gr.token, y, p.U, p.b, p.E, q.W, q.Ws, q.bs)
    errs = {"loss": abs(got[0] - ref[0]) / abs(ref[0])}
    for name, x, r in zip(("dU", "db", "dE", "dW", "dWs", "dbs"), got[1:], ref[1:]):
        errs[name] = rel_err(x, r)
    for k, e in errs.items():
        assert e <= TOL[prec], (prec, k, e, errs)
    return errs


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_sst_parse_trees_s300(prec):
    _check(foldgen.config_c3(48), 300, prec)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_sst_complete_trees(prec):
    _check(foldgen.config_c2(3, vocab=500), 128, prec)


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("S", [1, 7, 33])
def test_sst_small_odd_states(prec, S):
    rng = np.random.default_rng(S)
    shapes = [foldgen.parse_skew_shape(rng, int(rng.integers(1, 20))) for _ in range(12)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.zipf_tokens(rng, 40), 40)
    _check(gr, S, prec)


def test_sst_dag_with_sharing():
    rng = np.random.default_rng(8)
    gr = random_dag(rng, 200, 13, G=3)
    gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
    _check(gr, 24, "fp32")


def test_sst_deterministic_and_accumulate():
    import torch
    from paper_1702_02181_b200 import fold
    gr = foldgen.config_c3(64)
    S = 64
    p = foldgen.make_params("treelstm", S, gr.vocab)
    q = foldgen.make_sst_params(S)
    y = foldgen.make_labels(gr.n_nodes)
    a, b = _gpu(gr, S, "fp32", y, p, q, reps=2)
    assert a[0] == b[0]
    for x, z in zip(a[1:], b[1:]):
        assert np.array_equal(x, z)
    # accumulate = 1 adds a second backward's gradients
    dev = "cuda"
    t = lambda x: torch.tensor(x, device=dev)
    model = fold.Model(t(p.U), t(p.b), t(p.E), prec="fp32")
    head = fold.SstHead(t(q.W), t(q.Ws), t(q.bs), torch.tensor(y, dtype=torch.int32, device=dev))
    s = fold.schedule(*fold.graphs_to_device(gr, dev), gr.vocab)
    _, acts = fold.sst_forward(s, model, head)
    g1 = [g.clone() for g in fold.sst_backward(s, model, head, acts)]
    g2 = fold.sst_backward(s, model, head, acts, grads=tuple(x.clone() for x in g1), accumulate=True)
    for x, z in zip(g2, g1):
        x, z = x.double().cpu().numpy(), z.double().cpu().numpy()
        assert np.abs(x - 2 * z).max() <= 1e-5 * 2 * max(np.abs(z).max(), 1e-30)


def test_sst_rejects_bf16():
    import torch
    from paper_1702_02181_b200 import fold
    gr = foldgen.config_c1()
    S = 16
    p = foldgen.make_params("treelstm", S, gr.vocab)
    q = foldgen.make_sst_params(S)
    t = lambda x: torch.tensor(x, device="cuda")
    model = fold.Model(t(p.U), t(p.b), t(p.E), prec="bf16")
    head = fold.SstHead(t(q.W), t(q.Ws), t(q.bs), t(foldgen.make_labels(gr.n_nodes)))
    s = fold.schedule(*fold.graphs_to_device(gr, "cuda"), gr.vocab)
    with pytest.raises(fold.FoldError) as e:
        fold.sst_forward(s, model, head)
    assert e.value.status == "UNSUPPORTED"
