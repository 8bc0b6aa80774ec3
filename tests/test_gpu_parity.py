"""Forward / backward parity of the CUDA path against the fp64 oracle.

Bar (BASELINE.json north_star): normwise max relative error <= 1e-5 in FOLD_PREC_FP32,
<= 1e-2 in FOLD_PREC_BF16 (bf16 states/operands, fp32 accumulate), on root h, root c,
dU, db, dE. Sizes span several 128-row tiles per level and ragged tails; S values
include non-multiples of 64 (TMA zero-fill) and of 8 (scalar epilogue tails)."""
import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import random_dag, rel_err

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-5, "bf16": 1e-2}


def _run(gr, cell, prec, S, g=None, gc=None, params=None, want_pool=False):
    import torch
    from paper_1702_02181_b200 import fold
    p = params or foldgen.make_params(cell, S, gr.vocab)
    dev = "cuda"
    model = fold.Model(torch.tensor(p.U, device=dev), torch.tensor(p.b, device=dev), torch.tensor(p.E, device=dev),
                       cell=cell, prec=prec)
    op, child, token, root = fold.graphs_to_device(gr)
    s = fold.schedule(op, child, token, root, gr.vocab)
    h, c, acts = fold.forward(s, model)
    out = {"h": h.cpu().numpy(), "c": c.cpu().numpy(), "sched": s}
    if want_pool:
        H, C = acts.views(s, model)
        out["H"] = H[:, :S].float().cpu().numpy()
        out["C"] = C[:, :S].cpu().numpy()
    if g is not None:
        gd = torch.tensor(g, device=dev)
        gcd = torch.tensor(gc, device=dev) if gc is not None else None
        dU, db, dE = fold.backward(s, model, acts, gd, gcd)
        out.update(dU=dU.cpu().numpy(), db=db.cpu().numpy(), dE=dE.cpu().numpy())
    torch.cuda.synchronize()
    return out, p


def _check_fwd(gr, cell, prec, S):
    got, p = _run(gr, cell, prec, S)
    hr, cr = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E)
    eh = rel_err(got["h"], hr)
    assert eh <= TOL[prec], eh
    if cell == "treelstm":
        ec = rel_err(got["c"], cr)
        assert ec <= TOL[prec], ec
    return eh


def _check_bwd(gr, cell, prec, S, with_dc=False, seed=foldgen.GRAD_SEED):
    g = foldgen.make_upstream(gr.n_graphs, S, seed)
    gc = foldgen.make_upstream(gr.n_graphs, S, seed + 1) if with_dc else None
    got, p = _run(gr, cell, prec, S, g=g, gc=gc)
    dU, db, dE = oracle.backward(cell, gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, g, gc)
    errs = {k: rel_err(got[k], ref) for k, ref in (("dU", dU), ("db", db), ("dE", dE))}
    for k, e in errs.items():
        assert e <= TOL[prec], (k, e)
    return errs


# ------------------------------------------------------------------ forward

@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_c1_treernn_forward(prec):
    """BASELINE configs[0]: TreeRNN over 8 random trees of <= 16 leaves, S=16, V=32."""
    _check_fwd(foldgen.config_c1(), "treernn", prec, 16)


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("S", [16, 80, 128])
def test_treelstm_forward_random_trees(prec, S):
    rng = np.random.default_rng(S)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 40))) for _ in range(40)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 50), 50)
    _check_fwd(gr, "treelstm", prec, S)


def test_pool_states_fp32():
    """Every pool row (not just roots) equals the oracle's node state (fp32 mode)."""
    gr = foldgen.config_c3(32)
    got, p = _run(gr, "treelstm", "fp32", 24, want_pool=True)
    hr, cr, H, C = oracle.forward("treelstm", gr.op, gr.child, gr.token, gr.root, p.U, p.b, p.E, all_nodes=True)
    perm = got["sched"].to_numpy()["perm"]
    assert rel_err(got["H"], H[perm]) <= 1e-5
    assert rel_err(got["C"], C[perm]) <= 1e-5


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_dag_forward(prec):
    rng = np.random.default_rng(9)
    for _ in range(3):
        gr = random_dag(rng, 400, 11)
        gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
        _check_fwd(gr, "treelstm", prec, 32)


def test_c3_forward_bf16_full_state():
    """Parse-shaped trees at the paper's state 300 (§3.5: 'state size from 150 to 300'):
    S=300 is not a multiple of 64 (TMA OOB zero-fill) nor of 8 (scalar tails)."""
    _check_fwd(foldgen.config_c3(64), "treelstm", "bf16", 300)


def test_c2_forward_bf16_full_state():
    """configs[1] shape at full state 1024 on 2 complete 128-leaf trees."""
    _check_fwd(foldgen.config_c2(2), "treelstm", "bf16", 1024)


def test_c4_chain_forward_bf16():
    """configs[3]: depth-256 chains (one row per level per tree): bf16 error over 255
    dependent levels stays within the bar."""
    _check_fwd(foldgen.config_c4(2, leaves=256), "treelstm", "bf16", 128)


# ------------------------------------------------------------------ backward

@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("cell", ["treernn", "treelstm"])
def test_backward_random_trees(prec, cell):
    rng = np.random.default_rng(3)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 30))) for _ in range(30)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 20), 20)
    _check_bwd(gr, cell, prec, 32, with_dc=(cell == "treelstm"))


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_backward_dag(prec):
    """Multi-consumer nodes (pull-reduce over the consumer CSR), cell(x,x), roots that are
    also consumed, shuffled ids."""
    rng = np.random.default_rng(13)
    gr = random_dag(rng, 500, 9, G=6)
    gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
    _check_bwd(gr, "treelstm", prec, 48, with_dc=True)


def test_backward_c3_bf16():
    _check_bwd(foldgen.config_c3(48), "treelstm", "bf16", 300)


def test_backward_c2_bf16_full_state():
    _check_bwd(foldgen.config_c2(2), "treelstm", "bf16", 1024)


def test_backward_zipf_tokens_fp32():
    """Zipf(1) tokens: long token segments in the segmented dE reduction."""
    _check_bwd(foldgen.config_c3(200, vocab=64), "treelstm", "fp32", 16)


def test_single_leaf_and_leaf_only_batch():
    gr = foldgen.batch_from_shapes([foldgen.complete_shape(1)] * 5, lambda n: np.arange(n) % 3, 3)
    _check_bwd(gr, "treelstm", "fp32", 8)
    _check_bwd(gr, "treelstm", "bf16", 8)


def test_determinism_bitwise():
    """Two runs -> bitwise-identical outputs and gradients (no float atomics)."""
    gr = foldgen.config_c3(64)
    g = foldgen.make_upstream(gr.n_graphs, 64)
    a, _ = _run(gr, "treelstm", "bf16", 64, g=g)
    b, _ = _run(gr, "treelstm", "bf16", 64, g=g)
    for k in ("h", "c", "dU", "db", "dE"):
        assert np.array_equal(a[k], b[k]), k


def test_batch_composition_bitwise_fp32():
    """a merged batch gives each tree the result it gets alone. In fp32 mode
    each row's arithmetic does not depend on its batch-mates -> bitwise equality."""
    rng = np.random.default_rng(21)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 20))) for _ in range(6)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 10), 10)
    p = foldgen.make_params("treelstm", 40, 10)
    full, _ = _run(gr, "treelstm", "fp32", 40, params=p)
    for t in range(len(shapes)):
        one = foldgen.sub_batch(gr, t, t + 1)
        o, _ = _run(one, "treelstm", "fp32", 40, params=p)
        assert np.array_equal(o["h"][0], full["h"][t])


@pytest.mark.parametrize("prec", ["fp32", "bf16"])
@pytest.mark.parametrize("S", [1, 7, 33, 130])
def test_odd_and_tiny_state_sizes(prec, S):
    """S not a multiple of 8 / 64, odd S (the tree-like fused backward needs even S and the
    library falls back to the per-level backward), S = 1."""
    rng = np.random.default_rng(100 + S)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(1, 25))) for _ in range(9)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 50), 50)
    _check_fwd(gr, "treelstm", prec, S)
    _check_bwd(gr, "treelstm", prec, S)


def test_large_state_2048_bf16():
    """S = 2048 (K = 4096 per cell GEMM; above the narrow kernels' stationary-U limit, so
    every level runs in the wide kernels)."""
    rng = np.random.default_rng(2048)
    shapes = [foldgen.random_split_shape(rng, int(rng.integers(2, 9))) for _ in range(3)]
    gr = foldgen.batch_from_shapes(shapes, foldgen.uniform_tokens(rng, 40), 40)
    _check_fwd(gr, "treelstm", "bf16", 2048)
    _check_bwd(gr, "treelstm", "bf16", 2048)


def test_very_deep_chain():
    """A caterpillar 5000 levels deep (more levels than fold_schedule's level_off prefix copy
    of 4096 entries, and than any tile counter window): schedule bit-exact, fwd/bwd parity."""
    gr = foldgen.config_c4(2, vocab=64, leaves=5000)
    ref = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    got, p = _run(gr, "treelstm", "bf16", 32)
    assert got["sched"].n_levels == ref["n_levels"] == 5000
    assert np.array_equal(got["sched"].to_numpy()["level_off"], ref["level_off"])
    for prec in ("fp32", "bf16"):
        _check_fwd(gr, "treelstm", prec, 32)
        _check_bwd(gr, "treelstm", prec, 32)


# ------------------------------------------------------------------ instrumentation

@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_profile_classes_bracket_each_sweep_once(prec):
    """fold_profile_enable brackets each level sweep once per call (cell_fwd, gemm_dA), and
    fold_profile_enable_classes records only the requested classes."""
    from paper_1702_02181_b200 import fold
    gr = foldgen.config_c3(32)
    S = 64
    g = foldgen.make_upstream(gr.n_graphs, S)
    fold.profile_enable(True)
    _run(gr, "treelstm", prec, S, g=g)
    allp = fold.profile_read()
    fold.profile_enable(True, classes=("cell_fwd",))
    _run(gr, "treelstm", prec, S, g=g)
    onep = fold.profile_read()
    fold.profile_enable(False)
    assert allp["cell_fwd"][1] == 1 and allp["gemm_dA"][1] == 1 and allp["schedule"][1] == 1
    assert allp["cell_fwd"][0] > 0 and allp["gemm_dA"][0] > 0
    assert onep["cell_fwd"][1] == 1
    assert all(n == 0 for k, (_, n) in onep.items() if k != "cell_fwd")
