"""GPU scheduler parity: every schedule array bit-exact with the oracle,
status codes and offending ids identical on invalid inputs."""
import json
import os

import numpy as np
import pytest

import foldgen
import oracle
from tests.helpers import random_dag

pytestmark = pytest.mark.gpu

KEYS = ("depth", "perm", "rank", "gather", "level_off", "group_off", "cons_off", "cons_edge", "leaf_perm",
        "tok_seg", "root_row", "root_perm")


def _gpu_sched(gr):
    import torch
    from paper_1702_02181_b200 import fold
    op, child, token, root = fold.graphs_to_device(gr)
    s = fold.schedule(op, child, token, root, gr.vocab)
    torch.cuda.synchronize()
    return s.to_numpy()


def _compare(gr):
    ref = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    got = _gpu_sched(gr)
    for k in KEYS:
        assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), k
    for k in ("n_levels", "n_leaves", "n_cells", "n_tok_segs"):
        assert got[k] == ref[k], k
    # the depth-0 constants in pool order (leaf_token) = token[perm[r]]
    assert np.array_equal(got["leaf_token"], gr.token[ref["perm"][:ref["n_leaves"]]])
    return ref


def test_fig1():
    here = os.path.dirname(os.path.abspath(__file__))
    g = json.load(open(os.path.join(here, "golden", "fig1.json")))
    gr = foldgen.Graphs(np.asarray(g["op"], np.int32), np.asarray(g["child"], np.int32),
                        np.asarray(g["token"], np.int32), np.asarray(g["root"], np.int32), g["vocab"],
                        np.asarray([5], np.int32))
    _compare(gr)


@pytest.mark.parametrize("name,B", [("c1", None), ("c2", 1), ("c2", 3), ("c3", 64), ("c4", 2), ("c5", 16)])
def test_configs(name, B):
    _compare(foldgen.make_config(name, B))


def test_shuffled_ids_and_dags():
    rng = np.random.default_rng(5)
    for _ in range(20):
        gr = random_dag(rng, int(rng.integers(1, 300)), 7)
        gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
        _compare(gr)


def test_adversarial():
    # single leaf; a cell(x, x); chain-256 with reversed ids; big fan-in DAG (one leaf feeding all)
    _compare(foldgen.Graphs(np.asarray([0], np.int32), np.asarray([[-1, -1]], np.int32),
                            np.asarray([3], np.int32), np.asarray([0], np.int32), 4, np.asarray([1])))
    _compare(foldgen.Graphs(np.asarray([0, 1], np.int32), np.asarray([[-1, -1], [0, 0]], np.int32),
                            np.asarray([1, 0], np.int32), np.asarray([1, 1], np.int32), 4, np.asarray([2])))
    gr = foldgen.config_c4(1)
    _compare(foldgen.permute_nodes(gr, np.arange(gr.n_nodes)[::-1].copy()))
    N = 3000
    op = np.ones(N, np.int32); op[0] = 0
    child = np.zeros((N, 2), np.int32); child[0] = -1
    child[1:, 1] = np.arange(N - 1)
    _compare(foldgen.Graphs(op, child, np.zeros(N, np.int32), np.asarray([N - 1], np.int32), 1, np.asarray([N])))


def test_large_batches():
    """Full-size schedules at the bench configurations (C2 B=1024, C5 8192 trees) and a
    parse-shaped batch with shuffled ids: still bit-exact."""
    _compare(foldgen.config_c2(1024))
    _compare(foldgen.config_c5(8192))
    gr = foldgen.config_c3(1024)
    rng = np.random.default_rng(1)
    _compare(foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes)))


def test_empty():
    import torch
    from paper_1702_02181_b200 import fold
    e = torch.zeros(0, dtype=torch.int32, device="cuda")
    s = fold.schedule(e, torch.zeros((0, 2), dtype=torch.int32, device="cuda"), e, e, 4)
    assert s.n_levels == 0 and s.n_nodes == 0


@pytest.mark.parametrize("case,status,node", [
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, 5], [0, 1]], token=[0, 0, 0], root=[2]), "CHILD_RANGE", 1),
    (dict(op=[0, 2, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 0, 0], root=[2]), "OP_RANGE", 1),
    (dict(op=[0, 0, 1, 1], child=[[-1, -1], [-1, -1], [0, -1], [0, 1]], token=[0, 0, 0, 0], root=[3]), "ARITY", 2),
    (dict(op=[0, 1], child=[[0, -1], [0, 0]], token=[0, 0], root=[1]), "ARITY", 0),
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 9, 0], root=[2]), "TOKEN_RANGE", 1),
    (dict(op=[0, 0, 1], child=[[-1, -1], [-1, -1], [0, 1]], token=[0, 0, 0], root=[2, 3]), "ROOT_RANGE", 1),
    (dict(op=[0, 1, 1, 1], child=[[-1, -1], [0, 2], [1, 0], [0, 0]], token=[0, 0, 0, 0], root=[3]), "CYCLE", 1),
    (dict(op=[0, 1, 1], child=[[-1, -1], [0, 2], [0, 1]], token=[0, 0, 0], root=[0]), "CYCLE", 1),
    (dict(op=[0, 1], child=[[-1, -1], [1, 0]], token=[0, 0], root=[0]), "CYCLE", 1),
])
def test_errors_match_oracle(case, status, node):
    from paper_1702_02181_b200 import fold
    with pytest.raises(oracle.OracleError) as eo:
        oracle.schedule(case["op"], case["child"], case["token"], case["root"], 4)
    gr = foldgen.Graphs(np.asarray(case["op"], np.int32), np.asarray(case["child"], np.int32),
                        np.asarray(case["token"], np.int32), np.asarray(case["root"], np.int32), 4,
                        np.asarray([len(case["op"])]))
    with pytest.raises(fold.FoldError) as eg:
        _gpu_sched(gr)
    assert eg.value.status == eo.value.status == status
    assert eg.value.detail == eo.value.node == node
    # (node, depth, op) context: op is the offending node's op id as given
    ctx = fold.last_error_context()
    assert ctx[0] == node
    assert ctx[2] == (-1 if status == "ROOT_RANGE" else case["op"][node])
    assert ctx[1] == -1


def test_error_context_level():
    """FOLD_E_LEVEL reports the offending node's caller-fixed level as its depth."""
    import torch
    from paper_1702_02181_b200 import fold
    op = np.asarray([0, 0, 1, 1], np.int32)
    child = np.asarray([[-1, -1], [-1, -1], [0, 1], [2, 0]], np.int32)
    level = np.asarray([1, 1, 3, 3], np.int32)  # node 3 must be above its child 2
    t = lambda a: torch.from_numpy(a).cuda()
    with pytest.raises(fold.FoldError) as eg:
        fold.schedule(t(op), t(child), t(np.zeros(4, np.int32)), t(np.asarray([3], np.int32)), 4, level=t(level))
    assert eg.value.status == "LEVEL"
    assert fold.last_error_context() == (3, 3, 1)


def test_determinism():
    gr = foldgen.config_c3(256)
    a = _gpu_sched(gr)
    b = _gpu_sched(gr)
    for k in KEYS:
        assert np.array_equal(a[k], b[k])


@pytest.mark.parametrize("name,B", [("c2", 64), ("c4", 32), ("c3", 1024)])
def test_grid_cap_bit_exact(name, B):
    """fold_schedule_ex: a capped scheduler grid (the pipelined schedule beside the dU GEMM)
    gives the oracle's schedule bit for bit, for caps from 1 (acts as 2) to above the default."""
    import torch
    from paper_1702_02181_b200 import fold
    gr = foldgen.make_config(name, B)
    ref = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab)
    op, child, token, root = fold.graphs_to_device(gr)
    for cap in (1, 2, 3, 8, 16, 1000):
        got = fold.schedule(op, child, token, root, gr.vocab, max_blocks=cap).to_numpy()
        torch.cuda.synchronize()
        for k in KEYS:
            assert np.array_equal(np.asarray(got[k]), np.asarray(ref[k])), (cap, k)


@pytest.mark.parametrize("N,seed", [(6000, 1), (20000, 2), (9000, 3)])
def test_multiblock_dag_walk(N, seed):
    """DAGs large enough for the cooperative scheduler (> 4096 nodes): the depth walk with
    pending counts and overflow rounds (shared nodes, cell(x, x)) on shuffled ids, bit-exact
    with the oracle, five times over (a race in the walk would show as a flipped depth)."""
    rng = np.random.default_rng(seed)
    gr = random_dag(rng, N, 50)
    gr = foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes))
    for _ in range(5):
        _compare(gr)


@pytest.mark.parametrize("name,B", [("c4", 64), ("c2", 128), ("c5", 64)])
def test_multiblock_tree_walk_repeat(name, B):
    """Tree-like batches through the exchange-slot walk, repeated with shuffled ids."""
    rng = np.random.default_rng(7)
    gr = foldgen.make_config(name, B)
    _compare(gr)
    _compare(foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes)))


@pytest.mark.parametrize("leaves,B", [(3000, 1), (1200, 3)])
def test_multiblock_deep_chains(leaves, B):
    """Caterpillars deeper than any bench config (depth 3000, one chain walked by one thread in
    the cooperative scheduler), mixed with shuffled ids: bit-exact with the oracle."""
    rng = np.random.default_rng(leaves)
    gr = foldgen.config_c4(B, leaves=leaves)
    _compare(gr)
    _compare(foldgen.permute_nodes(gr, rng.permutation(gr.n_nodes)))
