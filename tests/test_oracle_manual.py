"""Pins for the oracle's manual-batching schedule (caller-fixed levels; PAPER.md L83 and
Table 1: "For the manual batching tests, we construct a static data-flow graph of
operations corresponding to the shape of the tree"). Expected values are hand-derived
or follow from the definition (rows ordered by (level, op, id)), independently of the
oracle's code."""
import json
import os

import numpy as np
import pytest

import foldgen
import oracle

HERE = os.path.dirname(os.path.abspath(__file__))


def test_fig1_manual_equals_dynamic():
    """Fig. 1 (L58-77): post-order cells n2, n4 are cell positions 0, 1 -> levels 2, 3,
    which are also their L40 depths, so the manual schedule IS the golden dynamic one."""
    g = json.load(open(os.path.join(HERE, "golden", "fig1.json")))
    gr = foldgen.Graphs(np.asarray(g["op"], np.int32), np.asarray(g["child"], np.int32),
                        np.asarray(g["token"], np.int32), np.asarray(g["root"], np.int32), g["vocab"],
                        np.asarray([5], np.int32))
    lv = foldgen.manual_levels(gr)
    assert lv.tolist() == [1, 1, 2, 1, 3]
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab, level=lv)
    exp = g["executor_form"]
    for k in ("depth", "perm", "rank", "level_off", "group_off", "cons_off", "cons_edge", "root_row"):
        assert s[k].tolist() == exp[k], k


def test_four_leaf_complete_manual():
    """4-leaf complete tree, post-order ids 0=E 1=E 2=C(0,1) 3=E 4=E 5=C(3,4) 6=C(2,5).
    Manual levels [1,1,2,1,1,3,4] (hand-derived): one row per cell level, so cell 5 no
    longer shares a level with cell 2 as it does under L40 depths."""
    o, l, r = foldgen.complete_shape(4)
    gr = foldgen.replicate_shape((o, l, r), 1, lambda n: np.zeros(n), 1)
    lv = foldgen.manual_levels(gr)
    assert lv.tolist() == [1, 1, 2, 1, 1, 3, 4]
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 1, level=lv)
    assert s["perm"].tolist() == [0, 1, 3, 4, 2, 5, 6]
    assert s["level_off"].tolist() == [0, 0, 4, 5, 6, 7]
    assert s["gather"][4:].tolist() == [[0, 1], [2, 3], [4, 5]]
    assert s["n_levels"] == 4
    d = oracle.schedule(gr.op, gr.child, gr.token, gr.root, 1)
    assert d["level_off"].tolist() == [0, 0, 4, 6, 7]


@pytest.mark.parametrize("B", [1, 2, 5])
def test_same_shape_batches_position_by_position(B):
    """Table 1 'manual' column: B trees of one random shape; each cell position is its
    own op, so every cell level holds exactly B rows (one per tree, in tree order) and
    there are (cells per tree) + 1 levels. B = 1 is the unbatched evaluation."""
    gr = foldgen.table1_batch(B, True, leaves=20)
    lv = foldgen.manual_levels(gr)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab, level=lv)
    n = int(gr.tree_sizes[0])
    ncell = 19
    assert s["n_levels"] == ncell + 1
    assert s["level_off"].tolist() == [0, 0] + [20 * B + j * B for j in range(0, ncell + 1)]
    cells_of_tree0 = np.nonzero(gr.op[:n] == 1)[0]
    for j in range(ncell):
        rows = s["perm"][20 * B + j * B: 20 * B + (j + 1) * B]
        assert rows.tolist() == [t * n + cells_of_tree0[j] for t in range(B)]


def test_manual_invariants_random_shapes():
    """Level order is a topological order: every gather points below the row's level."""
    gr = foldgen.table1_batch(7, False, leaves=30)
    lv = foldgen.manual_levels(gr)
    s = oracle.schedule(gr.op, gr.child, gr.token, gr.root, gr.vocab, level=lv)
    lo = s["level_off"]
    for r in range(s["n_leaves"], gr.n_nodes):
        d = s["depth"][s["perm"][r]]
        assert (s["gather"][r] < lo[d]).all() and (s["gather"][r] >= 0).all()
    # ragged: levels beyond the smallest tree's cell count hold fewer than B rows
    widths = np.diff(lo)[2:]
    assert widths.max() == 7 and widths.min() >= 1


@pytest.mark.parametrize("case,node", [
    (dict(level=[1, 1, 1]), 2),            # cell not above its children
    (dict(level=[2, 1, 3]), 0),            # EMBED must be level 1
    (dict(level=[1, 1, 4]), 2),            # level > n_nodes
    (dict(level=[1, 1, 0]), 2),            # level < 1
])
def test_level_errors(case, node):
    with pytest.raises(oracle.OracleError) as ei:
        oracle.schedule([0, 0, 1], [[-1, -1], [-1, -1], [0, 1]], [0, 0, 0], [2], 4, level=case["level"])
    assert ei.value.status == "LEVEL" and ei.value.node == node


def test_level_error_after_root_range():
    """Class order: ROOT_RANGE is reported before LEVEL (fold.h error order)."""
    with pytest.raises(oracle.OracleError) as ei:
        oracle.schedule([0, 0, 1], [[-1, -1], [-1, -1], [0, 1]], [0, 0, 0], [5], 4, level=[2, 1, 3])
    assert ei.value.status == "ROOT_RANGE"


def test_empty_levels_allowed():
    """Levels may skip values: level 2 is empty, offsets repeat."""
    s = oracle.schedule([0, 0, 1], [[-1, -1], [-1, -1], [0, 1]], [0, 0, 0], [2], 4, level=[1, 1, 3])
    assert s["n_levels"] == 3 and s["level_off"].tolist() == [0, 0, 2, 2, 3]


@pytest.mark.parametrize("cell", ["treernn", "treelstm"])
def test_manual_forward_bitwise_equals_node_at_a_time(cell):
    """the result does not depend on how nodes are batched; manual levels
    through the level loop equal node-at-a-time evaluation bit for bit."""
    rng = np.random.default_rng(11)
    S, V = 6, 9
    g = foldgen.gates_of(cell)
    U = rng.uniform(-0.5, 0.5, (g * S, 2 * S)); b = rng.uniform(-0.1, 0.1, g * S); E = rng.uniform(-0.5, 0.5, (V, S))
    gr = foldgen.table1_batch(5, False, leaves=13, vocab=V)
    _, _, H, C = oracle.forward(cell, gr.op, gr.child, gr.token, gr.root, U, b, E, all_nodes=True)
    H2, C2 = oracle.forward_levels(cell, gr.op, gr.child, gr.token, gr.root, U, b, E,
                                   level=foldgen.manual_levels(gr))
    assert np.array_equal(H, H2) and np.array_equal(C, C2)
