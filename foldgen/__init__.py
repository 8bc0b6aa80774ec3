"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NONE of the method's arithmetic: it only produces input graphs
(node op ids, child indices, tokens, roots) and parameter / upstream-gradient
arrays. Depths, schedules, cell math and gradients live in `oracle/` (reference)
and in `paper_1702_02181_b200/` (product); neither is imported here.

Graph encoding (our encoding of PAPER.md L37 "a batch of
multiple input graphs can be treated as a single disconnected graph"):
  op[n]        int32, 0 = EMBED (leaf: embedding lookup of the depth-0 constant
               token[n]), 1 = CELL (binary TreeRNN / TreeLSTM cell).
  child[n, 2]  int32, (left, right) node ids of a CELL; (-1, -1) for EMBED.
  token[n]     int32, word id of an EMBED node (0 for CELL nodes).
  root[g]      int32, node id whose output is graph g's result.
Nodes are numbered in post-order per tree (left subtree, right subtree, node)
and trees are concatenated in batch order; root[g] is the last node of tree g.

Input recipe: graph seed 1702, parameter seed 2181,
upstream-gradient seed 17022181, numpy PCG64.
  C1 TreeRNN tiny   : 8 random-split trees, leaves ~ U{1..16}, S=16, V=32.
  C2 complete-128   : B complete 128-leaf trees ("tree size is 128"),
                      S=1024, V=16384, tokens uniform.
  C3 parse-shaped   : leaves ~ U{1..60}, parse-skew split, S=300, V=16384, Zipf(1) tokens.
  C4 chain-256      : caterpillar of 256 leaves (Fold chain), S=1024.
  C5 train-8192     : 8192 random-split 128-leaf trees, S=1024, V=16384.
"""
from __future__ import annotations

import dataclasses
import numpy as np

EMBED = 0
CELL = 1

GRAPH_SEED = 1702
PARAM_SEED = 2181
GRAD_SEED = 17022181
LABEL_SEED = 297  # §3.5 synthetic per-node sentiment labels
SST_CLASSES = 5


@dataclasses.dataclass
class Graphs:
    op: np.ndarray      # [N] int32
    child: np.ndarray   # [N, 2] int32
    token: np.ndarray   # [N] int32
    root: np.ndarray    # [G] int32
    vocab: int
    tree_sizes: np.ndarray  # [G] nodes per tree (contiguous blocks)

    @property
    def n_nodes(self) -> int:
        return int(self.op.shape[0])

    @property
    def n_graphs(self) -> int:
        return int(self.root.shape[0])


# ----------------------------------------------------------------------------- shapes
# A tree shape is produced as local post-order arrays (op, left, right) with
# child ids local to the tree.

def _shape_from_splits(n_leaves: int, split) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Build a binary tree over a span of `n_leaves` leaves; `split(k)` returns the
    size of the left part (1..k-1) for a span of k >= 2 leaves. Iterative post-order."""
    ops: list[int] = []
    left: list[int] = []
    right: list[int] = []
    # stack entries: (k, state, left_id)
    stack = [[n_leaves, 0, -1, 0]]  # k, stage, left id, split
    ret = -1
    while stack:
        top = stack[-1]
        k, stage = top[0], top[1]
        if k == 1:
            ops.append(EMBED); left.append(-1); right.append(-1)
            ret = len(ops) - 1
            stack.pop()
            continue
        if stage == 0:
            s = int(split(k))
            assert 1 <= s <= k - 1
            top[3] = s
            top[1] = 1
            stack.append([s, 0, -1, 0])
        elif stage == 1:
            top[2] = ret
            top[1] = 2
            stack.append([k - top[3], 0, -1, 0])
        else:
            ops.append(CELL); left.append(top[2]); right.append(ret)
            ret = len(ops) - 1
            stack.pop()
    return (np.asarray(ops, np.int32), np.asarray(left, np.int32), np.asarray(right, np.int32))


def complete_shape(n_leaves: int):
    """Balanced split (left gets ceil(k/2)); for 2^k leaves this is the complete tree."""
    return _shape_from_splits(n_leaves, lambda k: (k + 1) // 2)


def random_split_shape(rng: np.random.Generator, n_leaves: int):
    """Random binary tree: a span of k leaves splits at s ~ U{1..k-1}."""
    return _shape_from_splits(n_leaves, lambda k: rng.integers(1, k))


def parse_skew_shape(rng: np.random.Generator, n_leaves: int):
    """Parse-shaped tree: s = 1 with probability 1/2 (right-branching skew), else U{1..k-1}."""
    def split(k):
        if rng.random() < 0.5:
            return 1
        return rng.integers(1, k)
    return _shape_from_splits(n_leaves, split)


def caterpillar_shape(n_leaves: int):
    """Chain: c_1 = cell(leaf_0, leaf_1), c_k = cell(c_{k-1}, leaf_k)."""
    return _shape_from_splits(n_leaves, lambda k: k - 1)


# ----------------------------------------------------------------------------- batches

def batch_from_shapes(shapes, tokens_fn, vocab: int) -> Graphs:
    """Concatenate tree shapes in batch order; tokens_fn(n) -> int array of n tokens."""
    sizes = np.asarray([len(s[0]) for s in shapes], np.int64)
    N = int(sizes.sum())
    op = np.empty(N, np.int32)
    child = np.full((N, 2), -1, np.int32)
    off = 0
    roots = np.empty(len(shapes), np.int32)
    for g, (o, l, r) in enumerate(shapes):
        n = len(o)
        op[off:off + n] = o
        cl = np.where(l >= 0, l + off, -1)
        cr = np.where(r >= 0, r + off, -1)
        child[off:off + n, 0] = cl
        child[off:off + n, 1] = cr
        roots[g] = off + n - 1
        off += n
    token = np.zeros(N, np.int32)
    leaves = np.nonzero(op == EMBED)[0]
    token[leaves] = tokens_fn(len(leaves)).astype(np.int32)
    return Graphs(op, child, token, roots, vocab, sizes.astype(np.int32))


def replicate_shape(shape, B: int, tokens_fn, vocab: int) -> Graphs:
    """B copies of one shape (vectorised; used for complete trees and chains)."""
    o, l, r = shape
    n = len(o)
    offs = (np.arange(B, dtype=np.int64) * n)[:, None]
    op = np.tile(o, B).astype(np.int32)
    cl = np.where(l[None, :] >= 0, l[None, :] + offs, -1).reshape(-1)
    cr = np.where(r[None, :] >= 0, r[None, :] + offs, -1).reshape(-1)
    child = np.stack([cl, cr], axis=1).astype(np.int32)
    roots = (np.arange(B, dtype=np.int64) * n + n - 1).astype(np.int32)
    token = np.zeros(B * n, np.int32)
    leaves = np.nonzero(op == EMBED)[0]
    token[leaves] = tokens_fn(len(leaves)).astype(np.int32)
    return Graphs(op, child, token, roots, vocab, np.full(B, n, np.int32))


def uniform_tokens(rng: np.random.Generator, vocab: int):
    return lambda n: rng.integers(0, vocab, size=n)


def zipf_tokens(rng: np.random.Generator, vocab: int, s: float = 1.0):
    """Bounded Zipf over [0, vocab): p(k) proportional to 1/(k+1)^s."""
    p = 1.0 / np.power(np.arange(1, vocab + 1, dtype=np.float64), s)
    p /= p.sum()
    cdf = np.cumsum(p)
    def draw(n):
        u = rng.random(n)
        return np.minimum(np.searchsorted(cdf, u, side="right"), vocab - 1)
    return draw


# ----------------------------------------------------------------------------- configs

def config_c1(seed: int = GRAPH_SEED) -> Graphs:
    rng = np.random.default_rng(seed)
    shapes = [random_split_shape(rng, int(rng.integers(1, 17))) for _ in range(8)]
    return batch_from_shapes(shapes, uniform_tokens(rng, 32), 32)


def config_c2(B: int, seed: int = GRAPH_SEED, vocab: int = 16384) -> Graphs:
    rng = np.random.default_rng(seed)
    return replicate_shape(complete_shape(128), B, uniform_tokens(rng, vocab), vocab)


def config_c3(B: int, seed: int = GRAPH_SEED, vocab: int = 16384) -> Graphs:
    rng = np.random.default_rng(seed)
    shapes = [parse_skew_shape(rng, int(rng.integers(1, 61))) for _ in range(B)]
    return batch_from_shapes(shapes, zipf_tokens(rng, vocab), vocab)


def config_c4(B: int, seed: int = GRAPH_SEED, vocab: int = 16384, leaves: int = 256) -> Graphs:
    rng = np.random.default_rng(seed)
    return replicate_shape(caterpillar_shape(leaves), B, uniform_tokens(rng, vocab), vocab)


def config_c5(B: int = 8192, seed: int = GRAPH_SEED, vocab: int = 16384) -> Graphs:
    rng = np.random.default_rng(seed)
    shapes = [random_split_shape(rng, 128) for _ in range(B)]
    return batch_from_shapes(shapes, uniform_tokens(rng, vocab), vocab)


def table1_batch(B: int, same_shape: bool, seed: int = GRAPH_SEED, vocab: int = 16384,
                 leaves: int = 128) -> Graphs:
    """PAPER.md L83/L86 Table 1 inputs: random binary trees of 128 leaves. same_shape=True:
    "a batch of random binary trees, all of which have the same shape" (the manual and
    "dynamic" columns); False: each tree its own random shape ("full dynamic")."""
    rng = np.random.default_rng(seed)
    if same_shape:
        return replicate_shape(random_split_shape(rng, leaves), B, uniform_tokens(rng, vocab), vocab)
    shapes = [random_split_shape(rng, leaves) for _ in range(B)]
    return batch_from_shapes(shapes, uniform_tokens(rng, vocab), vocab)


def manual_levels(gr: Graphs) -> np.ndarray:
    """Caller-fixed levels of the manual-batching baseline ("For the manual
    batching tests, we construct a static data-flow graph of operations corresponding to
    the shape of the tree"): every tree position is its own operation. Leaves (EMBED,
    no dependencies) are level 1; the j-th cell of a tree in node (post-)order is level
    2 + j, so trees of one shape batch position by position and a single tree runs one
    node at a time (the unbatched, batch-size-1 evaluation). Input preparation only:
    the levels are the static graph's op order, not a schedule computation."""
    level = np.ones(gr.n_nodes, np.int32)
    off = 0
    for n in gr.tree_sizes.tolist():
        cells = np.nonzero(gr.op[off:off + n] == CELL)[0]
        level[off + cells] = 2 + np.arange(len(cells), dtype=np.int32)
        off += n
    return level


CONFIG_STATE = {"c1": 16, "c2": 1024, "c3": 300, "c4": 1024, "c5": 1024}


def make_config(name: str, B: int | None = None, seed: int = GRAPH_SEED) -> Graphs:
    name = name.lower()
    if name == "c1":
        return config_c1(seed)
    if name == "c2":
        return config_c2(B or 1024, seed)
    if name == "c3":
        return config_c3(B or 1024, seed)
    if name == "c4":
        return config_c4(B or 1024, seed)
    if name == "c5":
        return config_c5(B or 8192, seed)
    raise ValueError(name)


# ----------------------------------------------------------------------------- params

@dataclasses.dataclass
class Params:
    U: np.ndarray  # [gates*S, 2S] float32 (out x in; gate row blocks i, fL, fR, o, u)
    b: np.ndarray  # [gates*S] float32
    E: np.ndarray  # [V, S] float32


def gates_of(cell: str) -> int:
    return {"treernn": 1, "treelstm": 5}[cell]


def make_params(cell: str, S: int, vocab: int, seed: int = PARAM_SEED) -> Params:
    """U ~ U(+-sqrt(6/(2S + gates*S))), b ~ U(+-0.1), E ~ U(+-0.5)."""
    rng = np.random.default_rng(seed)
    g = gates_of(cell)
    a = np.sqrt(6.0 / (2 * S + g * S))
    U = rng.uniform(-a, a, size=(g * S, 2 * S)).astype(np.float32)
    b = rng.uniform(-0.1, 0.1, size=(g * S,)).astype(np.float32)
    E = rng.uniform(-0.5, 0.5, size=(vocab, S)).astype(np.float32)
    return Params(U, b, E)


def make_upstream(G: int, S: int, seed: int = GRAD_SEED) -> np.ndarray:
    """dL/dh_root, g ~ U(+-1) (L = sum_g <g_g, h_root(g)>)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(G, S)).astype(np.float32)


# ----------------------------------------------------------------------------- misc

def sub_batch(gr: Graphs, t0: int, t1: int) -> Graphs:
    """Trees [t0, t1) of a batch, renumbered from 0 (trees are contiguous node blocks)."""
    cum = np.concatenate([[0], np.cumsum(gr.tree_sizes.astype(np.int64))])
    n0, n1 = int(cum[t0]), int(cum[t1])
    op = gr.op[n0:n1].copy()
    child = gr.child[n0:n1].copy()
    child = np.where(child >= 0, child - n0, -1).astype(np.int32)
    token = gr.token[n0:n1].copy()
    root = (gr.root[t0:t1] - n0).astype(np.int32)
    return Graphs(op, child, token, root, gr.vocab, gr.tree_sizes[t0:t1].copy())


def permute_nodes(gr: Graphs, perm: np.ndarray) -> Graphs:
    """Renumber nodes: new id of old node n is inv[n] where perm[new] = old."""
    N = gr.n_nodes
    inv = np.empty(N, np.int64)
    inv[perm] = np.arange(N)
    op = gr.op[perm].copy()
    child = gr.child[perm].copy()
    child = np.where(child >= 0, inv[np.maximum(child, 0)], -1).astype(np.int32)
    token = gr.token[perm].copy()
    root = inv[gr.root].astype(np.int32)
    return Graphs(op, child, token, root, gr.vocab, gr.tree_sizes.copy())


# ----------------------------------------------------------------------------- §3.5 model (NEXT-2)

@dataclasses.dataclass
class SstParams:
    W: np.ndarray   # [3S, S] leaf input weights, row blocks i, o, u (Tai W^(i), W^(o), W^(u))
    Ws: np.ndarray  # [C, S] per-node classifier
    bs: np.ndarray  # [C]


def make_sst_params(S: int, C: int = SST_CLASSES, seed: int = PARAM_SEED + 1) -> SstParams:
    """W ~ U(+-sqrt(6/(S + 3S))), Ws ~ U(+-sqrt(6/(S + C))), bs ~ U(+-0.1)."""
    rng = np.random.default_rng(seed)
    a = np.sqrt(6.0 / (4 * S))
    W = rng.uniform(-a, a, size=(3 * S, S)).astype(np.float32)
    a2 = np.sqrt(6.0 / (S + C))
    Ws = rng.uniform(-a2, a2, size=(C, S)).astype(np.float32)
    bs = rng.uniform(-0.1, 0.1, size=(C,)).astype(np.float32)
    return SstParams(W, Ws, bs)


def make_labels(N: int, C: int = SST_CLASSES, seed: int = LABEL_SEED) -> np.ndarray:
    """Synthetic per-node labels in node-id order (SST labels every node, PAPER.md L297;
    no dataset: uniform over the C classes)."""
    rng = np.random.default_rng(seed)
    return rng.integers(0, C, size=N).astype(np.int32)


# ----------------------------------------------------------------------------- multi-op (NEXT-3)
# SURVEY §8(f) NEXT-3 / PAPER.md L31-44: several operations and tensor types per depth.
# An op table (enumeration order = op id; "it enumerates them") is input
# data: kind, arity, input / output tensor type, vocabulary; tensor types have state sizes.
# Graph encoding as above with op ids into the table; child[n, k] for k < arity, -1 else.
MO_EMBED, MO_LSTM, MO_RNN = 0, 1, 2
MO_MAXA = 2
MO_SEED = 3133  # the C6 multi-op workload's graph seed


@dataclasses.dataclass
class MoTable:
    kind: np.ndarray      # [n_ops] int32 MO_EMBED / MO_LSTM / MO_RNN
    arity: np.ndarray     # [n_ops] int32 (0 for EMBED, 1..2 else)
    in_type: np.ndarray   # [n_ops] int32 (EMBED: -1)
    out_type: np.ndarray  # [n_ops] int32
    vocab: np.ndarray     # [n_ops] int32 (EMBED: table rows, else 0)
    S: np.ndarray         # [n_types] int32 state size of each tensor type

    @property
    def n_ops(self) -> int:
        return int(self.kind.shape[0])

    @property
    def n_types(self) -> int:
        return int(self.S.shape[0])


def mo_table(ops, S) -> MoTable:
    """ops: list of (kind, arity, in_type, out_type, vocab)."""
    a = np.asarray(ops, np.int64).reshape(-1, 5)
    return MoTable(*(a[:, i].astype(np.int32) for i in range(5)), np.asarray(S, np.int32))


def mo_table_c6(S0: int = 300, S1: int = 128, vocab: int = 16384) -> MoTable:
    """C6 (NEXT-3 workload): constituency-style trees with binary and unary (chain) nodes
    and a typed sentence projection at the root:
      op 0 EMBED  word      -> type 0 (S0)
      op 1 LSTM   arity 2   type 0 -> 0   (binary TreeLSTM)
      op 2 LSTM   arity 1   type 0 -> 0   (unary production: the N = 1 TreeLSTM)
      op 3 RNN    arity 1   type 0 -> 1   (sentence projection into tensor type 1, S1)"""
    return mo_table([(MO_EMBED, 0, -1, 0, vocab), (MO_LSTM, 2, 0, 0, 0), (MO_LSTM, 1, 0, 0, 0),
                     (MO_RNN, 1, 0, 1, 0)], [S0, S1])


@dataclasses.dataclass
class MoGraphs:
    op: np.ndarray      # [N] int32 op ids
    child: np.ndarray   # [N, MO_MAXA] int32
    token: np.ndarray   # [N] int32
    root: np.ndarray    # [G] int32
    table: MoTable

    @property
    def n_nodes(self) -> int:
        return int(self.op.shape[0])

    @property
    def n_graphs(self) -> int:
        return int(self.root.shape[0])


def mo_batch_c6(B: int, seed: int = MO_SEED, table: MoTable | None = None, max_leaves: int = 60,
                p_unary: float = 0.3, zipf: bool = True) -> MoGraphs:
    """B trees: parse-skew binary shapes over 1..max_leaves leaves (C3's distribution); every
    node gets a chain of unary LSTM parents (length ~ Geometric: each link with probability
    p_unary); the root gets the RNN projection (op 3). Post-order numbering per tree."""
    table = table or mo_table_c6()
    rng = np.random.default_rng(seed)
    V = int(table.vocab[0])
    draw = zipf_tokens(rng, V) if zipf else uniform_tokens(rng, V)
    ops, kids, toks, roots = [], [], [], []
    for _ in range(B):
        n_leaves = int(rng.integers(1, max_leaves + 1))
        sop, sl, sr = parse_skew_shape(rng, n_leaves)
        remap = np.empty(len(sop), np.int64)
        for i in range(len(sop)):
            if sop[i] == EMBED:
                ops.append(0); kids.append((-1, -1)); toks.append(int(draw(1)[0]))
            else:
                ops.append(1); kids.append((int(remap[sl[i]]), int(remap[sr[i]]))); toks.append(0)
            top = len(ops) - 1
            while rng.random() < p_unary:
                ops.append(2); kids.append((top, -1)); toks.append(0)
                top = len(ops) - 1
            remap[i] = top
        ops.append(3); kids.append((int(remap[len(sop) - 1]), -1)); toks.append(0)
        roots.append(len(ops) - 1)
    return MoGraphs(np.asarray(ops, np.int32), np.asarray(kids, np.int32).reshape(-1, MO_MAXA),
                    np.asarray(toks, np.int32), np.asarray(roots, np.int32), table)


def make_mo_params(table: MoTable, seed: int = PARAM_SEED) -> list:
    """Per op, in enumeration order: EMBED -> (E [V, S_out],); LSTM / RNN -> (U [rows, a*S_in],
    b [rows]) with rows = (3 + a) S (LSTM) or S_out (RNN); U ~ U(+-sqrt(6/(fan_in + rows))),
    b ~ U(+-0.1), E ~ U(+-0.5). float32 masters."""
    rng = np.random.default_rng(seed)
    out = []
    for o in range(table.n_ops):
        k, a = int(table.kind[o]), int(table.arity[o])
        So = int(table.S[table.out_type[o]])
        if k == MO_EMBED:
            out.append((rng.uniform(-0.5, 0.5, size=(int(table.vocab[o]), So)).astype(np.float32),))
            continue
        Si = int(table.S[table.in_type[o]])
        rows = (3 + a) * So if k == MO_LSTM else So
        lim = np.sqrt(6.0 / (a * Si + rows))
        U = rng.uniform(-lim, lim, size=(rows, a * Si)).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, size=(rows,)).astype(np.float32)
        out.append((U, b))
    return out


def make_mo_upstream(G: int, table: MoTable, seed: int = GRAD_SEED) -> np.ndarray:
    """dL/dh_root as [G, S_max], g ~ U(+-1) (graph g reads the first S_{type(root)} entries)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, size=(G, int(table.S.max()))).astype(np.float32)
