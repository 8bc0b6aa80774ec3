"""Paper-form dynamic-batching schedule with pass-through operations — TEST INFRASTRUCTURE ONLY.

Follows PAPER.md §2 (L37-44) step by step, in the paper's notation:
  1. "Assign a depth to each node ... constants ... depth zero" (L40).
  2. "Insert pass-through (identity) operations so that an operation at depth d+1
     only refers to results at depth d" (L41) — one chain per (source, depth),
     shared by all consumers (our reading, R7 / SPEC S:L405).
  3. "Batch together all nodes invoking the same operation at the same depth" (L42).
  4. "Concatenate all outputs which have the same depth and tensor type. The order of
     concatenation corresponds to the order in which the dynamic batching operations
     were enumerated" (L43) — enumeration [embed, cell], pass-throughs last, ordered by
     their source's row at d-1 (reading R6/R7).
  5. "Assign a label (d, t, i) to each edge ... The schedule ... consists of the indices
     i for all edges, which are grouped together by depth and operation" (L44).
Tensor types: 'int32[]' (the token constants, depth 0) and 'state' (for the TreeLSTM
the (h, c) pair is one fixed-shape [2,S] type; for the TreeRNN it is h).

Pure Python, for tiny graphs (Fig. 1, brute-force shapes); independent of
fold_oracle.c and of the product.
"""
from __future__ import annotations

EMBED, CELL = 0, 1
T_TOK, T_STATE = "int32[]", "state"


def depths(op, child):
    """constants depth 0; otherwise 1 + max depth of dependencies. EMBED's
    dependency is its (depth-0) token constant. Iterative memoised evaluation."""
    N = len(op)
    d = [None] * N
    for s in range(N):
        stack = [s]
        while stack:
            n = stack[-1]
            if d[n] is not None:
                stack.pop(); continue
            if op[n] == EMBED:
                d[n] = 1; stack.pop(); continue
            kids = [int(child[n][0]), int(child[n][1])]
            pend = [k for k in kids if d[k] is None]
            if pend:
                stack.extend(pend); continue
            d[n] = 1 + max(d[k] for k in kids)
            stack.pop()
    return d


def schedule(op, child, token, root):
    """Returns dict with
       'const': the depth-0 int32[] state (tokens of EMBED nodes in id order),
       'levels': list over d = 1..D of list of groups
                 {'op': 'embed'|'cell'|'pass', 'in': [list per input slot], 'rows': n, 'type': t},
       'rows': per d the concatenated row contents [('node', n) | ('pass', src)],
       'results': per graph the label (d, t, i),
       'n_pass': number of pass-through rows inserted."""
    op = [int(x) for x in op]
    child = [(int(c[0]), int(c[1])) for c in child]
    N = len(op)
    d = depths(op, child)
    D = max(d) if N else 0
    # depth-0 constants (not deduplicated): one per EMBED node, in id order
    const_nodes = [n for n in range(N) if op[n] == EMBED]
    const_row = {n: i for i, n in enumerate(const_nodes)}
    # pass-throughs needed: (src, depth) for every edge spanning more than one depth
    need = set()
    for n in range(N):
        if op[n] == CELL:
            for p in child[n]:
                for dd in range(d[p] + 1, d[n]):
                    need.add((p, dd))
    rows = {0: [("const", n) for n in const_nodes]}
    row_of = {}  # (d, ('node', n) | ('pass', p)) -> row index in the d 'state' concat

    def value_row(p, at):
        """row at depth `at` holding node p's value (its own row or its pass-through)."""
        key = ("node", p) if d[p] == at else ("pass", p)
        return row_of[(at, key)]

    levels = []
    for dd in range(1, D + 1):
        groups = []
        embeds = [n for n in range(N) if d[n] == dd and op[n] == EMBED]
        cells = [n for n in range(N) if d[n] == dd and op[n] == CELL]
        passes = [p for (p, x) in need if x == dd]
        # ordered by the source's row at dd-1
        passes.sort(key=lambda p: value_row(p, dd - 1))
        contents = [("node", n) for n in embeds] + [("node", n) for n in cells] + \
                   [("pass", p) for p in passes]
        if embeds:
            groups.append({"op": "embed", "in": [[const_row[n] for n in embeds]],
                           "rows": len(embeds), "type": T_STATE})
        if cells:
            groups.append({"op": "cell",
                           "in": [[value_row(child[n][0], dd - 1) for n in cells],
                                  [value_row(child[n][1], dd - 1) for n in cells]],
                           "rows": len(cells), "type": T_STATE})
        if passes:
            groups.append({"op": "pass", "in": [[value_row(p, dd - 1) for p in passes]],
                           "rows": len(passes), "type": T_STATE})
        for i, key in enumerate(contents):
            row_of[(dd, key)] = i
        rows[dd] = contents
        levels.append(groups)
    results = [(d[r], T_STATE, row_of[(d[r], ("node", int(r)))]) for r in root]
    return {"const": [int(token[n]) for n in const_nodes], "levels": levels, "rows": rows,
            "results": results, "n_pass": len(need), "depth": d}


def dump(sched) -> str:
    """SPEC S:L450 dump format: one line per (depth, op) group, then result labels."""
    out = [f"d=0 const={sched['const']} type={T_TOK}"]
    for dd, groups in enumerate(sched["levels"], start=1):
        for g in groups:
            ins = " ".join(f"in{k}={lst}" for k, lst in enumerate(g["in"]))
            out.append(f"d={dd} op={g['op']} {ins} out_rows={g['rows']} type={g['type']}")
    for lab in sched["results"]:
        out.append(f"result ({lab[0]},{lab[1]},{lab[2]})")
    return "\n".join(out).replace(", ", ",")
