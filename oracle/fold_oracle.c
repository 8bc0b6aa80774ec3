/*
 * oracle/fold_oracle.c — fp64 CPU ORACLE for dynamic batching (arXiv 1702.02181).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. The product path
 * (paper_1702_02181_b200/, include/fold.h, libfold.so) never links, includes or
 * calls anything here, and this file includes nothing from the product.
 *
 * What it computes, each function citing the passage it follows:
 *   oracle_schedule      — the dynamic-batching schedule by its definition
 *                          (§2 bullets 1-5), executor form
 *                          (global append-only pool, no pass-throughs; the
 *                          paper form with pass-throughs is oracle/paper_form.py).
 *   oracle_forward       — every node evaluated individually, one at a time, in a
 *                          topological order (batching reaches the
 *                          unbatched result; L86 "no measurable penalty ...").
 *   oracle_forward_levels— the same values computed level by level from this
 *                          oracle's own schedule (PAPER.md L47 loop model); used
 *                          only to pin "batched == unbatched" bitwise.
 *   (both schedule functions take optional caller-fixed levels: the manual-batching
 *    baseline of PAPER.md L83 / Table 1, where each tree position is its own op)
 *   oracle_backward      — hand-derived reverse mode ("gradients ...
 *                          do not require any additional code" in TF; here written
 *                          out), pinned by finite differences in tests/.
 *   oracle_sst_forward / oracle_sst_backward
 *                        — the §3.5 sentiment model: leaves
 *                          h = TreeLSTM(E[w], 0, 0), internal TreeLSTM(0, h_L, h_R),
 *                          5-way softmax cross-entropy at every node (NEXT-2).
 * All floating point is fp64; parameters arrive as fp64 copies of the fp32 masters.
 *
 * Cell equations (Tai et al. eqs 9-14 with x = 0, N = 2, cited
 * at PAPER.md L301-304; TreeRNN form read from Fig. 1 "RNN Cell"):
 *   TreeRNN  (gates=1): z = W [h_L; h_R] + b,   h = tanh(z),  c = 0
 *   TreeLSTM (gates=5, row blocks i, fL, fR, o, u of U[5S][2S]):
 *     z = U [h_L; h_R] + b
 *     i = s(z_i), fL = s(z_fL), fR = s(z_fR), o = s(z_o), u = tanh(z_u)
 *     c = i*u + fL*c_L + fR*c_R,   h = o*tanh(c)
 *   EMBED: h = E[token], c = 0        (leaf; its token is the depth-0 constant)
 *   s(x) = 1 / (1 + exp(-x))
 *
 * Status codes are this file's own (the product's fold.h defines its own; tests
 * compare by name).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { OR_OK = 0, OR_E_INVALID = 1, OR_E_CHILD_RANGE = 2, OR_E_ARITY = 3,
       OR_E_TOKEN_RANGE = 4, OR_E_ROOT_RANGE = 5, OR_E_CYCLE = 6, OR_E_OP_RANGE = 10,
       OR_E_LEVEL = 12 };
enum { OR_EMBED = 0, OR_CELL = 1, OR_N_OPS = 2 };
enum { OR_TREERNN = 0, OR_TREELSTM = 1 };

/* ---------------------------------------------------------------- validation */
/* Error classes checked in this order; the smallest offending node id (graph id
 * for ROOT_RANGE) of the first failing class is reported. */
static int validate(int N, int G, int V, const int32_t *op, const int32_t *child,
                    const int32_t *token, const int32_t *root, int32_t *err)
{
    for (int n = 0; n < N; n++)
        for (int k = 0; k < 2; k++)
            if (child[2 * n + k] < -1 || child[2 * n + k] >= N) { *err = n; return OR_E_CHILD_RANGE; }
    for (int n = 0; n < N; n++)
        if (op[n] != OR_EMBED && op[n] != OR_CELL) { *err = n; return OR_E_OP_RANGE; }
    for (int n = 0; n < N; n++) {
        int nch = (child[2 * n] >= 0) + (child[2 * n + 1] >= 0);
        int ok = (op[n] == OR_EMBED) ? (child[2 * n] == -1 && child[2 * n + 1] == -1)
                                     : (nch == 2);
        if (!ok) { *err = n; return OR_E_ARITY; }
    }
    for (int n = 0; n < N; n++)
        if (op[n] == OR_EMBED && (token[n] < 0 || token[n] >= V)) { *err = n; return OR_E_TOKEN_RANGE; }
    for (int g = 0; g < G; g++)
        if (root[g] < 0 || root[g] >= N) { *err = g; return OR_E_ROOT_RANGE; }
    return OR_OK;
}

/* Caller-fixed levels (manual batching: "For the manual batching tests, we
 * construct a static data-flow graph of operations corresponding to the shape of the
 * tree"): a level replaces the L40 depth. Valid when every EMBED has level 1, every
 * level is in [1, N] and every CELL's level exceeds both children's levels (so the
 * level order is a topological order). Smallest offending node id. */
static int validate_levels(int N, const int32_t *op, const int32_t *child, const int32_t *level,
                           int32_t *err)
{
    for (int n = 0; n < N; n++) {
        int bad = level[n] < 1 || level[n] > N;
        if (op[n] == OR_EMBED && level[n] != 1) bad = 1;
        if (op[n] == OR_CELL && (level[n] <= level[child[2 * n]] || level[n] <= level[child[2 * n + 1]])) bad = 1;
        if (bad) { *err = n; return OR_E_LEVEL; }
    }
    return OR_OK;
}

/* ---------------------------------------------------------------- depth
 * "Nodes with no dependencies (constants) are assigned depth zero. Nodes with only
 * dependencies of depth zero are assigned depth one, nodes whose dependencies have
 * a maximum depth of one get assigned depth two, etc."
 * EMBED's only dependency is its token constant (depth 0) => depth 1.
 * CELL => 1 + max(depth(L), depth(R)).
 * Memoised DFS with an explicit stack and white/grey/black colouring. A node that
 * reaches a cycle (grey child) or a bad child is "bad"; the cycle error reports the
 * smallest bad id. Also emits a post-order (children before parents) in `topo`. */
static int assign_depths(int N, const int32_t *op, const int32_t *child,
                         int32_t *depth, int32_t *topo, int32_t *err)
{
    enum { WHITE = 0, GREY = 1, OK = 2, BAD = 3 };
    unsigned char *col = (unsigned char *)calloc((size_t)N + 1, 1);
    int32_t *stk = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
    int32_t *nxt = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1)); /* next child slot */
    int ntopo = 0, any_bad = 0;
    for (int s = 0; s < N; s++) {
        if (col[s] != WHITE) continue;
        int sp = 0;
        stk[sp++] = s; col[s] = GREY; nxt[s] = 0;
        while (sp > 0) {
            int n = stk[sp - 1];
            int nc = (op[n] == OR_CELL) ? 2 : 0;
            if (nxt[n] < nc) {
                int c = child[2 * n + nxt[n]];
                nxt[n]++;
                if (col[c] == WHITE) { col[c] = GREY; nxt[c] = 0; stk[sp++] = c; }
                /* grey child = back edge (cycle); handled when n finishes */
                continue;
            }
            /* all children visited: finish n */
            int bad = 0, dmax = 0;
            for (int k = 0; k < nc; k++) {
                int c = child[2 * n + k];
                if (col[c] == GREY || col[c] == BAD) bad = 1;
                else if (depth[c] > dmax) dmax = depth[c];
            }
            if (bad) { col[n] = BAD; depth[n] = -1; any_bad = 1; }
            else { col[n] = OK; depth[n] = (op[n] == OR_EMBED) ? 1 : 1 + dmax; topo[ntopo++] = n; }
            sp--;
        }
    }
    int st = OR_OK;
    if (any_bad) {
        for (int n = 0; n < N; n++) if (col[n] == BAD) { *err = n; break; }
        st = OR_E_CYCLE;
    }
    free(col); free(stk); free(nxt);
    return st;
}

/* ---------------------------------------------------------------- schedule
 * Executor form:
 *  perm: for d = 1..D, for op in enumeration order (EMBED=0, CELL=1; PAPER.md L43
 *        "The order of concatenation corresponds to the order in which the dynamic
 *        batching operations were enumerated"), for n ascending with (depth, op) =
 *        (d, op): append n  ("Batch together all nodes invoking the same
 *        operation at the same depth"). Filled with bucket lists in one id-ordered pass.
 *  rank = perm^-1 (the pool row of each node).
 *  level_off[d] = #rows with depth < d, d = 0..D+1.
 *  group_off[k] = #rows with key < k, key = 2*depth + op, k = 0..2(D+1).
 *  gather[r][k] = rank[child[perm[r]][k]] for CELL rows, -1 otherwise (PAPER.md L44:
 *        the label i of an edge; here the global pool row; the paper's per-depth
 *        index is gather - level_off[depth(child)]).
 *  cons_off/cons_edge: for every child row (ascending), its consumer edges e = 2c + k
 *        in ascending e, where c = r - n_leaves is the cell index of consumer row r
 *        (all EMBED rows precede all CELL rows: EMBED depth = 1 < CELL depth).
 *  leaf_perm: EMBED rows sorted by (token, row); tok_seg: segment starts + end.
 *  root_row[g] = rank[root[g]]; root_perm: graph ids sorted by (root_row, g).
 * info[0..4] = n_levels (D), n_leaves, n_cells, n_tok_segs, err_node.
 */
int oracle_schedule(int N, int G, int V, const int32_t *op, const int32_t *child,
                    const int32_t *token, const int32_t *root, const int32_t *level,
                    int32_t *depth, int32_t *perm, int32_t *rank, int32_t *gather,
                    int32_t *level_off, int32_t *group_off, int32_t *cons_off,
                    int32_t *cons_edge, int32_t *leaf_perm, int32_t *tok_seg,
                    int32_t *root_row, int32_t *root_perm, int32_t *info)
{
    int32_t err = -1;
    info[0] = info[1] = info[2] = info[3] = 0; info[4] = -1;
    if (N < 0 || G < 0 || V < 0) return OR_E_INVALID;
    int st = validate(N, G, V, op, child, token, root, &err);
    if (st != OR_OK) { info[4] = err; return st; }
    if (level) {   /* manual batching: the caller's levels are the depths */
        st = validate_levels(N, op, child, level, &err);
        if (st != OR_OK) { info[4] = err; return st; }
        for (int n = 0; n < N; n++) depth[n] = level[n];
    } else {
        int32_t *topo = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
        st = assign_depths(N, op, child, depth, topo, &err);
        free(topo);
        if (st != OR_OK) { info[4] = err; return st; }
    }

    int D = 0;
    for (int n = 0; n < N; n++) if (depth[n] > D) D = depth[n];
    int nkeys = 2 * (D + 1);
    /* bucket lists: count, then append in ascending id */
    int32_t *cnt = (int32_t *)calloc((size_t)nkeys + 1, sizeof(int32_t));
    for (int n = 0; n < N; n++) cnt[2 * depth[n] + op[n]]++;
    group_off[0] = 0;
    for (int k = 0; k < nkeys; k++) group_off[k + 1] = group_off[k] + cnt[k];
    int32_t *fill = (int32_t *)malloc(sizeof(int32_t) * ((size_t)nkeys + 1));
    for (int k = 0; k <= nkeys; k++) fill[k] = group_off[k];
    for (int n = 0; n < N; n++) perm[fill[2 * depth[n] + op[n]]++] = n;
    for (int r = 0; r < N; r++) rank[perm[r]] = r;
    for (int d = 0; d <= D + 1; d++) level_off[d] = group_off[2 * d];
    int n_leaves = 0;
    for (int n = 0; n < N; n++) n_leaves += (op[n] == OR_EMBED);
    int n_cells = N - n_leaves;

    for (int r = 0; r < N; r++) {
        int n = perm[r];
        for (int k = 0; k < 2; k++)
            gather[2 * r + k] = (op[n] == OR_CELL) ? rank[child[2 * n + k]] : -1;
    }
    /* consumer CSR */
    for (int r = 0; r <= N; r++) cons_off[r] = 0;
    for (int c = 0; c < n_cells; c++)
        for (int k = 0; k < 2; k++) cons_off[gather[2 * (n_leaves + c) + k] + 1]++;
    for (int r = 0; r < N; r++) cons_off[r + 1] += cons_off[r];
    int32_t *pos = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
    for (int r = 0; r < N; r++) pos[r] = cons_off[r];
    for (int e = 0; e < 2 * n_cells; e++) {   /* ascending e => ascending within a row */
        int r = gather[2 * n_leaves + e];
        cons_edge[pos[r]++] = e;
    }
    free(pos);
    /* leaves by (token, row): insertion into token buckets in ascending row order */
    int32_t *tcnt = (int32_t *)calloc((size_t)V + 1, sizeof(int32_t));
    for (int r = 0; r < n_leaves; r++) tcnt[token[perm[r]] + 1]++;
    for (int t = 0; t < V; t++) tcnt[t + 1] += tcnt[t];
    int nseg = 0;
    for (int t = 0; t < V; t++) if (tcnt[t + 1] > tcnt[t]) tok_seg[nseg++] = tcnt[t];
    tok_seg[nseg] = n_leaves;
    for (int r = 0; r < n_leaves; r++) leaf_perm[tcnt[token[perm[r]]]++] = r;
    free(tcnt);
    for (int g = 0; g < G; g++) root_row[g] = rank[root[g]];
    /* roots by (root_row, g): stable insertion sort (G is small in tests) */
    for (int g = 0; g < G; g++) {
        int j = g;
        while (j > 0 && root_row[root_perm[j - 1]] > root_row[g]) { root_perm[j] = root_perm[j - 1]; j--; }
        root_perm[j] = g;
    }
    free(cnt); free(fill);
    info[0] = D; info[1] = n_leaves; info[2] = n_cells; info[3] = nseg; info[4] = -1;
    return OR_OK;
}

/* ---------------------------------------------------------------- cell math */
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

/* z[j] = b[j] + sum_{k<S} U[j][k] hL[k] + sum_{k<S} U[j][S+k] hR[k], k ascending */
static void cell_z(int rows, int S, const double *U, const double *b,
                   const double *hL, const double *hR, double *z)
{
    for (int j = 0; j < rows; j++) {
        const double *u = U + (size_t)j * 2 * S;
        double acc = b[j];
        for (int k = 0; k < S; k++) acc += u[k] * hL[k];
        for (int k = 0; k < S; k++) acc += u[S + k] * hR[k];
        z[j] = acc;
    }
}

/* one node, given its children's (h, c); writes h, c and (optionally) the gate
 * activations act[gates*S] = (i, fL, fR, o, u) or (h) for TreeRNN */
static void cell_forward(int cell, int S, const double *U, const double *b,
                         const double *hL, const double *cL, const double *hR, const double *cR,
                         double *h, double *c, double *z, double *act)
{
    int gates = (cell == OR_TREELSTM) ? 5 : 1;
    cell_z(gates * S, S, U, b, hL, hR, z);
    if (cell == OR_TREERNN) {
        for (int j = 0; j < S; j++) { h[j] = tanh(z[j]); c[j] = 0.0; if (act) act[j] = h[j]; }
        return;
    }
    for (int j = 0; j < S; j++) {
        double i = sigm(z[j]), fl = sigm(z[S + j]), fr = sigm(z[2 * S + j]);
        double o = sigm(z[3 * S + j]), u = tanh(z[4 * S + j]);
        double cc = i * u + fl * cL[j] + fr * cR[j];
        c[j] = cc;
        h[j] = o * tanh(cc);
        if (act) { act[j] = i; act[S + j] = fl; act[2 * S + j] = fr; act[3 * S + j] = o; act[4 * S + j] = u; }
    }
}

/* post-order of all nodes (children first), assuming a validated acyclic input */
static int topo_order(int N, const int32_t *op, const int32_t *child, int32_t *topo)
{
    int32_t *depth = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
    int32_t err;
    int st = assign_depths(N, op, child, depth, topo, &err);
    free(depth);
    return st;
}

/* ---------------------------------------------------------------- forward
 * Evaluates every node individually in a topological order (each node exactly once,
 * a DAG node shared by several consumers is evaluated once). Outputs root h/c
 * [G][S]; optionally all node states H_all/C_all [N][S] (node-id order).
 */
int oracle_forward(int cell, int S, int N, int G, int V,
                   const int32_t *op, const int32_t *child, const int32_t *token, const int32_t *root,
                   const double *U, const double *b, const double *E,
                   double *h_root, double *c_root, double *H_all, double *C_all)
{
    if (S <= 0 || (cell != OR_TREERNN && cell != OR_TREELSTM)) return OR_E_INVALID;
    int32_t err;
    int st = validate(N, G, V, op, child, token, root, &err);
    if (st) return st;
    int gates = (cell == OR_TREELSTM) ? 5 : 1;
    double *H = H_all ? H_all : (double *)malloc(sizeof(double) * (size_t)N * S + 8);
    double *C = C_all ? C_all : (double *)malloc(sizeof(double) * (size_t)N * S + 8);
    double *z = (double *)malloc(sizeof(double) * (size_t)gates * S);
    int32_t *topo = (int32_t *)malloc(sizeof(int32_t) * ((size_t)N + 1));
    st = topo_order(N, op, child, topo);
    if (st == OR_OK) {
        for (int t = 0; t < N; t++) {
            int n = topo[t];
            double *h = H + (size_t)n * S, *c = C + (size_t)n * S;
            if (op[n] == OR_EMBED) {
                for (int j = 0; j < S; j++) { h[j] = E[(size_t)token[n] * S + j]; c[j] = 0.0; }
            } else {
                int L = child[2 * n], R = child[2 * n + 1];
                cell_forward(cell, S, U, b, H + (size_t)L * S, C + (size_t)L * S,
                             H + (size_t)R * S, C + (size_t)R * S, h, c, z, NULL);
            }
        }
        for (int g = 0; g < G; g++)
            for (int j = 0; j < S; j++) {
                if (h_root) h_root[(size_t)g * S + j] = H[(size_t)root[g] * S + j];
                if (c_root) c_root[(size_t)g * S + j] = C[(size_t)root[g] * S + j];
            }
    }
    free(z); free(topo);
    if (!H_all) free(H);
    if (!C_all) free(C);
    return st;
}

/* Level-ordered evaluation driven by this oracle's own schedule (each
 * loop iteration evaluates all operations at one depth, gathering from earlier
 * results). Row r of the pool holds node perm[r]. Outputs in node-id order. */
int oracle_forward_levels(int cell, int S, int N, int G, int V,
                          const int32_t *op, const int32_t *child, const int32_t *token,
                          const int32_t *root, const int32_t *level,
                          const double *U, const double *b, const double *E,
                          double *H_out, double *C_out)
{
    int32_t *depth = malloc(sizeof(int32_t) * (N + 1)), *perm = malloc(sizeof(int32_t) * (N + 1));
    int32_t *rank = malloc(sizeof(int32_t) * (N + 1)), *gat = malloc(sizeof(int32_t) * (2 * N + 2));
    int32_t *lo = malloc(sizeof(int32_t) * (N + 3)), *go = malloc(sizeof(int32_t) * (2 * N + 5));
    int32_t *co = malloc(sizeof(int32_t) * (N + 2)), *ce = malloc(sizeof(int32_t) * (2 * N + 2));
    int32_t *lp = malloc(sizeof(int32_t) * (N + 1)), *ts = malloc(sizeof(int32_t) * (N + 2));
    int32_t *rr = malloc(sizeof(int32_t) * (G + 1)), *rp = malloc(sizeof(int32_t) * (G + 1));
    int32_t info[5];
    int gates = (cell == OR_TREELSTM) ? 5 : 1;
    int st = oracle_schedule(N, G, V, op, child, token, root, level, depth, perm, rank, gat, lo, go,
                             co, ce, lp, ts, rr, rp, info);
    if (st == OR_OK) {
        int D = info[0];
        double *Hp = malloc(sizeof(double) * (size_t)N * S + 8), *Cp = malloc(sizeof(double) * (size_t)N * S + 8);
        double *z = malloc(sizeof(double) * (size_t)gates * S);
        for (int d = 1; d <= D; d++) {
            for (int r = lo[d]; r < lo[d + 1]; r++) {
                int n = perm[r];
                double *h = Hp + (size_t)r * S, *c = Cp + (size_t)r * S;
                if (op[n] == OR_EMBED) {
                    for (int j = 0; j < S; j++) { h[j] = E[(size_t)token[n] * S + j]; c[j] = 0.0; }
                } else {
                    int gl = gat[2 * r], gr = gat[2 * r + 1];
                    cell_forward(cell, S, U, b, Hp + (size_t)gl * S, Cp + (size_t)gl * S,
                                 Hp + (size_t)gr * S, Cp + (size_t)gr * S, h, c, z, NULL);
                }
            }
        }
        for (int n = 0; n < N; n++)
            for (int j = 0; j < S; j++) {
                H_out[(size_t)n * S + j] = Hp[(size_t)rank[n] * S + j];
                C_out[(size_t)n * S + j] = Cp[(size_t)rank[n] * S + j];
            }
        free(Hp); free(Cp); free(z);
    }
    free(depth); free(perm); free(rank); free(gat); free(lo); free(go); free(co); free(ce);
    free(lp); free(ts); free(rr); free(rp);
    return st;
}

/* ---------------------------------------------------------------- backward
 * Loss L = sum_g <dh_root[g], h_root(g)> + <dc_root[g], c_root(g)> (dc_root nullable;
 * SURVEY §8(c.8) #10). Reverse-mode over the reverse of the topological order, so
 * every consumer is processed before its children; a node's (dh, dc) is the sum over
 * its consumers and root seeds (DAG: several terms). Per CELL node:
 *   TreeLSTM: tc = tanh(c); do = dh*tc; dc += dh*o*(1-tc^2)
 *             dz_i = dc*u*i(1-i); dz_fL = dc*c_L*fL(1-fL); dz_fR = dc*c_R*fR(1-fR)
 *             dz_o = do*o(1-o);   dz_u  = dc*i*(1-u^2)
 *             dc_L += dc*fL; dc_R += dc*fR
 *   TreeRNN:  dz = dh*(1-h^2)
 *   both:     dU += dz (x) [h_L; h_R]; db += dz; dh_L += U_L^T dz; dh_R += U_R^T dz
 *   EMBED:    dE[token] += dh   (its c is the constant 0; dc is dropped)
 * Outputs dU [gates*S][2S], db [gates*S], dE [V][S] are overwritten (not accumulated).
 */
int oracle_backward(int cell, int S, int N, int G, int V,
                    const int32_t *op, const int32_t *child, const int32_t *token, const int32_t *root,
                    const double *U, const double *b, const double *E,
                    const double *dh_root, const double *dc_root,
                    double *dU, double *db, double *dE)
{
    if (S <= 0 || (cell != OR_TREERNN && cell != OR_TREELSTM)) return OR_E_INVALID;
    int32_t err;
    int st = validate(N, G, V, op, child, token, root, &err);
    if (st) return st;
    int gates = (cell == OR_TREELSTM) ? 5 : 1;
    size_t NS = (size_t)N * S;
    double *H = malloc(sizeof(double) * NS + 8), *C = malloc(sizeof(double) * NS + 8);
    double *A = malloc(sizeof(double) * (size_t)N * gates * S + 8);   /* gate activations */
    double *dH = calloc(NS + 1, sizeof(double)), *dC = calloc(NS + 1, sizeof(double));
    double *z = malloc(sizeof(double) * (size_t)gates * S), *dz = malloc(sizeof(double) * (size_t)gates * S);
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    st = topo_order(N, op, child, topo);
    if (st != OR_OK) goto done;
    /* forward, saving activations */
    for (int t = 0; t < N; t++) {
        int n = topo[t];
        double *h = H + (size_t)n * S, *c = C + (size_t)n * S;
        if (op[n] == OR_EMBED) {
            for (int j = 0; j < S; j++) { h[j] = E[(size_t)token[n] * S + j]; c[j] = 0.0; }
        } else {
            int L = child[2 * n], R = child[2 * n + 1];
            cell_forward(cell, S, U, b, H + (size_t)L * S, C + (size_t)L * S,
                         H + (size_t)R * S, C + (size_t)R * S, h, c, z, A + (size_t)n * gates * S);
        }
    }
    memset(dU, 0, sizeof(double) * (size_t)gates * S * 2 * S);
    memset(db, 0, sizeof(double) * (size_t)gates * S);
    memset(dE, 0, sizeof(double) * (size_t)V * S);
    for (int g = 0; g < G; g++)
        for (int j = 0; j < S; j++) {
            dH[(size_t)root[g] * S + j] += dh_root[(size_t)g * S + j];
            if (dc_root) dC[(size_t)root[g] * S + j] += dc_root[(size_t)g * S + j];
        }
    for (int t = N - 1; t >= 0; t--) {
        int n = topo[t];
        double *dh = dH + (size_t)n * S, *dc = dC + (size_t)n * S;
        if (op[n] == OR_EMBED) {
            for (int j = 0; j < S; j++) dE[(size_t)token[n] * S + j] += dh[j];
            continue;
        }
        int L = child[2 * n], R = child[2 * n + 1];
        const double *a = A + (size_t)n * gates * S, *c = C + (size_t)n * S;
        const double *hL = H + (size_t)L * S, *hR = H + (size_t)R * S;
        const double *cL = C + (size_t)L * S, *cR = C + (size_t)R * S;
        if (cell == OR_TREERNN) {
            for (int j = 0; j < S; j++) dz[j] = dh[j] * (1.0 - a[j] * a[j]);
        } else {
            for (int j = 0; j < S; j++) {
                double i = a[j], fl = a[S + j], fr = a[2 * S + j], o = a[3 * S + j], u = a[4 * S + j];
                double tc = tanh(c[j]);
                double dO = dh[j] * tc;
                double dcc = dc[j] + dh[j] * o * (1.0 - tc * tc);
                dz[j] = dcc * u * i * (1.0 - i);
                dz[S + j] = dcc * cL[j] * fl * (1.0 - fl);
                dz[2 * S + j] = dcc * cR[j] * fr * (1.0 - fr);
                dz[3 * S + j] = dO * o * (1.0 - o);
                dz[4 * S + j] = dcc * i * (1.0 - u * u);
                dC[(size_t)L * S + j] += dcc * fl;
                dC[(size_t)R * S + j] += dcc * fr;
            }
        }
        for (int r = 0; r < gates * S; r++) {
            double *du = dU + (size_t)r * 2 * S;
            for (int k = 0; k < S; k++) { du[k] += dz[r] * hL[k]; du[S + k] += dz[r] * hR[k]; }
            db[r] += dz[r];
        }
        double *dhL = dH + (size_t)L * S, *dhR = dH + (size_t)R * S;
        for (int r = 0; r < gates * S; r++) {
            const double *u = U + (size_t)r * 2 * S;
            for (int k = 0; k < S; k++) { dhL[k] += u[k] * dz[r]; dhR[k] += u[S + k] * dz[r]; }
        }
    }
done:
    free(H); free(C); free(A); free(dH); free(dC); free(z); free(dz); free(topo);
    return st;
}

/* ---------------------------------------------------------------- §3.5 model (NEXT-2)
 * The sentiment model of PAPER.md L297-304 (§3.5 "Recursive definitions"):
 *   h_word = TreeLSTM(Embedding(word), 0, 0)           (L300, leaves)
 *   h_{left,right} = TreeLSTM(0, h_left, h_right)       (L301, internal nodes)
 * with TreeLSTM = Tai et al. eqs 9-14, N = 2 (L304), and a per-node 5-way softmax
 * classifier with cross-entropy, "every node has a sentiment label" (L297).
 * Leaf (x = E[token], h_L = h_R = 0, c_L = c_R = 0; W = the input weights W^(i), W^(o),
 * W^(u) stacked as row blocks of W[3S][S]; the bias b is the cell's, blocks i, o, u):
 *   i = s(W_i x + b_i), o = s(W_o x + b_o), u = tanh(W_u x + b_u)
 *   c = i*u   (the forget-gate terms f_k * c_k vanish: c_k = 0, so W^(f) never matters)
 *   h = o*tanh(c)
 * Internal nodes: the x = 0 cell above (cell_forward, TreeLSTM).
 * Every node n: l = Ws h_n + bs (Ws[C][S], bs[C]), p = softmax(l),
 *   loss_n = log(sum_k exp(l_k)) - l[label[n]];   L = sum over all nodes of loss_n.
 */
static void leaf_forward(int S, const double *W, const double *b, const double *x, double *h, double *c, double *act)
{
    for (int j = 0; j < S; j++) {
        double zi = b[j], zo = b[3 * S + j], zu = b[4 * S + j];
        const double *wi = W + (size_t)j * S, *wo = W + (size_t)(S + j) * S, *wu = W + (size_t)(2 * S + j) * S;
        for (int k = 0; k < S; k++) { zi += wi[k] * x[k]; zo += wo[k] * x[k]; zu += wu[k] * x[k]; }
        double i = sigm(zi), o = sigm(zo), u = tanh(zu);
        c[j] = i * u;
        h[j] = o * tanh(c[j]);
        if (act) { act[j] = i; act[S + j] = o; act[2 * S + j] = u; }
    }
}

/* log-softmax cross-entropy of one node: returns loss_n, writes dl = p - e_y */
static double node_ce(int S, int C, const double *Ws, const double *bs, const double *h, int y, double *dl)
{
    double mx = -INFINITY;
    for (int k = 0; k < C; k++) {
        double l = bs[k];
        for (int j = 0; j < S; j++) l += Ws[(size_t)k * S + j] * h[j];
        dl[k] = l;
        if (l > mx) mx = l;
    }
    double se = 0.0;
    for (int k = 0; k < C; k++) se += exp(dl[k] - mx);
    double lse = mx + log(se);
    double loss = lse - dl[y];
    for (int k = 0; k < C; k++) dl[k] = exp(dl[k] - lse) - (k == y ? 1.0 : 0.0);
    return loss;
}

static int sst_eval(int S, int N, const int32_t *op, const int32_t *child, const int32_t *token,
                    const double *U, const double *b, const double *E, const double *W,
                    double *H, double *Cs, double *A, double *AL, int32_t *topo)
{
    int st = topo_order(N, op, child, topo);
    if (st != OR_OK) return st;
    double *z = malloc(sizeof(double) * 5 * (size_t)S);
    for (int t = 0; t < N; t++) {
        int n = topo[t];
        double *h = H + (size_t)n * S, *c = Cs + (size_t)n * S;
        if (op[n] == OR_EMBED) {
            leaf_forward(S, W, b, E + (size_t)token[n] * S, h, c, AL ? AL + (size_t)n * 3 * S : NULL);
        } else {
            int L = child[2 * n], R = child[2 * n + 1];
            cell_forward(OR_TREELSTM, S, U, b, H + (size_t)L * S, Cs + (size_t)L * S, H + (size_t)R * S,
                         Cs + (size_t)R * S, h, c, z, A ? A + (size_t)n * 5 * S : NULL);
        }
    }
    free(z);
    return OR_OK;
}

/* Forward of the §3.5 model: total loss, optionally every node's h / c (node-id order). */
int oracle_sst_forward(int S, int N, int V, int C, const int32_t *op, const int32_t *child, const int32_t *token,
                       const int32_t *label, const double *U, const double *b, const double *E, const double *W,
                       const double *Ws, const double *bs, double *loss, double *H_all, double *C_all)
{
    if (S <= 0 || C <= 0) return OR_E_INVALID;
    int32_t err;
    int32_t root0 = 0;
    int st = validate(N, 0, V, op, child, token, &root0, &err);
    if (st) return st;
    for (int n = 0; n < N; n++)
        if (label[n] < 0 || label[n] >= C) return OR_E_INVALID;
    double *H = H_all ? H_all : malloc(sizeof(double) * (size_t)N * S + 8);
    double *Cs = C_all ? C_all : malloc(sizeof(double) * (size_t)N * S + 8);
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    double *dl = malloc(sizeof(double) * (size_t)C);
    st = sst_eval(S, N, op, child, token, U, b, E, W, H, Cs, NULL, NULL, topo);
    if (st == OR_OK) {
        double L = 0.0;
        for (int n = 0; n < N; n++) L += node_ce(S, C, Ws, bs, H + (size_t)n * S, label[n], dl);
        *loss = L;
    }
    free(topo); free(dl);
    if (!H_all) free(H);
    if (!C_all) free(Cs);
    return st;
}

/* Reverse mode of the §3.5 loss (hand-derived; pinned by finite differences in tests/):
 * every node first gets its classifier's dh += Ws^T (p - e_y), dWs += (p - e_y) (x) h,
 * dbs += p - e_y; then nodes in reverse topological order: cells as oracle_backward;
 * leaves: tc = tanh(c); do = dh*tc; dc' = dc + dh*o*(1-tc^2);
 *   dz_i = dc'*u*i(1-i), dz_o = do*o(1-o), dz_u = dc'*i*(1-u^2);
 *   dW_g += dz_g (x) x, db[block g] += dz_g (g in i, o, u), dE[token] += sum_g W_g^T dz_g.
 * All outputs overwritten. */
int oracle_sst_backward(int S, int N, int V, int C, const int32_t *op, const int32_t *child, const int32_t *token,
                        const int32_t *label, const double *U, const double *b, const double *E, const double *W,
                        const double *Ws, const double *bs, double *loss, double *dU, double *db, double *dE,
                        double *dW, double *dWs, double *dbs)
{
    if (S <= 0 || C <= 0) return OR_E_INVALID;
    int32_t err, root0 = 0;
    int st = validate(N, 0, V, op, child, token, &root0, &err);
    if (st) return st;
    for (int n = 0; n < N; n++)
        if (label[n] < 0 || label[n] >= C) return OR_E_INVALID;
    size_t NS = (size_t)N * S;
    double *H = malloc(sizeof(double) * NS + 8), *Cs = malloc(sizeof(double) * NS + 8);
    double *A = malloc(sizeof(double) * NS * 5 + 8), *AL = malloc(sizeof(double) * NS * 3 + 8);
    double *dH = calloc(NS + 1, sizeof(double)), *dC = calloc(NS + 1, sizeof(double));
    double *dz = malloc(sizeof(double) * 5 * (size_t)S), *dl = malloc(sizeof(double) * (size_t)C);
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    st = sst_eval(S, N, op, child, token, U, b, E, W, H, Cs, A, AL, topo);
    if (st != OR_OK) goto done;
    memset(dU, 0, sizeof(double) * (size_t)5 * S * 2 * S);
    memset(db, 0, sizeof(double) * (size_t)5 * S);
    memset(dE, 0, sizeof(double) * (size_t)V * S);
    memset(dW, 0, sizeof(double) * (size_t)3 * S * S);
    memset(dWs, 0, sizeof(double) * (size_t)C * S);
    memset(dbs, 0, sizeof(double) * (size_t)C);
    double L = 0.0;
    for (int n = 0; n < N; n++) {
        const double *h = H + (size_t)n * S;
        L += node_ce(S, C, Ws, bs, h, label[n], dl);
        for (int k = 0; k < C; k++) {
            dbs[k] += dl[k];
            for (int j = 0; j < S; j++) {
                dWs[(size_t)k * S + j] += dl[k] * h[j];
                dH[(size_t)n * S + j] += Ws[(size_t)k * S + j] * dl[k];
            }
        }
    }
    *loss = L;
    for (int t = N - 1; t >= 0; t--) {
        int n = topo[t];
        double *dh = dH + (size_t)n * S, *dc = dC + (size_t)n * S;
        const double *c = Cs + (size_t)n * S;
        if (op[n] == OR_EMBED) {
            const double *a = AL + (size_t)n * 3 * S, *x = E + (size_t)token[n] * S;
            for (int j = 0; j < S; j++) {
                double i = a[j], o = a[S + j], u = a[2 * S + j];
                double tc = tanh(c[j]);
                double dO = dh[j] * tc;
                double dcc = dc[j] + dh[j] * o * (1.0 - tc * tc);
                dz[j] = dcc * u * i * (1.0 - i);
                dz[S + j] = dO * o * (1.0 - o);
                dz[2 * S + j] = dcc * i * (1.0 - u * u);
            }
            const int blk[3] = {0, 3, 4};  /* bias blocks of i, o, u */
            double *de = dE + (size_t)token[n] * S;
            for (int g = 0; g < 3; g++)
                for (int j = 0; j < S; j++) {
                    double d = dz[g * S + j];
                    const double *w = W + (size_t)(g * S + j) * S;
                    double *dw = dW + (size_t)(g * S + j) * S;
                    db[blk[g] * S + j] += d;
                    for (int k = 0; k < S; k++) { dw[k] += d * x[k]; de[k] += w[k] * d; }
                }
            continue;
        }
        int Lc = child[2 * n], R = child[2 * n + 1];
        const double *a = A + (size_t)n * 5 * S;
        const double *hL = H + (size_t)Lc * S, *hR = H + (size_t)R * S;
        const double *cL = Cs + (size_t)Lc * S, *cR = Cs + (size_t)R * S;
        for (int j = 0; j < S; j++) {
            double i = a[j], fl = a[S + j], fr = a[2 * S + j], o = a[3 * S + j], u = a[4 * S + j];
            double tc = tanh(c[j]);
            double dO = dh[j] * tc;
            double dcc = dc[j] + dh[j] * o * (1.0 - tc * tc);
            dz[j] = dcc * u * i * (1.0 - i);
            dz[S + j] = dcc * cL[j] * fl * (1.0 - fl);
            dz[2 * S + j] = dcc * cR[j] * fr * (1.0 - fr);
            dz[3 * S + j] = dO * o * (1.0 - o);
            dz[4 * S + j] = dcc * i * (1.0 - u * u);
            dC[(size_t)Lc * S + j] += dcc * fl;
            dC[(size_t)R * S + j] += dcc * fr;
        }
        for (int r = 0; r < 5 * S; r++) {
            double *du = dU + (size_t)r * 2 * S;
            for (int k = 0; k < S; k++) { du[k] += dz[r] * hL[k]; du[S + k] += dz[r] * hR[k]; }
            db[r] += dz[r];
        }
        double *dhL = dH + (size_t)Lc * S, *dhR = dH + (size_t)R * S;
        for (int r = 0; r < 5 * S; r++) {
            const double *u = U + (size_t)r * 2 * S;
            for (int k = 0; k < S; k++) { dhL[k] += u[k] * dz[r]; dhR[k] += u[S + k] * dz[r]; }
        }
    }
done:
    free(H); free(Cs); free(A); free(AL); free(dH); free(dC); free(dz); free(dl); free(topo);
    return st;
}
