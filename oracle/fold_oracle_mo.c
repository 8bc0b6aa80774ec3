/*
 * oracle/fold_oracle_mo.c — fp64 CPU ORACLE for MULTI-OP dynamic batching (SURVEY §8(f)
 * NEXT-3: several operations and tensor types per depth).
 *
 * TEST INFRASTRUCTURE ONLY (see fold_oracle.c's header: only tests/, smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it; it includes nothing from the product).
 *
 * The method (§2):
 *   L31 "We distinguish between individual operations ... dynamic batching schedules
 *       operations ... it enumerates them for scheduling purposes."
 *   L33 "The inputs and outputs of operations have tensor types ... fixed and fully
 *       specified in advance"
 *   L40 depth: constants depth 0; a node's depth = 1 + max depth of its dependencies.
 *   L42 "Batch together all nodes invoking the same operation at the same depth"
 *   L43 "Concatenate all outputs which have the same depth and tensor type. The order of
 *       concatenation corresponds to the order in which the dynamic batching operations
 *       were enumerated."
 *   L44 "Assign a label (d, t, i) to each edge ... d is the depth, t is the tensor type,
 *       and i is the integer index for that edge into the (concatenated) outputs for d, t."
 *
 * Model (reading R30): an op table of n_ops operations in enumeration order
 * (op id = position), each {kind, arity, in_type, out_type, vocab}; tensor types t carry
 * (h, c) in R^{S_t} (c = 0 for ops without a memory cell).
 *   MO_EMBED (arity 0):   h = E_o[token], c = 0                        (Fig. 1 "embed lookup")
 *   MO_LSTM  (arity a):   N-ary TreeLSTM with x = 0 (Tai et al. eqs 9-14 as cited at
 *                         PAPER.md L301-304, N = a): row blocks of U_o[(3+a)S][aS] are
 *                         (i, f_1..f_a, o, u), column block k multiplies child k's h:
 *                         z = U_o [h_1; ..; h_a] + b_o, i = s(z_i), f_k = s(z_fk),
 *                         o = s(z_o), u = tanh(z_u), c = i u + sum_k f_k c_k, h = o tanh(c)
 *                         (in_type = out_type: the cell state passes through f_k)
 *   MO_RNN   (arity a):   h = tanh(U_o [h_1; ..; h_a] + b_o), c = 0, U_o[S_out][a S_in]
 *                         (Fig. 1 "RNN Cell"; with in_type != out_type a typed projection)
 * Parameters: one flat fp64 array, op o's block at poff[o] (mo_param_offsets): EMBED E_o
 * [V_o][S]; LSTM / RNN U_o then b_o. Gradients use the same layout.
 * Loss for the backward: L = sum_g <g_g, h_root(g)>, g stored as [G][S_max] (graph g uses
 * the first S_{type(root g)} entries).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { MO_OK = 0, MO_E_INVALID = 1, MO_E_CHILD_RANGE = 2, MO_E_ARITY = 3, MO_E_TOKEN_RANGE = 4,
       MO_E_ROOT_RANGE = 5, MO_E_CYCLE = 6, MO_E_OP_RANGE = 10, MO_E_TYPE = 11 };
enum { MO_EMBED = 0, MO_LSTM = 1, MO_RNN = 2 };
#define MO_MAXA 2

typedef struct {
    int n_ops, n_types;
    const int32_t *kind, *arity, *in_type, *out_type, *vocab;  /* [n_ops] */
    const int32_t *S;                                          /* [n_types] */
} mo_table;

static int rows_of(const mo_table *T, int o)    /* output rows of U_o */
{
    int S = T->S[T->out_type[o]];
    return T->kind[o] == MO_LSTM ? (3 + T->arity[o]) * S : S;
}
static int kin_of(const mo_table *T, int o) { return T->arity[o] * T->S[T->in_type[o]]; }

/* parameter block offsets poff[0..n_ops] (doubles / floats) */
int64_t mo_param_offsets(int n_ops, int n_types, const int32_t *kind, const int32_t *arity,
                         const int32_t *in_type, const int32_t *out_type, const int32_t *vocab,
                         const int32_t *S, int64_t *poff)
{
    mo_table T = {n_ops, n_types, kind, arity, in_type, out_type, vocab, S};
    int64_t off = 0;
    for (int o = 0; o < n_ops; o++) {
        poff[o] = off;
        if (kind[o] == MO_EMBED) off += (int64_t)vocab[o] * S[out_type[o]];
        else off += (int64_t)rows_of(&T, o) * kin_of(&T, o) + rows_of(&T, o);
    }
    poff[n_ops] = off;
    return off;
}

/* op table well-formed: kinds, arities, types in range, LSTM in == out, vocab > 0 */
static int table_ok(const mo_table *T)
{
    if (T->n_ops <= 0 || T->n_types <= 0) return 0;
    for (int t = 0; t < T->n_types; t++) if (T->S[t] <= 0) return 0;
    for (int o = 0; o < T->n_ops; o++) {
        int k = T->kind[o], a = T->arity[o];
        if (T->out_type[o] < 0 || T->out_type[o] >= T->n_types) return 0;
        if (k == MO_EMBED) { if (a != 0 || T->vocab[o] <= 0) return 0; continue; }
        if (k != MO_LSTM && k != MO_RNN) return 0;
        if (a < 1 || a > MO_MAXA) return 0;
        if (T->in_type[o] < 0 || T->in_type[o] >= T->n_types) return 0;
        if (k == MO_LSTM && T->in_type[o] != T->out_type[o]) return 0;
    }
    return 1;
}

/* Error classes in this order, smallest offending node id (graph id for ROOT_RANGE):
 * CHILD_RANGE (a slot outside [-1, N)), OP_RANGE, ARITY (slots [0, a) set, the rest -1),
 * TYPE (child's output type != the op's input type), TOKEN_RANGE, ROOT_RANGE. */
static int mo_validate(const mo_table *T, int N, int G, const int32_t *op, const int32_t *child,
                       const int32_t *token, const int32_t *root, int32_t *err)
{
    for (int n = 0; n < N; n++)
        for (int k = 0; k < MO_MAXA; k++)
            if (child[MO_MAXA * n + k] < -1 || child[MO_MAXA * n + k] >= N) { *err = n; return MO_E_CHILD_RANGE; }
    for (int n = 0; n < N; n++)
        if (op[n] < 0 || op[n] >= T->n_ops) { *err = n; return MO_E_OP_RANGE; }
    for (int n = 0; n < N; n++) {
        int a = T->arity[op[n]], ok = 1;
        for (int k = 0; k < MO_MAXA; k++) ok &= (k < a) ? child[MO_MAXA * n + k] >= 0 : child[MO_MAXA * n + k] == -1;
        if (!ok) { *err = n; return MO_E_ARITY; }
    }
    for (int n = 0; n < N; n++) {
        int o = op[n];
        for (int k = 0; k < T->arity[o]; k++)
            if (T->out_type[op[child[MO_MAXA * n + k]]] != T->in_type[o]) { *err = n; return MO_E_TYPE; }
    }
    for (int n = 0; n < N; n++)
        if (T->kind[op[n]] == MO_EMBED && (token[n] < 0 || token[n] >= T->vocab[op[n]])) { *err = n; return MO_E_TOKEN_RANGE; }
    for (int g = 0; g < G; g++)
        if (root[g] < 0 || root[g] >= N) { *err = g; return MO_E_ROOT_RANGE; }
    return MO_OK;
}

/* depth by PAPER.md L40 (EMBED: its token constant is the depth-0 dependency => 1; other
 * ops 1 + max over children), memoised DFS; also a post-order `topo`. Cycle: the smallest
 * id of a node that reaches a cycle. */
static int mo_depths(const mo_table *T, int N, const int32_t *op, const int32_t *child,
                     int32_t *depth, int32_t *topo, int32_t *err)
{
    enum { WHITE = 0, GREY = 1, DONE = 2, BAD = 3 };
    unsigned char *col = calloc((size_t)N + 1, 1);
    int32_t *stk = malloc(sizeof(int32_t) * ((size_t)N + 1)), *nxt = malloc(sizeof(int32_t) * ((size_t)N + 1));
    int nt = 0, any_bad = 0;
    for (int s = 0; s < N; s++) {
        if (col[s] != WHITE) continue;
        int sp = 0;
        stk[sp++] = s; col[s] = GREY; nxt[s] = 0;
        while (sp > 0) {
            int n = stk[sp - 1], a = T->arity[op[n]];
            if (nxt[n] < a) {
                int c = child[MO_MAXA * n + nxt[n]++];
                if (col[c] == WHITE) { col[c] = GREY; nxt[c] = 0; stk[sp++] = c; }
                continue;
            }
            int bad = 0, dmax = 0;
            for (int k = 0; k < a; k++) {
                int c = child[MO_MAXA * n + k];
                if (col[c] == GREY || col[c] == BAD) bad = 1;
                else if (depth[c] > dmax) dmax = depth[c];
            }
            if (bad) { col[n] = BAD; depth[n] = -1; any_bad = 1; }
            else { col[n] = DONE; depth[n] = 1 + dmax; topo[nt++] = n; }  /* EMBED: 1 + 0 */
            sp--;
        }
    }
    int st = MO_OK;
    if (any_bad) { for (int n = 0; n < N; n++) if (col[n] == BAD) { *err = n; break; } st = MO_E_CYCLE; }
    free(col); free(stk); free(nxt);
    return st;
}

/* ---------------------------------------------------------------- schedule
 * Outputs (caller-allocated):
 *   depth[N]
 *   group_off[(D+1)*n_ops + 1]: rows with key < k, key = depth*n_ops + op (the batched
 *        operation instances of L42, in depth then enumeration order)
 *   type_off[n_types + 1]: first row of each tensor type's pool in `pool`
 *   pool[N]: for t ascending, the nodes of output type t ordered by (depth, op, id): the
 *        L43 concatenation of all outputs of one (depth, type), concatenated over depths
 *   pool_row[N]: a node's row within its own type's pool (pool[type_off[t] + row] = n)
 *   tlevel_off[n_types*(D+2)]: per type t, tlevel_off[t*(D+2) + d] = rows of type t with
 *        depth < d (d = 0..D+1): the (d, t) block of the concatenation starts there
 *   label[N*MO_MAXA*3]: edge (n, k) -> (d, t, i) of its child (L44); -1 for unused slots.
 *        i = pool_row(child) - tlevel_off[t*(D+2) + d]
 *   info[0..1] = D, err node
 * Caller sizes group_off / tlevel_off for D <= N.
 */
int oracle_mo_schedule(int n_ops, int n_types, const int32_t *kind, const int32_t *arity,
                       const int32_t *in_type, const int32_t *out_type, const int32_t *vocab,
                       const int32_t *S, int N, int G, const int32_t *op, const int32_t *child,
                       const int32_t *token, const int32_t *root, int32_t *depth, int32_t *group_off,
                       int32_t *type_off, int32_t *pool, int32_t *pool_row, int32_t *tlevel_off,
                       int32_t *label, int32_t *info)
{
    mo_table T = {n_ops, n_types, kind, arity, in_type, out_type, vocab, S};
    int32_t err = -1;
    info[0] = 0; info[1] = -1;
    if (N < 0 || G < 0 || !table_ok(&T)) return MO_E_INVALID;
    int st = mo_validate(&T, N, G, op, child, token, root, &err);
    if (st) { info[1] = err; return st; }
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    st = mo_depths(&T, N, op, child, depth, topo, &err);
    free(topo);
    if (st) { info[1] = err; return st; }
    int D = 0;
    for (int n = 0; n < N; n++) if (depth[n] > D) D = depth[n];
    int nkeys = (D + 1) * n_ops;
    for (int k = 0; k <= nkeys; k++) group_off[k] = 0;
    for (int n = 0; n < N; n++) group_off[depth[n] * n_ops + op[n] + 1]++;
    for (int k = 0; k < nkeys; k++) group_off[k + 1] += group_off[k];
    /* type pools: count, then for t, d, op, n ascending append */
    type_off[0] = 0;
    for (int t = 0; t < n_types; t++) {
        int c = 0;
        for (int n = 0; n < N; n++) c += out_type[op[n]] == t;
        type_off[t + 1] = type_off[t] + c;
    }
    for (int t = 0; t < n_types; t++) {
        int r = 0;
        for (int d = 0; d <= D + 1; d++) {
            tlevel_off[t * (D + 2) + d] = r;
            if (d > D) break;
            for (int o = 0; o < n_ops; o++) {
                if (out_type[o] != t) continue;
                for (int n = 0; n < N; n++)
                    if (depth[n] == d && op[n] == o) { pool[type_off[t] + r] = n; pool_row[n] = r; r++; }
            }
        }
    }
    for (int n = 0; n < N; n++)
        for (int k = 0; k < MO_MAXA; k++) {
            int32_t *l = label + ((size_t)n * MO_MAXA + k) * 3;
            int c = child[MO_MAXA * n + k];
            if (c < 0) { l[0] = l[1] = l[2] = -1; continue; }
            int t = out_type[op[c]];
            l[0] = depth[c]; l[1] = t; l[2] = pool_row[c] - tlevel_off[t * (D + 2) + depth[c]];
        }
    info[0] = D;
    return MO_OK;
}

/* ---------------------------------------------------------------- one node */
static double sigm(double x) { return 1.0 / (1.0 + exp(-x)); }

/* x = [h_1; ..; h_a] (a S_in), z = U x + b (rows), k ascending */
static void mo_z(int rows, int kin, const double *U, const double *b, const double *x, double *z)
{
    for (int j = 0; j < rows; j++) {
        const double *u = U + (size_t)j * kin;
        double acc = b[j];
        for (int k = 0; k < kin; k++) acc += u[k] * x[k];
        z[j] = acc;
    }
}

/* node n's (h, c) from its children's rows of H / C (stride Smax); act = gate activations
 * (LSTM: i, f_1..f_a, o, u; RNN: h) for the backward */
static void mo_node(const mo_table *T, int Smax, const double *P, const int64_t *poff, int o, int tok,
                    const int32_t *ch, const double *H, const double *C, double *h, double *c, double *x,
                    double *z, double *act)
{
    int S = T->S[T->out_type[o]];
    if (T->kind[o] == MO_EMBED) {
        const double *E = P + poff[o];
        for (int j = 0; j < S; j++) { h[j] = E[(size_t)tok * S + j]; c[j] = 0.0; }
        return;
    }
    int a = T->arity[o], Sin = T->S[T->in_type[o]], rows = rows_of(T, o), kin = a * Sin;
    const double *U = P + poff[o], *b = U + (size_t)rows * kin;
    for (int k = 0; k < a; k++)
        for (int j = 0; j < Sin; j++) x[k * Sin + j] = H[(size_t)ch[k] * Smax + j];
    mo_z(rows, kin, U, b, x, z);
    if (T->kind[o] == MO_RNN) {
        for (int j = 0; j < S; j++) { h[j] = tanh(z[j]); c[j] = 0.0; if (act) act[j] = h[j]; }
        return;
    }
    for (int j = 0; j < S; j++) {
        double i = sigm(z[j]), og = sigm(z[(1 + a) * S + j]), u = tanh(z[(2 + a) * S + j]);
        double cc = i * u;
        for (int k = 0; k < a; k++) {
            double f = sigm(z[(1 + k) * S + j]);
            cc += f * C[(size_t)ch[k] * Smax + j];
            if (act) act[(1 + k) * S + j] = f;
        }
        c[j] = cc;
        h[j] = og * tanh(cc);
        if (act) { act[j] = i; act[(1 + a) * S + j] = og; act[(2 + a) * S + j] = u; }
    }
}

static int mo_prepare(const mo_table *T, int N, int G, const int32_t *op, const int32_t *child,
                      const int32_t *token, const int32_t *root, int32_t *topo)
{
    int32_t err;
    if (N < 0 || G < 0 || !table_ok(T)) return MO_E_INVALID;
    int st = mo_validate(T, N, G, op, child, token, root, &err);
    if (st) return st;
    int32_t *depth = malloc(sizeof(int32_t) * ((size_t)N + 1));
    st = mo_depths(T, N, op, child, depth, topo, &err);
    free(depth);
    return st;
}

static int smax_of(const mo_table *T)
{
    int m = 0;
    for (int t = 0; t < T->n_types; t++) if (T->S[t] > m) m = T->S[t];
    return m;
}

static int rows_max(const mo_table *T)
{
    int m = 0;
    for (int o = 0; o < T->n_ops; o++) if (T->kind[o] != MO_EMBED && rows_of(T, o) > m) m = rows_of(T, o);
    return m > 0 ? m : 1;
}

/* ---------------------------------------------------------------- forward
 * Every node individually in a topological order (batching reaches the
 * node-at-a-time result). H_all / C_all [N][S_max] in node-id order (a node of type t fills
 * its first S_t entries, the rest 0).
 */
int oracle_mo_forward(int n_ops, int n_types, const int32_t *kind, const int32_t *arity,
                      const int32_t *in_type, const int32_t *out_type, const int32_t *vocab, const int32_t *S,
                      int N, int G, const int32_t *op, const int32_t *child, const int32_t *token,
                      const int32_t *root, const double *P, double *H_all, double *C_all)
{
    mo_table T = {n_ops, n_types, kind, arity, in_type, out_type, vocab, S};
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    int st = mo_prepare(&T, N, G, op, child, token, root, topo);
    if (st == MO_OK) {
        int64_t poff[17];
        mo_param_offsets(n_ops, n_types, kind, arity, in_type, out_type, vocab, S, poff);
        int Sm = smax_of(&T), RM = rows_max(&T);
        double *x = malloc(sizeof(double) * (size_t)MO_MAXA * Sm), *z = malloc(sizeof(double) * (size_t)RM);
        memset(H_all, 0, sizeof(double) * (size_t)N * Sm);
        memset(C_all, 0, sizeof(double) * (size_t)N * Sm);
        for (int t = 0; t < N; t++) {
            int n = topo[t];
            mo_node(&T, Sm, P, poff, op[n], token[n], child + MO_MAXA * n, H_all, C_all,
                    H_all + (size_t)n * Sm, C_all + (size_t)n * Sm, x, z, NULL);
        }
        free(x); free(z);
    }
    free(topo);
    return st;
}

/* ---------------------------------------------------------------- backward
 * L = sum_g <g_g, h_root(g)>. Reverse of the topological order (consumers before their
 * children; a shared node's (dh, dc) sums all its consumers). Per node of op o:
 *   EMBED: dE_o[token] += dh
 *   RNN:   dz = dh (1 - h^2)
 *   LSTM:  tc = tanh(c); dc' = dc + dh o (1 - tc^2); dz_i = dc' u i(1-i);
 *          dz_fk = dc' c_k f_k(1-f_k); dz_o = dh tc o(1-o); dz_u = dc' i (1-u^2);
 *          dc_k += dc' f_k
 *   both:  dU_o += dz (x) x, db_o += dz, dh_k += U_o[:, block k]^T dz
 * dP is overwritten (same layout as P).
 */
int oracle_mo_backward(int n_ops, int n_types, const int32_t *kind, const int32_t *arity,
                       const int32_t *in_type, const int32_t *out_type, const int32_t *vocab, const int32_t *S,
                       int N, int G, const int32_t *op, const int32_t *child, const int32_t *token,
                       const int32_t *root, const double *P, const double *g, double *dP)
{
    mo_table T = {n_ops, n_types, kind, arity, in_type, out_type, vocab, S};
    int32_t *topo = malloc(sizeof(int32_t) * ((size_t)N + 1));
    int st = mo_prepare(&T, N, G, op, child, token, root, topo);
    if (st != MO_OK) { free(topo); return st; }
    int64_t poff[17];
    int64_t np = mo_param_offsets(n_ops, n_types, kind, arity, in_type, out_type, vocab, S, poff);
    int Sm = smax_of(&T), RM = rows_max(&T);
    size_t NS = (size_t)N * Sm;
    double *H = calloc(NS + 1, sizeof(double)), *C = calloc(NS + 1, sizeof(double));
    double *A = calloc((size_t)N * RM + 1, sizeof(double));
    double *dH = calloc(NS + 1, sizeof(double)), *dC = calloc(NS + 1, sizeof(double));
    double *x = malloc(sizeof(double) * (size_t)MO_MAXA * Sm), *z = malloc(sizeof(double) * (size_t)RM);
    double *dz = malloc(sizeof(double) * (size_t)RM);
    for (int t = 0; t < N; t++) {
        int n = topo[t];
        mo_node(&T, Sm, P, poff, op[n], token[n], child + MO_MAXA * n, H, C, H + (size_t)n * Sm,
                C + (size_t)n * Sm, x, z, A + (size_t)n * RM);
    }
    memset(dP, 0, sizeof(double) * (size_t)np);
    for (int gi = 0; gi < G; gi++) {
        int r = root[gi], Sr = S[out_type[op[r]]];
        for (int j = 0; j < Sr; j++) dH[(size_t)r * Sm + j] += g[(size_t)gi * Sm + j];
    }
    for (int t = N - 1; t >= 0; t--) {
        int n = topo[t], o = op[n], So = S[out_type[o]];
        const double *dh = dH + (size_t)n * Sm, *dc = dC + (size_t)n * Sm;
        if (kind[o] == MO_EMBED) {
            double *dE = dP + poff[o];
            for (int j = 0; j < So; j++) dE[(size_t)token[n] * So + j] += dh[j];
            continue;
        }
        int a = arity[o], Sin = S[in_type[o]], rows = rows_of(&T, o), kin = a * Sin;
        const int32_t *ch = child + MO_MAXA * n;
        const double *act = A + (size_t)n * RM;
        if (kind[o] == MO_RNN) {
            for (int j = 0; j < So; j++) dz[j] = dh[j] * (1.0 - act[j] * act[j]);
        } else {
            const double *c = C + (size_t)n * Sm;
            for (int j = 0; j < So; j++) {
                double i = act[j], og = act[(1 + a) * So + j], u = act[(2 + a) * So + j];
                double tc = tanh(c[j]);
                double dcc = dc[j] + dh[j] * og * (1.0 - tc * tc);
                dz[j] = dcc * u * i * (1.0 - i);
                for (int k = 0; k < a; k++) {
                    double f = act[(1 + k) * So + j];
                    dz[(1 + k) * So + j] = dcc * C[(size_t)ch[k] * Sm + j] * f * (1.0 - f);
                    dC[(size_t)ch[k] * Sm + j] += dcc * f;
                }
                dz[(1 + a) * So + j] = dh[j] * tc * og * (1.0 - og);
                dz[(2 + a) * So + j] = dcc * i * (1.0 - u * u);
            }
        }
        for (int k = 0; k < a; k++)
            for (int j = 0; j < Sin; j++) x[k * Sin + j] = H[(size_t)ch[k] * Sm + j];
        const double *U = P + poff[o];
        double *dU = dP + poff[o], *db = dU + (size_t)rows * kin;
        for (int r = 0; r < rows; r++) {
            double *du = dU + (size_t)r * kin;
            for (int k = 0; k < kin; k++) du[k] += dz[r] * x[k];
            db[r] += dz[r];
        }
        for (int k = 0; k < a; k++) {
            double *dhk = dH + (size_t)ch[k] * Sm;
            for (int r = 0; r < rows; r++) {
                const double *u = U + (size_t)r * kin + (size_t)k * Sin;
                for (int j = 0; j < Sin; j++) dhk[j] += u[j] * dz[r];
            }
        }
    }
    free(H); free(C); free(A); free(dH); free(dC); free(x); free(z); free(dz); free(topo);
    return MO_OK;
}
