/*
 * kitc_oracle.c -- CPU ORACLE for the barycentric Lagrange KITC (arXiv:1902.02250).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_1902_02250_b200/) never links, imports or calls it, and shares no code,
 * header, table or constant generator with it.
 *
 * Plain, slow, single-threaded C99, compiled with -O2 -ffp-contract=off.  Pair
 * terms in double, per-target accumulators in long double.
 * Every function cites the PAPER.md passage (P:<line>) it follows; where the
 * paper is silent or garbled the reading is named (A1..A18 = DESIGN.md
 * "Readings of the paper").
 *
 * Pinned by tests/test_oracle_*.py (-m "not gpu") against closed forms,
 * invariants and brute force -- see DESIGN.md "Oracle pins" (including the
 * separate-target functions, test_oracle_targets.py, and the size-check
 * variant, test_oracle_sizecheck.py).
 */
#include <float.h>
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846
/* A7: the paper's tolerance "DBL_MIN = 2.22507e-308". */
#define ORC_TOL DBL_MIN
/* A2/A3: split iff side > lmax/sqrt(2); 1/sqrt(2) rounded to nearest. */
#define ORC_INV_SQRT2 0.7071067811865476

enum { ORC_STOKESLET = 0, ORC_ROTLET = 1, ORC_STOKESLET_ROTLET = 2, ORC_POLY = 99 };

/* ------------------------------------------------------------------------- */
/* L0: interpolation math (§3)                                        */
/* ------------------------------------------------------------------------- */

/* Chebyshev points of the 2nd kind, s_k = cos(k pi / n), k = 0..n.
 * Reading A12: evaluated as sin(pi (n - 2k) / (2n)) -- the same number
 * mathematically, but exact 0 at k = n/2 and exact +-symmetry. */
void orc_cheb_nodes(int n, double* t)
{
    for (int k = 0; k <= n; ++k)
        t[k] = sin(ORC_PI * (double)(n - 2 * k) / (2.0 * (double)n));
}

/* Simple barycentric weights w_k = (-1)^k delta_k, delta = 1/2 at k = 0, n
 * (P:312-319). */
void orc_bary_weights(int n, double* w)
{
    for (int k = 0; k <= n; ++k) {
        double d = (k == 0 || k == n) ? 0.5 : 1.0;
        w[k] = (k % 2 == 0) ? d : -d;
    }
}

/* Chebyshev points linearly mapped to [lo, hi]: t -> (a+b)/2 + t (b-a)/2
 * (P:337-346).  Reading A13: s_0 = hi and s_n = lo pinned exactly. */
void orc_grid(int n, double lo, double hi, double* s)
{
    double t[64];
    orc_cheb_nodes(n, t);
    double c = 0.5 * (lo + hi), h = 0.5 * (hi - lo);
    for (int k = 0; k <= n; ++k) s[k] = c + h * t[k];
    s[0] = hi;
    s[n] = lo;
}

/* 1D barycentric Lagrange basis L_k(y) on the mapped grid s (Eq.
 * Barycentric-1D) with the coincidence flag of Algorithm 1 lines
 * 9-17: if |y - s_k| <= DBL_MIN then L = e_k (last k wins). */
void orc_basis(int n, const double* s, double y, double* L)
{
    double w[64], a[64], sum = 0.0;
    int flag = -1;
    orc_bary_weights(n, w);
    for (int k = 0; k <= n; ++k) {
        double diff = y - s[k];
        if (fabs(diff) <= ORC_TOL) {
            flag = k;
            a[k] = 0.0;
        } else {
            a[k] = w[k] / diff;
            sum += a[k];
        }
    }
    if (flag > -1) {
        for (int k = 0; k <= n; ++k) a[k] = 0.0;
        a[flag] = 1.0;
        sum = 1.0;
    }
    for (int k = 0; k <= n; ++k) L[k] = a[k] / sum;
}

/* ------------------------------------------------------------------------- */
/* L1: MRS kernels (§7)                                               */
/* ------------------------------------------------------------------------- */

/* H1, H2, Q, D1, D2 of Eq. MRS_kernels, literal; r2 = r^2. */
void orc_mrs_scalars(double r2, double eps, double* out5)
{
    double e2 = eps * eps;
    double s = r2 + e2;              /* r^2 + eps^2 */
    double s32 = s * sqrt(s);        /* (r^2+eps^2)^{3/2} */
    double s52 = s32 * s;
    double s72 = s52 * s;
    out5[0] = (2.0 * e2 + r2) / (8.0 * ORC_PI * s32);                          /* H1 */
    out5[1] = 1.0 / (8.0 * ORC_PI * s32);                                      /* H2 */
    out5[2] = (5.0 * e2 + 2.0 * r2) / (8.0 * ORC_PI * s52);                    /* Q  */
    out5[3] = (10.0 * e2 * e2 - 7.0 * e2 * r2 - 2.0 * r2 * r2) / (8.0 * ORC_PI * s72); /* D1 */
    out5[4] = (21.0 * e2 + 6.0 * r2) / (8.0 * ORC_PI * s72);                   /* D2 */
}

typedef struct {
    int id;     /* ORC_STOKESLET / ORC_ROTLET / ORC_STOKESLET_ROTLET / ORC_POLY */
    int m, p;   /* weight and output dimension */
    double eps;
    int poly_deg;
} orc_kernel;

static int kernel_dims(int id, int* m, int* p)
{
    switch (id) {
    case ORC_STOKESLET: *m = 3; *p = 3; return 0;
    case ORC_ROTLET: *m = 3; *p = 6; return 0;
    case ORC_STOKESLET_ROTLET: *m = 6; *p = 6; return 0;
    case ORC_POLY: *m = 1; *p = 1; return 0;
    }
    return -1;
}

/* One pair term k(x, y) f added to out[p].
 *  Stokeslet (Eq. Velocity_1): u = f H1 + [f.d] d H2,  d = x - y.
 *  Rotlet (Eqs. Velocity_2 / AngularVelocity with f = 0, reading A10):
 *     u = 1/2 [g x d] Q,  w = 1/4 g D1 + 1/4 [g.d] d D2   (reading A9 for d D2).
 *  Stokeslet+rotlet: both, weights (f, n), outputs (u, w).
 *  POLY (test kernel, not in the paper): k = prod_l (1 + (x_l - y_l)/2)^deg,
 *     a polynomial of degree deg in each source coordinate (far-field pin). */
static void pair_term(const orc_kernel* K, const double* x, const double* y,
                      const double* f, double* t)
{
    double d[3] = {x[0] - y[0], x[1] - y[1], x[2] - y[2]};
    if (K->id == ORC_POLY) {
        double q = 1.0;
        for (int l = 0; l < 3; ++l) q *= pow(1.0 + 0.5 * d[l], (double)K->poly_deg);
        t[0] = q * f[0];
        return;
    }
    double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    double S[5];
    orc_mrs_scalars(r2, K->eps, S);
    const double H1 = S[0], H2 = S[1], Q = S[2], D1 = S[3], D2 = S[4];
    if (K->id == ORC_STOKESLET || K->id == ORC_STOKESLET_ROTLET) {
        double fd = f[0] * d[0] + f[1] * d[1] + f[2] * d[2];
        for (int c = 0; c < 3; ++c) t[c] = f[c] * H1 + fd * d[c] * H2;
    } else {
        for (int c = 0; c < 3; ++c) t[c] = 0.0;
    }
    if (K->id == ORC_STOKESLET) return;
    const double* g = (K->id == ORC_ROTLET) ? f : f + 3; /* torque n_j */
    double gxd[3] = {g[1] * d[2] - g[2] * d[1], g[2] * d[0] - g[0] * d[2], g[0] * d[1] - g[1] * d[0]};
    double gd = g[0] * d[0] + g[1] * d[1] + g[2] * d[2];
    for (int c = 0; c < 3; ++c) t[c] += 0.5 * gxd[c] * Q;
    for (int c = 0; c < 3; ++c) t[3 + c] = 0.25 * g[c] * D1 + 0.25 * gd * d[c] * D2;
    if (K->id == ORC_STOKESLET_ROTLET) {
        double fxd[3] = {f[1] * d[2] - f[2] * d[1], f[2] * d[0] - f[0] * d[2], f[0] * d[1] - f[1] * d[0]};
        for (int c = 0; c < 3; ++c) t[3 + c] += 0.5 * fxd[c] * Q;
    }
}

/* Single pair, exported for the kernel pins. */
int orc_pair(int kernel, double eps, int poly_deg, const double* x, const double* y,
             const double* f, double* out)
{
    orc_kernel K = {kernel, 0, 0, eps, poly_deg};
    if (kernel_dims(kernel, &K.m, &K.p)) return -1;
    pair_term(&K, x, y, f, out);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* L2: tree (§6)                                           */
/* ------------------------------------------------------------------------- */

typedef struct {
    int64_t begin, end; /* sorted-index range [begin, end) */
    int level, parent;
    int nchild;
    int child[8];
    double lo[3], hi[3];
    int degenerate;     /* leaf with count > N0 (reading A3) */
} orc_node;

typedef struct {
    int64_t N;
    int N0;
    double* xs;      /* sorted positions, AoS N x 3 */
    int64_t* perm;   /* perm[s] = original index of sorted particle s */
    int64_t* iperm;  /* iperm[i] = sorted position of original particle i */
    orc_node* nodes; /* BFS order: sorted by (level, begin) */
    int nnodes, cap, depth, ndegenerate;
} orc_tree;

static int push_node(orc_tree* T)
{
    if (T->nnodes == T->cap) {
        int nc = T->cap ? 2 * T->cap : 64;
        orc_node* p = (orc_node*)realloc(T->nodes, (size_t)nc * sizeof(orc_node));
        if (!p) return -1;
        T->nodes = p;
        T->cap = nc;
    }
    memset(&T->nodes[T->nnodes], 0, sizeof(orc_node));
    return T->nnodes++;
}

/* Recursive bisection of cluster `id`:
 *  - box = minimal bounding box of the cluster's particles (root: P:584;
 *    every cluster: reading A3 / BASELINE.json "minimal bounding boxes");
 *  - leaf iff count <= N0 (reading A1);
 *  - bisect axis l iff L_l > lmax/sqrt(2), lmax = this cluster's own max side
 *    (reading A2), at the midpoint; x_l >= mid -> upper half (A3);
 *  - child code bx | by<<1 | bz<<2, stable partition in ascending code, empty
 *    children dropped (so 8, 4 or 2 children);
 *  - degenerate: lmax == 0, or only one nonempty child -> leaf (A3). */
static int build_rec(orc_tree* T, int id, int64_t* tmp_perm, double* tmp_x, unsigned char* code)
{
    orc_node* C = &T->nodes[id];
    int64_t b = C->begin, e = C->end;
    for (int l = 0; l < 3; ++l) {
        C->lo[l] = T->xs[3 * b + l];
        C->hi[l] = T->xs[3 * b + l];
    }
    for (int64_t j = b + 1; j < e; ++j)
        for (int l = 0; l < 3; ++l) {
            double v = T->xs[3 * j + l];
            if (v < C->lo[l]) C->lo[l] = v;
            if (v > C->hi[l]) C->hi[l] = v;
        }
    if (C->level > T->depth) T->depth = C->level;
    if (e - b <= T->N0) return 0;
    double L[3], lmax = 0.0;
    for (int l = 0; l < 3; ++l) {
        L[l] = C->hi[l] - C->lo[l];
        if (L[l] > lmax) lmax = L[l];
    }
    if (lmax == 0.0) {
        C->degenerate = 1;
        T->ndegenerate++;
        return 0;
    }
    int split[3];
    double mid[3];
    for (int l = 0; l < 3; ++l) {
        split[l] = L[l] > lmax * ORC_INV_SQRT2;
        mid[l] = 0.5 * (C->lo[l] + C->hi[l]);
    }
    int64_t cnt[8] = {0};
    for (int64_t j = b; j < e; ++j) {
        int c = 0;
        for (int l = 0; l < 3; ++l)
            if (split[l] && T->xs[3 * j + l] >= mid[l]) c |= 1 << l;
        code[j] = (unsigned char)c;
        cnt[c]++;
    }
    int nonempty = 0;
    for (int c = 0; c < 8; ++c) nonempty += cnt[c] > 0;
    if (nonempty < 2) {
        C->degenerate = 1;
        T->ndegenerate++;
        return 0;
    }
    /* stable partition by ascending code */
    int64_t o = b;
    for (int c = 0; c < 8; ++c)
        for (int64_t j = b; j < e; ++j)
            if (code[j] == c) {
                tmp_perm[o] = T->perm[j];
                for (int l = 0; l < 3; ++l) tmp_x[3 * o + l] = T->xs[3 * j + l];
                ++o;
            }
    memcpy(T->perm + b, tmp_perm + b, (size_t)(e - b) * sizeof(int64_t));
    memcpy(T->xs + 3 * b, tmp_x + 3 * b, (size_t)(e - b) * 3 * sizeof(double));
    int64_t start = b;
    int level = C->level;
    for (int c = 0; c < 8; ++c) {
        if (!cnt[c]) continue;
        int k = push_node(T);
        if (k < 0) return -1;
        C = &T->nodes[id]; /* realloc may move */
        T->nodes[k].begin = start;
        T->nodes[k].end = start + cnt[c];
        T->nodes[k].level = level + 1;
        T->nodes[k].parent = id;
        C->child[C->nchild++] = k;
        start += cnt[c];
    }
    int nch = C->nchild, kids[8];
    memcpy(kids, C->child, sizeof(kids));
    for (int i = 0; i < nch; ++i)
        if (build_rec(T, kids[i], tmp_perm, tmp_x, code)) return -1;
    return 0;
}

static orc_tree* g_sort_tree;
static int cmp_bfs(const void* a, const void* b)
{
    const orc_node* x = &g_sort_tree->nodes[*(const int*)a];
    const orc_node* y = &g_sort_tree->nodes[*(const int*)b];
    if (x->level != y->level) return x->level < y->level ? -1 : 1;
    return (x->begin < y->begin) ? -1 : (x->begin > y->begin);
}

/* Build the tree of particle clusters (Algorithm 2 line 5).
 * Clusters are exported in BFS order (level, then begin) -- a labelling choice
 * only; perm and ranges do not depend on it. Returns 0, or -1 on bad input. */
int orc_build_tree(int64_t N, const double* xyz, int N0, orc_tree** out)
{
    *out = NULL;
    if (N < 1 || N0 < 1) return -1;
    for (int64_t i = 0; i < 3 * N; ++i)
        if (!isfinite(xyz[i])) return -1;
    orc_tree* T = (orc_tree*)calloc(1, sizeof(orc_tree));
    T->N = N;
    T->N0 = N0;
    T->xs = (double*)malloc((size_t)N * 3 * sizeof(double));
    T->perm = (int64_t*)malloc((size_t)N * sizeof(int64_t));
    T->iperm = (int64_t*)malloc((size_t)N * sizeof(int64_t));
    memcpy(T->xs, xyz, (size_t)N * 3 * sizeof(double));
    for (int64_t i = 0; i < N; ++i) T->perm[i] = i;
    int64_t* tmp_perm = (int64_t*)malloc((size_t)N * sizeof(int64_t));
    double* tmp_x = (double*)malloc((size_t)N * 3 * sizeof(double));
    unsigned char* code = (unsigned char*)malloc((size_t)N);
    int r = push_node(T);
    T->nodes[r].begin = 0;
    T->nodes[r].end = N;
    T->nodes[r].parent = -1;
    int rc = build_rec(T, r, tmp_perm, tmp_x, code);
    free(tmp_perm);
    free(tmp_x);
    free(code);
    if (rc) return -1;
    /* relabel to BFS order */
    int nn = T->nnodes;
    int* order = (int*)malloc((size_t)nn * sizeof(int));
    int* newid = (int*)malloc((size_t)nn * sizeof(int));
    for (int i = 0; i < nn; ++i) order[i] = i;
    g_sort_tree = T;
    qsort(order, (size_t)nn, sizeof(int), cmp_bfs);
    for (int i = 0; i < nn; ++i) newid[order[i]] = i;
    orc_node* nodes = (orc_node*)malloc((size_t)nn * sizeof(orc_node));
    for (int i = 0; i < nn; ++i) {
        nodes[i] = T->nodes[order[i]];
        if (nodes[i].parent >= 0) nodes[i].parent = newid[nodes[i].parent];
        for (int c = 0; c < nodes[i].nchild; ++c) nodes[i].child[c] = newid[nodes[i].child[c]];
    }
    free(T->nodes);
    T->nodes = nodes;
    T->cap = nn;
    free(order);
    free(newid);
    for (int64_t s = 0; s < N; ++s) T->iperm[T->perm[s]] = s;
    *out = T;
    return 0;
}

void orc_tree_free(orc_tree* T)
{
    if (!T) return;
    free(T->xs);
    free(T->perm);
    free(T->iperm);
    free(T->nodes);
    free(T);
}

void orc_tree_info(const orc_tree* T, int64_t* nclusters, int* depth, int* ndegenerate)
{
    *nclusters = T->nnodes;
    *depth = T->depth;
    *ndegenerate = T->ndegenerate;
}

/* Export: perm[N]; per cluster begin, end, level, parent, first_child (-1 for
 * leaves; children are contiguous in BFS order), nchild, lo[3], hi[3]. */
void orc_tree_export(const orc_tree* T, int64_t* perm, int64_t* begin, int64_t* end,
                     int32_t* level, int32_t* parent, int32_t* first_child,
                     int32_t* nchild, double* lo, double* hi)
{
    memcpy(perm, T->perm, (size_t)T->N * sizeof(int64_t));
    for (int i = 0; i < T->nnodes; ++i) {
        const orc_node* C = &T->nodes[i];
        begin[i] = C->begin;
        end[i] = C->end;
        level[i] = C->level;
        parent[i] = C->parent;
        nchild[i] = C->nchild;
        first_child[i] = C->nchild ? C->child[0] : -1;
        for (int l = 0; l < 3; ++l) {
            lo[3 * i + l] = C->lo[l];
            hi[3 * i + l] = C->hi[l];
        }
    }
}

/* ------------------------------------------------------------------------- */
/* L3a: modified weights, Algorithm 1                             */
/* ------------------------------------------------------------------------- */

/* Grids of cluster C, reading A3/A13: s_{l,k} on [lo_l, hi_l]. */
static void cluster_grids(const orc_node* C, int n, double* s /* 3 x (n+1) */)
{
    for (int l = 0; l < 3; ++l) orc_grid(n, C->lo[l], C->hi[l], s + l * (n + 1));
}

/* Algorithm 1 for one cluster, literally.  y: sorted positions,
 * f: sorted weights (N x m).  fhat[m][(n+1)^3], k3 fastest. */
static void alg1_cluster(const orc_node* C, int n, int m, const double* xs, const double* f,
                         double* fhat)
{
    int P = n + 1, P3 = P * P * P;
    double s[3 * 64], w[64], a[3][64], sum[3];
    int flag[3];
    cluster_grids(C, n, s);
    orc_bary_weights(n, w);
    for (int i = 0; i < m * P3; ++i) fhat[i] = 0.0;                 /* line 4 */
    for (int64_t j = C->begin; j < C->end; ++j) {                   /* line 6 */
        for (int l = 0; l < 3; ++l) { flag[l] = -1; sum[l] = 0.0; } /* line 7 */
        for (int k = 0; k <= n; ++k)                                /* line 9 */
            for (int l = 0; l < 3; ++l) {
                double diff = xs[3 * j + l] - s[l * P + k];
                if (fabs(diff) <= ORC_TOL) {                        /* line 10 */
                    flag[l] = k;
                } else {                                            /* line 11 */
                    a[l][k] = w[k] / diff;
                    sum[l] += a[l][k];
                }
            }
        for (int l = 0; l < 3; ++l)                                 /* lines 15-17 */
            if (flag[l] > -1) {
                sum[l] = 1.0;
                for (int k = 0; k <= n; ++k) a[l][k] = 0.0;
                a[l][flag[l]] = 1.0;
            }
        double denom = sum[0] * sum[1] * sum[2];                    /* line 18 */
        for (int k1 = 0; k1 <= n; ++k1)                             /* lines 20-22 */
            for (int k2 = 0; k2 <= n; ++k2)
                for (int k3 = 0; k3 <= n; ++k3) {
                    double coef = a[0][k1] * a[1][k2] * a[2][k3] / denom;
                    int idx = (k1 * P + k2) * P + k3;
                    for (int c = 0; c < m; ++c) fhat[c * P3 + idx] += coef * f[j * m + c];
                }
    }
}

/* Modified weights of every cluster (Algorithm 2 line 6); w is in
 * ORIGINAL particle order (N x m).  fhat: nclusters x m x (n+1)^3. */
int orc_modified_weights(const orc_tree* T, int n, int m, const double* w, double* fhat)
{
    if (n < 1 || n > 60 || m < 1) return -1;
    int64_t N = T->N;
    double* fs = (double*)malloc((size_t)N * m * sizeof(double));
    for (int64_t s = 0; s < N; ++s)
        for (int c = 0; c < m; ++c) fs[s * m + c] = w[T->perm[s] * m + c];
    size_t per = (size_t)m * (n + 1) * (n + 1) * (n + 1);
    for (int i = 0; i < T->nnodes; ++i) alg1_cluster(&T->nodes[i], n, m, T->xs, fs, fhat + per * i);
    free(fs);
    return 0;
}

/* Same, for clusters [cb, ce) only (bounded-sample timing in bench.py). */
int orc_modified_weights_range(const orc_tree* T, int n, int m, const double* w, int64_t cb,
                               int64_t ce, double* fhat)
{
    if (n < 1 || n > 60 || m < 1 || cb < 0 || ce > T->nnodes || cb > ce) return -1;
    int64_t N = T->N;
    double* fs = (double*)malloc((size_t)N * m * sizeof(double));
    for (int64_t s = 0; s < N; ++s)
        for (int c = 0; c < m; ++c) fs[s * m + c] = w[T->perm[s] * m + c];
    size_t per = (size_t)m * (n + 1) * (n + 1) * (n + 1);
    for (int64_t i = cb; i < ce; ++i) alg1_cluster(&T->nodes[i], n, m, T->xs, fs, fhat + per * i);
    free(fs);
    return 0;
}

/* NOT IN THE PAPER: the modified weights of an internal
 * cluster from its children's.  Eq. modified_weights defines
 * fhat_k = sum_j L_k(y_j) f_j; L_k is a tensor product of degree-n polynomials
 * and a child's fhat reproduces every such moment of its particles
 * (sum_k' fhat_C,k' q(s_C,k') = sum_{j in C} f_j q(y_j)), so Algorithm 1 applied
 * to the children's proxy points s_C,k' carrying the charges fhat_C,k' gives the
 * parent's fhat exactly in exact arithmetic, at a cost independent of N_C
 * (the cost argument of P:465-469).  Leaves use Algorithm 1 on their particles.
 * Literal: the children in order, each child's proxies in lexicographic
 * (k1, k2, k3) order are the "particles" of alg1_cluster on the parent's grid.
 * Clusters are processed in decreasing BFS id (children before parents). */
int orc_modified_weights_upward(const orc_tree* T, int n, int m, const double* w, double* fhat)
{
    if (n < 1 || n > 60 || m < 1) return -1;
    int64_t N = T->N;
    int P = n + 1, P3 = P * P * P;
    size_t per = (size_t)m * P3;
    double* fs = (double*)malloc((size_t)N * m * sizeof(double));
    for (int64_t s = 0; s < N; ++s)
        for (int c = 0; c < m; ++c) fs[s * m + c] = w[T->perm[s] * m + c];
    double* py = (double*)malloc((size_t)8 * P3 * 3 * sizeof(double));  /* children's proxy points */
    double* pf = (double*)malloc((size_t)8 * P3 * m * sizeof(double));  /* and their charges */
    for (int i = T->nnodes - 1; i >= 0; --i) {
        const orc_node* C = &T->nodes[i];
        if (C->nchild == 0) {
            alg1_cluster(C, n, m, T->xs, fs, fhat + per * i);
            continue;
        }
        int64_t q = 0;
        for (int ch = 0; ch < C->nchild; ++ch) {
            const orc_node* K = &T->nodes[C->child[ch]];
            const double* fk = fhat + per * C->child[ch];
            double s[3 * 64];
            cluster_grids(K, n, s);
            for (int k1 = 0; k1 <= n; ++k1)
                for (int k2 = 0; k2 <= n; ++k2)
                    for (int k3 = 0; k3 <= n; ++k3, ++q) {
                        int idx = (k1 * P + k2) * P + k3;
                        py[3 * q] = s[k1];
                        py[3 * q + 1] = s[P + k2];
                        py[3 * q + 2] = s[2 * P + k3];
                        for (int c = 0; c < m; ++c) pf[q * m + c] = fk[c * P3 + idx];
                    }
        }
        orc_node proxy = *C;  /* the parent's box, its children's proxies as the particles */
        proxy.begin = 0;
        proxy.end = q;
        alg1_cluster(&proxy, n, m, py, pf, fhat + per * i);
    }
    free(py);
    free(pf);
    free(fs);
    return 0;
}

/* Modified weights of one explicit particle set on an explicit box (for the
 * moment-identity pins): y N x 3, f N x m, box lo/hi -> fhat m x (n+1)^3. */
int orc_modified_weights_box(int64_t N, const double* y, const double* f, int m, int n,
                             const double* lo, const double* hi, double* fhat)
{
    orc_node C;
    memset(&C, 0, sizeof(C));
    C.begin = 0;
    C.end = N;
    for (int l = 0; l < 3; ++l) { C.lo[l] = lo[l]; C.hi[l] = hi[l]; }
    alg1_cluster(&C, n, m, y, f, fhat);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* L3b: treecode evaluation, Algorithm 2                          */
/* ------------------------------------------------------------------------- */

typedef struct {
    const orc_tree* T;
    orc_kernel K;
    int n;
    double tt;        /* theta * theta, RN */
    int self_omit;
    int size_check;   /* variant: accepted cluster with N_C < (n+1)^3 -> direct */
    const double* fhat;
    const double* fs; /* sorted weights */
    long double acc[6];
    uint64_t st[5];   /* far clusters, far pairs, near leaves, near pairs, covered */
} eval_ctx;

/* MAC r/R <= theta (Eq. MAC), reading A4/A5: R^2 > 0 and
 * r^2 <= (theta*theta) R^2; r = half-diagonal, centre = box centre; all RN. */
static int mac(const orc_node* C, const double* x, double tt)
{
    double c[3], h[3];
    for (int l = 0; l < 3; ++l) {
        c[l] = 0.5 * (C->lo[l] + C->hi[l]);
        h[l] = 0.5 * (C->hi[l] - C->lo[l]);
    }
    double r2 = (h[0] * h[0] + h[1] * h[1]) + h[2] * h[2];
    double dx = x[0] - c[0], dy = x[1] - c[1], dz = x[2] - c[2];
    double R2 = (dx * dx + dy * dy) + dz * dz;
    return R2 > 0.0 && r2 <= tt * R2;
}

/* compute_velocity(x, C). xi_s = sorted index of the target. */
static void compute_velocity(eval_ctx* E, const double* x, int64_t xi_s, int id)
{
    const orc_tree* T = E->T;
    const orc_node* C = &T->nodes[id];
    int p = E->K.p, m = E->K.m, P = E->n + 1, P3 = P * P * P;
    double t[6];
    int accept = mac(C, x, E->tt);
    if (accept && E->size_check && C->end - C->begin < (int64_t)P3) {
        /* size-check variant (not in the paper; motivated by its cost argument
         * "a cost reduction when N_c >> n^3"): an accepted cluster
         * holding fewer particles than proxies is summed directly over its
         * particles (Eq. pc_interaction_3D).  The target lies outside an
         * accepted box (r <= theta R < R), so no self term can occur. */
        for (int64_t j = C->begin; j < C->end; ++j) {
            pair_term(&E->K, x, T->xs + 3 * j, E->fs + j * m, t);
            for (int c = 0; c < p; ++c) E->acc[c] += t[c];
            E->st[3] += 1;
        }
        E->st[2] += 1;
        E->st[4] += (uint64_t)(C->end - C->begin);
        return;
    }
    if (accept) {
        /* far field, Eq. pc_approximation_3D: target vs the (n+1)^3
         * Chebyshev points s_k with modified weights fhat_k */
        double s[3 * 64], fk[6], y[3];
        cluster_grids(C, E->n, s);
        const double* F = E->fhat + (size_t)id * m * P3;
        for (int k1 = 0; k1 < P; ++k1)
            for (int k2 = 0; k2 < P; ++k2)
                for (int k3 = 0; k3 < P; ++k3) {
                    int idx = (k1 * P + k2) * P + k3;
                    y[0] = s[k1];
                    y[1] = s[P + k2];
                    y[2] = s[2 * P + k3];
                    for (int c = 0; c < m; ++c) fk[c] = F[c * P3 + idx];
                    pair_term(&E->K, x, y, fk, t);
                    for (int c = 0; c < p; ++c) E->acc[c] += t[c];
                }
        E->st[0] += 1;
        E->st[1] += (uint64_t)P3;
        E->st[4] += (uint64_t)(C->end - C->begin);
    } else if (C->nchild == 0) {
        /* leaf: direct sum, Eq. pc_interaction_3D; self term by
         * index (reading A8) */
        for (int64_t j = C->begin; j < C->end; ++j) {
            if (E->self_omit && j == xi_s) continue;
            pair_term(&E->K, x, T->xs + 3 * j, E->fs + j * m, t);
            for (int c = 0; c < p; ++c) E->acc[c] += t[c];
            E->st[3] += 1;
        }
        E->st[2] += 1;
        E->st[4] += (uint64_t)(C->end - C->begin);
    } else {
        for (int i = 0; i < C->nchild; ++i) compute_velocity(E, x, xi_s, C->child[i]);
    }
}

/* Treecode velocities (Algorithm 2 line 7) for the targets `tgt`
 * (ORIGINAL indices; NULL = all N in order), targets = sources.
 * out: nt x p; stats (optional): nt x 5.  w: original order N x m. */
int orc_treecode_ex(const orc_tree* T, int kernel, double eps, int n, double theta, int self_omit,
                    int size_check, const double* fhat, const double* w, const int64_t* tgt, int64_t nt,
                    double* out, uint64_t* stats);
int orc_treecode(const orc_tree* T, int kernel, double eps, int n, double theta, int self_omit,
                 const double* fhat, const double* w, const int64_t* tgt, int64_t nt,
                 double* out, uint64_t* stats)
{
    return orc_treecode_ex(T, kernel, eps, n, theta, self_omit, 0, fhat, w, tgt, nt, out, stats);
}

/* As orc_treecode, with the size-check variant selectable (size_check != 0). */
int orc_treecode_ex(const orc_tree* T, int kernel, double eps, int n, double theta, int self_omit,
                    int size_check, const double* fhat, const double* w, const int64_t* tgt, int64_t nt,
                    double* out, uint64_t* stats)
{
    eval_ctx E;
    memset(&E, 0, sizeof(E));
    E.T = T;
    E.K.id = kernel;
    E.K.eps = eps;
    E.K.poly_deg = n;
    if (kernel_dims(kernel, &E.K.m, &E.K.p)) return -1;
    E.n = n;
    E.tt = theta * theta;
    E.self_omit = self_omit;
    E.size_check = size_check;
    E.fhat = fhat;
    int64_t N = T->N;
    int m = E.K.m, p = E.K.p;
    double* fs = (double*)malloc((size_t)N * m * sizeof(double));
    for (int64_t s = 0; s < N; ++s)
        for (int c = 0; c < m; ++c) fs[s * m + c] = w[T->perm[s] * m + c];
    E.fs = fs;
    if (!tgt) nt = N;
    for (int64_t q = 0; q < nt; ++q) {
        int64_t i = tgt ? tgt[q] : q;
        int64_t si = T->iperm[i];
        for (int c = 0; c < 6; ++c) E.acc[c] = 0.0L;
        memset(E.st, 0, sizeof(E.st));
        compute_velocity(&E, T->xs + 3 * si, si, 0);
        for (int c = 0; c < p; ++c) out[q * p + c] = (double)E.acc[c];
        if (stats)
            for (int c = 0; c < 5; ++c) stats[q * 5 + c] = E.st[c];
    }
    free(fs);
    return 0;
}

/* Treecode velocities at a SEPARATE target set (Algorithm 2 with targets x_i
 * that need not be sources; "the targets and sources coincide, but
 * this is not an essential restriction").  Same traversal as orc_treecode, no self term (no target is a
 * source); the root and every ancestor of a target's position may be accepted
 * when the target lies outside them.  xt: nt x 3; out: nt x p; stats optional;
 * size_check: the variant of orc_treecode_ex. */
int orc_treecode_targets(const orc_tree* T, int kernel, double eps, int n, double theta, int size_check,
                         const double* fhat, const double* w, const double* xt, int64_t nt,
                         double* out, uint64_t* stats)
{
    eval_ctx E;
    memset(&E, 0, sizeof(E));
    E.T = T;
    E.K.id = kernel;
    E.K.eps = eps;
    E.K.poly_deg = n;
    if (kernel_dims(kernel, &E.K.m, &E.K.p)) return -1;
    E.n = n;
    E.tt = theta * theta;
    E.self_omit = 0;
    E.size_check = size_check;
    E.fhat = fhat;
    int64_t N = T->N;
    int m = E.K.m, p = E.K.p;
    double* fs = (double*)malloc((size_t)N * m * sizeof(double));
    for (int64_t s = 0; s < N; ++s)
        for (int c = 0; c < m; ++c) fs[s * m + c] = w[T->perm[s] * m + c];
    E.fs = fs;
    for (int64_t q = 0; q < nt; ++q) {
        for (int c = 0; c < 6; ++c) E.acc[c] = 0.0L;
        memset(E.st, 0, sizeof(E.st));
        compute_velocity(&E, xt + 3 * q, -1, 0);
        for (int c = 0; c < p; ++c) out[q * p + c] = (double)E.acc[c];
        if (stats)
            for (int c = 0; c < 5; ++c) stats[q * 5 + c] = E.st[c];
    }
    free(fs);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* Direct sum and error                                   */
/* ------------------------------------------------------------------------- */

/* u(x_i) = sum_j k(x_i, x_j) f_j over j ascending in original order, j != i
 * skipped iff self_omit (reading A8).  Targets = sources; tgt as above. */
int orc_direct(int kernel, double eps, int poly_deg, int self_omit, int64_t N, const double* xyz,
               const double* w, const int64_t* tgt, int64_t nt, double* out)
{
    orc_kernel K = {kernel, 0, 0, eps, poly_deg};
    if (kernel_dims(kernel, &K.m, &K.p)) return -1;
    if (!tgt) nt = N;
    double t[6];
    for (int64_t q = 0; q < nt; ++q) {
        int64_t i = tgt ? tgt[q] : q;
        long double acc[6] = {0};
        for (int64_t j = 0; j < N; ++j) {
            if (self_omit && j == i) continue;
            pair_term(&K, xyz + 3 * i, xyz + 3 * j, w + j * K.m, t);
            for (int c = 0; c < K.p; ++c) acc[c] += t[c];
        }
        for (int c = 0; c < K.p; ++c) out[q * K.p + c] = (double)acc[c];
    }
    return 0;
}

/* u(x_q) = sum_j k(x_q, y_j) f_j (Eq. N-body) at separate targets xt
 * (nt x 3), all j ascending (no self term: no target is a source). */
int orc_direct_targets(int kernel, double eps, int poly_deg, int64_t N, const double* xyz,
                       const double* w, const double* xt, int64_t nt, double* out)
{
    orc_kernel K = {kernel, 0, 0, eps, poly_deg};
    if (kernel_dims(kernel, &K.m, &K.p)) return -1;
    double t[6];
    for (int64_t q = 0; q < nt; ++q) {
        long double acc[6] = {0};
        for (int64_t j = 0; j < N; ++j) {
            pair_term(&K, xt + 3 * q, xyz + 3 * j, w + j * K.m, t);
            for (int c = 0; c < K.p; ++c) acc[c] += t[c];
        }
        for (int c = 0; c < K.p; ++c) out[q * K.p + c] = (double)acc[c];
    }
    return 0;
}

/* Relative error E of Eq. error: rows of p components concatenated
 * per particle. Returns -1 if the reference is identically zero. */
double orc_rel_error(const double* ref, const double* approx, int64_t rows, int p)
{
    long double num = 0.0L, den = 0.0L;
    for (int64_t i = 0; i < rows * p; ++i) {
        long double d = (long double)ref[i] - (long double)approx[i];
        num += d * d;
        den += (long double)ref[i] * (long double)ref[i];
    }
    if (den == 0.0L) return -1.0;
    return (double)sqrtl(num / den);
}
