/*
 * kitc.h -- C ABI of libkitc.so, the B200 (sm_100a) hot path of the
 * barycentric Lagrange kernel-independent treecode (KITC) of Wang, Krasny and
 * Tlupova, arXiv:1902.02250.  P:<n> = PAPER.md line n.
 *
 * The library computes, for targets = sources x_i (i = 0..N-1) -- or for a
 * separate target set (kitc_eval_targets) --
 *     u(x_i) = sum_j k(x_i, x_j) f_j                       (Eq. N-body)
 * with the particle-cluster treecode of Algorithm 2: a tree of
 * rectangular clusters, modified weights at (n+1)^3 Chebyshev
 * points per cluster (Eq. modified_weights, Algorithm 1),
 * and a per-target traversal under the MAC r/R <= theta (Eq. MAC)
 * summing far clusters through their proxies (Eq. pc_approximation_3D,
 * P:436-440) and near leaves directly (Eq. pc_interaction_3D).
 * Kernels: the regularized Stokeslet (Eq. Velocity_1), the rotlet
 * (Eqs. Velocity_2 / AngularVelocity with f = 0) and the combined
 * Stokeslet+rotlet.  kitc_direct is the O(N^2) sum.
 *
 * Conventions (all entry points):
 *  - Pointers named *_dev are CUDA device pointers; *_host are host pointers.
 *    The CALLER owns every buffer passed in.  The device memory of a tree
 *    handle comes from the caller's kitc_allocator (kitc_tree_create_with_
 *    allocator; the Python binding passes PyTorch's caching allocator), or, for
 *    kitc_tree_create, from cudaMallocAsync on the device's default pool (whose
 *    attributes the library never changes).  It is requested on the stream of
 *    the call that needs it, retained across rebuilds (reallocated only to
 *    grow) and released by kitc_tree_free.  kitc_tree_workspace_bytes bounds it.
 *  - Layouts: coordinates are AoS double[N][3]; weights are AoS double[N][m];
 *    outputs are AoS double[N][p]; all in the caller's ORIGINAL particle order.
 *  - Work is enqueued on the caller's stream `s` (cudaStream_t passed as void*;
 *    NULL = legacy default stream).  Only kitc_build_tree and kitc_tree_export
 *    synchronize that stream.
 *  - Errors never cross the ABI as exceptions: every call returns a
 *    kitc_status; kitc_last_error() returns a thread-local message for the
 *    last non-OK status.  KITC_ECUDA is returned for launch or asynchronous
 *    CUDA errors observed by the call.
 *  - Everything is fp64.  Results are deterministic: bitwise identical run to
 *    run and independent of how batch / cluster ranges are split across calls
 *    or ranks (kitc_eval, kitc_eval_ex, kitc_eval_part, the peer-replicated
 *    modified weights).  The treecode evaluation uses a one-Newton-step
 *    s^{-1/2} (relative error < 2e-12; reading A19); kitc_direct
 *    keeps ~4 ulp.
 */
#ifndef KITC_H
#define KITC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    KITC_OK = 0,
    KITC_EINVAL = -1, /* bad argument (range, NULL, non-finite coordinate, ...) */
    KITC_ENOMEM = -2, /* device or host allocation failed */
    KITC_ECUDA = -3,  /* CUDA launch / runtime error */
    KITC_ESTATE = -4  /* call order violated (e.g. eval before weights) */
} kitc_status;

typedef enum {
    KITC_STOKESLET = 0,         /* m = 3 (force f),  p = 3 (u)         Eq. Velocity_1 */
    KITC_ROTLET = 1,            /* m = 3 (torque n), p = 6 (u, w)      Eqs. Velocity_2/AngularVelocity, f = 0 */
    KITC_STOKESLET_ROTLET = 2   /* m = 6 (f, n),     p = 6 (u, w)      Eqs. Velocity_2/AngularVelocity */
} kitc_kernel;

typedef enum {
    KITC_SELF_OMIT = 0,   /* skip j == i (by index) -- BASELINE configs, reading A8 */
    KITC_SELF_INCLUDE = 1 /* sum over all j (the regularized kernels are finite at r = 0) */
} kitc_self;

typedef struct kitc_tree kitc_tree; /* opaque, library-owned handle */

/* Weight and output dimensions (m, p) of a kernel.  EINVAL for unknown k. */
kitc_status kitc_kernel_dims(int32_t kernel, int32_t* m, int32_t* p);

/* Doubles per cluster in the fhat layout of kernel k at degree n in [1, 16]
 * (see kitc_modified_weights): R (n+1) m 8 with R = ceil((n+1)^2 / 8).
 * EINVAL for unknown k or n out of range. */
kitc_status kitc_fhat_cluster_len(int32_t kernel, int32_t n, int64_t* len);

/* Device-memory provider of a tree handle (device memory is
 * the caller's).  alloc(bytes, stream, ctx) returns a 16-byte aligned device
 * pointer usable in stream order on `stream` (a cudaStream_t as void*), or NULL
 * (-> KITC_ENOMEM); release(ptr, stream, ctx) gives it back once the work
 * enqueued on `stream` is done with it.  Called from inside kitc_build_tree,
 * kitc_modified_weights, kitc_eval_targets (growth only) and kitc_tree_free. */
typedef struct {
    void* (*alloc)(size_t bytes, void* stream, void* ctx);
    void (*release)(void* ptr, void* stream, void* ctx);
    void* ctx;
} kitc_allocator;

/* Create an empty tree handle (no device memory yet) whose device memory comes
 * from *a (copied; NULL = cudaMallocAsync).  EINVAL if a has a NULL member.
 * *out = NULL on error. */
kitc_status kitc_tree_create_with_allocator(const kitc_allocator* a, kitc_tree** out);

/* kitc_tree_create_with_allocator(NULL, out). */
kitc_status kitc_tree_create(kitc_tree** out);

/* Build the cluster tree of N particles (Algorithm 2 line 5; rule
 * P:583-596 with DESIGN.md readings A1-A4): every cluster's box is the minimal
 * bounding box of its particles; a cluster with count > N0 is bisected at its
 * midpoint along every side longer than lmax/sqrt(2) (lmax = its own longest
 * side), particles with x_l >= mid go to the upper half; children are the
 * nonempty groups in ascending code bx|by<<1|bz<<2, stably partitioned; a
 * cluster whose split leaves one nonempty child (or lmax = 0) stays a leaf.
 *  xyz_dev: device, double[N][3], original order, finite (else EINVAL).
 *  N in [1, 2^30 - 1], N0 >= 1.  Rebuilding an existing handle is allowed.
 * The whole build is ONE cooperative kernel on the device (no host work per
 * level); the call then reads back a block of counters -- its only
 * synchronisation of the stream.  EINVAL for a tree deeper than 4000 levels. */
kitc_status kitc_build_tree(kitc_tree* t, const double* xyz_dev, int64_t N, int32_t N0, void* s);

/* Upper bound of the device memory (bytes) a tree handle requests from its
 * allocator for N particles at leaf size N0 (kitc_build_tree) and modified
 * weights of `kernel` at degree n (kitc_modified_weights; kitc_eval needs no
 * more), assuming the worst-case tree of 2N - 1 clusters.  Lets a caller size
 * an arena for kitc_tree_create_with_allocator up front.  Excludes the
 * separate-target scratch of kitc_eval_targets (~44 Nt bytes + radix-sort temp).
 * EINVAL for N < 1, N0 < 1, unknown kernel, n outside [1, 16]. */
kitc_status kitc_tree_workspace_bytes(int64_t N, int32_t N0, int32_t kernel, int32_t n, size_t* bytes);

/* Sizes of the built tree.  Any output pointer may be NULL.
 *  n_clusters: number of clusters C (BFS order: by level, then by range start);
 *  depth: deepest level (root = 0); n_batches: number of warp batches of
 *  <= 4 targets (never straddling a leaf; ordered by leaf, Morton order inside);
 *  n_degenerate: leaves with count > N0 (coincident points). */
kitc_status kitc_tree_info(const kitc_tree* t, int64_t* n_clusters, int32_t* depth,
                           int64_t* n_batches, int32_t* n_degenerate);

/* Copy the tree structure to host buffers (for parity checks; synchronizes).
 * Any pointer may be NULL.  perm_host[N]: sorted position -> original index;
 * per cluster (C entries): begin, end (sorted-index range), level, parent
 * (-1 for the root), first_child (-1 for leaves; children are contiguous),
 * nchild, lo_host[C][3], hi_host[C][3] (the minimal box). */
kitc_status kitc_tree_export(const kitc_tree* t, int64_t* perm_host, int64_t* begin_host,
                             int64_t* end_host, int32_t* level_host, int32_t* parent_host,
                             int32_t* first_child_host, int32_t* nchild_host, double* lo_host,
                             double* hi_host);

/* Modified weights (Eq. modified_weights, Algorithm 1)
 * of clusters [cluster_begin, cluster_end) at degree n in [1, 16]:
 *   fhat_k = sum_{y_j in C} L_k1(y_j1) L_k2(y_j2) L_k3(y_j3) f_j
 * with L in barycentric form (Eq. Barycentric-1D) on the cluster's Chebyshev
 * grid s_{l,k} = c_l + h_l cos(k pi / n) (s_{l,0} = hi_l and s_{l,n} = lo_l
 * exactly), simple weights (-1)^k delta_k, and the coincidence flag
 * |y - s_k| <= DBL_MIN -> L = e_k (last k wins).
 *  w_dev: device, double[N][m] in ORIGINAL order (m from kitc_kernel_dims).
 *  fhat_dev: device, 16-byte aligned, double[C][L] with L from
 *  kitc_fhat_cluster_len, in the order [c][r][k3][comp][j]: the (n+1)^2 rows
 *  row = k1 (n+1) + k2 = 8 r + j are grouped in blocks of 8 ("rounds"), each
 *  block holding all k3 and components of its 8 rows contiguously (one bulk
 *  copy per round in kitc_eval); rows >= (n+1)^2 of the last block are written
 *  as 0.  Only the requested clusters' slices are written (a contiguous byte
 *  range per cluster range).  Also gathers w into the tree's sorted layout and
 *  computes every cluster's grid (both used by kitc_eval).
 *  0 <= cluster_begin <= cluster_end <= C.  ESTATE if no tree is built.
 *  Enqueue-only: the work items are generated on the device (no host sync). */
kitc_status kitc_modified_weights(kitc_tree* t, int32_t kernel, int32_t n, const double* w_dev,
                                  int64_t cluster_begin, int64_t cluster_end, double* fhat_dev,
                                  void* s);

/* Modified-weights variants (flags of kitc_modified_weights_ex). */
typedef enum {
    /* Not in the paper (the cost argument of P:465-469): the
     * fhat of an internal cluster is computed from its children's -- Algorithm 1
     * applied to the children's proxy points carrying their fhat, done as three 1D
     * interpolation transforms -- instead of from its N_C particles; leaves use
     * Algorithm 1.  Exact in exact arithmetic (a child's fhat reproduces every
     * moment of degree <= n per axis), so it changes results by rounding only
     * (reading A24); the oracle mirrors it (orc_modified_weights_upward).
     * Requires cluster_end = C (every child of a computed cluster is computed). */
    KITC_WEIGHTS_UPWARD = 1
} kitc_weights_flag;

/* kitc_modified_weights with variant flags (0 = Algorithm 1 for every cluster;
 * unknown bits -> EINVAL). */
kitc_status kitc_modified_weights_ex(kitc_tree* t, int32_t kernel, int32_t n, const double* w_dev,
                                     int64_t cluster_begin, int64_t cluster_end, uint32_t flags,
                                     double* fhat_dev, void* s);

/* Fused modified weights + replication for the multi-GPU path (SURVEY.md §8(e),
 * §8(f) f3): as kitc_modified_weights, but every computed cluster slice is
 * stored into each of the npeers buffers fhat_peers[0..npeers-1] (host array
 * of device pointers, npeers in [1, 8], each a full double[C][L] f-hat in the
 * same layout).  On a node the entries are the peer GPUs' f-hat buffers mapped
 * into this process (CUDA IPC / symmetric memory over NVLink 5 / NVSwitch), so
 * when every rank calls this for its own cluster range and then all ranks pass
 * a barrier, every rank holds the full f-hat -- the all-gather is done by the
 * kernel's own stores, overlapped with its compute.  The caller provides the
 * barrier (stream-ordered after this call).  npeers = 1 is kitc_modified_weights. */
kitc_status kitc_modified_weights_peers(kitc_tree* t, int32_t kernel, int32_t n, const double* w_dev,
                                        int64_t cluster_begin, int64_t cluster_end,
                                        double* const* fhat_peers, int32_t npeers, void* s);

/* Treecode evaluation (Algorithm 2 lines 7-17) for the targets of
 * batches [batch_begin, batch_end): per target, depth-first over the tree;
 * MAC accept iff R^2 > 0 and r^2 <= (theta*theta) R^2 (R = distance to the box
 * centre, r = half-diagonal, all round-to-nearest, no FMA: DESIGN.md A4/A5);
 * accepted -> far field over the (n+1)^3 proxies with fhat; rejected leaf ->
 * direct sum over its particles (j == i skipped under KITC_SELF_OMIT);
 * rejected internal -> children.
 *  n, kernel: must match the last kitc_modified_weights call; N0 must equal
 *  the tree's N0; 0 <= theta < 1; eps >= 0 (eps = 0 requires SELF_OMIT).
 *  fhat_dev: the FULL double[C][L] of kitc_modified_weights (every cluster),
 *  16-byte aligned (else EINVAL).
 *  out_dev: device double[N][p], original order; only the targets of the given
 *  batches are written.  It may also be pinned host memory (cudaMallocHost /
 *  cudaHostAlloc, mapped into the device address space under unified
 *  addressing): each target's row is then written over the host link as the
 *  kernel finishes it (zero-copy; the caller synchronises before reading).
 *  stats_dev: optional (NULL = off) device uint64[N][5], original order:
 *  far clusters, far pairs, near leaves, near pairs, covered sources. */
kitc_status kitc_eval(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0,
                      double eps, int32_t self, const double* fhat_dev, int64_t batch_begin,
                      int64_t batch_end, double* out_dev, uint64_t* stats_dev, void* s);

/* Treecode at a SEPARATE set of Nt targets (targets need not be
 * sources): the same traversal, MAC, far field and
 * near field as kitc_eval, with no self term (every source j is summed), so the
 * root and the ancestors of a target's position may be accepted when it lies
 * outside them.  Targets are batched internally along a Morton curve of their
 * bounding box (scratch owned by the tree handle; one call per handle at a time).
 *  xt_dev: device double[Nt][3] (any positions; eps = 0 and a target on a
 *  source gives a non-finite row -- the singular kernel); out_dev: device
 *  double[Nt][p] in the order of xt_dev; stats_dev optional uint64[Nt][5] as
 *  kitc_eval.  Other arguments and errors as kitc_eval.  Multi-GPU: each rank
 *  passes its own slice of the targets. */
kitc_status kitc_eval_targets(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0,
                              double eps, const double* fhat_dev, const double* xt_dev, int64_t Nt,
                              double* out_dev, uint64_t* stats_dev, void* s);

/* Evaluation variants (flags of kitc_eval_ex / kitc_eval_targets_ex). */
typedef enum {
    /* Not in the paper, motivated by its cost argument
     * "a cost reduction when N_c >> n^3": an ACCEPTED cluster with
     * N_C < (n+1)^3 particles is summed directly over its particles instead of
     * its (n+1)^3 proxies (counted as a near interaction in stats).  Changes the
     * result (more exact); the oracle mirrors it (orc_treecode_ex). */
    KITC_EVAL_SIZE_CHECK = 1
} kitc_eval_flag;

/* kitc_eval / kitc_eval_targets with variant flags (0 = the paper's method;
 * unknown bits -> EINVAL). */
kitc_status kitc_eval_ex(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                         int32_t self, uint32_t flags, const double* fhat_dev, int64_t batch_begin,
                         int64_t batch_end, double* out_dev, uint64_t* stats_dev, void* s);
kitc_status kitc_eval_targets_ex(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0,
                                 double eps, uint32_t flags, const double* fhat_dev, const double* xt_dev,
                                 int64_t Nt, double* out_dev, uint64_t* stats_dev, void* s);

/* kitc_eval_ex for part `part` of an interleaved split of ALL batches into
 * nparts parts (multi-GPU: part = rank, nparts = world size): the batches come
 * in chunks of 64 dealt round-robin, so every part samples the whole domain and
 * the parts' work is balanced (contiguous ranges balanced by target count leave
 * up to 7% imbalance, tools/balance_check.py).  The batches themselves do not
 * change, so every target's result is bitwise that of the single-GPU run.
 *  0 <= part < nparts.  Other arguments as kitc_eval_ex. */
kitc_status kitc_eval_part(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                           int32_t self, uint32_t flags, const double* fhat_dev, int32_t part, int32_t nparts,
                           double* out_dev, uint64_t* stats_dev, void* s);

/* Number of targets in batches [0, batch_end) -- for splitting work. */
kitc_status kitc_batch_targets(const kitc_tree* t, int64_t batch_end, int64_t* n_targets);

/* O(N^2) direct sum u(x_i) = sum_j k(x_i, y_j) f_j (Eq. N-body).
 *  x_tgt_dev double[Nt][3], x_src_dev double[Ns][3], w_src_dev double[Ns][m],
 *  out_dev double[Nt][p] (all device).  KITC_SELF_OMIT requires x_tgt_dev ==
 *  x_src_dev and Nt == Ns (skip j == i); otherwise EINVAL. */
kitc_status kitc_direct(int32_t kernel, double eps, int32_t self, const double* x_tgt_dev,
                        int64_t Nt, const double* x_src_dev, const double* w_src_dev, int64_t Ns,
                        double* out_dev, void* s);

/* Direct sum at a SAMPLE of the sources as targets (the paper samples targets
 * at large N): target q is source idx_dev[q] (device int64[nt],
 * each in [0, Ns), not checked), self pair j == idx[q] skipped under
 * KITC_SELF_OMIT.  out_dev double[nt][p].  Other arguments as kitc_direct. */
kitc_status kitc_direct_sample(int32_t kernel, double eps, int32_t self, const int64_t* idx_dev, int64_t nt,
                               const double* x_src_dev, const double* w_src_dev, int64_t Ns, double* out_dev,
                               void* s);

/* Relative error E (Eq. error) of approx vs ref, both device
 * double[count] (rows of p components concatenated):
 *   E = ( sum_i (ref_i - approx_i)^2 / sum_i ref_i^2 )^(1/2).
 * scratch_dev: caller-owned device double[KITC_REL_ERROR_SCRATCH] (per-block
 * partial sums; no allocation inside).  Writes E to *E_host (synchronizes the
 * stream; the partials are added in long double on the host).  EINVAL if the
 * reference is identically zero, count < 1 or a pointer is NULL. */
#define KITC_REL_ERROR_SCRATCH 1184
kitc_status kitc_rel_error(const double* ref_dev, const double* approx_dev, int64_t count,
                           double* scratch_dev, double* E_host, void* s);

/* Free the handle and its device memory.  Waits for the device (cudaDeviceSynchronize)
 * first: calls on any stream may still be using the handle's buffers. */
void kitc_tree_free(kitc_tree* t);

/* Thread-local message for the last non-OK status ("" if none). */
const char* kitc_last_error(void);

/* Number of CUDA kernels this library has launched in the process so far
 * (monotone counter; bench.py reports the difference over the timed region). */
uint64_t kitc_launch_count(void);

/* Build flags of the loaded library: bit 0 (KITC_BUILD_CHECKS) = device-side invariant
 * checks compiled in (the verification build libkitc_checks.so: index bounds of the
 * traversal, TMA stages, scatter and weights work items; a violation traps and the next
 * synchronising call returns KITC_ECUDA).  0 for the product build. */
#define KITC_BUILD_CHECKS 1
uint32_t kitc_build_flags(void);

#ifdef __cplusplus
}
#endif
#endif /* KITC_H */
