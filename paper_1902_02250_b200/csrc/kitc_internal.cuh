// kitc_internal.cuh -- shared internals of libkitc.so (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

#include "../../include/kitc.h"

namespace kitc {

constexpr int kMaxDegree = 16;        // n in [1, 16]
constexpr int kMaxPeers = 8;          // fhat replicas written by one modified-weights call (GPUs per node)
constexpr int kMaxLevels = 4000;      // tree levels supported by the device build
#ifndef KITC_GROUP
#define KITC_GROUP 8
#endif
constexpr int kGroup = KITC_GROUP;    // lanes cooperating on one target in k_eval
constexpr int kBatch = 32 / kGroup;   // targets per warp batch
constexpr double kPi = 3.14159265358979323846;

// fhat layout (include/kitc.h): per cluster [r][k3][m][j], row = k1 P + k2 = kRows r + j.
constexpr int kRows = 8;  // rows per round block = lanes per target in k_eval
inline int fhat_rounds(int P) { return (P * P + kRows - 1) / kRows; }
inline long long fhat_cluster_len(int P, int M) { return (long long)fhat_rounds(P) * P * M * kRows; }

extern std::atomic<unsigned long long> g_launches;  // kernels launched by the library
inline void note_launch(unsigned long long n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ---- device-side invariant checks (verification builds: -DKITC_CHECKS) ------
// A violated index bound prints its location and traps; the next synchronising call
// reports KITC_ECUDA.  tests/test_gpu_checks.py runs the parity cases on such a build
// (compute-sanitizer is not available on the GPU pool).  Compiled out by default.
#ifdef KITC_CHECKS
#include <cstdio>
#define KITC_DCHECK(cond)                                                            \
    do {                                                                             \
        if (!(cond)) {                                                               \
            printf("KITC_CHECKS %s:%d: %s\n", __FILE__, __LINE__, #cond);            \
            __trap();                                                                \
        }                                                                            \
    } while (0)
#else
#define KITC_DCHECK(cond) \
    do {                  \
    } while (0)
#endif

// ---- error plumbing ---------------------------------------------------------
kitc_status set_error(kitc_status st, const std::string& msg);
kitc_status check_cuda(cudaError_t e, const char* what);
#define KITC_TRY(expr)                                   \
    do {                                                 \
        kitc_status _st = (expr);                        \
        if (_st != KITC_OK) return _st;                  \
    } while (0)
#define KITC_CUDA(expr) KITC_TRY(::kitc::check_cuda((expr), #expr))

// Stream-ordered device buffer, grown on demand, retained across rebuilds.  Memory
// comes from the handle's kitc_allocator (include/kitc.h) when it has one (the
// Python binding passes torch's caching allocator), else cudaMallocAsync from the
// device's default pool (its attributes are left untouched).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    const kitc_allocator* al = nullptr;  // the owning handle's provider (nullptr: cudaMallocAsync)
    kitc_status ensure(size_t need, cudaStream_t s, bool keep = false);
    void release(cudaStream_t s);
    template <class T> T* as() const { return static_cast<T*>(p); }
};

// Pinned host staging buffer.
struct HostBuf {
    void* p = nullptr;
    size_t bytes = 0;
    kitc_status ensure(size_t need);
    void release();
    template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace kitc

// The opaque handle.
struct kitc_tree {
    cudaStream_t stream = nullptr;  // stream of the last build (for frees)
    int64_t N = 0;
    int32_t N0 = 0;
    int32_t depth = 0;
    int32_t ndegenerate = 0;
    int64_t nclusters = 0;
    int64_t nleaves = 0;
    int64_t nbatches = 0;
    int64_t ccap = 0;                    // cluster-table capacity (grown if a build overflows it)
    bool built = false;

    // sorted particles (SoA)
    kitc::DevBuf x, y, z, perm;          // double x3, int32
    kitc::DevBuf x2, y2, z2, perm2;      // partition scratch
    kitc::DevBuf w;                      // sorted weights, m planes of N
    int32_t w_m = 0;
    kitc::DevBuf src;                    // packed near-field records (x, y, z, w.., pad), src_ld doubles each
    int32_t src_ld = 0;
    bool weights_ready = false;
    int32_t grid_n = -1;                 // degree of the stored grids
    int32_t weights_kernel = -1;

    // clusters (BFS order, capacity ccap)
    kitc::DevBuf box;     // double[C][6]  lo xyz, hi xyz
    kitc::DevBuf cr;      // double4[C]    centre xyz, r^2
    kitc::DevBuf topo;    // int4[C]       begin, end, first_child (-1: leaf), nchild
    kitc::DevBuf clevel;  // int[C]
    kitc::DevBuf cparent; // int[C]        (-1 for the root)
    kitc::DevBuf grid;    // double[C][3][n+1]
    kitc::DevBuf tord;    // int32[N] targets in Morton order inside each leaf (batching only)
    kitc::DevBuf leaves;  // int4[nleaves] begin, end, cluster id, first batch (range order)
    kitc::DevBuf bstart;  // int32[nbatches] first position (in tord) of the batch
    kitc::DevBuf bcount;  // int32[nbatches]

    // host mirrors of the topology, copied on demand (kitc_tree_export, kitc_batch_targets)
    mutable bool host_topo = false;
    mutable std::vector<int32_t> h_begin, h_end, h_level, h_parent, h_first, h_nchild;
    mutable std::vector<int32_t> h_leaf_begin;   // leaves in range order: first sorted position
    mutable std::vector<int64_t> h_leaf_boff;    // first batch of each leaf (+ total at the end)

    // device-build scratch (tree.cu) and its pinned counter block
    kitc::DevBuf b_split, b_pre, b_kids, b_tot8, b_bpart, b_cnt, b_sub, b_ctr;
    kitc::HostBuf h_ctr;
    // weights scratch: device-generated work items, per-chunk partial fhat
    kitc::DevBuf d_witems, d_wpart;
    // separate-target scratch (kitc_eval_targets): Morton keys / indices (double
    // buffers for the radix sort), sorted coordinates, cub temp, bounding box
    mutable kitc::DevBuf d_tkey, d_tkey2, d_tidx, d_tidx2, d_txyz, d_tcub, d_tbox;

    // device-memory provider (include/kitc.h kitc_allocator); alloc == NULL: cudaMallocAsync
    kitc_allocator allocator{};
    template <class F> void for_each_buf(F&& f) {
        for (kitc::DevBuf* b : {&x, &y, &z, &perm, &x2, &y2, &z2, &perm2, &w, &src, &box, &cr, &topo, &clevel,
                                &cparent, &grid, &tord, &leaves, &bstart, &bcount, &b_split, &b_pre, &b_kids,
                                &b_tot8, &b_bpart, &b_cnt, &b_sub, &b_ctr, &d_witems, &d_wpart, &d_tkey, &d_tkey2,
                                &d_tidx, &d_tidx2, &d_txyz, &d_tcub, &d_tbox})
            f(*b);
    }
};

namespace kitc {
// tree.cu
kitc_status build_tree(kitc_tree* t, const double* xyz, int64_t N, int32_t N0, cudaStream_t s);
kitc_status ensure_host_topology(const kitc_tree* t);
const int* tree_level_starts(const kitc_tree* t);  // device int[depth + 2]: first cluster of each level
int64_t tree_cluster_cap(int64_t N, int32_t N0);
size_t tree_bytes(int64_t N, int64_t ccap);
size_t dev_alloc_bytes(size_t need);  // what DevBuf::ensure requests for `need` bytes
// weights.cu
size_t weights_bytes(int64_t N, int64_t C, int32_t depth, int kernel, int n);
// weights.cu
kitc_status modified_weights(kitc_tree* t, int kernel, int n, const double* w, int64_t cb,
                             int64_t ce, double* const* fhat_peers, int npeers, cudaStream_t s, unsigned flags = 0);
// eval.cu
// A separate target set, Morton-sorted (targets.cu): coordinates SoA by sorted
// position, the original row of each, count.  Batches are kBatch consecutive
// sorted targets.
struct TargetSet {
    const double *x, *y, *z;
    const int* row;
    int64_t n;
};
kitc_status eval(const kitc_tree* t, int kernel, int n, double theta, double eps, int self,
                 const double* fhat, int64_t bb, int64_t be, double* out, uint64_t* stats,
                 cudaStream_t s, const TargetSet* ts = nullptr, unsigned flags = 0, int part = 0,
                 int nparts = 1);
// targets.cu
kitc_status eval_targets(const kitc_tree* t, int kernel, int n, double theta, double eps,
                         const double* fhat, const double* xt, int64_t Nt, double* out,
                         uint64_t* stats, cudaStream_t s, unsigned flags = 0);
// direct.cu
kitc_status direct(int kernel, double eps, int self, const double* xt, int64_t Nt,
                   const double* xs, const double* ws, int64_t Ns, double* out, cudaStream_t s,
                   const int64_t* tidx = nullptr);
kitc_status rel_error(const double* ref, const double* approx, int64_t count, double* scratch, double* E,
                      cudaStream_t s);
}  // namespace kitc
