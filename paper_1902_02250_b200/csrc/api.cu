#include <algorithm>
// api.cu -- the extern "C" entry points of libkitc.so (include/kitc.h).
// Argument checks + exception barrier; the work is in tree.cu, weights.cu,
// eval.cu and direct.cu.
#include <new>

#include "kitc_internal.cuh"

using namespace kitc;

#define KITC_GUARD(...)                                                        \
    try {                                                                       \
        __VA_ARGS__                                                                 \
    } catch (const std::bad_alloc&) {                                           \
        return set_error(KITC_ENOMEM, "host allocation failed");                \
    } catch (...) {                                                             \
        return set_error(KITC_ECUDA, "unexpected C++ exception");               \
    }

extern "C" {

kitc_status kitc_fhat_cluster_len(int32_t kernel, int32_t n, int64_t* len) {
    int32_t m = 0;
    KITC_TRY(kitc_kernel_dims(kernel, &m, nullptr));
    if (n < 1 || n > kitc::kMaxDegree) return kitc::set_error(KITC_EINVAL, "kitc_fhat_cluster_len: n must be in [1, 16]");
    if (len) *len = kitc::fhat_cluster_len(n + 1, m);
    return KITC_OK;
}

kitc_status kitc_kernel_dims(int32_t kernel, int32_t* m, int32_t* p) {
    int mm, pp;
    switch (kernel) {
        case KITC_STOKESLET: mm = 3; pp = 3; break;
        case KITC_ROTLET: mm = 3; pp = 6; break;
        case KITC_STOKESLET_ROTLET: mm = 6; pp = 6; break;
        default: return set_error(KITC_EINVAL, "unknown kernel");
    }
    if (m) *m = mm;
    if (p) *p = pp;
    return KITC_OK;
}

kitc_status kitc_tree_create(kitc_tree** out) { return kitc_tree_create_with_allocator(nullptr, out); }

kitc_status kitc_tree_create_with_allocator(const kitc_allocator* a, kitc_tree** out) {
    if (!out) return set_error(KITC_EINVAL, "kitc_tree_create: out is NULL");
    *out = nullptr;
    if (a && (!a->alloc || !a->release))
        return set_error(KITC_EINVAL, "kitc_tree_create_with_allocator: alloc and release are both required");
    KITC_GUARD({
        kitc_tree* t = new kitc_tree();
        if (a) t->allocator = *a;
        t->for_each_buf([t](DevBuf& b) { b.al = &t->allocator; });
        *out = t;
        return KITC_OK;
    })
}

kitc_status kitc_tree_workspace_bytes(int64_t N, int32_t N0, int32_t kernel, int32_t n, size_t* bytes) {
    if (!bytes) return set_error(KITC_EINVAL, "kitc_tree_workspace_bytes: bytes is NULL");
    if (N < 1 || N > 0x3fffffffLL || N0 < 1) return set_error(KITC_EINVAL, "kitc_tree_workspace_bytes: bad N or N0");
    int32_t m = 0;
    KITC_TRY(kitc_kernel_dims(kernel, &m, nullptr));
    if (n < 1 || n > kitc::kMaxDegree) return set_error(KITC_EINVAL, "kitc_tree_workspace_bytes: n must be in [1, 16]");
    // worst case: C <= 2N - 1 clusters (every internal cluster has >= 2 children, every
    // leaf >= 1 particle), depth < min(N, kMaxLevels)
    const int64_t C = 2 * N - 1;
    const int32_t depth = (int32_t)std::min<int64_t>(N, kitc::kMaxLevels);
    *bytes = tree_bytes(N, C) + weights_bytes(N, C, depth, kernel, n);
    return KITC_OK;
}

kitc_status kitc_build_tree(kitc_tree* t, const double* xyz, int64_t N, int32_t N0, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_build_tree: NULL handle");
    KITC_GUARD(return build_tree(t, xyz, N, N0, (cudaStream_t)s);)
}

kitc_status kitc_tree_info(const kitc_tree* t, int64_t* nc, int32_t* depth, int64_t* nb, int32_t* ndeg) {
    if (!t) return set_error(KITC_EINVAL, "kitc_tree_info: NULL handle");
    if (!t->built) return set_error(KITC_ESTATE, "kitc_tree_info: tree not built");
    if (nc) *nc = t->nclusters;
    if (depth) *depth = t->depth;
    if (nb) *nb = t->nbatches;
    if (ndeg) *ndeg = t->ndegenerate;
    return KITC_OK;
}

kitc_status kitc_tree_export(const kitc_tree* t, int64_t* perm, int64_t* begin, int64_t* end, int32_t* level,
                             int32_t* parent, int32_t* first_child, int32_t* nchild, double* lo, double* hi) {
    if (!t) return set_error(KITC_EINVAL, "kitc_tree_export: NULL handle");
    if (!t->built) return set_error(KITC_ESTATE, "kitc_tree_export: tree not built");
    KITC_GUARD({
        cudaStream_t s = t->stream;
        const int64_t C = t->nclusters, N = t->N;
        KITC_TRY(ensure_host_topology(t));
        if (perm) {
            std::vector<int> p(N);
            KITC_CUDA(cudaMemcpyAsync(p.data(), t->perm.p, N * sizeof(int), cudaMemcpyDeviceToHost, s));
            KITC_CUDA(cudaStreamSynchronize(s));
            for (int64_t i = 0; i < N; ++i) perm[i] = p[i];
        }
        if (lo || hi) {
            std::vector<double> b(C * 6);
            KITC_CUDA(cudaMemcpyAsync(b.data(), t->box.p, C * 6 * sizeof(double), cudaMemcpyDeviceToHost, s));
            KITC_CUDA(cudaStreamSynchronize(s));
            for (int64_t c = 0; c < C; ++c)
                for (int l = 0; l < 3; ++l) {
                    if (lo) lo[c * 3 + l] = b[c * 6 + l];
                    if (hi) hi[c * 3 + l] = b[c * 6 + 3 + l];
                }
        }
        for (int64_t c = 0; c < C; ++c) {
            if (begin) begin[c] = t->h_begin[c];
            if (end) end[c] = t->h_end[c];
            if (level) level[c] = t->h_level[c];
            if (parent) parent[c] = t->h_parent[c];
            if (first_child) first_child[c] = t->h_first[c];
            if (nchild) nchild[c] = t->h_nchild[c];
        }
        return KITC_OK;
    })
}

kitc_status kitc_modified_weights(kitc_tree* t, int32_t kernel, int32_t n, const double* w, int64_t cb,
                                  int64_t ce, double* fhat, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_modified_weights: NULL handle");
    KITC_GUARD(return modified_weights(t, kernel, n, w, cb, ce, &fhat, 1, (cudaStream_t)s);)
}

kitc_status kitc_modified_weights_ex(kitc_tree* t, int32_t kernel, int32_t n, const double* w, int64_t cb,
                                     int64_t ce, uint32_t flags, double* fhat, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_modified_weights_ex: NULL handle");
    KITC_GUARD(return modified_weights(t, kernel, n, w, cb, ce, &fhat, 1, (cudaStream_t)s, flags);)
}

kitc_status kitc_modified_weights_peers(kitc_tree* t, int32_t kernel, int32_t n, const double* w, int64_t cb,
                                        int64_t ce, double* const* fhat_peers, int32_t npeers, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_modified_weights_peers: NULL handle");
    if (!fhat_peers) return set_error(KITC_EINVAL, "kitc_modified_weights_peers: NULL peer array");
    KITC_GUARD(return modified_weights(t, kernel, n, w, cb, ce, fhat_peers, npeers, (cudaStream_t)s);)
}

kitc_status kitc_eval(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                      int32_t self, const double* fhat, int64_t bb, int64_t be, double* out, uint64_t* stats,
                      void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_eval: NULL handle");
    if (t->built && N0 != t->N0) return set_error(KITC_EINVAL, "kitc_eval: N0 differs from the tree's N0");
    KITC_GUARD(return eval(t, kernel, n, theta, eps, self, fhat, bb, be, out, stats, (cudaStream_t)s);)
}

kitc_status kitc_eval_part(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                           int32_t self, uint32_t flags, const double* fhat, int32_t part, int32_t nparts,
                           double* out, uint64_t* stats, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_eval_part: NULL handle");
    if (t->built && N0 != t->N0) return set_error(KITC_EINVAL, "kitc_eval_part: N0 differs from the tree's N0");
    KITC_GUARD(return eval(t, kernel, n, theta, eps, self, fhat, 0, t->nbatches, out, stats, (cudaStream_t)s,
                           nullptr, flags, part, nparts);)
}

kitc_status kitc_eval_ex(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                         int32_t self, uint32_t flags, const double* fhat, int64_t bb, int64_t be, double* out,
                         uint64_t* stats, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_eval_ex: NULL handle");
    if (t->built && N0 != t->N0) return set_error(KITC_EINVAL, "kitc_eval_ex: N0 differs from the tree's N0");
    KITC_GUARD(return eval(t, kernel, n, theta, eps, self, fhat, bb, be, out, stats, (cudaStream_t)s, nullptr,
                           flags);)
}

kitc_status kitc_eval_targets(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0, double eps,
                              const double* fhat, const double* xt, int64_t Nt, double* out, uint64_t* stats,
                              void* s) {
    return kitc_eval_targets_ex(t, kernel, n, theta, N0, eps, 0u, fhat, xt, Nt, out, stats, s);
}

kitc_status kitc_eval_targets_ex(const kitc_tree* t, int32_t kernel, int32_t n, double theta, int32_t N0,
                                 double eps, uint32_t flags, const double* fhat, const double* xt, int64_t Nt,
                                 double* out, uint64_t* stats, void* s) {
    if (!t) return set_error(KITC_EINVAL, "kitc_eval_targets: NULL handle");
    if (t->built && N0 != t->N0) return set_error(KITC_EINVAL, "kitc_eval_targets: N0 differs from the tree's N0");
    KITC_GUARD(return eval_targets(t, kernel, n, theta, eps, fhat, xt, Nt, out, stats, (cudaStream_t)s, flags);)
}

kitc_status kitc_batch_targets(const kitc_tree* t, int64_t be, int64_t* nt) {
    if (!t || !nt) return set_error(KITC_EINVAL, "kitc_batch_targets: NULL argument");
    if (!t->built) return set_error(KITC_ESTATE, "kitc_batch_targets: tree not built");
    if (be < 0 || be > t->nbatches) return set_error(KITC_EINVAL, "kitc_batch_targets: bad batch index");
    KITC_TRY(ensure_host_topology(t));
    // batches tile the sorted positions leaf by leaf: batch b of leaf l starts at
    // leaf_begin_l + kBatch (b - boff_l), and that is the number of targets before it
    const auto& bo = t->h_leaf_boff;
    if (be == t->nbatches) {
        *nt = t->N;
        return KITC_OK;
    }
    const size_t l = (size_t)(std::upper_bound(bo.begin(), bo.end() - 1, be) - bo.begin()) - 1;
    *nt = t->h_leaf_begin[l] + (int64_t)kBatch * (be - bo[l]);
    return KITC_OK;
}

kitc_status kitc_direct(int32_t kernel, double eps, int32_t self, const double* xt, int64_t Nt, const double* xs,
                        const double* ws, int64_t Ns, double* out, void* s) {
    KITC_GUARD(return direct(kernel, eps, self, xt, Nt, xs, ws, Ns, out, (cudaStream_t)s);)
}

kitc_status kitc_direct_sample(int32_t kernel, double eps, int32_t self, const int64_t* idx, int64_t nt,
                               const double* xs, const double* ws, int64_t Ns, double* out, void* s) {
    if (nt > 0 && !idx) return set_error(KITC_EINVAL, "kitc_direct_sample: NULL index array");
    KITC_GUARD(return direct(kernel, eps, self, xs, nt, xs, ws, Ns, out, (cudaStream_t)s, idx);)
}

kitc_status kitc_rel_error(const double* ref, const double* ap, int64_t n, double* scratch, double* E, void* s) {
    KITC_GUARD(return rel_error(ref, ap, n, scratch, E, (cudaStream_t)s);)
}

void kitc_tree_free(kitc_tree* t) {
    if (!t) return;
    // calls on other streams may still use the handle's buffers: wait for the whole
    // device before releasing them (freeing is rare; correctness over latency)
    cudaDeviceSynchronize();
    cudaStream_t s = t->stream;
    t->for_each_buf([s](DevBuf& b) { b.release(s); });
    t->h_ctr.release();
    delete t;
}

}  // extern "C"
