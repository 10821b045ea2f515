// targets.cu -- treecode evaluation at a SEPARATE target set (the
// targets need not be the sources).
//
// The targets are ordered along a Morton curve of their own bounding box so
// that the kBatch targets of a warp batch are spatially compact (they then
// agree on most MAC decisions, as the in-leaf Morton batches of the sources do):
//   k_tbox     bounding box (order-preserving integer min/max atomics)
//   k_tmorton  63-bit Morton key per target (21 bits per axis)
//   cub radix sort of (key, index)
//   k_tgather  sorted SoA coordinates + original row of every sorted target
// then k_eval runs with batches of kBatch consecutive sorted targets and no
// self term.  Which batch a target lands in does not change its result.
#include <cub/cub.cuh>

#include "kitc_internal.cuh"

namespace kitc {

namespace {

__device__ __forceinline__ unsigned long long ord_key(double v) {
    const unsigned long long b = static_cast<unsigned long long>(__double_as_longlong(v));
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double ord_val(unsigned long long k) {
    const unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
    return __longlong_as_double(static_cast<long long>(b));
}

// box[0..2] = min keys (init all ones), box[3..5] = max keys (init 0)
__global__ void k_tbox(const double* __restrict__ xt, long long n, unsigned long long* box) {
    unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < n; q += (long long)gridDim.x * blockDim.x)
        for (int l = 0; l < 3; ++l) {
            const unsigned long long k = ord_key(xt[3 * q + l]);
            lo[l] = min(lo[l], k);
            hi[l] = max(hi[l], k);
        }
    for (int l = 0; l < 3; ++l)
        for (int o = 16; o > 0; o >>= 1) {
            lo[l] = min(lo[l], __shfl_xor_sync(0xffffffffu, lo[l], o));
            hi[l] = max(hi[l], __shfl_xor_sync(0xffffffffu, hi[l], o));
        }
    if ((threadIdx.x & 31) == 0)
        for (int l = 0; l < 3; ++l) {
            atomicMin(box + l, lo[l]);
            atomicMax(box + 3 + l, hi[l]);
        }
}

__device__ __forceinline__ unsigned long long spread21(unsigned long long v) {
    v &= 0x1fffffull;
    v = (v | v << 32) & 0x1f00000000ffffull;
    v = (v | v << 16) & 0x1f0000ff0000ffull;
    v = (v | v << 8) & 0x100f00f00f00f00full;
    v = (v | v << 4) & 0x10c30c30c30c30c3ull;
    v = (v | v << 2) & 0x1249249249249249ull;
    return v;
}

__global__ void k_tmorton(const double* __restrict__ xt, long long n, const unsigned long long* __restrict__ box,
                          unsigned long long* __restrict__ key, int* __restrict__ idx) {
    const long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (q >= n) return;
    unsigned long long k = 0;
    for (int l = 0; l < 3; ++l) {
        const double lo = ord_val(box[l]), hi = ord_val(box[3 + l]);
        const double ext = hi - lo;
        double u = ext > 0.0 ? (xt[3 * q + l] - lo) / ext : 0.0;  // [0, 1]; NaN -> 0 below
        u = u >= 0.0 ? (u <= 1.0 ? u : 1.0) : 0.0;
        k |= spread21(static_cast<unsigned long long>(u * 2097151.0)) << l;
    }
    key[q] = k;
    idx[q] = (int)q;
}

__global__ void k_tgather(const double* __restrict__ xt, long long n, const int* __restrict__ idx,
                          double* __restrict__ tx, double* __restrict__ ty, double* __restrict__ tz) {
    const long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (i >= n) return;
    const long long q = idx[i];
    tx[i] = xt[3 * q];
    ty[i] = xt[3 * q + 1];
    tz[i] = xt[3 * q + 2];
}

}  // namespace

kitc_status eval_targets(const kitc_tree* t, int kernel, int n, double theta, double eps, const double* fhat,
                         const double* xt, int64_t Nt, double* out, uint64_t* stats, cudaStream_t s,
                         unsigned flags) {
    if (!t->built) return set_error(KITC_ESTATE, "kitc_eval_targets: tree not built");
    if (Nt < 0 || Nt > 0x7fffffffLL) return set_error(KITC_EINVAL, "kitc_eval_targets: Nt out of range");
    if (Nt == 0) return KITC_OK;
    if (!xt || !out) return set_error(KITC_EINVAL, "kitc_eval_targets: NULL buffer");
    const size_t n8 = (size_t)Nt * 8, n4 = (size_t)Nt * 4;
    KITC_TRY(t->d_tkey.ensure(n8, s));
    KITC_TRY(t->d_tkey2.ensure(n8, s));
    KITC_TRY(t->d_tidx.ensure(n4, s));
    KITC_TRY(t->d_tidx2.ensure(n4, s));
    KITC_TRY(t->d_txyz.ensure(3 * n8, s));
    KITC_TRY(t->d_tbox.ensure(6 * sizeof(unsigned long long), s));
    unsigned long long* box = t->d_tbox.as<unsigned long long>();
    KITC_CUDA(cudaMemsetAsync(box, 0xff, 3 * sizeof(unsigned long long), s));
    KITC_CUDA(cudaMemsetAsync(box + 3, 0, 3 * sizeof(unsigned long long), s));
    const int nb = (int)std::min<int64_t>((Nt + 255) / 256, 148 * 8);
    k_tbox<<<nb, 256, 0, s>>>(xt, Nt, box); note_launch();
    const int g = (int)((Nt + 255) / 256);
    k_tmorton<<<g, 256, 0, s>>>(xt, Nt, box, t->d_tkey.as<unsigned long long>(), t->d_tidx.as<int>()); note_launch();
    cub::DoubleBuffer<unsigned long long> keys(t->d_tkey.as<unsigned long long>(), t->d_tkey2.as<unsigned long long>());
    cub::DoubleBuffer<int> vals(t->d_tidx.as<int>(), t->d_tidx2.as<int>());
    size_t tmp = 0;
    KITC_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, tmp, keys, vals, (int)Nt, 0, 63, s));
    KITC_TRY(t->d_tcub.ensure(tmp, s));
    KITC_CUDA(cub::DeviceRadixSort::SortPairs(t->d_tcub.p, tmp, keys, vals, (int)Nt, 0, 63, s));
    // (the radix sort's CUB kernels are library code: not counted by note_launch)
    double* txyz = t->d_txyz.as<double>();
    k_tgather<<<g, 256, 0, s>>>(xt, Nt, vals.Current(), txyz, txyz + Nt, txyz + 2 * Nt); note_launch();
    KITC_CUDA(cudaGetLastError());
    TargetSet ts{txyz, txyz + Nt, txyz + 2 * Nt, vals.Current(), Nt};
    return eval(t, kernel, n, theta, eps, KITC_SELF_INCLUDE, fhat, 0, (Nt + kBatch - 1) / kBatch, out, stats, s, &ts,
                flags);
}

}  // namespace kitc
