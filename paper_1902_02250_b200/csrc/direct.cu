// direct.cu -- O(N^2) direct sum u(x_i) = sum_j k(x_i, y_j) f_j (Eq. N-body,
// P:42-67) and the relative error E (Eq. error), sm_100a fp64.
//
// Two targets per thread (two independent pair chains); sources are staged
// through shared memory in tiles of kTile (broadcast reads); each tile's
// contribution is summed into a tile partial that is then added to the running
// total (two-level summation keeps the rounding of N = 1e7 sums ~10x below the
// 1e-12 parity gate).  The self-pair test runs only in tiles that can hold it.
#include <algorithm>
#include <cmath>

#include "kitc_internal.cuh"
#include "pair.cuh"

namespace kitc {

namespace {

constexpr int kTile = 256;

#ifndef KITC_DIRECT_TPT
#define KITC_DIRECT_TPT 1  // measured at N = 1e6: 1 (55.2% of FP64 peak) ~ 3 > 2 > 4
#endif
constexpr int kTPT = KITC_DIRECT_TPT;  // targets per thread (independent pair chains per source)

// The source tile's contribution to one target; SELF: the tile may hold the
// target's own source `si` -- that pair is evaluated with f = 0, s = 1 (an exact
// zero), otherwise no per-pair test at all.
template <int KER, bool SELF>
__device__ __forceinline__ void tile_pairs(const double* x, const double* y, const double* z, const long long* si,
                                           int tile, int cnt, const double* sx, const double* sy, const double* sz,
                                           const double (*sw)[kTile], double (*part)[Kern<KER>::P],
                                           const KParams& kp) {
    using K = Kern<KER>;
    constexpr int M = K::M;
    for (int jj = 0; jj < cnt; ++jj) {
        double f[M];
#pragma unroll
        for (int m = 0; m < M; ++m) f[m] = sw[m][jj];
        const double xj = sx[jj], yj = sy[jj], zj = sz[jj];
#pragma unroll
        for (int q = 0; q < kTPT; ++q) {
            const double dx = x[q] - xj, dy = y[q] - yj, dz = z[q] - zj;
            const bool me = SELF && (tile + jj == si[q]);
            double g[M];
#pragma unroll
            for (int m = 0; m < M; ++m) g[m] = me ? 0.0 : f[m];
            const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, kp.e2)));
            K::pair(dx, dy, dz, s, g, part[q], kp);
        }
    }
}

// tidx (optional): target q is source tidx[q] (sampled targets; its self pair is
// the one skipped under SELF_OMIT); otherwise target q is xt[q] (self = q).
// Each thread owns kTPT targets (i, i + kTile); summation order per target is
// sources ascending within a tile, tiles ascending (two-level).
template <int KER>
__global__ void __launch_bounds__(kTile) k_direct(const double* __restrict__ xt, int Nt,
                                                  const long long* __restrict__ tidx,
                                                  const double* __restrict__ xs,
                                                  const double* __restrict__ ws, int Ns,
                                                  double* __restrict__ out, KParams kp, int self_omit) {
    using K = Kern<KER>;
    constexpr int M = K::M, NP = K::P;
    __shared__ double sx[kTile], sy[kTile], sz[kTile], sw[M][kTile];
    double x[kTPT], y[kTPT], z[kTPT];
    long long si[kTPT];
    int ii[kTPT];
#pragma unroll
    for (int q = 0; q < kTPT; ++q) {
        ii[q] = blockIdx.x * (kTPT * kTile) + q * kTile + threadIdx.x;
        si[q] = self_omit ? ii[q] : -1;
        x[q] = y[q] = z[q] = 0.0;
        if (ii[q] < Nt) {
            const double* p = tidx ? xs + 3 * tidx[ii[q]] : xt + 3 * (size_t)ii[q];
            if (tidx && self_omit) si[q] = tidx[ii[q]];
            x[q] = p[0];
            y[q] = p[1];
            z[q] = p[2];
        } else {
            si[q] = -1;
        }
    }
    double tot[kTPT][NP];
#pragma unroll
    for (int q = 0; q < kTPT; ++q)
#pragma unroll
        for (int c = 0; c < NP; ++c) tot[q][c] = 0.0;
    for (int tile = 0; tile < Ns; tile += kTile) {
        const int j = tile + threadIdx.x;
        if (j < Ns) {
            sx[threadIdx.x] = xs[3 * (size_t)j];
            sy[threadIdx.x] = xs[3 * (size_t)j + 1];
            sz[threadIdx.x] = xs[3 * (size_t)j + 2];
#pragma unroll
            for (int m = 0; m < M; ++m) sw[m][threadIdx.x] = ws[(size_t)j * M + m];
        }
        __syncthreads();
        const int cnt = min(kTile, Ns - tile);
        double part[kTPT][NP];
#pragma unroll
        for (int q = 0; q < kTPT; ++q)
#pragma unroll
            for (int c = 0; c < NP; ++c) part[q][c] = 0.0;
        bool mine = false;
#pragma unroll
        for (int q = 0; q < kTPT; ++q) mine |= si[q] >= tile && si[q] < tile + cnt;
        if (__any_sync(0xffffffffu, mine))  // warp-uniform: some lane's own source is in this tile
            tile_pairs<KER, true>(x, y, z, si, tile, cnt, sx, sy, sz, sw, part, kp);
        else
            tile_pairs<KER, false>(x, y, z, si, tile, cnt, sx, sy, sz, sw, part, kp);
#pragma unroll
        for (int q = 0; q < kTPT; ++q)
#pragma unroll
            for (int c = 0; c < NP; ++c) tot[q][c] += part[q][c];
        __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < kTPT; ++q)
        if (ii[q] < Nt)
#pragma unroll
            for (int c = 0; c < NP; ++c) out[(size_t)ii[q] * NP + c] = tot[q][c] * K::scale(c);
}

constexpr int kErrBlocks = 592;  // 4 x 148 SMs; fixed -> deterministic

__global__ void __launch_bounds__(256) k_relerr(const double* __restrict__ ref, const double* __restrict__ ap,
                                                long long n, double* __restrict__ part) {
    double num = 0.0, den = 0.0;
    for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += (long long)kErrBlocks * 256) {
        const double r = ref[i], d = r - ap[i];
        num = fma(d, d, num);
        den = fma(r, r, den);
    }
    __shared__ double sn[256], sd[256];
    sn[threadIdx.x] = num;
    sd[threadIdx.x] = den;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) {
            sn[threadIdx.x] += sn[threadIdx.x + o];
            sd[threadIdx.x] += sd[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[2 * blockIdx.x] = sn[0];
        part[2 * blockIdx.x + 1] = sd[0];
    }
}

}  // namespace

kitc_status direct(int kernel, double eps, int self, const double* xt, int64_t Nt, const double* xs,
                   const double* ws, int64_t Ns, double* out, cudaStream_t s, const int64_t* tidx) {
    if (Nt < 0 || Ns < 0 || Nt > 0x7fffffffLL || Ns > 0x7fffffffLL)
        return set_error(KITC_EINVAL, "kitc_direct: size out of range");
    if (!(eps >= 0.0) || !std::isfinite(eps)) return set_error(KITC_EINVAL, "kitc_direct: eps must be >= 0");
    if (self != KITC_SELF_OMIT && self != KITC_SELF_INCLUDE) return set_error(KITC_EINVAL, "kitc_direct: bad self");
    if (tidx) xt = xs;  // sampled targets: validated by the caller (indices in [0, Ns))
    if (self == KITC_SELF_OMIT && !tidx && (xt != xs || Nt != Ns))
        return set_error(KITC_EINVAL, "kitc_direct: KITC_SELF_OMIT needs targets == sources");
    if (eps == 0.0 && self != KITC_SELF_OMIT)
        return set_error(KITC_EINVAL, "kitc_direct: eps = 0 requires KITC_SELF_OMIT");
    if (Nt == 0) return KITC_OK;
    if (!xt || !out || (Ns > 0 && (!xs || !ws))) return set_error(KITC_EINVAL, "kitc_direct: NULL buffer");
    const KParams kp = make_kparams(eps);
    const int grid = (int)((Nt + kTPT * kTile - 1) / (kTPT * kTile));
    const int so = self == KITC_SELF_OMIT;
    switch (kernel) {
        case KITC_STOKESLET: k_direct<0><<<grid, kTile, 0, s>>>(xt, (int)Nt, reinterpret_cast<const long long*>(tidx), xs, ws, (int)Ns, out, kp, so); note_launch(); break;
        case KITC_ROTLET: k_direct<1><<<grid, kTile, 0, s>>>(xt, (int)Nt, reinterpret_cast<const long long*>(tidx), xs, ws, (int)Ns, out, kp, so); note_launch(); break;
        case KITC_STOKESLET_ROTLET: k_direct<2><<<grid, kTile, 0, s>>>(xt, (int)Nt, reinterpret_cast<const long long*>(tidx), xs, ws, (int)Ns, out, kp, so); note_launch(); break;
        default: return set_error(KITC_EINVAL, "kitc_direct: unknown kernel");
    }
    KITC_CUDA(cudaGetLastError());
    return KITC_OK;
}

static_assert(2 * kErrBlocks == KITC_REL_ERROR_SCRATCH, "include/kitc.h KITC_REL_ERROR_SCRATCH");

kitc_status rel_error(const double* ref, const double* ap, int64_t n, double* part, double* E, cudaStream_t s) {
    if (!ref || !ap || !E || n < 1) return set_error(KITC_EINVAL, "kitc_rel_error: bad arguments");
    if (!part) return set_error(KITC_EINVAL, "kitc_rel_error: NULL scratch");
    k_relerr<<<kErrBlocks, 256, 0, s>>>(ref, ap, n, part); note_launch();
    KITC_CUDA(cudaGetLastError());
    std::vector<double> h(2 * kErrBlocks);
    KITC_CUDA(cudaMemcpyAsync(h.data(), part, h.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    KITC_CUDA(cudaStreamSynchronize(s));
    long double num = 0.0L, den = 0.0L;
    for (int b = 0; b < kErrBlocks; ++b) {
        num += h[2 * b];
        den += h[2 * b + 1];
    }
    if (den == 0.0L) return set_error(KITC_EINVAL, "kitc_rel_error: reference is identically zero");
    *E = (double)sqrtl(num / den);
    return KITC_OK;
}

}  // namespace kitc
