// eval.cu -- treecode evaluation (Algorithm 2 lines 7-17) on sm_100a.
//
// One warp = one batch of <= kBatch targets of one leaf, consecutive in the
// leaf's Morton order (spatially compact); kGroup lanes cooperate on each
// target (they split its proxies / sources and combine at the end).  The warp walks the tree depth-first with an explicit
// shared-memory stack of (cluster, lane mask) entries, so every lane keeps the
// paper's PER-TARGET semantics: a lane stops descending below a cluster it
// accepted; lanes that reject a cluster descend into its children.  At each
// popped cluster:
//   MAC   r^2 <= (theta^2) R^2, R^2 > 0   (RN intrinsics, no FMA; readings A4/A5)
//   far   accepted lanes sum the kernel against the (n+1)^3 proxies s_k with the
//         modified weights fhat_k (Eq. pc_approximation_3D);
//         uniform (broadcast) loads of fhat, tensor-product reuse of dx, dy, dz
//   near  rejecting lanes at a leaf sum over its particles directly
//         (Eq. pc_interaction_3D), j == i skipped by index (reading A8)
//   else  rejecting lanes push the children.
// Outputs are scaled once and scattered to original order (out[perm[t]]).
#include <algorithm>

#include "kitc_internal.cuh"
#include "pair.cuh"

namespace kitc {

namespace {

#ifndef KITC_EVAL_WARPS
#define KITC_EVAL_WARPS 4
#endif
#ifndef KITC_EVAL_MINB
#define KITC_EVAL_MINB 6  // resident CTAs per SM (register budget), Stokeslet
#endif
#ifndef KITC_EVAL_MINB1
#define KITC_EVAL_MINB1 4  // rotlet / combined (measured: 4 beats 5 and 6 on C4)
#endif
#ifndef KITC_EVAL_PREFETCH
#define KITC_EVAL_PREFETCH 0  // bit 0: far-field rows, bit 1: near-field sources
#endif
constexpr int kWarps = KITC_EVAL_WARPS;  // warps (batches) per CTA

// L1 prefetch of one line (the next round's fhat rows / near-field sources, so
// the loads of that round hit L1 instead of waiting on L2).
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

struct EvalArgs {
    const double* x;
    const double* y;
    const double* z;
    const int* perm;
    const int* tord;
    const double* w;  // sorted weights, M planes of N
    const double4* cr;
    const int4* topo;
    const double* grid;
    const double* fhat;
    const int* bstart;
    const int* bcount;
    double* out;
    unsigned long long* stats;
    long long bb, be;
    int N;
    int P;  // n + 1 (runtime copy)
    int stack_cap;
    int self_omit;
    double tt;  // theta * theta (RN)
    KParams kp;
};

// Far field of one accepted cluster for the lanes of one target group: lane
// group g (of kGroup) sums rows (k1, k2) = g, g + kGroup, ... of the (n+1)^2
// rows, all k3 per row (dx, dy, dx^2 + dy^2 per row and dz, dz^2 + eps^2 per
// plane are reused; Kern::pair_row folds the terms linear in d along the row);
// the rows left after the last full round are split pair by pair over the
// groups.  F layout: F[k3][m][row], row = k1 (n+1) + k2 (weights.cu).
template <int PT, int KER>
__device__ __forceinline__ void far_field(double x, double y, double z, const double* __restrict__ g,
                                          const double* __restrict__ F, double* acc, const KParams& kp, int Prt,
                                          int grp) {
    using K = EvalKern<KER>;
    constexpr int M = K::M;
    const int P = PT > 0 ? PT : Prt, P2 = P * P;
    const int full = (P2 / kGroup) * kGroup;
    if constexpr (PT > 0) {
        double dz[PT];
#pragma unroll
        for (int k3 = 0; k3 < PT; ++k3) dz[k3] = z - __ldg(g + 2 * PT + k3);
        // the next row's grid coordinates are loaded one row ahead
        double gx = 0.0, gy = 0.0;
        if (grp < full) {
            gx = __ldg(g + grp / PT);
            gy = __ldg(g + PT + grp % PT);
        }
        for (int row = grp; row < full; row += kGroup) {
            const double dx = x - gx;
            const double dy = y - gy;
            const int nrow = row + kGroup;
            if (nrow < full) {
                gx = __ldg(g + nrow / PT);
                gy = __ldg(g + PT + nrow % PT);
                if (KITC_EVAL_PREFETCH & 1) {
                    // the next round's kGroup rows of the P * M planes: 64 B each
                    const double* nb = F + (nrow - grp);
#pragma unroll
                    for (int q = grp; q < PT * M; q += kGroup) prefetch_l1(nb + q * P2);
                }
            }
            const double pxye = fma(dy, dy, dx * dx) + kp.e2;
            typename K::Row r;
#pragma unroll
            for (int k3 = 0; k3 < PT; ++k3) {
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = __ldg(F + (k3 * M + m) * P2 + row);
                K::pair_row(dx, dy, dz[k3], fma(dz[k3], dz[k3], pxye), f, acc, r, kp);
            }
            K::row_end(dx, dy, r, acc);
        }
    } else {
        for (int row = grp; row < full; row += kGroup) {
            const int k1 = row / P, k2 = row - k1 * P;
            const double dx = x - __ldg(g + k1);
            const double dy = y - __ldg(g + P + k2);
            const double pxye = fma(dy, dy, dx * dx) + kp.e2;
            typename K::Row r;
            for (int k3 = 0; k3 < P; ++k3) {
                const double dz = z - __ldg(g + 2 * P + k3);
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = __ldg(F + (k3 * M + m) * P2 + row);
                K::pair_row(dx, dy, dz, fma(dz, dz, pxye), f, acc, r, kp);
            }
            K::row_end(dx, dy, r, acc);
        }
    }
    const int rem = (P2 - full) * P;  // pairs of the leftover rows
    for (int q = grp; q < rem; q += kGroup) {
        const int row = full + q / P, k3 = q - (q / P) * P;
        const int k1 = row / P, k2 = row - k1 * P;
        const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2), dz = z - __ldg(g + 2 * P + k3);
        double f[M];
#pragma unroll
        for (int m = 0; m < M; ++m) f[m] = __ldg(F + (k3 * M + m) * P2 + row);
        K::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, acc, kp);
    }
}

// Near field of one rejected leaf: lane group g sums sources b + g, b + g + kGroup, ...
// (unrolled x4 with the loads hoisted).
template <int KER>
__device__ __forceinline__ void near_field(double x, double y, double z, int t, int b, int e, int grp,
                                           const EvalArgs& a, double* acc) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, U = 4;
    // The self pair (j == t under SELF_OMIT) is evaluated with f = 0 and s = 1:
    // its contribution is exactly zero, so the loop stays branch-free.
    const int self = a.self_omit ? t : -1;
    int j = b + grp;
    for (; j + (U - 1) * kGroup < e; j += U * kGroup) {
        if (KITC_EVAL_PREFETCH & 2) {
            // next iteration's U * kGroup sources: 2 lines of 128 B in each of 3 + M arrays
            const int nj = j - grp + U * kGroup + 16 * (grp & 1);
            const int arr = grp >> 1;  // 0..3
            const double* base = arr == 0 ? a.x : arr == 1 ? a.y : arr == 2 ? a.z : a.w;
            if (nj < e) {
                prefetch_l1(base + nj);
                if (arr == 3)
                    for (int m = 1; m < M; ++m) prefetch_l1(a.w + (size_t)m * a.N + nj);
            }
        }
        double sx[U], sy[U], sz[U], f[U][M];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = j + u * kGroup;
            sx[u] = __ldg(a.x + jj);
            sy[u] = __ldg(a.y + jj);
            sz[u] = __ldg(a.z + jj);
#pragma unroll
            for (int m = 0; m < M; ++m) f[u][m] = __ldg(a.w + (size_t)m * a.N + jj);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool me = (j + u * kGroup) == self;
            const double dx = x - sx[u], dy = y - sy[u], dz = z - sz[u];
#pragma unroll
            for (int m = 0; m < M; ++m) f[u][m] = me ? 0.0 : f[u][m];
            const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
            K::pair(dx, dy, dz, s, f[u], acc, a.kp);
        }
    }
    for (; j < e; j += kGroup) {
        const bool me = j == self;
        const double dx = x - __ldg(a.x + j), dy = y - __ldg(a.y + j), dz = z - __ldg(a.z + j);
        double f[M];
#pragma unroll
        for (int m = 0; m < M; ++m) f[m] = me ? 0.0 : __ldg(a.w + (size_t)m * a.N + j);
        const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
        K::pair(dx, dy, dz, s, f, acc, a.kp);
    }
}

// Lane l works for target l / kGroup of the batch, as member l % kGroup of its
// group; the kGroup lanes of a target share every MAC decision.
// STATS: also write the per-target interaction counts (a.stats != nullptr).
template <int PT, int KER, bool STATS>
__global__ void __launch_bounds__(kWarps * 32, KER == 0 ? KITC_EVAL_MINB : KITC_EVAL_MINB1) k_eval(const EvalArgs a) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, NP = K::P, NA = K::NA;
    extern __shared__ int2 smem_stack[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int grp = lane % kGroup, ti = lane / kGroup;
    int2* stk = smem_stack + wl * a.stack_cap;
    const long long b = a.bb + (long long)blockIdx.x * kWarps + wl;
    if (b >= a.be) return;  // whole warp
    const int p0 = a.bstart[b], tc = a.bcount[b];
    const bool valid = ti < tc;
    const int t = a.tord[p0 + (valid ? ti : 0)];
    const double x = a.x[t], y = a.y[t], z = a.z[t];
    const int P = PT > 0 ? PT : a.P;
    const int P3 = P * P * P;
    double acc[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) acc[c] = 0.0;
    unsigned long long st[5] = {0, 0, 0, 0, 0};
    const unsigned live = __ballot_sync(0xffffffffu, valid);
    if (lane == 0) stk[0] = make_int2(0, (int)live);
    __syncwarp();
    int sp = 1;
    while (sp > 0) {
        --sp;
        const int2 ent = stk[sp];
        __syncwarp();
        const int c = ent.x;
        const unsigned mask = (unsigned)ent.y;
        const bool in = (mask >> lane) & 1u;
        const double4 cr = a.cr[c];
        bool ok = false;
        if (in) {
            const double dx = __dsub_rn(x, cr.x), dy = __dsub_rn(y, cr.y), dz = __dsub_rn(z, cr.z);
            const double R2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
            ok = R2 > 0.0 && cr.w <= __dmul_rn(a.tt, R2);
        }
        const unsigned am = __ballot_sync(0xffffffffu, ok);
        const unsigned rm = mask & ~am;
        const int4 tp = a.topo[c];
        if (am && ok) {
            far_field<PT, KER>(x, y, z, a.grid + (size_t)c * 3 * P, a.fhat + (size_t)c * M * P3, acc, a.kp, P, grp);
            if (STATS) {
                st[0] += 1;
                st[1] += (unsigned long long)P3;
                st[4] += (unsigned long long)(tp.y - tp.x);
            }
        }
        if (rm) {
            if (tp.w == 0) {
                if (in && !ok) {
                    near_field<KER>(x, y, z, t, tp.x, tp.y, grp, a, acc);
                    if (STATS) {
                        const int self = (a.self_omit && t >= tp.x && t < tp.y) ? 1 : 0;
                        st[2] += 1;
                        st[3] += (unsigned long long)(tp.y - tp.x - self);
                        st[4] += (unsigned long long)(tp.y - tp.x);
                    }
                }
            } else {
                // children pushed in reverse so the first child is popped first (A17)
                if (lane < tp.w) stk[sp + tp.w - 1 - lane] = make_int2(tp.z + lane, (int)rm);
                sp += tp.w;
                __syncwarp();
            }
        }
    }
    // combine the kGroup partial sums of each target (fixed order -> deterministic)
#pragma unroll
    for (int c = 0; c < NA; ++c)
#pragma unroll
        for (int o = 1; o < kGroup; o <<= 1) acc[c] += __shfl_xor_sync(0xffffffffu, acc[c], o);
    if (!valid || grp != 0) return;
    const int o = a.perm[t];
#pragma unroll
    for (int c = 0; c < NP; ++c) a.out[(size_t)o * NP + c] = K::out(acc, c);
    if (STATS)
        for (int k = 0; k < 5; ++k) a.stats[(size_t)o * 5 + k] = st[k];
}

template <int PT, int KER, bool STATS>
static void launch_k(const EvalArgs& a, int grid, size_t smem, cudaStream_t s) {
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_eval<PT, KER, STATS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_eval<PT, KER, STATS><<<grid, kWarps * 32, smem, s>>>(a); note_launch();
}

template <int PT, int KER>
static void launch(const EvalArgs& a, int grid, size_t smem, cudaStream_t s) {
    if (a.stats)
        launch_k<PT, KER, true>(a, grid, smem, s);
    else
        launch_k<PT, KER, false>(a, grid, smem, s);
}

template <int KER>
static void dispatch(int P, const EvalArgs& a, int grid, size_t smem, cudaStream_t s) {
    switch (P) {
        case 2: launch<2, KER>(a, grid, smem, s); break;
        case 3: launch<3, KER>(a, grid, smem, s); break;
        case 4: launch<4, KER>(a, grid, smem, s); break;
        case 5: launch<5, KER>(a, grid, smem, s); break;
        case 6: launch<6, KER>(a, grid, smem, s); break;
        case 7: launch<7, KER>(a, grid, smem, s); break;
        case 8: launch<8, KER>(a, grid, smem, s); break;
        case 9: launch<9, KER>(a, grid, smem, s); break;
        case 10: launch<10, KER>(a, grid, smem, s); break;
        case 11: launch<11, KER>(a, grid, smem, s); break;
        default: launch<0, KER>(a, grid, smem, s); break;
    }
}

}  // namespace

kitc_status eval(const kitc_tree* t, int kernel, int n, double theta, double eps, int self, const double* fhat,
                 int64_t bb, int64_t be, double* out, uint64_t* stats, cudaStream_t s) {
    if (!t->built) return set_error(KITC_ESTATE, "kitc_eval: tree not built");
    if (!t->weights_ready || t->grid_n != n || t->weights_kernel != kernel)
        return set_error(KITC_ESTATE, "kitc_eval: call kitc_modified_weights with the same kernel and n first");
    if (!(theta >= 0.0 && theta < 1.0)) return set_error(KITC_EINVAL, "kitc_eval: theta must be in [0, 1)");
    if (!(eps >= 0.0) || !std::isfinite(eps)) return set_error(KITC_EINVAL, "kitc_eval: eps must be >= 0");
    if (self != KITC_SELF_OMIT && self != KITC_SELF_INCLUDE) return set_error(KITC_EINVAL, "kitc_eval: bad self");
    if (eps == 0.0 && self != KITC_SELF_OMIT)
        return set_error(KITC_EINVAL, "kitc_eval: eps = 0 requires KITC_SELF_OMIT (singular kernel)");
    if (bb < 0 || be > t->nbatches || bb > be) return set_error(KITC_EINVAL, "kitc_eval: bad batch range");
    if (!fhat || !out) return set_error(KITC_EINVAL, "kitc_eval: NULL buffer");
    if (be == bb) return KITC_OK;
    EvalArgs a;
    a.x = t->x.as<double>();
    a.y = t->y.as<double>();
    a.z = t->z.as<double>();
    a.perm = t->perm.as<int>();
    a.tord = t->tord.as<int>();
    a.w = t->w.as<double>();
    a.cr = t->cr.as<double4>();
    a.topo = t->topo.as<int4>();
    a.grid = t->grid.as<double>();
    a.fhat = fhat;
    a.bstart = t->bstart.as<int>();
    a.bcount = t->bcount.as<int>();
    a.out = out;
    a.stats = reinterpret_cast<unsigned long long*>(stats);
    a.bb = bb;
    a.be = be;
    a.N = (int)t->N;
    a.P = n + 1;
    a.stack_cap = 8 * (t->depth + 1);
    a.self_omit = self == KITC_SELF_OMIT;
    a.tt = theta * theta;
    a.kp = make_kparams(eps);
    const size_t smem = (size_t)kWarps * a.stack_cap * sizeof(int2);
    if (smem > 200 * 1024) return set_error(KITC_EINVAL, "kitc_eval: tree too deep for the traversal stack");
    const long long nb = be - bb;
    const int grid = (int)((nb + kWarps - 1) / kWarps);
    switch (kernel) {
        case KITC_STOKESLET: dispatch<0>(n + 1, a, grid, smem, s); break;
        case KITC_ROTLET: dispatch<1>(n + 1, a, grid, smem, s); break;
        case KITC_STOKESLET_ROTLET: dispatch<2>(n + 1, a, grid, smem, s); break;
        default: return set_error(KITC_EINVAL, "kitc_eval: unknown kernel");
    }
    KITC_CUDA(cudaGetLastError());
    return KITC_OK;
}

}  // namespace kitc
