// weights.cu -- modified weights (Eq. modified_weights, Algorithm 1
// P:528-557) as an sm_100a fp64 kernel.
//
// Work item = (cluster, chunk of <= kChunk of its particles).  Per tile of kTile
// particles, phase 1 forms the three per-axis barycentric vectors
//   L_l,k = a_k / sum_k' a_k',  a_k = w_k / (y_l - s_l,k)       (Eq. Barycentric-1D)
// with the DBL_MIN coincidence flag (Algorithm 1 lines 10, 15-17: L = e_flag,
// last k wins) and stages them with the weights in shared memory; phase 2 has
// thread (k2, k3) accumulate fhat[m][k1][k2][k3] += Lx[k1] (Ly[k2] Lz[k3] f_m)
// in registers for all k1 and m (the tensor-product loop of lines 20-22).
// Layout (include/kitc.h): fhat[c][r][k3][m][j], row = k1 (n+1) + k2 = 8 r + j:
// blocks of 8 rows ("rounds") hold all k3 and m of those rows contiguously, so
// k_eval stages one round with one bulk copy; padding rows of the last round are 0.
// Chunks of one cluster write partials that a second kernel sums in chunk
// order (deterministic).  Reading A15: L per axis instead of
// (a1 a2 a3 / denom), reciprocals by Newton-refined MUFU seeds -- rounding-only
// differences (parity gate 1e-13 per cluster).
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "kitc_internal.cuh"

namespace kitc {

namespace {

#ifndef KITC_W_MINB
#define KITC_W_MINB 6  // resident CTAs per SM (n <= 10); measured: 6 > 1 (128 regs) > 8 > 10
#endif
constexpr int kChunk = 4096;       // particles per work item (large calls)
constexpr int kChunkSmall = 1024;  // ... when the call has too few items to fill the GPU
// Chunk size of a tree: small chunks when the whole tree holds fewer than ~2 waves of work items
// (N ~ 1e6: a rank's shard at 8 GPUs then still fills the GPU; measured C3 8-rank shard 0.62 ->
// 0.36 ms), large ones otherwise (fewer partial slots to sum; C5 17.2 ms vs 18.2 ms with small
// chunks).  It depends on the tree only, never on the cluster range, so fhat (and every result) is
// bitwise the same however the clusters are split over calls or ranks.
static int weights_chunk(int64_t particle_clusters) {
    return particle_clusters / kChunk < 2 * 148 * KITC_W_MINB ? kChunkSmall : kChunk;
}
#ifndef KITC_W_TILE
#define KITC_W_TILE 32  // measured: 32 > 64 > 16
#endif
constexpr int kTile = KITC_W_TILE;  // particles staged per shared-memory tile

struct WItem {
    int32_t c;     // cluster id
    int32_t b, e;  // particle range (sorted indices)
    int32_t slot;  // -1: write fhat directly; >= 0: partial slot
};

struct Nodes {
    double t[kMaxDegree + 1];
};

// Destination replicas of fhat: the computed slice of every cluster is stored
// into each of them (same layout and offsets).  n = 1: the caller's buffer; n > 1:
// the fused modified-weights + all-gather of the multi-GPU path -- the other
// entries are peer GPUs' buffers mapped into this process (symmetric memory over
// NVLink), so the exchange is the kernel's own stores, with no separate collective.
struct Peers {
    double* p[kMaxPeers];
    int n;
};

// ws[c][i] = w[perm[i]][c] (SoA planes, Algorithm 1) and the packed near-field
// source records src[i] = (x, y, z, w_0 .. w_{m-1}, 0 pad) of sld doubles (16-B
// multiple), read by k_eval's near field with 16-byte loads.
__global__ void k_gather_w(const double* __restrict__ w, const int* __restrict__ perm, int N, int m,
                           double* __restrict__ ws, const double* __restrict__ x, const double* __restrict__ y,
                           const double* __restrict__ z, int sld, double* __restrict__ src) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    const size_t o = (size_t)perm[i] * m;
    double* r = src + (size_t)i * sld;
    r[0] = x[i];
    r[1] = y[i];
    r[2] = z[i];
    for (int c = 0; c < m; ++c) {
        const double v = w[o + c];
        ws[(size_t)c * N + i] = v;
        r[3 + c] = v;
    }
    for (int c = 3 + m; c < sld; ++c) r[c] = 0.0;
}

// grid s_{l,k} = c_l + h_l t_k, s_{l,0} = hi_l, s_{l,n} = lo_l (reading A13), RN.
__global__ void k_grids(int C, int n, Nodes nd, const double* __restrict__ box, double* __restrict__ grid) {
    int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= C) return;
    const int P = n + 1;
    for (int l = 0; l < 3; ++l) {
        const double lo = box[(size_t)c * 6 + l], hi = box[(size_t)c * 6 + 3 + l];
        const double ctr = __dmul_rn(0.5, __dadd_rn(lo, hi)), h = __dmul_rn(0.5, __dsub_rn(hi, lo));
        double* g = grid + ((size_t)c * 3 + l) * P;
        for (int k = 0; k <= n; ++k) g[k] = __dadd_rn(ctr, __dmul_rn(h, nd.t[k]));
        g[0] = hi;
        g[n] = lo;
    }
}

// 1/d for normal |d| (> DBL_MIN here): MUFU seed + two Newton steps (~1 ulp), no
// IEEE-division slow path (its branch serialises the warp).
__device__ __forceinline__ double rcp_nr(double d) {
    double y;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
    double e = fma(-d, y, 1.0);
    y = fma(y, e, y);
    e = fma(-d, y, 1.0);
    return fma(y, e, y);
}

// 1D barycentric vector of coordinate v on nodes s (Algorithm 1 lines 9-17).
template <int P>
__device__ __forceinline__ void bary(double v, const double* s, double* L) {
    double sum = 0.0;
    int flag = -1;
    double a[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
        const double diff = v - s[k];
        const double wk = (k == 0 || k == P - 1) ? ((k & 1) ? -0.5 : 0.5) : ((k & 1) ? -1.0 : 1.0);
        const bool hit = fabs(diff) <= DBL_MIN;
        flag = hit ? k : flag;
        a[k] = hit ? 0.0 : wk * rcp_nr(hit ? 1.0 : diff);
        sum += a[k];
    }
    const double inv = rcp_nr(flag >= 0 ? 1.0 : sum);
#pragma unroll
    for (int k = 0; k < P; ++k) L[k] = flag >= 0 ? (k == flag ? 1.0 : 0.0) : a[k] * inv;
}

template <int P, int M>
__global__ void __launch_bounds__((P * P + 31) / 32 * 32, P <= 11 ? KITC_W_MINB : 1) k_weights(
    const WItem* __restrict__ items, const double* __restrict__ x, const double* __restrict__ y,
    const double* __restrict__ z, const double* __restrict__ ws, int N, const double* __restrict__ grid,
    const Peers fhat, double* __restrict__ part, const int* __restrict__ nitems) {
    constexpr int P2 = P * P, NT = (P2 + 31) / 32 * 32, R = (P2 + kRows - 1) / kRows;
    constexpr int LEN = R * P * M * kRows;
    // rows padded to an even length: the x vector and the weights are read as 16-byte pairs
    constexpr int PP = (P + 1) & ~1, MP = (M + 1) & ~1;
    constexpr int QC = (3 * kTile + NT - 1) / NT, QW = (M * kTile + NT - 1) / NT;  // phase-1 items per thread
    __shared__ double sg[3 * P];
    // two tile buffers: phase 1 of tile t + 1 fills one while no thread can still read it
    // (they all passed tile t's barrier after finishing phase 2 of tile t - 1) -> one barrier per tile
    __shared__ __align__(16) double Lx[2][kTile][PP];
    __shared__ double Ly[2][kTile][P], Lz[2][kTile][P];
    __shared__ __align__(16) double sw[2][kTile][MP];
    if ((int)blockIdx.x >= *nitems) return;  // grid sized by an upper bound (no host sync)
    const WItem it = items[blockIdx.x];
    KITC_DCHECK(it.b >= 0 && it.b <= it.e && it.e <= N && it.c >= 0);
    const int tid = threadIdx.x;
    for (int i = tid; i < 3 * P; i += NT) sg[i] = grid[(size_t)it.c * 3 * P + i];
    const int k2 = tid / P, k3 = tid % P;
    const bool owner = tid < P2;
    double acc[M][P];
#pragma unroll
    for (int m = 0; m < M; ++m)
#pragma unroll
        for (int k = 0; k < P; ++k) acc[m][k] = 0.0;
    // the next tile's coordinates and weights, loaded into registers one tile ahead (their
    // global latency overlaps phase 2 of the current tile)
    double pc[QC], pw[QW];
    auto prefetch = [&](int tile) {
        const int cnt = min(kTile, it.e - tile);
#pragma unroll
        for (int i = 0; i < QC; ++i) {
            const int q = tid + i * NT, l = q / cnt, j = q - l * cnt;
            if (q < 3 * cnt) pc[i] = (l == 0 ? x : l == 1 ? y : z)[tile + j];
        }
#pragma unroll
        for (int i = 0; i < QW; ++i) {
            const int q = tid + i * NT, m = q / cnt, j = q - m * cnt;
            if (q < M * cnt) pw[i] = ws[(size_t)m * N + tile + j];
        }
    };
    if (it.b < it.e) prefetch(it.b);
    __syncthreads();
    int buf = 0;
    for (int tile = it.b; tile < it.e; tile += kTile, buf ^= 1) {
        const int cnt = min(kTile, it.e - tile);
        // phase 1: the 3 cnt per-axis vectors and the cnt weights, spread over all threads
#pragma unroll
        for (int i = 0; i < QC; ++i) {
            const int q = tid + i * NT, l = q / cnt, j = q - l * cnt;
            if (q < 3 * cnt) bary<P>(pc[i], sg + l * P, l == 0 ? Lx[buf][j] : l == 1 ? Ly[buf][j] : Lz[buf][j]);
        }
#pragma unroll
        for (int i = 0; i < QW; ++i) {
            const int q = tid + i * NT, m = q / cnt, j = q - m * cnt;
            if (q < M * cnt) sw[buf][j][m] = pw[i];
        }
        if (tile + kTile < it.e) prefetch(tile + kTile);
        __syncthreads();
        if (owner) {
            for (int j = 0; j < cnt; ++j) {
                const double q = Ly[buf][j][k2] * Lz[buf][j][k3];
                double g[MP];
#pragma unroll
                for (int m = 0; m < MP; m += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(&sw[buf][j][m]);
                    g[m] = q * v.x;
                    g[m + 1] = q * v.y;
                }
#pragma unroll
                for (int k1 = 0; k1 < PP; k1 += 2) {
                    const double2 v = *reinterpret_cast<const double2*>(&Lx[buf][j][k1]);
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        acc[m][k1] = fma(v.x, g[m], acc[m][k1]);
                        if (k1 + 1 < P) acc[m][k1 + 1] = fma(v.y, g[m], acc[m][k1 + 1]);
                    }
                }
            }
        }
    }
    const int nd = it.slot < 0 ? fhat.n : 1;
    for (int r = 0; r < nd; ++r) {
        double* dst = it.slot < 0 ? fhat.p[r] + (size_t)it.c * LEN : part + (size_t)it.slot * LEN;
        // zero padding rows P2 .. R kRows - 1
        for (int q = tid; q < (R * kRows - P2) * P * M; q += NT) {
            const int row = P2 + q / (P * M), km = q % (P * M);
            dst[((row / kRows) * P * M + km) * kRows + row % kRows] = 0.0;
        }
        if (!owner) continue;
#pragma unroll
        for (int m = 0; m < M; ++m)
#pragma unroll
            for (int k1 = 0; k1 < P; ++k1) {
                const int row = k1 * P + k2;
                dst[(((row / kRows) * P + k3) * M + m) * kRows + row % kRows] = acc[m][k1];
            }
    }
}

struct RItem {
    int32_t c, first_slot, nslots, pad;
};

// fhat[c] = sum of its partial slots in chunk order (deterministic).
__global__ void k_reduce(const RItem* __restrict__ r, int len, const double* __restrict__ part,
                         const Peers fhat, const int* __restrict__ nred) {
    if ((int)blockIdx.x >= *nred) return;
    const RItem it = r[blockIdx.x];
    for (int i = threadIdx.x; i < len; i += blockDim.x) {
        double s = part[(size_t)it.first_slot * len + i];
        for (int k = 1; k < it.nslots; ++k) s += part[(size_t)(it.first_slot + k) * len + i];
        for (int q = 0; q < fhat.n; ++q) fhat.p[q][(size_t)it.c * len + i] = s;
    }
}

// Work items of clusters [cb, ce) built on the device (one CTA): per cluster
// nch = ceil(N_C / chunk) chunks; one chunk writes fhat directly, several write
// partial slots that k_reduce sums in chunk order.  counts[0] = items, [1] = reduce
// entries.  Exclusive scans in cluster order (three at once).
__global__ void __launch_bounds__(1024) k_witems(const int4* __restrict__ topo, int cb, int ce, int leaves_only, int chunk,
                                                 WItem* __restrict__ items, RItem* __restrict__ red,
                                                 int* __restrict__ counts) {
    __shared__ int3 wsum[33];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
    int3 run = make_int3(0, 0, 0);  // items, slots, reduce entries before this chunk of clusters
    for (int c0 = cb; c0 < ce; c0 += blockDim.x) {
        const int c = c0 + threadIdx.x;
        int4 tp = make_int4(0, 0, 0, 0);
        int nch = 0;
        if (c < ce) {
            tp = topo[c];
            nch = (leaves_only && tp.w > 0) ? 0 : (tp.y - tp.x + chunk - 1) / chunk;
        }
        const int3 v = make_int3(nch, nch > 1 ? nch : 0, nch > 1 ? 1 : 0);
        int3 inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int a = __shfl_up_sync(0xffffffffu, inc.x, o), b = __shfl_up_sync(0xffffffffu, inc.y, o),
                      d = __shfl_up_sync(0xffffffffu, inc.z, o);
            if (lane >= o) {
                inc.x += a;
                inc.y += b;
                inc.z += d;
            }
        }
        if (lane == 31) wsum[w] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int3 sacc = make_int3(0, 0, 0);
            for (int k = 0; k < nw; ++k) {
                const int3 tt = wsum[k];
                wsum[k] = sacc;
                sacc.x += tt.x;
                sacc.y += tt.y;
                sacc.z += tt.z;
            }
            wsum[32] = sacc;
        }
        __syncthreads();
        if (c < ce) {
            const int io = run.x + wsum[w].x + inc.x - v.x, so = run.y + wsum[w].y + inc.y - v.y,
                      ro = run.z + wsum[w].z + inc.z - v.z;
            for (int q = 0; q < nch; ++q)
                items[io + q] = WItem{c, tp.x + q * chunk, min(tp.y, tp.x + (q + 1) * chunk), nch == 1 ? -1 : so + q};
            if (nch > 1) red[ro] = RItem{c, so, nch, 0};
        }
        run.x += wsum[32].x;
        run.y += wsum[32].y;
        run.z += wsum[32].z;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        counts[0] = run.x;
        counts[1] = run.z;
    }
}

// Upward pass (flag KITC_WEIGHTS_UPWARD; not in the paper): the
// fhat of an internal cluster from its children's.  Algorithm 1 applied to a child's
// proxy points s_C,k' (charges fhat_C,k') on the parent's grid factorises over the
// axes: fhat_P[k1 k2 k3] += sum_k' A_x[k1][k1'] A_y[k2][k2'] A_z[k3][k3'] fhat_C[k1' k2' k3'],
// A_l[kp][kc] = L^P_kp(s_C,l,kc) (the 1D barycentric vector of Algorithm 1 lines 9-17,
// coincidence flag included), so it runs as three 1D transforms of P^4 FMAs each
// instead of (n+1)^3 "particles" x (n+1)^3 terms; exact in exact arithmetic (the
// children's fhat reproduce every moment of degree <= n per axis).  One CTA per
// internal cluster of one level (children first: the host launches deepest level
// first); one component at a time in shared memory [F | T | ACC | A | grids].
template <int P, int M>
__global__ void __launch_bounds__(256) k_upward(const int4* __restrict__ topo, const int* __restrict__ lstart, int lv,
                                                int cb, const double* __restrict__ grid, const Peers fhat) {
    constexpr int P2 = P * P, P3 = P2 * P, R = (P2 + kRows - 1) / kRows, LEN = R * P * M * kRows;
    extern __shared__ __align__(16) double upw[];
    double* F = upw;            // child fhat, one component [k1][k2][k3]; then T2
    double* T = F + P3;         // T1
    double* ACC = T + P3;       // parent fhat, one component
    double* A = ACC + P3;       // [3][P][P]
    double* sP = A + 3 * P2;    // parent grid [3][P]
    const int tid = threadIdx.x;
    const int L0 = max(lstart[lv], cb), L1 = lstart[lv + 1];
    const double* src = fhat.p[0];
    for (int c = L0 + (int)blockIdx.x; c < L1; c += gridDim.x) {
        const int4 tp = topo[c];
        if (tp.w == 0) continue;  // leaves: Algorithm 1 on their particles (k_weights)
        __syncthreads();
        for (int i = tid; i < 3 * P; i += blockDim.x) sP[i] = grid[(size_t)c * 3 * P + i];
        for (int m = 0; m < M; ++m) {
            for (int i = tid; i < P3; i += blockDim.x) ACC[i] = 0.0;
            for (int ch = tp.z; ch < tp.z + tp.w; ++ch) {
                __syncthreads();
                // A_l[kp][kc] = L^P_kp(s_C,l,kc); the child's fhat component m
                for (int q = tid; q < 3 * P; q += blockDim.x) {
                    const int l = q / P, kc = q - l * P;
                    double Lv[P];
                    bary<P>(grid[((size_t)ch * 3 + l) * P + kc], sP + l * P, Lv);
#pragma unroll
                    for (int kp = 0; kp < P; ++kp) A[(l * P + kp) * P + kc] = Lv[kp];
                }
                const double* Fc = src + (size_t)ch * LEN;
                for (int i = tid; i < P3; i += blockDim.x) {
                    const int row = i / P, k3 = i - row * P;
                    F[i] = Fc[(((row / kRows) * P + k3) * M + m) * kRows + row % kRows];
                }
                __syncthreads();
                for (int i = tid; i < P3; i += blockDim.x) {  // T[k1][k2'][k3'] = sum_k1' A_x[k1][k1'] F[k1'][k2'][k3']
                    const int k1 = i / P2, r = i - k1 * P2;
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < P; ++k) v = fma(A[k1 * P + k], F[k * P2 + r], v);
                    T[i] = v;
                }
                __syncthreads();
                for (int i = tid; i < P3; i += blockDim.x) {  // F[k1][k2][k3'] = sum_k2' A_y[k2][k2'] T[k1][k2'][k3']
                    const int k1 = i / P2, k2 = (i / P) % P, k3 = i % P;
                    double v = 0.0;
#pragma unroll
                    for (int k = 0; k < P; ++k) v = fma(A[(P + k2) * P + k], T[(k1 * P + k) * P + k3], v);
                    F[i] = v;
                }
                __syncthreads();
                for (int i = tid; i < P3; i += blockDim.x) {  // ACC[k1][k2][k3] += sum_k3' A_z[k3][k3'] F[k1][k2][k3']
                    const int r = i / P, k3 = i % P;
                    double v = ACC[i];
#pragma unroll
                    for (int k = 0; k < P; ++k) v = fma(A[(2 * P + k3) * P + k], F[r * P + k], v);
                    ACC[i] = v;
                }
            }
            __syncthreads();
            for (int q = 0; q < fhat.n; ++q) {
                double* dst = fhat.p[q] + (size_t)c * LEN;
                for (int i = tid; i < P3; i += blockDim.x) {
                    const int row = i / P, k3 = i - row * P;
                    dst[(((row / kRows) * P + k3) * M + m) * kRows + row % kRows] = ACC[i];
                }
                for (int i = tid; i < (R * kRows - P2) * P; i += blockDim.x) {  // padding rows
                    const int row = P2 + i / P, k3 = i % P;
                    dst[(((row / kRows) * P + k3) * M + m) * kRows + row % kRows] = 0.0;
                }
            }
        }
    }
}

template <int P, int M>
static void launch_upward(const kitc_tree* t, const int* lstart, int cb, const Peers& fhat, cudaStream_t s) {
    const size_t smem = (size_t)(3 * P * P * P + 3 * P * P + 3 * P) * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_upward<P, M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int lv = t->depth - 1; lv >= 0; --lv) {  // children before parents
        k_upward<P, M><<<148 * 4, 256, smem, s>>>(t->topo.as<int4>(), lstart, lv, cb, t->grid.as<double>(), fhat);
        note_launch();
    }
}

template <int M>
static kitc_status dispatch_upward(int n, const kitc_tree* t, const int* lstart, int cb, const Peers& fhat,
                                   cudaStream_t s) {
    switch (n + 1) {
#define KITC_U(P) \
    case P: launch_upward<P, M>(t, lstart, cb, fhat, s); break;
        KITC_U(2) KITC_U(3) KITC_U(4) KITC_U(5) KITC_U(6) KITC_U(7) KITC_U(8) KITC_U(9) KITC_U(10)
        KITC_U(11) KITC_U(12) KITC_U(13) KITC_U(14) KITC_U(15) KITC_U(16) KITC_U(17)
#undef KITC_U
        default: return set_error(KITC_EINVAL, "kitc_modified_weights: n out of range");
    }
    return KITC_OK;
}

template <int P, int M>
static void launch_weights(int nitems, const WItem* items, const kitc_tree* t, const double* ws,
                           const double* grid, const Peers& fhat, double* part, const int* counts, cudaStream_t s) {
    constexpr int NT = (P * P + 31) / 32 * 32;
    k_weights<P, M><<<nitems, NT, 0, s>>>(items, t->x.as<double>(), t->y.as<double>(), t->z.as<double>(), ws,
                                          (int)t->N, grid, fhat, part, counts); note_launch();
}

template <int M>
static kitc_status dispatch(int n, int nitems, const WItem* items, const kitc_tree* t, const double* ws,
                            const double* grid, const Peers& fhat, double* part, const int* counts, cudaStream_t s) {
    switch (n + 1) {
#define KITC_W(P) \
    case P: launch_weights<P, M>(nitems, items, t, ws, grid, fhat, part, counts, s); break;
        KITC_W(2) KITC_W(3) KITC_W(4) KITC_W(5) KITC_W(6) KITC_W(7) KITC_W(8) KITC_W(9) KITC_W(10)
        KITC_W(11) KITC_W(12) KITC_W(13) KITC_W(14) KITC_W(15) KITC_W(16) KITC_W(17)
#undef KITC_W
        default: return set_error(KITC_EINVAL, "kitc_modified_weights: n out of range");
    }
    return KITC_OK;
}

}  // namespace

kitc_status modified_weights(kitc_tree* t, int kernel, int n, const double* w, int64_t cb, int64_t ce,
                             double* const* fhat_peers, int npeers, cudaStream_t s, unsigned flags) {
    if (flags & ~(unsigned)KITC_WEIGHTS_UPWARD) return set_error(KITC_EINVAL, "kitc_modified_weights: unknown flags");
    const bool upward = (flags & KITC_WEIGHTS_UPWARD) != 0;
    if (npeers < 1 || npeers > kMaxPeers) return set_error(KITC_EINVAL, "kitc_modified_weights: npeers out of range");
    Peers fhat;
    fhat.n = npeers;
    for (int q = 0; q < kMaxPeers; ++q) fhat.p[q] = q < npeers ? fhat_peers[q] : nullptr;
    for (int q = 0; q < npeers; ++q)
        if (!fhat.p[q] && ce > cb) return set_error(KITC_EINVAL, "kitc_modified_weights: NULL buffer");
    int32_t m = 0, p = 0;
    KITC_TRY(kitc_kernel_dims(kernel, &m, &p));
    if (n < 1 || n > kMaxDegree) return set_error(KITC_EINVAL, "kitc_modified_weights: n must be in [1, 16]");
    if (!t->built) return set_error(KITC_ESTATE, "kitc_modified_weights: tree not built");
    if (cb < 0 || ce > t->nclusters || cb > ce) return set_error(KITC_EINVAL, "kitc_modified_weights: bad cluster range");
    if (!w) return set_error(KITC_EINVAL, "kitc_modified_weights: NULL buffer");
    const int N = (int)t->N, C = (int)t->nclusters, P = n + 1;
    const long long LEN = fhat_cluster_len(P, m);
    // sorted weights (SoA, m planes)
    KITC_TRY(t->w.ensure((size_t)m * N * sizeof(double), s));
    const int sld = (3 + m + 1) & ~1;
    KITC_TRY(t->src.ensure((size_t)N * sld * sizeof(double), s));
    t->src_ld = sld;
    k_gather_w<<<(N + 255) / 256, 256, 0, s>>>(w, t->perm.as<int>(), N, m, t->w.as<double>(), t->x.as<double>(),
                                               t->y.as<double>(), t->z.as<double>(), sld, t->src.as<double>());
    note_launch();
    // grids of every cluster (reading A12: t_k = sin(pi (n - 2k) / (2n)))
    Nodes nd;
    for (int k = 0; k <= n; ++k) nd.t[k] = std::sin(kPi * (double)(n - 2 * k) / (2.0 * (double)n));
    KITC_TRY(t->grid.ensure((size_t)C * 3 * P * sizeof(double), s));
    k_grids<<<(C + 127) / 128, 128, 0, s>>>(C, n, nd, t->box.as<double>(), t->grid.as<double>()); note_launch();
    KITC_CUDA(cudaGetLastError());
    t->w_m = m;
    t->grid_n = n;
    t->weights_kernel = kernel;
    t->weights_ready = true;
    if (ce == cb) return KITC_OK;
    if (upward && (ce != C || npeers != 1))
        return set_error(KITC_EINVAL, "kitc_modified_weights: KITC_WEIGHTS_UPWARD needs cluster_end = C (children "
                                      "in range) and one fhat buffer");
    // work items on the device; grids sized by upper bounds (items: each particle lies in
    // depth + 1 clusters, each cluster adds at most one partial chunk) -- no host sync
    const int64_t ncl = ce - cb;
    const int chunk = weights_chunk((int64_t)N * (t->depth + 1));
    const int64_t ub_items = std::min<int64_t>((int64_t)N * (t->depth + 1) / chunk + ncl, 0x7fffffff);
    const size_t o1 = ((size_t)ub_items * sizeof(WItem) + 15) / 16 * 16;
    const size_t o2 = o1 + ((size_t)ncl * sizeof(RItem) + 15) / 16 * 16;
    KITC_TRY(t->d_witems.ensure(o2 + 16, s));
    WItem* di = t->d_witems.as<WItem>();
    RItem* dr = reinterpret_cast<RItem*>(t->d_witems.as<char>() + o1);
    int* counts = reinterpret_cast<int*>(t->d_witems.as<char>() + o2);
    k_witems<<<1, 1024, 0, s>>>(t->topo.as<int4>(), (int)cb, (int)ce, upward ? 1 : 0, chunk, di, dr, counts);
    note_launch();
    KITC_TRY(t->d_wpart.ensure((size_t)std::max<int64_t>(ub_items, 1) * LEN * sizeof(double), s));
    if (m == 3)
        KITC_TRY(dispatch<3>(n, (int)ub_items, di, t, t->w.as<double>(), t->grid.as<double>(), fhat,
                             t->d_wpart.as<double>(), counts, s));
    else
        KITC_TRY(dispatch<6>(n, (int)ub_items, di, t, t->w.as<double>(), t->grid.as<double>(), fhat,
                             t->d_wpart.as<double>(), counts, s));
    k_reduce<<<(int)ncl, 256, 0, s>>>(dr, (int)LEN, t->d_wpart.as<double>(), fhat, counts + 1); note_launch();
    if (upward && t->depth > 0) {
        if (m == 3)
            KITC_TRY(dispatch_upward<3>(n, t, tree_level_starts(t), (int)cb, fhat, s));
        else
            KITC_TRY(dispatch_upward<6>(n, t, tree_level_starts(t), (int)cb, fhat, s));
    }
    KITC_CUDA(cudaGetLastError());
    return KITC_OK;
}

size_t weights_bytes(int64_t N, int64_t C, int32_t depth, int kernel, int n) {
    int32_t m = 0;
    if (kitc_kernel_dims(kernel, &m, nullptr) != KITC_OK || n < 1 || n > kMaxDegree) return 0;
    const int P = n + 1;
    const int64_t LEN = fhat_cluster_len(P, m);
    const int sld = (3 + m + 1) & ~1;
    const int64_t ub_items = N * (depth + 1) / kChunkSmall + C;
    const size_t witems = ((size_t)ub_items * sizeof(WItem) + 15) / 16 * 16 + ((size_t)C * sizeof(RItem) + 15) / 16 * 16 + 16;
    return dev_alloc_bytes((size_t)m * N * sizeof(double)) + dev_alloc_bytes((size_t)N * sld * sizeof(double)) +
           dev_alloc_bytes((size_t)C * 3 * P * sizeof(double)) + dev_alloc_bytes(witems) +
           dev_alloc_bytes((size_t)std::max<int64_t>(ub_items, 1) * LEN * sizeof(double));
}

}  // namespace kitc
