// tree.cu -- the KITC cluster tree, built on the device by ONE cooperative kernel.
//
// Rule (§6; readings A1-A4): minimal bounding
// box per cluster; a cluster with count > N0 is bisected at its midpoint along
// every side L_l > lmax / sqrt(2); x_l >= mid_l -> upper half; children = the
// nonempty code groups (code = bx | by<<1 | bz<<2) in ascending code, formed by
// a STABLE partition; a split leaving < 2 nonempty children is a (degenerate)
// leaf.  Clusters are numbered BFS (level, then range start).
//
// k_build runs every level of the build without returning to the host: grid-wide
// barriers (cooperative launch, one CTA per SM) separate the phases of a level,
//   SB  min/max of every work item (<= kChk particles of one cluster)
//   S1  per cluster: box, centre, r^2, split axes (round-to-nearest intrinsics)
//   S2  CTA 0: exclusive scan of the partition items of the splitting clusters
//   S3  per item: counts of the 8 child codes
//   S4  warp per splitting cluster: child sizes, per-item scatter offsets
//       (warp scans in item order -> the partition is stable)
//   S5  CTA 0: child numbering (scan), child records, next level's work items
//   S6  per item: stable scatter (warp __match_any_sync ranks + per-warp prefix)
//   S7  per item: copy back (overlaps the next level's SB, which reads the copy)
// then the leaves in range order with their warp-batch offsets (bottom-up and
// top-down passes over the levels) and each leaf's targets in Morton order of
// their position in the leaf box (batching only; no result depends on it).
// The host reads back ONE block of counters at the end (kitc_build_tree's only
// synchronisation); a cluster table too small for the tree sets a flag and the
// build is repeated with a larger one (never for the BASELINE configs).
#include <cooperative_groups.h>

#include <cub/block/block_radix_sort.cuh>

#include <algorithm>
#include <cfloat>
#include <cmath>

#include "kitc_internal.cuh"

namespace cg = cooperative_groups;

namespace kitc {

namespace {

constexpr int kBT = 512;           // threads per CTA of k_build
constexpr int kNW = kBT / 32;
constexpr int kChk = 4096;         // particles per work item
constexpr int kUW = 8;             // box / count phases: loads of each axis in flight per lane
constexpr int kUS = 4;             // scatter phase: tiles in flight per warp
constexpr int kU = 4;              // CTA-per-item phases: loads in flight per thread
constexpr int kWarpMode = 2;       // a level's items are done warp-per-item if >= kWarpMode per warp
constexpr double kInvSqrt2 = 0.7071067811865476;  // 1/sqrt(2), RN (reading A2)
constexpr int kSortMax = 2048;     // leaves up to this size are Morton-ordered

// counters (int32) at the head of the control block; level starts follow
enum { kC = 0, kLevels, kDeg, kOverflow, kNonFinite, kLeaves, kBatches, kItems, kBoxItems, kNCtr = 16 };

struct BuildArgs {
    const double* xyz;
    int N, N0, ccap, maxlev, nbatch_cap;
    double *x, *y, *z;
    int* perm;
    double *x2, *y2, *z2;
    int* perm2;
    int4* topo;      // [ccap] begin, end, first child (-1: leaf), nchild
    int* level;      // [ccap]
    int* parent;     // [ccap]
    double* box;     // [ccap][6]
    double4* cr;     // [ccap] centre, r^2
    double4* split;  // [ccap] level-local: centre, axis mask
    int* bpre;       // [ccap + 1] level-local: first box item of each cluster
    int* ipre;       // [ccap + 1] level-local: first partition item
    int* kids;       // [ccap] level-local: children (0: leaf)
    int* tot8;       // [ccap][8] level-local: child sizes by code
    double* bpart;   // [icap][6] box partials of the items
    int* cnt;        // [icap][8]
    int* off;        // [icap][8]
    int* subl;       // [ccap] leaves in the subtree
    int* subb;       // [ccap] warp batches in the subtree
    int* loff;       // [ccap] first leaf (range order) of the subtree
    int* boff;       // [ccap] first batch of the subtree
    int* ctr;        // [kNCtr + maxlev + 2]
    int4* leaves;    // [ccap] begin, end, cluster, first batch (range order)
    int* tord;       // [N]
    int* bstart;     // [nbatch_cap]
    int* bcount;
};

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct Smem {
    union {
        double red[kNW][6];
        struct {
            int wcnt[kNW][8];
            int base[8];
        } sc;
        int scan[kNW + 1];
    };
    int hist[8];
    int item_cl;  // level-local cluster of the CTA's current item
};

// block min/max of (mn[3], mx[3]) -> written by thread 0 to dst[6]
__device__ void block_minmax(double* mn, double* mx, double* dst, Smem& sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        mn[l] = warp_min(mn[l]);
        mx[l] = warp_max(mx[l]);
    }
    if (lane == 0)
        for (int l = 0; l < 3; ++l) {
            sm.red[w][l] = mn[l];
            sm.red[w][3 + l] = mx[l];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = sm.red[0][threadIdx.x];
        for (int k = 1; k < kNW; ++k) v = threadIdx.x < 3 ? fmin(v, sm.red[k][threadIdx.x]) : fmax(v, sm.red[k][threadIdx.x]);
        dst[threadIdx.x] = v;
    }
    __syncthreads();
}

// exclusive scan of val(i), i in [0, n), by one CTA: out[i], out[n] = total (returned)
template <class F>
__device__ int block_scan(int n, F val, int* out, Smem& sm) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int run = 0;
    for (int c0 = 0; c0 < n; c0 += kBT) {
        const int i = c0 + threadIdx.x;
        const int v = i < n ? val(i) : 0;
        int inc = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        if (lane == 31) sm.scan[w] = inc;
        __syncthreads();
        if (threadIdx.x == 0) {
            int s = 0;
            for (int k = 0; k < kNW; ++k) {
                const int t = sm.scan[k];
                sm.scan[k] = s;
                s += t;
            }
            sm.scan[kNW] = s;
        }
        __syncthreads();
        if (i < n) out[i] = run + sm.scan[w] + inc - v;
        run += sm.scan[kNW];
        __syncthreads();
    }
    if (threadIdx.x == 0) out[n] = run;
    __syncthreads();
    return run;
}

// level-local cluster of work item q: the largest i with pre[i] <= q (pre ascending,
// pre[n] = total), by a 32-ary search of the warp (about log32 n dependent loads)
__device__ __forceinline__ int warp_find(const int* pre, int n, int q) {
    const int lane = threadIdx.x & 31;
    int lo = 0, hi = n;  // answer in [lo, hi)
    while (hi - lo > 1) {
        const int step = (hi - lo + 31) / 32;
        const int probe = lo + lane * step;
        const int v = probe < hi ? pre[probe] : 0x7fffffff;
        const unsigned m = __ballot_sync(0xffffffffu, v <= q);
        const int k = 31 - __clz(m);  // lane 0 always qualifies (pre[lo] <= q)
        lo += k * step;
        hi = min(hi, lo + step);
    }
    return lo;
}

__device__ __forceinline__ int child_code(double px, double py, double pz, const double4& sp) {
    const int mask = (int)sp.w;
    int code = 0;
    if ((mask & 1) && px >= sp.x) code |= 1;
    if ((mask & 2) && py >= sp.y) code |= 2;
    if ((mask & 4) && pz >= sp.z) code |= 4;
    return code;
}

__device__ __forceinline__ unsigned int spread3(unsigned int v) {  // 10 bits -> every 3rd bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__device__ __forceinline__ int ld(const int* p) { return *(volatile const int*)p; }

#ifdef KITC_BUILD_PROF  // tuning builds: globaltimer at every grid barrier (CTA 0)
__device__ unsigned long long g_bprof[1024];
__device__ int g_bprof_n;
#endif
// grid-wide barrier; `tag` labels the phase that just ended (profiling builds only)
__device__ __forceinline__ void gsync(cg::grid_group& G, int tag) {
    G.sync();
#ifdef KITC_BUILD_PROF
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        const int k = g_bprof_n;
        if (k < 1024) g_bprof[k] = ((unsigned long long)tag << 56) | (t & 0x00ffffffffffffffull);
        g_bprof_n = k + 1;
    }
#else
    (void)tag;
#endif
}

__global__ void __launch_bounds__(kBT, 1) k_build(const BuildArgs a) {
    cg::grid_group G = cg::this_grid();
    __shared__ Smem sm;
    const int nb = gridDim.x, tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int gt = blockIdx.x * kBT + tid, gsz = nb * kBT;
    int* lstart = a.ctr + kNCtr;

    // ---- level 0: stage the input (AoS -> SoA), identity permutation, root box partials
    {
        double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
        bool bad = false;
        for (int i = gt; i < a.N; i += gsz) {
            const double v[3] = {a.xyz[3 * (size_t)i], a.xyz[3 * (size_t)i + 1], a.xyz[3 * (size_t)i + 2]};
            a.x[i] = v[0];
            a.y[i] = v[1];
            a.z[i] = v[2];
            a.perm[i] = i;
#pragma unroll
            for (int l = 0; l < 3; ++l) {
                bad |= !isfinite(v[l]);
                mn[l] = fmin(mn[l], v[l]);
                mx[l] = fmax(mx[l], v[l]);
            }
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(a.ctr + kNonFinite, 1);
        block_minmax(mn, mx, a.bpart + (size_t)blockIdx.x * 6, sm);
        if (blockIdx.x == 0 && tid == 0) {
            a.topo[0] = make_int4(0, a.N, -1, 0);
            a.level[0] = 0;
            a.parent[0] = -1;
            lstart[0] = 0;
            lstart[1] = 1;
            a.bpre[0] = 0;
            a.bpre[1] = nb;  // the root's box items are the CTAs' partials
        }
    }
    gsync(G, 0);
    if (ld(a.ctr + kNonFinite)) return;

    int l = 0;
    for (;; ++l) {
        const int L0 = ld(lstart + l), L1 = ld(lstart + l + 1), nl = L1 - L0;
        if (nl == 0) break;
        // ---- SB: box partials of the level's work items (level 0: done above).  Level l's
        // particles live in buffer l % 2 (the scatter of level l - 1 ping-pongs).
        const double* cx = (l & 1) ? a.x2 : a.x;
        const double* cy = (l & 1) ? a.y2 : a.y;
        const double* cz = (l & 1) ? a.z2 : a.z;
        if (l > 0) {
            const int B = ld(a.ctr + kBoxItems);
            if (B >= kWarpMode * nb * kNW) {  // many (small) items: a warp per item
                for (int q = blockIdx.x * kNW + w; q < B; q += nb * kNW) {
                    const int i = warp_find(a.bpre, nl, q);
                    const int4 tp = a.topo[L0 + i];
                    const int b = tp.x + (q - a.bpre[i]) * kChk, e = min(tp.y, b + kChk);
                    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
                    for (int t0 = b; t0 < e; t0 += kUW * 32) {  // kUW loads of each axis in flight
                        double v[kUW][3];
#pragma unroll
                        for (int u = 0; u < kUW; ++u) {
                            const int j = min(t0 + u * 32 + lane, e - 1);  // duplicates of a valid point: harmless
                            v[u][0] = cx[j];
                            v[u][1] = cy[j];
                            v[u][2] = cz[j];
                        }
#pragma unroll
                        for (int u = 0; u < kUW; ++u)
#pragma unroll
                            for (int k = 0; k < 3; ++k) {
                                mn[k] = fmin(mn[k], v[u][k]);
                                mx[k] = fmax(mx[k], v[u][k]);
                            }
                    }
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        mn[k] = warp_min(mn[k]);
                        mx[k] = warp_max(mx[k]);
                    }
                    if (lane < 6) a.bpart[(size_t)q * 6 + lane] = lane < 3 ? mn[lane] : mx[lane - 3];
                }
            } else {  // few (large) items: a CTA per item
                for (int q = blockIdx.x; q < B; q += nb) {
                    const int fi = warp_find(a.bpre, nl, q);
                    if (tid == 0) sm.item_cl = fi;
                    __syncthreads();
                    const int i = sm.item_cl;
                    const int4 tp = a.topo[L0 + i];
                    const int b = tp.x + (q - a.bpre[i]) * kChk, e = min(tp.y, b + kChk);
                    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
                    for (int t0 = b; t0 < e; t0 += kU * kBT) {
                        double v[kU][3];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const int j = min(t0 + u * kBT + tid, e - 1);
                            v[u][0] = cx[j];
                            v[u][1] = cy[j];
                            v[u][2] = cz[j];
                        }
#pragma unroll
                        for (int u = 0; u < kU; ++u)
#pragma unroll
                            for (int k = 0; k < 3; ++k) {
                                mn[k] = fmin(mn[k], v[u][k]);
                                mx[k] = fmax(mx[k], v[u][k]);
                            }
                    }
                    block_minmax(mn, mx, a.bpart + (size_t)q * 6, sm);
                }
            }
            gsync(G, 10);
        }
        // ---- S1: box, centre, r^2, split decision; partition items of splitting clusters
        for (int i = gt; i < nl; i += gsz) {
            const int c = L0 + i;
            double lo[3], hi[3];
            const int q0 = a.bpre[i], q1 = a.bpre[i + 1];
            for (int k = 0; k < 3; ++k) {
                lo[k] = a.bpart[(size_t)q0 * 6 + k];
                hi[k] = a.bpart[(size_t)q0 * 6 + 3 + k];
            }
            for (int q = q0 + 1; q < q1; ++q)
                for (int k = 0; k < 3; ++k) {
                    lo[k] = fmin(lo[k], a.bpart[(size_t)q * 6 + k]);
                    hi[k] = fmax(hi[k], a.bpart[(size_t)q * 6 + 3 + k]);
                }
            double ctr[3], h[3], L[3];
            for (int k = 0; k < 3; ++k) {
                a.box[(size_t)c * 6 + k] = lo[k];
                a.box[(size_t)c * 6 + 3 + k] = hi[k];
                ctr[k] = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
                L[k] = __dsub_rn(hi[k], lo[k]);
                h[k] = __dmul_rn(0.5, L[k]);
            }
            const double r2 = __dadd_rn(__dadd_rn(__dmul_rn(h[0], h[0]), __dmul_rn(h[1], h[1])), __dmul_rn(h[2], h[2]));
            a.cr[c] = make_double4(ctr[0], ctr[1], ctr[2], r2);
            double lmax = 0.0;
            for (int k = 0; k < 3; ++k)
                if (L[k] > lmax) lmax = L[k];
            const double thr = __dmul_rn(lmax, kInvSqrt2);
            int mask = 0;
            if (lmax > 0.0)
                for (int k = 0; k < 3; ++k)
                    if (L[k] > thr) mask |= 1 << k;
            a.split[i] = make_double4(ctr[0], ctr[1], ctr[2], (double)mask);
            const int4 tp = a.topo[c];
            const int n = tp.y - tp.x;
            a.kids[i] = n > a.N0 ? (n + kChk - 1) / kChk : 0;  // partition items (-> children in S4)
        }
        gsync(G, 11);
        // ---- S2: partition items
        if (blockIdx.x == 0) {
            const int I = block_scan(nl, [&](int i) { return a.kids[i]; }, a.ipre, sm);
            if (tid == 0) a.ctr[kItems] = I;
        }
        gsync(G, 12);
        const int I = ld(a.ctr + kItems);
        if (I == 0) break;  // no cluster of this level splits: they are all leaves
        // ---- S3: child-code counts per item
        if (I >= kWarpMode * nb * kNW) {  // a warp per item
            for (int q = blockIdx.x * kNW + w; q < I; q += nb * kNW) {
                const int i = warp_find(a.ipre, nl, q);
                const int4 tp = a.topo[L0 + i];
                const int b = tp.x + (q - a.ipre[i]) * kChk, e = min(tp.y, b + kChk);
                const double4 sp = a.split[i];
                int c8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                for (int t0 = b; t0 < e; t0 += kUW * 32) {
                    double v[kUW][3];
#pragma unroll
                    for (int u = 0; u < kUW; ++u) {
                        const int j = min(t0 + u * 32 + lane, e - 1);
                        v[u][0] = cx[j];
                        v[u][1] = cy[j];
                        v[u][2] = cz[j];
                    }
#pragma unroll
                    for (int u = 0; u < kUW; ++u) {
                        const int code = t0 + u * 32 + lane < e ? child_code(v[u][0], v[u][1], v[u][2], sp) : 8;
#pragma unroll
                        for (int k = 0; k < 8; ++k) c8[k] += code == k;
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k)
                    for (int o = 16; o; o >>= 1) c8[k] += __shfl_xor_sync(0xffffffffu, c8[k], o);
                if (lane == 0)
#pragma unroll
                    for (int k = 0; k < 8; ++k) a.cnt[(size_t)q * 8 + k] = c8[k];
            }
        } else {  // a CTA per item
            for (int q = blockIdx.x; q < I; q += nb) {
                const int fi = warp_find(a.ipre, nl, q);
                if (tid < 8) sm.hist[tid] = 0;
                if (tid == 0) sm.item_cl = fi;
                __syncthreads();
                const int i = sm.item_cl;
                const int4 tp = a.topo[L0 + i];
                const int b = tp.x + (q - a.ipre[i]) * kChk, e = min(tp.y, b + kChk);
                const double4 sp = a.split[i];
                for (int t0 = b; t0 < e; t0 += kU * kBT) {  // CTA-uniform trip count (__match_any_sync below)
                    double v[kU][3];
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int j = min(t0 + u * kBT + tid, e - 1);
                        v[u][0] = cx[j];
                        v[u][1] = cy[j];
                        v[u][2] = cz[j];
                    }
#pragma unroll
                    for (int u = 0; u < kU; ++u) {
                        const int code = t0 + u * kBT + tid < e ? child_code(v[u][0], v[u][1], v[u][2], sp) : 8;
                        const unsigned peers = __match_any_sync(0xffffffffu, code);
                        if (code < 8 && lane == __ffs(peers) - 1) atomicAdd(&sm.hist[code], __popc(peers));
                    }
                }
                __syncthreads();
                if (tid < 8) a.cnt[(size_t)q * 8 + tid] = sm.hist[tid];
                __syncthreads();
            }
        }
        gsync(G, 13);
        // ---- S4: warp per splitting cluster: child sizes, stable per-item offsets
        for (int i = (blockIdx.x * kNW + w); i < nl; i += nb * kNW) {
            const int q0 = a.ipre[i], q1 = a.ipre[i + 1];
            if (q1 == q0) {
                if (lane == 0) a.kids[i] = 0;
                continue;
            }
            int tot[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) tot[k] = 0;
            for (int q = q0 + lane; q < q1; q += 32)
#pragma unroll
                for (int k = 0; k < 8; ++k) tot[k] += a.cnt[(size_t)q * 8 + k];
            int ne = 0;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                for (int o = 16; o; o >>= 1) tot[k] += __shfl_xor_sync(0xffffffffu, tot[k], o);
                ne += tot[k] > 0;
            }
            if (ne < 2) {  // degenerate: lmax == 0 or all particles on one side
                if (lane == 0) {
                    a.kids[i] = 0;
                    atomicAdd(a.ctr + kDeg, 1);
                }
                continue;
            }
            const int4 tp = a.topo[L0 + i];
            int run[8], pos = tp.x;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                run[k] = pos;
                pos += tot[k];
            }
            for (int q = q0; q < q1; q += 32) {
                const int qq = q + lane;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int v = qq < q1 ? a.cnt[(size_t)qq * 8 + k] : 0;
                    int inc = v;
                    for (int o = 1; o < 32; o <<= 1) {
                        const int t = __shfl_up_sync(0xffffffffu, inc, o);
                        if (lane >= o) inc += t;
                    }
                    if (qq < q1) a.off[(size_t)qq * 8 + k] = run[k] + inc - v;
                    run[k] += __shfl_sync(0xffffffffu, inc, 31);
                }
            }
            if (lane == 0) {
                a.kids[i] = ne;
                for (int k = 0; k < 8; ++k) a.tot8[(size_t)i * 8 + k] = tot[k];
            }
        }
        gsync(G, 14);
        // ---- S5: children (BFS ids L1 + prefix), their records, the next level's box items
        if (blockIdx.x == 0) {
            int* kpre = a.bpre;  // the level's box prefix is no longer needed
            const int NL = block_scan(nl, [&](int i) { return a.kids[i]; }, kpre, sm);
            const bool over = L1 + NL > a.ccap || l + 2 > a.maxlev;
            if (over) {  // table too small (or too deep): no split at this level; the host rebuilds
                for (int i = tid; i < nl; i += kBT) a.kids[i] = 0;
                if (tid == 0) {
                    a.ctr[kOverflow] = 1;
                    lstart[l + 2] = L1;
                }
            } else {
                for (int i = tid; i < nl; i += kBT) {
                    const int ne = a.kids[i];
                    if (!ne) continue;
                    const int c = L0 + i, fc = L1 + kpre[i];
                    int4 tp = a.topo[c];
                    int st = tp.x, id = fc;
                    for (int k = 0; k < 8; ++k) {
                        const int n = a.tot8[(size_t)i * 8 + k];
                        if (!n) continue;
                        a.topo[id] = make_int4(st, st + n, -1, 0);
                        a.level[id] = l + 1;
                        a.parent[id] = c;
                        st += n;
                        ++id;
                    }
                    tp.z = fc;
                    tp.w = ne;
                    a.topo[c] = tp;
                }
                __syncthreads();
                // box items of the next level (its clusters are [L1, L1 + NL))
                const int B = block_scan(NL, [&](int j) {
                    const int4 tp = a.topo[L1 + j];
                    return (tp.y - tp.x + kChk - 1) / kChk;
                }, a.bpre, sm);
                if (tid == 0) {
                    a.ctr[kBoxItems] = B;
                    lstart[l + 2] = L1 + NL;
                }
            }
        }
        gsync(G, 15);
        // ---- S6: stable scatter of the splitting clusters' items into x2.. ; S7: copy back
        {
            const int* cp = (l & 1) ? a.perm2 : a.perm;
            double* nx = (l & 1) ? a.x : a.x2;
            double* ny = (l & 1) ? a.y : a.y2;
            double* nz = (l & 1) ? a.z : a.z2;
            int* np = (l & 1) ? a.perm : a.perm2;
            const unsigned lt = (1u << lane) - 1u;
            if (I >= kWarpMode * nb * kNW) {  // a warp per item, 32-element tiles in order
                for (int q = blockIdx.x * kNW + w; q < I; q += nb * kNW) {
                    const int i = warp_find(a.ipre, nl, q);
                    if (a.kids[i] == 0) continue;  // degenerate leaf: its particles stay
                    const int4 tp = a.topo[L0 + i];
                    const int b = tp.x + (q - a.ipre[i]) * kChk, e = min(tp.y, b + kChk);
                    const double4 sp = a.split[i];
                    int base = lane < 8 ? a.off[(size_t)q * 8 + lane] : 0;  // lane k: next position of code k
                    for (int t0 = b; t0 < e; t0 += kUS * 32) {
                        double px[kUS], py[kUS], pz[kUS];
                        int pi[kUS];
#pragma unroll
                        for (int u = 0; u < kUS; ++u) {  // kUS tiles' loads in flight, then the tiles in order (stable)
                            const int j = min(t0 + u * 32 + lane, e - 1);
                            px[u] = cx[j];
                            py[u] = cy[j];
                            pz[u] = cz[j];
                            pi[u] = cp[j];
                        }
#pragma unroll
                        for (int u = 0; u < kUS; ++u) {
                            const int tile = t0 + u * 32;
                            if (tile >= e) break;  // warp-uniform
                            const bool valid = tile + lane < e;
                            const int code = valid ? child_code(px[u], py[u], pz[u], sp) : 8;
                            const unsigned peers = __match_any_sync(0xffffffffu, code);
                            const int pos = __shfl_sync(0xffffffffu, base, code & 7) + __popc(peers & lt);
                            KITC_DCHECK(!valid || (pos >= tp.x && pos < tp.y));  // children partition the parent
                            if (valid) {
                                nx[pos] = px[u];
                                ny[pos] = py[u];
                                nz[pos] = pz[u];
                                np[pos] = pi[u];
                            }
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                const unsigned mk = __ballot_sync(0xffffffffu, code == k);
                                if (lane == k) base += __popc(mk);
                            }
                        }
                    }
                }
            } else {  // a CTA per item, kBT-element tiles in order (warp ranks + per-warp prefix)
                for (int q = blockIdx.x; q < I; q += nb) {
                    const int fi = warp_find(a.ipre, nl, q);
                    if (tid == 0) sm.item_cl = fi;
                    __syncthreads();
                    const int i = sm.item_cl;
                    if (a.kids[i] == 0) {
                        __syncthreads();
                        continue;
                    }
                    const int4 tp = a.topo[L0 + i];
                    const int b = tp.x + (q - a.ipre[i]) * kChk, e = min(tp.y, b + kChk);
                    const double4 sp = a.split[i];
                    if (tid < 8) sm.sc.base[tid] = a.off[(size_t)q * 8 + tid];
                    for (int t0 = b; t0 < e; t0 += kU * kBT) {
                        double px[kU], py[kU], pz[kU];
                        int pi[kU];
#pragma unroll
                        for (int u = 0; u < kU; ++u) {  // kU tiles' loads in flight, then the tiles in order (stable)
                            const int j = min(t0 + u * kBT + tid, e - 1);
                            px[u] = cx[j];
                            py[u] = cy[j];
                            pz[u] = cz[j];
                            pi[u] = cp[j];
                        }
#pragma unroll
                        for (int u = 0; u < kU; ++u) {
                            const int tile = t0 + u * kBT;
                            if (tile >= e) break;  // CTA-uniform
                            if (tid < kNW * 8) sm.sc.wcnt[tid / 8][tid % 8] = 0;
                            __syncthreads();
                            const bool valid = tile + tid < e;
                            const int code = valid ? child_code(px[u], py[u], pz[u], sp) : 8;
                            const unsigned peers = __match_any_sync(0xffffffffu, code);
                            const int rank = __popc(peers & lt);
                            if (valid && rank == 0) sm.sc.wcnt[w][code] = __popc(peers);
                            __syncthreads();
                            if (valid) {
                                int pos = sm.sc.base[code] + rank;
                                for (int k = 0; k < w; ++k) pos += sm.sc.wcnt[k][code];
                                KITC_DCHECK(pos >= tp.x && pos < tp.y);  // children partition the parent
                                nx[pos] = px[u];
                                ny[pos] = py[u];
                                nz[pos] = pz[u];
                                np[pos] = pi[u];
                            }
                            __syncthreads();
                            if (tid < 8) {
                                int sum = 0;
                                for (int k = 0; k < kNW; ++k) sum += sm.sc.wcnt[k][tid];
                                sm.sc.base[tid] += sum;
                            }
                            __syncthreads();
                        }
                    }
                }
            }
        }
        gsync(G, 16);
        if (ld(lstart + l + 2) == L1) {  // no children (overflow): stop
            ++l;
            break;
        }
    }
    // levels 0 .. nlev-1 hold clusters [lstart[0], lstart[nlev])
    gsync(G, 20);
    int nlev = 0;
    while (nlev <= a.maxlev && ld(lstart + nlev + 1) > ld(lstart + nlev)) ++nlev;
    const int C = ld(lstart + nlev);
    // ---- leaves and warp batches in range order: bottom-up subtree counts ...
    for (int lv = nlev - 1; lv >= 0; --lv) {
        const int b0 = ld(lstart + lv), b1 = ld(lstart + lv + 1);
        for (int c = b0 + gt; c < b1; c += gsz) {
            const int4 tp = a.topo[c];
            int sl = 0, sb = 0;
            if (tp.w == 0) {
                sl = 1;
                sb = (tp.y - tp.x + kBatch - 1) / kBatch;
            } else {
                for (int k = 0; k < tp.w; ++k) {
                    sl += a.subl[tp.z + k];
                    sb += a.subb[tp.z + k];
                }
            }
            a.subl[c] = sl;
            a.subb[c] = sb;
        }
        gsync(G, 21);
    }
    // ... and top-down offsets (children in code order = range order)
    if (gt == 0) {
        a.loff[0] = 0;
        a.boff[0] = 0;
    }
    gsync(G, 22);
    for (int lv = 0; lv < nlev; ++lv) {
        const int b0 = ld(lstart + lv), b1 = ld(lstart + lv + 1);
        for (int c = b0 + gt; c < b1; c += gsz) {
            const int4 tp = a.topo[c];
            const int lo_ = a.loff[c], bo = a.boff[c];
            if (tp.w == 0) {
                a.leaves[lo_] = make_int4(tp.x, tp.y, c, bo);
            } else {
                int r = lo_, rb = bo;
                for (int k = 0; k < tp.w; ++k) {
                    a.loff[tp.z + k] = r;
                    a.boff[tp.z + k] = rb;
                    r += a.subl[tp.z + k];
                    rb += a.subb[tp.z + k];
                }
            }
        }
        gsync(G, 23);
    }
    const int nleaves = a.subl[0], nbatches = a.subb[0];
    if (gt == 0) {
        a.ctr[kC] = C;
        a.ctr[kLevels] = nlev;
        a.ctr[kLeaves] = nleaves;
        a.ctr[kBatches] = nbatches;
    }
}

// Each leaf's particles into buffer 0 (a leaf of odd level was left in buffer 1 by
// the ping-pong scatter), its targets in Morton order of their position in the
// leaf box (7 bits per axis; a stable block radix sort of (key, index), so ties
// keep the sorted order), and its warp batches = kBatch consecutive entries of
// that order.  Batching only: no result depends on it.  Leaves larger than
// kSortMax (degenerate ones) keep the sorted order.  Grid-stride over the leaves
// (their number is read on the device).
constexpr int kLT = 256, kLI = kSortMax / kLT;
__global__ void __launch_bounds__(kLT) k_leaf_order(const BuildArgs a) {
    using Sort = cub::BlockRadixSort<unsigned, kLT, kLI, int, 4>;
    __shared__ typename Sort::TempStorage tmp;
    const int nleaves = a.ctr[kLeaves];
    for (int li = blockIdx.x; li < nleaves; li += gridDim.x) {
        const int4 lf = a.leaves[li];
        const int b = lf.x, n = lf.y - lf.x, c = lf.z;
        if (a.level[c] & 1)
            for (int i = b + threadIdx.x; i < lf.y; i += kLT) {
                a.x[i] = a.x2[i];
                a.y[i] = a.y2[i];
                a.z[i] = a.z2[i];
                a.perm[i] = a.perm2[i];
            }
        for (int i = threadIdx.x; i * kBatch < n; i += kLT) {
            a.bstart[lf.w + i] = b + i * kBatch;
            a.bcount[lf.w + i] = min(kBatch, n - i * kBatch);
        }
        if (n > kSortMax) {
            for (int i = threadIdx.x; i < n; i += kLT) a.tord[b + i] = b + i;
            continue;
        }
        const double* X = (a.level[c] & 1) ? a.x2 : a.x;
        const double* Y = (a.level[c] & 1) ? a.y2 : a.y;
        const double* Z = (a.level[c] & 1) ? a.z2 : a.z;
        double lo[3], sc[3];
        for (int k = 0; k < 3; ++k) {
            lo[k] = a.box[(size_t)c * 6 + k];
            const double wd = a.box[(size_t)c * 6 + 3 + k] - lo[k];
            sc[k] = wd > 0.0 ? 127.999 / wd : 0.0;
        }
        unsigned key[kLI];
        int val[kLI];
#pragma unroll
        for (int u = 0; u < kLI; ++u) {  // blocked arrangement: thread t holds items t kLI + u
            const int i = threadIdx.x * kLI + u;
            key[u] = 0xffffffffu;  // padding sorts last
            val[u] = i;
            if (i < n) {
                const unsigned qx = (unsigned)fmin(fmax((X[b + i] - lo[0]) * sc[0], 0.0), 127.0);
                const unsigned qy = (unsigned)fmin(fmax((Y[b + i] - lo[1]) * sc[1], 0.0), 127.0);
                const unsigned qz = (unsigned)fmin(fmax((Z[b + i] - lo[2]) * sc[2], 0.0), 127.0);
                key[u] = spread3(qx) | (spread3(qy) << 1) | (spread3(qz) << 2);
            }
        }
        Sort(tmp).Sort(key, val, 0, 21);
#pragma unroll
        for (int u = 0; u < kLI; ++u) {
            const int i = threadIdx.x * kLI + u;
            if (i < n) a.tord[b + i] = b + val[u];
        }
        __syncthreads();  // tmp is reused by the next leaf
    }
}

template <class T>
static size_t bytes_of(int64_t n) {
    return (size_t)std::max<int64_t>(n, 1) * sizeof(T);
}

}  // namespace

#ifdef KITC_BUILD_PROF
extern "C" int kitc_build_prof(unsigned long long* out, int cap) {
    int n = 0;
    cudaMemcpyFromSymbol(&n, g_bprof_n, sizeof(int));
    n = n < cap ? n : cap;
    cudaMemcpyFromSymbol(out, g_bprof, n * sizeof(unsigned long long));
    int z = 0;
    cudaMemcpyToSymbol(g_bprof_n, &z, sizeof(int));
    return n;
}
#endif

int64_t tree_cluster_cap(int64_t N, int32_t N0) {
    // first guess of the cluster-table size: ~16 N / (N0 + 1) + 1024, never above the
    // worst case 2N - 1 (every internal cluster has >= 2 children, every leaf >= 1 particle)
    const int64_t guess = 16 * (N / ((int64_t)N0 + 1)) + 1024;
    return std::max<int64_t>(1, std::min<int64_t>(2 * N - 1, guess));
}

// device bytes of every build buffer, in the order build_tree ensures them
struct BuildSizes {
    int64_t icap, nbcap;
    size_t b[26];
};
static BuildSizes build_sizes(int64_t N, int64_t ccap, int grid) {
    BuildSizes z;
    z.icap = N / kChk + ccap + 1 + grid;
    z.nbcap = (N + kBatch - 1) / kBatch + ccap;
    const size_t d = bytes_of<double>(N), i = bytes_of<int>(N);
    const size_t v[25] = {d, d, d, i, d, d, d, i, i,                                        // x y z perm x2 y2 z2 perm2 tord
                          bytes_of<int4>(ccap), bytes_of<int>(ccap), bytes_of<int>(ccap),    // topo level parent
                          bytes_of<double>(6 * ccap), bytes_of<double4>(ccap),              // box cr
                          bytes_of<double4>(ccap), 2 * bytes_of<int>(ccap + 1), bytes_of<int>(ccap),
                          bytes_of<int>(8 * ccap), bytes_of<double>(6 * z.icap), 2 * bytes_of<int>(8 * z.icap),
                          4 * bytes_of<int>(ccap), bytes_of<int4>(ccap), bytes_of<int>(z.nbcap),
                          bytes_of<int>(z.nbcap), bytes_of<int>(kNCtr + kMaxLevels + 2)};
    for (int k = 0; k < 25; ++k) z.b[k] = v[k];
    return z;
}

size_t tree_bytes(int64_t N, int64_t ccap) {
    const BuildSizes z = build_sizes(N, ccap, 1024);
    size_t tot = 0;
    for (size_t v : z.b) tot += dev_alloc_bytes(v);
    return tot;
}

kitc_status build_tree(kitc_tree* t, const double* xyz, int64_t N64, int32_t N0, cudaStream_t s) {
    if (N64 < 1 || N64 > 0x3fffffffLL) return set_error(KITC_EINVAL, "kitc_build_tree: N out of range");
    if (N0 < 1) return set_error(KITC_EINVAL, "kitc_build_tree: N0 < 1");
    if (!xyz) return set_error(KITC_EINVAL, "kitc_build_tree: xyz is NULL");
    const int N = (int)N64;
    t->built = false;
    t->weights_ready = false;
    t->grid_n = -1;
    t->host_topo = false;
    t->stream = s;
    t->N = N;
    t->N0 = N0;
    static int grid = 0;
    if (!grid) {
        int dev = 0, sms = 0, occ = 0;
        KITC_CUDA(cudaGetDevice(&dev));
        KITC_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        KITC_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_build, kBT, 0));
        if (occ < 1) return set_error(KITC_ECUDA, "kitc_build_tree: build kernel cannot be resident");
        grid = sms;  // one CTA per SM (grid-wide barriers: fewer arrivals)
    }
    int64_t ccap = std::max<int64_t>(t->ccap, tree_cluster_cap(N, N0));
    for (int attempt = 0;; ++attempt) {
        ccap = std::min<int64_t>(ccap, 2 * (int64_t)N - 1);
        const BuildSizes z = build_sizes(N, ccap, grid);
        const int64_t icap = z.icap, nbcap = z.nbcap;
        kitc::DevBuf* bufs[25] = {&t->x, &t->y, &t->z, &t->perm, &t->x2, &t->y2, &t->z2, &t->perm2, &t->tord,
                                  &t->topo, &t->clevel, &t->cparent, &t->box, &t->cr, &t->b_split, &t->b_pre,
                                  &t->b_kids, &t->b_tot8, &t->b_bpart, &t->b_cnt, &t->b_sub, &t->leaves, &t->bstart,
                                  &t->bcount, &t->b_ctr};
        for (int k = 0; k < 25; ++k) KITC_TRY(bufs[k]->ensure(z.b[k], s));
        KITC_TRY(t->h_ctr.ensure(kNCtr * sizeof(int)));
        KITC_CUDA(cudaMemsetAsync(t->b_ctr.p, 0, (kNCtr + kMaxLevels + 2) * sizeof(int), s));
        BuildArgs a;
        a.xyz = xyz;
        a.N = N;
        a.N0 = N0;
        a.ccap = (int)ccap;
        a.maxlev = kMaxLevels;
        a.nbatch_cap = (int)nbcap;
        a.x = t->x.as<double>();
        a.y = t->y.as<double>();
        a.z = t->z.as<double>();
        a.perm = t->perm.as<int>();
        a.x2 = t->x2.as<double>();
        a.y2 = t->y2.as<double>();
        a.z2 = t->z2.as<double>();
        a.perm2 = t->perm2.as<int>();
        a.topo = t->topo.as<int4>();
        a.level = t->clevel.as<int>();
        a.parent = t->cparent.as<int>();
        a.box = t->box.as<double>();
        a.cr = t->cr.as<double4>();
        a.split = t->b_split.as<double4>();
        a.bpre = t->b_pre.as<int>();
        a.ipre = a.bpre + (ccap + 1);
        a.kids = t->b_kids.as<int>();
        a.tot8 = t->b_tot8.as<int>();
        a.bpart = t->b_bpart.as<double>();
        a.cnt = t->b_cnt.as<int>();
        a.off = a.cnt + 8 * icap;
        a.subl = t->b_sub.as<int>();
        a.subb = a.subl + ccap;
        a.loff = a.subb + ccap;
        a.boff = a.loff + ccap;
        a.ctr = t->b_ctr.as<int>();
        a.leaves = t->leaves.as<int4>();
        a.tord = t->tord.as<int>();
        a.bstart = t->bstart.as<int>();
        a.bcount = t->bcount.as<int>();
        void* args[] = {&a};
        KITC_CUDA(cudaLaunchCooperativeKernel((void*)k_build, dim3(grid), dim3(kBT), args, 0, s));
        note_launch();
        k_leaf_order<<<grid * 8, kLT, 0, s>>>(a);
        note_launch();
        int* hc = t->h_ctr.as<int>();
        KITC_CUDA(cudaMemcpyAsync(hc, t->b_ctr.p, kNCtr * sizeof(int), cudaMemcpyDeviceToHost, s));
        KITC_CUDA(cudaStreamSynchronize(s));  // the build's one host synchronisation
        if (hc[kNonFinite]) return set_error(KITC_EINVAL, "kitc_build_tree: non-finite coordinate");
        if (hc[kOverflow]) {
            if (ccap >= 2 * (int64_t)N - 1 || attempt > 8)
                return set_error(KITC_EINVAL, "kitc_build_tree: tree deeper than the supported number of levels");
            ccap *= 4;
            continue;
        }
        t->ccap = ccap;
        t->nclusters = hc[kC];
        t->depth = hc[kLevels] - 1;
        t->ndegenerate = hc[kDeg];
        t->nleaves = hc[kLeaves];
        t->nbatches = hc[kBatches];
        t->built = true;
        return KITC_OK;
    }
}

const int* tree_level_starts(const kitc_tree* t) { return t->b_ctr.as<int>() + kNCtr; }

// host copies of the topology (kitc_tree_export, kitc_batch_targets): read once per build
kitc_status ensure_host_topology(const kitc_tree* t) {
    if (t->host_topo) return KITC_OK;
    const int64_t C = t->nclusters, L = t->nleaves;
    std::vector<int4> tp(C), lv(L);
    std::vector<int> level(C), parent(C);
    cudaStream_t s = t->stream;
    KITC_CUDA(cudaMemcpyAsync(tp.data(), t->topo.p, C * sizeof(int4), cudaMemcpyDeviceToHost, s));
    KITC_CUDA(cudaMemcpyAsync(level.data(), t->clevel.p, C * sizeof(int), cudaMemcpyDeviceToHost, s));
    KITC_CUDA(cudaMemcpyAsync(parent.data(), t->cparent.p, C * sizeof(int), cudaMemcpyDeviceToHost, s));
    KITC_CUDA(cudaMemcpyAsync(lv.data(), t->leaves.p, L * sizeof(int4), cudaMemcpyDeviceToHost, s));
    KITC_CUDA(cudaStreamSynchronize(s));
    t->h_begin.resize(C);
    t->h_end.resize(C);
    t->h_first.resize(C);
    t->h_nchild.resize(C);
    for (int64_t c = 0; c < C; ++c) {
        t->h_begin[c] = tp[c].x;
        t->h_end[c] = tp[c].y;
        t->h_first[c] = tp[c].z;
        t->h_nchild[c] = tp[c].w;
    }
    t->h_level.assign(level.begin(), level.end());
    t->h_parent.assign(parent.begin(), parent.end());
    t->h_leaf_begin.resize(L);
    t->h_leaf_boff.resize(L + 1);
    for (int64_t i = 0; i < L; ++i) {
        t->h_leaf_begin[i] = lv[i].x;
        t->h_leaf_boff[i] = lv[i].w;
    }
    t->h_leaf_boff[L] = t->nbatches;
    t->host_topo = true;
    return KITC_OK;
}

}  // namespace kitc
