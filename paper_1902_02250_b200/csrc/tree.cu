// tree.cu -- level-synchronous device build of the KITC cluster tree.
//
// Rule (§6; readings A1-A4): minimal bounding
// box per cluster; a cluster with count > N0 is bisected at its midpoint along
// every side L_l > lmax / sqrt(2); x_l >= mid_l -> upper half; children = the
// nonempty code groups (code = bx | by<<1 | bz<<2) in ascending code, formed by
// a STABLE partition; a split leaving < 2 nonempty children is a (degenerate)
// leaf.  The ordering is integer-exact: per level, (1) a min/max reduction over
// (cluster, chunk) work items, (2) the split decision with round-to-nearest
// intrinsics (no FMA contraction), (3) per-chunk code counts, (4) a host
// exclusive scan of the counts in chunk order, (5) a stable in-chunk scatter
// (warp __match_any_sync ranks + per-warp prefix).  Clusters are numbered BFS
// (level, then range start); the host keeps the topology.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "kitc_internal.cuh"

namespace kitc {

namespace {

constexpr int kBoxChunk = 8192;   // particles per bbox work item
constexpr int kPartChunk = 4096;  // particles per partition work item
constexpr int kThreads = 256;
constexpr double kInvSqrt2 = 0.7071067811865476;  // 1/sqrt(2), RN (reading A2)

struct Item {
    int32_t cl;  // level-local cluster index
    int32_t b, e;
    int32_t pad;
};

__global__ void k_init(const double* __restrict__ xyz, int N, double* __restrict__ x,
                       double* __restrict__ y, double* __restrict__ z, int* __restrict__ perm,
                       int* __restrict__ flag) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= N) return;
    double a = xyz[3 * (size_t)i], b = xyz[3 * (size_t)i + 1], c = xyz[3 * (size_t)i + 2];
    x[i] = a;
    y[i] = b;
    z[i] = c;
    perm[i] = i;
    if (!isfinite(a) || !isfinite(b) || !isfinite(c)) atomicOr(flag, 1);
}

__device__ __forceinline__ double warp_min(double v) {
    for (int o = 16; o; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_max(double v) {
    for (int o = 16; o; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// (1) per work item: min/max of x, y, z over [b, e)  -> part[item][6]
__global__ void __launch_bounds__(kThreads) k_bbox_partial(const Item* __restrict__ items,
                                                           const double* __restrict__ x,
                                                           const double* __restrict__ y,
                                                           const double* __restrict__ z,
                                                           double* __restrict__ part) {
    const Item it = items[blockIdx.x];
    double mn[3] = {INFINITY, INFINITY, INFINITY}, mx[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int i = it.b + threadIdx.x; i < it.e; i += kThreads) {
        double v[3] = {x[i], y[i], z[i]};
#pragma unroll
        for (int l = 0; l < 3; ++l) {
            mn[l] = fmin(mn[l], v[l]);
            mx[l] = fmax(mx[l], v[l]);
        }
    }
    __shared__ double sm[kThreads / 32][6];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int l = 0; l < 3; ++l) {
        mn[l] = warp_min(mn[l]);
        mx[l] = warp_max(mx[l]);
    }
    if (lane == 0)
        for (int l = 0; l < 3; ++l) {
            sm[w][l] = mn[l];
            sm[w][3 + l] = mx[l];
        }
    __syncthreads();
    if (threadIdx.x < 6) {
        double v = sm[0][threadIdx.x];
        for (int k = 1; k < kThreads / 32; ++k)
            v = threadIdx.x < 3 ? fmin(v, sm[k][threadIdx.x]) : fmax(v, sm[k][threadIdx.x]);
        part[(size_t)blockIdx.x * 6 + threadIdx.x] = v;
    }
}

// (2) per cluster of the level: box, centre, r^2 and the split decision.
//   centre c = 0.5 (lo + hi), h = 0.5 (hi - lo), r^2 = (hx^2 + hy^2) + hz^2
//   (reading A4); split_l = L_l > lmax * (1/sqrt 2); mid = c.  All RN.
__global__ void k_bbox_final(int nl, const int* __restrict__ first_item,
                             const int* __restrict__ cid, const double* __restrict__ part,
                             double* __restrict__ box, double4* __restrict__ cr,
                             double4* __restrict__ split) {
    int l = blockIdx.x * blockDim.x + threadIdx.x;
    if (l >= nl) return;
    double lo[3], hi[3];
    const int i0 = first_item[l], i1 = first_item[l + 1];
    for (int k = 0; k < 3; ++k) {
        lo[k] = part[(size_t)i0 * 6 + k];
        hi[k] = part[(size_t)i0 * 6 + 3 + k];
    }
    for (int i = i0 + 1; i < i1; ++i)
        for (int k = 0; k < 3; ++k) {
            lo[k] = fmin(lo[k], part[(size_t)i * 6 + k]);
            hi[k] = fmax(hi[k], part[(size_t)i * 6 + 3 + k]);
        }
    const int c = cid[l];
    double ctr[3], h[3], L[3];
    for (int k = 0; k < 3; ++k) {
        box[(size_t)c * 6 + k] = lo[k];
        box[(size_t)c * 6 + 3 + k] = hi[k];
        ctr[k] = __dmul_rn(0.5, __dadd_rn(lo[k], hi[k]));
        L[k] = __dsub_rn(hi[k], lo[k]);
        h[k] = __dmul_rn(0.5, L[k]);
    }
    double r2 = __dadd_rn(__dadd_rn(__dmul_rn(h[0], h[0]), __dmul_rn(h[1], h[1])), __dmul_rn(h[2], h[2]));
    cr[c] = make_double4(ctr[0], ctr[1], ctr[2], r2);
    double lmax = 0.0;
    for (int k = 0; k < 3; ++k)
        if (L[k] > lmax) lmax = L[k];
    const double thr = __dmul_rn(lmax, kInvSqrt2);
    int mask = 0;
    if (lmax > 0.0)
        for (int k = 0; k < 3; ++k)
            if (L[k] > thr) mask |= 1 << k;
    split[l] = make_double4(ctr[0], ctr[1], ctr[2], (double)mask);
}

__device__ __forceinline__ int child_code(double px, double py, double pz, const double4& sp) {
    const int mask = (int)sp.w;
    int code = 0;
    if ((mask & 1) && px >= sp.x) code |= 1;
    if ((mask & 2) && py >= sp.y) code |= 2;
    if ((mask & 4) && pz >= sp.z) code |= 4;
    return code;
}

// (3) per partition work item: counts of each child code.
__global__ void __launch_bounds__(kThreads) k_part_count(const Item* __restrict__ items,
                                                         const double* __restrict__ x,
                                                         const double* __restrict__ y,
                                                         const double* __restrict__ z,
                                                         const double4* __restrict__ split,
                                                         int* __restrict__ cnt) {
    __shared__ int c8[8];
    if (threadIdx.x < 8) c8[threadIdx.x] = 0;
    __syncthreads();
    const Item it = items[blockIdx.x];
    const double4 sp = split[it.cl];
    for (int i = it.b + threadIdx.x; i < it.e; i += kThreads)
        atomicAdd(&c8[child_code(x[i], y[i], z[i], sp)], 1);
    __syncthreads();
    if (threadIdx.x < 8) cnt[(size_t)blockIdx.x * 8 + threadIdx.x] = c8[threadIdx.x];
}

// (5) stable scatter of a work item into the scratch arrays at the host-scanned
// offsets off[item][code]; in-tile ranks from __match_any_sync + warp prefix.
__global__ void __launch_bounds__(kThreads) k_part_scatter(
    const Item* __restrict__ items, const int* __restrict__ off, const double* __restrict__ x,
    const double* __restrict__ y, const double* __restrict__ z, const int* __restrict__ perm,
    const double4* __restrict__ split, double* __restrict__ x2, double* __restrict__ y2,
    double* __restrict__ z2, int* __restrict__ perm2) {
    constexpr int NW = kThreads / 32;
    __shared__ int wcnt[NW][8];
    __shared__ int base[8];
    const Item it = items[blockIdx.x];
    const double4 sp = split[it.cl];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x < 8) base[threadIdx.x] = off[(size_t)blockIdx.x * 8 + threadIdx.x];
    const unsigned lt = (1u << lane) - 1u;
    for (int tile = it.b; tile < it.e; tile += kThreads) {
        if (threadIdx.x < NW * 8) wcnt[threadIdx.x / 8][threadIdx.x % 8] = 0;
        __syncthreads();
        const int i = tile + threadIdx.x;
        const bool valid = i < it.e;
        double px = 0, py = 0, pz = 0;
        int pi = 0, code = 8;
        if (valid) {
            px = x[i];
            py = y[i];
            pz = z[i];
            pi = perm[i];
            code = child_code(px, py, pz, sp);
        }
        const unsigned peers = __match_any_sync(0xffffffffu, code);
        const int rank = __popc(peers & lt);
        if (valid && rank == 0) wcnt[w][code] = __popc(peers);
        __syncthreads();
        if (valid) {
            int pos = base[code] + rank;
            for (int k = 0; k < w; ++k) pos += wcnt[k][code];
            x2[pos] = px;
            y2[pos] = py;
            z2[pos] = pz;
            perm2[pos] = pi;
        }
        __syncthreads();
        if (threadIdx.x < 8) {
            int s = 0;
            for (int k = 0; k < NW; ++k) s += wcnt[k][threadIdx.x];
            base[threadIdx.x] += s;
        }
        __syncthreads();  // wcnt is cleared at the top of the next tile
    }
}

__global__ void __launch_bounds__(kThreads) k_copy_back(const Item* __restrict__ items,
                                                        const double* __restrict__ x2,
                                                        const double* __restrict__ y2,
                                                        const double* __restrict__ z2,
                                                        const int* __restrict__ perm2,
                                                        double* __restrict__ x, double* __restrict__ y,
                                                        double* __restrict__ z, int* __restrict__ perm) {
    const Item it = items[blockIdx.x];
    for (int i = it.b + threadIdx.x; i < it.e; i += kThreads) {
        x[i] = x2[i];
        y[i] = y2[i];
        z[i] = z2[i];
        perm[i] = perm2[i];
    }
}

// Targets of each leaf in Morton order of their position inside the leaf box,
// so that a warp batch (kBatch consecutive entries) is spatially compact and
// its lanes take the same MAC decisions more often.  Batching only: every
// target's traversal and sums are independent of it.  Leaves larger than
// kSortMax (degenerate ones) keep their sorted order.
constexpr int kSortMax = 2048;

__device__ __forceinline__ unsigned int spread3(unsigned int v) {  // 10 bits -> every 3rd bit
    v &= 0x3ffu;
    v = (v | (v << 16)) & 0x030000ffu;
    v = (v | (v << 8)) & 0x0300f00fu;
    v = (v | (v << 4)) & 0x030c30c3u;
    v = (v | (v << 2)) & 0x09249249u;
    return v;
}

__global__ void __launch_bounds__(256) k_leaf_order(const int4* __restrict__ leaves, const double* __restrict__ box,
                                                    const double* __restrict__ x, const double* __restrict__ y,
                                                    const double* __restrict__ z, int* __restrict__ tord,
                                                    int* __restrict__ bstart, int* __restrict__ bcount) {
    __shared__ unsigned long long key[kSortMax];
    const int4 lf = leaves[blockIdx.x];
    const int b = lf.x, n = lf.y - lf.x, c = lf.z;
    // the leaf's warp batches: kBatch consecutive positions of its Morton order
    for (int i = threadIdx.x; i * kBatch < n; i += blockDim.x) {
        bstart[lf.w + i] = b + i * kBatch;
        bcount[lf.w + i] = min(kBatch, n - i * kBatch);
    }
    if (n > kSortMax) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) tord[b + i] = b + i;
        return;
    }
    int n2 = 1;
    while (n2 < n) n2 <<= 1;
    double lo[3], sc[3];
    for (int l = 0; l < 3; ++l) {
        lo[l] = box[(size_t)c * 6 + l];
        const double w = box[(size_t)c * 6 + 3 + l] - lo[l];
        sc[l] = w > 0.0 ? 1023.999 / w : 0.0;
    }
    for (int i = threadIdx.x; i < n2; i += blockDim.x) {
        unsigned long long k = ~0ull;
        if (i < n) {
            const unsigned qx = (unsigned)fmin(fmax((x[b + i] - lo[0]) * sc[0], 0.0), 1023.0);
            const unsigned qy = (unsigned)fmin(fmax((y[b + i] - lo[1]) * sc[1], 0.0), 1023.0);
            const unsigned qz = (unsigned)fmin(fmax((z[b + i] - lo[2]) * sc[2], 0.0), 1023.0);
            const unsigned m = spread3(qx) | (spread3(qy) << 1) | (spread3(qz) << 2);
            k = ((unsigned long long)m << 32) | (unsigned)i;
        }
        key[i] = k;
    }
    __syncthreads();
    for (int k = 2; k <= n2; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < n2; i += blockDim.x) {
                const int ixj = i ^ j;
                if (ixj > i) {
                    const unsigned long long a = key[i], bb = key[ixj];
                    if ((a > bb) == ((i & k) == 0)) {
                        key[i] = bb;
                        key[ixj] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < n; i += blockDim.x) tord[b + i] = b + (int)(key[i] & 0xffffffffu);
}

template <class T>
static size_t pad16(size_t n) {
    return (n * sizeof(T) + 15) / 16 * 16;
}

}  // namespace

// KITC_TRACE=1: host timestamps of the build phases on stderr (latency tuning only)
static bool trace_on() {
    static const bool on = [] {
        const char* e = std::getenv("KITC_TRACE");
        return e && *e == '1';
    }();
    return on;
}
static void trace(const char* what, int level) {
    if (!trace_on()) return;
    static auto t0 = std::chrono::steady_clock::now();
    const auto now = std::chrono::steady_clock::now();
    if (level < 0) t0 = now;
    std::fprintf(stderr, "[kitc build] %8.1f us  %s %d\n",
                 std::chrono::duration<double, std::micro>(now - t0).count(), what, level);
}

kitc_status build_tree(kitc_tree* t, const double* xyz, int64_t N64, int32_t N0, cudaStream_t s) {
    trace("start", -1);
    if (t->ev_stage) KITC_CUDA(cudaEventSynchronize(t->ev_stage));  // previous build's staging copies
    if (N64 < 1 || N64 > 0x7fffffffLL) return set_error(KITC_EINVAL, "kitc_build_tree: N out of range");
    if (N0 < 1) return set_error(KITC_EINVAL, "kitc_build_tree: N0 < 1");
    if (!xyz) return set_error(KITC_EINVAL, "kitc_build_tree: xyz is NULL");
    const int N = (int)N64;
    t->built = false;
    t->weights_ready = false;
    t->grid_n = -1;
    t->stream = s;
    t->N = N;
    t->N0 = N0;
    const size_t nd = (size_t)N * sizeof(double), ni = (size_t)N * sizeof(int);
    KITC_TRY(t->x.ensure(nd, s));
    KITC_TRY(t->y.ensure(nd, s));
    KITC_TRY(t->z.ensure(nd, s));
    KITC_TRY(t->perm.ensure(ni, s));
    KITC_TRY(t->x2.ensure(nd, s));
    KITC_TRY(t->y2.ensure(nd, s));
    KITC_TRY(t->z2.ensure(nd, s));
    KITC_TRY(t->perm2.ensure(ni, s));
    KITC_TRY(t->d_flag.ensure(sizeof(int), s));
    KITC_CUDA(cudaMemsetAsync(t->d_flag.p, 0, sizeof(int), s));
    double *x = t->x.as<double>(), *y = t->y.as<double>(), *z = t->z.as<double>();
    int* perm = t->perm.as<int>();
    k_init<<<(N + 255) / 256, 256, 0, s>>>(xyz, N, x, y, z, perm, t->d_flag.as<int>()); note_launch();
    KITC_CUDA(cudaGetLastError());

    auto& hb = t->h_begin;
    auto& he = t->h_end;
    auto& hl = t->h_level;
    auto& hp = t->h_parent;
    auto& hf = t->h_first;
    auto& hn = t->h_nchild;
    hb.assign(1, 0);
    he.assign(1, N);
    hl.assign(1, 0);
    hp.assign(1, -1);
    hf.assign(1, -1);
    hn.assign(1, 0);
    std::vector<int> cur(1, 0), next;
    int depth = 0, ndeg = 0;
    std::vector<Item> bitems, pitems, sitems;
    std::vector<int> first_item, pfirst, cand, offs;
    std::vector<int> host_cnt;
    int level = 0;
    while (!cur.empty()) {
        const int nl = (int)cur.size();
        const int ntot = (int)hb.size();
        KITC_TRY(t->box.ensure((size_t)ntot * 6 * sizeof(double), s, true));
        KITC_TRY(t->cr.ensure((size_t)ntot * sizeof(double4), s, true));
        // work items of this level
        bitems.clear();
        first_item.assign(1, 0);
        pitems.clear();
        pfirst.clear();
        cand.clear();
        for (int l = 0; l < nl; ++l) {
            const int c = cur[l];
            for (int b = hb[c]; b < he[c]; b += kBoxChunk)
                bitems.push_back(Item{l, b, std::min(he[c], b + kBoxChunk), 0});
            first_item.push_back((int)bitems.size());
            if (he[c] - hb[c] > N0) {
                cand.push_back(l);
                pfirst.push_back((int)pitems.size());
                for (int b = hb[c]; b < he[c]; b += kPartChunk)
                    pitems.push_back(Item{l, b, std::min(he[c], b + kPartChunk), 0});
            }
        }
        pfirst.push_back((int)pitems.size());
        const int nbi = (int)bitems.size(), npi = (int)pitems.size();
        // stage: bitems | pitems | first_item | cid
        const size_t o1 = pad16<Item>(nbi), o2 = o1 + pad16<Item>(npi), o3 = o2 + pad16<int>(nl + 1),
                     o4 = o3 + pad16<int>(nl);
        KITC_TRY(t->h_stage.ensure(o4));
        KITC_TRY(t->d_items.ensure(o4, s));
        char* hs = t->h_stage.as<char>();
        std::copy(bitems.begin(), bitems.end(), reinterpret_cast<Item*>(hs));
        std::copy(pitems.begin(), pitems.end(), reinterpret_cast<Item*>(hs + o1));
        std::copy(first_item.begin(), first_item.end(), reinterpret_cast<int*>(hs + o2));
        for (int l = 0; l < nl; ++l) reinterpret_cast<int*>(hs + o3)[l] = cur[l];
        KITC_CUDA(cudaMemcpyAsync(t->d_items.p, hs, o4, cudaMemcpyHostToDevice, s));
        char* ds = t->d_items.as<char>();
        KITC_TRY(t->d_part.ensure((size_t)nbi * 6 * sizeof(double), s));
        KITC_TRY(t->d_split.ensure((size_t)nl * sizeof(double4), s));
        KITC_TRY(t->d_cnt.ensure((size_t)std::max(npi, 1) * 8 * sizeof(int) + 16, s));
        k_bbox_partial<<<nbi, kThreads, 0, s>>>(reinterpret_cast<Item*>(ds), x, y, z, t->d_part.as<double>()); note_launch();
        k_bbox_final<<<(nl + 127) / 128, 128, 0, s>>>(nl, reinterpret_cast<int*>(ds + o2),
                                                    reinterpret_cast<int*>(ds + o3), t->d_part.as<double>(),
                                                    t->box.as<double>(), t->cr.as<double4>(),
                                                    t->d_split.as<double4>()); note_launch();
        if (npi)
            k_part_count<<<npi, kThreads, 0, s>>>(reinterpret_cast<Item*>(ds + o1), x, y, z,
                                                 t->d_split.as<double4>(), t->d_cnt.as<int>()); note_launch();
        KITC_CUDA(cudaGetLastError());
        trace("enqueued bbox/count", level);
        // read counts (+ the non-finite flag at level 0)
        const size_t cb = (size_t)npi * 8 * sizeof(int);
        KITC_TRY(t->h_cnt.ensure(cb + 16));
        int* hc = t->h_cnt.as<int>();
        if (npi) KITC_CUDA(cudaMemcpyAsync(hc, t->d_cnt.p, cb, cudaMemcpyDeviceToHost, s));
        if (level == 0) KITC_CUDA(cudaMemcpyAsync(hc + npi * 8, t->d_flag.p, sizeof(int), cudaMemcpyDeviceToHost, s));
        KITC_CUDA(cudaStreamSynchronize(s));
        trace("counts on host", level);
        if (level == 0 && hc[npi * 8] != 0)
            return set_error(KITC_EINVAL, "kitc_build_tree: non-finite coordinate");
        // (4) scan: offsets per (item, code); children
        next.clear();
        sitems.clear();
        offs.clear();
        for (size_t q = 0; q < cand.size(); ++q) {
            const int l = cand[q], c = cur[l];
            int tot[8] = {0};
            for (int i = pfirst[q]; i < pfirst[q + 1]; ++i)
                for (int k = 0; k < 8; ++k) tot[k] += hc[i * 8 + k];
            int ne = 0;
            for (int k = 0; k < 8; ++k) ne += tot[k] > 0;
            if (ne < 2) {  // degenerate: lmax == 0 or all particles on one side
                ++ndeg;
                continue;
            }
            int run[8], pos = hb[c];
            for (int k = 0; k < 8; ++k) {
                run[k] = pos;
                pos += tot[k];
            }
            for (int i = pfirst[q]; i < pfirst[q + 1]; ++i) {
                sitems.push_back(pitems[i]);
                for (int k = 0; k < 8; ++k) {
                    offs.push_back(run[k]);
                    run[k] += hc[i * 8 + k];
                }
            }
            hf[c] = (int)hb.size();
            hn[c] = ne;
            int st = hb[c];
            for (int k = 0; k < 8; ++k) {
                if (!tot[k]) continue;
                const int id = (int)hb.size();
                hb.push_back(st);
                he.push_back(st + tot[k]);
                hl.push_back(level + 1);
                hp.push_back(c);
                hf.push_back(-1);
                hn.push_back(0);
                next.push_back(id);
                st += tot[k];
            }
        }
        if (!sitems.empty()) {
            const int nsi = (int)sitems.size();
            const size_t p1 = pad16<Item>(nsi), p2 = p1 + pad16<int>((size_t)nsi * 8);
            KITC_TRY(t->d_off.ensure(p2, s));
            char* hs2 = t->h_cnt.as<char>();  // counts already consumed
            KITC_TRY(t->h_cnt.ensure(p2));
            hs2 = t->h_cnt.as<char>();
            std::copy(sitems.begin(), sitems.end(), reinterpret_cast<Item*>(hs2));
            std::copy(offs.begin(), offs.end(), reinterpret_cast<int*>(hs2 + p1));
            KITC_CUDA(cudaMemcpyAsync(t->d_off.p, hs2, p2, cudaMemcpyHostToDevice, s));
            char* dd = t->d_off.as<char>();
            k_part_scatter<<<nsi, kThreads, 0, s>>>(reinterpret_cast<Item*>(dd), reinterpret_cast<int*>(dd + p1),
                                                    x, y, z, perm, t->d_split.as<double4>(), t->x2.as<double>(),
                                                    t->y2.as<double>(), t->z2.as<double>(), t->perm2.as<int>()); note_launch();
            k_copy_back<<<nsi, kThreads, 0, s>>>(reinterpret_cast<Item*>(dd), t->x2.as<double>(), t->y2.as<double>(),
                                                 t->z2.as<double>(), t->perm2.as<int>(), x, y, z, perm); note_launch();
            KITC_CUDA(cudaGetLastError());
            trace("enqueued scatter", level);
            // no sync: the host next writes h_cnt after the next level's count sync, which
            // (stream order) follows this copy
        }
        if (!next.empty()) depth = level + 1;
        cur.swap(next);
        ++level;
    }
    const int C = (int)hb.size();
    t->nclusters = C;
    t->depth = depth;
    t->ndegenerate = ndeg;
    // topology table + batches: leaves in order of their ranges (they tile [0, N)); leaf l owns
    // batches [boff_l, boff_l + ceil(n_l / kBatch)), written on the device by k_leaf_order
    std::vector<std::pair<int, int>> leaves;
    for (int c = 0; c < C; ++c)
        if (hn[c] == 0) leaves.emplace_back(hb[c], c);
    std::sort(leaves.begin(), leaves.end());
    const int nlv = (int)leaves.size();
    t->h_leaf_begin.resize(nlv);
    t->h_leaf_boff.resize(nlv + 1);
    int64_t nb = 0;
    for (int i = 0; i < nlv; ++i) {
        const int c = leaves[i].second;
        t->h_leaf_begin[i] = hb[c];
        t->h_leaf_boff[i] = nb;
        nb += (he[c] - hb[c] + kBatch - 1) / kBatch;
    }
    t->h_leaf_boff[nlv] = nb;
    t->nbatches = nb;
    const size_t q1 = pad16<int4>(C), q2 = q1 + pad16<int4>(nlv);
    KITC_TRY(t->h_stage.ensure(q2));
    int4* ht = t->h_stage.as<int4>();
    for (int c = 0; c < C; ++c) ht[c] = make_int4(hb[c], he[c], hf[c], hn[c]);
    int4* hlv = reinterpret_cast<int4*>(t->h_stage.as<char>() + q1);
    for (int i = 0; i < nlv; ++i)
        hlv[i] = make_int4(hb[leaves[i].second], he[leaves[i].second], leaves[i].second, (int)t->h_leaf_boff[i]);
    KITC_TRY(t->topo.ensure(q1, s));
    KITC_TRY(t->bstart.ensure((size_t)std::max<int64_t>(nb, 1) * sizeof(int), s));
    KITC_TRY(t->bcount.ensure((size_t)std::max<int64_t>(nb, 1) * sizeof(int), s));
    KITC_TRY(t->leaves.ensure(q2 - q1, s));
    KITC_TRY(t->tord.ensure((size_t)N * sizeof(int), s));
    KITC_CUDA(cudaMemcpyAsync(t->topo.p, t->h_stage.p, (size_t)C * sizeof(int4), cudaMemcpyHostToDevice, s));
    KITC_CUDA(cudaMemcpyAsync(t->leaves.p, hlv, (size_t)nlv * sizeof(int4), cudaMemcpyHostToDevice, s));
    k_leaf_order<<<nlv, 256, 0, s>>>(t->leaves.as<int4>(), t->box.as<double>(), x, y, z, t->tord.as<int>(),
                                      t->bstart.as<int>(), t->bcount.as<int>()); note_launch();
    KITC_CUDA(cudaGetLastError());
    // h_stage may still be read by the copies above: the next writer waits on this event
    if (!t->ev_stage) KITC_CUDA(cudaEventCreateWithFlags(&t->ev_stage, cudaEventDisableTiming));
    KITC_CUDA(cudaEventRecord(t->ev_stage, s));
    trace("enqueued topology", level);
    t->built = true;
    return KITC_OK;
}

}  // namespace kitc
