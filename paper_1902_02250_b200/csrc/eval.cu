// eval.cu -- treecode evaluation (Algorithm 2 lines 7-17) on sm_100a.
//
// One warp = one batch of <= kBatch = 4 targets of one leaf, consecutive in the
// leaf's Morton order (spatially compact); kGroup = 8 lanes cooperate on each
// target (they split its proxy rows / sources and combine at the end).  The warp
// walks the tree depth-first with an explicit shared-memory stack of (cluster,
// lane mask) entries, so every lane keeps the paper's PER-TARGET semantics: a
// lane stops descending below a cluster it accepted; lanes that reject a cluster
// descend into its children.  At each popped cluster:
//   MAC   r^2 <= (theta^2) R^2, R^2 > 0   (RN intrinsics, no FMA; readings A4/A5)
//   far   accepting lanes sum the kernel against the (n+1)^3 proxies s_k with the
//         modified weights fhat_k (Eq. pc_approximation_3D): fhat
//         staged into shared memory by cp.async.bulk (TMA) two stages ahead,
//         tensor-product reuse of dx, dy, dz, two rows per lane (far_field) or,
//         for the Stokeslet at P = 10 with all 4 targets accepting, one row for
//         two targets per lane; for the Stokeslet at P <= 8 the whole cluster in
//         one stage (far_small); a cluster accepted by only 1 or 2 targets is
//         done by the whole warp (far_field_team)
//   near  rejecting lanes at a leaf sum over its particles directly
//         (Eq. pc_interaction_3D), j == i skipped by index (reading A8); idle
//         target groups join 1 or 2 participating targets (near_leaf)
//   else  rejecting lanes push the children.
// Outputs are scaled once and scattered to original order (out[perm[t]]).
// DESIGN.md §6 has the measured effect of each choice.
#include <algorithm>

#include "kitc_internal.cuh"
#include "pair.cuh"

namespace kitc {

namespace {

#ifndef KITC_EVAL_WARPS
#define KITC_EVAL_WARPS 4
#endif
#ifndef KITC_EVAL_MINB
#define KITC_EVAL_MINB 4  // resident CTAs per SM (register budget), Stokeslet at n = 8 (round 2: 4 CTAs with the
                          // target-pair near field (below) beat 5 CTAs without it: C3 95.0 -> 93.8 ms)
#endif
#ifndef KITC_EVAL_MINB_P8
#define KITC_EVAL_MINB_P8 4  // Stokeslet at n = 7, 9, 10 (measured: 4 beats 5 on X1 / X1L and the C2 sweep)
#endif
#ifndef KITC_EVAL_MINB_OTHER
#define KITC_EVAL_MINB_OTHER 4  // Stokeslet at n <= 6 (round 2, with the target-pair near field: n = 3, 5, 6 on the C3 input 32.6 -> 30.6, 49.7 -> 47.6, 59.6 -> 59.1 ms; n = 4 39.6 both)
#endif
#ifndef KITC_EVAL_MINB1
#define KITC_EVAL_MINB1 4  // rotlet / combined (measured: 4 beats 5 and 6 on C4)
#endif
#ifndef KITC_NEAR_U
#define KITC_NEAR_U 4  // near field: sources per lane per unrolled iteration (loads hoisted)
#endif
#ifndef KITC_NEAR_PACKED
#define KITC_NEAR_PACKED 1  // near field reads the packed (x, y, z, w) records
#endif
#ifndef KITC_NEAR_TEAMS
#define KITC_NEAR_TEAMS 1  // near field: idle target groups join the participating ones
#endif
#ifndef KITC_FAR_TEAMS
#define KITC_FAR_TEAMS 1  // far field: idle target groups join 1 or 2 accepting targets
#endif
#ifndef KITC_DZ_SMEM
#define KITC_DZ_SMEM 1  // far field: per-plane dz of the batch's targets in shared memory
#endif
#ifndef KITC_DZ_REG9
#define KITC_DZ_REG9 1  // ... but in registers for these kernels (bit k) at P = 9 (4 CTAs/SM, 128 registers)
#endif
#ifndef KITC_EVAL_SB
#define KITC_EVAL_SB 2
#endif
#ifndef KITC_ROWPF
#define KITC_ROWPF 1  // far field: load the next stage's row grid coordinates one stage ahead (see kRowPF)
#endif
#ifndef KITC_FAR_TB
// far field with all 4 targets accepting: one row for TWO targets per lane, Stokeslet at
// P = 10 (measured on the C3 input: n = 9 -6%; slower at P = 9 (spills at 5 CTAs/SM, 4 CTAs/SM
// loses more), P = 11, P <= 7 and for the rotlet; at P = 8 (n = 7 -8%) superseded by far_small)
#define KITC_FAR_TB 1
#endif
#ifndef KITC_FAR_TB_P9
#define KITC_FAR_TB_P9 0  // tuning builds only (with KITC_EVAL_MINB=4: no spills)
#endif
constexpr int kWarps = KITC_EVAL_WARPS;  // warps (batches) per CTA
template <int PT, int KER>
__host__ __device__ constexpr int eval_min_blocks() {  // CTAs/SM per instantiation (measured, see the macros above)
    return KER == 0 ? (PT == 9 ? KITC_EVAL_MINB : (PT == 8 || PT >= 10) ? KITC_EVAL_MINB_P8 : KITC_EVAL_MINB_OTHER)
                    : KITC_EVAL_MINB1;
}
#ifndef KITC_PART_CHUNK
#define KITC_PART_CHUNK 64
#endif
constexpr int kPartChunk = KITC_PART_CHUNK;  // batches per chunk of the interleaved multi-GPU split
#ifdef KITC_EVAL_HIST
__device__ unsigned long long g_hist[10];
}  // namespace
extern "C" void kitc_eval_hist(unsigned long long* h) { cudaMemcpyFromSymbol(h, g_hist, sizeof(g_hist)); }
namespace {
#endif
constexpr int kSB = KITC_EVAL_SB;         // fhat blocks per pipeline stage (1 or 2)
static_assert(kSB == 1 || kSB == 2, "kSB");
static_assert(kGroup == kRows, "k_eval: one fhat row per lane of a target group");

struct EvalArgs {
    const double* x;  // sorted sources (SoA)
    const double* y;
    const double* z;
    const double* tx;  // targets by position t (= x, y, z when targets = sources)
    const double* ty;
    const double* tz;
    int tpack;  // 1: targets = sources, coordinates read from the packed records (src)
    const int* perm;  // output row of target position t
    const int* tord;  // batch slot -> target position (nullptr: identity)
    const double* w;  // sorted weights, M planes of N
    const double* src;  // packed near-field records (x, y, z, w.., pad), sld doubles each
    int sld;
    const double4* cr;
    const int4* topo;
    const double* grid;
    const double* fhat;
    const int* bstart;  // nullptr: batch b = positions [kBatch b, kBatch b + kBatch) of nt
    const int* bcount;
    long long nt;
    double* out;
    unsigned long long* stats;
    long long bb, be;
    int part, nparts;  // interleaved multi-GPU split (nparts > 1): chunks of kPartChunk batches
    int N;
    int ncl;   // clusters in the tree (index bound; KITC_CHECKS)
    long long nout;  // output rows (index bound; KITC_CHECKS)
    int P;  // n + 1 (runtime copy)
    int stack_cap;
    int warp_smem;  // bytes of shared memory per warp (WarpSmem)
    int self_omit;
    int size_check;  // KITC_EVAL_SIZE_CHECK
    double tt;  // theta * theta (RN)
    KParams kp;
};

// ---- per-warp shared memory: two fhat stage buffers (TMA destinations), their
// mbarriers, the number of stages issued so far (-> buffer and phase parity of
// the next stage), the per-plane dz of the batch's targets, and the DFS stack.
struct WarpSmem {
    double* dzs;               // kBatch x P doubles (KITC_DZ_SMEM)
    double* buf;               // 2 x blk doubles
    unsigned long long* bar;   // 2 mbarriers
    int* nround;
    int2* stk;
    int stage_bytes;  // bytes available for the two stage buffers (KITC_CHECKS)
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// One elected lane: arm the barrier with the byte count and start the bulk
// copy global -> shared, which completes the transaction on the barrier.
__device__ __forceinline__ void tma_round(double* dst, const double* src, unsigned bytes, unsigned long long* bar) {
    const unsigned b = smem_u32(bar);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(b)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "KITC_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra KITC_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

// Far field of one accepted cluster (Eq. pc_approximation_3D) for
// the accepted lanes `am` of the warp.  fhat comes in blocks of kRows = 8 rows
// (k1, k2) x all k3 x all m (weights.cu layout); kSB consecutive blocks form a
// stage, staged into shared memory by ONE bulk copy two stages ahead of its use
// (double buffer, mbarrier completion), so the FP64 work never waits on L2.
// Every row is summed over all k3 with dx, dy, dx^2 + dy^2 + eps^2 per row and
// dz per plane reused (EvalKern::pair_row folds the terms linear in d along the
// row).  In a stage of two full blocks lane g of a target group takes the two
// adjacent rows 2(g%4), 2(g%4)+1 of block g/4 (one 16-byte shared load fetches
// both rows' weights; two independent pair chains); a stage with one full block
// gives each lane one row; the rows of a partial last block are split pair by
// pair over the lanes.
template <int PT, int KER>
__device__ __forceinline__ void far_field(double x, double y, double z, const double* __restrict__ g,
                                          const double* __restrict__ F, double* acc, const KParams& kp, int Prt,
                                          int grp, int lane, unsigned am, const WarpSmem& ws) {
    using K = EvalKern<KER>;
    constexpr int M = K::M;
    const int P = PT > 0 ? PT : Prt, P2 = P * P;
    const int R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;  // blocks, full blocks
    const int blk = P * M * kRows;                            // doubles per block
    const int NS = (R + kSB - 1) / kSB;                       // stages
    const bool leader = lane == __ffs(am) - 1;
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {  // stage st of this cluster -> buffer k & 1
        const int nb = min(kSB, R - st * kSB);
        KITC_DCHECK(nb >= 1 && (st * kSB + nb) * blk <= R * blk && 2 * kSB * blk * 8 <= ws.stage_bytes);
        tma_round(ws.buf + (k & 1) * kSB * blk, F + (size_t)st * kSB * blk, (unsigned)(nb * blk * 8),
                  ws.bar + (k & 1));
    };
    if (leader) {
        // the buffers were last read through the generic proxy (previous cluster): order
        // those reads before the async-proxy (bulk copy) writes, as for the refills below
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    // dz per plane of this lane's target: in shared memory (frees registers; the target-pair
    // path also reads the sibling's), or in registers where the budget allows (kDzReg)
    constexpr bool kDzReg = PT > 0 && (!KITC_DZ_SMEM || (((KITC_DZ_REG9 >> KER) & 1) && PT == 9));
    double dzr[PT > 0 ? PT : 1];
    double* dzp = ws.dzs + (lane / kGroup) * P;
    if constexpr (kDzReg) {
#pragma unroll
        for (int k3 = 0; k3 < (PT > 0 ? PT : 1); ++k3) dzr[k3] = z - __ldg(g + 2 * P + k3);
    } else {
        for (int k3 = grp; k3 < P; k3 += kGroup) dzp[k3] = z - __ldg(g + 2 * P + k3);
        __syncwarp(am);
    }
#define KITC_DZ(k3) (kDzReg ? dzr[k3] : dzp[k3])
#if KITC_FAR_TB
    // register blocking over targets (all 4 accept): lane L evaluates row L & 15 of the
    // stage for its own target (acc) and for the sibling target of lane L ^ 8 (oth); the
    // f-hat row is read once for both, and oth is folded into the sibling's lanes below
    constexpr bool kTB = KITC_FAR_TB && KITC_DZ_SMEM && K::kPairRows && kSB == 2 && KER == 0 &&
                         (PT == 8 || PT == 10 || (KITC_FAR_TB_P9 && PT == 9));
    const bool tb = kTB && am == 0xffffffffu;
    double oth[K::NA];
    double ox = 0.0, oy = 0.0;
    if constexpr (kTB) if (tb) {
#pragma unroll
        for (int c = 0; c < K::NA; ++c) oth[c] = 0.0;
        ox = __shfl_xor_sync(0xffffffffu, x, kGroup);
        oy = __shfl_xor_sync(0xffffffffu, y, kGroup);
    }
#endif
    // the Stokeslet's 4-CTA/SM instantiations without target-pair blocking (128 registers) keep the
    // grid coordinates (x of k1, y of k2) of the lane's two rows of the NEXT two-block stage in
    // registers: C3 93.8 -> 93.4 ms, C5 857.7 -> 854.3 ms (slower for the rotlet and at P = 8)
    constexpr bool kRowPF = KITC_ROWPF && KER == 0 && eval_min_blocks<PT, KER>() == 4 && PT != 8 && PT != 10;
    double rg[4];
    auto row_grid = [&](int sq) {
        const int ra = (sq * kSB + (grp >> 2)) * kRows + 2 * (grp & 3);
        const int k1a = ra / P, k2a = ra - k1a * P;
        const int k1b = k2a + 1 == P ? k1a + 1 : k1a, k2b = k2a + 1 == P ? 0 : k2a + 1;
        rg[0] = __ldg(g + k1a);
        rg[1] = __ldg(g + P + k2a);
        rg[2] = __ldg(g + k1b);
        rg[3] = __ldg(g + P + k2b);
    };
    if constexpr (kRowPF) row_grid(0);
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * kSB * blk;
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int b0 = st * kSB;  // first block of the stage
#if KITC_FAR_TB
        if (kTB && tb && b0 + 1 < RF) {
            const int q = lane & 15, h = q >> 3, j = q & 7;
            const int row = (b0 + h) * kRows + j;
            const int k1 = row / P, k2 = row - k1 * P;
            const double gx = __ldg(g + k1), gy = __ldg(g + P + k2);
            const double dxa = x - gx, dya = y - gy, dxb = ox - gx, dyb = oy - gy;
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Bj = B + h * blk + j;
            const double* dzb = ws.dzs + ((lane / kGroup) ^ 1) * P;  // the sibling target's dz
            typename K::Row rA, rB;
            if constexpr (PT > 0) {
#pragma unroll
                for (int k3 = 0; k3 < PT; ++k3) {
                    double f[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) f[m] = Bj[(k3 * M + m) * kRows];
                    const double za = KITC_DZ(k3), zb = dzb[k3];
                    K::pair_row(dxa, dya, za, fma(za, za, pa), f, acc, rA, kp);
                    K::pair_row(dxb, dyb, zb, fma(zb, zb, pb), f, oth, rB, kp);
                }
            }
            K::row_end(dxa, dya, rA, acc);
            K::row_end(dxb, dyb, rB, oth);
        } else
#endif
        if (K::kPairRows && kSB == 2 && b0 + 1 < RF) {
            // two full blocks: rows ra, ra + 1 of block h = grp / 4
            const int h = grp >> 2, j = 2 * (grp & 3);
            double dxa, dya, dxb, dyb;
            if constexpr (kRowPF) {  // loaded during the previous stage
                dxa = x - rg[0];
                dya = y - rg[1];
                dxb = x - rg[2];
                dyb = y - rg[3];
                if (st + 1 < NS) row_grid(st + 1);
            } else {
                const int ra = (b0 + h) * kRows + j;
                const int k1a = ra / P, k2a = ra - k1a * P;
                const int k1b = k2a + 1 == P ? k1a + 1 : k1a, k2b = k2a + 1 == P ? 0 : k2a + 1;
                dxa = x - __ldg(g + k1a);
                dya = y - __ldg(g + P + k2a);
                dxb = x - __ldg(g + k1b);
                dyb = y - __ldg(g + P + k2b);
            }
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Bh = B + h * blk + j;
            typename K::Row rA, rB;
            if constexpr (PT > 0) {
#pragma unroll
                for (int k3 = 0; k3 < PT; ++k3) {
                    double fa[M], fb[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const double2 v = *reinterpret_cast<const double2*>(Bh + (k3 * M + m) * kRows);
                        fa[m] = v.x;
                        fb[m] = v.y;
                    }
                    const double zk = KITC_DZ(k3);
                    K::pair_row(dxa, dya, zk, fma(zk, zk, pa), fa, acc, rA, kp);
                    K::pair_row(dxb, dyb, zk, fma(zk, zk, pb), fb, acc, rB, kp);
                }
            } else {
                for (int k3 = 0; k3 < P; ++k3) {
                    const double dzk = z - __ldg(g + 2 * P + k3);
                    double fa[M], fb[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) {
                        const double2 v = *reinterpret_cast<const double2*>(Bh + (k3 * M + m) * kRows);
                        fa[m] = v.x;
                        fb[m] = v.y;
                    }
                    K::pair_row(dxa, dya, dzk, fma(dzk, dzk, pa), fa, acc, rA, kp);
                    K::pair_row(dxb, dyb, dzk, fma(dzk, dzk, pb), fb, acc, rB, kp);
                }
            }
            K::row_end(dxa, dya, rA, acc);
            K::row_end(dxb, dyb, rB, acc);
        } else {
            for (int bb = b0; bb < min(b0 + kSB, R); ++bb) {
                const double* Bb = B + (bb - b0) * blk;
                if (bb < RF) {  // full block: one row per lane
                    const int row = bb * kRows + grp;
                    const int k1 = row / P, k2 = row - k1 * P;
                    const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2);
                    const double pxye = fma(dy, dy, dx * dx) + kp.e2;
                    typename K::Row r;
                    if constexpr (PT > 0) {
#pragma unroll
                        for (int k3 = 0; k3 < PT; ++k3) {
                            double f[M];
#pragma unroll
                            for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + grp];
                            const double zk = KITC_DZ(k3);
                            K::pair_row(dx, dy, zk, fma(zk, zk, pxye), f, acc, r, kp);
                        }
                    } else {
                        for (int k3 = 0; k3 < P; ++k3) {
                            const double dzk = z - __ldg(g + 2 * P + k3);
                            double f[M];
#pragma unroll
                            for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + grp];
                            K::pair_row(dx, dy, dzk, fma(dzk, dzk, pxye), f, acc, r, kp);
                        }
                    }
                    K::row_end(dx, dy, r, acc);
                } else if (!kDzReg && (P2 - RF * kRows == 2 || P2 - RF * kRows == 4)) {
                    // partial block of 2 or 4 rows (even P): kRows / nrem lanes per row, each
                    // summing a contiguous k3 range in row form (partial row sums are linear)
                    const int nrem = P2 - RF * kRows, L = kRows / max(nrem, 1), KL = (P + L - 1) / L;
                    const int jj = grp / L, q = grp - jj * L, row = RF * kRows + jj;
                    const int k1 = row / P, k2 = row - k1 * P;
                    const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2);
                    const double pxye = fma(dy, dy, dx * dx) + kp.e2;
                    typename K::Row r;
                    for (int k3 = q * KL; k3 < min(P, (q + 1) * KL); ++k3) {
                        double f[M];
#pragma unroll
                        for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + jj];
                        K::pair_row(dx, dy, dzp[k3], fma(dzp[k3], dzp[k3], pxye), f, acc, r, kp);
                    }
                    K::row_end(dx, dy, r, acc);
                } else {  // partial last block: pair by pair
                    const int pairs = (P2 - RF * kRows) * P;
                    for (int q = grp; q < pairs; q += kRows) {
                        const int jj = q / P, k3 = q - jj * P, row = RF * kRows + jj;
                        const int k1 = row / P, k2 = row - k1 * P;
                        const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2),
                                     dzk = z - __ldg(g + 2 * P + k3);
                        double f[M];
#pragma unroll
                        for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + jj];
                        K::pair(dx, dy, dzk, fma(dy, dy, dx * dx) + fma(dzk, dzk, kp.e2), f, acc, kp);
                    }
                }
            }
        }
        __syncwarp(am);  // every accepted lane is done with buffer k & 1
        if (leader && st + 2 < NS) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + 2, k);
        }
    }
    if (leader) *ws.nround = base + NS;
#if KITC_FAR_TB
    if constexpr (kTB) if (tb) {
#pragma unroll
        for (int c = 0; c < K::NA; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, oth[c], kGroup);
    }
#endif
    __syncwarp(am);
#undef KITC_DZ
}

#ifndef KITC_FAR_SMALL
#define KITC_FAR_SMALL 1  // Stokeslet at P <= 8: the whole cluster in one stage (far_small)
#endif
__host__ __device__ constexpr bool far_small_on(int P, int KER) {
    return KITC_FAR_SMALL && KER == 0 && P >= 2 && P <= 8;
}
// f-hat blocks of stage buffer per warp: the whole cluster (far_small) or two kSB-block stages
__host__ __device__ constexpr int stage_blocks(int P, int KER) {
    return far_small_on(P, KER) && (P * P + kRows - 1) / kRows > 2 * kSB ? (P * P + kRows - 1) / kRows : 2 * kSB;
}

// Far field of one accepted cluster at low degree (Stokeslet, P <= 8): the cluster's f-hat
// (R blocks of 8 rows) comes in ONE bulk copy with one wait, and every lane of a target group
// sums the rows grp, grp + 8, grp + 16, .. of the full blocks in groups of RG independent row
// chains (RG = all of them when there are <= 3, else 2), the P^2 mod 8 leftover rows pair by
// pair.  Against far_field's two-block stages this drops the per-stage handshake and the
// one-row-per-lane stage: far-field loop alone (tools/far_small_probe.cu, all 4 targets
// accepting) P = 4 46.5 -> 50.0%, P = 5 49.9 -> 56.2%, P = 6 52.7 -> 57.0%, P = 7 60.3 -> 63.5%,
// P = 8 (vs target pairs) 67.8 -> 70.0% of the FP64 peak.  The stage is one round of the
// warp's round counter, so it interleaves with far_field_team's two-buffer rounds.
template <int PT, int KER>
__device__ __forceinline__ void far_small(double x, double y, double z, const double* __restrict__ g,
                                          const double* __restrict__ F, double* acc, const KParams& kp, int grp,
                                          int lane, unsigned am, const WarpSmem& ws) {
    using K = EvalKern<KER>;
    constexpr int P = PT, M = K::M, P2 = P * P, R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    constexpr int blk = P * M * kRows, RG = RF <= 3 ? (RF > 0 ? RF : 1) : 2;
    static_assert(RF <= 3 || RF % 2 == 0, "far_small: row groups of 2");
    const int k = *ws.nround;
    if (lane == __ffs(am) - 1) {
        KITC_DCHECK(R * blk * 8 <= ws.stage_bytes);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // buffer last read by the generic proxy
        tma_round(ws.buf, F, (unsigned)(R * blk * 8), ws.bar + (k & 1));
    }
    double dzr[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) dzr[k3] = z - __ldg(g + 2 * P + k3);
    mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
    const double* B = ws.buf;
#pragma unroll 1
    for (int r0 = 0; r0 < RF; r0 += RG) {
        double dx[RG], dy[RG], pp[RG];
        typename K::Row rw[RG];
#pragma unroll
        for (int i = 0; i < RG; ++i) {
            const int row = (r0 + i) * kRows + grp, k1 = row / P, k2 = row - k1 * P;
            dx[i] = x - __ldg(g + k1);
            dy[i] = y - __ldg(g + P + k2);
            pp[i] = fma(dy[i], dy[i], dx[i] * dx[i]) + kp.e2;
        }
#pragma unroll
        for (int k3 = 0; k3 < P; ++k3) {
            const double zk = dzr[k3];
#pragma unroll
            for (int i = 0; i < RG; ++i) {
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = B[((r0 + i) * P + k3) * M * kRows + m * kRows + grp];
                K::pair_row(dx[i], dy[i], zk, fma(zk, zk, pp[i]), f, acc, rw[i], kp);
            }
        }
#pragma unroll
        for (int i = 0; i < RG; ++i) K::row_end(dx[i], dy[i], rw[i], acc);
    }
    if constexpr (P2 > RF * kRows) {  // the partial block's rows, pair by pair over the group's lanes
        const double* Bb = B + RF * blk;
        constexpr int pairs = (P2 - RF * kRows) * P;
        for (int q = grp; q < pairs; q += kRows) {
            const int jj = q / P, k3 = q - jj * P, row = RF * kRows + jj;
            const int k1 = row / P, k2 = row - k1 * P;
            const double ddx = x - __ldg(g + k1), ddy = y - __ldg(g + P + k2), dzk = z - __ldg(g + 2 * P + k3);
            double f[M];
#pragma unroll
            for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + jj];
            K::pair(ddx, ddy, dzk, fma(ddy, ddy, ddx * ddx) + fma(dzk, dzk, kp.e2), f, acc, kp);
        }
    }
    __syncwarp(am);  // every accepted lane is done with the buffer
    if (lane == __ffs(am) - 1) *ws.nround = k + 1;
    __syncwarp(am);
}

// Far field of one cluster accepted by only 1 or 2 of the batch's targets, by the
// WHOLE warp ("teams", as near_leaf): the idle target groups join the accepting
// ones.  Two targets: teams of 16 lanes, one row of the 16-row stage per lane.
// One target: 32 lanes, each row split between two lanes by k3 halves (the row
// sums of EvalKern::pair_row are linear, so partial rows fold like full ones).
// Same TMA-staged double buffer and round counter as far_field; partial sums are
// folded into the accepting groups' lanes with butterfly shuffles.
template <int PT, int KER>
__device__ __forceinline__ void far_field_team(double x, double y, double z, const double* __restrict__ g,
                                               const double* __restrict__ F, double* acc, const KParams& kp,
                                               int Prt, int lane, unsigned am, const WarpSmem& ws) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, NA = K::NA;
    const int P = PT > 0 ? PT : Prt, P2 = P * P;
    const int R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    const int blk = P * M * kRows;
    const int NS = (R + kSB - 1) / kSB;
    const int grp = lane % kGroup, gl = lane / kGroup;
    const bool mine = (am >> lane) & 1u;
    const unsigned gm = am & 0x01010101u;
    const int nt = __popc(gm);
    const int ga = (__ffs(gm) - 1) / kGroup;
    int src, rk, TS, xm;
    if (nt == 1) {
        TS = 32;
        src = ga;
        rk = ((gl - ga) & 3) * kGroup + grp;
        xm = 0;
    } else {
        const int gb = (31 - __clz(gm)) / kGroup;
        TS = 16;
        xm = ((ga ^ gb) == 1) ? 2 : 1;
        const bool act = gl == ga || gl == gb;
        src = act ? gl : (gl ^ xm);
        rk = (act ? 0 : kGroup) + grp;
    }
    const int sl = src * kGroup;
    const double tx = __shfl_sync(0xffffffffu, x, sl), ty = __shfl_sync(0xffffffffu, y, sl);
    const double tz = __shfl_sync(0xffffffffu, z, sl);
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nb = min(kSB, R - st * kSB);
        KITC_DCHECK(nb >= 1 && (st * kSB + nb) * blk <= R * blk && 2 * kSB * blk * 8 <= ws.stage_bytes);
        tma_round(ws.buf + (k & 1) * kSB * blk, F + (size_t)st * kSB * blk, (unsigned)(nb * blk * 8),
                  ws.bar + (k & 1));
    };
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // as in far_field
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    // this lane's rows: row j of block h of every stage; one target: k3 in [klo, klo + KH)
    const int r16 = rk & 15, h = r16 >> 3, j = r16 & 7;
    constexpr int KH = PT > 0 ? (PT + 1) / 2 : 1;
    const int khalf = (P + 1) / 2;
    const int klo = (TS == 32 && rk >= 16) ? khalf : 0;
    const int kn = TS == 32 ? (rk >= 16 ? P - khalf : khalf) : P;  // k3 count of this lane's rows
    double tmp[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) tmp[c] = 0.0;
    double dzh[PT > 0 ? PT : 1];
    if constexpr (PT > 0) {
#pragma unroll
        for (int i = 0; i < PT; ++i) dzh[i] = tz - __ldg(g + 2 * PT + min(klo + i, PT - 1));
    }
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * kSB * blk;
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int b0 = st * kSB, bb = b0 + h;
        if (bb < RF) {
            const int row = bb * kRows + j;
            const int k1 = row / P, k2 = row - k1 * P;
            const double dx = tx - __ldg(g + k1), dy = ty - __ldg(g + P + k2);
            const double pxye = fma(dy, dy, dx * dx) + kp.e2;
            const double* Bj = B + h * blk + j;
            typename K::Row r;
            if constexpr (PT > 0) {
                if (TS == 16) {
#pragma unroll
                    for (int k3 = 0; k3 < PT; ++k3) {
                        double f[M];
#pragma unroll
                        for (int m = 0; m < M; ++m) f[m] = Bj[(k3 * M + m) * kRows];
                        K::pair_row(dx, dy, dzh[k3], fma(dzh[k3], dzh[k3], pxye), f, tmp,
                                    r, kp);
                    }
                } else {
#pragma unroll
                    for (int i = 0; i < KH; ++i) {
                        if (i < kn) {
                            double f[M];
#pragma unroll
                            for (int m = 0; m < M; ++m) f[m] = Bj[((klo + i) * M + m) * kRows];
                            K::pair_row(dx, dy, dzh[i], fma(dzh[i], dzh[i], pxye), f, tmp, r, kp);
                        }
                    }
                }
            } else {
                for (int i = 0; i < kn; ++i) {
                    const int k3 = klo + i;
                    const double dzk = tz - __ldg(g + 2 * P + k3);
                    double f[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) f[m] = Bj[(k3 * M + m) * kRows];
                    K::pair_row(dx, dy, dzk, fma(dzk, dzk, pxye), f, tmp, r, kp);
                }
            }
            K::row_end(dx, dy, r, tmp);
        }
        if (RF < R && RF >= b0 && RF < b0 + kSB) {  // the partial last block, pair by pair
            const double* Bb = B + (RF - b0) * blk;
            const int pairs = (P2 - RF * kRows) * P;
            for (int q = rk; q < pairs; q += TS) {
                const int jj = q / P, k3 = q - jj * P, row = RF * kRows + jj;
                const int k1 = row / P, k2 = row - k1 * P;
                const double dx = tx - __ldg(g + k1), dy = ty - __ldg(g + P + k2), dzk = tz - __ldg(g + 2 * P + k3);
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + jj];
                K::pair(dx, dy, dzk, fma(dy, dy, dx * dx) + fma(dzk, dzk, kp.e2), f, tmp, kp);
            }
        }
        __syncwarp();
        if (lane == 0 && st + 2 < NS) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + 2, k);
        }
    }
    if (lane == 0) *ws.nround = base + NS;
    __syncwarp();
#pragma unroll
    for (int c = 0; c < NA; ++c) {
        if (nt == 1) {
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], 8);
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], 16);
        } else {
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], xm * kGroup);
        }
        if (mine) acc[c] += tmp[c];
    }
}

// Near field of one rejected leaf: the lane of rank `rk` in a team of TS lanes
// working for a target at (x, y, z) sums sources b + rk, b + rk + TS, ...
// (unrolled x4 with the loads hoisted).  SELF: the target is source `self` of
// this leaf, whose pair is evaluated with f = 0 and s = 1 -- an exact zero
// contribution, no branch.
template <int KER, bool SELF>
__device__ __forceinline__ void near_field_impl(double x, double y, double z, int self, int b, int e, int rk, int TS,
                                                const EvalArgs& a, double* acc) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, U = KITC_NEAR_U;
    int j = b + rk;
    for (; j + (U - 1) * TS < e; j += U * TS) {
        double sx[U], sy[U], sz[U], f[U][M];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = j + u * TS;
            if (KITC_NEAR_PACKED) {  // one record: (x, y) (z, w0) (w1, w2) ... 16-byte loads
                const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)jj * a.sld);
                double v[((3 + M + 1) / 2) * 2];
#pragma unroll
                for (int q = 0; q < (3 + M + 1) / 2; ++q) {
                    const double2 d2 = __ldg(r + q);
                    v[2 * q] = d2.x;
                    v[2 * q + 1] = d2.y;
                }
                sx[u] = v[0];
                sy[u] = v[1];
                sz[u] = v[2];
#pragma unroll
                for (int m = 0; m < M; ++m) f[u][m] = v[3 + m];
            } else {
                sx[u] = __ldg(a.x + jj);
                sy[u] = __ldg(a.y + jj);
                sz[u] = __ldg(a.z + jj);
#pragma unroll
                for (int m = 0; m < M; ++m) f[u][m] = __ldg(a.w + (size_t)m * a.N + jj);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const bool me = SELF && (j + u * TS) == self;
            const double dx = x - sx[u], dy = y - sy[u], dz = z - sz[u];
            if (SELF) {
#pragma unroll
                for (int m = 0; m < M; ++m) f[u][m] = me ? 0.0 : f[u][m];
            }
            const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
            K::pair(dx, dy, dz, s, f[u], acc, a.kp);
        }
    }
    for (; j < e; j += TS) {
        const bool me = SELF && j == self;
        const double dx = x - __ldg(a.x + j), dy = y - __ldg(a.y + j), dz = z - __ldg(a.z + j);
        double f[M];
#pragma unroll
        for (int m = 0; m < M; ++m) f[m] = me ? 0.0 : __ldg(a.w + (size_t)m * a.N + j);
        const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
        K::pair(dx, dy, dz, s, f, acc, a.kp);
    }
}

#ifndef KITC_NEAR_TB
// kernels (bit k = kernel k) whose near field is blocked over target pairs: the rotlet (C4n4, n = 4:
// 57.9 -> 55.4 ms; C4, n = 8: 140.7 -> 140.3 ms); slower for the Stokeslet (C3 +0.5%) and the
// combined kernel (X2 +0.5%)
#define KITC_NEAR_TB 2
#endif
#ifndef KITC_NEAR_TB_AT4
// also the Stokeslet instantiations that run at 4 CTAs/SM (128 registers: the record loads of 4 sources
// stay in flight for 2 targets): C3 95.0 -> 93.8 ms, X1 40.2 -> 39.5 ms, C5 856.8 -> 858.8 ms
#define KITC_NEAR_TB_AT4 1
#endif
#ifndef KITC_NEAR_TB_U0
#define KITC_NEAR_TB_U0 4  // Stokeslet: source records per lane in flight (C3, 4 CTAs/SM: U = 3, 4, 6, 8 -> 93.9, 93.7, 94.5, 96.8 ms)
#endif
#ifndef KITC_NEAR_TB_U1
#define KITC_NEAR_TB_U1 2  // rotlet
#endif
// Near field blocked over target pairs: the lane of rank rk (of TS) sums sources
// b + rk, b + rk + TS, ... for TWO targets A and B, so every source record it loads
// feeds two pair evaluations (half the loads per pair, two independent chains).
// SELF: A or B may be a source of this leaf (pair with f = 0, s = 1: exact zero).
template <int KER, bool SELF>
__device__ __forceinline__ void near_field_tb(double xa, double ya, double za, int ta, double xb, double yb,
                                              double zb, int tb, int b, int e, int rk, int TS, const EvalArgs& a,
                                              double* accA, double* accB) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, U = KER == 0 ? KITC_NEAR_TB_U0 : KITC_NEAR_TB_U1, NQ = (3 + M + 1) / 2;
    int j = b + rk;
    for (; j + (U - 1) * TS < e; j += U * TS) {
        double v[U][NQ * 2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)(j + u * TS) * a.sld);
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const double2 d2 = __ldg(r + q);
                v[u][2 * q] = d2.x;
                v[u][2 * q + 1] = d2.y;
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int jj = j + u * TS;
            {
                const bool me = SELF && jj == ta;
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = SELF && me ? 0.0 : v[u][3 + m];
                const double dx = xa - v[u][0], dy = ya - v[u][1], dz = za - v[u][2];
                const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
                K::pair(dx, dy, dz, s, f, accA, a.kp);
            }
            {
                const bool me = SELF && jj == tb;
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = SELF && me ? 0.0 : v[u][3 + m];
                const double dx = xb - v[u][0], dy = yb - v[u][1], dz = zb - v[u][2];
                const double s = me ? 1.0 : fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2)));
                K::pair(dx, dy, dz, s, f, accB, a.kp);
            }
        }
    }
    for (; j < e; j += TS) {
        const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)j * a.sld);
        double v[NQ * 2];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const double2 d2 = __ldg(r + q);
            v[2 * q] = d2.x;
            v[2 * q + 1] = d2.y;
        }
        const bool mea = SELF && j == ta, meb = SELF && j == tb;
        double fa[M], fb[M];
#pragma unroll
        for (int m = 0; m < M; ++m) {
            fa[m] = mea ? 0.0 : v[3 + m];
            fb[m] = meb ? 0.0 : v[3 + m];
        }
        const double dxa = xa - v[0], dya = ya - v[1], dza = za - v[2];
        const double dxb = xb - v[0], dyb = yb - v[1], dzb = zb - v[2];
        K::pair(dxa, dya, dza, mea ? 1.0 : fma(dxa, dxa, fma(dya, dya, fma(dza, dza, a.kp.e2))), fa, accA, a.kp);
        K::pair(dxb, dyb, dzb, meb ? 1.0 : fma(dxb, dxb, fma(dyb, dyb, fma(dzb, dzb, a.kp.e2))), fb, accB, a.kp);
    }
}

// The self pair can only occur in the leaf holding the target; every other leaf
// runs the select-free loop (warp-uniform: a batch never straddles leaves).
template <int KER>
__device__ __forceinline__ void near_field(double x, double y, double z, int t, int b, int e, int rk, int TS,
                                           const EvalArgs& a, double* acc) {
    if (a.self_omit && t >= b && t < e)
        near_field_impl<KER, true>(x, y, z, t, b, e, rk, TS, a, acc);
    else
        near_field_impl<KER, false>(x, y, z, -1, b, e, rk, TS, a, acc);
}

// Near field of leaf [b, e) for the participating lanes `rm` (whole target groups).
// With 3 or 4 participating targets each sums with its own kGroup lanes.  With 1
// or 2, the idle groups join them ("teams" of 32 or 16 lanes): every lane sums a
// strided share of the sources for its team's target into scratch accumulators,
// and the team's partial sums are folded into the owning group's lanes with
// butterfly shuffles -- the per-target result is the same sum (rounding order
// aside), with no idle lanes.  Called by ALL lanes of the warp.
template <int KER, int PT>
__device__ __forceinline__ void near_leaf(double x, double y, double z, int t, int b, int e, int lane, unsigned rm,
                                          const EvalArgs& a, double* acc) {
    using K = EvalKern<KER>;
    constexpr int NA = K::NA;
    const int grp = lane % kGroup, g = lane / kGroup;
    const int nt = __popc(rm) / kGroup;
    KITC_DCHECK(b >= 0 && b <= e && e <= a.N && (rm & 0x01010101u) * 0xffu == rm);
    const bool mine = (rm >> lane) & 1u;
    constexpr bool kTB = ((KITC_NEAR_TB >> KER) & 1) ||
                         (KITC_NEAR_TB_AT4 && KER == 0 && eval_min_blocks<PT, KER>() == 4);
    if (kTB && nt >= 3) {
        // 3 or 4 participating targets: each half-warp takes the target pair of its two groups,
        // 16 lanes striding the sources, every record feeding both targets; a lane's partial for
        // the partner group's target is handed over with one shuffle (lane ^ 8).  A target that
        // does not take this leaf directly (nt = 3) is computed and discarded.
        const int la = (lane >> 4) * 16, lb = la + kGroup;
        const double xa = __shfl_sync(0xffffffffu, x, la), ya = __shfl_sync(0xffffffffu, y, la);
        const double za = __shfl_sync(0xffffffffu, z, la);
        const double xb = __shfl_sync(0xffffffffu, x, lb), yb = __shfl_sync(0xffffffffu, y, lb);
        const double zb = __shfl_sync(0xffffffffu, z, lb);
        const int ta = __shfl_sync(0xffffffffu, t, la), tb = __shfl_sync(0xffffffffu, t, lb);
        double accA[NA], accB[NA];
#pragma unroll
        for (int c = 0; c < NA; ++c) accA[c] = accB[c] = 0.0;
        if (a.self_omit && t >= b && t < e)  // warp-uniform: the batch's leaf
            near_field_tb<KER, true>(xa, ya, za, ta, xb, yb, zb, tb, b, e, lane & 15, 16, a, accA, accB);
        else
            near_field_tb<KER, false>(xa, ya, za, -1, xb, yb, zb, -1, b, e, lane & 15, 16, a, accA, accB);
        const bool inB = (lane & kGroup) != 0;
#pragma unroll
        for (int c = 0; c < NA; ++c) {
            const double other = __shfl_xor_sync(0xffffffffu, inB ? accA[c] : accB[c], kGroup);
            if (mine) acc[c] += (inB ? accB[c] : accA[c]) + other;
        }
        return;
    }
    if (!KITC_NEAR_TEAMS || nt >= 3) {
        if (mine) near_field<KER>(x, y, z, t, b, e, grp, kGroup, a, acc);
        return;
    }
    // groups of the participating targets (ascending): ga [, gb]
    const unsigned gm = rm & 0x01010101u;  // one bit per participating group (its lane 0)
    const int ga = (__ffs(gm) - 1) / kGroup;
    int src, rk, TS, xm;
    if (nt == 1) {
        TS = 32;
        src = ga;
        rk = ((g - ga) & 3) * kGroup + grp;
        xm = 0;
    } else {
        const int gb = (31 - __clz(gm)) / kGroup;
        TS = 16;
        // partner groups: lane ^ xm*kGroup, chosen so each active group pairs with an idle one
        xm = ((ga ^ gb) == 1) ? 2 : 1;
        const bool act = g == ga || g == gb;
        src = act ? g : (g ^ xm);
        rk = (act ? 0 : kGroup) + grp;
    }
    const int sl = src * kGroup;
    const double tx = __shfl_sync(0xffffffffu, x, sl), ty = __shfl_sync(0xffffffffu, y, sl);
    const double tz = __shfl_sync(0xffffffffu, z, sl);
    const int tt = __shfl_sync(0xffffffffu, t, sl);
    double tmp[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) tmp[c] = 0.0;
    near_field<KER>(tx, ty, tz, tt, b, e, rk, TS, a, tmp);
#pragma unroll
    for (int c = 0; c < NA; ++c) {
        if (nt == 1) {
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], 8);
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], 16);
        } else {
            tmp[c] += __shfl_xor_sync(0xffffffffu, tmp[c], xm * kGroup);
        }
        if (mine) acc[c] += tmp[c];
    }
}

// Lane l works for target l / kGroup of the batch, as member l % kGroup of its
// group; the kGroup lanes of a target share every MAC decision.
// STATS: also write the per-target interaction counts (a.stats != nullptr).
template <int PT, int KER, bool STATS>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, KER>()) k_eval(const EvalArgs a) {
    using K = EvalKern<KER>;
    constexpr int M = K::M, NP = K::P, NA = K::NA;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int grp = lane % kGroup, ti = lane / kGroup;
    WarpSmem ws;
    {
        const int P = PT > 0 ? PT : a.P;
        const int blk = P * M * kRows;
        unsigned char* base = smem_raw + (size_t)wl * a.warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + (PT > 0 ? stage_blocks(PT, KER) : 2 * kSB) * blk *
                                                                     sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        ws.dzs = reinterpret_cast<double*>(ws.bar + 3);
        ws.stk = reinterpret_cast<int2*>(ws.dzs + (KITC_DZ_SMEM ? kBatch * P : 0));
        ws.stage_bytes = (int)(reinterpret_cast<unsigned char*>(ws.bar) - base);
        KITC_DCHECK(reinterpret_cast<unsigned char*>(ws.stk + a.stack_cap) <= base + a.warp_smem);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    int2* stk = ws.stk;
    long long b = a.bb + (long long)blockIdx.x * kWarps + wl;
    if (a.nparts > 1) {  // part-local index -> global batch of the interleaved chunks
        const long long i = b;
        b = ((i / kPartChunk) * a.nparts + a.part) * kPartChunk + i % kPartChunk;
    }
    if (b >= a.be) return;  // whole warp
    int p0, tc;
    if (a.bstart) {
        p0 = a.bstart[b];
        tc = a.bcount[b];
    } else {
        p0 = (int)(b * kBatch);
        tc = (int)min((long long)kBatch, a.nt - p0);
    }
    KITC_DCHECK(p0 >= 0 && tc >= 1 && tc <= kBatch && (long long)p0 + tc <= a.nt);
    const bool valid = ti < tc;
    const int t = a.tord ? a.tord[p0 + (valid ? ti : 0)] : p0 + (valid ? ti : 0);
    KITC_DCHECK(t >= 0 && t < a.nt);
    double x, y, z;
    if (a.tpack) {  // targets = sources: the coordinates from the packed record (no separate read of x, y, z)
        const double* r = a.src + (size_t)t * a.sld;
        const double2 xy = __ldg(reinterpret_cast<const double2*>(r));
        x = xy.x;
        y = xy.y;
        z = __ldg(r + 2);
    } else {
        x = a.tx[t];
        y = a.ty[t];
        z = a.tz[t];
    }
    const int P = PT > 0 ? PT : a.P;
    const int P3 = P * P * P;
    const long long LEN = (long long)((P * P + kRows - 1) / kRows) * P * M * kRows;  // fhat doubles per cluster
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
        KITC_DCHECK(c >= 0 && c < a.ncl && (mask & ~live) == 0u);
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
        // a cluster's particles lie in [0, N); children (BFS numbering) follow their parent
        KITC_DCHECK(tp.x >= 0 && tp.x <= tp.y && tp.y <= a.N && tp.w >= 0 && tp.w <= 8 &&
                    (tp.w == 0 || (tp.z > c && tp.z + tp.w <= a.ncl)));
#ifdef KITC_EVAL_HIST
        // tuning only: histogram of accepting targets per (warp, far cluster) and of
        // near-field participants per (warp, leaf) -> g_hist[0..4], g_hist[5..9]
        if (lane == 0) {
            if (am) atomicAdd(&g_hist[__popc(am) / kGroup], 1ull);
            if (rm && tp.w == 0) atomicAdd(&g_hist[5 + __popc(rm) / kGroup], 1ull);
        }
#endif
        if (am && a.size_check && tp.y - tp.x < P3) {
            // size-check variant (flag KITC_EVAL_SIZE_CHECK): an accepted cluster with
            // fewer particles than proxies is summed directly (the target is outside it)
            if (ok) {
                near_field<KER>(x, y, z, t, tp.x, tp.y, grp, kGroup, a, acc);
                if (STATS) {
                    st[2] += 1;
                    st[3] += (unsigned long long)(tp.y - tp.x);
                    st[4] += (unsigned long long)(tp.y - tp.x);
                }
            }
        } else if (am && KITC_FAR_TEAMS && kSB == 2 && __popc(am) <= 2 * kGroup) {
            far_field_team<PT, KER>(x, y, z, a.grid + (size_t)c * 3 * P, a.fhat + (size_t)c * LEN, acc, a.kp, P,
                                    lane, am, ws);
            if (STATS && ok) {
                st[0] += 1;
                st[1] += (unsigned long long)P3;
                st[4] += (unsigned long long)(tp.y - tp.x);
            }
        } else if (am && ok) {
            if constexpr (PT > 0 && far_small_on(PT, KER))
                far_small<PT, KER>(x, y, z, a.grid + (size_t)c * 3 * P, a.fhat + (size_t)c * LEN, acc, a.kp, grp,
                                   lane, am, ws);
            else
                far_field<PT, KER>(x, y, z, a.grid + (size_t)c * 3 * P, a.fhat + (size_t)c * LEN, acc, a.kp, P,
                                   grp, lane, am, ws);
            if (STATS) {
                st[0] += 1;
                st[1] += (unsigned long long)P3;
                st[4] += (unsigned long long)(tp.y - tp.x);
            }
        }
        if (rm) {
            if (tp.w == 0) {
                near_leaf<KER, PT>(x, y, z, t, tp.x, tp.y, lane, rm, a, acc);
                if (in && !ok) {
                    if (STATS) {
                        const int self = (a.self_omit && t >= tp.x && t < tp.y) ? 1 : 0;
                        st[2] += 1;
                        st[3] += (unsigned long long)(tp.y - tp.x - self);
                        st[4] += (unsigned long long)(tp.y - tp.x);
                    }
                }
            } else {
                // children pushed in reverse so the first child is popped first (A17).  The
                // stack holds <= 7 depth + 1 entries (8 (depth + 1) allocated); overflowing it
                // would be a library bug: trap (the next synchronising call reports KITC_ECUDA)
                if (sp + tp.w > a.stack_cap) __trap();
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
    KITC_DCHECK(o >= 0 && o < a.nout);
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
#ifdef KITC_ONLY_P  // tuning builds (tools/build_variant.py): one specialised degree, the rest generic
    if (P == KITC_ONLY_P)
        launch<KITC_ONLY_P, KER>(a, grid, smem, s);
    else
        launch<0, KER>(a, grid, smem, s);
    return;
#endif
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
                 int64_t bb, int64_t be, double* out, uint64_t* stats, cudaStream_t s, const TargetSet* ts,
                 unsigned flags, int part, int nparts) {
    if (nparts < 1 || part < 0 || part >= nparts) return set_error(KITC_EINVAL, "kitc_eval: bad part / nparts");
    if (flags & ~(unsigned)KITC_EVAL_SIZE_CHECK) return set_error(KITC_EINVAL, "kitc_eval: unknown flags");
    if (!t->built) return set_error(KITC_ESTATE, "kitc_eval: tree not built");
    if (!t->weights_ready || t->grid_n != n || t->weights_kernel != kernel)
        return set_error(KITC_ESTATE, "kitc_eval: call kitc_modified_weights with the same kernel and n first");
    if (!(theta >= 0.0 && theta < 1.0)) return set_error(KITC_EINVAL, "kitc_eval: theta must be in [0, 1)");
    if (!(eps >= 0.0) || !std::isfinite(eps)) return set_error(KITC_EINVAL, "kitc_eval: eps must be >= 0");
    if (self != KITC_SELF_OMIT && self != KITC_SELF_INCLUDE) return set_error(KITC_EINVAL, "kitc_eval: bad self");
    if (eps == 0.0 && self != KITC_SELF_OMIT && !ts)
        return set_error(KITC_EINVAL, "kitc_eval: eps = 0 requires KITC_SELF_OMIT (singular kernel)");
    const int64_t nbatch = ts ? (ts->n + kBatch - 1) / kBatch : t->nbatches;
    if (bb < 0 || be > nbatch || bb > be) return set_error(KITC_EINVAL, "kitc_eval: bad batch range");
    if (!fhat || !out) return set_error(KITC_EINVAL, "kitc_eval: NULL buffer");
    if (be == bb) return KITC_OK;
    EvalArgs a;
    a.x = t->x.as<double>();
    a.y = t->y.as<double>();
    a.z = t->z.as<double>();
    a.perm = t->perm.as<int>();
    a.tord = t->tord.as<int>();
    a.tx = a.x;
    a.ty = a.y;
    a.tz = a.z;
    a.tpack = 1;
    a.w = t->w.as<double>();
    a.src = t->src.as<double>();
    a.sld = t->src_ld;
    a.cr = t->cr.as<double4>();
    a.topo = t->topo.as<int4>();
    a.grid = t->grid.as<double>();
    a.fhat = fhat;
    a.bstart = t->bstart.as<int>();
    a.bcount = t->bcount.as<int>();
    a.nt = t->N;
    if (ts) {  // separate targets: no self term (reading A8 applies to targets = sources only)
        a.tx = ts->x;
        a.ty = ts->y;
        a.tz = ts->z;
        a.tpack = 0;
        a.perm = ts->row;
        a.tord = nullptr;
        a.bstart = a.bcount = nullptr;
        a.nt = ts->n;
        self = KITC_SELF_INCLUDE;
    }
    a.out = out;
    a.stats = reinterpret_cast<unsigned long long*>(stats);
    a.bb = bb;
    a.be = be;
    a.part = part;
    a.nparts = nparts;
    a.N = (int)t->N;
    a.ncl = (int)t->nclusters;
    a.nout = ts ? ts->n : t->N;
    a.P = n + 1;
    a.stack_cap = 8 * (t->depth + 1);
    a.self_omit = self == KITC_SELF_OMIT;
    a.size_check = (flags & KITC_EVAL_SIZE_CHECK) != 0;
    a.tt = theta * theta;
    a.kp = make_kparams(eps);
    int m = 0;
    KITC_TRY(kitc_kernel_dims(kernel, &m, nullptr));
    if (reinterpret_cast<uintptr_t>(fhat) % 16) return set_error(KITC_EINVAL, "kitc_eval: fhat must be 16-byte aligned");
    // per warp: 2 stage buffers + 2 mbarriers + round counter (8 B) + stack, 128-B multiple
    a.warp_smem = (int)(((size_t)stage_blocks(n + 1, kernel) * (n + 1) * m * kRows * sizeof(double) + 24 +
                         (size_t)a.stack_cap * sizeof(int2) +
                         (KITC_DZ_SMEM ? (size_t)kBatch * (n + 1) * sizeof(double) : 0) +
                         127) / 128 * 128);
    const size_t smem = (size_t)kWarps * a.warp_smem;
    if (smem > 200 * 1024) return set_error(KITC_EINVAL, "kitc_eval: tree too deep for the traversal stack");
    long long nb = be - bb;
    if (nparts > 1) {  // batches [0, be) split into chunks dealt round-robin; this part's count
        if (bb != 0) return set_error(KITC_EINVAL, "kitc_eval: an interleaved split covers batches [0, end)");
        const long long nch = (be + kPartChunk - 1) / kPartChunk;
        nb = 0;
        for (long long c = part; c < nch; c += nparts) nb += std::min<long long>(kPartChunk, be - c * kPartChunk);
        if (nb == 0) return KITC_OK;
        nb = ((nch - 1 - part) / nparts) * kPartChunk + kPartChunk;  // part-local index range (last chunk may be short)
    }
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
