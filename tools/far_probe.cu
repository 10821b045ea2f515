// Far-field loop in isolation (tuning probe, not part of libkitc): every warp sums the
// production far_field<PT, 0> (eval.cu) of a random sequence of clusters for a batch
// of 4 targets that all accept (am = full warp) -- no traversal, no near field, no lane
// masks.  f-hat of 1169 clusters (the C3 tree's count) is L2-resident like in k_eval.
// Prints pairs/clk/SM and the algorithmic rate (32 flop/pair) against the derived peak.
//   nvcc ... -I paper_1902_02250_b200/csrc tools/far_probe.cu -L paper_1902_02250_b200 -lkitc
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1902_02250_b200/csrc/eval.cu"

namespace kitc {
namespace {

template <int PT>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, 0>())
    k_far_probe(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out,
                KParams kp, int warp_smem) {
    using K = EvalKern<0>;
    constexpr int M = K::M, NA = K::NA, P = PT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int grp = lane % kGroup, ti = lane / kGroup;
    WarpSmem ws;
    {
        const int blk = P * M * kRows;
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + 2 * kSB * blk * sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        ws.dzs = reinterpret_cast<double*>(ws.bar + 3);
        ws.stk = reinterpret_cast<int2*>(ws.dzs + kBatch * P);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const long long LEN = (long long)((P * P + kRows - 1) / kRows) * P * M * kRows;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 3.0 + 0.01 * ti, y = 2.5 - 0.003 * ti, z = 2.0 + 0.002 * ti;
    double acc[NA];
#pragma unroll
    for (int c = 0; c < NA; ++c) acc[c] = 0.0;
    for (int i = 0; i < ncalls; ++i) {
        const int c = seq[(int)(((long long)gw * 7919 + i) % nseq)];
        far_field<PT, 0>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, P, grp, lane,
                         0xffffffffu, ws);
    }
    double t = 0.0;
#pragma unroll
    for (int c = 0; c < NA; ++c) t += acc[c];
    if (t == 1.2345) out[0] = t;
}


// Variant 1: far field blocked over target pairs with merged accumulators (3 per target) and
// the plane offsets dz of BOTH targets in registers: lane L takes row (L & 15) of each 16-row
// stage for its own target (group L / 8) and the sibling group's target (L ^ 8).
template <int PT>
__device__ __forceinline__ void far_tb(double xA, double yA, double zA, double xB, double yB, double zB,
                                       const double* __restrict__ g, const double* __restrict__ F, double* accA,
                                       double* accB, const KParams& kp, int lane, const WarpSmem& ws) {
    constexpr int P = PT, M = 3, P2 = P * P, R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    constexpr int blk = P * M * kRows, NS = (R + 1) / 2;
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nb = min(2, R - st * 2);
        tma_round(ws.buf + (k & 1) * 2 * blk, F + (size_t)st * 2 * blk, (unsigned)(nb * blk * 8), ws.bar + (k & 1));
    };
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    double dzA[P], dzB[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) {
        const double gz = __ldg(g + 2 * P + k3);
        dzA[k3] = zA - gz;
        dzB[k3] = zB - gz;
    }
    const int q = lane & 15, h = q >> 3, j = q & 7;
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * 2 * blk;
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int b0 = st * 2;
        if (b0 + 1 < RF) {
            const int row = (b0 + h) * kRows + j;
            const int k1 = row / P, k2 = row - k1 * P;
            const double gx = __ldg(g + k1), gy = __ldg(g + P + k2);
            const double dxa = xA - gx, dya = yA - gy, dxb = xB - gx, dyb = yB - gy;
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Bj = B + h * blk + j;
            double CA = 0.0, ZA = 0.0, CB = 0.0, ZB = 0.0;
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                const double f0 = Bj[(k3 * M + 0) * kRows], f1 = Bj[(k3 * M + 1) * kRows],
                             f2 = Bj[(k3 * M + 2) * kRows];
                {
                    const double dz = dzA[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pa));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxa, fma(f1, dya, f2 * dz)) * Y3;
                    CA += c;
                    ZA = fma(c, dz, ZA);
                    accA[0] = fma(f0, hh, accA[0]);
                    accA[1] = fma(f1, hh, accA[1]);
                    accA[2] = fma(f2, hh, accA[2]);
                }
                {
                    const double dz = dzB[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pb));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxb, fma(f1, dyb, f2 * dz)) * Y3;
                    CB += c;
                    ZB = fma(c, dz, ZB);
                    accB[0] = fma(f0, hh, accB[0]);
                    accB[1] = fma(f1, hh, accB[1]);
                    accB[2] = fma(f2, hh, accB[2]);
                }
            }
            CA *= 0.25;
            CB *= 0.25;
            accA[0] = fma(CA, dxa, accA[0]);
            accA[1] = fma(CA, dya, accA[1]);
            accA[2] = fma(0.25, ZA, accA[2]);
            accB[0] = fma(CB, dxb, accB[0]);
            accB[1] = fma(CB, dyb, accB[1]);
            accB[2] = fma(0.25, ZB, accB[2]);
        } else {
            // last stage: full block b0 (if any) row by row, then the partial block pair by pair
            for (int bb = b0; bb < min(b0 + 2, R); ++bb) {
                const double* Bb = B + (bb - b0) * blk;
                const int nrow = bb < RF ? kRows : P2 - RF * kRows;
                for (int qq = q; qq < nrow * P; qq += 16) {
                    const int jj = qq / P, k3 = qq - jj * P, row = bb * kRows + jj;
                    const int k1 = row / P, k2 = row - k1 * P;
                    const double gx = __ldg(g + k1), gy = __ldg(g + P + k2), gz = __ldg(g + 2 * P + k3);
                    const double f[3] = {Bb[(k3 * M + 0) * kRows + jj], Bb[(k3 * M + 1) * kRows + jj],
                                         Bb[(k3 * M + 2) * kRows + jj]};
                    double t6[6] = {0, 0, 0, 0, 0, 0};
                    {
                        const double dx = xA - gx, dy = yA - gy, dz = zA - gz;
                        EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, t6, kp);
                        accA[0] = fma(0.25, t6[3], accA[0] + t6[0]);
                        accA[1] = fma(0.25, t6[4], accA[1] + t6[1]);
                        accA[2] = fma(0.25, t6[5], accA[2] + t6[2]);
                    }
                    double u6[6] = {0, 0, 0, 0, 0, 0};
                    {
                        const double dx = xB - gx, dy = yB - gy, dz = zB - gz;
                        EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, u6, kp);
                        accB[0] = fma(0.25, u6[3], accB[0] + u6[0]);
                        accB[1] = fma(0.25, u6[4], accB[1] + u6[1]);
                        accB[2] = fma(0.25, u6[5], accB[2] + u6[2]);
                    }
                }
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
}

template <int PT>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, 0>())
    k_far_tb(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out,
             KParams kp, int warp_smem) {
    constexpr int M = 3, P = PT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ti = lane / kGroup;
    WarpSmem ws;
    {
        const int blk = P * M * kRows;
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + 2 * kSB * blk * sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        ws.dzs = reinterpret_cast<double*>(ws.bar + 3);
        ws.stk = reinterpret_cast<int2*>(ws.dzs + kBatch * P);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const long long LEN = (long long)((P * P + kRows - 1) / kRows) * P * M * kRows;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 3.0 + 0.01 * ti, y = 2.5 - 0.003 * ti, z = 2.0 + 0.002 * ti;
    const double xb = __shfl_xor_sync(0xffffffffu, x, kGroup), yb = __shfl_xor_sync(0xffffffffu, y, kGroup),
                 zb = __shfl_xor_sync(0xffffffffu, z, kGroup);
    double acc[3] = {0, 0, 0}, oth[3] = {0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int c = seq[(int)(((long long)gw * 7919 + i) % nseq)];
        far_tb<PT>(x, y, z, xb, yb, zb, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, oth, kp, lane, ws);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, oth[c], kGroup);
    double t = acc[0] + acc[1] + acc[2];
    if (t == 1.2345) out[0] = t;
}


__device__ __forceinline__ void pair_row_nomufu(double dx, double dy, double dz, double s, const double* f,
                                                double* acc, EvalKern<0>::Row& r, const KParams& k) {
    const double y = s;
    const double Y = y * fma(-(s * y), y, 3.0);
    const double Y3 = (Y * Y) * Y;
    const double h = fma(k.e2q, Y3, Y);
    const double c = fma(f[0], dx, fma(f[1], dy, f[2] * dz)) * Y3;
    r.C += c;
    r.Z = fma(c, dz, r.Z);
    acc[0] = fma(f[0], h, acc[0]);
    acc[1] = fma(f[1], h, acc[1]);
    acc[2] = fma(f[2], h, acc[2]);
}

// Variant 2 (ablation): the production two-rows-per-lane path (dz in registers) with
//   V & 1: no TMA / mbarrier (the stage buffers are read as they are)
//   V & 2: no shared loads (f-hat values formed from registers)
//   V & 4: no partial last block
template <int PT, int V>
__device__ __forceinline__ void far_var(double x, double y, double z, const double* __restrict__ g,
                                        const double* __restrict__ F, double* acc, const KParams& kp, int grp,
                                        int lane, const WarpSmem& ws, const double* __restrict__ Fn = nullptr) {
    using K = EvalKern<0>;
    constexpr int P = PT, M = 3, P2 = P * P, R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    constexpr int blk = P * M * kRows, NS = (R + 1) / 2;
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nb = min(2, R - st * 2);
        tma_round(ws.buf + (k & 1) * 2 * blk, F + (size_t)st * 2 * blk, (unsigned)(nb * blk * 8), ws.bar + (k & 1));
    };
    // V & 64: cross-cluster prefetch -- this cluster's first two stages were issued by the
    // previous call; the last two stage slots issue the NEXT cluster's (Fn) first two stages
    auto issue_n = [&](int st, int k) {
        const int nb = min(2, R - st * 2);
        tma_round(ws.buf + (k & 1) * 2 * blk, Fn + (size_t)st * 2 * blk, (unsigned)(nb * blk * 8), ws.bar + (k & 1));
    };
    if (!(V & 1) && !(V & 64) && lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    double dzr[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) dzr[k3] = z - __ldg(g + 2 * P + k3);
#pragma unroll((V & 32) ? NS : 1)
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * 2 * blk;
        if (!(V & 1)) mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int b0 = st * 2;
        if (b0 + 1 < RF) {
            const int h = grp >> 2, j = 2 * (grp & 3);
            const int ra = (b0 + h) * kRows + j;
            const int k1a = ra / P, k2a = ra - k1a * P;
            const int k1b = k2a + 1 == P ? k1a + 1 : k1a, k2b = k2a + 1 == P ? 0 : k2a + 1;
            const double dxa = x - __ldg(g + k1a), dya = y - __ldg(g + P + k2a);
            const double dxb = x - __ldg(g + k1b), dyb = y - __ldg(g + P + k2b);
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Bh = B + h * blk + j;
            typename K::Row rA, rB;
            double fa_prev[M] = {0, 0, 0}, fb_prev[M] = {0, 0, 0};
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                double fa[M], fb[M];
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    if (V & 2) {
                        fa[m] = dzr[(k3 + m + 1) % P];
                        fb[m] = dzr[(k3 + m + 2) % P];
                    } else if ((V & 8) && (k3 & 1)) {  // half the shared loads: odd k3 reuse the even k3's values
                        fa[m] = fa_prev[m];
                        fb[m] = fb_prev[m];
                    } else {
                        const double2 v = *reinterpret_cast<const double2*>(Bh + (k3 * M + m) * kRows);
                        fa[m] = v.x;
                        fb[m] = v.y;
                    }
                }
#pragma unroll
                for (int m = 0; m < M; ++m) {
                    fa_prev[m] = fa[m];
                    fb_prev[m] = fb[m];
                }
                const double zk = dzr[k3];
                if (V & 16) {  // no MUFU: the seed is s itself (same FP64 instruction count)
                    pair_row_nomufu(dxa, dya, zk, fma(zk, zk, pa), fa, acc, rA, kp);
                    pair_row_nomufu(dxb, dyb, zk, fma(zk, zk, pb), fb, acc, rB, kp);
                } else {
                    K::pair_row(dxa, dya, zk, fma(zk, zk, pa), fa, acc, rA, kp);
                    K::pair_row(dxb, dyb, zk, fma(zk, zk, pb), fb, acc, rB, kp);
                }
            }
            K::row_end(dxa, dya, rA, acc);
            K::row_end(dxb, dyb, rB, acc);
        } else if (!(V & 4)) {
            for (int bb = b0; bb < min(b0 + 2, R); ++bb) {
                const double* Bb = B + (bb - b0) * blk;
                const int pairs = (bb < RF ? kRows : P2 - RF * kRows) * P;
                for (int q = grp; q < pairs; q += kRows) {
                    const int jj = q / P, k3 = q - jj * P, row = bb * kRows + jj;
                    const int k1 = row / P, k2 = row - k1 * P;
                    const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2), dzk = z - __ldg(g + 2 * P + k3);
                    double f[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) f[m] = Bb[(k3 * M + m) * kRows + jj];
                    K::pair(dx, dy, dzk, fma(dy, dy, dx * dx) + fma(dzk, dzk, kp.e2), f, acc, kp);
                }
            }
        }
        if (!(V & 32)) __syncwarp();
        if (!(V & 1) && lane == 0 && st + 2 < NS) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(st + 2, k);
        } else if ((V & 64) && lane == 0 && Fn && st + 2 - NS < NS) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_n(st + 2 - NS, k);
        }
    }
    if (!(V & 1) && lane == 0) *ws.nround = base + NS;
    __syncwarp();
}

template <int PT, int V>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, 0>())
    k_far_var(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out,
              KParams kp, int warp_smem) {
    constexpr int M = 3, P = PT;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int grp = lane % kGroup, ti = lane / kGroup;
    WarpSmem ws;
    {
        const int blk = P * M * kRows;
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + 2 * kSB * blk * sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        ws.dzs = reinterpret_cast<double*>(ws.bar + 3);
        ws.stk = reinterpret_cast<int2*>(ws.dzs + kBatch * P);
        for (int i = lane; i < 4 * blk; i += 32) ws.buf[i] = 0.001 * (i % 97) - 0.04;
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const long long LEN = (long long)((P * P + kRows - 1) / kRows) * P * M * kRows;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 3.0 + 0.01 * ti, y = 2.5 - 0.003 * ti, z = 2.0 + 0.002 * ti;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    if (V & 64) {  // prime: the first cluster's first two stages
        const int c0 = seq[(int)(((long long)gw * 7919) % nseq)];
        constexpr int blk = P * M * kRows, R = (P * P + kRows - 1) / kRows;
        if (lane == 0) {
            tma_round(ws.buf, fhat + (size_t)c0 * LEN, (unsigned)(min(2, R) * blk * 8), ws.bar);
            if (R > 2) tma_round(ws.buf + 2 * blk, fhat + (size_t)c0 * LEN + 2 * blk, (unsigned)(min(2, R - 2) * blk * 8), ws.bar + 1);
        }
        __syncwarp();
    }
    for (int i = 0; i < ncalls; ++i) {
        const int c = seq[(int)(((long long)gw * 7919 + i) % nseq)];
        const int cn = seq[(int)(((long long)gw * 7919 + i + 1) % nseq)];
        far_var<PT, V>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, grp, lane, ws,
                       (V & 64) && i + 1 < ncalls ? fhat + (size_t)cn * LEN : nullptr);
    }
    double t = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5];
    if (t == 1.2345) out[0] = t;
}

// Variant 3: target pairs (as far_tb) with a ROW-CONTIGUOUS f-hat layout: row r of a cluster
// holds its P x M values (k3-major, m fastest) at stride RS doubles, so a lane fetches its
// row with 16-byte loads and every loaded value feeds two pairs (0.78 loads per pair).
template <int PT>
__device__ __forceinline__ void far_tb2(double xA, double yA, double zA, double xB, double yB, double zB,
                                        const double* __restrict__ g, const double* __restrict__ F, double* accA,
                                        double* accB, const KParams& kp, int lane, const WarpSmem& ws) {
    constexpr int P = PT, M = 3, P2 = P * P, NV = P * M, RS = ((NV + 1) / 2 * 2) | 2;  // 30 at P = 9
    constexpr int SR = 16, NS = (P2 + SR - 1) / SR;  // rows per stage, stages
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nr = min(SR, P2 - st * SR);
        tma_round(ws.buf + (k & 1) * SR * RS, F + (size_t)st * SR * RS, (unsigned)(nr * RS * 8), ws.bar + (k & 1));
    };
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    double dzA[P], dzB[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) {
        const double gz = __ldg(g + 2 * P + k3);
        dzA[k3] = zA - gz;
        dzB[k3] = zB - gz;
    }
    const int q = lane & 15;
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * SR * RS;
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int nr = min(SR, P2 - st * SR);
        if (nr == SR) {
            const int row = st * SR + q;
            const int k1 = row / P, k2 = row - k1 * P;
            const double gx = __ldg(g + k1), gy = __ldg(g + P + k2);
            const double dxa = xA - gx, dya = yA - gy, dxb = xB - gx, dyb = yB - gy;
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Br = B + q * RS;
            double v[NV + 1];
#pragma unroll
            for (int i = 0; i < NV / 2; ++i) {
                const double2 t = *reinterpret_cast<const double2*>(Br + 2 * i);
                v[2 * i] = t.x;
                v[2 * i + 1] = t.y;
            }
            if (NV & 1) v[NV - 1] = Br[NV - 1];
            double CA = 0.0, ZA = 0.0, CB = 0.0, ZB = 0.0;
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                const double f0 = v[3 * k3], f1 = v[3 * k3 + 1], f2 = v[3 * k3 + 2];
                {
                    const double dz = dzA[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pa));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxa, fma(f1, dya, f2 * dz)) * Y3;
                    CA += c;
                    ZA = fma(c, dz, ZA);
                    accA[0] = fma(f0, hh, accA[0]);
                    accA[1] = fma(f1, hh, accA[1]);
                    accA[2] = fma(f2, hh, accA[2]);
                }
                {
                    const double dz = dzB[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pb));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxb, fma(f1, dyb, f2 * dz)) * Y3;
                    CB += c;
                    ZB = fma(c, dz, ZB);
                    accB[0] = fma(f0, hh, accB[0]);
                    accB[1] = fma(f1, hh, accB[1]);
                    accB[2] = fma(f2, hh, accB[2]);
                }
            }
            CA *= 0.25;
            CB *= 0.25;
            accA[0] = fma(CA, dxa, accA[0]);
            accA[1] = fma(CA, dya, accA[1]);
            accA[2] = fma(0.25, ZA, accA[2]);
            accB[0] = fma(CB, dxb, accB[0]);
            accB[1] = fma(CB, dyb, accB[1]);
            accB[2] = fma(0.25, ZB, accB[2]);
        } else {
            // partial last stage: (row, k3) pairs over the 16 lanes of the half-warp
            for (int qq = q; qq < nr * P; qq += 16) {
                const int jj = qq / P, k3 = qq - jj * P, row = st * SR + jj;
                const int k1 = row / P, k2 = row - k1 * P;
                const double gx = __ldg(g + k1), gy = __ldg(g + P + k2), gz = __ldg(g + 2 * P + k3);
                const double* Br = B + jj * RS + 3 * k3;
                const double f[3] = {Br[0], Br[1], Br[2]};
                double t6[6] = {0, 0, 0, 0, 0, 0};
                {
                    const double dx = xA - gx, dy = yA - gy, dz = zA - gz;
                    EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, t6, kp);
                    accA[0] = fma(0.25, t6[3], accA[0] + t6[0]);
                    accA[1] = fma(0.25, t6[4], accA[1] + t6[1]);
                    accA[2] = fma(0.25, t6[5], accA[2] + t6[2]);
                }
                double u6[6] = {0, 0, 0, 0, 0, 0};
                {
                    const double dx = xB - gx, dy = yB - gy, dz = zB - gz;
                    EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, u6, kp);
                    accB[0] = fma(0.25, u6[3], accB[0] + u6[0]);
                    accB[1] = fma(0.25, u6[4], accB[1] + u6[1]);
                    accB[2] = fma(0.25, u6[5], accB[2] + u6[2]);
                }
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
}

template <int PT>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, 0>())
    k_far_tb2(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out,
              KParams kp, int warp_smem) {
    constexpr int P = PT, M = 3, NV = P * M, RS = ((NV + 1) / 2 * 2) | 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ti = lane / kGroup;
    WarpSmem ws;
    {
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + 2 * 16 * RS * sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const long long LEN = (long long)P * P * RS;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 3.0 + 0.01 * ti, y = 2.5 - 0.003 * ti, z = 2.0 + 0.002 * ti;
    const double xb = __shfl_xor_sync(0xffffffffu, x, kGroup), yb = __shfl_xor_sync(0xffffffffu, y, kGroup),
                 zb = __shfl_xor_sync(0xffffffffu, z, kGroup);
    double acc[3] = {0, 0, 0}, oth[3] = {0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int c = seq[(int)(((long long)gw * 7919 + i) % nseq)];
        far_tb2<PT>(x, y, z, xb, yb, zb, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, oth, kp, lane, ws);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, oth[c], kGroup);
    double t = acc[0] + acc[1] + acc[2];
    if (t == 1.2345) out[0] = t;
}

// Variant 4: as far_tb2 with the row stored m-major ([m][k3], m stride 10), loaded per k3 pair: row r of a cluster
// holds its P x M values (k3-major, m fastest) at stride RS doubles, so a lane fetches its
// row with 16-byte loads and every loaded value feeds two pairs (0.78 loads per pair).
template <int PT>
__device__ __forceinline__ void far_tb3(double xA, double yA, double zA, double xB, double yB, double zB,
                                        const double* __restrict__ g, const double* __restrict__ F, double* accA,
                                        double* accB, const KParams& kp, int lane, const WarpSmem& ws) {
    constexpr int P = PT, M = 3, P2 = P * P, MS = (P + 1) / 2 * 2, RS = 3 * MS;  // 30 at P = 9
    constexpr int SR = 16, NS = (P2 + SR - 1) / SR;  // rows per stage, stages
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nr = min(SR, P2 - st * SR);
        tma_round(ws.buf + (k & 1) * SR * RS, F + (size_t)st * SR * RS, (unsigned)(nr * RS * 8), ws.bar + (k & 1));
    };
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NS > 1) issue(1, base + 1);
    }
    double dzA[P], dzB[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) {
        const double gz = __ldg(g + 2 * P + k3);
        dzA[k3] = zA - gz;
        dzB[k3] = zB - gz;
    }
    const int q = lane & 15;
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (k & 1) * SR * RS;
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int nr = min(SR, P2 - st * SR);
        if (nr == SR) {
            const int row = st * SR + q;
            const int k1 = row / P, k2 = row - k1 * P;
            const double gx = __ldg(g + k1), gy = __ldg(g + P + k2);
            const double dxa = xA - gx, dya = yA - gy, dxb = xB - gx, dyb = yB - gy;
            const double pa = fma(dya, dya, dxa * dxa) + kp.e2;
            const double pb = fma(dyb, dyb, dxb * dxb) + kp.e2;
            const double* Br = B + q * RS;
            double CA = 0.0, ZA = 0.0, CB = 0.0, ZB = 0.0;
            double w[3][2];
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                if ((k3 & 1) == 0) {
#pragma unroll
                    for (int m = 0; m < 3; ++m) {
                        const double2 t = *reinterpret_cast<const double2*>(Br + m * MS + k3);
                        w[m][0] = t.x;
                        w[m][1] = t.y;
                    }
                }
                const double f0 = w[0][k3 & 1], f1 = w[1][k3 & 1], f2 = w[2][k3 & 1];
                {
                    const double dz = dzA[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pa));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxa, fma(f1, dya, f2 * dz)) * Y3;
                    CA += c;
                    ZA = fma(c, dz, ZA);
                    accA[0] = fma(f0, hh, accA[0]);
                    accA[1] = fma(f1, hh, accA[1]);
                    accA[2] = fma(f2, hh, accA[2]);
                }
                {
                    const double dz = dzB[k3];
                    const double Y = rsqrt2_newton(fma(dz, dz, pb));
                    const double Y3 = (Y * Y) * Y;
                    const double hh = fma(kp.e2q, Y3, Y);
                    const double c = fma(f0, dxb, fma(f1, dyb, f2 * dz)) * Y3;
                    CB += c;
                    ZB = fma(c, dz, ZB);
                    accB[0] = fma(f0, hh, accB[0]);
                    accB[1] = fma(f1, hh, accB[1]);
                    accB[2] = fma(f2, hh, accB[2]);
                }
            }
            CA *= 0.25;
            CB *= 0.25;
            accA[0] = fma(CA, dxa, accA[0]);
            accA[1] = fma(CA, dya, accA[1]);
            accA[2] = fma(0.25, ZA, accA[2]);
            accB[0] = fma(CB, dxb, accB[0]);
            accB[1] = fma(CB, dyb, accB[1]);
            accB[2] = fma(0.25, ZB, accB[2]);
        } else {
            // partial last stage: (row, k3) pairs over the 16 lanes of the half-warp
            for (int qq = q; qq < nr * P; qq += 16) {
                const int jj = qq / P, k3 = qq - jj * P, row = st * SR + jj;
                const int k1 = row / P, k2 = row - k1 * P;
                const double gx = __ldg(g + k1), gy = __ldg(g + P + k2), gz = __ldg(g + 2 * P + k3);
                const double* Br = B + jj * RS + k3;
                const double f[3] = {Br[0], Br[MS], Br[2 * MS]};
                double t6[6] = {0, 0, 0, 0, 0, 0};
                {
                    const double dx = xA - gx, dy = yA - gy, dz = zA - gz;
                    EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, t6, kp);
                    accA[0] = fma(0.25, t6[3], accA[0] + t6[0]);
                    accA[1] = fma(0.25, t6[4], accA[1] + t6[1]);
                    accA[2] = fma(0.25, t6[5], accA[2] + t6[2]);
                }
                double u6[6] = {0, 0, 0, 0, 0, 0};
                {
                    const double dx = xB - gx, dy = yB - gy, dz = zB - gz;
                    EvalKern<0>::pair(dx, dy, dz, fma(dy, dy, dx * dx) + fma(dz, dz, kp.e2), f, u6, kp);
                    accB[0] = fma(0.25, u6[3], accB[0] + u6[0]);
                    accB[1] = fma(0.25, u6[4], accB[1] + u6[1]);
                    accB[2] = fma(0.25, u6[5], accB[2] + u6[2]);
                }
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
}

template <int PT>
__global__ void __launch_bounds__(kWarps * 32, eval_min_blocks<PT, 0>())
    k_far_tb3(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out,
              KParams kp, int warp_smem) {
    constexpr int P = PT, M = 3, NV = P * M, RS = ((NV + 1) / 2 * 2) | 2;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ti = lane / kGroup;
    WarpSmem ws;
    {
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + 2 * 16 * RS * sizeof(double));
        ws.nround = reinterpret_cast<int*>(ws.bar + 2);
        if (lane == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar)));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(ws.bar + 1)));
            *ws.nround = 0;
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();
    }
    const long long LEN = (long long)P * P * RS;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 3.0 + 0.01 * ti, y = 2.5 - 0.003 * ti, z = 2.0 + 0.002 * ti;
    const double xb = __shfl_xor_sync(0xffffffffu, x, kGroup), yb = __shfl_xor_sync(0xffffffffu, y, kGroup),
                 zb = __shfl_xor_sync(0xffffffffu, z, kGroup);
    double acc[3] = {0, 0, 0}, oth[3] = {0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int c = seq[(int)(((long long)gw * 7919 + i) % nseq)];
        far_tb3<PT>(x, y, z, xb, yb, zb, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, oth, kp, lane, ws);
    }
#pragma unroll
    for (int c = 0; c < 3; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, oth[c], kGroup);
    double t = acc[0] + acc[1] + acc[2];
    if (t == 1.2345) out[0] = t;
}

template <int PT>
void run(int sms, int clk_khz) {
    constexpr int M = 3, P = PT;
    const int nclu = 1169;
    const long long LEN = std::max((long long)((P * P + kRows - 1) / kRows) * P * M * kRows, (long long)P * P * 30);
    std::vector<double> hg((size_t)nclu * 3 * P), hf((size_t)nclu * LEN);
    srand(1);
    for (auto& v : hg) v = -1.0 + 2.0 * rand() / RAND_MAX;
    for (auto& v : hf) v = -1.0 + 2.0 * rand() / RAND_MAX;
    const int nseq = 1 << 16;
    std::vector<int> hs(nseq);
    for (auto& v : hs) v = rand() % nclu;
    double *g, *f, *o;
    int* s;
    cudaMalloc(&g, hg.size() * 8);
    cudaMalloc(&f, hf.size() * 8);
    cudaMalloc(&o, 8);
    cudaMalloc(&s, nseq * 4);
    cudaMemcpy(g, hg.data(), hg.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(f, hf.data(), hf.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(s, hs.data(), nseq * 4, cudaMemcpyHostToDevice);
    const int warp_smem = (int)(((size_t)2 * kSB * P * M * kRows * 8 + 24 + 64 * 8 + (size_t)kBatch * P * 8 + 127) /
                                128 * 128);
    // FAR_PROBE_EXTRA_SMEM (bytes per CTA): enlarge the shared-memory carve-out (less L1) without using it
    const size_t smem = (size_t)kWarps * warp_smem + (getenv("FAR_PROBE_EXTRA_SMEM") ? atoi(getenv("FAR_PROBE_EXTRA_SMEM")) : 0);
    cudaFuncSetAttribute(k_far_probe<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_tb<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 9>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 17>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 23>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_tb3<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_tb2<PT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 33>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_far_var<PT, 37>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ctas = sms * eval_min_blocks<PT, 0>() * 8, ncalls = 48;
    const KParams kp = make_kparams(0.01);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[13] = {"far_field (prod)", "far_tb (v1)", "var 0 (copy of prod)", "var 1 no TMA",
                            "var 3 no TMA, no LDS", "var 4 no tail", "var 7 math only", "var 9 no TMA, half LDS",
                            "var 17 no TMA, no MUFU", "var 23 math, no MUFU", "far_tb2 row-contiguous", "var 64 cross-cluster prefetch", "far_tb3 m-major k3 pairs"};
    for (int rep = 0; rep < 39; ++rep) {
        const int V = rep % 13;
        cudaEventRecord(e0);
        if (V == 0) k_far_probe<PT><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 1) k_far_tb<PT><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 2) k_far_var<PT, 0><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 3) k_far_var<PT, 1><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 4) k_far_var<PT, 3><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 5) k_far_var<PT, 4><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 6) k_far_var<PT, 7><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 7) k_far_var<PT, 9><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 8) k_far_var<PT, 17><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 9) k_far_var<PT, 23><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 10) k_far_tb2<PT><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 11) k_far_var<PT, 64><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else k_far_tb3<PT><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double pairs = (double)ctas * kWarps * ncalls * 4 * P * P * P;
        const double rate = pairs / (ms * 1e-3);
        if (rep >= 13)
            printf("P %2d %-22s %.3f ms, %.3f pairs/clk/SM, %.2f TFLOP/s = %.1f%% of %.2f (err %s)\n", P, names[V],
                   ms, rate / (sms * clk_khz * 1e3), rate * 32e-12,
                   100.0 * rate * 32 / (sms * 128.0 * clk_khz * 1e3), sms * 128.0 * clk_khz * 1e-9,
                   cudaGetErrorString(cudaGetLastError()));
    }
    cudaFree(g);
    cudaFree(f);
    cudaFree(o);
    cudaFree(s);
}

}  // namespace
}  // namespace kitc

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int clk = 1965000;  // sm_max_mhz (MEASURED_PEAKS.json): the derived peak's clock
    kitc::run<9>(sms, clk);
    return 0;
}
