// Far field at low degree in isolation (tuning probe): the production far_field<PT, 0> against
// far_small<PT> -- the whole cluster's f-hat in ONE bulk copy and one wait, every lane of a target
// group taking the rows grp, grp + 8, grp + 16, .. (independent row chains) and the P^2 mod 8
// leftover rows pair by pair.  All 4 targets accept; 1169 clusters, L2-resident.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1902_02250_b200/csrc/eval.cu"

namespace kitc {
namespace {

template <int PT, int KER, int RG>
__device__ __forceinline__ void far_small(double x, double y, double z, const double* __restrict__ g,
                                          const double* __restrict__ F, double* acc, const KParams& kp, int grp,
                                          int lane, const WarpSmem& ws) {
    using K = EvalKern<KER>;
    constexpr int P = PT, M = K::M, P2 = P * P, R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    constexpr int blk = P * M * kRows;
    const int k = *ws.nround;
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        tma_round(ws.buf, F, (unsigned)(R * blk * 8), ws.bar + (k & 1));
    }
    double dzr[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) dzr[k3] = z - __ldg(g + 2 * P + k3);
    mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
    const double* B = ws.buf;
#pragma unroll 1
    for (int r0 = 0; r0 < RF; r0 += RG) {
        constexpr int NR = RG;
        double dx[NR], dy[NR], pp[NR];
        typename K::Row rw[NR];
#pragma unroll
        for (int i = 0; i < NR; ++i) {
            const int r = min(r0 + i, RF - 1);
            const int row = r * kRows + grp, k1 = row / P, k2 = row - k1 * P;
            dx[i] = x - __ldg(g + k1);
            dy[i] = y - __ldg(g + P + k2);
            pp[i] = fma(dy[i], dy[i], dx[i] * dx[i]) + kp.e2;
        }
#pragma unroll
        for (int k3 = 0; k3 < P; ++k3) {
            const double zk = dzr[k3];
#pragma unroll
            for (int i = 0; i < NR; ++i) {
                if (RF % RG != 0 && r0 + i >= RF) continue;
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = B[((r0 + i) * P + k3) * M * kRows + m * kRows + grp];
                K::pair_row(dx[i], dy[i], zk, fma(zk, zk, pp[i]), f, acc, rw[i], kp);
            }
        }
#pragma unroll
        for (int i = 0; i < NR; ++i)
            if (RF % RG == 0 || r0 + i < RF) K::row_end(dx[i], dy[i], rw[i], acc);
    }
    if (P2 > RF * kRows) {  // leftover rows of the partial block, pair by pair over the group's lanes
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
    __syncwarp();
    if (lane == 0) *ws.nround = k + 1;
    __syncwarp();
}


// Variant for larger P: stages of SBK blocks (all rows of a stage: one per lane per full block,
// in row groups of <= 3 chains), NBUF = 1 (one buffer, stages in sequence) or 2 (double buffer).
template <int PT, int KER, int SBK, int NBUF>
__device__ __forceinline__ void far_stages(double x, double y, double z, const double* __restrict__ g,
                                           const double* __restrict__ F, double* acc, const KParams& kp, int grp,
                                           int lane, const WarpSmem& ws) {
    using K = EvalKern<KER>;
    constexpr int P = PT, M = K::M, P2 = P * P, R = (P2 + kRows - 1) / kRows, RF = P2 / kRows;
    constexpr int blk = P * M * kRows, NS = (R + SBK - 1) / SBK;
    const int base = *ws.nround;
    auto issue = [&](int st, int k) {
        const int nb = min(SBK, R - st * SBK);
        tma_round(ws.buf + (NBUF == 2 ? (k & 1) * SBK * blk : 0), F + (size_t)st * SBK * blk, (unsigned)(nb * blk * 8),
                  ws.bar + (k & 1));
    };
    if (lane == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(0, base);
        if (NBUF == 2 && NS > 1) issue(1, base + 1);
    }
    double dzr[P];
#pragma unroll
    for (int k3 = 0; k3 < P; ++k3) dzr[k3] = z - __ldg(g + 2 * P + k3);
#pragma unroll 1
    for (int st = 0; st < NS; ++st) {
        const int k = base + st;
        const double* B = ws.buf + (NBUF == 2 ? (k & 1) * SBK * blk : 0);
        mbar_wait(ws.bar + (k & 1), (unsigned)(k >> 1) & 1u);
        const int b0 = st * SBK, nfull = max(0, min(SBK, RF - b0));
        // full blocks of this stage in row groups of 3 / 2 / 1
        int r = 0;
#pragma unroll 1
        for (; r + 3 <= nfull; r += 3) {
            double dx[3], dy[3], pp[3];
            typename K::Row rw[3];
#pragma unroll
            for (int i = 0; i < 3; ++i) {
                const int row = (b0 + r + i) * kRows + grp, k1 = row / P, k2 = row - k1 * P;
                dx[i] = x - __ldg(g + k1);
                dy[i] = y - __ldg(g + P + k2);
                pp[i] = fma(dy[i], dy[i], dx[i] * dx[i]) + kp.e2;
            }
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                const double zk = dzr[k3];
#pragma unroll
                for (int i = 0; i < 3; ++i) {
                    double f[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) f[m] = B[((r + i) * P + k3) * M * kRows + m * kRows + grp];
                    K::pair_row(dx[i], dy[i], zk, fma(zk, zk, pp[i]), f, acc, rw[i], kp);
                }
            }
#pragma unroll
            for (int i = 0; i < 3; ++i) K::row_end(dx[i], dy[i], rw[i], acc);
        }
#pragma unroll 1
        for (; r + 2 <= nfull; r += 2) {
            double dx[2], dy[2], pp[2];
            typename K::Row rw[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) {
                const int row = (b0 + r + i) * kRows + grp, k1 = row / P, k2 = row - k1 * P;
                dx[i] = x - __ldg(g + k1);
                dy[i] = y - __ldg(g + P + k2);
                pp[i] = fma(dy[i], dy[i], dx[i] * dx[i]) + kp.e2;
            }
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                const double zk = dzr[k3];
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    double f[M];
#pragma unroll
                    for (int m = 0; m < M; ++m) f[m] = B[((r + i) * P + k3) * M * kRows + m * kRows + grp];
                    K::pair_row(dx[i], dy[i], zk, fma(zk, zk, pp[i]), f, acc, rw[i], kp);
                }
            }
#pragma unroll
            for (int i = 0; i < 2; ++i) K::row_end(dx[i], dy[i], rw[i], acc);
        }
        if (r < nfull) {
            const int row = (b0 + r) * kRows + grp, k1 = row / P, k2 = row - k1 * P;
            const double dx = x - __ldg(g + k1), dy = y - __ldg(g + P + k2);
            const double pp = fma(dy, dy, dx * dx) + kp.e2;
            typename K::Row rw;
#pragma unroll
            for (int k3 = 0; k3 < P; ++k3) {
                double f[M];
#pragma unroll
                for (int m = 0; m < M; ++m) f[m] = B[(r * P + k3) * M * kRows + m * kRows + grp];
                K::pair_row(dx, dy, dzr[k3], fma(dzr[k3], dzr[k3], pp), f, acc, rw, kp);
            }
            K::row_end(dx, dy, rw, acc);
        }
        if (b0 + SBK >= R && P2 > RF * kRows) {  // partial block (last stage)
            const double* Bb = B + (RF - b0) * blk;
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
        __syncwarp();
        if (lane == 0) {
            const int nx = NBUF == 2 ? st + 2 : st + 1;
            if (nx < NS) {
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                issue(nx, NBUF == 2 ? k + 2 : k + 1);
            }
        }
    }
    if (lane == 0) *ws.nround = base + NS;
    __syncwarp();
}

#ifndef FSP_MINB
#define FSP_MINB 4
#endif
template <int PT, int KER, int V>
__global__ void __launch_bounds__(kWarps * 32, FSP_MINB)
    k_probe(const double* grid, const double* fhat, const int* seq, int nseq, int ncalls, double* out, KParams kp,
            int warp_smem) {
    constexpr int M = EvalKern<KER>::M, P = PT, NA = EvalKern<KER>::NA;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int grp = lane % kGroup, ti = lane / kGroup;
    WarpSmem ws;
    {
        const int R = (P * P + kRows - 1) / kRows, blk = P * M * kRows;
        unsigned char* base = smem_raw + (size_t)wl * warp_smem;
        ws.buf = reinterpret_cast<double*>(base);
        ws.bar = reinterpret_cast<unsigned long long*>(base + (size_t)(V >= 6 ? 6 : V ? R : 2 * kSB) * blk * sizeof(double));
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
        if constexpr (V == 0)
            far_field<PT, KER>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, P, grp, lane,
                               0xffffffffu, ws);
        else if constexpr (V == 6)
            far_stages<PT, KER, 6, 1>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, grp, lane, ws);
        else if constexpr (V == 7)
            far_stages<PT, KER, 3, 2>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, grp, lane, ws);
        else if constexpr (V == 8)
            far_stages<PT, KER, 4, 1>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, grp, lane, ws);
        else
            far_small<PT, KER, V>(x, y, z, grid + (size_t)c * 3 * P, fhat + (size_t)c * LEN, acc, kp, grp, lane, ws);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < NA; ++c) t += acc[c];
    if (t == 1.2345) out[0] = t;
}

template <int PT, int KER>
void run(int sms, int clk_khz) {
    constexpr int M = EvalKern<KER>::M, P = PT;
    const int nclu = 1169;
    const long long LEN = (long long)((P * P + kRows - 1) / kRows) * P * M * kRows;
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
    const int R = (P * P + kRows - 1) / kRows;
    const int warp_smem = (int)(((size_t)std::max(std::max(2 * kSB, R), 6) * P * M * kRows * 8 + 24 + 64 * 8 + (size_t)kBatch * P * 8 +
                                 127) / 128 * 128);
    const size_t smem = (size_t)kWarps * warp_smem;
    cudaFuncSetAttribute(k_probe<PT, KER, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_probe<PT, KER, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int ctas = sms * 4 * 8, ncalls = 192;
    const KParams kp = make_kparams(0.01);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
#ifdef FSP_BIG
    const int VS[4] = {0, 2, 5, 0};
#else
    const int VS[4] = {0, 6, 7, 8};
#endif
    for (int rep = 0; rep < 8; ++rep) {
        const int V = VS[rep % 4];
        cudaEventRecord(e0);
        if (V == 0) k_probe<PT, KER, 0><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 6) k_probe<PT, KER, 6><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 7) k_probe<PT, KER, 7><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 2) k_probe<PT, KER, 2><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else if (V == 5) k_probe<PT, KER, 5><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        else k_probe<PT, KER, 8><<<ctas, kWarps * 32, smem>>>(g, f, s, nseq, ncalls, o, kp, warp_smem);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        const double pairs = (double)ctas * kWarps * ncalls * 4 * P * P * P;
        const double rate = pairs / (ms * 1e-3);
        const double fl = KER == 0 ? 32 : 59;
        if (rep >= 4)
            printf("K %d P %2d %-18s %.3f ms, %.3f pairs/clk/SM, %.1f%% of %.2f TFLOP/s (err %s)\n", KER, P,
                   V == 0 ? "far_field (prod)" : V == 6 ? "stages 6 blk x1 buf" : V == 7 ? "stages 3 blk x2 buf" : V == 2 ? "whole cluster RG2" : V == 5 ? "whole cluster RG5" : "stages 4 blk x1 buf", ms,
                   rate / (sms * clk_khz * 1e3), 100.0 * rate * fl / (sms * 128.0 * clk_khz * 1e3),
                   sms * 128.0 * clk_khz * 1e-9,
                   cudaGetErrorString(cudaGetLastError()));
    }
}

}  // namespace
}  // namespace kitc

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    kitc::run<9, 0>(sms, 1965000);
    kitc::run<10, 0>(sms, 1965000);
    return 0;
}
