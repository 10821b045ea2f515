// Near-field loop in isolation (tuning probe, not part of libkitc): every warp runs the
// production near_leaf<0, 9> (eval.cu: target pairs, 4 records in flight) for a batch of
// 4 targets over a random sequence of "leaves" (ranges of 250..2000 packed source records
// of an N = 1e6 array, L2-resident as in k_eval at C3).  Prints pairs/clk/SM and the
// algorithmic rate (32 flop/pair) against the derived FP64 peak.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1902_02250_b200/csrc/eval.cu"

namespace kitc {
namespace {

template <int V>
__global__ void __launch_bounds__(kWarps * 32, 4) k_near_probe(EvalArgs a, const int2* leaves, int nleaf, int ncalls) {
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ti = lane / kGroup;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 0.1 + 0.001 * ti, y = -0.2 + 0.0007 * ti, z = 0.3 - 0.0003 * ti;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int2 L = leaves[(int)(((long long)gw * 7919 + i) % nleaf)];
        near_leaf<0, 9>(x, y, z, -1, L.x, L.y, lane, 0xffffffffu, a, acc);
    }
    double t = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5];
    if (t == 1.2345) a.out[0] = t;
}


// Variants of near_field_tb (Stokeslet, no self pair): V = 0 global records (copy of prod),
// 1 records from shared memory (a 512-record window: timing only), 2 no loads (register records)
template <int V, int U>
__device__ __forceinline__ void near_var(double xa, double ya, double za, double xb, double yb, double zb, int b, int e,
                                         int rk, const EvalArgs& a, const double* sm, double* accA, double* accB) {
    using K = EvalKern<0>;
    constexpr int M = 3, NQ = 3, TS = 16;
    double base[U][NQ * 2];
    if (V == 2) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int q = 0; q < NQ * 2; ++q) base[u][q] = a.src[(size_t)(b + rk + u) * a.sld + q];
    }
    int j = b + rk;
    for (; j + (U - 1) * TS < e; j += U * TS) {
        double v[U][NQ * 2];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if ((V & 3) == 0) {
                const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)(j + u * TS) * a.sld);
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const double2 d2 = __ldg(r + q);
                    v[u][2 * q] = d2.x;
                    v[u][2 * q + 1] = d2.y;
                }
            } else if ((V & 3) == 1) {
                const double2* r = reinterpret_cast<const double2*>(sm + ((j + u * TS) & 511) * 6);
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const double2 d2 = r[q];
                    v[u][2 * q] = d2.x;
                    v[u][2 * q + 1] = d2.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < NQ * 2; ++q) {
                    v[u][q] = base[u][q];
                    asm volatile("" : "+d"(v[u][q]));
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            {
                const double dx = xa - v[u][0], dy = ya - v[u][1], dz = za - v[u][2];
                K::pair(dx, dy, dz, fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))), &v[u][3], accA, a.kp);
            }
            {
                const double dx = xb - v[u][0], dy = yb - v[u][1], dz = zb - v[u][2];
                K::pair(dx, dy, dz, fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))), &v[u][3], accB, a.kp);
            }
        }
    }
    if (V & 4) {  // prod-style serial remainder
        for (; j < e; j += TS) {
            const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)j * a.sld);
            double v[NQ * 2];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const double2 d2 = __ldg(r + q);
                v[2 * q] = d2.x;
                v[2 * q + 1] = d2.y;
            }
            const double dxa = xa - v[0], dya = ya - v[1], dza = za - v[2];
            const double dxb = xb - v[0], dyb = yb - v[1], dzb = zb - v[2];
            K::pair(dxa, dya, dza, fma(dxa, dxa, fma(dya, dya, fma(dza, dza, a.kp.e2))), &v[3], accA, a.kp);
            K::pair(dxb, dyb, dzb, fma(dxb, dxb, fma(dyb, dyb, fma(dzb, dzb, a.kp.e2))), &v[3], accB, a.kp);
        }
    }
    if (V & 8) {  // masked unrolled remainder: out-of-range records read record e-1 with f = 0, s = 1
        if (j < e) {
            double v[U][NQ * 2];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int jj = min(j + u * TS, e - 1);
                const double2* r = reinterpret_cast<const double2*>(a.src + (size_t)jj * a.sld);
#pragma unroll
                for (int q = 0; q < NQ; ++q) {
                    const double2 d2 = __ldg(r + q);
                    v[u][2 * q] = d2.x;
                    v[u][2 * q + 1] = d2.y;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const bool in = j + u * TS < e;
#pragma unroll
                for (int m = 0; m < M; ++m) v[u][3 + m] = in ? v[u][3 + m] : 0.0;
                {
                    const double dx = xa - v[u][0], dy = ya - v[u][1], dz = za - v[u][2];
                    K::pair(dx, dy, dz, in ? fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))) : 1.0, &v[u][3], accA, a.kp);
                }
                {
                    const double dx = xb - v[u][0], dy = yb - v[u][1], dz = zb - v[u][2];
                    K::pair(dx, dy, dz, in ? fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))) : 1.0, &v[u][3], accB, a.kp);
                }
            }
        }
    }
}

template <int V, int U>
__global__ void __launch_bounds__(kWarps * 32, 4) k_near_var(EvalArgs a, const int2* leaves, int nleaf, int ncalls) {
    __shared__ __align__(16) double sm[512 * 6];
    for (int i = threadIdx.x; i < 512 * 6; i += blockDim.x) sm[i] = a.src[i];
    __syncthreads();
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int gw = blockIdx.x * kWarps + wl;
    const int la = (lane >> 4) * 16, lb = la + kGroup;
    const double xa = 0.1 + 0.001 * (la / 8), ya = -0.2, za = 0.3, xb = 0.1 + 0.001 * (lb / 8), yb = -0.2, zb = 0.3;
    double accA[6] = {0, 0, 0, 0, 0, 0}, accB[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int2 L = leaves[(int)(((long long)gw * 7919 + i) % nleaf)];
        if (V == 16) near_field_tb<0, false>(xa, ya, za, -1, xb, yb, zb, -1, L.x, L.y, lane & 15, 16, a, accA, accB);
        else near_var<V, U>(xa, ya, za, xb, yb, zb, L.x, L.y, lane & 15, a, sm, accA, accB);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < 6; ++c) t += accA[c] + accB[c];
    if (t == 1.2345) a.out[0] = t;
}


// near_leaf2: target pairs with the lane's OWN target accumulated straight into acc and only
// the partner group's target (lane ^ 8) into a per-leaf oth[], folded by one shuffle at the end
template <int U>
__device__ __forceinline__ void near_leaf2(double x, double y, double z, int b, int e, int lane, const EvalArgs& a,
                                           double* acc) {
    using K = EvalKern<0>;
    constexpr int M = 3, NQ = 3, TS = 16;
    const double xb = __shfl_xor_sync(0xffffffffu, x, kGroup), yb = __shfl_xor_sync(0xffffffffu, y, kGroup),
                 zb = __shfl_xor_sync(0xffffffffu, z, kGroup);
    double oth[6] = {0, 0, 0, 0, 0, 0};
    int j = b + (lane & 15);
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
            {
                const double dx = x - v[u][0], dy = y - v[u][1], dz = z - v[u][2];
                K::pair(dx, dy, dz, fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))), &v[u][3], acc, a.kp);
            }
            {
                const double dx = xb - v[u][0], dy = yb - v[u][1], dz = zb - v[u][2];
                K::pair(dx, dy, dz, fma(dx, dx, fma(dy, dy, fma(dz, dz, a.kp.e2))), &v[u][3], oth, a.kp);
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
        const double dxa = x - v[0], dya = y - v[1], dza = z - v[2];
        const double dxb = xb - v[0], dyb = yb - v[1], dzb = zb - v[2];
        K::pair(dxa, dya, dza, fma(dxa, dxa, fma(dya, dya, fma(dza, dza, a.kp.e2))), &v[3], acc, a.kp);
        K::pair(dxb, dyb, dzb, fma(dxb, dxb, fma(dyb, dyb, fma(dzb, dzb, a.kp.e2))), &v[3], oth, a.kp);
    }
#pragma unroll
    for (int c = 0; c < 6; ++c) acc[c] += __shfl_xor_sync(0xffffffffu, oth[c], kGroup);
}

template <int U>
__global__ void __launch_bounds__(kWarps * 32, 4) k_near2(EvalArgs a, const int2* leaves, int nleaf, int ncalls) {
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int ti = lane / kGroup;
    const int gw = blockIdx.x * kWarps + wl;
    const double x = 0.1 + 0.001 * ti, y = -0.2 + 0.0007 * ti, z = 0.3 - 0.0003 * ti;
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int i = 0; i < ncalls; ++i) {
        const int2 L = leaves[(int)(((long long)gw * 7919 + i) % nleaf)];
        near_leaf2<U>(x, y, z, L.x, L.y, lane, a, acc);
    }
    double t = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5];
    if (t == 1.2345) a.out[0] = t;
}

void run(int sms, int clk_khz) {
    const int N = 1000000, sld = 6;
    std::vector<double> hs((size_t)N * sld);
    srand(3);
    for (int j = 0; j < N; ++j) {
        for (int q = 0; q < 3; ++q) hs[(size_t)j * sld + q] = -1.0 + 2.0 * rand() / RAND_MAX;
        for (int q = 3; q < 6; ++q) hs[(size_t)j * sld + q] = -1.0 + 2.0 * rand() / RAND_MAX;
    }
    const int nleaf = 4096;
    std::vector<int2> hl(nleaf);
    long long tot = 0;
    for (auto& l : hl) {
        const int len = 250 + rand() % 1751;
        l.x = rand() % (N - len);
        l.y = l.x + len;
        tot += len;
    }
    double *s, *o;
    int2* lv;
    cudaMalloc(&s, hs.size() * 8);
    cudaMalloc(&o, 8);
    cudaMalloc(&lv, nleaf * sizeof(int2));
    cudaMemcpy(s, hs.data(), hs.size() * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(lv, hl.data(), nleaf * sizeof(int2), cudaMemcpyHostToDevice);
    EvalArgs a{};
    a.src = s;
    a.sld = sld;
    a.out = o;
    a.N = N;
    a.self_omit = 0;
    a.kp = make_kparams(0.01);
    const int ctas = sms * 4 * 4, ncalls = 32;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[5] = {"near_leaf (prod)", "var 0 U4 no tail", "prod near_field_tb", "var 4 U4 serial tail", "near_leaf2 U4 own->acc"};
    for (int rep = 0; rep < 15; ++rep) {
        const int V = rep % 5;
        cudaEventRecord(e0);
        if (V == 0) k_near_probe<0><<<ctas, kWarps * 32>>>(a, lv, nleaf, ncalls);
        else if (V == 1) k_near_var<0, 4><<<ctas, kWarps * 32>>>(a, lv, nleaf, ncalls);
        else if (V == 2) k_near_var<16, 4><<<ctas, kWarps * 32>>>(a, lv, nleaf, ncalls);
        else if (V == 3) k_near_var<4, 4><<<ctas, kWarps * 32>>>(a, lv, nleaf, ncalls);
        else k_near2<4><<<ctas, kWarps * 32>>>(a, lv, nleaf, ncalls);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        double pairs = 0;
        for (int w = 0; w < ctas * kWarps; ++w)
            for (int i = 0; i < ncalls; ++i) {
                const int2 L = hl[(int)(((long long)w * 7919 + i) % nleaf)];
                pairs += 4.0 * (L.y - L.x);
            }
        const double rate = pairs / (ms * 1e-3);
        if (rep >= 5)
            printf("%-22s %.3f ms, %.3f pairs/clk/SM, %.2f TFLOP/s = %.1f%% of %.2f (err %s)\n", names[V],
                   ms, rate / (sms * clk_khz * 1e3), rate * 32e-12, 100.0 * rate * 32 / (sms * 128.0 * clk_khz * 1e3),
                   sms * 128.0 * clk_khz * 1e-9, cudaGetErrorString(cudaGetLastError()));
    }
}

}  // namespace
}  // namespace kitc

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    kitc::run(sms, 1965000);
    return 0;
}
