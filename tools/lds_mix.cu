// FP64 issue cost of shared loads (tuning probe): 8 independent DFMA chains per thread,
// 16 DFMA per iteration, plus L shared loads of W bytes per lane whose values are the
// FMA addends (no extra FP64 instructions).  Prints DFMA/clk/SM per (W, L).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/lds_mix.cu -o tools/lds_mix
#include <cstdio>
#include <cuda_runtime.h>

template <int W, int L, int A>
__global__ void __launch_bounds__(128, 4) k(double* out, int iters) {
    __shared__ __align__(16) double sm[1024];
    for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = 1e-3 * (i % 37);
    __syncthreads();
    double c[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) c[i] = 1.0 + threadIdx.x * 1e-6 + i;
    const double a = 0.999999;
    // A = 0: contiguous (W bytes per lane), 1: each quarter-warp reads the same 128 B, 2: all lanes one address
    const int lane = threadIdx.x & 31;
    const int off = A == 0 ? lane * (W / 8) : A == 1 ? (lane & 7) * (W / 8) : 0;
    for (int it = 0; it < iters; ++it) {
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = 1e-9;
#pragma unroll
        for (int l = 0; l < L; ++l) {
            const int o = (off + l * 64 + it * 2) & 1023;
            if (W == 16) {
                const double2 t = *reinterpret_cast<const double2*>(sm + o);
                v[(2 * l) & 7] = t.x;
                v[(2 * l + 1) & 7] = t.y;
            } else if (W == 8) {
                v[l & 7] = sm[o];
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, v[i]);
#pragma unroll
        for (int i = 0; i < 8; ++i) c[i] = fma(c[i], a, 1e-9);
    }
    double t = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) t += c[i];
    if (t == 1.2345) out[0] = t;
}

template <int W, int L, int A>
void run(int sms, double* o) {
    const int iters = 20000, ctas = sms * 4 * 4;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k<W, L, A><<<ctas, 128>>>(o, iters);
    cudaEventRecord(e0);
    k<W, L, A><<<ctas, 128>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double dfma = (double)ctas * 128 * iters * 16;
    printf("W %2d A %d L %d (%.3f loads per DFMA): %.1f DFMA/clk/SM at 1965 MHz\n", W, A, L, L / 16.0,
           dfma / (ms * 1e-3) / (sms * 1965e6));
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* o;
    cudaMalloc(&o, 8);
    run<16, 0, 0>(sms, o);
    run<16, 1, 0>(sms, o); run<16, 2, 0>(sms, o); run<16, 4, 0>(sms, o);
    run<16, 1, 1>(sms, o); run<16, 2, 1>(sms, o); run<16, 4, 1>(sms, o);
    run<16, 1, 2>(sms, o); run<16, 2, 2>(sms, o); run<16, 4, 2>(sms, o);
    run<8, 2, 0>(sms, o); run<8, 4, 0>(sms, o); run<8, 8, 0>(sms, o);
    run<8, 2, 2>(sms, o); run<8, 4, 2>(sms, o); run<8, 8, 2>(sms, o);
    return 0;
}
