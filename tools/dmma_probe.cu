// Is the FP64 tensor path (DMMA, mma.sync m8n8k4 f64) a separate unit from the
// DFMA pipe on B200?  Throughput of DMMA alone, DFMA alone, and both interleaved.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double* d, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1]) : "d"(a), "d"(b));
}
template <int NM, int NF>
__global__ void k(double* out, int iters) {
  double acc[4][2];
  double f[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) { acc[i][0] = threadIdx.x; acc[i][1] = 1; }
#pragma unroll
  for (int i = 0; i < 8; ++i) f[i] = 1.0 + i * 1e-3 + threadIdx.x * 1e-9;
  double a = 1e-3 * threadIdx.x, b = 0.5;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < NM; ++r) dmma(acc[r % 4], a, b);
#pragma unroll
    for (int r = 0; r < NF; ++r) f[r % 8] = fma(f[r % 8], 0.999999, 1e-9);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) s += acc[i][0] + acc[i][1];
#pragma unroll
  for (int i = 0; i < 8; ++i) s += f[i];
  if (s == 1.2345) out[0] = s;
}
template <int NM, int NF> void run(double* o, int sms, int clk) {
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<NM, NF><<<sms * 4, 256>>>(o, iters);
  cudaEventRecord(e0); k<NM, NF><<<sms * 4, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double warps = sms * 4 * 8.0, cyc = ms * 1e-3 * clk * 1e3;
  double dmma_flops = 2.0 * 8 * 8 * 4 * NM * iters * warps;  // per warp-level mma: 8x8x4 MACs
  double dfma_flops = 2.0 * 32 * NF * iters * warps;
  printf("DMMA/iter %2d DFMA/iter %2d: %.3f ms  DMMA %.1f TFLOP/s  DFMA %.1f TFLOP/s  total %.1f TFLOP/s\n", NM, NF, ms,
         dmma_flops / ms / 1e9, dfma_flops / ms / 1e9, (dmma_flops + dfma_flops) / ms / 1e9);
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* o; cudaMalloc(&o, 8);
  run<8, 0>(o, sms, clk); run<0, 16>(o, sms, clk); run<8, 16>(o, sms, clk); run<4, 16>(o, sms, clk); run<8, 8>(o, sms, clk);
  return 0;
}
