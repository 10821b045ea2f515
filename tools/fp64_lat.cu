// FP64 pipe: throughput vs independent chains per thread (ILP) and warps per SM (TLP).
#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void k(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 1.2345) out[0] = s;
}
template <int CH> void run(int warps_per_sm, double* o, int sms, int clk) {
  int threads = 32 * warps_per_sm; if (threads > 1024) threads = 1024;
  int blocks = sms * (32 * warps_per_sm / threads);
  int iters = 20000 / CH * 8;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<CH><<<blocks, threads>>>(o, iters, 0.9999, 1e-7);
  cudaEventRecord(e0); k<CH><<<blocks, threads>>>(o, iters, 0.9999, 1e-7); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fma_per_clk_sm = (double)iters * CH * threads * blocks / (ms * 1e-3) / sms / (clk * 1e3);
  printf("chains %d warps/SM %2d : %.1f DFMA/clk/SM\n", CH, warps_per_sm, fma_per_clk_sm);
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* o; cudaMalloc(&o, 8);
  for (int w : {4, 8, 16, 24, 32}) { run<1>(w, o, sms, clk); run<2>(w, o, sms, clk); run<4>(w, o, sms, clk); run<8>(w, o, sms, clk); }
  return 0;
}
