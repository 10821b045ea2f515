// Peak Stokeslet pair throughput on B200 (no memory traffic): KC independent
// pairs per step, the production pair math (pair.cuh).  Reports pairs/clk/SM
// and the algorithmic TFLOP/s (32 flops/pair).
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1902_02250_b200/csrc/pair.cuh"
using namespace kitc;
template <int KC, int BLK>
__global__ void __launch_bounds__(BLK) k(double* out, int iters, KParams kp) {
  double x = 0.1 + threadIdx.x * 1e-6, y = 0.2, z = 0.3;
  double acc[KC][3] = {};
  double f[KC][3];
#pragma unroll
  for (int i = 0; i < KC; ++i) { f[i][0] = 0.5 + i; f[i][1] = -0.25; f[i][2] = 0.125 * i; }
  double sz = 0.01;
  for (int it = 0; it < iters; ++it) {
    double dx[KC], dy[KC], dz[KC], s[KC];
#pragma unroll
    for (int i = 0; i < KC; ++i) { dx[i] = x; dy[i] = y; dz[i] = z - sz * i; s[i] = fma(dz[i], dz[i], fma(dy[i], dy[i], fma(dx[i], dx[i], kp.e2))); }
    pairs<0, KC>(dx, dy, dz, s, f, acc, kp);
    x += 1e-7;
  }
  double t = 0;
#pragma unroll
  for (int i = 0; i < KC; ++i) t += acc[i][0] + acc[i][1] + acc[i][2];
  if (t == 1.2345) out[0] = t;
}
template <int KC, int BLK> void run(int bps, double* o, int sms, int clk) {
  int iters = 2000;
  KParams kp = make_kparams(0.01);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<KC, BLK><<<sms * bps, BLK>>>(o, iters, kp);
  cudaEventRecord(e0); k<KC, BLK><<<sms * bps, BLK>>>(o, iters, kp); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pairs = (double)iters * KC * BLK * sms * bps;
  printf("KC %d warps/SM %2d: %.2f pairs/clk/SM, %.2f TFLOP/s algorithmic\n", KC, BLK / 32 * bps, pairs / (ms * 1e-3) / sms / (clk * 1e3), 32 * pairs / ms / 1e9);
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* o; cudaMalloc(&o, 8);
  run<1, 256>(2, o, sms, clk); run<1, 256>(4, o, sms, clk);
  run<2, 256>(2, o, sms, clk); run<2, 256>(4, o, sms, clk);
  run<3, 256>(2, o, sms, clk); run<3, 256>(4, o, sms, clk);
  run<4, 256>(2, o, sms, clk); run<4, 256>(3, o, sms, clk);
  run<6, 256>(2, o, sms, clk); run<8, 256>(1, o, sms, clk); run<8, 256>(2, o, sms, clk);
  return 0;
}
