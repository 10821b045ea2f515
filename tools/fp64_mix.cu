// Throughput of DFMA / DMUL / DADD / MUFU.RSQ64H and mixes on B200 (per SM per clock).
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double seed(double s) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(s)); return y; }
template <int MODE>
__global__ void k(double* out, int iters) {
  double a[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) a[c] = 1.0 + threadIdx.x * 1e-9 + c * 1e-3;
  const double m = 0.99999, b = 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (MODE == 0) a[c] = fma(a[c], m, b);
      if (MODE == 1) a[c] = a[c] * m;
      if (MODE == 2) a[c] = a[c] + b;
      if (MODE == 3) a[c] = seed(a[c]) + 1.0;  // 1 MUFU + 1 DADD
      if (MODE == 4) { double y = seed(a[c]); a[c] = fma(fma(fma(fma(y, m, b), m, b), m, b), m, 1.0); } // 1 MUFU + 4 DFMA
      if (MODE == 5) { double y = a[c]; a[c] = fma(fma(fma(fma(y, m, b), m, b), m, b), m, 1.0); }  // 4 DFMA (same dep shape)
      if (MODE == 6) { double y = (double)rsqrtf((float)a[c]); a[c] = fma(fma(fma(fma(y, m, b), m, b), m, b), m, 1.0); } // F2F+MUFU.RSQ+F2F + 4 DFMA
    }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c];
  if (s == 1.2345) out[0] = s;
}
template <int MODE> void run(const char* nm, double ops_per, double* o, int sms, int clk) {
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<sms * 8, 256>>>(o, iters);
  cudaEventRecord(e0); k<MODE><<<sms * 8, 256>>>(o, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double per = (double)iters * 8 * 256 * sms * 8 / (ms * 1e-3) / sms / (clk * 1e3);
  printf("%-28s %.2f items/clk/SM  (%.1f FP64-pipe ops/clk/SM if %.0f ops/item)\n", nm, per, per * ops_per, ops_per);
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* o; cudaMalloc(&o, 8);
  run<0>("DFMA", 1, o, sms, clk); run<1>("DMUL", 1, o, sms, clk); run<2>("DADD", 1, o, sms, clk);
  run<3>("MUFU.RSQ64H + DADD", 1, o, sms, clk); run<4>("MUFU.RSQ64H + 4 DFMA", 4, o, sms, clk); run<5>("4 DFMA", 4, o, sms, clk);
  run<6>("F2F+MUFU.RSQ(f32)+F2F + 4 DFMA", 4, o, sms, clk);
  return 0;
}
