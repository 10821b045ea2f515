// Does DFMA throughput depend on the number of distinct register operands
// (register-file read bandwidth)?  8 independent chains per thread.
#include <cstdio>
#include <cuda_runtime.h>
template <int MODE>
__global__ void k(double* out, int iters, double c1, double c2) {
  double a[8], b[8], d[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) { a[c] = 1.0 + threadIdx.x * 1e-9 + c; b[c] = 0.9999 + c * 1e-7; d[c] = 1e-9 * (c + 1); }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      if (MODE == 0) a[c] = fma(a[c], c1, c2);            // 1 register operand (+ uniform/const)
      if (MODE == 1) a[c] = fma(a[c], b[c], c2);          // 2 distinct registers
      if (MODE == 2) a[c] = fma(a[c], b[c], d[c]);        // 3 distinct registers
      if (MODE == 3) a[c] = fma(b[c], d[c], a[c]);        // 3 distinct, accumulator last
      if (MODE == 4) a[c] = a[c] * b[c];                  // DMUL 2 regs
    }
#pragma unroll
    for (int c = 0; c < 8; ++c) { asm volatile("" : "+d"(b[c]), "+d"(d[c])); }
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += a[c] + b[c] + d[c];
  if (s == 1.2345) out[0] = s;
}
template <int MODE> void run(const char* nm, double* o, int sms, int clk) {
  int iters = 4000;
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<MODE><<<sms * 8, 256>>>(o, iters, 0.9999, 1e-9);
  cudaEventRecord(e0); k<MODE><<<sms * 8, 256>>>(o, iters, 0.9999, 1e-9); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-40s %.1f ops/clk/SM\n", nm, (double)iters * 8 * 256 * sms * 8 / (ms * 1e-3) / sms / (clk * 1e3));
}
int main() {
  int sms, clk; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0); cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* o; cudaMalloc(&o, 8);
  run<0>("DFMA a = a*c1 + c2", o, sms, clk); run<1>("DFMA a = a*b + c2", o, sms, clk);
  run<2>("DFMA a = a*b + d", o, sms, clk); run<3>("DFMA a = b*d + a", o, sms, clk); run<4>("DMUL a = a*b", o, sms, clk);
  return 0;
}
