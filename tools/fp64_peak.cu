// FP64 DFMA peak probe for the roofline denominator.
// Independent DFMA chains per thread; grid = SMs x resident CTAs.
#include <cstdio>
#include <cuda_runtime.h>
template <int CHAINS>
__global__ void dfma_loop(double* out, long iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (long i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}
#ifndef KITC_PROBE_LIB
int main(int argc, char** argv) {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("gpu %s sms %d clock_khz %d cc %d.%d\n", p.name, sms, clk, p.major, p.minor);
  double* out; cudaMalloc(&out, 8);
  const int threads = 256; const int CH = 8;
  for (int blocksPerSM : {4, 8}) {
    for (double seconds : {0.2, 4.0}) {
      long iters = 1 << 14;
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      // calibrate
      dfma_loop<CH><<<sms * blocksPerSM, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e0);
      dfma_loop<CH><<<sms * blocksPerSM, threads>>>(out, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      long it2 = (long)(iters * (seconds * 1e3 / ms));
      cudaEventRecord(e0);
      dfma_loop<CH><<<sms * blocksPerSM, threads>>>(out, it2, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * CH * (double)it2 * threads * sms * blocksPerSM;
      printf("blocks/SM %d target %.1fs: %.3f ms, %.2f TFLOP/s (fp64 fma), per SM per clk at max clock: %.1f FMA\n",
             blocksPerSM, seconds, ms, flops / ms / 1e9, flops / 2 / (ms * 1e-3) / sms / (clk * 1e3));
    }
  }
  cudaError_t e = cudaGetLastError(); printf("err %s\n", cudaGetErrorString(e));
  return 0;
}
#endif

// Library form for bench.py (built by __graft_entry__.build() into
// tools/libfp64_peak.so): the DFMA rate of the box, measured untimed before the
// bench's timed region and reported beside the derived roofline peak.
extern "C" int kitc_probe_dfma_tflops(double seconds, double* tflops, double* fma_per_sm_clk) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceProp p;
  if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return -1;
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  const int sms = p.multiProcessorCount, threads = 256, bps = 4, CH = 8;
  double* out = nullptr;
  if (cudaMalloc(&out, 8) != cudaSuccess) return -1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  long iters = 1 << 14;
  dfma_loop<CH><<<sms * bps, threads>>>(out, iters, 0.999999, 1e-7);  // warm-up + calibration
  cudaEventRecord(e0);
  dfma_loop<CH><<<sms * bps, threads>>>(out, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, e0, e1);
  const long it2 = (long)(iters * (seconds * 1e3 / ms));
  cudaEventRecord(e0);
  dfma_loop<CH><<<sms * bps, threads>>>(out, it2, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * CH * (double)it2 * threads * sms * bps;
  *tflops = flops / (ms * 1e-3) / 1e12;
  if (fma_per_sm_clk) *fma_per_sm_clk = flops / 2 / (ms * 1e-3) / sms / (clk * 1e3);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
