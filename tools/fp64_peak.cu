// FP64 DFMA throughput microbenchmark (SURVEY.md §8(d) "FP64 peak"): 8 independent
// DFMA chains per thread, full occupancy, timed with CUDA events. Prints one JSON line.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void dfma_loop(double* out, long iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; i++) r[i] = threadIdx.x * 1e-9 + i;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) r[i] = fma(r[i], a, b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += r[i];
  if (s == 12345.678) out[0] = s;
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* d; cudaMalloc(&d, 8);
  int threads = 512, blocks = p.multiProcessorCount * 4;
  long iters = 200000;
  dfma_loop<<<blocks, threads>>>(d, 1000, 0.999999, 1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * iters * (double)threads * blocks;
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp64_tflops\": %.3f, \"ms\": %.3f, \"sms\": %d, \"max_clock_mhz\": %.0f, \"theoretical_at_max_clock_tflops\": %.3f}\n",
         flops / best / 1e9, best, p.multiProcessorCount, clk / 1e3,
         p.multiProcessorCount * 64 * 2 * (clk * 1e3) / 1e12);
  return 0;
}
