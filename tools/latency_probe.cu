// Dependent-chain latency probe (cycles) for the instructions on the tracker's critical path:
// DFMA, DMUL, LDS.128 (shared), SHFL (32-bit), REDUX (redux.sync max), MUFU.RCP64H.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void probe(double *out, long long *cyc, int iters) {
  __shared__ double2 sm[64];
  const int lane = threadIdx.x;
  if (lane < 64) sm[lane] = make_double2(lane * 0.5, 1.0);
  __syncwarp();
  double a = 1.0 + lane * 1e-9, b = 0.999999;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) a = fma(a, b, 1e-7);
  long long t1 = clock64();
  for (int i = 0; i < iters; ++i) a = a * b;
  long long t2 = clock64();
  int idx = lane & 7;
  for (int i = 0; i < iters; ++i) { double2 v = sm[idx]; idx = ((int)v.y + idx) & 7; }
  long long t3 = clock64();
  unsigned u = lane;
  for (int i = 0; i < iters; ++i) u = __shfl_xor_sync(0xffffffff, u, 1) + 1;
  long long t4 = clock64();
  unsigned w = lane;
  for (int i = 0; i < iters; ++i) w = __reduce_max_sync(0xffffffff, w) - lane;
  long long t5 = clock64();
  double r = 1.5 + lane;
  for (int i = 0; i < iters; ++i) { double q; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(q) : "d"(r)); r = q + 1.0; }
  long long t6 = clock64();
  if (lane == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4; cyc[5] = t6 - t5;
  }
  out[lane] = a + idx + u + w + r;
}
int main() {
  double *o; long long *c; cudaMalloc(&o, 64 * 8); cudaMalloc(&c, 8 * 8);
  const int iters = 4096;
  probe<<<1, 32>>>(o, c, iters);
  probe<<<1, 32>>>(o, c, iters);
  long long h[6]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  const char *n[6] = {"DFMA", "DMUL", "LDS.128", "SHFL", "REDUX", "MUFU.RCP64H(+DADD)"};
  printf("{");
  for (int i = 0; i < 6; ++i) printf("%s\"%s\": %.2f", i ? ", " : "", n[i], (double)h[i] / iters);
  printf("}\n");
  return 0;
}
