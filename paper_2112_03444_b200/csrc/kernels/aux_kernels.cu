// aux_kernels.cu -- coefficient prologue, standalone batched fused LU solve, FP64 probe (sm_100a).
#include <cstdint>
#include <cuda_runtime.h>

#include "tracker.cuh"

namespace hcb {

// ------------------------------------------------------------------------------------------
// Coefficient prologue.  For instance b, c_j(p(t)) with
// p(t) = (1-t) p0 + t p1[b] (reading R3) is a polynomial in t of degree <= D:
// each coefficient monomial w * prod_m p_{f_m}(t) is a product of linear factors
// (p0_q + t (p1_q - p0_q)), expanded here once per instance.  One thread per (b, j);
// output coef_t[b][d][j] so the tracker's Horner loads are coalesced over j.
// ------------------------------------------------------------------------------------------
__global__ void coef_prologue_kernel(const PrologueArgs A) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= A.B * A.ncoef) return;
  const long long b = idx / A.ncoef;
  const int j = (int)(idx % A.ncoef);
  const double2 *p1 = A.p1 + (size_t)b * A.P;
  double2 res[MAX_COEF_DEG + 1];
#pragma unroll
  for (int d = 0; d <= MAX_COEF_DEG; ++d) res[d] = make_double2(0.0, 0.0);
  for (int m = A.coef_mono_ptr[j]; m < A.coef_mono_ptr[j + 1]; ++m) {
    const CoefMono mo = A.mono[m];
    double2 poly[MAX_COEF_DEG + 1];
#pragma unroll
    for (int d = 0; d <= MAX_COEF_DEG; ++d) poly[d] = make_double2(0.0, 0.0);
    poly[0] = make_double2(mo.wre, mo.wim);
    for (int f = 0; f < mo.deg; ++f) {
      const int q = mo.fac[f];
      const double2 a0 = A.p0[q];
      const double2 d1 = make_double2(p1[q].x - a0.x, p1[q].y - a0.y);
      // poly *= (a0 + t d1): new[d] = poly[d] a0 + poly[d-1] d1 (high to low, in place)
#pragma unroll
      for (int d = MAX_COEF_DEG; d >= 1; --d) {
        const double2 u = cmul(poly[d], a0), v = cmul(poly[d - 1], d1);
        poly[d] = make_double2(u.x + v.x, u.y + v.y);
      }
      poly[0] = cmul(poly[0], a0);
    }
#pragma unroll
    for (int d = 0; d <= MAX_COEF_DEG; ++d) res[d] = make_double2(res[d].x + poly[d].x, res[d].y + poly[d].y);
  }
  for (int d = 0; d <= A.D; ++d) A.coef_t[((size_t)b * (A.D + 1) + d) * A.ncoef + j] = res[d];
}

cudaError_t launch_prologue(const PrologueArgs &A, cudaStream_t stream) {
  const long long n = A.B * A.ncoef;
  if (n == 0) return cudaSuccess;
  const int threads = 256;
  coef_prologue_kernel<<<(unsigned)((n + threads - 1) / threads), threads, 0, stream>>>(A);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------
// FP64 DFMA throughput probe: 8 independent chains per thread.
// ------------------------------------------------------------------------------------------
__global__ void fp64_probe_kernel(double *out, long iters, double a, double c) {
  double r[8];
#pragma unroll
  for (int i = 0; i < 8; i++) r[i] = threadIdx.x * 1e-9 + i;
  for (long it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++) r[i] = fma(r[i], a, c);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++) s += r[i];
  if (s == 12345.678) out[0] = s;
}

cudaError_t run_fp64_probe(int device, double *tflops) {
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return e;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double *d = nullptr;
  if ((e = cudaMalloc(&d, 8)) != cudaSuccess) return e;
  const int threads = 512, blocks = sms * 4;
  const long iters = 200000;
  fp64_probe_kernel<<<blocks, threads>>>(d, 2000, 0.999999, 1e-7);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; rep++) {
    cudaEventRecord(e0);
    fp64_probe_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  e = cudaGetLastError();
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(d);
  *tflops = 2.0 * 8 * iters * (double)threads * blocks / (best * 1e-3) / 1e12;
  return e;
}

}  // namespace hcb
