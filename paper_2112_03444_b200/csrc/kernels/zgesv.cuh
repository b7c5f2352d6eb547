// zgesv.cuh -- standalone batched fused LU + solve kernel template (instantiated per N).
#pragma once
#include "tracker.cuh"

namespace hcb {

// ------------------------------------------------------------------------------------------
// Standalone batched fused LU + solve (Fig. 3): one
// sub-warp of L lanes per system, row r of [A | b] in lane r's registers, the same lu_rows as the
// tracker.  4 warps per CTA, grid-stride over systems.
// ------------------------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(128) batched_zgesv_kernel(const double2 *__restrict__ A, const double2 *__restrict__ b,
                                                            double2 *__restrict__ x, int32_t *__restrict__ info,
                                                            long long batch, double pivot_rel) {
  constexpr int L = (N <= 1) ? 1 : (N <= 2) ? 2 : (N <= 4) ? 4 : (N <= 8) ? 8 : (N <= 16) ? 16 : 32;
  constexpr int TPW = 32 / L;
  __shared__ double2 prow_s[4 * TPW][2 * (N + 1)];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / L, r = lane % L;
  double2 *prow = prow_s[warp * TPW + seg];
  const long long slots = (long long)gridDim.x * 4 * TPW;
  for (long long base = ((long long)blockIdx.x * 4 + warp) * TPW; base < batch; base += slots) {
    const long long k = base + seg;   // warp-uniform loop; idle segments solve a dummy copy
    const long long kk = k < batch ? k : batch - 1;
    double2 a[N + 1];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = (r < N) ? A[((size_t)kk * N + r) * N + j] : make_double2(0.0, 0.0);
    a[N] = (r < N) ? b[(size_t)kk * N + r] : make_double2(0.0, 0.0);
    double2 y;
    double amax = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) amax = fmax(amax, abs2(a[j]));
    const bool ok = lu_rows<N, L>(a, r, seg, prow, pivot_rel, amax, y);
    if (k < batch) {
      if (r < N) x[(size_t)k * N + r] = y;
      if (r == 0) info[k] = ok ? 0 : 1;
    }
  }
}

template <int N>
cudaError_t launch_zgesv_n(int64_t batch, const double2 *A, const double2 *b, double2 *x, int32_t *info,
                                  double pivot_rel, cudaStream_t s) {
  constexpr int L = (N <= 1) ? 1 : (N <= 2) ? 2 : (N <= 4) ? 4 : (N <= 8) ? 8 : (N <= 16) ? 16 : 32;
  constexpr int TPW = 32 / L;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_zgesv_kernel<N>, 128, 0);
  long long need = (batch + 4 * TPW - 1) / (4 * TPW);
  long long ctas = (long long)sms * (per_sm > 0 ? per_sm : 1);
  if (need < ctas) ctas = need;
  if (ctas < 1) ctas = 1;
  batched_zgesv_kernel<N><<<(unsigned)ctas, 128, 0, s>>>(A, b, x, info, batch, pivot_rel);
  return cudaGetLastError();
}

}  // namespace hcb
