// zgesv.cuh -- standalone batched fused LU + solve kernel template (instantiated per N).
#pragma once
#include "tracker.cuh"

namespace hcb {

// ------------------------------------------------------------------------------------------
// Standalone batched fused LU + solve (Fig. 3): one
// sub-warp of L lanes per system, row r of [A | b] in lane r's registers, the same lu_rows as the
// tracker.  4 warps per CTA, grid-stride over systems.  A warp's TPW systems are contiguous in
// memory: the warp loads them with consecutive lanes on consecutive elements (coalesced) into a
// shared staging tile with an odd row stride (conflict-free row reads), then each lane takes its row.
// ------------------------------------------------------------------------------------------
template <int N>
struct ZgesvShape {
  static constexpr int L = (N <= 1) ? 1 : (N <= 2) ? 2 : (N <= 4) ? 4 : (N <= 8) ? 8 : (N <= 16) ? 16 : 32;
  static constexpr int TPW = 32 / L;
  static constexpr int SP = (N % 2) ? N : N + 1;   // staging row stride (odd: 16-byte rows conflict-free)
  static constexpr int STAGE = TPW * N * SP;       // double2 per warp
  static constexpr int PROW = TPW * 2 * (N + 1);   // double2 per warp
  static constexpr size_t SMEM = (size_t)4 * (STAGE + PROW) * sizeof(double2);
};

template <int N>
__global__ void __launch_bounds__(128) batched_zgesv_kernel(const double2 *__restrict__ A, const double2 *__restrict__ b,
                                                            double2 *__restrict__ x, int32_t *__restrict__ info,
                                                            long long batch, double pivot_rel) {
  using Z = ZgesvShape<N>;
  constexpr int L = Z::L, TPW = Z::TPW, SP = Z::SP;
  extern __shared__ __align__(16) double2 zsmem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / L, r = lane % L;
  double2 *stage = zsmem + warp * (Z::STAGE + Z::PROW);
  double2 *prow = stage + Z::STAGE + seg * 2 * (N + 1);
  const long long slots = (long long)gridDim.x * 4 * TPW;
  const long long total = batch * N * N;
  for (long long base = ((long long)blockIdx.x * 4 + warp) * TPW; base < batch; base += slots) {
    // ---- coalesced load of the warp's TPW systems into the staging tile ----
    const long long off = base * N * N;
#pragma unroll 4
    for (int i = lane; i < TPW * N * N; i += 32) {
      const int sys = i / (N * N), row = (i / N) % N, col = i % N;
      stage[(sys * N + row) * SP + col] = (off + i < total) ? __ldg(&A[off + i]) : make_double2(0.0, 0.0);
    }
    __syncwarp();
    const long long k = base + seg;   // warp-uniform loop; idle segments solve a dummy (zero) system
    const bool valid = k < batch;
    double2 a[N + 1];
#pragma unroll
    for (int j = 0; j < N; ++j) a[j] = (r < N) ? stage[(seg * N + r) * SP + j] : make_double2(0.0, 0.0);
    a[N] = (r < N && valid) ? __ldg(&b[(size_t)k * N + r]) : make_double2(0.0, 0.0);
    __syncwarp();   // the staging tile is reused by the next iteration's load
    double2 y;
    double amax = 0.0;
#pragma unroll
    for (int j = 0; j < N; ++j) amax = fmax(amax, abs2(a[j]));
    const bool ok = lu_rows<N, L>(a, r, seg, prow, stage + seg * N * SP, pivot_rel, amax, y);   // (the staging tile is dead here)
    if (valid) {
      if (r < N) x[(size_t)k * N + r] = y;
      if (r == 0) info[k] = ok ? 0 : 1;
    }
  }
}

template <int N>
cudaError_t launch_zgesv_n(int64_t batch, const double2 *A, const double2 *b, double2 *x, int32_t *info,
                                  double pivot_rel, cudaStream_t s) {
  using Z = ZgesvShape<N>;
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute((const void *)batched_zgesv_kernel<N>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Z::SMEM);
  if (e != cudaSuccess) return e;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, batched_zgesv_kernel<N>, 128, Z::SMEM);
  long long need = (batch + 4 * Z::TPW - 1) / (4 * Z::TPW);
  long long ctas = (long long)sms * (per_sm > 0 ? per_sm : 1);
  if (need < ctas) ctas = need;
  if (ctas < 1) ctas = 1;
  batched_zgesv_kernel<N><<<(unsigned)ctas, 128, Z::SMEM, s>>>(A, b, x, info, batch, pivot_rel);
  return cudaGetLastError();
}

}  // namespace hcb
