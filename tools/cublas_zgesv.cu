// cublas_zgesv.cu -- the library baseline of the Fig. 3 re-run (SURVEY.md
// N1): cuBLAS batched LU (cublasZgetrfBatched) + triangular solves (cublasZgetrsBatched) called
// directly, timed with CUDA events.  Benchmark tooling only (scripts/bench_zgesv.py loads it with
// ctypes); the product path never links cuBLAS.
//
// Layout: our matrices are row-major [batch][n][n]; cuBLAS is column-major, so the buffer is A^T:
// getrf factors A^T and getrs with CUBLAS_OP_T solves (A^T)^T x = A x = b.
//
// extern "C" int cublas_zgesv_time(int n, long long batch, const void *A, const void *b, void *x,
//                                  int reps, float *ms_median, int *info_nonzero)
//   A, b: device buffers (row-major), x: device [batch][n] output, both left untouched except x.
//   Each repetition copies A and b into work buffers (outside the timed region), then times
//   getrf + getrs between CUDA events.  Returns 0 on success.
#include <algorithm>
#include <cstdio>
#include <vector>

#include <cublas_v2.h>
#include <cuComplex.h>
#include <cuda_runtime.h>

__global__ void fill_ptrs(cuDoubleComplex **pa, cuDoubleComplex *a, long long stride, long long batch) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < batch) pa[i] = a + i * stride;
}

extern "C" int cublas_zgesv_time(int n, long long batch, const void *A, const void *b, void *x, int reps,
                                 float *ms_median, int *info_nonzero) {
  cublasHandle_t h;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return 1;
  const size_t na = (size_t)batch * n * n, nb = (size_t)batch * n;
  cuDoubleComplex *wa = nullptr, *wb = nullptr, **pa = nullptr, **pb = nullptr;
  int *piv = nullptr, *info = nullptr;
  cudaMalloc(&wa, na * sizeof(cuDoubleComplex));
  cudaMalloc(&wb, nb * sizeof(cuDoubleComplex));
  cudaMalloc(&pa, batch * sizeof(void *));
  cudaMalloc(&pb, batch * sizeof(void *));
  cudaMalloc(&piv, (size_t)batch * n * sizeof(int));
  cudaMalloc(&info, batch * sizeof(int));
  const int thr = 256;
  const unsigned blocks = (unsigned)((batch + thr - 1) / thr);
  fill_ptrs<<<blocks, thr>>>(pa, wa, (long long)n * n, batch);
  fill_ptrs<<<blocks, thr>>>(pb, wb, n, batch);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  std::vector<float> ts;
  int host_info = 0, rc = 0;
  for (int rep = 0; rep < reps + 3; ++rep) {
    cudaMemcpy(wa, A, na * sizeof(cuDoubleComplex), cudaMemcpyDeviceToDevice);
    cudaMemcpy(wb, b, nb * sizeof(cuDoubleComplex), cudaMemcpyDeviceToDevice);
    cudaEventRecord(e0);
    if (cublasZgetrfBatched(h, n, pa, n, piv, info, (int)batch) != CUBLAS_STATUS_SUCCESS) rc = 2;
    if (cublasZgetrsBatched(h, CUBLAS_OP_T, n, 1, (const cuDoubleComplex *const *)pa, n, piv, pb, n, &host_info,
                            (int)batch) != CUBLAS_STATUS_SUCCESS)
      rc = 3;
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep >= 3) ts.push_back(ms);   // 3 warm-up repetitions
  }
  std::vector<int> hinfo(batch);
  cudaMemcpy(hinfo.data(), info, batch * sizeof(int), cudaMemcpyDeviceToHost);
  int nz = 0;
  for (int v : hinfo) nz += v != 0;
  cudaMemcpy(x, wb, nb * sizeof(cuDoubleComplex), cudaMemcpyDeviceToDevice);
  std::sort(ts.begin(), ts.end());
  *ms_median = ts.empty() ? -1.f : ts[ts.size() / 2];
  *info_nonzero = nz;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(wa);
  cudaFree(wb);
  cudaFree(pa);
  cudaFree(pb);
  cudaFree(piv);
  cudaFree(info);
  cublasDestroy(h);
  if (cudaGetLastError() != cudaSuccess) return 4;
  return rc;
}
