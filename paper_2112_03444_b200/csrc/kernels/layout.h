// layout.h -- shared-memory layout of the tracker kernel (host and device agree on sizes).
#pragma once

#include <cstddef>
#include <cuda_runtime.h>

namespace hcb {

__host__ __device__ inline size_t align16(size_t b) { return (b + 15) & ~size_t(15); }

// Per track slot: the endgame sampling state (80 bytes, EgSample), the shared-memory tracker state (state_bytes, below), cval[ncoef + ncoef_src]
// (c(t) for every slot, c'(t) for the rhs slots), mono[n_mono + 1] (x_0..x_{N-1}, 1, shared products, a constant zero),
// M[n_entries] (non-zero entries of [dH/dx | rhs]), prow[2 * (N + 1)] (double-buffered pivot row),
// rabs[N] (doubles).
constexpr size_t EG_SAMPLE_BYTES = 80;
// Per-lane tracker state kept in shared memory (the 128-register kernels): the RK / corrector vectors
// [kacc | kprev | xc][lnc] (double2) and one copy of the slot's scalars (64 bytes: track id, step, h,
// t1, the t of the cached coefficients, four counters).  lnc = state lanes x unknowns per lane: the
// lanes without a row (r >= N) share one dummy entry, so a 32-lane track of N unknowns keeps N + 1.
__host__ __device__ constexpr int state_lanes(int N, int L, int NC) { return (NC == 1 && L > N) ? N + 1 : L * NC; }
__host__ __device__ inline size_t state_bytes(int lnc) { return lnc ? (size_t)48 * lnc + 64 : 0; }
__host__ __device__ inline size_t slot_bytes(int N, int lnc, int ncoef, int ncoef_src, int n_mono, int n_entries) {
  return EG_SAMPLE_BYTES + state_bytes(lnc) +
         align16(sizeof(double) * 2 * ((size_t)ncoef + ncoef_src + n_mono + 1 + n_entries + 2 * (N + 1)) +
                 sizeof(double) * N);
}

// Per CTA, before the slots: the op table [Q * L] (8 B each), the monomial program (4 B each) and
// the dense -> compact entry map (2 B each).
__host__ __device__ inline size_t table_bytes(int Q, int L, int nprog, int N) {
  return align16((size_t)8 * Q * L) + align16((size_t)4 * nprog) + align16((size_t)2 * N * (N + 1));
}

}  // namespace hcb
