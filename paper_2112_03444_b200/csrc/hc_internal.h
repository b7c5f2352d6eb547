// hc_internal.h -- shared between the host runtime (csrc/host) and the kernels (csrc/kernels)
// of the B200 path.  Not part of the ABI (include/hc.h is).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hc.h"

namespace hcb {

// ------------------------------------------------------------------------------------------
// Evaluation op: one term contribution  out(row, col) += scale * c_j * x_{f0} * ... * x_{f7}
// (the paper's homogenised term (s_k, a_{k,j}, x_{k,m1}, ..., x_{k,mM})).  Unused
// factor slots hold N, the constant-one slot.  Ops are lane-balanced by the host
// compiler: at step q lane r executes ops[q * L + r]; ops of one output entry are contiguous in
// a lane and the last one carries OP_LAST, which stores the register accumulator to M[dest].
//   x: coefficient index (bits 0..15) | dest entry row*(N+1)+col (bits 16..31, 0xFFFF = none)
//   y: flags (bit 0 OP_LAST, bit 1 OP_RHS) | scale (bits 8..15, real integer exponent)
//   z, w: factor variable indices, one byte each (f0..f3 in z, f4..f7 in w)
// ------------------------------------------------------------------------------------------
enum : uint32_t { OP_LAST = 1u, OP_RHS = 2u };
constexpr uint32_t OP_NO_DEST = 0xFFFFu;
constexpr int MAX_FACTORS = HC_MAX_FACTORS;
constexpr int MAX_COEF_DEG = 7;   // coefficient polynomials in t: degree <= 7

// Coefficient monomial for the prologue: weight * prod_{m < deg} p_{fac[m]}  (deg <= MAX_COEF_DEG)
struct CoefMono {
  double wre, wim;
  int32_t coef;   // coefficient expression id
  int32_t deg;
  int16_t fac[MAX_COEF_DEG + 1];
};

struct DevSettings {
  double dt_init, dt_min, dt_max, grow, shrink, newton_tol, inf_norm, end_tol, res_abs, res_rel, pivot_rel;
  int32_t predictor, grow_after, max_newton, max_steps, end_newton;
};

struct TrackArgs {
  // system tables
  const uint4 *ops;          // [Q * L]
  const uint8_t *step_nfac;  // [Q]
  int32_t Q;
  int32_t ncoef;
  int32_t D;                 // degree of coefficient polynomials in t
  // batch
  const double2 *coef_t;     // [B][D+1][ncoef]
  const double2 *start_x;    // [S][N]
  int64_t S, total;          // tracks = B * S
  unsigned long long *queue; // work counter (zeroed before launch)
  double2 *x_out;            // [total][N]
  int32_t *status_out;       // [total]
  int32_t *counters_out;     // [total][4]
  double *resid_out;         // [total][2]
  DevSettings st;
};

struct PrologueArgs {
  const CoefMono *mono;      // [n_mono], sorted by coef
  const int32_t *coef_mono_ptr;  // [ncoef + 1]
  int32_t ncoef, D, P;
  const double2 *p0;         // [P]
  const double2 *p1;         // [B][P]
  int64_t B;
  double2 *coef_t;           // [B][D+1][ncoef]
};

// Launch plan for one N (filled by the per-N instantiation units).
struct TrackerPlan {
  int lanes;          // L
  int warps_per_cta;
  int ctas;           // persistent grid
  size_t smem_bytes;  // dynamic shared memory per CTA
};

size_t slot_smem_bytes(int N, int ncoef);
size_t table_smem_bytes(int Q, int L);

// Per-N launchers (csrc/kernels/tracker_n*.cu); return cudaError_t.
typedef cudaError_t (*tracker_launch_fn)(const TrackArgs &, int device, cudaStream_t, TrackerPlan *);
tracker_launch_fn tracker_launcher(int N);

cudaError_t launch_prologue(const PrologueArgs &, cudaStream_t);
cudaError_t launch_batched_zgesv(int n, int64_t batch, const double2 *A, const double2 *b, double2 *x,
                                 int32_t *info, double pivot_rel, cudaStream_t);
cudaError_t run_fp64_probe(int device, double *tflops);

inline int lanes_for(int N) {
  int L = 1;
  while (L < N) L <<= 1;
  return L;
}

}  // namespace hcb
