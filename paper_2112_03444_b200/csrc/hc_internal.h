// hc_internal.h -- shared between the host runtime (csrc/host) and the kernels (csrc/kernels)
// of the B200 path.  Not part of the ABI (include/hc.h is).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "hc.h"

namespace hcb {

// ------------------------------------------------------------------------------------------
// Evaluation tables (the paper's homogenised term records (s_k, a_{k,j}, x_{k,m1..mM}),
// P:432-434, re-laid out for the B200 kernel):
//  * coefficient slots: the prologue turns every coefficient expression c_j(p) -- with the
//    derivative scale s_k already folded in ("fold s_k into coefficients") -- into a polynomial
//    in t; the kernel evaluates c_j(t) and c_j'(t) by Horner into shared memory;
//  * monomial program: every monomial needed by dH/dx or H is computed once per evaluation as
//    mono[k] = mono[parent_k] * x[var_k], level by level (degree d from degree d-1); slots
//    0..N-1 are the unknowns, slot N the constant one (P:430's auxiliary variable x_{M+1} = 1);
//    entry = parent (bits 0..15) | var (bits 16..31);
//  * ops: out(row, col) += coef[slot] * mono[k], lane-balanced: at step q lane r executes
//    ops[q * L + r]; ops of one output entry are contiguous in a lane and the last carries
//    OP_LAST, which stores the register accumulator to M[dest]; padding ops sit after a lane's
//    last entry and never store.
//      x: coefficient slot (bits 0..15) | monomial index (bits 16..31)
//      y: dest entry (bits 0..15, 0xFFFF = none) | flags << 16 (OP_LAST, OP_RHS)
//  * entries are stored compactly (only structurally non-zero entries of [dH/dx | rhs]);
//    mpos[row*(N+1)+col] is the compact index or -1 for a structural zero.
// ------------------------------------------------------------------------------------------
enum : uint32_t { OP_LAST = 1u, OP_RHS = 2u };
constexpr uint32_t OP_NO_DEST = 0xFFFFu;
constexpr int MAX_FACTORS = HC_MAX_FACTORS;   // max monomial degree
constexpr int MAX_LEVELS = MAX_FACTORS;       // monomial program levels (degrees 2..MAX_FACTORS)
constexpr int MAX_COEF_DEG = 7;               // coefficient polynomials in t: degree <= 7

// Coefficient monomial for the prologue: weight * prod_{m < deg} p_{fac[m]}  (deg <= MAX_COEF_DEG)
struct CoefMono {
  double wre, wim;
  int32_t coef;   // coefficient expression id
  int32_t deg;
  int16_t fac[MAX_COEF_DEG + 1];
};

struct DevSettings {
  double dt_init, dt_min, dt_max, grow, shrink, newton_tol, inf_norm, end_tol, res_abs, res_rel, pivot_rel;
  // endgame (reading R26; hc.h documents each field)
  double eg_start, eg_inf_mu, eg_sing_mu, eg_stab, eg_inf_s, eg_inf_norm, eg_tol;
  int32_t predictor, grow_after, max_newton, max_steps, end_newton;
  int32_t eg_samples, eg_max_winding, eg_max_radii;
};

// Internal track status: handed from the tracker to the Cauchy endgame kernel (never returned).
constexpr int32_t HC_EG_PENDING = 7;

// Per-slot endgame sampling state of the tracker kernel (shared memory, written by lane 0 of the
// slot): next sample point, the previous sample (log s, log ||x||, log s||dx/dt||), previous mu,
// the current norms, and the run lengths of the at-infinity / singular conditions (reading R26).
struct EgSample {
  double s_next, pls, plx, pld, mu_prev;
  double xn2, kn2;   // ||x||_inf^2 at the last accepted point, ||k1||_inf^2 of the current step
  int32_t nsamp, inf_run, sing_run, pad;
};

struct TrackArgs {
  // system tables
  const uint2 *ops;          // [Q * L]
  int32_t Q;                 // op steps (paired table: 2 x pair steps, the table's size in uint2 units)
  int32_t Qp;                // pair steps of a paired op table (0: single ops; abi.cpp pair_ops)
  const uint32_t *mono_prog; // [n_mono - (N + 1)]
  int32_t n_mono;            // monomial table size including the N unknowns and the constant
  int32_t n_levels;
  int32_t level_end[MAX_LEVELS];  // level l covers [level_end[l-1] (or N+1), level_end[l])
  int32_t ncoef;             // coefficient slots
  int32_t ncoef_src;         // slots [0, ncoef_src) are the descriptor's coefficients (used by rhs ops)
  int32_t D;                 // degree of coefficient polynomials in t
  const int16_t *mpos;       // [N * (N + 1)] dense -> compact entry index, -1 = structural zero
  int32_t n_entries;         // compact entries
  // batch
  const double2 *coef_t;     // [B][D+1][ncoef]
  const double2 *start_x;    // [S][N]
  int64_t S, total;          // tracks = B * S
  unsigned long long *queue; // work counter (zeroed before launch)
  double2 *x_out;            // [total][N]
  int32_t *status_out;       // [total]
  int32_t *counters_out;     // [total][4]
  double *resid_out;         // [total][2]
  int32_t *winding_out;      // [total] Cauchy endgame winding number (0: not used)
  int64_t *eg_list;          // [total] tracks handed to the Cauchy endgame (status HC_EG_PENDING)
  unsigned long long *eg_count;  // [2]: tracks in eg_list; the endgame kernel's work counter
  DevSettings st;
  unsigned long long *phase_cycles;  // [8] per-phase clock sums (only in HCB_PHASE_TIMING builds), or null
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

// Per-N launchers (csrc/kernels/tracker_n*.cu); return cudaError_t.
typedef cudaError_t (*tracker_launch_fn)(const TrackArgs &, int device, cudaStream_t, TrackerPlan *);
tracker_launch_fn tracker_launcher(int N);

cudaError_t launch_prologue(const PrologueArgs &, cudaStream_t);
cudaError_t launch_batched_zgesv(int n, int64_t batch, const double2 *A, const double2 *b, double2 *x,
                                 int32_t *info, double pivot_rel, cudaStream_t);
cudaError_t run_fp64_probe(int device, double *tflops);

// Track layouts.  Default: a sub-warp of L = next_pow2(N) lanes, lane r owns row r.  Hybrid
// layout for 17 <= N <= 18: L = 16 lanes (two tracks per warp); lane r owns row r, and the
// E = N - 16 "extra" rows 16..N-1 are held column-distributed (lane r holds their columns r and
// r + 16), see tracker.cuh lu_rows_hy.  Host (op balancing over L lanes) and device agree here.
#ifndef HCB_HYBRID_LAYOUT
#define HCB_HYBRID_LAYOUT 0   // experiment switch: measured slower on trifocal
#endif
__host__ __device__ constexpr bool hy_layout(int N) { return HCB_HYBRID_LAYOUT && (N == 17 || N == 18); }
__host__ __device__ constexpr int lanes_for(int N) {
  return hy_layout(N) ? 16 : (N <= 1) ? 1 : (N <= 2) ? 2 : (N <= 4) ? 4 : (N <= 8) ? 8 : (N <= 16) ? 16 : 32;
}

// CTA shape of the tracker kernel (warps per CTA, minimum resident CTAs per SM), shared by the
// kernel's __launch_bounds__ and the host's layout policy (hc_track_batch).
#ifndef HCB_MAXW_MID   // warps per CTA for 17 <= N <= 20 (A/B experiments override it)
#define HCB_MAXW_MID 12
#endif
#ifndef HCB_MAXW_MID16   // warps per CTA for N = 15, 16 (16-lane tracks; A/B experiments override it)
#define HCB_MAXW_MID16 16
#endif
#ifndef HCB_MAXW_LOW   // warps per CTA and CTAs per SM for N <= 14 (A/B experiments override them)
#define HCB_MAXW_LOW 4
#endif
#ifndef HCB_MINB_LOW
#define HCB_MINB_LOW 4
#endif
__host__ __device__ constexpr int tracker_maxw(int N, int LW) {
  return (hy_layout(N) && LW == lanes_for(N)) ? 8
         : (N == 15 || N == 16)               ? HCB_MAXW_MID16
         : (N >= 17 && N <= 20)               ? HCB_MAXW_MID
         : (N <= 14)                          ? HCB_MAXW_LOW
                                              : 4;
}
__host__ __device__ constexpr int tracker_minb(int N) { return (N <= 14) ? HCB_MINB_LOW : (N <= 20) ? 1 : 2; }
// The 128-register kernels (16 resident warps per SM) keep the RK / corrector vectors and the slot's
// rarely touched scalars in shared memory, so their registers go to the rows being eliminated;
// N <= HCB_SS_MIN_N keeps them in registers (small rows leave room).
#ifndef HCB_SS_MIN_N
#define HCB_SS_MIN_N 8
#endif
__host__ __device__ constexpr bool tracker_smem_state(int N, int LW) {
  return tracker_maxw(N, LW) * tracker_minb(N) >= 16 && N > HCB_SS_MIN_N;
}

}  // namespace hcb
