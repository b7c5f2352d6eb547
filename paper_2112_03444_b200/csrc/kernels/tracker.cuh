// tracker.cuh -- the fused persistent HC path-tracking kernel for sm_100a (one template per N).
//
// One sub-warp of L = next_pow2(N) lanes owns one track ("a track to a warp", with
// sub-warps when N <= 16); lane r owns Jacobian row r, right-hand-side entry r and unknown x_r
// ("one row per thread").  Every loop iteration performs exactly one
//     evaluate (dH/dx | rhs)  ->  fused LU + solve on [A | b]
// per track slot, where the rhs is dH/dt (RK4 stage, Eq. 3 P:168 / P:175) or H (Newton, Eq. 6
// P:182).  Each slot runs its own state machine (RK stage s, Newton iteration, endpoint polish,
// residual), so slots of one warp never wait for each other, and the single solve call site keeps
// the unrolled LU in the instruction cache once (no loop-invariant branch may guard code inside the
// loop: the compiler would unswitch the loop and duplicate that call site -- DESIGN.md §7c).
// Finished slots pull the next track id from a
// global atomic queue (persistent kernel); tracks are ordered instance-major so concurrently
// running slots share an instance's coefficient table in L1/L2.
//
// Evaluation: the host compiler turned dH/dx, H and dH/dt into coefficient slots, a
// shared monomial program and a lane-balanced op list (a constant-one slot pads); the tables sit
// in shared memory for the whole kernel (staged by bulk async copies; the wide layout reads paired
// op records, two terms per record).  Coefficient values c_j(t), c_j'(t) come from
// per-instance polynomials in t (prologue kernel) by Horner.  The elimination keeps row r of
// [J | rhs] in lane r's registers, pivots by an arg-max of |a|^2 (REDUX for 32-lane tracks,
// shuffles otherwise; ties -> lower row), broadcasts the pivot row through shared memory, and
// eliminates above and below the pivot (Gauss-Jordan), so the solution needs one division per row
// and no back-substitution (kernel fusion + augmented matrix).
// Lane layouts: L = next_pow2(N) lanes per track (throughput) or 32 (wide latency layout, N <= 16).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "../hc_internal.h"
#include "layout.h"
#include "bulk.cuh"

namespace hcb {

constexpr unsigned FULL = 0xffffffffu;

// Optional per-phase cycle accounting (experiments only: -DHCB_PHASE_TIMING).
#ifdef HCB_PHASE_TIMING
#define HCB_T(var) const long long var = clock64()
#define HCB_ACC(i, a, b) (hcb_phase[i] += (unsigned long long)((b) - (a)))
#else
#define HCB_T(var)
#define HCB_ACC(i, a, b)
#endif
// Warps per CTA and minimum resident CTAs per SM, by N (register budget 65536 / (32 * warps * ctas)):
//   N <= 14: 4 warps x 4 CTAs (128 regs);  N = 15, 16 (two 16-lane tracks per warp): one 16-warp CTA
//   (128 regs; 5-point relpose: 2.7 % faster than 12 warps at 168);  17..20: one 12-warp CTA per SM
//   (168 regs; measured on the trifocal system: 12 warps at 168 regs beat 16 at 128 (spills) and 8
//   at 218);  N > 20: 4 warps x 2 CTAs.  The launcher shrinks the CTA when the shared memory does
//   not fit.
//   Hybrid layout (hy_layout(N), 16-lane tracks with column-distributed extra rows): one 8-warp CTA
//   (16 tracks; shared memory bound).
// LW: lanes per track -- lanes_for(N) (throughput layout, 32/LW tracks per warp) or 32 (the wide
// latency layout for N <= 16: one track per warp, its op list and monomial program spread over 32
// lanes and REDUX-based reductions; chosen by the host for batches that under-fill the GPU).
template <int N, int LW = lanes_for(N)>
struct TrackerShape {
  static constexpr bool HY = hy_layout(N) && LW == lanes_for(N);
  static constexpr int L = LW;
  static constexpr int E = HY ? N - 16 : 0;   // extra rows (hybrid layout)
  static constexpr int NC = HY ? 2 : 1;       // unknown components per lane
  static constexpr int MAXW = tracker_maxw(N, LW);
  static constexpr int MINB = tracker_minb(N);
  // 128-register kernels (16 resident warps per SM) keep the RK / corrector vectors and the rarely
  // touched per-track scalars in shared memory, the others (N >= 17: 168 registers) in registers,
  // where the shared memory would only shrink the L1 that serves the coefficient tables
#ifdef HCB_SMEM_STATE_ALL   // A/B switch: per-lane state in shared memory for every N
  static constexpr bool SMEM_STATE = true;
#else
  static constexpr bool SMEM_STATE = tracker_smem_state(N, LW);
#endif
  static constexpr int LNC = SMEM_STATE ? state_lanes(N, L, NC) : 0;   // state lanes in the slot (layout.h)
  static constexpr int LV = SMEM_STATE ? LNC / NC : 1;                 // ... per unknown component
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// c + a * b
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {
  return make_double2(fma(a.x, b.x, fma(-a.y, b.y, c.x)), fma(a.x, b.y, fma(a.y, b.x, c.y)));
}
// c - a * b
__device__ __forceinline__ double2 cfms(double2 c, double2 a, double2 b) {
  return make_double2(fma(-a.x, b.x, fma(a.y, b.y, c.x)), fma(-a.x, b.y, fma(-a.y, b.x, c.y)));
}
__device__ __forceinline__ double abs2(double2 a) { return fma(a.x, a.x, a.y * a.y); }
// 1/x for x > 0: MUFU reciprocal estimate + two Newton steps (full FP64 accuracy, no slow-path
// call; non-finite or zero x gives a non-finite or huge result, and such pivots fail the
// singularity test anyway).
__device__ __forceinline__ double frcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  double e = fma(-x, r, 1.0);
  r = fma(r, e, r);
  e = fma(-x, r, 1.0);
  return fma(r, e, r);
}
__device__ __forceinline__ double2 crecip(double2 a) {
  const double d = frcp(abs2(a));
  return make_double2(a.x * d, -a.y * d);
}
__device__ __forceinline__ bool cfinite(double2 a) { return isfinite(a.x) && isfinite(a.y); }
// max that propagates NaN from b (a is >= 0 or NaN already)
__device__ __forceinline__ double nmax(double a, double b) { return (b > a || b != b) ? b : a; }
__device__ __forceinline__ double2 shfl2(double2 v, int src, int width) {
  return make_double2(__shfl_sync(FULL, v.x, src, width), __shfl_sync(FULL, v.y, src, width));
}

#ifndef HCB_OUT_EXPERIMENT   // DRAM-traffic experiments (scripts/gpu.sh traffic_ab): 1 = no status/counter/
#define HCB_OUT_EXPERIMENT 0  // residual writes, 2 = no x writes (results invalid)
#endif
#ifndef HCB_EG_SAMPLING   // endgame sampling in the tracker (A/B switch; 0 = no endgame hand-off)
#define HCB_EG_SAMPLING 1
#endif
#ifndef HCB_SEG16_REDUX   // 8- and 16-lane tracks: REDUX-based segment max / arg-max (A/B switch)
#define HCB_SEG16_REDUX 1
#endif
template <int L>
__host__ __device__ constexpr unsigned seg_mask();
// Per-segment maximum of an unsigned value for 32/L tracks per warp: one full-warp REDUX per segment
// (lanes of the other segments contribute 0), each lane takes its own segment's result.
template <int L>
__device__ __forceinline__ unsigned seg_redux_max(unsigned x) {
  const int sg = (threadIdx.x & 31) / L;
  unsigned m = 0u;
#pragma unroll
  for (int k = 0; k < 32 / L; ++k) {
    const unsigned mk = __reduce_max_sync(FULL, sg == k ? x : 0u);
    if (sg == k) m = mk;
  }
  return m;
}

// Maximum over the L lanes of a segment of a value that is >= 0 or NaN.  L == 32, 16, 8: exact max
// by REDUX on the high then the low words of the IEEE bit pattern (non-negative doubles order like
// their bits; a NaN lane yields a NaN result, which every caller treats like a failure; one REDUX
// per segment and pass for 16 and 8 lanes); L < 8: butterfly of the NaN-propagating nmax (a NaN residual or step norm
// classifies the same way for every lane width, as the oracle's max does).
template <int L>
__device__ __forceinline__ double seg_max(double v) {
  if constexpr ((L == 16 || L == 8) && HCB_SEG16_REDUX) {   // per-segment REDUX (as for 32 lanes)
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned mhi = seg_redux_max<L>((unsigned)(bits >> 32));
    const unsigned mlo = seg_redux_max<L>(((unsigned)(bits >> 32) == mhi) ? (unsigned)bits : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  } else if constexpr (L == 32) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned mhi = __reduce_max_sync(FULL, (unsigned)(bits >> 32));
    const unsigned mlo = __reduce_max_sync(FULL, ((unsigned)(bits >> 32) == mhi) ? (unsigned)bits : 0u);
    return __longlong_as_double((long long)(((unsigned long long)mhi << 32) | mlo));
  } else {
#pragma unroll
    for (int off = L / 2; off >= 1; off >>= 1) v = nmax(v, __shfl_xor_sync(FULL, v, off));
    return v;
  }
}
template <int L>
__host__ __device__ constexpr unsigned seg_mask() {
  if constexpr (L == 32) return FULL;
  else return (1u << L) - 1u;
}
template <int L>
__device__ __forceinline__ bool seg_all(bool p, int seg) {
  const unsigned b = __ballot_sync(FULL, p);
  const unsigned m = seg_mask<L>() << ((L == 32) ? 0 : seg * L);
  return (b & m) == m;
}

enum SlotState : int { ST_RK = 0, ST_NEWTON = 1, ST_POLISH = 2, ST_RESID = 3, ST_DONE = 4, ST_EGFIN = 5 };

// ------------------------------------------------------------------------------------------
// Arg-max of v over the L lanes of a segment; ties -> lowest lane.  v < 0 marks a non-candidate.
// L == 32: two REDUX (max of the high, then low words of the IEEE bit pattern, which orders
// non-negative doubles like their values) + one ballot; L < 32: shuffle butterfly.
// Returns the winning lane (segment-relative) and the maximum value (-1 when no candidate).
// ------------------------------------------------------------------------------------------
// Arg-max with the singularity test folded in: returns the pivot lane and sets sing when the maximum
// is <= thr (or there is no candidate).  L == 32: the common case -- a unique maximum in the high
// words that differs from thr's high word -- needs a single REDUX; ties or a high word equal to
// thr's take the exact two-REDUX path of seg_argmax.
template <int L>
__device__ __forceinline__ int seg_argmax(double v, int r, double &vmax);
#ifndef HCB_PACKED_ARGMAX   // 32-lane arg-max by one REDUX on a packed (|a|^2 bits, lane) key (A/B switch)
#define HCB_PACKED_ARGMAX 0
#endif
template <int L>
__device__ __forceinline__ int seg_argmax_thr(double v, int r, double thr, bool &sing) {
  if constexpr (L == 32 && HCB_PACKED_ARGMAX) {
    // key = the top 27 bits of |a|^2's IEEE pattern (exponent + 16 mantissa bits; sign is 0) above
    // 31 - lane: one REDUX gives the pivot and ties (to 2^-16 relative) go to the lowest row;
    // non-candidates (used rows, padding, NaN) have key 0
    const unsigned hi = (unsigned)((unsigned long long)__double_as_longlong(v) >> 36);
    const unsigned key = (v >= 0.0) ? ((hi << 5) | (31u - (unsigned)r)) : 0u;
    const unsigned mk = __reduce_max_sync(FULL, key);
    const unsigned thr_hi = (unsigned)((unsigned long long)__double_as_longlong(thr) >> 36);
    sing |= (mk == 0u) || ((mk >> 5) <= thr_hi);
    return 31 - (int)(mk & 31u);
  } else if constexpr (L == 32) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (v >= 0.0) ? (unsigned)(bits >> 32) + 1u : 0u;
    const unsigned mhi = __reduce_max_sync(FULL, hi);
    const unsigned b1 = __ballot_sync(FULL, hi == mhi);
    const unsigned thr_hi1 = (unsigned)((unsigned long long)__double_as_longlong(thr) >> 32) + 1u;
    if (__popc(b1) == 1 && mhi != thr_hi1 && mhi != 0u) {   // warp-uniform branch
      sing |= (mhi < thr_hi1);
      return __ffs(b1) - 1;
    }
    double vmax;
    const int idx = seg_argmax<L>(v, r, vmax);
    sing |= !(vmax > thr);
    return idx;
  } else if constexpr ((L == 16 || L == 8) && HCB_SEG16_REDUX) {
    // 32/L tracks per warp: the high-word maximum of each segment by one full-warp REDUX each (the
    // other segments contribute 0), then the same unique-maximum test as for 32 lanes; the fast
    // path is taken only when every segment passes it (warp-uniform), else the exact butterfly
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (v >= 0.0) ? (unsigned)(bits >> 32) + 1u : 0u;
    const unsigned mhi = seg_redux_max<L>(hi);
    const int sg = (threadIdx.x & 31) / L;
    const unsigned b1 = __ballot_sync(FULL, hi == mhi) & (seg_mask<L>() << (L * sg));
    const unsigned thr_hi1 = (unsigned)((unsigned long long)__double_as_longlong(thr) >> 32) + 1u;
    if (__all_sync(FULL, __popc(b1) == 1 && mhi != thr_hi1 && mhi != 0u)) {
      sing |= (mhi < thr_hi1);
      return __ffs(b1) - 1 - L * sg;
    }
    double vmax;
    const int idx = seg_argmax<L>(v, r, vmax);
    sing |= !(vmax > thr);
    return idx;
  } else {
    double vmax;
    const int idx = seg_argmax<L>(v, r, vmax);
    sing |= !(vmax > thr);
    return idx;
  }
}

template <int L>
__device__ __forceinline__ int seg_argmax(double v, int r, double &vmax) {
  if constexpr (L == 32) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    const unsigned hi = (v >= 0.0) ? (unsigned)(bits >> 32) + 1u : 0u;
    const unsigned mhi = __reduce_max_sync(FULL, hi);
    const unsigned lo = (hi == mhi) ? (unsigned)bits : 0u;
    const unsigned mlo = __reduce_max_sync(FULL, lo);
    const unsigned ball = __ballot_sync(FULL, hi == mhi && lo == mlo);
    vmax = (mhi == 0u) ? -1.0 : __longlong_as_double((long long)(((unsigned long long)(mhi - 1u) << 32) | mlo));
    return __ffs(ball) - 1;
  } else {
    int idx = r;
#pragma unroll
    for (int off = L / 2; off >= 1; off >>= 1) {
      const double ov = __shfl_xor_sync(FULL, v, off);
      const int oi = __shfl_xor_sync(FULL, idx, off);
      if (ov > v || (ov == v && oi < idx)) {
        v = ov;
        idx = oi;
      }
    }
    vmax = v;
    return idx;
  }
}

// ------------------------------------------------------------------------------------------
// Fused elimination with partial pivoting on [A | b] held one row per lane (a[0..N-1] = row r of
// A, a[N] = b_r) (one kernel, the augmented matrix carries the triangular solve with L).
// The paper back-substitutes on the cached U; here the rows already pivoted also eliminate the
// current column (Gauss-Jordan), which costs nothing extra in the one-row-per-lane SIMT layout and
// replaces the N-step sequential back-substitution by one division per row.
// Pivot = max |a|^2 over the not-yet-pivoted rows (ties -> lowest row, reading R13); singular when
// |pivot| <= pivot_rel * max|A_ij| (R9) or anything is non-finite.
// Latency schedule (one warp owns the whole factorisation, so the per-column dependency chain is
// the cost): every lane computes 1/a_rk of its candidate speculatively; once the arg-max names the
// pivot lane, 1/pivot and the pivot row's column k+1 are shuffled from it while the rest of its row
// goes through a double-buffered shared row (one __syncwarp per column); every other row updates
// column k+1 first, and the arg-max for step k+1 starts on it while the remaining columns are
// updated.  The pivot lane also parks 1/pivot in pinv[k] (scratch that is dead during the solve)
// for the final division.  Solution components are collected through shared memory.
// Returns the solution component y_r in lane r and a slot-uniform success flag.
// prow: 2 * (N + 1) double2, pinv: N double2 (per slot shared memory).
// ------------------------------------------------------------------------------------------
#ifndef HCB_LU_PRED_PUBLISH   // 32-lane tracks publish the pivot row with predicated stores (A/B switch)
#define HCB_LU_PRED_PUBLISH 1
#endif
#ifndef HCB_LU_PINV   // 1/pivot parked in shared scratch (1) or kept in registers (0) (A/B switch)
#define HCB_LU_PINV (-1)   // -1: scratch for 32-lane tracks (one more predicated store in the publish
#endif                     // run), registers for narrower ones (A/B: 4-view +2.7 %, trifocal -2.5 %)
#ifndef HCB_LU_SYNC_EARLY   // __syncwarp right after the publish (1), or after the next arg-max (0)
#define HCB_LU_SYNC_EARLY (-1)   // -1: by N (measured: N <= 16 +4.5 %, N = 18 -0.7 %)
#endif
// 16-byte shared-memory store under a predicate (a predicated st.shared, not a divergent branch)
__device__ __forceinline__ void st_shared_if(bool pred, double2 *dst, double2 v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.u32 p, %0, 0;\n @p st.shared.v2.f64 [%1], {%2, %3};\n}" ::"r"((unsigned)pred),
               "r"(smem_u32(dst)), "d"(v.x), "d"(v.y)
               : "memory");
}
template <int N, int L>
__device__ __forceinline__ bool lu_rows(double2 (&a)[N + 1], int r, int seg, double2 *prow, double2 *pinv,
                                        double pivot_rel, double lane_max, double2 &y) {
  constexpr bool SYNC_EARLY = (HCB_LU_SYNC_EARLY < 0) ? (N <= 16) : (HCB_LU_SYNC_EARLY != 0);
  constexpr bool PINV = (HCB_LU_PINV < 0) ? (L == 32) : (HCB_LU_PINV != 0);
  // rows already pivoted (and padding rows) are excluded from the arg-max by a -inf bias on |a|^2
  // (one DADD per column; a NaN result is never a candidate either)
  double vbias = (r >= N) ? -INFINITY : 0.0;
  int mystep = (r >= N) ? N : -1;
  double2 myinv = make_double2(0.0, 0.0);   // (HCB_LU_PINV == 0: 1/pivot kept in registers)
  // lane_max: max |A_ij|^2 over the entries this lane holds or produced (NaN entries are ignored by
  // fmax; they make the solve fail through the non-finite solution check)
  const double am = seg_max<L>(lane_max);
  const double thr = pivot_rel * pivot_rel * am;
  bool sing = !(am < INFINITY);
  // pivot of step 0
  double v0 = abs2(a[0]) + vbias;
  if (!(v0 >= 0.0)) v0 = -1.0;   // NaN is never a pivot
  int p = seg_argmax_thr<L>(v0, r, thr, sing);
  double2 spec = crecip(a[0]);   // speculative 1/a_rk of this lane's candidate (overlaps the search)
#pragma unroll
  for (int k = 0; k < N; ++k) {
    double2 *pr = prow + (k & 1) * (N + 1);
    // early broadcast from the pivot lane by shuffles: 1/pivot and the pivot row's column k+1
    const double2 inv = shfl2(spec, p, L);
    const double2 u1 = shfl2(a[k + 1], p, L);
    const bool me = (r == p);
    // the pivot lane publishes the rest of its row (columns k+2..N) through shared memory, and parks
    // 1/pivot for the final division (pinv: slot scratch, dead during the solve).  32-lane tracks:
    // predicated stores (not a branch), so the scheduler interleaves them with the FP64 work around
    // them (trifocal +2.3 %); narrower tracks keep the branch (4-view: 2.3 % faster with it).
    if constexpr (L == 32 && HCB_LU_PRED_PUBLISH) {
#pragma unroll
      for (int j = k + 2; j <= N; ++j) st_shared_if(me, &pr[j], a[j]);
      if constexpr (PINV) st_shared_if(me, &pinv[k], spec);
    } else if (me) {
#pragma unroll
      for (int j = k + 2; j <= N; ++j) pr[j] = a[j];
      if constexpr (PINV) pinv[k] = spec;
    }
    if (me) {
      vbias = -INFINITY;
      mystep = k;
      if constexpr (!PINV) myinv = spec;
    }
    if constexpr (SYNC_EARLY) __syncwarp();   // the published row is visible: its loads may start early
    // Gauss-Jordan: every row except the pivot row eliminates column k -- the rows pivoted earlier
    // too, which in this one-row-per-lane layout costs no extra instruction (the whole warp runs
    // the update anyway) and removes the sequential back-substitution.  Padding rows are zero.
    const double2 lc = cmul(a[k], inv);
    const double2 l = me ? make_double2(0.0, 0.0) : lc;
    a[k + 1] = cfms(a[k + 1], l, u1);   // column k+1 first (k + 1 == N: the right-hand side)
    if (k + 1 < N) {
      double v = abs2(a[k + 1]) + vbias;
      if (L < 32 && !(v >= 0.0)) v = -1.0;   // NaN is never a pivot (the REDUX path excludes it itself)
      spec = crecip(a[k + 1]);
      p = seg_argmax_thr<L>(v, r, thr, sing);
      if constexpr (!SYNC_EARLY) __syncwarp();   // the published row is visible
      // trailing update in chunks of 4 columns: the 4 shared loads are issued before their FMAs so
      // the load latency overlaps (the compiler otherwise keeps only ~2 loads in flight)
#pragma unroll
      for (int j0 = k + 2; j0 <= N; j0 += 4) {
        double2 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (j0 + i <= N) u[i] = pr[j0 + i];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (j0 + i <= N) a[j0 + i] = cfms(a[j0 + i], l, u[i]);
      }
    }
  }
  // ---- the system is now diagonal in pivot order: x_{mystep} = b' / pivot, routed through shared memory ----
  double2 *xsol = prow;
  // a row that was never a pivot (mystep == -1: only when the search found no usable candidate, i.e.
  // a singular solve) writes nothing -- xsol[-1] would be the slot's always-zero entry of M
  if (mystep >= 0 && mystep < N) xsol[mystep] = cmul(a[N], PINV ? pinv[mystep] : myinv);
  __syncwarp();
  const double2 sol = (r < N) ? xsol[r] : make_double2(0.0, 0.0);
  y = sol;
  return seg_all<L>(!sing && cfinite(sol), seg);
}

// ------------------------------------------------------------------------------------------
// The same elimination in the hybrid layout (hy_layout(N), 17 <= N <= 18): 16 lanes per track,
// two tracks per warp.  Lane r holds row r of [A | b] in a[0..N] and, for each extra row
// 16 + q (q < E = N - 16), the entries of columns r and r + 16 in e[q][0], e[q][1] (the second
// exists when r + 16 <= N).  A 32-lane track would leave 14 of 32 lanes idle for N = 18; here the
// idle work is 2 extra rows spread over 16 lanes, and the per-column pivot overhead is shared by
// two tracks.  Same pivots (max |a|^2, ties -> lowest row, R13), same Gauss-Jordan update order.
// Per column k: arg-max over own rows and the extras' column k (held by lane k & 15) by a
// 16-lane (value, row) butterfly; 1/pivot and the pivot row's column k+1 are shuffled from the
// lane(s) holding them; the extras' column-k entries are shuffled to every lane for their
// multipliers; column k+1 is updated first; the pivot row's columns k+2..N go through shared
// memory (an own row by its lane, an extra row by all lanes); then the trailing update.
// Returns x_r in y[0] and x_{16+r} (r < E) in y[1].
// ------------------------------------------------------------------------------------------
template <int N, int E>
__device__ __forceinline__ bool lu_rows_hy(double2 (&a)[N + 1], double2 (&e)[E][2], int r, int seg, double2 *prow,
                                           double pivot_rel, double lane_max, double2 (&y)[2]) {
  constexpr int L = 16;
  const double2 zero = make_double2(0.0, 0.0);
  bool used = false;
  int mystep = N;
  double2 myinv = zero;
  bool eused[E];
  int estep[E];
  double2 einv[E];
#pragma unroll
  for (int q = 0; q < E; ++q) {
    eused[q] = false;
    estep[q] = N;
    einv[q] = zero;
  }
  const double am = seg_max<L>(lane_max);
  const double thr = pivot_rel * pivot_rel * am;
  bool sing = !(am < INFINITY);
#pragma unroll
  for (int k = 0; k < N; ++k) {
    const int kc = k & 15, ks = k >> 4;               // lane and slot of the extras' column k
    const int kc1 = (k + 1) & 15, ks1 = (k + 1) >> 4;  // ... and of column k+1
    double2 *pr = prow + (k & 1) * (N + 1);
    // ---- pivot: (value, row) arg-max over the own rows and the extras' column k ----
    double v = used ? -1.0 : abs2(a[k]);
    if (!(v >= 0.0)) v = -1.0;   // NaN is never a pivot
    int row = r;
#pragma unroll
    for (int q = 0; q < E; ++q) {
      double ve = abs2(e[q][ks]);
      if (eused[q] || r != kc || !(ve >= 0.0)) ve = -1.0;
      if (ve > v) {
        v = ve;
        row = 16 + q;
      }
    }
#pragma unroll
    for (int off = L / 2; off >= 1; off >>= 1) {
      const double ov = __shfl_xor_sync(FULL, v, off);
      const int orow = __shfl_xor_sync(FULL, row, off);
      if (ov > v || (ov == v && orow < row)) {
        v = ov;
        row = orow;
      }
    }
    const int pid = row;   // uniform over the segment
    sing |= !(v > thr);
    // ---- 1/pivot and the pivot row's column k+1 ----
    double2 pv = a[k], pu = a[k + 1];
    int src = pid, src1 = pid;
    if (pid >= 16) {
#pragma unroll
      for (int q = 0; q < E; ++q)
        if (pid == 16 + q) {
          pv = e[q][ks];
          pu = e[q][ks1];
        }
      src = kc;
      src1 = kc1;
    }
    const double2 inv = crecip(shfl2(pv, src, L));
    const double2 u1 = shfl2(pu, src1, L);
    // ---- multipliers (the pivot row keeps its entries; every other row is eliminated) ----
    const bool me = (r == pid);
    const double2 l = me ? zero : cmul(a[k], inv);
    double2 le[E];
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const double2 ek = shfl2(e[q][ks], kc, L);
      le[q] = (pid == 16 + q) ? zero : cmul(ek, inv);
    }
    // ---- column k+1 first (k + 1 == N: the right-hand side) ----
    a[k + 1] = cfms(a[k + 1], l, u1);
#pragma unroll
    for (int q = 0; q < E; ++q) {
      const double2 t1 = cfms(e[q][ks1], le[q], u1);
      if (r == kc1) e[q][ks1] = t1;
    }
    if (me) {
      used = true;
      mystep = k;
      myinv = inv;
    }
#pragma unroll
    for (int q = 0; q < E; ++q)
      if (pid == 16 + q) {
        eused[q] = true;
        estep[q] = k;
        einv[q] = inv;
      }
    if (k + 1 < N) {
      // ---- publish columns k+2..N of the pivot row ----
      if (me) {
#pragma unroll
        for (int j = k + 2; j <= N; ++j) pr[j] = a[j];
      }
      if (pid >= 16) {
        double2 s0 = zero, s1 = zero;
#pragma unroll
        for (int q = 0; q < E; ++q)
          if (pid == 16 + q) {
            s0 = e[q][0];
            s1 = e[q][1];
          }
        pr[r] = s0;
        if (r + 16 <= N) pr[r + 16] = s1;
      }
      __syncwarp();
      // ---- trailing update: own row, columns k+2..N (4 loads in flight per chunk) ----
#pragma unroll
      for (int j0 = k + 2; j0 <= N; j0 += 4) {
        double2 u[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (j0 + i <= N) u[i] = pr[j0 + i];
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (j0 + i <= N) a[j0 + i] = cfms(a[j0 + i], l, u[i]);
      }
      // ---- trailing update of the extras: lane r's columns r and r + 16 when >= k+2 ----
      if (k + 2 <= 15) {
        const double2 u = pr[r];
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const double2 t0 = cfms(e[q][0], le[q], u);
          if (r >= k + 2) e[q][0] = t0;
        }
      }
      {
        const int c1 = (r + 16 <= N) ? r + 16 : N;
        const double2 u = pr[c1];
#pragma unroll
        for (int q = 0; q < E; ++q) {
          const double2 t0 = cfms(e[q][1], le[q], u);
          if (r + 16 >= k + 2 && r + 16 <= N) e[q][1] = t0;
        }
      }
    }
  }
  __syncwarp();
  // ---- the system is diagonal in pivot order: x_step = b' / pivot ----
  double2 *xsol = prow;
  if (mystep < N) xsol[mystep] = cmul(a[N], myinv);
  if (r == (N & 15)) {
#pragma unroll
    for (int q = 0; q < E; ++q)
      if (estep[q] < N) xsol[estep[q]] = cmul(e[q][N >> 4], einv[q]);
  }
  __syncwarp();
  y[0] = xsol[r];
  y[1] = (r < E) ? xsol[16 + r] : zero;
  return seg_all<L>(!sing && cfinite(y[0]) && cfinite(y[1]), seg);
}

// ------------------------------------------------------------------------------------------
// Op list: M[dest] = sum over the entry's ops of coef[slot] * mono[k] (P:432-434 terms with the
// products shared through the monomial program).  ABS also accumulates sum |c m| for the
// relative residual of the rhs rows (reading R10).
// ------------------------------------------------------------------------------------------
// One op: accumulate c*m; at the entry's last op store the entry and reset.  The complex product is
// split over two accumulators (c.x*m and the c.y part) so the four DFMAs of an op depend only on
// the previous op's same-part accumulator (chain of 1).
template <int N, bool ABS>
__device__ __forceinline__ void op_accumulate(uint2 op, double2 c, double2 m, double2 &acc, double2 &acc2,
                                              double &acc_abs, double2 *__restrict__ M, double *__restrict__ rabs,
                                              const int16_t *row_of) {
  const uint32_t fl = op.y >> 16;
  if (ABS) acc_abs += sqrt(abs2(cmul(c, m)));
  acc.x = fma(c.x, m.x, acc.x);
  acc.y = fma(c.x, m.y, acc.y);
  acc2.x = fma(-c.y, m.y, acc2.x);
  acc2.y = fma(c.y, m.x, acc2.y);
  if (fl & OP_LAST) {
    const uint32_t dest = op.y & 0xFFFFu;
    M[dest] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
    if (ABS && (fl & OP_RHS)) rabs[row_of[dest]] = acc_abs;
    acc = make_double2(0.0, 0.0);
    acc2 = make_double2(0.0, 0.0);
    acc_abs = 0.0;
  }
}

// Op list: M[dest] = sum over the entry's ops of coef[slot] * mono[k].  Ops are processed in blocks
// of 4 whose op records and operands are all loaded before any store of the block (the stores into
// M would otherwise serialise every op behind the previous op's store: the compiler cannot prove
// that M does not alias the op table, both being shared memory).
template <int N, int L, bool ABS>
__device__ __forceinline__ void run_ops(const uint2 *__restrict__ ops_s, int Q, int rhs_off,
                                        const double2 *__restrict__ cval, const double2 *__restrict__ mono,
                                        double2 *__restrict__ M, double *__restrict__ rabs, const int16_t *row_of,
                                        int r) {
  double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
  double acc_abs = 0.0;
  int q = 0;
  for (; q + 4 <= Q; q += 4) {
    uint2 op[4];
    double2 c[4], m[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) op[i] = ops_s[(q + i) * L + r];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[i] = cval[(int)(op[i].x & 0xFFFFu) + (((op[i].y >> 16) & OP_RHS) ? rhs_off : 0)];
      m[i] = mono[op[i].x >> 16];
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) op_accumulate<N, ABS>(op[i], c[i], m[i], acc, acc2, acc_abs, M, rabs, row_of);
  }
  for (; q < Q; ++q) {
    const uint2 o = ops_s[q * L + r];
    const double2 c = cval[(int)(o.x & 0xFFFFu) + (((o.y >> 16) & OP_RHS) ? rhs_off : 0)];
    op_accumulate<N, ABS>(o, c, mono[o.x >> 16], acc, acc2, acc_abs, M, rabs, row_of);
  }
}

// Paired op table (TrackArgs::Qp > 0, abi.cpp pair_ops): a record holds two terms of the same entry
// (x: slot_a | mono_a << 16, y: slot_b | mono_b << 16, z: dest | flags << 16), an odd entry's last
// record pairs its term with the constant-zero monomial.  The record decode, the rhs select and the
// entry-end bookkeeping (store + reset) are paid once per two terms.  Blocks of 2 records (4 terms).
template <int N, int L, bool ABS>
__device__ __forceinline__ void run_ops_pairs(const uint4 *__restrict__ ops4, int Q2, int rhs_off,
                                              const double2 *__restrict__ cval, const double2 *__restrict__ mono,
                                              double2 *__restrict__ M, double *__restrict__ rabs,
                                              const int16_t *row_of, int r) {
  double2 acc = make_double2(0.0, 0.0), acc2 = make_double2(0.0, 0.0);
  double acc_abs = 0.0;
  auto pair_step = [&](uint4 o, double2 ca, double2 ma, double2 cb, double2 mb) {
    if (ABS) {   // (in the single-op order, so the relative residual is bit-identical too)
      acc_abs += sqrt(abs2(cmul(ca, ma)));
      acc_abs += sqrt(abs2(cmul(cb, mb)));
    }
    acc.x = fma(ca.x, ma.x, acc.x);
    acc.y = fma(ca.x, ma.y, acc.y);
    acc2.x = fma(-ca.y, ma.y, acc2.x);
    acc2.y = fma(ca.y, ma.x, acc2.y);
    acc.x = fma(cb.x, mb.x, acc.x);
    acc.y = fma(cb.x, mb.y, acc.y);
    acc2.x = fma(-cb.y, mb.y, acc2.x);
    acc2.y = fma(cb.y, mb.x, acc2.y);
    const uint32_t fl = o.z >> 16;
    if (fl & OP_LAST) {
      const uint32_t dest = o.z & 0xFFFFu;
      M[dest] = make_double2(acc.x + acc2.x, acc.y + acc2.y);
      if (ABS && (fl & OP_RHS)) rabs[row_of[dest]] = acc_abs;
      acc = make_double2(0.0, 0.0);
      acc2 = make_double2(0.0, 0.0);
      acc_abs = 0.0;
    }
  };
  int q = 0;
  for (; q + 2 <= Q2; q += 2) {
    uint4 op[2];
    double2 c[4], m[4];
#pragma unroll
    for (int i = 0; i < 2; ++i) op[i] = ops4[(q + i) * L + r];
#pragma unroll
    for (int i = 0; i < 2; ++i) {
      const int roff = ((op[i].z >> 16) & OP_RHS) ? rhs_off : 0;
      c[2 * i] = cval[(int)(op[i].x & 0xFFFFu) + roff];
      m[2 * i] = mono[op[i].x >> 16];
      c[2 * i + 1] = cval[(int)(op[i].y & 0xFFFFu) + roff];
      m[2 * i + 1] = mono[op[i].y >> 16];
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) pair_step(op[i], c[2 * i], m[2 * i], c[2 * i + 1], m[2 * i + 1]);
  }
  if (q < Q2) {
    const uint4 o = ops4[q * L + r];
    const int roff = ((o.z >> 16) & OP_RHS) ? rhs_off : 0;
    pair_step(o, cval[(int)(o.x & 0xFFFFu) + roff], mono[o.x >> 16], cval[(int)(o.y & 0xFFFFu) + roff], mono[o.y >> 16]);
  }
}

// ------------------------------------------------------------------------------------------
// Coefficient values at t: c_j(t) for every slot and c_j'(t) for the rhs slots (j < nsrc), by
// Horner on the prologue's polynomials coef_t[d][j] (d <= D); two slots per lane per iteration,
// all loads issued before the FMA chains.
// ------------------------------------------------------------------------------------------
template <int D, int L>
__device__ __forceinline__ void horner(const double2 *__restrict__ ct, double t, int ncoef, int nsrc,
                                       double2 *__restrict__ cval, int r) {
  for (int j0 = r; j0 < ncoef; j0 += 2 * L) {
    const int j1 = j0 + L;
    const bool has1 = j1 < ncoef;
    double2 c0[D + 1], c1[D + 1];
#pragma unroll
    for (int d = 0; d <= D; ++d) {
      c0[d] = __ldg(&ct[(size_t)d * ncoef + j0]);
      c1[d] = has1 ? __ldg(&ct[(size_t)d * ncoef + j1]) : make_double2(0.0, 0.0);
    }
    double2 p0 = c0[D], p1 = c1[D], q0 = make_double2(0.0, 0.0), q1 = q0;
#pragma unroll
    for (int d = D - 1; d >= 0; --d) {
      q0 = make_double2(fma(q0.x, t, p0.x), fma(q0.y, t, p0.y));
      q1 = make_double2(fma(q1.x, t, p1.x), fma(q1.y, t, p1.y));
      p0 = make_double2(fma(p0.x, t, c0[d].x), fma(p0.y, t, c0[d].y));
      p1 = make_double2(fma(p1.x, t, c1[d].x), fma(p1.y, t, c1[d].y));
    }
    cval[j0] = p0;
    if (j0 < nsrc) cval[ncoef + j0] = q0;
    if (has1) {
      cval[j1] = p1;
      if (j1 < nsrc) cval[ncoef + j1] = q1;
    }
  }
}

// Coefficient values at a complex t (the Cauchy endgame tracks around |1 - t| = s, reading R26):
// the same Horner recurrences in complex arithmetic, any degree D.
template <int L>
__device__ __forceinline__ void horner_c(const double2 *__restrict__ ct, double2 t, int D, int ncoef, int nsrc,
                                         double2 *__restrict__ cval, int r) {
  for (int j = r; j < ncoef; j += L) {
    double2 p = __ldg(&ct[(size_t)D * ncoef + j]), q = make_double2(0.0, 0.0);
#pragma unroll 1
    for (int d = D - 1; d >= 0; --d) {
      const double2 c = __ldg(&ct[(size_t)d * ncoef + j]);
      q = cfma(q, t, p);   // q = q t + p
      p = cfma(p, t, c);   // p = p t + c
    }
    cval[j] = p;
    if (j < nsrc) cval[ncoef + j] = q;
  }
}

template <typename T>
struct is_complex_t { static constexpr bool value = false; };
template <>
struct is_complex_t<double2> { static constexpr bool value = true; };

// ------------------------------------------------------------------------------------------
// Evaluate [dH/dx | rhs] into the slot's M (shared), then fused LU + solve.  Returns the solution
// component y_r in lane r (r < N) and whether the solve succeeded (uniform over the slot).
// rhs_off = 0 -> rhs = H (coefficients c(t)); rhs_off = ncoef -> rhs = dH/dt (coefficients c'(t)).
// ------------------------------------------------------------------------------------------
template <int N, int L, int NC, typename TT>
__device__ __forceinline__ bool eval_solve(const TrackArgs &A, const uint2 *__restrict__ ops_s,
                                           const uint32_t *__restrict__ prog_s, const int16_t *__restrict__ mpos_s,
                                           const int16_t *__restrict__ row_of, const double2 *__restrict__ ct,
                                           TT t, bool need_coef, int rhs_off, bool want_abs, double2 *cval,
                                           double2 *mono,
                                           double2 *M, double2 *prow, double *rabs, int r, int seg,
                                           const double2 (&xr)[NC],
                                           double2 (&y)[NC], double2 (&fr)[NC], double (&fabs_r)[NC]
#ifdef HCB_PHASE_TIMING
                                           , unsigned long long (&hcb_phase)[8]
#endif
                                           ) {
  const int ncoef = A.ncoef, D = A.D;
  // ---- stage x (monomial slots 0..N-1) and coefficient values c(t) (all slots), c'(t) (rhs
  //      slots) by Horner on the prologue's polynomials in t ----
  HCB_T(c0);
  constexpr int E = TrackerShape<N, L>::E;
  if (r < N) mono[r] = xr[0];
  if constexpr (NC == 2) {
    if (r < E) mono[16 + r] = xr[NC - 1];
  }
  if constexpr (is_complex_t<TT>::value) {
    if (need_coef) horner_c<L>(ct, t, D, ncoef, A.ncoef_src, cval, r);
  } else if (need_coef) switch (D) {   // D is uniform: the common degrees keep all loads of a coefficient in flight together
    case 1: horner<1, L>(ct, t, ncoef, A.ncoef_src, cval, r); break;
    case 2: horner<2, L>(ct, t, ncoef, A.ncoef_src, cval, r); break;
    case 3: horner<3, L>(ct, t, ncoef, A.ncoef_src, cval, r); break;
    default:
      for (int j = r; j < ncoef; j += L) {
        double2 p = __ldg(&ct[(size_t)D * ncoef + j]), q = make_double2(0.0, 0.0);
#pragma unroll 1
        for (int d = D - 1; d >= 0; --d) {
          const double2 c = __ldg(&ct[(size_t)d * ncoef + j]);
          q = make_double2(fma(q.x, t, p.x), fma(q.y, t, p.y));
          p = make_double2(fma(p.x, t, c.x), fma(p.y, t, c.y));
        }
        cval[j] = p;
        if (j < A.ncoef_src) cval[ncoef + j] = q;
      }
  }
  __syncwarp();
  HCB_T(c1);
  HCB_ACC(0, c0, c1);
  // ---- monomial program: degree d products from degree d-1 (shared by all entries) ----
  int lo = N + 1;
  for (int l = 0; l < A.n_levels; ++l) {
    const int hi = A.level_end[l];
    int k = lo + r;
    // batches of 2 items per lane: both items' operands are loaded before either product is stored
    // (the parents come from earlier levels, but the compiler cannot move loads above a store)
    for (; k + L < hi; k += 2 * L) {
      const uint32_t e0 = prog_s[k - (N + 1)], e1 = prog_s[k + L - (N + 1)];
      const double2 a0 = mono[e0 & 0xFFFFu], b0 = mono[e0 >> 16], a1 = mono[e1 & 0xFFFFu], b1 = mono[e1 >> 16];
      mono[k] = cmul(a0, b0);
      mono[k + L] = cmul(a1, b1);
    }
    if (k < hi) {
      const uint32_t e = prog_s[k - (N + 1)];
      mono[k] = cmul(mono[e & 0xFFFFu], mono[e >> 16]);
    }
    lo = hi;
    __syncwarp();
  }
  HCB_T(c2);
  HCB_ACC(1, c1, c2);
  // ---- homogenised term evaluation, lane-balanced op list ----
  if (A.Qp > 0) {   // paired op table (uniform)
    const uint4 *ops4 = reinterpret_cast<const uint4 *>(ops_s);
    if (want_abs) run_ops_pairs<N, L, true>(ops4, A.Qp, rhs_off, cval, mono, M, rabs, row_of, r);
    else run_ops_pairs<N, L, false>(ops4, A.Qp, rhs_off, cval, mono, M, rabs, row_of, r);
  } else if (want_abs) run_ops<N, L, true>(ops_s, A.Q, rhs_off, cval, mono, M, rabs, row_of, r);
  else run_ops<N, L, false>(ops_s, A.Q, rhs_off, cval, mono, M, rabs, row_of, r);
  __syncwarp();
  HCB_T(c3);
  HCB_ACC(2, c2, c3);
  // ---- load row r of [A | b] into registers (structural zeros read the always-zero entry) ----
  if constexpr (NC == 2) {
    // hybrid layout: row r plus the extra rows' columns r and r + 16
    double2 a[N + 1], e[E][2];
    double jmax = 0.0;
#pragma unroll
    for (int j = 0; j <= N; ++j) {
      a[j] = M[mpos_s[r * (N + 1) + j]];
      if (j < N) jmax = fmax(jmax, abs2(a[j]));
    }
#pragma unroll
    for (int q = 0; q < E; ++q)
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        const int col = r + 16 * c;
        e[q][c] = (col <= N) ? M[mpos_s[(16 + q) * (N + 1) + col]] : make_double2(0.0, 0.0);
        if (col < N) jmax = fmax(jmax, abs2(e[q][c]));
      }
    fr[0] = a[N];
    fr[NC - 1] = (r < E) ? M[mpos_s[(16 + (r < E ? r : 0)) * (N + 1) + N]] : make_double2(0.0, 0.0);
    fabs_r[0] = want_abs ? rabs[r] : 0.0;
    fabs_r[NC - 1] = (r < E && want_abs) ? rabs[16 + r] : 0.0;
    HCB_T(c4h);
    HCB_ACC(3, c3, c4h);
    const bool okh = lu_rows_hy<N, E>(a, e, r, seg, prow, A.st.pivot_rel, jmax, y);
    HCB_T(c5h);
    HCB_ACC(4, c4h, c5h);
    return okh;
  }
  double2 a[N + 1];
  const int rr = (r < N) ? r : 0;
  double jmax = 0.0;   // max |A_rj|^2 of this row, for the singularity threshold (R9)
#pragma unroll
  for (int j = 0; j <= N; ++j) {
    a[j] = M[mpos_s[rr * (N + 1) + j]];
    if (j < N) jmax = fmax(jmax, abs2(a[j]));
  }
  if (r >= N) {
    jmax = 0.0;
#pragma unroll
    for (int j = 0; j <= N; ++j) a[j] = make_double2(0.0, 0.0);
  }
  fr[0] = a[N];
  fabs_r[0] = (r < N && want_abs) ? rabs[r] : 0.0;
  HCB_T(c4);
  HCB_ACC(3, c3, c4);
  const bool ok = lu_rows<N, L>(a, r, seg, prow, M, A.st.pivot_rel, jmax, y[0]);
  HCB_T(c5);
  HCB_ACC(4, c4, c5);
  return ok;
}

// ------------------------------------------------------------------------------------------
// The persistent tracker kernel.
// ------------------------------------------------------------------------------------------
template <int N, int LW>
__device__ __forceinline__ void track_body(const TrackArgs &A) {
  constexpr int L = TrackerShape<N, LW>::L;
  constexpr int NC = TrackerShape<N, LW>::NC;   // unknown components per lane (2: hybrid layout)
  constexpr int E = TrackerShape<N, LW>::E;
  constexpr int TPW = 32 / L;
  extern __shared__ __align__(16) unsigned char smem_raw[];

  // ---- stage the op table, the monomial program and the entry map in shared memory (constant for
  //      the kernel) with bulk async copies (TMA engine, 1-D; the device copies are zero-padded to
  //      16-byte multiples by the host), completed on an mbarrier ----
  __shared__ __align__(8) unsigned long long tables_bar;
  uint2 *ops_s = reinterpret_cast<uint2 *>(smem_raw);
  const int nops = A.Q * L;
  const int nprog = A.n_mono - (N + 1);
  uint32_t *prog_s = reinterpret_cast<uint32_t *>(smem_raw + align16((size_t)8 * nops));
  int16_t *mpos_s = reinterpret_cast<int16_t *>(smem_raw + align16((size_t)8 * nops) + align16((size_t)4 * nprog));
  if (threadIdx.x == 0) {
    const unsigned b_ops = (unsigned)align16((size_t)8 * nops), b_prog = (unsigned)align16((size_t)4 * nprog),
                   b_mpos = (unsigned)align16((size_t)2 * N * (N + 1));
    mbar_init(&tables_bar, 1);
    mbar_arrive_expect_tx(&tables_bar, b_ops + b_prog + b_mpos);
    if (b_ops) bulk_copy_g2s(ops_s, A.ops, b_ops, &tables_bar);
    if (b_prog) bulk_copy_g2s(prog_s, A.mono_prog, b_prog, &tables_bar);
    bulk_copy_g2s(mpos_s, A.mpos, b_mpos, &tables_bar);
  }
  unsigned char *slots_base = smem_raw + table_bytes(A.Q, L, nprog, N) + align16((size_t)2 * A.n_entries);
  // compact entry -> row (for the relative residual of rhs entries)
  int16_t *row_of = reinterpret_cast<int16_t *>(smem_raw + table_bytes(A.Q, L, nprog, N));
  for (int i = threadIdx.x; i < N * (N + 1); i += blockDim.x)
    if (A.mpos[i] < A.n_entries) row_of[A.mpos[i]] = (int16_t)(i / (N + 1));

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / L, r = lane % L;
  const int slot = warp * TPW + seg;
  const int ncoef = A.ncoef, D = A.D;
  constexpr bool SS = TrackerShape<N, LW>::SMEM_STATE;
  constexpr int LNC = TrackerShape<N, LW>::LNC;
  unsigned char *sb = slots_base + (size_t)slot * slot_bytes(N, LNC, ncoef, A.ncoef_src, A.n_mono, A.n_entries + 1);
  EgSample *egs = reinterpret_cast<EgSample *>(sb);   // endgame sampling state (R26), lane 0 writes
  double2 *vstate = reinterpret_cast<double2 *>(sb + EG_SAMPLE_BYTES);   // [3][NC][LV] (SS only)
  // one copy of the slot's rarely touched scalars (track id, step size, h, t1, the t of the cached
  // coefficients, step / rejection / Newton / consecutive-accept counters; every lane of the slot
  // reads and writes the same values) -- in shared memory for the 128-register kernels, so their
  // register budget goes to the rows being eliminated (SS only)
  long long *s_g = reinterpret_cast<long long *>(vstate + 3 * LNC);
  double *s_dt = reinterpret_cast<double *>(s_g + 1);   // dt, h, t1, cval_t
  int *s_cnt = reinterpret_cast<int *>(s_dt + 4);       // steps, rej, newt, acc
  double2 *cval = reinterpret_cast<double2 *>(reinterpret_cast<unsigned char *>(vstate) + state_bytes(LNC));
  double2 *mono = cval + ncoef + A.ncoef_src;
  double2 *M = mono + A.n_mono + 1;   // (mono[n_mono]: the constant zero of paired op tables)
  double2 *prow = M + A.n_entries + 1;
  double *rabs = reinterpret_cast<double *>(prow + 2 * (N + 1));
  if (r == 0) {
    mono[N] = make_double2(1.0, 0.0);            // constant-one slot
    mono[A.n_mono] = make_double2(0.0, 0.0);     // constant zero (pad term of paired op tables)
    M[A.n_entries] = make_double2(0.0, 0.0);     // the entry every structural zero reads
  }
  __syncthreads();                   // (the barrier's initialisation is visible to every waiter)
  mbar_wait_parity(&tables_bar, 0);  // the staged tables have landed

  const DevSettings &st = A.st;
  const int n_rk = (st.predictor == HC_EULER) ? 1 : 4;

  // ---- slot state (replicated over the slot's lanes) ----
  int state = ST_DONE;
  long long g_r = -1;
  long long &g = SS ? s_g[0] : g_r;
  g = -1;
  const double2 *ct = A.coef_t;   // instance coefficient table
  double t = 0.0;
  double dt_r = 0.0, h_r = 0.0, t1_r = 0.0, cval_t_r = -1.0;
  int steps_r = 0, rej_r = 0, newt_r = 0, acc_r = 0;
  double &dt = SS ? s_dt[0] : dt_r, &h = SS ? s_dt[1] : h_r, &t1 = SS ? s_dt[2] : t1_r;
  h = t1 = 0.0;
  int &steps = SS ? s_cnt[0] : steps_r, &rej = SS ? s_cnt[1] : rej_r, &newt = SS ? s_cnt[2] : newt_r,
      &acc = SS ? s_cnt[3] : acc_r;
  dt = 0.0;
  acc = steps = rej = newt = 0;
  int stage = 0, it = 0, solves = 0;
  // component c of lane r is unknown r (c = 0) or 16 + r (c = 1, hybrid layout, r < E)
  // x stays in registers; in the 128-register kernels (SS) the RK accumulators and the corrector's
  // point live in the slot's shared memory ([kacc | kprev | xc][NC][L], one conflict-free 16-byte word
  // per lane): they are touched a few times per iteration, and the registers they free keep the
  // N <= 16 kernels within 128
  double2 x[NC], kacc_r[NC], kprev_r[NC], xc_r[NC];
  constexpr int LV = TrackerShape<N, LW>::LV;
  const int vr = (SS && LV < L) ? (r < N ? r : N) : r;   // state lane (lanes without a row share a dummy)
  auto KACC = [&](int c) -> double2 & { return SS ? vstate[(0 * NC + c) * LV + vr] : kacc_r[c]; };
  auto KPREV = [&](int c) -> double2 & { return SS ? vstate[(1 * NC + c) * LV + vr] : kprev_r[c]; };
  auto XC = [&](int c) -> double2 & { return SS ? vstate[(2 * NC + c) * LV + vr] : xc_r[c]; };
#pragma unroll
  for (int c = 0; c < NC; ++c) x[c] = KACC(c) = KPREV(c) = XC(c) = make_double2(0.0, 0.0);
  auto comp_valid = [&](int c) -> bool { return c == 0 ? (r < N) : (r < E); };
  auto comp_row = [&](int c) -> int { return c == 0 ? r : 16 + r; };
  bool need_track = true;
  bool fresh_k1 = false;   // the last solve was a successful RK stage 1 (endgame sampling)
  double &cval_t = SS ? s_dt[3] : cval_t_r;   // t at which the slot's coefficient values were
  cval_t = -1.0;                                        // last evaluated (-1: none)
#ifdef HCB_PHASE_TIMING
  unsigned long long hcb_phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  long long hcb_iter0 = clock64();
  long long hcb_k0 = hcb_iter0;
#endif

  // begin a step attempt from (x, t) with dt; returns false when max_steps is exhausted
  auto begin_step = [&]() -> bool {
    if (steps >= st.max_steps) return false;
    ++steps;
    h = dt;
    t1 = t + dt;
    if (t1 >= 1.0) {
      t1 = 1.0;
      h = 1.0 - t;
    }
    stage = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) KACC(c) = KPREV(c) = make_double2(0.0, 0.0);
    state = ST_RK;
    return true;
  };
  auto finish = [&](int status, double ra, double rr) {
#pragma unroll
    for (int c = 0; c < NC; ++c)
      if (comp_valid(c) && HCB_OUT_EXPERIMENT != 2) A.x_out[(size_t)g * N + comp_row(c)] = x[c];
    if (r == 0 && HCB_OUT_EXPERIMENT != 1) {
      A.status_out[g] = status;
      reinterpret_cast<int4 *>(A.counters_out)[g] = make_int4(steps, rej, newt, solves);
      reinterpret_cast<double2 *>(A.resid_out)[g] = make_double2(ra, rr);
      if (A.winding_out) A.winding_out[g] = 0;
    }
    if (r == 0) {
      // a singular endpoint (reading R26): the Cauchy endgame kernel continues this track from
      // (x, t = 1 - ra) with step rr; the list entry is the track id
      if (status == HC_EG_PENDING) A.eg_list[atomicAdd(A.eg_count, 1ULL)] = g;
    }
    need_track = true;
    state = ST_DONE;
  };

  for (;;) {
    // ---- refill: slots without a track pull the next id (instance-major).  The shuffle runs on
    //      all 32 lanes (warp collectives are never inside slot-divergent branches). ----
    {
      unsigned long long got = 0;
      if (need_track && r == 0) got = atomicAdd(A.queue, 1ULL);
      got = __shfl_sync(FULL, got, seg * L);
      if (need_track) {
        need_track = false;
        if ((long long)got < A.total) {
          g = (long long)got;
          const long long b = g / A.S, s = g % A.S;
          ct = A.coef_t + (size_t)b * (D + 1) * ncoef;
          cval_t = -1.0;   // new instance: coefficient values are stale
#pragma unroll
          for (int c = 0; c < NC; ++c) x[c] = comp_valid(c) ? A.start_x[s * N + comp_row(c)] : make_double2(0.0, 0.0);
          t = 0.0;
          dt = st.dt_init;
          acc = steps = rej = newt = solves = 0;
          if (r == 0) {   // endgame sampling state (read again only after eval_solve's __syncwarp)
            egs->s_next = st.eg_start;
            egs->mu_prev = 0.0;
            egs->xn2 = 0.0;   // (no sample is taken at t = 0: s = 1 > eg_start)
            egs->nsamp = egs->inf_run = egs->sing_run = 0;
          }
          begin_step();
        } else {
          state = ST_DONE;
          ct = A.coef_t;
          g = -1;
        }
      }
    }
    // ---- endgame sampling (reading R26): at the first step start with s = 1 - t <= s_next, right
    //      after the predictor's first stage (k1 = dx/dt = -y), record log ||x||, log s||k1||;
    //      between samples v = dlog||x||/dlog s, mu = dlog(s||dx/dt||)/dlog s.  Three consecutive
    //      converged samples with mu = v < eg_inf_mu (and s <= eg_inf_s or ||x|| >= eg_inf_norm)
    //      -> AT_INFINITY; with 0 < mu < eg_sing_mu -> the Cauchy endgame kernel. ----
    //      (Taken at the top of the iteration after that stage, where fewer values are live; the norms
    //      come from the reductions the solves already did: ||x|| at the last accept, ||k1||.)
    // (no test of st.eg_start here: a loop-invariant branch makes the compiler unswitch the loop,
    // i.e. compile the whole evaluation + elimination twice -- the 4-view kernel 6.1 k -> 9.6 k SASS
    // instructions; with the endgame off s_next = eg_start = 0 and no sample is ever wanted)
    if (HCB_EG_SAMPLING) {
      // s_next was written by the slot's lane 0 at an earlier iteration, before that iteration's
      // evaluation (whose __syncwarps make it visible); xn2 / kn2 are written by lane 0 too, and only
      // lane 0 reads the sampling state below, so the block needs no __syncwarp of its own (a
      // warp-synchronous region here made ptxas compile the evaluation + elimination twice)
      const bool want = fresh_k1 && (1.0 - t) <= egs->s_next;
      fresh_k1 = false;
      int decision = 0;   // 1: at infinity, 2: the Cauchy endgame
      if (__builtin_expect(__any_sync(FULL, want), 0)) {
        if (want && r == 0) {
          EgSample e = *egs;
          const double s = 1.0 - t, xn = sqrt(e.xn2), kn = sqrt(e.kn2);
          // single-precision logarithms, as the oracle (reading R26: decisions against ~1e-2-wide
          // thresholds; the inlined double-precision log cost 4-5 % of the 4-view / 5-point
          // throughput through the hot loop's code, A/B in profiles/r02_ab_eg_sampling.log)
          const double ls = __logf((float)s), lx = __logf((float)xn), ldv = __logf((float)(s * kn));
          if (e.nsamp > 0) {
            const double v = (lx - e.plx) / (ls - e.pls), mu = (ldv - e.pld) / (ls - e.pls);
            const bool stable = e.nsamp > 1 && fabs(mu - e.mu_prev) < st.eg_stab;
            int inf_run = (stable && mu < st.eg_inf_mu && fabs(v - mu) < st.eg_stab) ? e.inf_run + 1 : 0;
            if (s > st.eg_inf_s && xn < st.eg_inf_norm) inf_run = 0;
            const int sing_run = (stable && mu > 0.0 && mu < st.eg_sing_mu) ? e.sing_run + 1 : 0;
            decision = inf_run >= 3 ? 1 : (sing_run >= 3 ? 2 : 0);
            e.mu_prev = mu;
            e.inf_run = inf_run;
            e.sing_run = sing_run;
          }
          e.pls = ls;
          e.plx = lx;
          e.pld = ldv;
          e.nsamp += 1;
          e.s_next = 0.5 * s;
#ifndef HCB_EG_BISECT_NOWRITE
          *egs = e;
#endif
        }
        decision = __shfl_sync(FULL, decision, seg * L);
      }
#ifdef HCB_EG_BISECT_NODECIDE
      decision = 0;
#endif
      // the decision is carried out by the state machine below (one finish() call site): this
      // iteration's evaluation is a dummy for the slot and counts no solve
      if (decision) {
        state = ST_EGFIN;
        stage = decision;
      }
    }

    // (a slot the sampling just finished refills at the next iteration: need_track)
    if (__all_sync(FULL, state == ST_DONE && !need_track)) break;
#ifdef HCB_PHASE_TIMING
    hcb_iter0 = clock64();
    hcb_phase[7] += 1;   // iterations
#endif

    // ---- what this slot evaluates in this iteration ----
    double te;
    double2 xe[NC];
    int rhs_off = 0;
    if (state == ST_RK) {
      const double cs = (stage == 0) ? 0.0 : (stage == 3 ? 1.0 : 0.5);
      te = t + cs * h;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        xe[c] = make_double2(fma(cs * h, KPREV(c).x, x[c].x), fma(cs * h, KPREV(c).y, x[c].y));
      rhs_off = ncoef;  // rhs = dH/dt
    } else if (state == ST_NEWTON) {
      te = t1;
#pragma unroll
      for (int c = 0; c < NC; ++c) xe[c] = XC(c);
    } else if (state == ST_POLISH || state == ST_RESID) {
      te = 1.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) xe[c] = x[c];
    } else {
      te = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) xe[c] = make_double2(0.0, 0.0);
    }
    const bool want_abs = __any_sync(FULL, state == ST_RESID);
    double2 yv[NC], fr[NC];
    double fa[NC];
    // coefficient values depend only on (instance, t): RK stages 2/3 share t + h/2, and stage 4,
    // the Newton iterations and the next step's stage 1 share t + h, so Horner is skipped then
    const bool need_coef = (te != cval_t);
    cval_t = te;
    const bool ok = eval_solve<N, L, NC>(A, ops_s, prog_s, mpos_s, row_of, ct, te, need_coef, rhs_off, want_abs, cval, mono,
                                     M, prow, rabs,
                                     r, seg, xe, yv, fr, fa
#ifdef HCB_PHASE_TIMING
                                     , hcb_phase
#endif
                                     );

#ifdef HCB_PHASE_TIMING
    const long long hcb_e = clock64();
#endif
    // ---- slot-uniform reductions, computed on all lanes before any slot-divergent branch ----
    double2 cand[NC];
    bool fin = true;
    double yd2 = 0.0, cd2 = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double2 base = (state == ST_POLISH) ? x[c] : XC(c);
      cand[c] = make_double2(base.x - yv[c].x, base.y - yv[c].y);   // Newton update x - dx
      fin = fin && cfinite(cand[c]);
      yd2 = nmax(yd2, abs2(yv[c]));
      cd2 = nmax(cd2, abs2(cand[c]));
    }
    const bool cand_fin = seg_all<L>(fin, seg);
    const double d2 = seg_max<L>(NC == 1 ? abs2(yv[0]) : yd2);
    const double c2 = seg_max<L>(NC == 1 ? abs2(cand[0]) : cd2);
    double res_abs = 0.0, res_rel = 0.0;
    if (want_abs) {   // warp-uniform: only when some slot classifies its endpoint
      double fm = 0.0, fq = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) {
        if (!comp_valid(c)) continue;
        const double m = sqrt(abs2(fr[c]));
        fm = nmax(fm, m);
        fq = nmax(fq, fa[c] > 0.0 ? m / fa[c] : (m == 0.0 ? 0.0 : INFINITY));
      }
      res_abs = seg_max<L>(fm);
      res_rel = seg_max<L>(fq);
    }

    // ---- advance the slot's state machine ----
    if (state == ST_DONE) continue;
    if (state != ST_RESID && state != ST_EGFIN) ++solves;
    bool accept = false, reject = false;
    if (state == ST_EGFIN) {   // endgame decision (R26): at infinity, or x, s = 1 - t, dt for the Cauchy kernel
      const bool inf = stage == 1;
      finish(inf ? HC_AT_INFINITY : HC_EG_PENDING, inf ? INFINITY : 1.0 - t, inf ? INFINITY : dt);
    } else if (state == ST_RK) {
      if (!ok) {
        reject = true;
      } else {
        const double w = (stage == 0 || stage == 3) ? 1.0 : 2.0;
        fresh_k1 = stage == 0;   // k1 = dx/dt at the step start: an endgame sample point (R26)
        if (stage == 0 && r == 0) egs->kn2 = d2;   // ||k1||^2 (k1 = -y)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const double2 k = make_double2(-yv[c].x, -yv[c].y);
          KACC(c) = make_double2(fma(w, k.x, KACC(c).x), fma(w, k.y, KACC(c).y));
          KPREV(c) = k;
        }
        if (stage + 1 < n_rk) {
          ++stage;
        } else {
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            if (n_rk == 1) {
              XC(c) = make_double2(fma(h, KPREV(c).x, x[c].x), fma(h, KPREV(c).y, x[c].y));
            } else {
              const double h6 = h / 6.0;
              XC(c) = make_double2(fma(h6, KACC(c).x, x[c].x), fma(h6, KACC(c).y, x[c].y));
            }
          }
          state = ST_NEWTON;
          it = 0;
        }
      }
    } else if (state == ST_NEWTON) {
      ++newt;
      if (!ok || !cand_fin) {
        reject = true;
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) XC(c) = cand[c];
        if (d2 <= st.newton_tol * st.newton_tol * fmax(1.0, c2)) accept = true;
        else if (++it >= st.max_newton) reject = true;
      }
    } else if (state == ST_POLISH) {
      if (!ok) {
        state = ST_RESID;
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) x[c] = cand[c];
        if (!cand_fin) {
          finish(HC_NONFINITE, INFINITY, INFINITY);
        } else if (d2 <= st.end_tol * st.end_tol * fmax(1.0, c2) || ++it >= st.end_newton) {
          state = ST_RESID;
        }
      }
    } else {  // ST_RESID: classify the endpoint (reading R10)
      const int status = (res_abs <= st.res_abs || res_rel <= st.res_rel) ? HC_CONVERGED : HC_SINGULAR;
      finish(status, res_abs, res_rel);
    }
    if (accept) {
#pragma unroll
      for (int c = 0; c < NC; ++c) x[c] = XC(c);
      if (r == 0) egs->xn2 = c2;   // ||x||^2 of the accepted point (endgame samples)
      t = t1;
      if (++acc >= st.grow_after) {
        dt = fmin(dt * st.grow, st.dt_max);
        acc = 0;
      }
      if (c2 > st.inf_norm * st.inf_norm) {   // c2 = ||xc||^2 of the accepted point
        finish(HC_DIVERGED, INFINITY, INFINITY);
      } else if (t >= 1.0) {
        state = ST_POLISH;
        it = 0;
      } else if (!begin_step()) {
        finish(HC_MAX_STEPS, INFINITY, INFINITY);
      }
    } else if (reject) {
      ++rej;
      acc = 0;
      dt *= st.shrink;
      if (dt < st.dt_min) finish(HC_STEP_UNDERFLOW, INFINITY, INFINITY);
      else if (!begin_step()) finish(HC_MAX_STEPS, INFINITY, INFINITY);
    }
#ifdef HCB_PHASE_TIMING
    hcb_phase[5] += (unsigned long long)(clock64() - hcb_e);          // reductions + state machine
    hcb_phase[6] += (unsigned long long)(hcb_e - hcb_iter0);          // whole eval + solve
#endif
  }
#ifdef HCB_PHASE_TIMING
  if ((threadIdx.x & 31) == 0 && A.phase_cycles) {
    for (int i = 0; i < 8; ++i) atomicAdd(&A.phase_cycles[i], hcb_phase[i]);
  }
  (void)hcb_k0;
#endif
}

// Kernel entry point: the register budget comes from __launch_bounds__ (MAXW warps, MINB CTAs per
// SM).  (An explicit __maxnreg__ entry for 13-15 warps at 136-152 registers was tried: the launch
// configuration was rejected on the device.)
template <int N, int LW>
__global__ void __launch_bounds__(TrackerShape<N, LW>::MAXW * 32, TrackerShape<N, LW>::MINB)
    hc_track_kernel(const TrackArgs A) {
  track_body<N, LW>(A);
}

template <int N, int LW = lanes_for(N)>
cudaError_t launch_tracker_n(const TrackArgs &A, int device, cudaStream_t stream, TrackerPlan *plan) {
  constexpr int L = TrackerShape<N, LW>::L;
  constexpr int TPW = 32 / L;
  const size_t tables = table_bytes(A.Q, L, A.n_mono - (N + 1), N) + align16((size_t)2 * A.n_entries);
  const size_t per_warp =
      (size_t)TPW * slot_bytes(N, TrackerShape<N, LW>::LNC, A.ncoef, A.ncoef_src, A.n_mono, A.n_entries + 1);
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int warps = TrackerShape<N, LW>::MAXW;
  if (const char *ev = getenv("HC_TRACKER_WARPS")) {   // experiment override (<= compile-time max)
    const int w = atoi(ev);
    if (w >= 1 && w < warps) warps = w;
  }
  while (warps > 1 && tables + warps * per_warp > (size_t)smem_max) --warps;
  const size_t smem = tables + warps * per_warp;
  if (smem > (size_t)smem_max) return cudaErrorInvalidConfiguration;
  const void *fn = (const void *)hc_track_kernel<N, LW>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, warps * 32, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const long long slots_needed = (A.total + TPW - 1) / TPW;
  long long ctas = (long long)per_sm * sms;
  const long long ctas_needed = (slots_needed + warps - 1) / warps;
  if (ctas_needed < ctas) ctas = ctas_needed;
  if (ctas < 1) ctas = 1;
  if (plan) {
    plan->lanes = L;
    plan->warps_per_cta = warps;
    plan->ctas = (int)ctas;
    plan->smem_bytes = smem;
  }
  hc_track_kernel<N, LW><<<(unsigned)ctas, warps * 32, smem, stream>>>(A);
  return cudaGetLastError();
}

}  // namespace hcb
