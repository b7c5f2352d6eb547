// endgame.cuh -- the Cauchy endgame kernel for sm_100a (reading R26; one template per N).
//
// The tracker hands a track to this kernel (status HC_EG_PENDING, id in eg_list) when its endgame
// samples show a singular endpoint: mu = dlog(s ||dx/dt||)/dlog s has converged to 0 < 1/m < 1
// (s = 1 - t).  Near t = 1 such a path is a Puiseux series in s^{1/m}; the paper only says that
// "extra verification steps are needed".  The endgame (Morgan-Sommese-Wampler's
// Cauchy integral, restated in DESIGN.md R26):
//   at radius s, track x around the circle t(theta) = 1 - s e^{i theta} in K = eg_samples equal
//   arcs per loop (Davidenko in theta: dx/dtheta = dx/dt * dt/dtheta, dt/dtheta = -i s e^{i theta};
//   RK4 predictor, Newton corrector at the complex t, step halving on rejection), summing x at the
//   K arc starts; after each loop test whether x is back at the loop's start point; the loop count
//   at closure is the winding number m; the estimate of x(1) is the mean of the m K samples (the
//   trapezoidal Cauchy integral).  Then move radially (ordinary real-t tracking) to s / 2 and
//   repeat; two consecutive estimates within eg_tol * max(1, |x_i|) end it, and the endpoint is
//   classified by its residuals at t = 1 (R10).  When the loops fail or the estimate is not a root
//   (the circle enclosed other branch points, e.g. of a near-double root: the mean of several roots)
//   the track resumes ordinary tracking (R5-R9, no sampling) from the hand-over point to t = 1 and
//   the R10 polish and classification -- exactly the oracle's order.
// Same evaluation and fused LU as the tracker (eval_solve with a complex t); slots of a warp run
// independent state machines, one eval + solve per slot per loop iteration, and pull work from
// eg_list through a global counter.  Only tracks with singular endpoints ever reach this kernel, so
// it is written for clarity, not speed.
#pragma once

#include "tracker.cuh"

namespace hcb {

enum EgMode : int { EG_ARC = 0, EG_RADIAL = 1, EG_PLAIN = 2, EG_POLISH = 3, EG_RESID = 4, EG_IDLE = 5 };

#ifndef HCB_EG_DEBUG   // experiment builds: a failed Cauchy attempt records its reason in resid[1]
#define HCB_EG_DEBUG 0
#endif

template <int N, int L>
__device__ __forceinline__ void endgame_body(const TrackArgs &A) {
  constexpr int TPW = 32 / L;
  // nothing handed over (the common case): leave before staging the tables (uniform over the grid;
  // the tracker finished before this kernel started, stream order)
  if (*reinterpret_cast<const volatile unsigned long long *>(A.eg_count) == 0ULL) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint2 *ops_s = reinterpret_cast<uint2 *>(smem_raw);
  const int nops = A.Q * L;
  for (int i = threadIdx.x; i < nops; i += blockDim.x) ops_s[i] = __ldg(&A.ops[i]);
  const int nprog = A.n_mono - (N + 1);
  uint32_t *prog_s = reinterpret_cast<uint32_t *>(smem_raw + align16((size_t)8 * nops));
  for (int i = threadIdx.x; i < nprog; i += blockDim.x) prog_s[i] = __ldg(&A.mono_prog[i]);
  int16_t *mpos_s = reinterpret_cast<int16_t *>(smem_raw + align16((size_t)8 * nops) + align16((size_t)4 * nprog));
  for (int i = threadIdx.x; i < N * (N + 1); i += blockDim.x) mpos_s[i] = __ldg(&A.mpos[i]);
  unsigned char *slots_base = smem_raw + table_bytes(A.Q, L, nprog, N) + align16((size_t)2 * A.n_entries);
  int16_t *row_of = reinterpret_cast<int16_t *>(smem_raw + table_bytes(A.Q, L, nprog, N));
  for (int i = threadIdx.x; i < N * (N + 1); i += blockDim.x)
    if (A.mpos[i] < A.n_entries) row_of[A.mpos[i]] = (int16_t)(i / (N + 1));

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int seg = lane / L, r = lane % L;
  const int slot = warp * TPW + seg;
  const int ncoef = A.ncoef, D = A.D;
  unsigned char *sb = slots_base + (size_t)slot * slot_bytes(N, L, ncoef, A.ncoef_src, A.n_mono, A.n_entries + 1);
  // (the tracker's per-lane state area is unused here)
  double2 *cval = reinterpret_cast<double2 *>(sb + EG_SAMPLE_BYTES + state_bytes(L));
  double2 *mono = cval + ncoef + A.ncoef_src;
  double2 *M = mono + A.n_mono + 1;   // (mono[n_mono]: the constant zero of paired op tables)
  double2 *prow = M + A.n_entries + 1;
  double *rabs = reinterpret_cast<double *>(prow + 2 * (N + 1));
  if (r == 0) {
    mono[N] = make_double2(1.0, 0.0);
    mono[A.n_mono] = make_double2(0.0, 0.0);
    M[A.n_entries] = make_double2(0.0, 0.0);
  }
  __syncthreads();

  const DevSettings &st = A.st;
  const int n_rk = (st.predictor == HC_EULER) ? 1 : 4;
  const int K = st.eg_samples;
  const double two_pi = 6.283185307179586476925286766559;
  const unsigned long long n_items = A.eg_count[0];

  // ---- slot state (replicated over the slot's lanes) ----
  int mode = EG_IDLE, phase = 0, stage = 0, it = 0, acc = 0;
  long long g = -1;
  const double2 *ct = A.coef_t;
  int steps = 0, rej = 0, newt = 0, solves = 0;
  double s = 0.0, th = 0.0, th_end = 0.0, h = 0.0, hh = 0.0, tn = 0.0;   // circle
  double tr = 0.0, t_end = 0.0, dtr = 0.0, hr = 0.0, t1 = 0.0;            // radial / plain
  double s_h = 0.0, dt_h = 0.0;                                           // hand-over point
  int arc = 0, loops = 0, radius = 0, m = 0;
  bool have_est = false, need_track = true, cauchy_est = false;
  double dbg_where = 0.0;
  double2 x = make_double2(0.0, 0.0), xr = x, sum = x, est = x, kacc = x, kprev = x, xc = x, xh = x;
  const bool valid = r < N;
  double2 cval_t = make_double2(-1.0, 0.0);   // t of the slot's cached coefficient values

  auto circ = [&](double theta) { double sn, cs; sincos(theta, &sn, &cs); return make_double2(cs, sn); };
  int dbg = 0;
  auto done = [&](int status, double ra, double rr, int wind) {
    if (valid) A.x_out[(size_t)g * N + r] = x;
    if (r == 0) {
      A.status_out[g] = status;
      reinterpret_cast<int4 *>(A.counters_out)[g] = make_int4(steps, rej, newt, solves);
      if (HCB_EG_DEBUG) {   // (failure reason, radius * 100 + loops at the failure, s there)
        ra = dbg;
        rr = dbg_where;
      }
      reinterpret_cast<double2 *>(A.resid_out)[g] = make_double2(ra, rr);
      if (A.winding_out) A.winding_out[g] = wind;
    }
    need_track = true;
    mode = EG_IDLE;
  };
  // real-t step attempt (radial move or plain tracking) from tr towards t_end with dtr
  auto begin_real_step = [&]() -> bool {
    if (steps >= st.max_steps) return false;
    ++steps;
    hr = dtr;
    t1 = tr + dtr;
    if (t1 >= t_end) {
      t1 = t_end;
      hr = t_end - tr;
    }
    phase = 0;
    stage = 0;
    kacc = kprev = make_double2(0.0, 0.0);
    return true;
  };
  // the Cauchy endgame failed (or its estimate is not a root): resume plain tracking from the
  // hand-over point to t = 1 (R5-R9), then polish and classify
  auto fallback = [&](int why) {
    dbg = why;
    dbg_where = radius * 100 + loops + 1e-3 * arc;
    x = xh;
    tr = 1.0 - s_h;
    t_end = 1.0;
    dtr = dt_h;
    acc = 0;
    cauchy_est = false;
    mode = EG_PLAIN;
    if (!begin_real_step()) done(HC_MAX_STEPS, INFINITY, INFINITY, 0);
  };
  auto begin_arc_step = [&]() -> bool {
    if (steps >= st.max_steps) return false;
    ++steps;
    hh = h;
    tn = th + h;
    if (tn >= th_end) {
      tn = th_end;
      hh = th_end - th;
    }
    phase = 0;
    stage = 0;
    kacc = kprev = make_double2(0.0, 0.0);
    return true;
  };
  auto begin_arc = [&]() -> bool {   // arc `arc` of the current loop: sample, then track it
    sum = make_double2(sum.x + x.x, sum.y + x.y);
    th = two_pi * arc / K;
    th_end = two_pi * (arc + 1) / K;
    h = th_end - th;
    mode = EG_ARC;
    return begin_arc_step();
  };
  auto begin_radius = [&]() -> bool {   // Cauchy loops at the current radius s
    xr = x;
    sum = make_double2(0.0, 0.0);
    loops = 0;
    arc = 0;
    return begin_arc();
  };

  for (;;) {
    {
      unsigned long long got = 0;
      if (need_track && r == 0) got = atomicAdd(A.eg_count + 1, 1ULL);
      got = __shfl_sync(FULL, got, seg * L);
      if (need_track) {
        need_track = false;
        if (got < n_items) {
          g = A.eg_list[got];
          const long long b = g / A.S;
          ct = A.coef_t + (size_t)b * (D + 1) * ncoef;
          cval_t = make_double2(-1.0, 0.0);
          x = valid ? A.x_out[(size_t)g * N + r] : make_double2(0.0, 0.0);
          xh = x;
          const int4 c0 = reinterpret_cast<const int4 *>(A.counters_out)[g];
          steps = c0.x;
          rej = c0.y;
          newt = c0.z;
          solves = c0.w;
          const double2 sd = reinterpret_cast<const double2 *>(A.resid_out)[g];   // (s = 1 - t, dt) at hand-over
          s = s_h = sd.x;
          dt_h = sd.y;
          radius = 0;
          have_est = false;
          m = 0;
          dbg = 0;
          if (!begin_radius()) fallback(5);
        } else {
          mode = EG_IDLE;
          g = -1;
        }
      }
    }
    if (__all_sync(FULL, mode == EG_IDLE && !need_track)) break;

    // ---- what this slot evaluates: te (complex), the point, and the rhs ----
    double2 te = make_double2(1.0, 0.0), xe = x, dtdth = make_double2(0.0, 0.0);
    int rhs_off = 0;
    if (mode == EG_ARC) {
      if (phase == 0) {
        const double cs = (stage == 0) ? 0.0 : (stage == 3 ? 1.0 : 0.5);
        const double2 e = circ(th + cs * hh);
        te = make_double2(1.0 - s * e.x, -s * e.y);
        dtdth = make_double2(s * e.y, -s * e.x);   // -i s e^{i theta}
        xe = make_double2(fma(cs * hh, kprev.x, x.x), fma(cs * hh, kprev.y, x.y));
        rhs_off = ncoef;
      } else {
        const double2 e = circ(tn);
        te = make_double2(1.0 - s * e.x, -s * e.y);
        xe = xc;
      }
    } else if (mode == EG_RADIAL || mode == EG_PLAIN) {
      if (phase == 0) {
        const double cs = (stage == 0) ? 0.0 : (stage == 3 ? 1.0 : 0.5);
        te = make_double2(tr + cs * hr, 0.0);
        dtdth = make_double2(1.0, 0.0);
        xe = make_double2(fma(cs * hr, kprev.x, x.x), fma(cs * hr, kprev.y, x.y));
        rhs_off = ncoef;
      } else {
        te = make_double2(t1, 0.0);
        xe = xc;
      }
    } else if (mode == EG_POLISH) {
      te = make_double2(1.0, 0.0);
      xe = xc;
    } else if (mode == EG_RESID) {
      te = make_double2(1.0, 0.0);
      xe = x;
    }
    const bool want_abs = __any_sync(FULL, mode == EG_RESID);
    const bool need_coef = te.x != cval_t.x || te.y != cval_t.y;
    cval_t = te;
    double2 xa[1] = {xe}, yv[1], fr[1];
    double fa[1];
#ifdef HCB_PHASE_TIMING
    unsigned long long hcb_phase[8] = {0, 0, 0, 0, 0, 0, 0, 0};   // (the phase build times the tracker only)
#endif
    const bool ok = eval_solve<N, L, 1>(A, ops_s, prog_s, mpos_s, row_of, ct, te, need_coef, rhs_off, want_abs, cval,
                                        mono, M, prow, rabs, r, seg, xa, yv, fr, fa
#ifdef HCB_PHASE_TIMING
                                        , hcb_phase
#endif
                                        );
    const double2 y = yv[0];

    // ---- slot-uniform reductions (all lanes, before any slot-divergent branch) ----
    const double2 cand = make_double2(xc.x - y.x, xc.y - y.y);   // Newton update
    const bool cand_fin = seg_all<L>(!valid || cfinite(cand), seg);
    const double d2 = seg_max<L>(valid ? abs2(y) : 0.0);
    const double c2 = seg_max<L>(valid ? abs2(cand) : 0.0);
    // loop closure: the accepted point vs the loop's start point
    const double dcl = seg_max<L>(valid ? abs2(make_double2(cand.x - xr.x, cand.y - xr.y)) : 0.0);
    const double xr2 = seg_max<L>(valid ? abs2(xr) : 0.0);
    // the estimate if this accept closes a loop, and its agreement with the previous radius
    const double2 enew = make_double2(sum.x / ((loops + 1) * K), sum.y / ((loops + 1) * K));
    const double em = sqrt(abs2(enew));
    const bool agree =
        seg_all<L>(!valid || sqrt(abs2(make_double2(enew.x - est.x, enew.y - est.y))) <= st.eg_tol * fmax(1.0, em), seg);
    const bool x_fin = seg_all<L>(!valid || cfinite(x), seg);
    double res_abs = 0.0, res_rel = 0.0;
    if (want_abs) {
      const double mg = valid ? sqrt(abs2(fr[0])) : 0.0;
      res_abs = seg_max<L>(mg);
      res_rel = seg_max<L>(valid ? (fa[0] > 0.0 ? mg / fa[0] : (mg == 0.0 ? 0.0 : INFINITY)) : 0.0);
    }

    // ---- advance the slot's state machine ----
    if (mode == EG_IDLE) continue;
    if (mode == EG_RESID) {
      const bool conv = res_abs <= st.res_abs || res_rel <= st.res_rel;
      if (cauchy_est) {   // the Cauchy estimate: a root, or back to plain tracking
        if (x_fin && conv) done(HC_CONVERGED, res_abs, res_rel, m);
        else fallback(6);
      } else if (!x_fin) {
        done(HC_NONFINITE, INFINITY, INFINITY, 0);
      } else {
        done(conv ? HC_CONVERGED : HC_SINGULAR, res_abs, res_rel, 0);
      }
      continue;
    }
    ++solves;
    if (mode == EG_POLISH) {   // R10 polish at t = 1 (as the tracker's ST_POLISH)
      if (!ok) {
        mode = EG_RESID;
      } else {
        x = xc = cand;
        if (!cand_fin) done(HC_NONFINITE, INFINITY, INFINITY, 0);
        else if (d2 <= st.end_tol * st.end_tol * fmax(1.0, c2) || ++it >= st.end_newton) mode = EG_RESID;
      }
      continue;
    }
    bool accept = false, reject = false;
    const double hstep = (mode == EG_ARC) ? hh : hr;
    if (phase == 0) {   // RK stage: k = (dx/dt) (dt/dtau) = -y dt/dtau
      if (!ok) {
        reject = true;
      } else {
        const double w = (stage == 0 || stage == 3) ? 1.0 : 2.0;
        const double2 k = cmul(make_double2(-y.x, -y.y), dtdth);
        kacc = make_double2(fma(w, k.x, kacc.x), fma(w, k.y, kacc.y));
        kprev = k;
        if (stage + 1 < n_rk) {
          ++stage;
        } else {
          if (n_rk == 1) xc = make_double2(fma(hstep, kprev.x, x.x), fma(hstep, kprev.y, x.y));
          else xc = make_double2(fma(hstep / 6.0, kacc.x, x.x), fma(hstep / 6.0, kacc.y, x.y));
          phase = 1;
          it = 0;
        }
      }
    } else {   // Newton at the step's end point
      ++newt;
      if (!ok || !cand_fin) {
        reject = true;
      } else {
        xc = cand;
        if (d2 <= st.newton_tol * st.newton_tol * fmax(1.0, c2)) accept = true;
        else if (++it >= st.max_newton) reject = true;
      }
    }
    if (accept) {
      x = xc;
      if (mode == EG_ARC) {
        th = tn;
        if (th < th_end) {
          if (!begin_arc_step()) fallback(1);
        } else if (++arc < K) {
          if (!begin_arc()) fallback(1);
        } else {   // a loop is complete
          ++loops;
          arc = 0;
          if (dcl <= 1e-12 * fmax(1.0, xr2)) {   // |x - xr|_inf <= 1e-6 max(1, |xr|_inf): closed
            x = xr;
            m = loops;
            if (have_est && agree) {
              x = enew;   // the endpoint estimate: classified at t = 1
              cauchy_est = true;
              mode = EG_RESID;
            } else {
              est = enew;
              have_est = true;
              if (radius + 1 < st.eg_max_radii) {   // radial move to s / 2
                tr = 1.0 - s;
                t_end = 1.0 - 0.5 * s;
                dtr = t_end - tr;
                mode = EG_RADIAL;
                if (!begin_real_step()) fallback(1);
              } else {
                fallback(3);
              }
            }
          } else if (loops < st.eg_max_winding) {
            if (!begin_arc()) fallback(1);
          } else {
            fallback(2);
          }
        }
      } else {   // radial move or plain tracking
        tr = t1;
        if (mode == EG_PLAIN) {
          if (++acc >= st.grow_after) {
            dtr = fmin(dtr * st.grow, st.dt_max);
            acc = 0;
          }
          if (c2 > st.inf_norm * st.inf_norm) {
            done(HC_DIVERGED, INFINITY, INFINITY, 0);
          } else if (tr >= 1.0) {
            xc = x;
            it = 0;
            mode = EG_POLISH;
          } else if (!begin_real_step()) {
            done(HC_MAX_STEPS, INFINITY, INFINITY, 0);
          }
        } else if (tr < t_end) {
          if (!begin_real_step()) fallback(1);
        } else {
          s *= 0.5;
          ++radius;
          if (!begin_radius()) fallback(1);
        }
      }
    } else if (reject) {
      ++rej;
      if (mode == EG_ARC) {
        h *= st.shrink;
        if (h < st.dt_min) fallback(4);
        else if (!begin_arc_step()) fallback(1);
      } else if (mode == EG_PLAIN) {
        acc = 0;
        dtr *= st.shrink;
        if (dtr < st.dt_min) done(HC_STEP_UNDERFLOW, INFINITY, INFINITY, 0);
        else if (!begin_real_step()) done(HC_MAX_STEPS, INFINITY, INFINITY, 0);
      } else {
        dtr *= st.shrink;
        if (dtr < st.dt_min) fallback(7);
        else if (!begin_real_step()) fallback(1);
      }
    }
  }
}

template <int N, int LW>
__global__ void __launch_bounds__(128) hc_endgame_kernel(const TrackArgs A) {
  endgame_body<N, LW>(A);
}

// Launch over the tracks the tracker handed over (the count is read on the device: no host sync).
// 4 warps per CTA, one CTA per SM (persistent), shared memory as in the tracker.  LW = 32 (N <= 16):
// the wide latency layout, one track per warp -- the few handed-over tracks are a latency chain.
template <int N, int LW = lanes_for(N)>
cudaError_t launch_endgame_n(const TrackArgs &A, int device, cudaStream_t stream) {
  constexpr int L = LW;
  constexpr int TPW = 32 / L;
  const size_t tables = table_bytes(A.Q, L, A.n_mono - (N + 1), N) + align16((size_t)2 * A.n_entries);
  const size_t per_warp = (size_t)TPW * slot_bytes(N, L, A.ncoef, A.ncoef_src, A.n_mono, A.n_entries + 1);
  int smem_max = 0;
  cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  int warps = 4;
  while (warps > 1 && tables + warps * per_warp > (size_t)smem_max) --warps;
  const size_t smem = tables + warps * per_warp;
  if (smem > (size_t)smem_max) return cudaErrorInvalidConfiguration;
  const void *fn = (const void *)hc_endgame_kernel<N, LW>;
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  hc_endgame_kernel<N, LW><<<(unsigned)sms, warps * 32, smem, stream>>>(A);
  return cudaGetLastError();
}

}  // namespace hcb
