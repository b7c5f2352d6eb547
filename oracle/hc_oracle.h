/*
 * hc_oracle.h -- CPU oracle for batched homotopy-continuation path tracking.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load or call this library.  It shares no
 * code, header, table or constant generator with the CUDA path
 * (paper_2112_03444_b200/): it evaluates the polynomial system directly from exponent
 * lists and solves with a textbook LU, following PAPER.md §3 step by step.
 *
 * Complex doubles are passed as interleaved (re, im) double pairs.
 */
#ifndef HC_ORACLE_H
#define HC_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* F(x; p): see hc_inputs/descriptor.py for the layout. */
typedef struct {
  int32_t n, P, nterms, ncoef;
  const int32_t *term_eq;    /* [nterms] */
  const int32_t *term_xexp;  /* [nterms * n] */
  const int32_t *term_coef;  /* [nterms] */
  const int32_t *coef_ptr;   /* [ncoef + 1] */
  const double  *coef_w;     /* [nnz * 2] */
  const int32_t *coef_pexp;  /* [nnz * P] */
} orc_sys;

/* Homotopy H(x, t).
 *   kind 0 (TD):  H = (1 - t) gamma G + t F,  G_i = x_i^{deg_i} - 1       (Eq. 1 P:155-158 + gamma, R1/R2)
 *   kind 1 (PH):  H = F(x; (1 - t) p0 + t p1)                              (P:429 + reading R3)        */
typedef struct {
  int32_t kind;
  const orc_sys *sys;
  const int32_t *deg;   /* TD: [n] */
  double gamma[2];      /* TD */
  const double *p0;     /* PH: [P * 2] */
  const double *p1;     /* PH: [P * 2] */
} orc_homotopy;

typedef struct {
  int32_t predictor;    /* 0 = RK4, 1 = Euler (Eq. 4) */
  double dt_init, dt_min, dt_max;
  int32_t grow_after;
  double grow, shrink;
  int32_t max_newton;
  double newton_tol;
  int32_t max_steps;
  double inf_norm;
  int32_t end_newton;
  double end_tol;
  double res_abs, res_rel;
  double pivot_rel;
  /* endgame (reading R26): 0 < eg_start < 1 enables it (s = 1 - t at which sampling starts) */
  double eg_start;
  double eg_inf_mu;      /* at infinity: converged mu = v < eg_inf_mu (three consecutive samples) */
  double eg_sing_mu;     /* Cauchy endgame: converged 0 < mu < eg_sing_mu (three consecutive samples) */
  double eg_stab;        /* converged: |mu - mu_prev| < eg_stab (and |v - mu| < eg_stab at infinity) */
  double eg_inf_s;       /* at infinity is decided only at s <= eg_inf_s or once ||x||_inf >= eg_inf_norm */
  double eg_inf_norm;
  int32_t eg_samples;    /* Cauchy: sample points per loop around |1 - t| = s */
  int32_t eg_max_winding;
  int32_t eg_max_radii;  /* Cauchy: radii s, s/2, s/4, ... tried */
  double eg_tol;         /* Cauchy: consecutive estimates agree within eg_tol * max(1, |x|) */
} orc_settings;

enum { ORC_CONVERGED = 0, ORC_DIVERGED = 1, ORC_STEP_UNDERFLOW = 2, ORC_MAX_STEPS = 3,
       ORC_SINGULAR = 4, ORC_NONFINITE = 5, ORC_AT_INFINITY = 6 };

void orc_settings_default(orc_settings *s);

/* Direct evaluations (for pins).  All outputs interleaved complex. */
void orc_eval_coefs(const orc_sys *s, const double *p, double *c /*[ncoef*2]*/);
void orc_eval_F(const orc_sys *s, const double *p, const double *x, double *F /*[n*2]*/);
void orc_eval_JF(const orc_sys *s, const double *p, const double *x, double *J /*[n*n*2]*/);
void orc_eval_H(const orc_homotopy *h, const double *x, double t, double *H, double *Hx, double *Ht);

/* Textbook LU with partial pivoting + two triangular solves.  Returns 0, or 1 when singular. */
int orc_lu_solve(int n, const double *A /*[n*n*2] row-major*/, const double *b, double *x, double pivot_rel);

/* Total-degree start solutions (reading R2): roots of unity, k_1 fastest.  Returns prod(deg). */
int64_t orc_td_start(int n, const int32_t *deg, double *x /*[prod*n*2] or NULL*/);

/* Track S start points through H for each of B instances (PH: p1 = p1s + b*P*2; TD: B = 1).
 * Outputs per track g = b*S + s: x[g*n*2], status[g], counters[g*4] = (steps, rejections,
 * newton iterations, linear solves), resid[g*2] = (abs, rel), winding[g] (0: no Cauchy endgame, else
 * the winding number it found; may be NULL).  Multithreaded, deterministic. */
void orc_track(const orc_homotopy *h, const double *p1s, int64_t B,
               const double *start_x, int64_t S, const orc_settings *st, int nthreads,
               double *x_out, int32_t *status, int32_t *counters, double *resid, int32_t *winding);

/* One predictor step from (x, t) with step dt (RK4 or Euler per st->predictor); 0 on success. */
int orc_predict(const orc_homotopy *h, const orc_settings *st, const double *x, double t, double dt, double *xp);
/* Newton at fixed t (Eq. 6), in place; returns 1 converged, 0 not converged, -1 singular. */
/* Endpoint residuals at x, t = 1 (reading R10): r = ||F||_inf, r_rel = max_i |F_i| / sum_k |c_ik||m_k(x)|. */
void orc_endpoint_residual(const orc_homotopy *h, const double *x, double *r, double *r_rel);
int orc_newton(const orc_homotopy *h, const orc_settings *st, double *x, double t, int iters, double tol);

#ifdef __cplusplus
}
#endif
#endif
