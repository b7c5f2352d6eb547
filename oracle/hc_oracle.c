/*
 * hc_oracle.c -- plain, slow, obviously-correct CPU oracle for HC path tracking.
 *
 * TEST INFRASTRUCTURE ONLY (see hc_oracle.h): only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may use it.  It shares no code with the
 * CUDA path.  Each function cites the passage of PAPER.md (P:line) or the SURVEY.md §8(c)
 * reading (R#) it follows.
 *
 * Pinned by tests/test_oracle_*.py against: closed forms (x(t)=1+t path, Newton on x^2-4,
 * roots of unity), library routines (numpy.linalg.solve, numpy.roots), finite differences,
 * textbook root counts (katsura-n = 2^n, cyclic-5/6/7 = 70/156/924), the paper's counts
 * (4-view = 296, Table 2) and planted ground truth.
 */
#include "hc_oracle.h"

#include <complex.h>
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef double complex cplx;

static cplx ld(const double *a, int64_t i) { return a[2 * i] + I * a[2 * i + 1]; }
static void st(double *a, int64_t i, cplx v) { a[2 * i] = creal(v); a[2 * i + 1] = cimag(v); }

static cplx cpow_int(cplx z, int e) {
  cplx r = 1.0;
  for (int k = 0; k < e; k++) r *= z;   /* powers by repeated multiplication */
  return r;
}

void orc_settings_default(orc_settings *s) {
  /* SURVEY.md §8(c) readings R5-R10 (paper silent; S:217 for the shape of the policy). */
  s->predictor = 0;
  s->dt_init = 0.01;
  s->dt_min = 1e-14;
  s->dt_max = 0.1;
  s->grow_after = 4;
  s->grow = 2.0;
  s->shrink = 0.5;
  s->max_newton = 3;
  s->newton_tol = 1e-8;
  s->max_steps = 10000;
  s->inf_norm = 1e14;
  s->end_newton = 3;
  s->end_tol = 1e-12;
  s->res_abs = 1e-10;
  s->res_rel = 1e-12;
  s->pivot_rel = 1e-14;
  /* endgame: reading R26 (the paper: "extra verification steps are needed") */
  s->eg_start = 0.1;
  s->eg_inf_mu = -0.05;
  s->eg_sing_mu = 0.75;
  s->eg_stab = 0.02;
  s->eg_inf_s = 1e-12;
  s->eg_inf_norm = 1e5;
  s->eg_samples = 16;
  s->eg_max_winding = 8;
  s->eg_max_radii = 12;
  s->eg_tol = 1e-10;
}

/* ---------------------------------------------------------------------------------------
 * Direct evaluation of F(x; p), its x-Jacobian, and coefficient derivatives.
 * c_j(p) = sum_m w_m prod_q p_q^{e_mq}; F_i = sum_{k in eq i} c_{coef(k)} prod_v x_v^{e_kv}.
 * --------------------------------------------------------------------------------------- */

static cplx coef_value(const orc_sys *s, int j, const cplx *p) {
  cplx c = 0;
  for (int m = s->coef_ptr[j]; m < s->coef_ptr[j + 1]; m++) {
    cplx v = ld(s->coef_w, m);
    for (int q = 0; q < s->P; q++) v *= cpow_int(p[q], s->coef_pexp[(int64_t)m * s->P + q]);
    c += v;
  }
  return c;
}

/* d/ds c_j(p + s dp) at s = 0 = sum_m w_m sum_q e_mq p_q^{e_mq-1} dp_q prod_{q' != q} p_q'^{e} */
static cplx coef_dir_deriv(const orc_sys *s, int j, const cplx *p, const cplx *dp) {
  cplx c = 0;
  for (int m = s->coef_ptr[j]; m < s->coef_ptr[j + 1]; m++) {
    const int32_t *e = s->coef_pexp + (int64_t)m * s->P;
    for (int q = 0; q < s->P; q++) {
      if (e[q] == 0) continue;
      cplx v = ld(s->coef_w, m) * (double)e[q] * cpow_int(p[q], e[q] - 1) * dp[q];
      for (int r = 0; r < s->P; r++)
        if (r != q) v *= cpow_int(p[r], e[r]);
      c += v;
    }
  }
  return c;
}

static cplx monomial(const orc_sys *s, int k, const cplx *x) {
  cplx m = 1.0;
  for (int v = 0; v < s->n; v++) m *= cpow_int(x[v], s->term_xexp[(int64_t)k * s->n + v]);
  return m;
}

/* d/dx_v of the monomial of term k (exponent decrement). */
static cplx monomial_dx(const orc_sys *s, int k, const cplx *x, int v) {
  int e = s->term_xexp[(int64_t)k * s->n + v];
  if (e == 0) return 0;
  cplx m = (double)e;
  for (int u = 0; u < s->n; u++) {
    int eu = s->term_xexp[(int64_t)k * s->n + u];
    m *= cpow_int(x[u], u == v ? eu - 1 : eu);
  }
  return m;
}

/* F(x) with given coefficient values c[ncoef] */
static void F_from_coefs(const orc_sys *s, const cplx *c, const cplx *x, cplx *F) {
  for (int i = 0; i < s->n; i++) F[i] = 0;
  for (int k = 0; k < s->nterms; k++) F[s->term_eq[k]] += c[s->term_coef[k]] * monomial(s, k, x);
}

/* J_F(x)[i][v] with given coefficient values */
static void JF_from_coefs(const orc_sys *s, const cplx *c, const cplx *x, cplx *J) {
  int n = s->n;
  for (int i = 0; i < n * n; i++) J[i] = 0;
  for (int k = 0; k < s->nterms; k++)
    for (int v = 0; v < n; v++)
      J[s->term_eq[k] * n + v] += c[s->term_coef[k]] * monomial_dx(s, k, x, v);
}

static void load_vec(const double *a, int n, cplx *out) {
  for (int i = 0; i < n; i++) out[i] = ld(a, i);
}

void orc_eval_coefs(const orc_sys *s, const double *p, double *c) {
  cplx *pp = malloc(sizeof(cplx) * (s->P + 1));
  load_vec(p, s->P, pp);
  for (int j = 0; j < s->ncoef; j++) st(c, j, coef_value(s, j, pp));
  free(pp);
}

void orc_eval_F(const orc_sys *s, const double *p, const double *x, double *F) {
  cplx *pp = malloc(sizeof(cplx) * (s->P + 1)), *c = malloc(sizeof(cplx) * s->ncoef);
  cplx *xx = malloc(sizeof(cplx) * s->n), *FF = malloc(sizeof(cplx) * s->n);
  load_vec(p, s->P, pp);
  load_vec(x, s->n, xx);
  for (int j = 0; j < s->ncoef; j++) c[j] = coef_value(s, j, pp);
  F_from_coefs(s, c, xx, FF);
  for (int i = 0; i < s->n; i++) st(F, i, FF[i]);
  free(pp); free(c); free(xx); free(FF);
}

void orc_eval_JF(const orc_sys *s, const double *p, const double *x, double *J) {
  int n = s->n;
  cplx *pp = malloc(sizeof(cplx) * (s->P + 1)), *c = malloc(sizeof(cplx) * s->ncoef);
  cplx *xx = malloc(sizeof(cplx) * n), *JJ = malloc(sizeof(cplx) * n * n);
  load_vec(p, s->P, pp);
  load_vec(x, n, xx);
  for (int j = 0; j < s->ncoef; j++) c[j] = coef_value(s, j, pp);
  JF_from_coefs(s, c, xx, JJ);
  for (int i = 0; i < n * n; i++) st(J, i, JJ[i]);
  free(pp); free(c); free(xx); free(JJ);
}

/* ---------------------------------------------------------------------------------------
 * The homotopy (Eq. 1; gamma trick R1; parameter homotopy R3) and its derivatives
 * ∂H/∂x (Eq. 3) and ∂H/∂t.
 * --------------------------------------------------------------------------------------- */

typedef struct {
  const orc_homotopy *h;
  const double *p1;      /* this instance's target parameters (PH) */
  cplx *c_t;             /* coefficient values at the current t [ncoef] */
  cplx *dc_t;            /* d/dt of coefficient values [ncoef] */
  cplx *c_one;           /* coefficient values at t = 1 (target) [ncoef] */
  cplx *p_t, *dp;        /* scratch [P] */
  cplx *F, *G, *J;       /* scratch */
  cplx t_cached;
  int cached;
} hctx;

/* t may be complex (the Cauchy endgame, R26, tracks around |1 - t| = s); p(t) and c(p(t)) are
 * polynomials, so the same formulas hold. */
static void ctx_coefs(hctx *cx, cplx t) {
  const orc_sys *s = cx->h->sys;
  if (cx->cached && cx->t_cached == t) return;
  if (cx->h->kind == 1) {
    for (int q = 0; q < s->P; q++) {
      cplx a = ld(cx->h->p0, q), b = ld(cx->p1, q);
      cx->p_t[q] = (1.0 - t) * a + t * b;   /* p(t) = (1-t) p0 + t p1 (R3) */
      cx->dp[q] = b - a;
    }
    for (int j = 0; j < s->ncoef; j++) {
      cx->c_t[j] = coef_value(s, j, cx->p_t);
      cx->dc_t[j] = coef_dir_deriv(s, j, cx->p_t, cx->dp);
    }
  } else {
    /* TD target: constant coefficients (parameters unused) */
    for (int j = 0; j < s->ncoef; j++) {
      cx->c_t[j] = coef_value(s, j, cx->p_t);
      cx->dc_t[j] = 0;
    }
  }
  cx->t_cached = t;
  cx->cached = 1;
}

/* H, ∂H/∂x, ∂H/∂t at (x, t); any output may be NULL. */
static void eval_H(hctx *cx, const cplx *x, cplx t, cplx *H, cplx *Hx, cplx *Ht) {
  const orc_homotopy *h = cx->h;
  const orc_sys *s = h->sys;
  int n = s->n;
  ctx_coefs(cx, t);
  if (h->kind == 1) {
    if (H) F_from_coefs(s, cx->c_t, x, H);
    if (Hx) JF_from_coefs(s, cx->c_t, x, Hx);
    if (Ht) F_from_coefs(s, cx->dc_t, x, Ht);  /* ∂H/∂t = sum_k (dc_k/dt) m_k(x) */
    return;
  }
  cplx gam = h->gamma[0] + I * h->gamma[1];
  F_from_coefs(s, cx->c_t, x, cx->F);
  for (int i = 0; i < n; i++) cx->G[i] = cpow_int(x[i], h->deg[i]) - 1.0;   /* G_i = x_i^{d_i} - 1 */
  if (H)
    for (int i = 0; i < n; i++) H[i] = (1.0 - t) * gam * cx->G[i] + t * cx->F[i];
  if (Ht)
    for (int i = 0; i < n; i++) Ht[i] = cx->F[i] - gam * cx->G[i];
  if (Hx) {
    JF_from_coefs(s, cx->c_t, x, cx->J);
    for (int i = 0; i < n; i++)
      for (int v = 0; v < n; v++) {
        cplx g = (i == v) ? (double)h->deg[i] * cpow_int(x[i], h->deg[i] - 1) : 0.0;
        Hx[i * n + v] = (1.0 - t) * gam * g + t * cx->J[i * n + v];
      }
  }
}

static int ctx_init(hctx *cx, const orc_homotopy *h, const double *p1) {
  const orc_sys *s = h->sys;
  int n = s->n, P = s->P > 0 ? s->P : 1;
  memset(cx, 0, sizeof(*cx));
  cx->h = h;
  cx->p1 = p1;
  cx->c_t = calloc(s->ncoef + 1, sizeof(cplx));
  cx->dc_t = calloc(s->ncoef + 1, sizeof(cplx));
  cx->c_one = calloc(s->ncoef + 1, sizeof(cplx));
  cx->p_t = calloc(P, sizeof(cplx));
  cx->dp = calloc(P, sizeof(cplx));
  cx->F = calloc(n, sizeof(cplx));
  cx->G = calloc(n, sizeof(cplx));
  cx->J = calloc(n * n, sizeof(cplx));
  return 0;
}

static void ctx_free(hctx *cx) {
  free(cx->c_t); free(cx->dc_t); free(cx->c_one); free(cx->p_t); free(cx->dp);
  free(cx->F); free(cx->G); free(cx->J);
}

void orc_eval_H(const orc_homotopy *h, const double *x, double t, double *H, double *Hx, double *Ht) {
  hctx cx;
  int n = h->sys->n;
  ctx_init(&cx, h, h->p1);
  cplx *xx = malloc(sizeof(cplx) * n), *a = malloc(sizeof(cplx) * n), *b = malloc(sizeof(cplx) * n * n),
       *c = malloc(sizeof(cplx) * n);
  load_vec(x, n, xx);
  eval_H(&cx, xx, t, a, b, c);
  for (int i = 0; i < n; i++) {
    if (H) st(H, i, a[i]);
    if (Ht) st(Ht, i, c[i]);
  }
  if (Hx)
    for (int i = 0; i < n * n; i++) st(Hx, i, b[i]);
  free(xx); free(a); free(b); free(c);
  ctx_free(&cx);
}

/* ---------------------------------------------------------------------------------------
 * Linear solve: "an LU factorization with partial pivoting followed by two triangular
 * solves".  Pivot = max |a| (R13; ties -> lowest row); singular when
 * |pivot| <= pivot_rel * max |A_ij| (R9).  Works on a copy of A and b.
 * --------------------------------------------------------------------------------------- */
static int lu_solve(int n, const cplx *A_in, const cplx *b_in, cplx *x, double pivot_rel) {
  cplx *A = malloc(sizeof(cplx) * n * n), *y = malloc(sizeof(cplx) * n);
  int *perm = malloc(sizeof(int) * n);
  double amax = 0;
  int singular = 0;
  memcpy(A, A_in, sizeof(cplx) * n * n);
  for (int i = 0; i < n * n; i++) {
    double a = cabs(A[i]);
    if (!isfinite(a)) singular = 1;
    if (a > amax) amax = a;
  }
  for (int i = 0; i < n; i++) perm[i] = i;
  /* factor: P A = L U, L unit lower (stored below diagonal), U upper */
  for (int k = 0; k < n && !singular; k++) {
    int piv = k;
    double best = cabs(A[k * n + k]);
    for (int i = k + 1; i < n; i++) {
      double a = cabs(A[i * n + k]);
      if (a > best) { best = a; piv = i; }
    }
    if (!(best > pivot_rel * amax)) { singular = 1; break; }
    if (piv != k) {
      for (int j = 0; j < n; j++) { cplx tmp = A[k * n + j]; A[k * n + j] = A[piv * n + j]; A[piv * n + j] = tmp; }
      int tp = perm[k]; perm[k] = perm[piv]; perm[piv] = tp;
    }
    for (int i = k + 1; i < n; i++) {
      cplx l = A[i * n + k] / A[k * n + k];
      A[i * n + k] = l;
      for (int j = k + 1; j < n; j++) A[i * n + j] -= l * A[k * n + j];
    }
  }
  if (!singular) {
    /* L y = P b */
    for (int i = 0; i < n; i++) {
      cplx v = b_in[perm[i]];
      for (int j = 0; j < i; j++) v -= A[i * n + j] * y[j];
      y[i] = v;
    }
    /* U x = y */
    for (int i = n - 1; i >= 0; i--) {
      cplx v = y[i];
      for (int j = i + 1; j < n; j++) v -= A[i * n + j] * x[j];
      x[i] = v / A[i * n + i];
    }
    for (int i = 0; i < n; i++)
      if (!isfinite(creal(x[i])) || !isfinite(cimag(x[i]))) singular = 1;
  }
  free(A); free(y); free(perm);
  return singular;
}

int orc_lu_solve(int n, const double *A, const double *b, double *x, double pivot_rel) {
  cplx *AA = malloc(sizeof(cplx) * n * n), *bb = malloc(sizeof(cplx) * n), *xx = malloc(sizeof(cplx) * n);
  load_vec(A, n * n, AA);
  load_vec(b, n, bb);
  int r = lu_solve(n, AA, bb, xx, pivot_rel);
  for (int i = 0; i < n; i++) st(x, i, r ? NAN : xx[i]);
  free(AA); free(bb); free(xx);
  return r;
}

/* ---------------------------------------------------------------------------------------
 * Start solutions of G_i = x_i^{d_i} - 1 (reading R2): x_i = exp(2 pi i k_i / d_i), k_1 fastest.
 * --------------------------------------------------------------------------------------- */
int64_t orc_td_start(int n, const int32_t *deg, double *x) {
  int64_t total = 1;
  for (int i = 0; i < n; i++) total *= deg[i];
  if (!x) return total;
  for (int64_t g = 0; g < total; g++) {
    int64_t r = g;
    for (int i = 0; i < n; i++) {
      int k = (int)(r % deg[i]);
      r /= deg[i];
      double s, c;
      /* exact quarter turns: sincospi-style reduction of 2k/d */
      double a = 2.0 * k / deg[i];   /* angle / pi in [0, 2) */
      if (a == 0.0) { c = 1; s = 0; }
      else if (a == 0.5) { c = 0; s = 1; }
      else if (a == 1.0) { c = -1; s = 0; }
      else if (a == 1.5) { c = 0; s = -1; }
      else { c = cos(M_PI * a); s = sin(M_PI * a); }
      x[2 * (g * n + i)] = c;
      x[2 * (g * n + i) + 1] = s;
    }
  }
  return total;
}

/* ---------------------------------------------------------------------------------------
 * Path tracking: predictor (Eq. 3-4; RK4 P:175, reading R5), Newton corrector
 * (Eq. 5-6, reading R6), step policy (R7), termination (R8, R9), endpoint (R10).
 * --------------------------------------------------------------------------------------- */

static double vec_norm_inf(int n, const cplx *v) {
  double m = 0;
  for (int i = 0; i < n; i++) {
    double a = cabs(v[i]);
    if (!(a <= m)) m = a;   /* propagates NaN */
  }
  return m;
}

static int all_finite(int n, const cplx *v) {
  for (int i = 0; i < n; i++)
    if (!isfinite(creal(v[i])) || !isfinite(cimag(v[i]))) return 0;
  return 1;
}

typedef struct {
  hctx cx;
  const orc_settings *st;
  int n;
  cplx *Hx, *rhs, *k1, *k2, *k3, *k4, *xs, *dx, *H;
  int32_t solves;
} tracker;

/* dx/dt = -(∂H/∂x)^{-1} ∂H/∂t  (Eq. 3).  Returns 0 on success. */
static int davidenko(tracker *T, const cplx *x, cplx t, cplx *dxdt) {
  int n = T->n;
  eval_H(&T->cx, x, t, NULL, T->Hx, T->rhs);
  T->solves++;
  if (lu_solve(n, T->Hx, T->rhs, dxdt, T->st->pivot_rel)) return 1;
  for (int i = 0; i < n; i++) dxdt[i] = -dxdt[i];
  return 0;
}

/* RK4 or Euler (Eq. 4): x* from (x, t) with step h, given k1 = dx/dt at (x, t) in T->k1.
 * Returns 0 on success. */
static int predict_from_k1(tracker *T, const cplx *x, double t, double h, cplx *xp) {
  int n = T->n;
  if (T->st->predictor == 1) {
    for (int i = 0; i < n; i++) xp[i] = x[i] + h * T->k1[i];
    return 0;
  }
  for (int i = 0; i < n; i++) T->xs[i] = x[i] + 0.5 * h * T->k1[i];
  if (davidenko(T, T->xs, t + 0.5 * h, T->k2)) return 1;
  for (int i = 0; i < n; i++) T->xs[i] = x[i] + 0.5 * h * T->k2[i];
  if (davidenko(T, T->xs, t + 0.5 * h, T->k3)) return 1;
  for (int i = 0; i < n; i++) T->xs[i] = x[i] + h * T->k3[i];
  if (davidenko(T, T->xs, t + h, T->k4)) return 1;
  for (int i = 0; i < n; i++)
    xp[i] = x[i] + (h / 6.0) * (T->k1[i] + 2.0 * T->k2[i] + 2.0 * T->k3[i] + T->k4[i]);
  return 0;
}

/* RK4 or Euler (Eq. 4): x* from (x, t) with step h.  Returns 0 on success. */
static int predict(tracker *T, const cplx *x, double t, double h, cplx *xp) {
  if (davidenko(T, x, t, T->k1)) return 1;
  return predict_from_k1(T, x, t, h, xp);
}

/* Newton (Eq. 6): x <- x - (∂H/∂x)^{-1} H at fixed t, <= iters iterations, converged when
 * ||Δ||_inf <= tol * max(1, ||x||_inf).  Returns 1 if converged. */
static int newton(tracker *T, cplx *x, cplx t, int iters, double tol, int32_t *count, int *singular) {
  int n = T->n;
  *singular = 0;
  for (int it = 0; it < iters; it++) {
    eval_H(&T->cx, x, t, T->H, T->Hx, NULL);
    T->solves++;
    (*count)++;
    if (lu_solve(n, T->Hx, T->H, T->dx, T->st->pivot_rel)) { *singular = 1; return 0; }
    for (int i = 0; i < n; i++) x[i] -= T->dx[i];
    if (!all_finite(n, x)) { *singular = 1; return 0; }
    double xn = vec_norm_inf(n, x);
    if (vec_norm_inf(n, T->dx) <= tol * (xn > 1.0 ? xn : 1.0)) return 1;
  }
  return 0;
}

/* Endpoint residuals at t = 1 (reading R10): r = ||F||_inf and
 * r_rel = max_i |F_i| / sum_{k in eq i} |c_k| |m_k(x)| (TD: target F alone). */
static void endpoint_residual(tracker *T, const cplx *x, double *r, double *r_rel) {
  const orc_sys *s = T->cx.h->sys;
  int n = s->n;
  ctx_coefs(&T->cx, 1.0);
  cplx *F = calloc(n, sizeof(cplx));
  double *den = calloc(n, sizeof(double));
  for (int k = 0; k < s->nterms; k++) {
    cplx c = T->cx.c_t[s->term_coef[k]], m = monomial(s, k, x);
    F[s->term_eq[k]] += c * m;
    den[s->term_eq[k]] += cabs(c) * cabs(m);
  }
  double ra = 0, rr = 0;
  for (int i = 0; i < n; i++) {
    double a = cabs(F[i]);
    double q = den[i] > 0 ? a / den[i] : (a == 0 ? 0 : INFINITY);
    if (!(a <= ra)) ra = a;
    if (!(q <= rr)) rr = q;
  }
  *r = ra;
  *r_rel = rr;
  free(F); free(den);
}

/* ---------------------------------------------------------------------------------------
 * Endgame (reading R26).  The paper tracks to t = 1 and notes that "the cardinality of the output
 * is not always correct, and extra verification steps are needed"; a path that ends
 * at a singular root or at infinity makes the step size collapse near t = 1.  Standard HC
 * endgames (Morgan, Sommese and Wampler's Cauchy endgame) handle both; this is the plain form:
 *
 *  sampling: with s = 1 - t, once s <= eg_start, the first step attempt at s <= s_next records,
 *    right after the predictor's first stage (k1 = dx/dt at that point, so no extra solve),
 *    log ||x||_inf and log (s ||dx/dt||_inf), and s_next = s / 2.  Between consecutive samples
 *    v  = d log ||x|| / d log s          (x ~ s^v: v < 0 means ||x|| grows as s -> 0)
 *    mu = d log (s ||dx/dt||) / d log s  (x = x* + c s^{1/m}: mu -> 1/m; x ~ s^{-q/m}: mu -> -q/m)
 *  An estimate is "stable" when mu changed by less than eg_stab since the previous sample (the
 *  Puiseux regime has been reached: before it a path may look divergent and turn back).
 *  at infinity: stable, mu < eg_inf_mu and |v - mu| < eg_stab (||x|| ~ s^mu) at three
 *               consecutive samples                                              -> AT_INFINITY;
 *  singular:    stable and 0 < mu < eg_sing_mu at three consecutive samples     -> Cauchy endgame;
 *  otherwise the path is tracked to t = 1 as before (a non-singular endpoint has mu -> 1).
 *
 *  Cauchy endgame at radius s: x is tracked around the circle t(theta) = 1 - s e^{i theta}
 *    (Davidenko in theta: dx/dtheta = dx/dt * dt/dtheta, dt/dtheta = -i s e^{i theta}) in
 *    eg_samples equal arcs per loop; the loop is repeated until x returns to its start (the
 *    winding number m = loops, <= eg_max_winding); the endpoint estimate is the mean of the
 *    m * eg_samples samples (the trapezoidal rule for the Cauchy integral
 *    x(1) = (1 / 2 pi m) int_0^{2 pi m} x(theta) dtheta, exact for the Puiseux terms below order
 *    m * eg_samples).  The path then moves radially to s / 2 (ordinary tracking in real t) and the
 *    loop is repeated; the endgame succeeds when two consecutive estimates agree within
 *    eg_tol * max(1, ||x||_inf), and the endpoint is classified by its residuals (R10).
 * --------------------------------------------------------------------------------------- */

/* One RK4 (or Euler) step along the circle t(theta) = 1 - s e^{i theta} from theta to theta + h. */
static int predict_circle(tracker *T, const cplx *x, double s, double th, double h, cplx *xp) {
  int n = T->n;
  cplx *k[4] = {T->k1, T->k2, T->k3, T->k4};
  const double cst[4] = {0.0, 0.5, 0.5, 1.0};
  int stages = T->st->predictor == 1 ? 1 : 4;
  for (int q = 0; q < stages; q++) {
    double thq = th + cst[q] * h;
    cplx tq = 1.0 - s * cexp(I * thq), dtdth = -I * s * cexp(I * thq);
    for (int i = 0; i < n; i++) T->xs[i] = q == 0 ? x[i] : x[i] + cst[q] * h * k[q - 1][i];
    if (davidenko(T, T->xs, tq, k[q])) return 1;
    for (int i = 0; i < n; i++) k[q][i] *= dtdth;
  }
  for (int i = 0; i < n; i++)
    xp[i] = stages == 1 ? x[i] + h * k[0][i]
                        : x[i] + (h / 6.0) * (k[0][i] + 2.0 * k[1][i] + 2.0 * k[2][i] + k[3][i]);
  return 0;
}

typedef struct { int32_t steps, rej, newt; } eg_ctr;

/* Track x along the circle of radius s from theta0 to theta1 (landing exactly on theta1) with
 * the corrector at every step and the step policy R7 in theta.  Returns 0 on success. */
static int circle_arc(tracker *T, cplx *x, double s, double th0, double th1, eg_ctr *c) {
  const orc_settings *st = T->st;
  int n = T->n, sing;
  cplx *xp = malloc(sizeof(cplx) * n);
  double th = th0, h = th1 - th0;
  int fail = 0;
  while (th < th1) {
    if (c->steps >= st->max_steps) { fail = 1; break; }
    c->steps++;
    double hh = h, tn = th + h;
    if (tn >= th1) { tn = th1; hh = th1 - th; }
    int ok = predict_circle(T, x, s, th, hh, xp) == 0;
    if (ok) ok = newton(T, xp, 1.0 - s * cexp(I * tn), st->max_newton, st->newton_tol, &c->newt, &sing);
    if (ok) {
      memcpy(x, xp, sizeof(cplx) * n);
      th = tn;
    } else {
      c->rej++;
      h *= st->shrink;
      if (h < st->dt_min) { fail = 1; break; }
    }
  }
  free(xp);
  return fail;
}

/* Ordinary tracking in real t from t0 to t1 < 1 (the radial move between Cauchy radii). */
static int radial(tracker *T, cplx *x, double t0, double t1, eg_ctr *c) {
  const orc_settings *st = T->st;
  int n = T->n, sing;
  cplx *xp = malloc(sizeof(cplx) * n);
  double t = t0, dt = t1 - t0;
  int fail = 0;
  while (t < t1) {
    if (c->steps >= st->max_steps) { fail = 1; break; }
    c->steps++;
    double h = dt, tn = t + dt;
    if (tn >= t1) { tn = t1; h = t1 - t; }
    int ok = predict(T, x, t, h, xp) == 0;
    if (ok) ok = newton(T, xp, tn, st->max_newton, st->newton_tol, &c->newt, &sing);
    if (ok) {
      memcpy(x, xp, sizeof(cplx) * n);
      t = tn;
    } else {
      c->rej++;
      dt *= st->shrink;
      if (dt < st->dt_min) { fail = 1; break; }
    }
  }
  free(xp);
  return fail;
}

/* Cauchy endgame from x at t = 1 - s (real).  On success x holds the endpoint estimate and *m the
 * winding number; returns 0.  On failure x holds the last tracked point; returns 1. */
static int cauchy_endgame(tracker *T, cplx *x, double s, eg_ctr *c, int *m) {
  const orc_settings *st = T->st;
  int n = T->n, K = st->eg_samples;
  cplx *xr = malloc(sizeof(cplx) * n), *sum = malloc(sizeof(cplx) * n), *est = malloc(sizeof(cplx) * n);
  int have_est = 0, fail = 1;
  for (int r = 0; r < st->eg_max_radii; r++) {
    memcpy(xr, x, sizeof(cplx) * n);
    for (int i = 0; i < n; i++) sum[i] = 0;
    int loops = 0, closed = 0, arc_fail = 0;
    while (loops < st->eg_max_winding && !closed && !arc_fail) {
      for (int j = 0; j < K && !arc_fail; j++) {
        for (int i = 0; i < n; i++) sum[i] += x[i];   /* sample at theta = 2 pi j / K of this loop */
        arc_fail = circle_arc(T, x, s, 2.0 * M_PI * j / K, 2.0 * M_PI * (j + 1) / K, c);
      }
      loops++;
      if (!arc_fail) {
        double dmax = 0, xm = vec_norm_inf(n, xr);
        for (int i = 0; i < n; i++) {
          double d = cabs(x[i] - xr[i]);
          if (!(d <= dmax)) dmax = d;
        }
        closed = dmax <= 1e-6 * (xm > 1.0 ? xm : 1.0);   /* back on the starting branch */
      }
    }
    if (arc_fail || !closed) break;
    /* the loop ended where it started: continue from the exact start point (the closed loop only
     * adds tracking error) */
    memcpy(x, xr, sizeof(cplx) * n);
    double scale = 0;
    int agree = have_est;
    for (int i = 0; i < n; i++) {
      cplx e = sum[i] / (double)(loops * K);
      if (have_est) {
        double em = cabs(e);
        if (!(cabs(e - est[i]) <= st->eg_tol * (em > 1.0 ? em : 1.0))) agree = 0;
      }
      est[i] = e;
      if (cabs(e) > scale) scale = cabs(e);
    }
    have_est = 1;
    *m = loops;
    if (agree) { fail = 0; break; }
    if (r + 1 < st->eg_max_radii && radial(T, x, 1.0 - s, 1.0 - 0.5 * s, c)) break;
    s *= 0.5;
    (void)scale;
  }
  if (!fail) memcpy(x, est, sizeof(cplx) * n);
  free(xr); free(sum); free(est);
  return fail;
}

/* Ordinary tracking (R5-R9, no endgame sampling) from (x, *t) with step *dt to t = 1; returns -1 when
 * t = 1 was reached (the caller polishes and classifies), else the terminal status. */
static int resume_plain(tracker *T, cplx *x, double *tp, double *dtp, int32_t *steps, int32_t *rej, int32_t *newt) {
  const orc_settings *st = T->st;
  int n = T->n, sing, stat = -1, acc = 0;
  double t = *tp, dt = *dtp;
  cplx *xp = malloc(sizeof(cplx) * n);
  while (t < 1.0) {
    if (*steps >= st->max_steps) { stat = ORC_MAX_STEPS; break; }
    (*steps)++;
    double h = dt, t1 = t + dt;
    if (t1 >= 1.0) { t1 = 1.0; h = 1.0 - t; }
    int ok = predict(T, x, t, h, xp) == 0;
    if (ok) ok = newton(T, xp, t1, st->max_newton, st->newton_tol, newt, &sing);
    if (ok) {
      memcpy(x, xp, sizeof(cplx) * n);
      t = t1;
      if (++acc >= st->grow_after) { dt = dt * st->grow; if (dt > st->dt_max) dt = st->dt_max; acc = 0; }
      if (vec_norm_inf(n, x) > st->inf_norm) { stat = ORC_DIVERGED; break; }
    } else {
      (*rej)++;
      acc = 0;
      dt *= st->shrink;
      if (dt < st->dt_min) { stat = ORC_STEP_UNDERFLOW; break; }
    }
  }
  free(xp);
  *tp = t;
  *dtp = dt;
  return stat;
}

static void track_one(tracker *T, const cplx *x0, cplx *x_out, int32_t *status, int32_t *ctr, double *resid,
                      int32_t *winding) {
  const orc_settings *st = T->st;
  int n = T->n;
  cplx *x = malloc(sizeof(cplx) * n), *xp = malloc(sizeof(cplx) * n);
  memcpy(x, x0, sizeof(cplx) * n);
  double t = 0.0, dt = st->dt_init;
  int32_t steps = 0, rej = 0, newt = 0, acc = 0;
  int stat = -1, sing, wind = 0;
  /* endgame sampling state (R26) */
  const int eg_on = st->eg_start > 0.0 && st->eg_start < 1.0;
  double s_next = st->eg_start, pls = 0, plx = 0, pld = 0, mu_prev = 0;
  int nsamp = 0, cauchy = 0, inf_run = 0, sing_run = 0;
  T->solves = 0;
  while (t < 1.0) {
    if (steps >= st->max_steps) { stat = ORC_MAX_STEPS; break; }
    steps++;
    double h = dt, t1 = t + dt;
    if (t1 >= 1.0) { t1 = 1.0; h = 1.0 - t; }
    /* predictor stage 1: k1 = dx/dt at (x, t) */
    int ok = davidenko(T, x, t, T->k1) == 0;
    if (eg_on && ok && 1.0 - t <= s_next) {
      /* endgame sample at s = 1 - t with k1 = dx/dt at (x, t); the logarithms are taken in single
       * precision (reading R26: the decisions compare slopes of log-log samples against thresholds
       * of width ~1e-2, eg_stab / eg_inf_mu / eg_sing_mu, so 1e-7 suffices; the CUDA path takes the
       * same decisions from single-precision logarithms) */
      double s = 1.0 - t, ls = logf((float)s), lx = logf((float)vec_norm_inf(n, x)),
             ldv = logf((float)(s * vec_norm_inf(n, T->k1)));
      if (nsamp > 0) {
        double v = (lx - plx) / (ls - pls), mu = (ldv - pld) / (ls - pls);
        int stable = nsamp > 1 && fabs(mu - mu_prev) < st->eg_stab;
        /* at infinity: ||x|| ~ s^v with v = mu < eg_inf_mu, converged (R26) */
        inf_run = (stable && mu < st->eg_inf_mu && fabs(v - mu) < st->eg_stab) ? inf_run + 1 : 0;
        if (s > st->eg_inf_s && exp(lx) < st->eg_inf_norm) inf_run = 0;   /* see eg_inf_s, eg_inf_norm */
        /* finite singular endpoint: mu -> 1/m, 0 < 1/m < eg_sing_mu, converged */
        sing_run = (stable && mu > 0.0 && mu < st->eg_sing_mu) ? sing_run + 1 : 0;
        if (inf_run >= 3) { stat = ORC_AT_INFINITY; break; }
        if (sing_run >= 3) { cauchy = 1; break; }
        mu_prev = mu;
      }
      pls = ls; plx = lx; pld = ldv;
      nsamp++;
      s_next = 0.5 * s;
    }
    if (ok) ok = predict_from_k1(T, x, t, h, xp) == 0;
    if (ok) ok = newton(T, xp, t1, st->max_newton, st->newton_tol, &newt, &sing);
    if (ok) {
      memcpy(x, xp, sizeof(cplx) * n);
      t = t1;
      if (++acc >= st->grow_after) { dt = dt * st->grow; if (dt > st->dt_max) dt = st->dt_max; acc = 0; }
      if (vec_norm_inf(n, x) > st->inf_norm) { stat = ORC_DIVERGED; break; }
    } else {
      rej++;
      acc = 0;
      dt *= st->shrink;
      if (dt < st->dt_min) { stat = ORC_STEP_UNDERFLOW; break; }
    }
  }
  double r = INFINITY, r_rel = INFINITY;
  if (cauchy) {
    /* the step attempt that took the sample is abandoned after its first stage */
    eg_ctr c = {steps, rej, newt};
    int m = 0;
    cplx *xh = malloc(sizeof(cplx) * n);
    memcpy(xh, x, sizeof(cplx) * n);
    int fail = cauchy_endgame(T, x, 1.0 - t, &c, &m);
    steps = c.steps; rej = c.rej; newt = c.newt;
    if (!fail && all_finite(n, x)) {
      endpoint_residual(T, x, &r, &r_rel);
      if (r <= st->res_abs || r_rel <= st->res_rel) { stat = ORC_CONVERGED; wind = m; }
      else fail = 1;
    } else {
      fail = 1;
    }
    if (fail) {
      /* the loops enclosed other branch points (e.g. a near-double root: the estimate is the mean of
       * several roots) or failed: resume ordinary tracking from the hand-over point, without
       * endgame sampling (R26) */
      memcpy(x, xh, sizeof(cplx) * n);
      free(xh);
      r = r_rel = INFINITY;
      cauchy = 0;
      stat = resume_plain(T, x, &t, &dt, &steps, &rej, &newt);
    } else {
      free(xh);
    }
  }
  if (cauchy) {
    /* done above */
  } else if (stat < 0) {
    /* endpoint polish on F(.; p1) = H(., 1) */
    int32_t pol = 0;
    newton(T, x, 1.0, st->end_newton, st->end_tol, &pol, &sing);
    if (!all_finite(n, x)) stat = ORC_NONFINITE;
    else {
      endpoint_residual(T, x, &r, &r_rel);
      if (r <= st->res_abs || r_rel <= st->res_rel) stat = ORC_CONVERGED;
      else stat = ORC_SINGULAR;
    }
  }
  memcpy(x_out, x, sizeof(cplx) * n);
  *status = stat;
  ctr[0] = steps; ctr[1] = rej; ctr[2] = newt; ctr[3] = T->solves;
  resid[0] = r; resid[1] = r_rel;
  if (winding) *winding = wind;
  free(x); free(xp);
}

static void tracker_init(tracker *T, const orc_homotopy *h, const double *p1, const orc_settings *st) {
  int n = h->sys->n;
  memset(T, 0, sizeof(*T));
  ctx_init(&T->cx, h, p1);
  T->st = st;
  T->n = n;
  T->Hx = malloc(sizeof(cplx) * n * n);
  T->rhs = malloc(sizeof(cplx) * n); T->k1 = malloc(sizeof(cplx) * n); T->k2 = malloc(sizeof(cplx) * n);
  T->k3 = malloc(sizeof(cplx) * n); T->k4 = malloc(sizeof(cplx) * n); T->xs = malloc(sizeof(cplx) * n);
  T->dx = malloc(sizeof(cplx) * n); T->H = malloc(sizeof(cplx) * n);
}

static void tracker_free(tracker *T) {
  free(T->Hx); free(T->rhs); free(T->k1); free(T->k2); free(T->k3); free(T->k4); free(T->xs);
  free(T->dx); free(T->H);
  ctx_free(&T->cx);
}

typedef struct {
  const orc_homotopy *h;
  const double *p1s;
  int64_t B, S;
  const double *start_x;
  const orc_settings *st;
  double *x_out;
  int32_t *status, *counters;
  double *resid;
  int32_t *winding;
  int64_t next;   /* dynamic chunking over track ids */
} job;

static void *worker(void *arg) {
  job *J = arg;
  int n = J->h->sys->n;
  int P = J->h->sys->P;
  cplx *x0 = malloc(sizeof(cplx) * n), *xo = malloc(sizeof(cplx) * n);
  int64_t total = J->B * J->S, cur_b = -1;
  tracker T;
  int have = 0;
  for (;;) {
    int64_t g = __atomic_fetch_add(&J->next, 1, __ATOMIC_RELAXED);
    if (g >= total) break;
    int64_t b = g / J->S, s = g % J->S;
    if (b != cur_b) {
      if (have) tracker_free(&T);
      tracker_init(&T, J->h, J->h->kind == 1 ? J->p1s + 2 * b * P : NULL, J->st);
      have = 1;
      cur_b = b;
    }
    load_vec(J->start_x + 2 * s * n, n, x0);
    track_one(&T, x0, xo, J->status + g, J->counters + 4 * g, J->resid + 2 * g, J->winding ? J->winding + g : NULL);
    for (int i = 0; i < n; i++) st(J->x_out, g * n + i, xo[i]);
  }
  if (have) tracker_free(&T);
  free(x0); free(xo);
  return NULL;
}

void orc_track(const orc_homotopy *h, const double *p1s, int64_t B, const double *start_x, int64_t S,
               const orc_settings *st, int nthreads, double *x_out, int32_t *status, int32_t *counters,
               double *resid, int32_t *winding) {
  job J = {h, p1s, B, S, start_x, st, x_out, status, counters, resid, winding, 0};
  if (nthreads < 1) nthreads = 1;
  if (nthreads == 1) { worker(&J); return; }
  pthread_t *th = malloc(sizeof(pthread_t) * nthreads);
  for (int i = 0; i < nthreads; i++) pthread_create(&th[i], NULL, worker, &J);
  for (int i = 0; i < nthreads; i++) pthread_join(th[i], NULL);
  free(th);
}

/* ---------------------------------------------------------------------------------------
 * Single-step entry points for pins: one predictor step and Newton at fixed t.
 * --------------------------------------------------------------------------------------- */
int orc_predict(const orc_homotopy *h, const orc_settings *cfg, const double *x, double t, double dt, double *xp) {
  tracker T;
  int n = h->sys->n;
  tracker_init(&T, h, h->p1, cfg);
  cplx *xx = malloc(sizeof(cplx) * n), *yy = malloc(sizeof(cplx) * n);
  load_vec(x, n, xx);
  int r = predict(&T, xx, t, dt, yy);
  for (int i = 0; i < n; i++) st(xp, i, yy[i]);
  free(xx); free(yy);
  tracker_free(&T);
  return r;
}

/* The endpoint residuals of reading R10 at x (t = 1) -- the same endpoint_residual() the tracker
 * classifies with; exported so the pins can check r and r_rel against hand-computed values. */
void orc_endpoint_residual(const orc_homotopy *h, const double *x, double *r, double *r_rel) {
  tracker T;
  orc_settings cfg;
  int n = h->sys->n;
  orc_settings_default(&cfg);
  tracker_init(&T, h, h->p1, &cfg);
  cplx *xx = malloc(sizeof(cplx) * n);
  load_vec(x, n, xx);
  endpoint_residual(&T, xx, r, r_rel);
  free(xx);
  tracker_free(&T);
}

int orc_newton(const orc_homotopy *h, const orc_settings *cfg, double *x, double t, int iters, double tol) {
  tracker T;
  int n = h->sys->n, sing;
  int32_t count = 0;
  tracker_init(&T, h, h->p1, cfg);
  cplx *xx = malloc(sizeof(cplx) * n);
  load_vec(x, n, xx);
  int conv = newton(&T, xx, t, iters, tol, &count, &sing);
  for (int i = 0; i < n; i++) st(x, i, xx[i]);
  free(xx);
  tracker_free(&T);
  return sing ? -1 : conv;
}
