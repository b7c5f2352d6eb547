/*
 * hc.h -- C ABI of the B200-native batched homotopy-continuation path tracker.
 *
 * Method: GPU-HC (Chien et al., arXiv 2112.03444; /root/reference/PAPER.md, cited "P:<line>").
 * For every start solution x0 of a start system and every problem instance, track the
 * solution path x(t) of H(x, t) = 0 from t = 0 to t = 1 (Eq. 1) with a
 * Runge-Kutta predictor on the Davidenko ODE  (dH/dx) dx/dt = -dH/dt  (Eq. 3, P:166-169;
 * RK4 P:175) and a Newton corrector (Eq. 5-6), adaptive step control, and
 * endpoint classification; complex FP64 throughout, N <= 32 unknowns.
 *
 * Homotopies: every homotopy is a parameter homotopy H(x,t) = F(x; (1-t) p0 + t p1)
 * ("coefficients ... are linear interpolation of corresponding elements in the start and
 * target systems").  A total-degree homotopy with the gamma
 * trick, H = (1-t) gamma G + t F with G_i = x_i^{d_i} - 1, is expressed in that form by
 * hc_system_create_total_degree + hc_total_degree_params (SURVEY.md §8(b) convention).
 *
 * Conventions
 *  - extern "C"; no C++ exception crosses this boundary; every call returns hc_status.
 *  - hc_complex is layout-compatible with std::complex<double>, cuDoubleComplex and
 *    torch.complex128 (interleaved re, im).
 *  - Errors: argument/shape errors return HC_E_INVALID_ARG (N not in [1,32], null pointers,
 *    non-finite coefficients, inconsistent sizes); unsupported sizes HC_E_TOO_LARGE; CUDA
 *    failures HC_E_CUDA; allocation failures HC_E_OOM.  hc_last_error() returns a
 *    thread-local message for the last failing call.  A per-track numerical failure is
 *    never an error: it is reported in the track's status ("the batch call never fails
 *    wholesale").
 *  - Device memory: the library allocates its per-batch buffers stream-ordered from its own memory
 *    pool per device (release threshold 4 GiB, so back-to-back batches reuse it); temporaries are
 *    released in stream order when the batch's kernels are enqueued, result-owned outputs by
 *    hc_result_destroy.
 *  - Determinism: a track's arithmetic depends only on its inputs and the lane layout, never on
 *    scheduling, CTA shape, batch size or GPU count: identical inputs in the same layout give
 *    identical output bits.  For N <= 16 the default layout choice (HC_LAYOUT_AUTO) depends on
 *    the batch size, so a sharded job pins hc_tracker_settings.lane_layout to get the same bits
 *    for every shard size (paper_2112_03444_b200.distributed does).
 */
#ifndef HC_H
#define HC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HC_MAX_VARS 32
#define HC_MAX_FACTORS 8   /* max total degree of one Jacobian/homotopy term after differentiation + 1 */

typedef struct { double re, im; } hc_complex;

typedef enum {
  HC_OK = 0,
  HC_E_INVALID_ARG = 1,
  HC_E_TOO_LARGE = 2,
  HC_E_CUDA = 3,
  HC_E_OOM = 4,
  HC_E_INTERNAL = 5
} hc_status;

/* Per-track endpoint status (readings R8-R10). */
typedef enum {
  HC_CONVERGED = 0,      /* reached t = 1, polished, residual <= res_abs or relative residual <= res_rel */
  HC_DIVERGED = 1,       /* ||x||_inf > inf_norm during tracking (path to infinity) */
  HC_STEP_UNDERFLOW = 2, /* step size fell below dt_min */
  HC_MAX_STEPS = 3,      /* more than max_steps step attempts */
  HC_SINGULAR = 4,       /* reached t = 1 but the endpoint failed the residual test (singular/ill-conditioned) */
  HC_NONFINITE = 5,      /* non-finite endpoint */
  HC_AT_INFINITY = 6     /* endgame (reading R26): converged valuation ||x|| ~ s^v, v < 0, with s = 1 - t */
} hc_track_status;

typedef enum { HC_RK4 = 0, HC_EULER = 1 } hc_predictor;
typedef enum { HC_MEM_DEVICE = 0, HC_MEM_HOST = 1 } hc_memory;
typedef enum { HC_LAYOUT_AUTO = 0, HC_LAYOUT_THROUGHPUT = 1, HC_LAYOUT_WIDE = 2 } hc_lane_layout;

typedef struct hc_system_s *hc_system;  /* opaque, library-owned */
typedef struct hc_result_s *hc_result;  /* opaque, library-owned */

/* ---------------------------------------------------------------------------------------------
 * System description: F(x; p) = 0, N equations in N unknowns, coefficients polynomial in P params.
 *   F_i(x; p) = sum_{k : term_eq[k] == i} c_{term_coef[k]}(p) * prod_v x_v^{term_xexp[k*N + v]}
 *   c_j(p)    = sum_{m = coef_ptr[j]}^{coef_ptr[j+1]-1} coef_w[m] * prod_q p_q^{coef_pexp[m*P + q]}
 * All pointers are host pointers, borrowed for the duration of the call.
 * --------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t n_vars;            /* N, 1..32 */
  int32_t n_params;          /* P >= 0 */
  int32_t n_terms;           /* number of (equation, x-monomial) terms */
  const int32_t *term_eq;    /* [n_terms] equation index in [0, N) */
  const int32_t *term_xexp;  /* [n_terms * N] exponents of x, >= 0 */
  const int32_t *term_coef;  /* [n_terms] coefficient-expression id in [0, n_coefs) */
  int32_t n_coefs;           /* number of coefficient expressions */
  const int32_t *coef_ptr;   /* [n_coefs + 1] CSR offsets into coef_w / coef_pexp */
  const hc_complex *coef_w;  /* [nnz] weights (finite) */
  const int32_t *coef_pexp;  /* [nnz * P] parameter exponents, >= 0 */
} hc_system_desc;

/* Compile the system (the paper's "indexing system": homogenised term tables for
 * dH/dx, dH/dt and H, the constant-one slot, lane-balanced op lists) and upload the tables to
 * `device`.  *out receives a handle owned by the caller until hc_system_destroy. */
hc_status hc_system_create(const hc_system_desc *desc, int device, hc_system *out);

/* Total-degree homotopy H = (1-t) gamma G + t F, G_i = x_i^{d_i} - 1 (Eq. 1 + gamma trick, R1/R2).
 * `target` must have constant coefficients (all coef_pexp zero).  The created system has
 * parameters p = (coefficients of G, coefficients of F); hc_total_degree_params fills the
 * p0/p1 that make the parameter homotopy equal Eq. 1 with gamma. */
hc_status hc_system_create_total_degree(const hc_system_desc *target, int device, hc_system *out);
hc_status hc_total_degree_params(hc_system sys, hc_complex gamma,
                                 hc_complex *p0 /* host [P] */, hc_complex *p1 /* host [P] */);
/* Number of total-degree start solutions prod_i d_i (or -1 when > 2^31). */
int64_t hc_total_degree_count(hc_system sys);
/* Start solutions x_i = exp(2 pi i k_i / d_i), k_1 fastest (reading R2); host [count * N]. */
hc_status hc_total_degree_start(hc_system sys, hc_complex *start_x);

typedef struct {
  int32_t n_vars, n_params, n_coefs;
  int32_t coef_degree_t;      /* D: degree of the coefficient polynomials in t */
  int32_t lanes_per_track;    /* L = next power of two >= N (throughput layout; see hc_track_batch) */
  int32_t tracks_per_warp;    /* 32 / L */
  int32_t op_steps;           /* Q: evaluation op steps per lane (lane-balanced) */
  int32_t max_factors;        /* M: max monomial degree (paper's M) */
  int32_t n_ops_J, n_ops_rhs; /* real (unpadded) ops of dH/dx and of the H / dH/dt vector */
  int32_t n_terms;            /* terms of F */
  int64_t flops_coef;         /* algorithmic FP64 flops per solve: coefficient polynomials at t */
  int64_t flops_eval;         /* ... evaluating dH/dx and one right-hand side */
  int64_t flops_lu;           /* ... fused LU + solve on [A | b] (SURVEY.md §8(d) rule) */
  int64_t flops_solve;        /* total per solve (coef + eval + lu + 8N vector work) */
  int64_t smem_per_track;     /* bytes of shared memory per track slot */
  int32_t n_coef_slots;       /* coefficient slots (descriptor coefficients + s_k-scaled copies) */
  int32_t n_monos;            /* monomial table size (N unknowns + constant one + shared products) */
  int32_t mono_levels;        /* levels of the monomial program (max degree - 1) */
  int64_t flops_eval_kernel;  /* flops the kernel's evaluation actually performs (shared monomials) */
  int64_t flops_solve_kernel; /* per solve, kernel's own count (coef slots + eval + lu + 8N) */
} hc_system_info;
hc_status hc_system_info_get(hc_system sys, hc_system_info *out);
/* Host-only (no GPU needed): compile `desc` and report its info / its evaluation tables
 * (layouts in csrc/hc_internal.h): ops [op_steps * lanes_per_track * 2] uint32
 * (x = coefficient slot | monomial << 16, y = dest | flags << 16), mono_prog
 * [n_monos - N - 1] uint32 (parent | var << 16), slot_map [n_coef_slots * 2] int32
 * (descriptor coefficient id, scale s_k), entry_map [N * (N + 1)] int16 (dense entry of
 * [dH/dx | rhs] -> compact index used by op destinations, -1 = structural zero).
 * Any output pointer may be NULL. */
hc_status hc_system_compile_info(const hc_system_desc *desc, hc_system_info *out);
hc_status hc_system_compile_tables(const hc_system_desc *desc, uint32_t *ops, uint32_t *mono_prog, int32_t *slot_map,
                                   int16_t *entry_map);
hc_status hc_system_destroy(hc_system sys);

/* ---------------------------------------------------------------------------------------------
 * Tracker settings (the paper fixes none of them).
 * --------------------------------------------------------------------------------------------- */
typedef struct {
  int32_t predictor;    /* HC_RK4 or HC_EULER (Eq. 4) */
  double dt_init;       /* initial step (0.01) */
  double dt_min;        /* STEP_UNDERFLOW below this (1e-14) */
  double dt_max;        /* (0.1) */
  int32_t grow_after;   /* consecutive accepted steps before growing (4) */
  double grow;          /* (2.0) */
  double shrink;        /* on rejection (0.5) */
  int32_t max_newton;   /* corrector iterations per step (3) */
  double newton_tol;    /* converged when ||dx||_inf <= tol * max(1, ||x||_inf) (1e-8) */
  int32_t max_steps;    /* step attempts (10000) */
  double inf_norm;      /* DIVERGED when ||x||_inf exceeds it (1e14) */
  int32_t end_newton;   /* endpoint polish iterations at t = 1 (3) */
  double end_tol;       /* polish tolerance (1e-12) */
  double res_abs;       /* CONVERGED if ||F(x)||_inf <= res_abs (1e-10) ... */
  double res_rel;       /* ... or max_i |F_i| / sum_k |c_ik||m_k(x)| <= res_rel (1e-12) */
  double pivot_rel;     /* a solve fails when |pivot| <= pivot_rel * max|A_ij| (1e-14) */
  /* Endgame (reading R26; the paper: "the cardinality of the output is not always
   * correct, and extra verification steps are needed").  With s = 1 - t, once
   * s <= eg_start every halving of s is sampled at a step start (right after the predictor's
   * first stage): v = dlog||x||/dlog s and mu = dlog(s ||dx/dt||)/dlog s between samples.
   * AT_INFINITY: three consecutive samples with |mu - mu_prev| < eg_stab, |v - mu| < eg_stab,
   * mu < eg_inf_mu, and s <= eg_inf_s or ||x||_inf >= eg_inf_norm.  Cauchy endgame (singular
   * endpoint, winding number m, mu -> 1/m): three consecutive samples with |mu - mu_prev| < eg_stab
   * and 0 < mu < eg_sing_mu; the path is tracked around |1 - t| = s in eg_samples arcs per loop until
   * it closes (m loops, m <= eg_max_winding), the endpoint estimate is the mean of the samples
   * (Cauchy integral), radii s, s/2, ... (at most eg_max_radii) until two estimates agree within
   * eg_tol * max(1, ||x||_inf). */
  double eg_start;      /* 0 disables the endgame (0.1) */
  double eg_inf_mu;     /* (-0.05) */
  double eg_sing_mu;    /* (0.75) */
  double eg_stab;       /* (0.02) */
  double eg_inf_s;      /* (1e-12) */
  double eg_inf_norm;   /* (1e5) */
  int32_t eg_samples;   /* (16) */
  int32_t eg_max_winding; /* (8) */
  int32_t eg_max_radii; /* (12) */
  double eg_tol;        /* (1e-10) */
  /* Lane layout of the tracker kernel for N <= 16 (a launch choice; results agree as solution
   * sets, bits may differ between layouts because the op list is balanced over a different number
   * of lanes): HC_LAYOUT_AUTO picks by batch size (see hc_track_batch), HC_LAYOUT_THROUGHPUT /
   * HC_LAYOUT_WIDE pin it, so a job sharded over GPUs gives the same bits for any shard size.
   * Ignored for N > 16 (one layout).  The environment variable HC_LANES=wide|narrow overrides
   * HC_LAYOUT_AUTO only. */
  int32_t lane_layout;  /* hc_lane_layout (HC_LAYOUT_AUTO) */
} hc_tracker_settings;
hc_status hc_tracker_settings_default(hc_tracker_settings *out);

/* ---------------------------------------------------------------------------------------------
 * One batch: B instances x S start solutions = B*S tracks, track id g = b*S + s.
 * memory == HC_MEM_DEVICE: every pointer is a device pointer on the system's device; the call
 *   enqueues work on `stream` and returns immediately; inputs must stay valid until the stream
 *   passes the batch (hc_result_wait or a stream synchronisation).
 * memory == HC_MEM_HOST: every pointer is a host pointer; the library stages host->device
 *   copies, runs, copies results back and returns after completion (end-to-end path).
 * Output pointers may be NULL: the result then owns device buffers, read with hc_result_get.
 * --------------------------------------------------------------------------------------------- */
typedef struct {
  int64_t n_instances;         /* B >= 1 */
  int64_t n_start;             /* S >= 1 */
  const hc_complex *start_x;   /* [S * N] start solutions */
  const hc_complex *p_start;   /* [P] p0 (may be NULL when P == 0) */
  const hc_complex *p_target;  /* [B * P] p1 per instance (may be NULL when P == 0) */
  hc_complex *x_out;           /* [B * S * N] endpoints, or NULL */
  int32_t *status_out;         /* [B * S] hc_track_status, or NULL */
  int32_t *counters_out;       /* [B * S * 4]: steps, rejections, newton iterations, solves; or NULL */
  double *resid_out;           /* [B * S * 2]: ||F||_inf, relative residual; or NULL */
  int32_t memory;              /* hc_memory */
  void *stream;                /* cudaStream_t (NULL = default stream) */
  int32_t *winding_out;        /* [B * S]: Cauchy endgame winding number (0: not used); or NULL */
} hc_batch;

/* Enqueue (or, for HC_MEM_HOST, run) one batch.  *out (may be NULL) receives a result handle that
 * must be released with hc_result_destroy; the system must outlive its results.
 * Lane layout (a launch choice; results agree as solution sets, bits may differ between layouts
 * because the op list is balanced over a different number of lanes): for N <= 16 a batch of at
 * most ~2.5 waves of one-track-per-warp slots runs in the wide latency layout (32 lanes per track,
 * e.g. single-instance katsura-6 / cyclic-7 solves), larger batches in the throughput layout
 * (next_pow2(N) lanes per track, 32 / that tracks per warp).  settings->lane_layout pins the
 * choice; with HC_LAYOUT_AUTO the environment HC_LANES=wide|narrow overrides it; hc_result_launch
 * reports it. */
hc_status hc_track_batch(hc_system sys, const hc_tracker_settings *settings, const hc_batch *batch,
                         hc_result *out);
/* Block until the batch finished. */
hc_status hc_result_wait(hc_result res);
/* Device time in ms between the start of the coefficient prologue and the end of the batch (the
 * tracker and, when enabled, the Cauchy endgame kernel), measured with CUDA events on the batch
 * stream; also the prologue alone and the tracker kernel alone. */
hc_status hc_result_elapsed_ms(hc_result res, float *total_ms, float *prologue_ms, float *tracker_ms);

/* Launch configuration the tracker kernel used (lanes per track, warps per CTA, persistent CTAs,
 * dynamic shared memory per CTA). */
hc_status hc_result_launch(hc_result res, int32_t *lanes, int32_t *warps_per_cta, int32_t *ctas, int64_t *smem_bytes);

typedef struct {
  int32_t status;       /* hc_track_status */
  int32_t steps, rejections, newton_iters, solves;
  double resid_abs, resid_rel;
} hc_track_info;
/* Copy one track's endpoint (host x [N]) and info; waits for the batch. */
hc_status hc_result_get(hc_result res, int64_t instance, int64_t track, hc_complex *x, hc_track_info *info);
hc_status hc_result_destroy(hc_result res);

/* ---------------------------------------------------------------------------------------------
 * Batched fused LU + solve (kernel fusion, augmented matrix [A b]; the elimination
 * runs Gauss-Jordan in the one-row-per-lane layout, so no separate back-substitution).  Solves
 * A_k x_k = b_k for k < batch; A row-major [batch][n][n], b [batch][n],
 * x [batch][n], info [batch] (0 ok, 1 singular: pivot <= pivot_rel * max|A_ij| or non-finite).
 * Device pointers, async on stream.  n in [1, 32].
 * --------------------------------------------------------------------------------------------- */
hc_status hc_batched_zgesv(int32_t n, int64_t batch, const hc_complex *A, const hc_complex *b, hc_complex *x,
                           int32_t *info, double pivot_rel, void *stream);

/* FP64 DFMA throughput probe (SURVEY.md §8(d) "FP64 peak"): runs ~`ms` milliseconds of
 * independent DFMA chains on every SM of `device`; *tflops receives the achieved FLOP/s / 1e12. */
hc_status hc_fp64_peak_probe(int device, double *tflops);

/* ---------------------------------------------------------------------------------------------
 * Endpoint post-processing (host, not timed; readings R11, R12 -- SPEC
 * S:266-274): greedy deduplication in track order of one instance's CONVERGED endpoints -- track s
 * merges into the first kept endpoint x with |x_i - y_i| <= dedup_tol * max(1, |x_i|) for every
 * i -- and real classification of the kept ones (max_i |Im x_i| <= real_tol * max(1, |x_i|)).
 * Host arrays: x [S * N] endpoints (e.g. one instance's slice of x_out), status [S] (hc_track_status,
 * NULL = all CONVERGED).  Caller-owned outputs, [S] each, may be NULL: rep[s] = the track index of
 * the kept endpoint s merged into (s itself when kept), -1 when s is not CONVERGED; is_real[s] = 1
 * for a kept real endpoint, else 0.  *n_unique = number of kept endpoints.
 * Errors: HC_E_INVALID_ARG for null n_unique, null x with S > 0, S < 0, N outside [1, 32], negative
 * tolerances.
 * --------------------------------------------------------------------------------------------- */
hc_status hc_solutions(const hc_complex *x, const int32_t *status, int64_t S, int32_t N, double dedup_tol,
                       double real_tol, int64_t *rep, int32_t *is_real, int64_t *n_unique);

/* Experiment hook: per-phase cycle sums of the tracker kernel (coefficients, monomials, ops, row
 * load, elimination, state machine, eval+solve, iterations) -- only in libraries built with
 * -DHCB_PHASE_TIMING (HCB_VARIANT=timing); HC_E_INVALID_ARG otherwise. out8: host [8]. */
hc_status hc_debug_phase_cycles(hc_result res, unsigned long long *out8);

/* Thread-local message of the last failing call (never NULL). */
const char *hc_last_error(void);
/* Library version string. */
const char *hc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* HC_H */
