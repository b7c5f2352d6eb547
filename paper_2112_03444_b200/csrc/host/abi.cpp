// abi.cpp -- the C ABI (include/hc.h): system handles, batch launch, results, helpers.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>   // header-only NVTX v3: ranges cost nothing unless a tool is attached

#include "../hc_internal.h"
#include "compiler.h"
#include "../kernels/layout.h"

namespace hcb {
// per-N launchers defined in csrc/kernels/tracker_n*.cu
#define HCB_DECLW(N)                                                                        \
  cudaError_t launch_tracker_wide_##N(const TrackArgs &, int, cudaStream_t, TrackerPlan *); \
  cudaError_t launch_endgame_wide_##N(const TrackArgs &, int, cudaStream_t);
HCB_DECLW(1) HCB_DECLW(2) HCB_DECLW(3) HCB_DECLW(4) HCB_DECLW(5) HCB_DECLW(6) HCB_DECLW(7) HCB_DECLW(8)
HCB_DECLW(9) HCB_DECLW(10) HCB_DECLW(11) HCB_DECLW(12) HCB_DECLW(13) HCB_DECLW(14) HCB_DECLW(15) HCB_DECLW(16)
#undef HCB_DECLW
#define HCB_DECL(N)                                                                                      \
  cudaError_t launch_tracker_##N(const TrackArgs &, int, cudaStream_t, TrackerPlan *);                  \
  cudaError_t launch_endgame_##N(const TrackArgs &, int, cudaStream_t);                                 \
  cudaError_t launch_zgesv_##N(int64_t, const double2 *, const double2 *, double2 *, int32_t *, double, \
                               cudaStream_t);
HCB_DECL(1) HCB_DECL(2) HCB_DECL(3) HCB_DECL(4) HCB_DECL(5) HCB_DECL(6) HCB_DECL(7) HCB_DECL(8)
HCB_DECL(9) HCB_DECL(10) HCB_DECL(11) HCB_DECL(12) HCB_DECL(13) HCB_DECL(14) HCB_DECL(15) HCB_DECL(16)
HCB_DECL(17) HCB_DECL(18) HCB_DECL(19) HCB_DECL(20) HCB_DECL(21) HCB_DECL(22) HCB_DECL(23) HCB_DECL(24)
HCB_DECL(25) HCB_DECL(26) HCB_DECL(27) HCB_DECL(28) HCB_DECL(29) HCB_DECL(30) HCB_DECL(31) HCB_DECL(32)
#undef HCB_DECL

typedef cudaError_t (*zgesv_fn)(int64_t, const double2 *, const double2 *, double2 *, int32_t *, double, cudaStream_t);
static const tracker_launch_fn kTrackers[33] = {
    nullptr,            launch_tracker_1,  launch_tracker_2,  launch_tracker_3,  launch_tracker_4,
    launch_tracker_5,   launch_tracker_6,  launch_tracker_7,  launch_tracker_8,  launch_tracker_9,
    launch_tracker_10,  launch_tracker_11, launch_tracker_12, launch_tracker_13, launch_tracker_14,
    launch_tracker_15,  launch_tracker_16, launch_tracker_17, launch_tracker_18, launch_tracker_19,
    launch_tracker_20,  launch_tracker_21, launch_tracker_22, launch_tracker_23, launch_tracker_24,
    launch_tracker_25,  launch_tracker_26, launch_tracker_27, launch_tracker_28, launch_tracker_29,
    launch_tracker_30,  launch_tracker_31, launch_tracker_32};
static const zgesv_fn kZgesv[33] = {
    nullptr,          launch_zgesv_1,  launch_zgesv_2,  launch_zgesv_3,  launch_zgesv_4,  launch_zgesv_5,
    launch_zgesv_6,   launch_zgesv_7,  launch_zgesv_8,  launch_zgesv_9,  launch_zgesv_10, launch_zgesv_11,
    launch_zgesv_12,  launch_zgesv_13, launch_zgesv_14, launch_zgesv_15, launch_zgesv_16, launch_zgesv_17,
    launch_zgesv_18,  launch_zgesv_19, launch_zgesv_20, launch_zgesv_21, launch_zgesv_22, launch_zgesv_23,
    launch_zgesv_24,  launch_zgesv_25, launch_zgesv_26, launch_zgesv_27, launch_zgesv_28, launch_zgesv_29,
    launch_zgesv_30,  launch_zgesv_31, launch_zgesv_32};

tracker_launch_fn tracker_launcher(int N) { return (N >= 1 && N <= 32) ? kTrackers[N] : nullptr; }
typedef cudaError_t (*endgame_fn)(const TrackArgs &, int, cudaStream_t);
static const endgame_fn kEndgame[33] = {
    nullptr,            launch_endgame_1,  launch_endgame_2,  launch_endgame_3,  launch_endgame_4,
    launch_endgame_5,   launch_endgame_6,  launch_endgame_7,  launch_endgame_8,  launch_endgame_9,
    launch_endgame_10,  launch_endgame_11, launch_endgame_12, launch_endgame_13, launch_endgame_14,
    launch_endgame_15,  launch_endgame_16, launch_endgame_17, launch_endgame_18, launch_endgame_19,
    launch_endgame_20,  launch_endgame_21, launch_endgame_22, launch_endgame_23, launch_endgame_24,
    launch_endgame_25,  launch_endgame_26, launch_endgame_27, launch_endgame_28, launch_endgame_29,
    launch_endgame_30,  launch_endgame_31, launch_endgame_32};
// the wide latency layout (32 lanes per track) for N <= 16
static const tracker_launch_fn kTrackersWide[17] = {
    nullptr,               launch_tracker_wide_1,  launch_tracker_wide_2,  launch_tracker_wide_3,
    launch_tracker_wide_4, launch_tracker_wide_5,  launch_tracker_wide_6,  launch_tracker_wide_7,
    launch_tracker_wide_8, launch_tracker_wide_9,  launch_tracker_wide_10, launch_tracker_wide_11,
    launch_tracker_wide_12, launch_tracker_wide_13, launch_tracker_wide_14, launch_tracker_wide_15,
    launch_tracker_wide_16};
static tracker_launch_fn tracker_launcher_wide(int N) { return (N >= 1 && N <= 16) ? kTrackersWide[N] : nullptr; }
static const endgame_fn kEndgameWide[17] = {
    nullptr,               launch_endgame_wide_1,  launch_endgame_wide_2,  launch_endgame_wide_3,
    launch_endgame_wide_4, launch_endgame_wide_5,  launch_endgame_wide_6,  launch_endgame_wide_7,
    launch_endgame_wide_8, launch_endgame_wide_9,  launch_endgame_wide_10, launch_endgame_wide_11,
    launch_endgame_wide_12, launch_endgame_wide_13, launch_endgame_wide_14, launch_endgame_wide_15,
    launch_endgame_wide_16};

cudaError_t launch_batched_zgesv(int n, int64_t batch, const double2 *A, const double2 *b, double2 *x,
                                 int32_t *info, double pivot_rel, cudaStream_t s) {
  if (n < 1 || n > 32) return cudaErrorInvalidValue;
  if (batch == 0) return cudaSuccess;
  return kZgesv[n](batch, A, b, x, info, pivot_rel, s);
}
}  // namespace hcb

using namespace hcb;

static thread_local std::string g_err;

static hc_status fail(hc_status s, const std::string &msg) {
  g_err = msg;
  return s;
}
static hc_status cuda_fail(cudaError_t e, const char *where) {
  g_err = std::string(where) + ": " + cudaGetErrorString(e);
  return e == cudaErrorMemoryAllocation ? HC_E_OOM : HC_E_CUDA;
}
#define CK(call)                                   \
  do {                                             \
    cudaError_t _e = (call);                       \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// A compiled table set on the device (one per lane layout).
struct DevTables {
  uint2 *d_ops = nullptr;
  int Qp = 0;                // pair steps when d_ops holds the paired table (pair_ops), else 0
  uint32_t *d_mono_prog = nullptr;
  int16_t *d_mpos = nullptr;
  CoefMono *d_mono = nullptr;
  int32_t *d_mono_ptr = nullptr;
};

struct hc_system_s {
  int device = 0;
  CompiledSystem cs;     // throughput layout: lanes_for(N) lanes per track
  DevTables dt;
  bool has_wide = false;  // N <= 16: the wide latency layout (32 lanes per track) as well
  CompiledSystem cs_w;
  DevTables dt_w;
  // total-degree metadata
  bool td = false;
  std::vector<hc_complex> td_fvals;
  std::vector<int32_t> td_degrees;
};

struct hc_result_s {
  hc_system sys = nullptr;   // must outlive the result (documented in hc.h)
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t B = 0, S = 0, total = 0;
  int memory = HC_MEM_DEVICE;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};   // prologue start, tracker start, end, endgame start
  // device buffers owned by the result (freed on destroy), and per-batch temporaries (freed in
  // stream order once the batch's kernels are enqueued; on destroy if the enqueue failed)
  std::vector<void *> owned, temps;
  // where the outputs are (device or host)
  hc_complex *x = nullptr;
  int32_t *status = nullptr, *counters = nullptr;
  double *resid = nullptr;
  int32_t *winding = nullptr;
  bool outputs_on_host = false;
  bool waited = false;
  TrackerPlan plan{};
  unsigned long long *phase_cycles = nullptr;
};

static void destroy_result(hc_result r) {
  if (!r) return;
  cudaSetDevice(r->device);
  for (void *p : r->owned) cudaFreeAsync(p, r->stream);
  for (void *p : r->temps) cudaFreeAsync(p, r->stream);
  for (auto &e : r->ev)
    if (e) cudaEventDestroy(e);
  if (r->outputs_on_host) {
  }
  delete r;
}

// The library's stream-ordered memory pool per device: memory freed by a batch stays in the pool
// (release threshold 4 GiB) for the next batch, so steady-state calls allocate without mapping new
// pages (the default pool returns everything at each synchronisation).
static cudaMemPool_t lib_pool(int device) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  if ((int)pools.size() <= device) pools.resize(device + 1, nullptr);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    cudaMemPool_t pool = nullptr;
    if (cudaMemPoolCreate(&pool, &props) != cudaSuccess) {
      (void)cudaGetLastError();
      return nullptr;   // fall back to the device's default pool
    }
    uint64_t thr = 4ull << 30;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    pools[device] = pool;
  }
  return pools[device];
}

// temp: a per-batch temporary, released in stream order right after the batch's kernels are
// enqueued (hc_track_batch), not when the result is destroyed
template <class T>
static hc_status dev_alloc(hc_result r, T **p, size_t count, bool temp = false) {
  void *q = nullptr;
  const size_t bytes = std::max<size_t>(1, count) * sizeof(T);
  cudaMemPool_t pool = lib_pool(r->device);
  cudaError_t e = pool ? cudaMallocFromPoolAsync(&q, bytes, pool, r->stream) : cudaMallocAsync(&q, bytes, r->stream);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMallocAsync");
  (temp ? r->temps : r->owned).push_back(q);
  *p = reinterpret_cast<T *>(q);
  return HC_OK;
}

extern "C" {

const char *hc_last_error(void) { return g_err.c_str(); }
const char *hc_version(void) { return "hc-b200 0.1 (sm_100a)"; }

hc_status hc_tracker_settings_default(hc_tracker_settings *s) {
  if (!s) return fail(HC_E_INVALID_ARG, "null settings");
  // SURVEY.md §8(c) readings R5-R10 (the paper fixes none of these constants).
  s->predictor = HC_RK4;
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
  // endgame, reading R26
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
  s->lane_layout = HC_LAYOUT_AUTO;
  return HC_OK;
}

// The op table, the monomial program and the entry map are staged into shared memory by the tracker
// with 1-D bulk async copies (cp.async.bulk, 16-byte granules): each device copy is zero-padded to
// a multiple of 16 bytes (the padded bytes land in the shared-memory alignment padding).
static hc_status upload_padded16(void **dst, const void *src, size_t bytes) {
  const size_t padded = std::max<size_t>(16, (bytes + 15) & ~size_t(15));
  std::vector<unsigned char> buf(padded, 0);
  if (bytes) std::memcpy(buf.data(), src, bytes);
  CK(cudaMalloc(dst, padded));
  CK(cudaMemcpy(*dst, buf.data(), padded, cudaMemcpyHostToDevice));
  return HC_OK;
}

// Paired op table (tracker.cuh run_ops_pairs): the ops of each entry two at a time in one 16-byte
// record {slot_a | mono_a << 16, slot_b | mono_b << 16, dest | flags << 16, 0}; an odd entry's last
// record pairs its term with the constant-zero monomial mono[n_mono] (same slot, so the coefficient
// is finite and the term exactly 0); entries re-balanced over the lanes by record count; lanes past
// their last entry get neutral records.  Returns the pair steps Qp; the table is [Qp][L] records.
static int pair_ops(const CompiledSystem &cs, std::vector<uint2> &out) {
  const int L = cs.L, Q = cs.Q;
  // the entries (op runs ending in OP_LAST) of every lane; the compiler's never-stored padding ops
  // after a lane's last entry are dropped
  std::vector<std::vector<uint2>> entries;
  for (int l = 0; l < L; ++l) {
    std::vector<uint2> cur;
    for (int q = 0; q < Q; ++q) {
      const uint2 o = cs.ops[(size_t)q * L + l];
      cur.push_back(o);
      if ((o.y >> 16) & OP_LAST) {
        entries.push_back(cur);
        cur.clear();
      }
    }
  }
  // re-balance over the lanes by record count (LPT, longest first; stable, deterministic)
  std::stable_sort(entries.begin(), entries.end(),
                   [](const std::vector<uint2> &a, const std::vector<uint2> &b) { return a.size() > b.size(); });
  std::vector<std::vector<uint4>> lanes(L);
  for (const auto &e : entries) {
    int l = 0;
    for (int k = 1; k < L; ++k)
      if (lanes[k].size() < lanes[l].size()) l = k;
    const uint32_t fl = e.back().y >> 16;
    for (size_t i = 0; i < e.size(); i += 2) {
      const uint2 a = e[i];
      const bool has_b = i + 1 < e.size();
      const uint2 b = has_b ? e[i + 1] : uint2{(a.x & 0xFFFFu) | ((uint32_t)cs.n_mono << 16), 0u};
      const bool last = i + 2 >= e.size();
      lanes[l].push_back(uint4{a.x, b.x, last ? e.back().y : (OP_NO_DEST | ((fl & OP_RHS) << 16)), 0u});
    }
  }
  int Qp = 0;
  for (auto &v : lanes) Qp = std::max(Qp, (int)v.size());
  const uint4 neutral{(uint32_t)cs.n_mono << 16, (uint32_t)cs.n_mono << 16, OP_NO_DEST, 0u};
  out.assign((size_t)Qp * L * 2, uint2{0u, 0u});
  for (int q = 0; q < Qp; ++q)
    for (int l = 0; l < L; ++l) {
      const uint4 r = q < (int)lanes[l].size() ? lanes[l][q] : neutral;
      out[((size_t)q * L + l) * 2] = uint2{r.x, r.y};
      out[((size_t)q * L + l) * 2 + 1] = uint2{r.z, r.w};
    }
  return Qp;
}

static hc_status upload_tables(const CompiledSystem &cs, DevTables &t, bool wide) {
  // Paired op table for the wide latency layout (A/B: katsura-6 1.50 -> 1.44 ms, cyclic-7 TD 8.2 ->
  // 7.7 ms: half the op-list iterations on a latency-bound chain), single ops for the throughput
  // layout (trifocal -3.5 %, 4-view -5.5 %, 5-point -5 % with pairs: the padding terms' extra work
  // and the gathers' bank pattern cost more than the saved bookkeeping).  HC_OP_PAIRS=0|1 overrides.
  const char *ev = getenv("HC_OP_PAIRS");
  const bool pairs = ev ? atoi(ev) == 1 : wide;
  std::vector<uint2> pops;
  t.Qp = pairs ? pair_ops(cs, pops) : 0;
  hc_status s = t.Qp ? upload_padded16((void **)&t.d_ops, pops.data(), sizeof(uint2) * pops.size())
                     : upload_padded16((void **)&t.d_ops, cs.ops.data(), sizeof(uint2) * cs.ops.size());
  if (s == HC_OK) s = upload_padded16((void **)&t.d_mono_prog, cs.mono_prog.data(), sizeof(uint32_t) * cs.mono_prog.size());
  // device copy of the entry map: structural zeros point at the extra always-zero entry n_entries
  std::vector<int16_t> mp(cs.mpos);
  for (auto &v : mp)
    if (v < 0) v = (int16_t)cs.n_entries;
  if (s == HC_OK) s = upload_padded16((void **)&t.d_mpos, mp.data(), sizeof(int16_t) * mp.size());
  if (s != HC_OK) return s;
  CK(cudaMalloc(&t.d_mono, sizeof(CoefMono) * std::max<size_t>(1, cs.mono.size())));
  CK(cudaMalloc(&t.d_mono_ptr, sizeof(int32_t) * cs.mono_ptr.size()));
  if (!cs.mono.empty())
    CK(cudaMemcpy(t.d_mono, cs.mono.data(), sizeof(CoefMono) * cs.mono.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(t.d_mono_ptr, cs.mono_ptr.data(), sizeof(int32_t) * cs.mono_ptr.size(), cudaMemcpyHostToDevice));
  return HC_OK;
}

static hc_status upload_system(hc_system sys) {
  CK(cudaSetDevice(sys->device));
  hc_status s = upload_tables(sys->cs, sys->dt, false);
  if (s == HC_OK && sys->has_wide) s = upload_tables(sys->cs_w, sys->dt_w, true);
  return s;
}

static void free_tables(DevTables &t) {
  cudaFree(t.d_ops);
  cudaFree(t.d_mono_prog);
  cudaFree(t.d_mpos);
  cudaFree(t.d_mono);
  cudaFree(t.d_mono_ptr);
}

static void free_system(hc_system sys) {
  if (!sys) return;
  cudaSetDevice(sys->device);
  free_tables(sys->dt);
  free_tables(sys->dt_w);
  delete sys;
}

hc_status hc_system_create(const hc_system_desc *desc, int device, hc_system *out) {
  if (!desc || !out) return fail(HC_E_INVALID_ARG, "null argument");
  *out = nullptr;
  hc_system sys = new (std::nothrow) hc_system_s();
  if (!sys) return fail(HC_E_OOM, "host allocation failed");
  sys->device = device;
  std::string err;
  hc_status s = compile_system(*desc, sys->cs, err);
  if (s == HC_OK && sys->cs.N <= 16 && sys->cs.L < 32) {
    s = compile_system(*desc, sys->cs_w, err, 32);
    sys->has_wide = (s == HC_OK);
  }
  if (s != HC_OK) {
    delete sys;
    return fail(s, err);
  }
  s = upload_system(sys);
  if (s != HC_OK) {
    free_system(sys);
    return s;
  }
  *out = sys;
  return HC_OK;
}

hc_status hc_system_create_total_degree(const hc_system_desc *target, int device, hc_system *out) {
  if (!target || !out) return fail(HC_E_INVALID_ARG, "null argument");
  *out = nullptr;
  OwnedDesc od;
  std::vector<hc_complex> fvals;
  std::vector<int32_t> degrees;
  std::string err;
  hc_status s = total_degree_desc(*target, od, fvals, degrees, err);
  if (s != HC_OK) return fail(s, err);
  hc_system_desc v = od.view();
  s = hc_system_create(&v, device, out);
  if (s != HC_OK) return s;
  (*out)->td = true;
  (*out)->td_fvals = fvals;
  (*out)->td_degrees = degrees;
  return HC_OK;
}

hc_status hc_total_degree_params(hc_system sys, hc_complex gamma, hc_complex *p0, hc_complex *p1) {
  if (!sys || !p0 || !p1) return fail(HC_E_INVALID_ARG, "null argument");
  if (!sys->td) return fail(HC_E_INVALID_ARG, "not a total-degree system");
  if (!std::isfinite(gamma.re) || !std::isfinite(gamma.im) || (gamma.re == 0.0 && gamma.im == 0.0))
    return fail(HC_E_INVALID_ARG, "gamma must be finite and non-zero");
  const int N = sys->cs.N, P = sys->cs.P;
  // H = F~(x; (1-t) p0 + t p1) = (1-t) gamma G + t F  (Eq. 1 with gamma, R1)
  for (int q = 0; q < P; ++q) p0[q] = p1[q] = hc_complex{0.0, 0.0};
  for (int i = 0; i < N; ++i) {
    p0[i] = gamma;                                     // gamma * x_i^{d_i}
    p0[N + i] = hc_complex{-gamma.re, -gamma.im};      // gamma * (-1)
  }
  for (size_t j = 0; j < sys->td_fvals.size(); ++j) p1[2 * N + j] = sys->td_fvals[j];
  return HC_OK;
}

int64_t hc_total_degree_count(hc_system sys) {
  if (!sys || !sys->td) return -1;
  int64_t c = 1;
  for (int d : sys->td_degrees) {
    c *= d;
    if (c > (1LL << 31)) return -1;
  }
  return c;
}

hc_status hc_total_degree_start(hc_system sys, hc_complex *x) {
  if (!sys || !x) return fail(HC_E_INVALID_ARG, "null argument");
  if (!sys->td) return fail(HC_E_INVALID_ARG, "not a total-degree system");
  const int64_t cnt = hc_total_degree_count(sys);
  if (cnt < 0) return fail(HC_E_TOO_LARGE, "Bezout number exceeds 2^31");
  const int N = sys->cs.N;
  for (int64_t g = 0; g < cnt; ++g) {
    int64_t rem = g;
    for (int i = 0; i < N; ++i) {
      const int d = sys->td_degrees[i];
      const int k = (int)(rem % d);
      rem /= d;
      // exp(2 pi i k / d); quarter turns exact (reading R2)
      const int num = 4 * k;   // angle in quarter turns = 4k/d
      double c, s;
      if (num % d == 0) {
        const int qt = (num / d) & 3;
        c = (qt == 0) ? 1.0 : (qt == 2 ? -1.0 : 0.0);
        s = (qt == 1) ? 1.0 : (qt == 3 ? -1.0 : 0.0);
      } else {
        const double ang = 2.0 * M_PI * (double)k / (double)d;
        c = std::cos(ang);
        s = std::sin(ang);
      }
      x[g * N + i] = hc_complex{c, s};
    }
  }
  return HC_OK;
}

static void fill_info(const CompiledSystem &cs, hc_system_info *o) {
  std::memset(o, 0, sizeof(*o));
  o->n_vars = cs.N;
  o->n_params = cs.P;
  o->n_coefs = cs.ncoef;
  o->coef_degree_t = cs.D;
  o->lanes_per_track = cs.L;
  o->tracks_per_warp = 32 / cs.L;
  o->op_steps = cs.Q;
  o->max_factors = cs.M;
  o->n_ops_J = cs.n_ops_J;
  o->n_ops_rhs = cs.n_ops_rhs;
  o->n_terms = cs.n_terms;
  o->flops_coef = cs.flops_coef;
  o->flops_eval = cs.flops_eval;
  o->flops_lu = cs.flops_lu;
  o->flops_solve = cs.flops_solve;
  o->n_coef_slots = cs.ncoef;
  o->n_monos = cs.n_mono;
  o->mono_levels = cs.n_levels;
  o->flops_eval_kernel = cs.flops_eval_kernel;
  o->flops_solve_kernel = cs.flops_solve_kernel;
  // (the tracker keeps its per-lane state in shared memory when its CTA shape is 16 warps per SM)
  const bool ss = tracker_smem_state(cs.N, cs.L);
  o->smem_per_track = (int64_t)slot_bytes(cs.N, ss ? state_lanes(cs.N, cs.L, hy_layout(cs.N) && cs.L == lanes_for(cs.N) ? 2 : 1) : 0,
                                          cs.ncoef, cs.ncoef_src,
                                          cs.n_mono, cs.n_entries + 1);
}

hc_status hc_system_info_get(hc_system sys, hc_system_info *o) {
  if (!sys || !o) return fail(HC_E_INVALID_ARG, "null argument");
  fill_info(sys->cs, o);
  return HC_OK;
}

hc_status hc_system_compile_info(const hc_system_desc *desc, hc_system_info *o) {
  if (!desc || !o) return fail(HC_E_INVALID_ARG, "null argument");
  CompiledSystem cs;
  std::string err;
  hc_status s = compile_system(*desc, cs, err);
  if (s != HC_OK) return fail(s, err);
  fill_info(cs, o);
  return HC_OK;
}

hc_status hc_system_compile_tables(const hc_system_desc *desc, uint32_t *ops, uint32_t *mono_prog, int32_t *slot_map,
                                   int16_t *entry_map) {
  if (!desc) return fail(HC_E_INVALID_ARG, "null argument");
  CompiledSystem cs;
  std::string err;
  hc_status s = compile_system(*desc, cs, err);
  if (s != HC_OK) return fail(s, err);
  if (ops) std::memcpy(ops, cs.ops.data(), sizeof(uint2) * cs.ops.size());
  if (mono_prog) std::memcpy(mono_prog, cs.mono_prog.data(), sizeof(uint32_t) * cs.mono_prog.size());
  if (slot_map) std::memcpy(slot_map, cs.slot_map.data(), sizeof(int32_t) * cs.slot_map.size());
  if (entry_map) std::memcpy(entry_map, cs.mpos.data(), sizeof(int16_t) * cs.mpos.size());
  return HC_OK;
}

hc_status hc_solutions(const hc_complex *x, const int32_t *status, int64_t S, int32_t N, double dedup_tol,
                       double real_tol, int64_t *rep, int32_t *is_real, int64_t *n_unique) {
  if ((!x && S > 0) || !n_unique) return fail(HC_E_INVALID_ARG, "null argument");
  if (S < 0 || N < 1 || N > 32) return fail(HC_E_INVALID_ARG, "S >= 0 and 1 <= N <= 32 required");
  if (!(dedup_tol >= 0.0) || !(real_tol >= 0.0)) return fail(HC_E_INVALID_ARG, "negative tolerance");
  std::vector<int64_t> kept;   // track indices of the kept endpoints, in track order (reading R11)
  for (int64_t s = 0; s < S; ++s) {
    const bool conv = !status || status[s] == HC_CONVERGED;
    if (is_real) is_real[s] = 0;
    if (!conv) {
      if (rep) rep[s] = -1;
      continue;
    }
    const hc_complex *y = x + s * N;
    int64_t into = -1;
    for (int64_t u : kept) {
      const hc_complex *k = x + u * N;
      bool same = true;
      for (int i = 0; i < N && same; ++i) {
        const double d = std::hypot(k[i].re - y[i].re, k[i].im - y[i].im);
        same = d <= dedup_tol * std::max(1.0, std::hypot(k[i].re, k[i].im));
      }
      if (same) {
        into = u;
        break;
      }
    }
    if (into < 0) {
      kept.push_back(s);
      into = s;
      if (is_real) {   // reading R12
        bool real = true;
        for (int i = 0; i < N && real; ++i)
          real = std::fabs(y[i].im) <= real_tol * std::max(1.0, std::hypot(y[i].re, y[i].im));
        is_real[s] = real ? 1 : 0;
      }
    }
    if (rep) rep[s] = into;
  }
  *n_unique = (int64_t)kept.size();
  return HC_OK;
}

hc_status hc_system_destroy(hc_system sys) {
  free_system(sys);
  return HC_OK;
}

static hc_status check_settings(const hc_tracker_settings &s) {
  if (s.predictor != HC_RK4 && s.predictor != HC_EULER) return fail(HC_E_INVALID_ARG, "predictor");
  if (!(s.dt_min > 0 && s.dt_min <= s.dt_init && s.dt_init <= s.dt_max && s.dt_max <= 1.0))
    return fail(HC_E_INVALID_ARG, "need 0 < dt_min <= dt_init <= dt_max <= 1");
  if (!(s.grow > 1.0) || !(s.shrink > 0.0 && s.shrink < 1.0)) return fail(HC_E_INVALID_ARG, "grow > 1, 0 < shrink < 1");
  if (s.grow_after < 1 || s.max_newton < 1 || s.max_steps < 1 || s.end_newton < 0)
    return fail(HC_E_INVALID_ARG, "iteration counts");
  if (!(s.newton_tol > 0) || !(s.inf_norm > 0) || !(s.end_tol > 0) || !(s.pivot_rel >= 0))
    return fail(HC_E_INVALID_ARG, "tolerances");
  if (!(s.eg_start >= 0.0 && s.eg_start < 1.0)) return fail(HC_E_INVALID_ARG, "need 0 <= eg_start < 1");
  if (s.eg_start > 0.0 && (s.eg_samples < 2 || s.eg_max_winding < 1 || s.eg_max_radii < 2 || !(s.eg_stab > 0) ||
                           !(s.eg_tol > 0) || !(s.eg_inf_s >= 0) || !(s.eg_inf_norm > 0) || !(s.eg_sing_mu > 0) ||
                           !(s.eg_inf_mu < 0)))
    return fail(HC_E_INVALID_ARG, "endgame settings");
  if (s.lane_layout < HC_LAYOUT_AUTO || s.lane_layout > HC_LAYOUT_WIDE) return fail(HC_E_INVALID_ARG, "lane_layout");
  return HC_OK;
}

static bool aligned16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

// Wide latency layout when the throughput layout would leave the GPU mostly idle: at most ~2.5
// waves of one-track-per-warp slots (the wide kernel's resident warps per SM, from the same CTA
// shape as its __launch_bounds__: 16 for N <= 16), i.e.
// small single-instance solves (katsura-6: 64 tracks, cyclic-7: 5040), where the makespan is one
// track's chain of solves and spreading its op list over 32 lanes shortens every solve.
static bool wide_layout(int device, int N, int64_t tracks, int32_t layout) {
  if (layout == HC_LAYOUT_WIDE) return true;
  if (layout == HC_LAYOUT_THROUGHPUT) return false;
  if (const char *ev = getenv("HC_LANES")) {
    if (!strcmp(ev, "wide")) return true;
    if (!strcmp(ev, "narrow")) return false;
  }
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const int64_t slots = (int64_t)sms * tracker_maxw(N, 32) * tracker_minb(N);
  return tracks * 2 <= slots * 5;
}

// NVTX range over a scope (host side: the enqueue, or the whole call for HC_MEM_HOST)
struct NvtxRange {
  explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static hc_status track_batch_impl(hc_system sys, const hc_tracker_settings *settings, const hc_batch *bt,
                                  hc_result *out);
hc_status hc_track_batch(hc_system sys, const hc_tracker_settings *settings, const hc_batch *bt, hc_result *out) {
  NvtxRange range("hc_track_batch");
  return track_batch_impl(sys, settings, bt, out);
}

static hc_status track_batch_impl(hc_system sys, const hc_tracker_settings *settings, const hc_batch *bt,
                                  hc_result *out) {
  if (out) *out = nullptr;
  if (!sys || !bt) return fail(HC_E_INVALID_ARG, "null argument");
  hc_tracker_settings st;
  if (settings) st = *settings;
  else hc_tracker_settings_default(&st);
  hc_status s = check_settings(st);
  if (s != HC_OK) return s;
  const int N = sys->cs.N, P = sys->cs.P;
  if (bt->n_instances < 1 || bt->n_start < 1) return fail(HC_E_INVALID_ARG, "n_instances and n_start must be >= 1");
  if (bt->n_instances > (1LL << 40) / bt->n_start) return fail(HC_E_TOO_LARGE, "too many tracks");
  // ---- lane layout: the wide latency layout (one track per warp, 32 lanes) when the batch
  //      under-fills the GPU in the throughput layout (policy in wide_layout()); HC_LANES=wide|narrow
  //      overrides it (experiments and tests) ----
  const bool wide = sys->has_wide && wide_layout(sys->device, N, bt->n_instances * bt->n_start, st.lane_layout);
  const CompiledSystem &cs = wide ? sys->cs_w : sys->cs;
  const DevTables &dt = wide ? sys->dt_w : sys->dt;
  if (!bt->start_x) return fail(HC_E_INVALID_ARG, "start_x is null");
  if (P > 0 && (!bt->p_start || !bt->p_target)) return fail(HC_E_INVALID_ARG, "p_start / p_target null with P > 0");
  if (bt->memory != HC_MEM_DEVICE && bt->memory != HC_MEM_HOST) return fail(HC_E_INVALID_ARG, "memory");
  const bool host = bt->memory == HC_MEM_HOST;
  if (!host) {
    for (const void *p : {(const void *)bt->start_x, (const void *)bt->p_start, (const void *)bt->p_target,
                          (const void *)bt->x_out, (const void *)bt->counters_out, (const void *)bt->resid_out})
      if (p && !aligned16(p)) return fail(HC_E_INVALID_ARG, "device buffers must be 16-byte aligned");
  }
  const int64_t B = bt->n_instances, S = bt->n_start, total = B * S;

  CK(cudaSetDevice(sys->device));
  (void)cudaGetLastError();   // clear a stale error left by a foreign caller
  hc_result r = new (std::nothrow) hc_result_s();
  if (!r) return fail(HC_E_OOM, "host allocation failed");
  r->sys = sys;
  r->device = sys->device;
  r->stream = reinterpret_cast<cudaStream_t>(bt->stream);
  r->B = B;
  r->S = S;
  r->total = total;
  r->memory = bt->memory;
  auto bail = [&](hc_status e) {
    destroy_result(r);
    return e;
  };
  for (auto &e : r->ev)
    if (cudaEventCreate(&e) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "cudaEventCreate"));

  // ---- inputs on the device ----
  const double2 *d_start = reinterpret_cast<const double2 *>(bt->start_x);
  const double2 *d_p0 = reinterpret_cast<const double2 *>(bt->p_start);
  const double2 *d_p1 = reinterpret_cast<const double2 *>(bt->p_target);
  double2 *d_x = reinterpret_cast<double2 *>(bt->x_out);
  int32_t *d_status = bt->status_out, *d_ctr = bt->counters_out, *d_wind = bt->winding_out;
  double *d_resid = bt->resid_out;
  if (host) {
    double2 *a, *b0 = nullptr, *b1 = nullptr;
    if ((s = dev_alloc(r, &a, (size_t)S * N, true)) != HC_OK) return bail(s);
    if (cudaMemcpyAsync(a, bt->start_x, sizeof(double2) * S * N, cudaMemcpyHostToDevice, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "H2D start_x"));
    d_start = a;
    if (P > 0) {
      if ((s = dev_alloc(r, &b0, (size_t)P, true)) != HC_OK) return bail(s);
      if ((s = dev_alloc(r, &b1, (size_t)B * P, true)) != HC_OK) return bail(s);
      if (cudaMemcpyAsync(b0, bt->p_start, sizeof(double2) * P, cudaMemcpyHostToDevice, r->stream) != cudaSuccess ||
          cudaMemcpyAsync(b1, bt->p_target, sizeof(double2) * B * P, cudaMemcpyHostToDevice, r->stream) != cudaSuccess)
        return bail(cuda_fail(cudaGetLastError(), "H2D params"));
      d_p0 = b0;
      d_p1 = b1;
    }
    d_x = nullptr;
    d_status = nullptr;
    d_ctr = nullptr;
    d_resid = nullptr;
    d_wind = nullptr;
    if (bt->winding_out && (s = dev_alloc(r, &d_wind, (size_t)total)) != HC_OK) return bail(s);
  }
  if (!d_x && (s = dev_alloc(r, &d_x, (size_t)total * N)) != HC_OK) return bail(s);
  if (!d_status && (s = dev_alloc(r, &d_status, (size_t)total)) != HC_OK) return bail(s);
  if (!d_ctr && (s = dev_alloc(r, &d_ctr, (size_t)total * 4)) != HC_OK) return bail(s);
  if (!d_resid && (s = dev_alloc(r, &d_resid, (size_t)total * 2)) != HC_OK) return bail(s);
  double2 *d_coef = nullptr;
  unsigned long long *d_queue = nullptr;
  if ((s = dev_alloc(r, &d_coef, (size_t)B * (cs.D + 1) * cs.ncoef, true)) != HC_OK) return bail(s);
  // work counters: [0] the tracker's queue, [1] tracks handed to the endgame, [2] the endgame's queue
  if ((s = dev_alloc(r, &d_queue, 3, true)) != HC_OK) return bail(s);
  if (cudaMemsetAsync(d_queue, 0, 3 * sizeof(unsigned long long), r->stream) != cudaSuccess)
    return bail(cuda_fail(cudaGetLastError(), "memset queue"));
  int64_t *d_eg_list = nullptr;
  if (st.eg_start > 0.0 && (s = dev_alloc(r, &d_eg_list, (size_t)total, true)) != HC_OK) return bail(s);
  // P == 0: coefficients are constants; feed the prologue a dummy parameter vector
  double2 *d_dummy = nullptr;
  if (P == 0) {
    if ((s = dev_alloc(r, &d_dummy, 1, true)) != HC_OK) return bail(s);
    d_p0 = d_dummy;
    d_p1 = d_dummy;
  }

  // ---- prologue: per-instance coefficient polynomials in t ----
  PrologueArgs pa{};
  pa.mono = dt.d_mono;
  pa.coef_mono_ptr = dt.d_mono_ptr;
  pa.ncoef = cs.ncoef;
  pa.D = cs.D;
  pa.P = P;
  pa.p0 = d_p0;
  pa.p1 = d_p1;
  pa.B = B;
  pa.coef_t = d_coef;
  cudaEventRecord(r->ev[0], r->stream);
  nvtxRangePushA("hc: coefficient prologue");
  cudaError_t e = launch_prologue(pa, r->stream);
  nvtxRangePop();
  if (e != cudaSuccess) return bail(cuda_fail(e, "coef prologue launch"));
  cudaEventRecord(r->ev[1], r->stream);

  // ---- the fused tracker ----
  TrackArgs ta{};
  ta.ops = dt.d_ops;
  ta.Q = dt.Qp ? 2 * dt.Qp : cs.Q;
  ta.Qp = dt.Qp;
  ta.mono_prog = dt.d_mono_prog;
  ta.n_mono = cs.n_mono;
  ta.n_levels = cs.n_levels;
  for (int l = 0; l < MAX_LEVELS; ++l) ta.level_end[l] = cs.level_end[l];
  ta.ncoef = cs.ncoef;
  ta.ncoef_src = cs.ncoef_src;
  ta.mpos = dt.d_mpos;
  ta.n_entries = cs.n_entries;
  ta.D = cs.D;
  ta.coef_t = d_coef;
  ta.start_x = d_start;
  ta.S = S;
  ta.total = total;
  ta.queue = d_queue;
  ta.x_out = d_x;
  ta.status_out = d_status;
  ta.counters_out = d_ctr;
  ta.resid_out = d_resid;
  ta.winding_out = d_wind;
  ta.eg_list = d_eg_list;
  ta.eg_count = d_queue + 1;
  ta.st.eg_start = st.eg_start;
  ta.st.eg_inf_mu = st.eg_inf_mu;
  ta.st.eg_sing_mu = st.eg_sing_mu;
  ta.st.eg_stab = st.eg_stab;
  ta.st.eg_inf_s = st.eg_inf_s;
  ta.st.eg_inf_norm = st.eg_inf_norm;
  ta.st.eg_tol = st.eg_tol;
  ta.st.eg_samples = st.eg_samples;
  ta.st.eg_max_winding = st.eg_max_winding;
  ta.st.eg_max_radii = st.eg_max_radii;
  ta.st.dt_init = st.dt_init;
  ta.st.dt_min = st.dt_min;
  ta.st.dt_max = st.dt_max;
  ta.st.grow = st.grow;
  ta.st.shrink = st.shrink;
  ta.st.newton_tol = st.newton_tol;
  ta.st.inf_norm = st.inf_norm;
  ta.st.end_tol = st.end_tol;
  ta.st.res_abs = st.res_abs;
  ta.st.res_rel = st.res_rel;
  ta.st.pivot_rel = st.pivot_rel;
  ta.st.predictor = st.predictor;
  ta.st.grow_after = st.grow_after;
  ta.st.max_newton = st.max_newton;
  ta.st.max_steps = st.max_steps;
  ta.st.end_newton = st.end_newton;
  ta.phase_cycles = nullptr;
#ifdef HCB_PHASE_TIMING
  {
    unsigned long long *pc = nullptr;
    if ((s = dev_alloc(r, &pc, 8)) != HC_OK) return bail(s);
    cudaMemsetAsync(pc, 0, 64, r->stream);
    ta.phase_cycles = pc;
    r->phase_cycles = pc;
  }
#endif
  nvtxRangePushA("hc: fused tracker");
  e = (wide ? tracker_launcher_wide(N) : tracker_launcher(N))(ta, sys->device, r->stream, &r->plan);
  nvtxRangePop();
  if (e != cudaSuccess) return bail(cuda_fail(e, "tracker launch"));
  cudaEventRecord(r->ev[3], r->stream);
  // ---- the Cauchy endgame (reading R26) over the tracks the tracker handed over; the count stays
  //      on the device, so an empty list costs one short launch and no host synchronisation.  It
  //      runs on the throughput-layout tables (after the wide layout, with their own coefficient
  //      polynomials: slots are relabelled per layout) ----
  if (st.eg_start > 0.0) {
    // the endgame's tracks are a latency chain: it runs in the wide layout (one track per warp on 32
    // lanes) for N <= 16, else in the throughput layout; coefficient slots are bank-relabelled per
    // layout, so a layout other than the tracker's gets its own coefficient polynomials
    const bool eg_wide = sys->has_wide;
    const CompiledSystem &ecs = eg_wide ? sys->cs_w : sys->cs;
    const DevTables &edt = eg_wide ? sys->dt_w : sys->dt;
    TrackArgs ea = ta;
    if (eg_wide != wide) {
      double2 *d_coef_e = nullptr;
      if ((s = dev_alloc(r, &d_coef_e, (size_t)B * (ecs.D + 1) * ecs.ncoef, true)) != HC_OK) return bail(s);
      PrologueArgs pe = pa;
      pe.mono = edt.d_mono;
      pe.coef_mono_ptr = edt.d_mono_ptr;
      pe.ncoef = ecs.ncoef;
      pe.D = ecs.D;
      pe.coef_t = d_coef_e;
      e = launch_prologue(pe, r->stream);
      if (e != cudaSuccess) return bail(cuda_fail(e, "coef prologue launch (endgame tables)"));
      ea.coef_t = d_coef_e;
    }
    ea.ops = edt.d_ops;
    ea.Q = edt.Qp ? 2 * edt.Qp : ecs.Q;
    ea.Qp = edt.Qp;
    ea.mono_prog = edt.d_mono_prog;
    ea.n_mono = ecs.n_mono;
    ea.n_levels = ecs.n_levels;
    for (int l = 0; l < MAX_LEVELS; ++l) ea.level_end[l] = ecs.level_end[l];
    ea.mpos = edt.d_mpos;
    ea.n_entries = ecs.n_entries;
    ea.ncoef = ecs.ncoef;
    ea.ncoef_src = ecs.ncoef_src;
    ea.D = ecs.D;
    nvtxRangePushA("hc: Cauchy endgame");
    e = (eg_wide ? kEndgameWide[N] : kEndgame[N])(ea, sys->device, r->stream);
    nvtxRangePop();
    if (e != cudaSuccess) return bail(cuda_fail(e, "endgame launch"));
  }
  cudaEventRecord(r->ev[2], r->stream);
  // per-batch temporaries (coefficient tables, work counters, endgame list, staged inputs): released
  // in stream order now, so the next batch on this stream reuses them from the pool
  for (void *p : r->temps) cudaFreeAsync(p, r->stream);
  r->temps.clear();

  if (host) {
    if (bt->x_out &&
        cudaMemcpyAsync(bt->x_out, d_x, sizeof(double2) * total * N, cudaMemcpyDeviceToHost, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "D2H x"));
    if (bt->status_out &&
        cudaMemcpyAsync(bt->status_out, d_status, sizeof(int32_t) * total, cudaMemcpyDeviceToHost, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "D2H status"));
    if (bt->counters_out && cudaMemcpyAsync(bt->counters_out, d_ctr, sizeof(int32_t) * total * 4,
                                            cudaMemcpyDeviceToHost, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "D2H counters"));
    if (bt->resid_out && cudaMemcpyAsync(bt->resid_out, d_resid, sizeof(double) * total * 2,
                                         cudaMemcpyDeviceToHost, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "D2H resid"));
    if (bt->winding_out && cudaMemcpyAsync(bt->winding_out, d_wind, sizeof(int32_t) * total,
                                           cudaMemcpyDeviceToHost, r->stream) != cudaSuccess)
      return bail(cuda_fail(cudaGetLastError(), "D2H winding"));
    if (cudaStreamSynchronize(r->stream) != cudaSuccess) return bail(cuda_fail(cudaGetLastError(), "sync"));
    r->waited = true;
  }
  r->x = reinterpret_cast<hc_complex *>(d_x);
  r->status = d_status;
  r->counters = d_ctr;
  r->resid = d_resid;
  r->winding = d_wind;
  if (out) *out = r;
  else if (!host) {
    // fire-and-forget: the caller owns all outputs; release our buffers after the stream passes
    destroy_result(r);
  } else {
    destroy_result(r);
  }
  return HC_OK;
}

hc_status hc_result_wait(hc_result r) {
  if (!r) return fail(HC_E_INVALID_ARG, "null result");
  CK(cudaSetDevice(r->device));
  CK(cudaEventSynchronize(r->ev[2]));
  r->waited = true;
  return HC_OK;
}

hc_status hc_result_elapsed_ms(hc_result r, float *total, float *prologue, float *tracker) {
  if (!r) return fail(HC_E_INVALID_ARG, "null result");
  hc_status s = hc_result_wait(r);
  if (s != HC_OK) return s;
  float a = 0, b = 0, c = 0;
  CK(cudaEventElapsedTime(&a, r->ev[0], r->ev[2]));
  CK(cudaEventElapsedTime(&b, r->ev[0], r->ev[1]));
  CK(cudaEventElapsedTime(&c, r->ev[1], r->ev[3]));   // the tracker kernel alone (not the endgame)
  if (total) *total = a;
  if (prologue) *prologue = b;
  if (tracker) *tracker = c;
  return HC_OK;
}

hc_status hc_result_launch(hc_result r, int32_t *lanes, int32_t *warps_per_cta, int32_t *ctas, int64_t *smem_bytes) {
  if (!r) return fail(HC_E_INVALID_ARG, "null result");
  if (lanes) *lanes = r->plan.lanes;
  if (warps_per_cta) *warps_per_cta = r->plan.warps_per_cta;
  if (ctas) *ctas = r->plan.ctas;
  if (smem_bytes) *smem_bytes = (int64_t)r->plan.smem_bytes;
  return HC_OK;
}

// Experiment builds (-DHCB_PHASE_TIMING) only: per-phase cycle sums of the tracker kernel.
hc_status hc_debug_phase_cycles(hc_result r, unsigned long long *out8) {
  if (!r || !out8) return fail(HC_E_INVALID_ARG, "null");
  if (!r->phase_cycles) return fail(HC_E_INVALID_ARG, "not a phase-timing build");
  hc_status s = hc_result_wait(r);
  if (s != HC_OK) return s;
  CK(cudaMemcpy(out8, r->phase_cycles, 64, cudaMemcpyDeviceToHost));
  return HC_OK;
}

hc_status hc_result_get(hc_result r, int64_t instance, int64_t track, hc_complex *x, hc_track_info *info) {
  if (!r) return fail(HC_E_INVALID_ARG, "null result");
  if (instance < 0 || instance >= r->B || track < 0 || track >= r->S) return fail(HC_E_INVALID_ARG, "index out of range");
  hc_status s = hc_result_wait(r);
  if (s != HC_OK) return s;
  const int N = r->sys->cs.N;
  const int64_t g = instance * r->S + track;
  if (x) CK(cudaMemcpy(x, r->x + g * N, sizeof(hc_complex) * N, cudaMemcpyDeviceToHost));
  if (info) {
    int32_t c[4], st;
    double rs[2];
    CK(cudaMemcpy(&st, r->status + g, sizeof(int32_t), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(c, r->counters + 4 * g, sizeof(c), cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(rs, r->resid + 2 * g, sizeof(rs), cudaMemcpyDeviceToHost));
    info->status = st;
    info->steps = c[0];
    info->rejections = c[1];
    info->newton_iters = c[2];
    info->solves = c[3];
    info->resid_abs = rs[0];
    info->resid_rel = rs[1];
  }
  return HC_OK;
}

hc_status hc_result_destroy(hc_result r) {
  destroy_result(r);
  return HC_OK;
}

hc_status hc_batched_zgesv(int32_t n, int64_t batch, const hc_complex *A, const hc_complex *b, hc_complex *x,
                           int32_t *info, double pivot_rel, void *stream) {
  if (n < 1 || n > 32) return fail(n > 32 ? HC_E_TOO_LARGE : HC_E_INVALID_ARG, "n must be in [1, 32]");
  if (batch < 0) return fail(HC_E_INVALID_ARG, "batch < 0");
  if (batch > 0 && (!A || !b || !x || !info)) return fail(HC_E_INVALID_ARG, "null pointer");
  cudaError_t e = launch_batched_zgesv(n, batch, reinterpret_cast<const double2 *>(A),
                                       reinterpret_cast<const double2 *>(b), reinterpret_cast<double2 *>(x), info,
                                       pivot_rel, reinterpret_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return cuda_fail(e, "batched zgesv");
  return HC_OK;
}

hc_status hc_fp64_peak_probe(int device, double *tflops) {
  if (!tflops) return fail(HC_E_INVALID_ARG, "null");
  cudaError_t e = run_fp64_probe(device, tflops);
  if (e != cudaSuccess) return cuda_fail(e, "fp64 probe");
  return HC_OK;
}

}  // extern "C"
