// compiler.cpp -- the host system compiler.
//
// The paper homogenises every entry of dH/dx, dH/dt and H into K padded terms
// (s_k, a_{k,j}, x_{k,m1..mM}) with a constant-one variable so a warp can evaluate them in a
// uniform format, one Jacobian row per thread.  Padding every entry to K
// terms wastes most of the work on sparse vision systems (trifocal J: 648 real of 3888 padded
// terms), and row-per-thread leaves lanes idle when rows differ in length.  Here the same
// homogeneous term record is kept (coefficient index, integer scale s_k, up to M factor indices,
// constant-one slot for unused factors), but entries are bin-packed over the L lanes of a track
// (longest-processing-time first), so each lane runs ~(total terms / L) ops, and each lane step q
// carries the max factor count of its ops so the product loop is uniform across the warp.
#include "compiler.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <sstream>

namespace hcb {

namespace {

struct RawOp {
  int coef;
  int scale;
  bool rhs;
  std::vector<int> fac;   // factor variable indices (repeated for powers)
};

struct Entry {
  int dest;               // row * (N + 1) + col
  std::vector<RawOp> ops;
  int64_t cost = 0;
  int maxnf = 0;
};

int64_t term_flops(int nf, int scale) {
  // a term of total degree d costs 6(d-1) + 8 (complex products, then a complex
  // FMA with the coefficient), a constant costs 2 (complex add); +2 for a real scale s_k != 1.
  int64_t f = (nf >= 1) ? 6 * (nf - 1) + 8 : 2;
  if (scale != 1) f += 2;
  return f;
}

}  // namespace

int64_t lu_flops(int N) {
  // augmented elimination sum_{j=0}^{N-1} j (6 + 8 (j+1)) + back-substitution
  // 8 N (N-1) / 2 + 6 N.
  int64_t f = 0;
  for (int j = 0; j < N; ++j) f += (int64_t)j * (6 + 8 * (j + 1));
  f += 8LL * N * (N - 1) / 2 + 6LL * N;
  return f;
}

hc_system_desc OwnedDesc::view() const {
  hc_system_desc d{};
  d.n_vars = n_vars;
  d.n_params = n_params;
  d.n_terms = n_terms;
  d.term_eq = term_eq.data();
  d.term_xexp = term_xexp.data();
  d.term_coef = term_coef.data();
  d.n_coefs = n_coefs;
  d.coef_ptr = coef_ptr.data();
  d.coef_w = coef_w.data();
  d.coef_pexp = coef_pexp.empty() ? nullptr : coef_pexp.data();
  return d;
}

static hc_status validate(const hc_system_desc &d, std::string &err) {
  std::ostringstream os;
  if (d.n_vars < 1 || d.n_vars > HC_MAX_VARS) {
    os << "n_vars must be in [1, " << HC_MAX_VARS << "], got " << d.n_vars;
    err = os.str();
    return d.n_vars > HC_MAX_VARS ? HC_E_TOO_LARGE : HC_E_INVALID_ARG;
  }
  if (d.n_params < 0 || d.n_terms < 1 || d.n_coefs < 1) {
    err = "n_params >= 0, n_terms >= 1 and n_coefs >= 1 required";
    return HC_E_INVALID_ARG;
  }
  if (!d.term_eq || !d.term_xexp || !d.term_coef || !d.coef_ptr || !d.coef_w || (d.n_params > 0 && !d.coef_pexp)) {
    err = "null descriptor array";
    return HC_E_INVALID_ARG;
  }
  if (d.n_coefs > 65535) {
    err = "more than 65535 coefficient expressions";
    return HC_E_TOO_LARGE;
  }
  std::vector<int> seen_eq(d.n_vars, 0);
  for (int k = 0; k < d.n_terms; ++k) {
    if (d.term_eq[k] < 0 || d.term_eq[k] >= d.n_vars) {
      err = "term_eq out of range at term " + std::to_string(k);
      return HC_E_INVALID_ARG;
    }
    seen_eq[d.term_eq[k]] = 1;
    if (d.term_coef[k] < 0 || d.term_coef[k] >= d.n_coefs) {
      err = "term_coef out of range at term " + std::to_string(k);
      return HC_E_INVALID_ARG;
    }
    for (int v = 0; v < d.n_vars; ++v)
      if (d.term_xexp[(size_t)k * d.n_vars + v] < 0 || d.term_xexp[(size_t)k * d.n_vars + v] > 255) {
        err = "term exponent out of range [0, 255] at term " + std::to_string(k);
        return HC_E_INVALID_ARG;
      }
  }
  for (int i = 0; i < d.n_vars; ++i)
    if (!seen_eq[i]) {
      err = "equation " + std::to_string(i) + " has no terms (system not square)";
      return HC_E_INVALID_ARG;
    }
  if (d.coef_ptr[0] != 0) {
    err = "coef_ptr[0] must be 0";
    return HC_E_INVALID_ARG;
  }
  for (int j = 0; j < d.n_coefs; ++j)
    if (d.coef_ptr[j + 1] < d.coef_ptr[j]) {
      err = "coef_ptr not non-decreasing";
      return HC_E_INVALID_ARG;
    }
  const int nnz = d.coef_ptr[d.n_coefs];
  for (int m = 0; m < nnz; ++m) {
    if (!std::isfinite(d.coef_w[m].re) || !std::isfinite(d.coef_w[m].im)) {
      err = "non-finite coefficient weight at " + std::to_string(m);
      return HC_E_INVALID_ARG;
    }
    for (int q = 0; q < d.n_params; ++q)
      if (d.coef_pexp[(size_t)m * d.n_params + q] < 0) {
        err = "negative parameter exponent";
        return HC_E_INVALID_ARG;
      }
  }
  return HC_OK;
}

hc_status compile_system(const hc_system_desc &d, CompiledSystem &cs, std::string &err) {
  hc_status s = validate(d, err);
  if (s != HC_OK) return s;
  const int N = d.n_vars, P = d.n_params;
  cs = CompiledSystem();
  cs.N = N;
  cs.P = P;
  cs.ncoef = d.n_coefs;
  cs.n_terms = d.n_terms;
  cs.L = lanes_for(N);

  // ---- coefficient expressions -> monomials in p with repeated factor lists ----
  cs.mono_ptr.assign(d.n_coefs + 1, 0);
  int D = 0;
  for (int j = 0; j < d.n_coefs; ++j) {
    for (int m = d.coef_ptr[j]; m < d.coef_ptr[j + 1]; ++m) {
      CoefMono mo{};
      mo.wre = d.coef_w[m].re;
      mo.wim = d.coef_w[m].im;
      mo.coef = j;
      int deg = 0;
      for (int q = 0; q < P; ++q) {
        const int e = d.coef_pexp[(size_t)m * P + q];
        for (int r = 0; r < e; ++r) {
          if (deg >= MAX_COEF_DEG) {
            err = "coefficient expression of degree > " + std::to_string(MAX_COEF_DEG) + " in the parameters";
            return HC_E_TOO_LARGE;
          }
          mo.fac[deg++] = (int16_t)q;
        }
      }
      mo.deg = deg;
      D = std::max(D, deg);
      cs.mono.push_back(mo);
    }
    cs.mono_ptr[j + 1] = (int32_t)cs.mono.size();
  }
  cs.D = D;

  // ---- degrees ----
  cs.degrees.assign(N, 0);
  for (int k = 0; k < d.n_terms; ++k) {
    int tot = 0;
    for (int v = 0; v < N; ++v) tot += d.term_xexp[(size_t)k * N + v];
    cs.degrees[d.term_eq[k]] = std::max(cs.degrees[d.term_eq[k]], tot);
  }

  // ---- ops: rhs entries (H / dH/dt, column N) and Jacobian entries (exponent decrement) ----
  std::map<int, Entry> entries;
  auto add_op = [&](int row, int col, RawOp op) -> bool {
    if ((int)op.fac.size() > MAX_FACTORS) return false;
    const int dest = row * (N + 1) + col;
    Entry &e = entries[dest];
    e.dest = dest;
    e.ops.push_back(std::move(op));
    return true;
  };
  for (int k = 0; k < d.n_terms; ++k) {
    const int i = d.term_eq[k], j = d.term_coef[k];
    const int32_t *e = d.term_xexp + (size_t)k * N;
    RawOp h{j, 1, true, {}};
    for (int v = 0; v < N; ++v)
      for (int r = 0; r < e[v]; ++r) h.fac.push_back(v);
    if (!add_op(i, N, h)) {
      err = "term of total degree > " + std::to_string(MAX_FACTORS);
      return HC_E_TOO_LARGE;
    }
    cs.n_ops_rhs++;
    for (int v = 0; v < N; ++v) {
      if (e[v] == 0) continue;
      RawOp jo{j, e[v], false, {}};
      for (int u = 0; u < N; ++u)
        for (int r = 0; r < (u == v ? e[u] - 1 : e[u]); ++r) jo.fac.push_back(u);
      add_op(i, v, jo);
      cs.n_ops_J++;
    }
  }
  // ---- flop model ----
  cs.flops_eval = 0;
  int M = 0;
  for (auto &kv : entries) {
    Entry &e = kv.second;
    std::sort(e.ops.begin(), e.ops.end(), [](const RawOp &a, const RawOp &b) { return a.fac.size() > b.fac.size(); });
    for (const RawOp &o : e.ops) {
      cs.flops_eval += term_flops((int)o.fac.size(), o.scale);
      e.cost += (int64_t)o.fac.size() + 2;
      e.maxnf = std::max(e.maxnf, (int)o.fac.size());
      M = std::max(M, (int)o.fac.size());
    }
  }
  cs.M = M;
  cs.flops_coef = (int64_t)d.n_coefs * 8 * D;
  cs.flops_lu = lu_flops(N);
  cs.flops_solve = cs.flops_coef + cs.flops_eval + cs.flops_lu + 8LL * N;

  // ---- lane balancing: LPT bin packing of entries over L lanes ----
  const int L = cs.L;
  std::vector<Entry *> order;
  for (auto &kv : entries) order.push_back(&kv.second);
  std::stable_sort(order.begin(), order.end(), [](const Entry *a, const Entry *b) { return a->cost > b->cost; });
  std::vector<std::vector<Entry *>> lane_entries(L);
  std::vector<int64_t> load(L, 0);
  for (Entry *e : order) {
    const int l = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    lane_entries[l].push_back(e);
    load[l] += e->cost;
  }
  std::vector<std::vector<const RawOp *>> lane_ops(L);
  std::vector<std::vector<int>> lane_last(L);   // dest for last op of an entry, -1 otherwise
  for (int l = 0; l < L; ++l) {
    auto &es = lane_entries[l];
    std::stable_sort(es.begin(), es.end(), [](const Entry *a, const Entry *b) { return a->maxnf > b->maxnf; });
    for (const Entry *e : es)
      for (size_t k = 0; k < e->ops.size(); ++k) {
        lane_ops[l].push_back(&e->ops[k]);
        lane_last[l].push_back(k + 1 == e->ops.size() ? e->dest : -1);
      }
  }
  int Q = 0;
  for (int l = 0; l < L; ++l) Q = std::max(Q, (int)lane_ops[l].size());
  cs.Q = Q;
  cs.ops.assign((size_t)Q * L, uint4{});
  cs.step_nfac.assign(Q, 0);
  for (int q = 0; q < Q; ++q) {
    int nf = 0;
    for (int l = 0; l < L; ++l) {
      uint4 w;
      uint8_t f[MAX_FACTORS];
      for (int m = 0; m < MAX_FACTORS; ++m) f[m] = (uint8_t)N;   // constant-one slot
      if (q < (int)lane_ops[l].size()) {
        const RawOp *o = lane_ops[l][q];
        const int dest = lane_last[l][q];
        w.x = (uint32_t)o->coef | ((uint32_t)(dest < 0 ? OP_NO_DEST : (uint32_t)dest) << 16);
        w.y = (dest >= 0 ? OP_LAST : 0u) | (o->rhs ? OP_RHS : 0u) | ((uint32_t)(o->scale & 0xFF) << 8);
        for (size_t m = 0; m < o->fac.size(); ++m) f[m] = (uint8_t)o->fac[m];
        nf = std::max(nf, (int)o->fac.size());
      } else {
        // padding op: scale 0, no store, coefficient 0 (any valid index), all factors = 1
        w.x = 0u | (OP_NO_DEST << 16);
        w.y = 0u;
      }
      w.z = (uint32_t)f[0] | ((uint32_t)f[1] << 8) | ((uint32_t)f[2] << 16) | ((uint32_t)f[3] << 24);
      w.w = (uint32_t)f[4] | ((uint32_t)f[5] << 8) | ((uint32_t)f[6] << 16) | ((uint32_t)f[7] << 24);
      cs.ops[(size_t)q * L + l] = w;
    }
    cs.step_nfac[q] = (uint8_t)nf;
  }
  return HC_OK;
}

hc_status total_degree_desc(const hc_system_desc &F, OwnedDesc &out, std::vector<hc_complex> &fvals,
                            std::vector<int32_t> &degrees, std::string &err) {
  hc_status s = validate(F, err);
  if (s != HC_OK) return s;
  const int N = F.n_vars;
  // target coefficient values (constant coefficients required)
  fvals.assign(F.n_coefs, hc_complex{0.0, 0.0});
  for (int j = 0; j < F.n_coefs; ++j)
    for (int m = F.coef_ptr[j]; m < F.coef_ptr[j + 1]; ++m) {
      for (int q = 0; q < F.n_params; ++q)
        if (F.coef_pexp[(size_t)m * F.n_params + q] != 0) {
          err = "total-degree target must have constant coefficients";
          return HC_E_INVALID_ARG;
        }
      fvals[j].re += F.coef_w[m].re;
      fvals[j].im += F.coef_w[m].im;
    }
  degrees.assign(N, 0);
  for (int k = 0; k < F.n_terms; ++k) {
    int tot = 0;
    for (int v = 0; v < N; ++v) tot += F.term_xexp[(size_t)k * N + v];
    degrees[F.term_eq[k]] = std::max(degrees[F.term_eq[k]], tot);
  }
  for (int i = 0; i < N; ++i)
    if (degrees[i] < 1) {
      err = "equation " + std::to_string(i) + " is constant";
      return HC_E_INVALID_ARG;
    }
  out = OwnedDesc();
  out.n_vars = N;
  out.n_params = 2 * N + F.n_coefs;
  out.n_coefs = 2 * N + F.n_coefs;   // one coefficient expression per parameter: c_q(p) = p_q
  out.n_terms = 2 * N + F.n_terms;
  const int P = out.n_params;
  for (int i = 0; i < N; ++i) {   // G_i = x_i^{d_i} - 1: coefficient p_i on x_i^{d_i}, p_{N+i} on 1
    out.term_eq.push_back(i);
    for (int v = 0; v < N; ++v) out.term_xexp.push_back(v == i ? degrees[i] : 0);
    out.term_coef.push_back(i);
    out.term_eq.push_back(i);
    for (int v = 0; v < N; ++v) out.term_xexp.push_back(0);
    out.term_coef.push_back(N + i);
  }
  for (int k = 0; k < F.n_terms; ++k) {
    out.term_eq.push_back(F.term_eq[k]);
    for (int v = 0; v < N; ++v) out.term_xexp.push_back(F.term_xexp[(size_t)k * N + v]);
    out.term_coef.push_back(2 * N + F.term_coef[k]);
  }
  out.coef_ptr.resize(out.n_coefs + 1);
  out.coef_pexp.assign((size_t)out.n_coefs * P, 0);
  for (int q = 0; q < out.n_coefs; ++q) {
    out.coef_ptr[q] = q;
    out.coef_w.push_back(hc_complex{1.0, 0.0});
    out.coef_pexp[(size_t)q * P + q] = 1;
  }
  out.coef_ptr[out.n_coefs] = out.n_coefs;
  return HC_OK;
}

}  // namespace hcb
