// compiler.cpp -- the host system compiler.
//
// The paper homogenises every entry of dH/dx, dH/dt and H into K padded terms
// (s_k, a_{k,j}, x_{k,m1..mM}) with a constant-one variable so a warp can evaluate them in a
// uniform format, one Jacobian row per thread.  Padding every entry to K
// terms wastes most of the work on sparse vision systems (trifocal J: 648 real of 3888 padded
// terms), row-per-thread leaves lanes idle when rows differ in length, and every term re-multiplies
// its M factors.  Here the homogeneous record survives as (coefficient slot, monomial index):
//  * s_k is folded into the coefficient (a slot per distinct (c_j, s_k)), evaluated by the
//    prologue as a polynomial in t;
//  * the products x_{m1} ... x_{mM} are shared: every monomial any entry needs is computed once
//    per evaluation as the product of two monomials of lower degree (a monomial program in
//    ceil(log2(max degree)) dependent levels; the unknowns and the constant one are its first N+1
//    slots);
//  * entries are bin-packed over the L lanes of a track (longest-processing-time first), so each
//    lane runs ~(total terms / L) uniform ops out(row,col) += coef[slot] * mono[k].
#include "compiler.h"

#include <algorithm>
#include <cmath>
#include <map>
#include <numeric>
#include <set>
#include <sstream>

namespace hcb {

namespace {

typedef std::vector<int> Expo;   // exponent vector of a monomial in x

struct RawOp {
  int slot;       // coefficient slot (scale folded in)
  Expo mono;      // monomial
  int scale;      // s_k (for the flop rule only)
  bool rhs;
};

struct Entry {
  int dest;       // row * (N + 1) + col
  std::vector<RawOp> ops;
};

int deg_of(const Expo &e) { return std::accumulate(e.begin(), e.end(), 0); }

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


// ------------------------------------------------------------------------------------------
// Shared-memory bank relabelling.  The op loop reads coef[slot] and mono[k] with LDS.128: a warp
// request is served in phases of 8 lanes, and two lanes of a phase that read different 16-byte
// entries with the same index mod 8 conflict.  Slot and monomial ids are free up to permutations
// within groups (rhs slots / other slots; monomials of one degree level), so a greedy swap search
// (deterministic seed) minimises sum over (step, phase) of the worst bank multiplicity.
// Returns perm: old label -> new label.
// ------------------------------------------------------------------------------------------
static std::vector<int> bank_relabel(const std::vector<int> &lab, int Q, int L, int nlabels,
                                     const std::vector<std::vector<int>> &groups, uint64_t seed, int iters) {
  const int W = std::min(8, L), P = std::max(1, L / 8), C = Q * P;
  std::vector<int> perm(nlabels);
  std::iota(perm.begin(), perm.end(), 0);
  std::vector<std::vector<int>> cell_labels(C), lab_cells(nlabels);
  for (int q = 0; q < Q; ++q)
    for (int p = 0; p < P; ++p) {
      std::vector<int> v;
      for (int l = p * W; l < p * W + W && l < L; ++l) v.push_back(lab[(size_t)q * L + l]);
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
      const int c = q * P + p;
      cell_labels[c] = v;
      for (int x : v) lab_cells[x].push_back(c);
    }
  auto cell_cost = [&](int c) {
    int b[8] = {0, 0, 0, 0, 0, 0, 0, 0}, m = 0;
    for (int x : cell_labels[c]) m = std::max(m, ++b[perm[x] & 7]);
    return m;
  };
  std::vector<int> cost(C);
  for (int c = 0; c < C; ++c) cost[c] = cell_cost(c);
  std::vector<const std::vector<int> *> gl;
  for (const auto &g : groups)
    if (g.size() > 1) gl.push_back(&g);
  if (gl.empty()) return perm;
  uint64_t st = seed * 0x9E3779B97F4A7C15ull + 1;
  auto rnd = [&]() {
    st ^= st << 13;
    st ^= st >> 7;
    st ^= st << 17;
    return st;
  };
  std::vector<int> stamp(C, -1), cells;
  for (int it = 0; it < iters; ++it) {
    const std::vector<int> &g = *gl[rnd() % gl.size()];
    const int a = g[rnd() % g.size()], b = g[rnd() % g.size()];
    if (a == b) continue;
    cells.clear();
    for (int c : lab_cells[a])
      if (stamp[c] != it) stamp[c] = it, cells.push_back(c);
    for (int c : lab_cells[b])
      if (stamp[c] != it) stamp[c] = it, cells.push_back(c);
    int old = 0, nw = 0;
    for (int c : cells) old += cost[c];
    std::swap(perm[a], perm[b]);
    std::vector<int> nc(cells.size());
    for (size_t i = 0; i < cells.size(); ++i) nw += (nc[i] = cell_cost(cells[i]));
    if (nw <= old) {
      for (size_t i = 0; i < cells.size(); ++i) cost[cells[i]] = nc[i];
    } else {
      std::swap(perm[a], perm[b]);
    }
  }
  return perm;
}

hc_status compile_system(const hc_system_desc &d, CompiledSystem &cs, std::string &err, int lanes) {
  hc_status s = validate(d, err);
  if (s != HC_OK) return s;
  const int N = d.n_vars, P = d.n_params;
  cs = CompiledSystem();
  cs.N = N;
  cs.P = P;
  cs.ncoef_src = d.n_coefs;
  cs.n_terms = d.n_terms;
  cs.L = lanes > 0 ? lanes : lanes_for(N);

  // ---- degrees ----
  cs.degrees.assign(N, 0);
  for (int k = 0; k < d.n_terms; ++k) {
    int tot = 0;
    for (int v = 0; v < N; ++v) tot += d.term_xexp[(size_t)k * N + v];
    cs.degrees[d.term_eq[k]] = std::max(cs.degrees[d.term_eq[k]], tot);
  }

  // ---- ops: H / dH/dt entries (column N) and dH/dx entries by exponent decrement; the exponent
  //      s_k = e_v becomes a coefficient slot s_k * c_j (scale folded into the coefficient) ----
  std::map<std::pair<int, int>, int> slot_of;   // (coef j, scale) -> slot
  std::vector<std::pair<int, int>> slots;
  for (int j = 0; j < d.n_coefs; ++j) {
    slot_of[{j, 1}] = j;
    slots.push_back({j, 1});
  }
  auto slot_for = [&](int j, int e) {
    auto it = slot_of.find({j, e});
    if (it != slot_of.end()) return it->second;
    const int id = (int)slots.size();
    slot_of[{j, e}] = id;
    slots.push_back({j, e});
    return id;
  };
  std::map<int, Entry> entries;
  int maxdeg = 0;
  for (int k = 0; k < d.n_terms; ++k) {
    const int i = d.term_eq[k], j = d.term_coef[k];
    Expo e(d.term_xexp + (size_t)k * N, d.term_xexp + (size_t)(k + 1) * N);
    const int de = deg_of(e);
    if (de > MAX_FACTORS) {
      err = "term of total degree > " + std::to_string(MAX_FACTORS);
      return HC_E_TOO_LARGE;
    }
    maxdeg = std::max(maxdeg, de);
    Entry &er = entries[i * (N + 1) + N];
    er.dest = i * (N + 1) + N;
    er.ops.push_back(RawOp{j, e, 1, true});
    cs.n_ops_rhs++;
    for (int v = 0; v < N; ++v) {
      if (e[v] == 0) continue;
      Expo e2 = e;
      e2[v] -= 1;
      Entry &ej = entries[i * (N + 1) + v];
      ej.dest = i * (N + 1) + v;
      ej.ops.push_back(RawOp{slot_for(j, e[v]), e2, e[v], false});
      cs.n_ops_J++;
    }
  }
  if ((int)slots.size() > 65535) {
    err = "more than 65535 coefficient slots";
    return HC_E_TOO_LARGE;
  }
  cs.ncoef = (int)slots.size();
  cs.M = maxdeg;

  // ---- coefficient slots -> prologue monomials (slot = scale * c_j) ----
  cs.mono_ptr.assign(cs.ncoef + 1, 0);
  cs.slot_map.resize(2 * cs.ncoef);
  int D = 0;
  for (int sl = 0; sl < cs.ncoef; ++sl) {
    const int j = slots[sl].first, sc = slots[sl].second;
    cs.slot_map[2 * sl] = j;
    cs.slot_map[2 * sl + 1] = sc;
    for (int m = d.coef_ptr[j]; m < d.coef_ptr[j + 1]; ++m) {
      CoefMono mo{};
      mo.wre = d.coef_w[m].re * sc;
      mo.wim = d.coef_w[m].im * sc;
      mo.coef = sl;
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
    cs.mono_ptr[sl + 1] = (int32_t)cs.mono.size();
  }
  cs.D = D;

  // ---- monomial program: every needed monomial of degree d >= 2 is one complex product of two
  //      monomials from earlier levels.  Log depth: level(d) = ceil(log2 d) (degree 2 -> 1, 3-4 -> 2,
  //      5-8 -> 3), i.e. ceil(log2 maxdeg) dependent levels (a warp sync each) instead of
  //      maxdeg - 1.  The split e = a * b (deg a >= deg b, level(deg a) < level(d)) prefers factors
  //      that are needed anyway (shared work), then the most balanced split. ----
  auto log_level = [](int dg) {
    int l = 0;
    while ((1 << l) < dg) ++l;
    return l;   // 1 -> 0, 2 -> 1, 3..4 -> 2, 5..8 -> 3
  };
  // log depth only when it saves at least two levels: with a single level saved the products whose
  // both operands are arbitrary monomials (instead of monomial x variable) cost more in bank
  // conflicts than the saved level (measured: trifocal, max degree 5, +1.5 %; cyclic-7, max degree
  // 7, 6 -> 3 levels, -3 %).  Otherwise the classic program: degree d = (degree d-1) x variable.
  const bool logdepth = maxdeg >= 2 && log_level(maxdeg) + 2 <= maxdeg - 1;
  auto level_of = [&](int dg) { return logdepth ? log_level(dg) : dg - 1; };
  std::map<Expo, int> mono_idx;
  std::set<Expo> need;
  for (auto &kv : entries)
    for (const RawOp &o : kv.second.ops)
      if (deg_of(o.mono) >= 2) need.insert(o.mono);
  std::vector<std::set<Expo>> by_deg(maxdeg + 1);
  for (const Expo &e : need) by_deg[deg_of(e)].insert(e);
  std::map<Expo, std::pair<Expo, Expo>> split;   // monomial -> (a, b)
  for (int dg = maxdeg; dg >= 2; --dg) {
    const int T = level_of(dg);
    for (const Expo &e : by_deg[dg]) {
      if (!logdepth) {
        // classic program: a parent of degree d-1 times a variable; prefer a parent that is already
        // needed (shared work, lowest variable first), else divide by the highest variable
        int best = -1;
        for (int v = 0; v < N && best < 0; ++v) {
          if (!e[v]) continue;
          Expo p2 = e;
          p2[v] -= 1;
          if (dg - 1 < 2 || by_deg[dg - 1].count(p2)) best = v;
        }
        if (best < 0)
          for (int v = N - 1; v >= 0; --v)
            if (e[v]) {
              best = v;
              break;
            }
        Expo p2 = e, xv(N, 0);
        p2[best] -= 1;
        xv[best] = 1;
        if (dg - 1 >= 2) by_deg[dg - 1].insert(p2);
        split[e] = {p2, xv};
        continue;
      }
      // log depth: enumerate sub-multisets a of e (the larger factor); b = e - a
      std::vector<int> fac;
      for (int v = 0; v < N; ++v)
        for (int c = 0; c < e[v]; ++c) fac.push_back(v);
      std::set<Expo> seen;
      int best_score = -1;
      std::pair<Expo, Expo> best;
      const int nf = (int)fac.size();
      for (int mask = 1; mask < (1 << nf); ++mask) {
        const int da = __builtin_popcount((unsigned)mask), db = dg - da;
        if (db < 1 || da < db || level_of(da) >= T) continue;
        Expo a(N, 0);
        for (int i = 0; i < nf; ++i)
          if (mask >> i & 1) a[fac[i]] += 1;
        if (!seen.insert(a).second) continue;
        Expo b = e;
        for (int v = 0; v < N; ++v) b[v] -= a[v];
        auto have = [&](const Expo &m) { const int dm = deg_of(m); return dm < 2 || by_deg[dm].count(m) > 0; };
        // score: factors already present count most, then balance (larger deg b)
        const int score = 100 * ((int)have(a) + (int)have(b)) + db;
        if (score > best_score) {
          best_score = score;
          best = {a, b};
        }
      }
      split[e] = best;
      if (deg_of(best.first) >= 2) by_deg[deg_of(best.first)].insert(best.first);
      if (deg_of(best.second) >= 2) by_deg[deg_of(best.second)].insert(best.second);
    }
  }
  auto index_of = [&](const Expo &e) -> int {
    const int dg = deg_of(e);
    if (dg == 0) return N;
    if (dg == 1)
      for (int v = 0; v < N; ++v)
        if (e[v]) return v;
    return mono_idx.at(e);
  };
  int next = N + 1;
  cs.n_levels = maxdeg >= 2 ? level_of(maxdeg) : 0;
  if (cs.n_levels > MAX_LEVELS) {
    err = "monomial degree too large";
    return HC_E_TOO_LARGE;
  }
  for (int l = 1; l <= cs.n_levels; ++l) {
    for (int dg = 2; dg <= maxdeg; ++dg) {
      if (level_of(dg) != l) continue;
      for (const Expo &e : by_deg[dg]) mono_idx[e] = next++;
    }
    // program entries in index order (the loop above numbers a level's monomials consecutively)
    for (int dg = 2; dg <= maxdeg; ++dg) {
      if (level_of(dg) != l) continue;
      for (const Expo &e : by_deg[dg]) {
        const auto &ab = split.at(e);
        cs.mono_prog.push_back((uint32_t)index_of(ab.first) | ((uint32_t)index_of(ab.second) << 16));
      }
    }
    cs.level_end[l - 1] = next;
  }
  cs.n_mono = next;
  if (cs.n_mono > 65535) {
    err = "too many monomials";
    return HC_E_TOO_LARGE;
  }

  // ---- flop models ----
  cs.flops_eval = 0;
  for (auto &kv : entries)
    for (const RawOp &o : kv.second.ops) cs.flops_eval += term_flops(deg_of(o.mono), o.scale);
  cs.flops_eval_kernel = 6LL * (cs.n_mono - N - 1) + 8LL * (cs.n_ops_J + cs.n_ops_rhs);
  cs.flops_coef = (int64_t)d.n_coefs * 8 * D;
  cs.flops_lu = lu_flops(N);
  cs.flops_solve = cs.flops_coef + cs.flops_eval + cs.flops_lu + 8LL * N;
  cs.flops_solve_kernel = (int64_t)cs.ncoef * 8 * D + cs.flops_eval_kernel + cs.flops_lu + 8LL * N;

  // ---- lane balancing: LPT bin packing of entries (cost = ops + 1 store) over the L lanes ----
  const int L = cs.L;
  std::vector<Entry *> order;
  for (auto &kv : entries) order.push_back(&kv.second);
  std::stable_sort(order.begin(), order.end(),
                   [](const Entry *a, const Entry *b) { return a->ops.size() > b->ops.size(); });
  std::vector<std::vector<Entry *>> lane_entries(L);
  std::vector<int64_t> load(L, 0);
  for (Entry *e : order) {
    const int l = (int)(std::min_element(load.begin(), load.end()) - load.begin());
    lane_entries[l].push_back(e);
    load[l] += (int64_t)e->ops.size() + 1;
  }
  int Q = 0;
  for (int l = 0; l < L; ++l) {
    int n = 0;
    for (const Entry *e : lane_entries[l]) n += (int)e->ops.size();
    Q = std::max(Q, n);
  }
  // the kernel runs the op list in blocks of 4 with all loads of a block issued first; a ragged
  // tail runs one op per shared-memory round trip.  In the wide latency layout the list is padded
  // to whole blocks (padding ops are neutral: never stored): measured -3..5 % per solve there, but
  // +1 % in the throughput layout, where the extra work outweighs the shorter chain.
  if (cs.L != lanes_for(N)) Q = (Q + 3) & ~3;
  cs.Q = Q;
  // compact entry numbering: row-major order of the structurally non-zero entries
  cs.mpos.assign((size_t)N * (N + 1), (int16_t)-1);
  {
    int c = 0;
    for (auto &kv : entries) cs.mpos[kv.first] = (int16_t)c++;   // std::map iterates row-major
    cs.n_entries = c;
  }
  cs.ops.assign((size_t)Q * L, uint2{0u, OP_NO_DEST});
  for (int l = 0; l < L; ++l) {
    int q = 0;
    for (const Entry *e : lane_entries[l])
      for (size_t k = 0; k < e->ops.size(); ++k, ++q) {
        const RawOp &o = e->ops[k];
        const bool last = (k + 1 == e->ops.size());
        uint2 w;
        w.x = (uint32_t)o.slot | ((uint32_t)index_of(o.mono) << 16);
        w.y = (last ? (uint32_t)cs.mpos[e->dest] : OP_NO_DEST) | ((last ? OP_LAST : 0u) | (o.rhs ? OP_RHS : 0u)) << 16;
        cs.ops[(size_t)q * L + l] = w;
      }
    // padding ops after the lane's last entry: slot 0 times the constant monomial, never stored
    for (; q < Q; ++q) cs.ops[(size_t)q * L + l] = uint2{(uint32_t)N << 16, OP_NO_DEST};
  }

  // ---- bank relabelling of coefficient slots and monomials (see bank_relabel) ----
  {
    const int nsrc = d.n_coefs;
    std::vector<int> sl((size_t)Q * L), mo((size_t)Q * L);
    for (size_t i = 0; i < cs.ops.size(); ++i) {
      sl[i] = (int)(cs.ops[i].x & 0xFFFFu);
      mo[i] = (int)(cs.ops[i].x >> 16);
    }
    std::vector<std::vector<int>> sg(2);
    for (int j = 0; j < cs.ncoef; ++j) sg[j < nsrc ? 0 : 1].push_back(j);
    const std::vector<int> ps = bank_relabel(sl, Q, L, cs.ncoef, sg, 2112, 40000);
    std::vector<std::vector<int>> mg(std::max(1, cs.n_levels));
    for (int k = N + 1, lvl = 0; k < cs.n_mono; ++k) {
      while (k >= cs.level_end[lvl]) ++lvl;
      mg[lvl].push_back(k);
    }
    const std::vector<int> pm = bank_relabel(mo, Q, L, cs.n_mono, mg, 3444, 40000);
    for (auto &w : cs.ops) w.x = (uint32_t)ps[w.x & 0xFFFFu] | ((uint32_t)pm[w.x >> 16] << 16);
    // monomial program in the new numbering (permutations stay within a level)
    std::vector<uint32_t> prog(cs.mono_prog.size());
    for (int k = N + 1; k < cs.n_mono; ++k) {
      const uint32_t e = cs.mono_prog[k - N - 1];
      const int fa = (int)(e & 0xFFFFu), fb = (int)(e >> 16);
      prog[pm[k] - N - 1] = (uint32_t)pm[fa] | ((uint32_t)pm[fb] << 16);
    }
    cs.mono_prog = prog;
    // coefficient slots in the new numbering; pad the slot count to a multiple of 8 so that the
    // c'(t) copy (slot + ncoef) falls in the same bank group as c(t)
    const int ncoef_pad = (cs.ncoef + 7) & ~7;
    std::vector<int32_t> smap(2 * ncoef_pad, 0);
    std::vector<std::vector<CoefMono>> per(ncoef_pad);
    for (int j = 0; j < cs.ncoef; ++j) {
      smap[2 * ps[j]] = cs.slot_map[2 * j];
      smap[2 * ps[j] + 1] = cs.slot_map[2 * j + 1];
      for (int m = cs.mono_ptr[j]; m < cs.mono_ptr[j + 1]; ++m) {
        CoefMono c = cs.mono[m];
        c.coef = ps[j];
        per[ps[j]].push_back(c);
      }
    }
    for (int j = cs.ncoef; j < ncoef_pad; ++j) {   // padding slots: zero coefficient, weight-0 monomial
      smap[2 * j] = 0;
      smap[2 * j + 1] = 0;
    }
    cs.mono.clear();
    cs.mono_ptr.assign(ncoef_pad + 1, 0);
    for (int j = 0; j < ncoef_pad; ++j) {
      for (const CoefMono &c : per[j]) cs.mono.push_back(c);
      cs.mono_ptr[j + 1] = (int32_t)cs.mono.size();
    }
    cs.slot_map = smap;
    cs.ncoef = ncoef_pad;
  }
  // ---- bank relabelling of the compact entries for the row loads (lane r reads row r's column
  //      j at step j; structural zeros all read the single zero entry, a broadcast) ----
  {
    const int NE = cs.n_entries;
    const int Lr = cs.L;
    std::vector<int> lab((size_t)(N + 1) * Lr, NE);
    for (int j = 0; j <= N; ++j)
      for (int r = 0; r < Lr && r < N; ++r) {
        const int e = cs.mpos[(size_t)r * (N + 1) + j];
        lab[(size_t)j * Lr + r] = e < 0 ? NE : e;
      }
    std::vector<std::vector<int>> eg(1);
    for (int e = 0; e < NE; ++e) eg[0].push_back(e);
    const std::vector<int> pe = bank_relabel(lab, N + 1, Lr, NE + 1, eg, 2021, 20000);
    for (auto &v : cs.mpos)
      if (v >= 0) v = (int16_t)pe[v];
    for (auto &w : cs.ops) {
      const uint32_t dest = w.y & 0xFFFFu;
      if (dest != OP_NO_DEST) w.y = (w.y & 0xFFFF0000u) | (uint32_t)pe[dest];
    }
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
