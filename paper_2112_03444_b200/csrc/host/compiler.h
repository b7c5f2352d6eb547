// compiler.h -- host-side system compiler: descriptor -> homogenised, lane-balanced evaluation
// tables (the paper's "indexing system") + coefficient-polynomial monomials.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../hc_internal.h"

namespace hcb {

struct CompiledSystem {
  int N = 0, P = 0, D = 0;
  int ncoef_src = 0;               // coefficient expressions of the descriptor
  int ncoef = 0;                   // coefficient slots (descriptor's + scaled copies s_k * c_j)
  int L = 1, Q = 0, M = 0;         // lanes, op steps, max monomial degree
  int n_ops_J = 0, n_ops_rhs = 0, n_terms = 0;
  int n_mono = 0, n_levels = 0;    // monomial table size (incl. N unknowns + constant), levels
  int level_end[MAX_LEVELS] = {0};
  std::vector<uint2> ops;          // [Q * L]
  std::vector<int16_t> mpos;       // [N * (N + 1)] dense -> compact entry, -1 = structural zero
  int n_entries = 0;
  std::vector<uint32_t> mono_prog; // [n_mono - N - 1]: parent | var << 16
  std::vector<int32_t> slot_map;   // [ncoef * 2]: (descriptor coefficient id, scale)
  std::vector<CoefMono> mono;      // prologue monomials, sorted by slot
  std::vector<int32_t> mono_ptr;   // [ncoef + 1]
  std::vector<int32_t> degrees;    // total degree of each equation
  int64_t flops_coef = 0, flops_eval = 0, flops_lu = 0, flops_solve = 0;   // SURVEY §8(d) rule
  int64_t flops_eval_kernel = 0, flops_solve_kernel = 0;                   // as the kernel computes
};

// Returns HC_OK or an error code with a message in `err`.
// lanes: lanes per track (0 = lanes_for(N); 32 = the wide latency layout for N <= 16)
hc_status compile_system(const hc_system_desc &d, CompiledSystem &out, std::string &err, int lanes = 0);

// Descriptor of the total-degree homotopy system built from a constant-coefficient target
// (SURVEY.md §8(b) "Total degree is a PH"): params = (G x^d coefficients [N], G constants [N],
// target coefficient values [ncoef]).  `fvals` receives the target's coefficient values.
struct OwnedDesc {
  int32_t n_vars = 0, n_params = 0, n_terms = 0, n_coefs = 0;
  std::vector<int32_t> term_eq, term_xexp, term_coef, coef_ptr, coef_pexp;
  std::vector<hc_complex> coef_w;
  hc_system_desc view() const;
};
hc_status total_degree_desc(const hc_system_desc &target, OwnedDesc &out, std::vector<hc_complex> &fvals,
                            std::vector<int32_t> &degrees, std::string &err);

int64_t lu_flops(int N);

}  // namespace hcb
