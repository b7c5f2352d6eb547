"""System descriptor: F(x; p) = 0 as a flat term list (the `hc_system_desc` of
include/hc.h and of oracle/hc_oracle.h).

F_i(x; p) = sum over terms k with term_eq[k] == i of  c_{term_coef[k]}(p) * prod_v x_v^{term_xexp[k, v]}
c_j(p)    = sum over m in [coef_ptr[j], coef_ptr[j+1]) of coef_w[m] * prod_q p_q^{coef_pexp[m, q]}

This is the paper's "coefficients a_{k,j}" written before
any homogenisation: the index tables of P:434 are built from it by the CUDA
path's own compiler, and the oracle evaluates it directly.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .poly import Poly


@dataclass
class SystemDesc:
    n_vars: int
    n_params: int
    term_eq: np.ndarray      # int32 [T]
    term_xexp: np.ndarray    # int32 [T, n]
    term_coef: np.ndarray    # int32 [T]
    coef_ptr: np.ndarray     # int32 [C+1]
    coef_w: np.ndarray       # complex128 [nnz]
    coef_pexp: np.ndarray    # int32 [nnz, P]  (shape [nnz, 0] when P == 0)
    name: str = ""
    var_names: list = field(default_factory=list)
    polys: list = field(default_factory=list, repr=False, compare=False)  # source equations (tests)

    @property
    def n_terms(self) -> int:
        return int(self.term_eq.shape[0])

    @property
    def n_coefs(self) -> int:
        return int(self.coef_ptr.shape[0] - 1)

    def degrees(self) -> list[int]:
        """Total degree d_i of each equation (for the total-degree start, Bezout count)."""
        d = [0] * self.n_vars
        tot = self.term_xexp.sum(axis=1)
        for k in range(self.n_terms):
            i = int(self.term_eq[k])
            d[i] = max(d[i], int(tot[k]))
        return d

    def coef_degree_p(self) -> int:
        """Max total degree in p over all coefficient expressions."""
        if self.coef_pexp.size == 0:
            return 0
        return int(self.coef_pexp.sum(axis=1).max())

    def is_constant(self) -> bool:
        return self.coef_pexp.size == 0 or not self.coef_pexp.any()

    def contiguous(self) -> "SystemDesc":
        for a in ("term_eq", "term_xexp", "term_coef", "coef_ptr", "coef_pexp"):
            setattr(self, a, np.ascontiguousarray(getattr(self, a), dtype=np.int32))
        self.coef_w = np.ascontiguousarray(self.coef_w, dtype=np.complex128)
        return self


def desc_from_equations(eqs: list[Poly], name: str = "", var_names=None) -> SystemDesc:
    """Expand polynomials F_i(x; p) into the flat descriptor.

    Monomials in x are grouped per equation; each group's coefficient is a
    polynomial in p.  Identical coefficient polynomials are shared (one
    coefficient expression id), which is what makes the paper's "a_{k,j}
    identifies a coefficient" indexing compact.
    """
    assert eqs, "empty system"
    n, P = eqs[0].n, eqs[0].P
    term_eq, term_xexp, term_coef = [], [], []
    coef_ids: dict = {}
    coef_list: list = []
    for i, f in enumerate(eqs):
        assert (f.n, f.P) == (n, P)
        groups: dict = {}
        for k, v in f.t.items():
            xe, pe = k[:n], k[n:]
            groups.setdefault(xe, {})
            groups[xe][pe] = groups[xe].get(pe, 0) + v
        for xe in sorted(groups, key=lambda e: (-sum(e), tuple(-a for a in e))):
            cp = {pe: w for pe, w in groups[xe].items() if w != 0}
            if not cp:
                continue
            key = tuple(sorted((pe, complex(w).real, complex(w).imag) for pe, w in cp.items()))
            j = coef_ids.get(key)
            if j is None:
                j = len(coef_list)
                coef_ids[key] = j
                coef_list.append(sorted(cp.items()))
            term_eq.append(i)
            term_xexp.append(list(xe))
            term_coef.append(j)
    coef_ptr = [0]
    coef_w, coef_pexp = [], []
    for cp in coef_list:
        for pe, w in cp:
            coef_w.append(complex(w))
            coef_pexp.append(list(pe))
        coef_ptr.append(len(coef_w))
    return SystemDesc(
        n_vars=n, n_params=P,
        term_eq=np.array(term_eq, dtype=np.int32),
        term_xexp=np.array(term_xexp, dtype=np.int32).reshape(len(term_eq), n),
        term_coef=np.array(term_coef, dtype=np.int32),
        coef_ptr=np.array(coef_ptr, dtype=np.int32),
        coef_w=np.array(coef_w, dtype=np.complex128),
        coef_pexp=np.array(coef_pexp, dtype=np.int32).reshape(len(coef_w), P),
        name=name, var_names=list(var_names or []), polys=list(eqs),
    ).contiguous()
