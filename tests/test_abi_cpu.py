"""C-ABI library checks that need no GPU: it loads, exports every symbol include/hc.h declares,
and its host-side compiler produces the paper's homogenised term format."""
import os
import re

import numpy as np
import pytest

from hc_inputs import rng, systems
from hc_inputs.poly import const, var_p, var_x

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def hc():
    import __graft_entry__
    __graft_entry__.build_lib()
    from paper_2112_03444_b200 import hc as hcmod
    return hcmod


def declared_symbols():
    txt = open(os.path.join(ROOT, "include", "hc.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol(hc):
    from paper_2112_03444_b200 import _lib
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTED)
    assert "sm_100a" in hc.version()


def test_settings_defaults_match_readings(hc):
    s = hc.hc_tracker_settings_default()
    assert (s.predictor, s.dt_init, s.dt_min, s.dt_max, s.grow_after, s.grow, s.shrink) == (0, 0.01, 1e-14, 0.1, 4, 2.0, 0.5)
    assert (s.max_newton, s.newton_tol, s.max_steps, s.inf_norm, s.end_newton) == (3, 1e-8, 10000, 1e14, 3)


def _decode(ops, nfac, N):
    """Interpret the op table: list of (lane, dest, coef, scale, rhs, last, factors)."""
    out = []
    Q, Lanes, _ = ops.shape
    for q in range(Q):
        for ln in range(Lanes):
            x, y, z, w = (int(v) for v in ops[q, ln])
            facs = [(z >> (8 * m)) & 0xFF for m in range(4)] + [(w >> (8 * m)) & 0xFF for m in range(4)]
            out.append(dict(q=q, lane=ln, coef=x & 0xFFFF, dest=x >> 16, last=bool(y & 1), rhs=bool(y & 2),
                            scale=(y >> 8) & 0xFF, fac=facs[: int(nfac[q])], allfac=facs))
    return out


def eval_ops(ops, nfac, N, cvals, cdvals, x, rhs_dt=False):
    """Direct interpretation of the compiled table (independent of the CUDA kernel):
    returns [A | b] with b = H (rhs_dt False) or dH/dt (True)."""
    xs = np.concatenate([x, [1.0]])
    M = np.zeros((N, N + 1), complex)
    Q, Lanes, _ = ops.shape
    for ln in range(Lanes):
        acc = 0j
        for q in range(Q):
            x_, y_, z_, w_ = (int(v) for v in ops[q, ln])
            rhs = bool(y_ & 2)
            c = (cdvals if (rhs and rhs_dt) else cvals)[x_ & 0xFFFF]
            v = c * ((y_ >> 8) & 0xFF)
            facs = [(z_ >> (8 * m)) & 0xFF for m in range(4)] + [(w_ >> (8 * m)) & 0xFF for m in range(4)]
            for m in range(int(nfac[q])):
                v *= xs[facs[m]]
            acc += v
            if y_ & 1:
                d = x_ >> 16
                M[d // (N + 1), d % (N + 1)] = acc
                acc = 0j
    return M


def test_paper_index_format_example(hc):
    """P:429-434 worked example.  F_1 = a1 x1^2 + 2 a2 x1^2 x2 + 8 a3 x1 x2^2 has dF_1/dx1 = A =
    2a1x1 + 4a2x1x2 + 8a3x2^2; F_2 = 5/2 a4 x1^2 x2 + 7 a5 x1 x2^2 has dF_2/dx1 = B = 5a4x1x2 + 7a5x2^2.
    A must compile to the paper's terms ((2,a1,x1,x3), (4,a2,x1,x2), (8,a3,x2,x2)) (reading R14: the third
    term's factors are (x2, x2); padding uses the constant-one slot x3 = 1) and B to
    ((5,a4,x1,x2), (7,a5,x2,x2)), up to the split of s_k between scale and coefficient weight."""
    n, P = 2, 5
    x1, x2 = var_x(n, P, 0), var_x(n, P, 1)
    a = [var_p(n, P, q) for q in range(P)]
    F1 = a[0] * x1 * x1 + 2 * a[1] * x1 * x1 * x2 + 8 * a[2] * x1 * x2 * x2
    F2 = 2.5 * a[3] * x1 * x1 * x2 + 7 * a[4] * x1 * x2 * x2
    d = systems.from_polys([F1, F2], "paper-example")
    ops, nfac, info = hc.hc_system_compile_ops(d)
    assert info["lanes_per_track"] == 2 and info["max_factors"] == 3
    recs = _decode(ops, nfac, n)
    # coefficient expression j -> (weight, parameter index)
    cw = {j: (complex(d.coef_w[d.coef_ptr[j]]), int(np.argmax(d.coef_pexp[d.coef_ptr[j]]))) for j in range(d.n_coefs)}

    def entry_terms(row, col):
        """(s_k, a index (1-based), sorted 1-based factor indices padded to 2 with the constant slot)."""
        terms, lanes = [], {}
        for r in recs:
            lanes.setdefault(r["lane"], []).append(r)
        for ln, rs in lanes.items():
            cur = []
            for r in rs:
                if r["scale"] == 0:
                    continue
                cur.append(r)
                if r["last"]:
                    if r["dest"] == row * (n + 1) + col:
                        for t in cur:
                            w, q = cw[t["coef"]]
                            f = sorted(i + 1 for i in t["fac"] if i != n)
                            f = f + [n + 1] * (2 - len(f))
                            terms.append((round((t["scale"] * w).real, 12), q + 1, tuple(f)))
                    cur = []
        return sorted(terms)

    assert entry_terms(0, 0) == sorted([(2.0, 1, (1, 3)), (4.0, 2, (1, 2)), (8.0, 3, (2, 2))])
    assert entry_terms(1, 0) == sorted([(5.0, 4, (1, 2)), (7.0, 5, (2, 2))])
    # every factor slot is a variable or the constant-one slot index N; padding ops have scale 0
    for r in recs:
        assert all(0 <= f <= n for f in r["allfac"])
        if r["dest"] == 0xFFFF and not r["last"] and r["scale"] == 0:
            assert all(f == n for f in r["allfac"])


@pytest.mark.parametrize("name", ["katsura-6", "cyclic-7", "4-view", "trifocal"])
def test_compiled_table_matches_oracle_evaluation(hc, orc, name):
    """The compiled op table, interpreted directly in Python, reproduces the oracle's J_F and F
    (PH: coefficients at p) -- pins the host compiler (differentiation, folding, lane packing)."""
    d = {"katsura-6": lambda: systems.katsura(6), "cyclic-7": lambda: systems.cyclic(7),
         "4-view": lambda: systems.nview_triangulation(4), "trifocal": systems.trifocal_unknown_f}[name]()
    ops, nfac, info = hc.hc_system_compile_ops(d)
    N = d.n_vars
    assert info["n_ops_rhs"] == d.n_terms
    g = rng.gen(3)
    for _ in range(3):
        p = (g.standard_normal(d.n_params) + 1j * g.standard_normal(d.n_params))
        x = g.standard_normal(N) + 1j * g.standard_normal(N)
        c = orc.eval_coefs(d, p)
        M = eval_ops(ops, nfac, N, c, np.zeros_like(c), x)
        J = orc.eval_JF(d, p, x)
        F = orc.eval_F(d, p, x)
        assert np.max(np.abs(M[:, :N] - J)) <= 1e-12 * (1 + np.max(np.abs(J)))
        assert np.max(np.abs(M[:, N] - F)) <= 1e-12 * (1 + np.max(np.abs(F)))
    # lane balance: no lane carries more than the ideal share + the largest entry
    assert info["op_steps"] * info["lanes_per_track"] >= info["n_ops_J"] + info["n_ops_rhs"]


def test_flop_model(hc):
    """SURVEY.md §8(d) LU rule: N=7 -> 1232, N=14 -> 8638, N=18 -> 17754, N=32 -> 94432 flops."""
    for N, want in ((7, 1232), (14, 8638), (18, 17754), (32, 94432)):
        X = [var_x(N, 0, i) for i in range(N)]
        d = systems.from_polys([X[i] * X[i] - 1 for i in range(N)])
        assert hc.hc_system_compile_info(d)["flops_lu"] == want


def test_invalid_descriptors_rejected(hc):
    from paper_2112_03444_b200._lib import HC_E_INVALID_ARG, HC_E_TOO_LARGE
    X = [var_x(33, 0, i) for i in range(33)]
    big = systems.from_polys([X[i] - 1 for i in range(33)])
    with pytest.raises(hc.HCError) as e:
        hc.hc_system_compile_info(big)
    assert e.value.code == HC_E_TOO_LARGE
    d = systems.katsura(3)
    bad = systems.katsura(3)
    bad.coef_w = bad.coef_w.copy()
    bad.coef_w[0] = np.nan
    with pytest.raises(hc.HCError) as e:
        hc.hc_system_compile_info(bad)
    assert e.value.code == HC_E_INVALID_ARG
    bad2 = systems.katsura(3)
    bad2.term_eq = np.zeros_like(bad2.term_eq)   # equations 1..3 have no terms
    with pytest.raises(hc.HCError) as e:
        hc.hc_system_compile_info(bad2)
    assert e.value.code == HC_E_INVALID_ARG
    x = var_x(1, 0, 0)
    deg9 = systems.from_polys([x ** 9 - 1])
    with pytest.raises(hc.HCError) as e:
        hc.hc_system_compile_info(deg9)
    assert e.value.code == HC_E_TOO_LARGE
    assert hc.hc_system_compile_info(d)["n_vars"] == 4


def test_product_never_imports_oracle():
    """The product path must not route through the oracle (prompt rule ③)."""
    pkg = os.path.join(ROOT, "paper_2112_03444_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "hc_oracle" not in txt, f
