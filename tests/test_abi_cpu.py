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
    assert s.lane_layout == hc.HC_LAYOUT_AUTO


def test_sharded_settings_pin_the_lane_layout(hc):
    """A sharded job pins the lane layout (the auto choice depends on the batch size for N <= 16,
    include/hc.h Determinism); an out-of-range layout is rejected by the C ABI."""
    from paper_2112_03444_b200.distributed import sharded_settings
    assert sharded_settings(hc.hc_tracker_settings_default()).lane_layout == hc.HC_LAYOUT_THROUGHPUT
    assert sharded_settings(hc.settings(lane_layout=hc.HC_LAYOUT_WIDE)).lane_layout == hc.HC_LAYOUT_WIDE


def mono_factors(prog, N):
    """Variable multiset of every monomial-table entry: k < N -> [k], k == N -> [] (constant one),
    k > N -> factors(a) + factors(b) for the entry's two factor indices (program order is by
    level, factors first)."""
    f = [[k] for k in range(N)] + [[]]
    for e in prog:
        a, b = int(e) & 0xFFFF, int(e) >> 16
        assert a < len(f) and b < len(f)   # factors come from earlier entries
        f.append(f[a] + f[b])
    return f


def decode_ops(ops, N):
    """Per lane, the op records as dicts (slot, mono, dest, last, rhs)."""
    Q, Lanes, _ = ops.shape
    lanes = []
    for ln in range(Lanes):
        rs = []
        for q in range(Q):
            x, y = int(ops[q, ln, 0]), int(ops[q, ln, 1])
            fl = y >> 16
            rs.append(dict(slot=x & 0xFFFF, mono=x >> 16, dest=y & 0xFFFF, last=bool(fl & 1), rhs=bool(fl & 2)))
        lanes.append(rs)
    return lanes


def eval_tables(ops, prog, smap, emap, N, cvals, x):
    """Direct interpretation of the compiled tables (independent of the CUDA kernel):
    returns [A | b] with b = H, coefficient slot value = scale * c_j."""
    mono = list(x) + [1.0 + 0j]
    for e in prog:
        mono.append(mono[int(e) & 0xFFFF] * mono[int(e) >> 16])
    slotv = [smap[s, 1] * cvals[smap[s, 0]] for s in range(smap.shape[0])]
    compact = {}
    for rs in decode_ops(ops, N):
        acc = 0j
        for r in rs:
            acc += slotv[r["slot"]] * mono[r["mono"]]
            if r["last"]:
                compact[r["dest"]] = acc
                acc = 0j
    M = np.zeros((N, N + 1), complex)
    for i in range(N):
        for j in range(N + 1):
            if emap[i, j] >= 0:
                M[i, j] = compact[int(emap[i, j])]
    assert sorted(compact) == list(range(len(compact)))   # every compact entry written exactly once
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
    ops, prog, smap, emap, info = hc.hc_system_compile_tables(d)
    dense = {int(emap[i, j]): i * (n + 1) + j for i in range(n) for j in range(n + 1) if emap[i, j] >= 0}
    assert info["lanes_per_track"] == 2 and info["max_factors"] == 3
    facs = mono_factors(prog, n)
    # coefficient expression j -> (weight, parameter index)
    cw = {j: (complex(d.coef_w[d.coef_ptr[j]]), int(np.argmax(d.coef_pexp[d.coef_ptr[j]]))) for j in range(d.n_coefs)}

    def entry_terms(row, col):
        """(s_k * weight, a index (1-based), sorted 1-based factors padded to 2 with the constant slot N+1)."""
        terms = []
        for rs in decode_ops(ops, n):
            cur = []
            for r in rs:
                cur.append(r)
                if r["last"]:
                    if dense[r["dest"]] == row * (n + 1) + col:
                        for t in cur:
                            j, sc = int(smap[t["slot"], 0]), int(smap[t["slot"], 1])
                            w, q = cw[j]
                            f = sorted(i + 1 for i in facs[t["mono"]])
                            f = f + [n + 1] * (2 - len(f))
                            terms.append((round((sc * w).real, 12), q + 1, tuple(f)))
                    cur = []
        return sorted(terms)

    assert entry_terms(0, 0) == sorted([(2.0, 1, (1, 3)), (4.0, 2, (1, 2)), (8.0, 3, (2, 2))])
    assert entry_terms(1, 0) == sorted([(5.0, 4, (1, 2)), (7.0, 5, (2, 2))])
    # the constant-one slot is monomial index N: a degree-1 term's partner is x3 = 1
    assert facs[n] == []


@pytest.mark.parametrize("name", ["katsura-6", "cyclic-7", "4-view", "trifocal", "5-point", "P3P", "eco-8",
                                  "cyclic-7 family"])
def test_compiled_table_matches_oracle_evaluation(hc, orc, name):
    """The compiled op table, interpreted directly in Python, reproduces the oracle's J_F and F
    (PH: coefficients at p) -- pins the host compiler (differentiation, folding, lane packing, the
    classic and the log-depth monomial programs: cyclic-7 uses the latter)."""
    d = {"katsura-6": lambda: systems.katsura(6), "cyclic-7": lambda: systems.cyclic(7),
         "4-view": lambda: systems.nview_triangulation(4), "trifocal": systems.trifocal_unknown_f,
         "5-point": systems.fivepoint_relpose_depth, "P3P": systems.p3p_depth, "eco-8": lambda: systems.eco(8),
         "cyclic-7 family": lambda: systems.cyclic_family(7)}[name]()
    ops, prog, smap, emap, info = hc.hc_system_compile_tables(d)
    N = d.n_vars
    assert info["n_ops_rhs"] == d.n_terms
    g = rng.gen(3)
    for _ in range(3):
        p = (g.standard_normal(d.n_params) + 1j * g.standard_normal(d.n_params))
        x = g.standard_normal(N) + 1j * g.standard_normal(N)
        c = orc.eval_coefs(d, p)
        M = eval_tables(ops, prog, smap, emap, N, c, x)
        J = orc.eval_JF(d, p, x)
        F = orc.eval_F(d, p, x)
        assert np.max(np.abs(M[:, :N] - J)) <= 1e-12 * (1 + np.max(np.abs(J)))
        assert np.max(np.abs(M[:, N] - F)) <= 1e-12 * (1 + np.max(np.abs(F)))
    # lane balance: every op placed; at most one entry's worth above the ideal share per lane
    nops = info["n_ops_J"] + info["n_ops_rhs"]
    assert info["op_steps"] * info["lanes_per_track"] >= nops
    assert info["op_steps"] <= nops / info["lanes_per_track"] + N + 2
    # monomial sharing: each table entry is one complex product
    assert info["n_monos"] - N - 1 == len(prog)


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


def test_solutions_post_processing_matches_oracle(hc, orc):
    """hc_solutions (a11, readings R11/R12) against the oracle's dedup / is_real on synthetic
    endpoints: planted near-duplicates (inside and well outside the 1e-6 tolerance), real and
    complex points, large coordinates, non-converged tracks."""
    g = rng.gen(5)
    S, N = 400, 6
    base = (g.standard_normal((60, N)) + 1j * g.standard_normal((60, N))) * 10.0 ** g.integers(-2, 5, (60, 1))
    base[::3] = base[::3].real   # some real points
    X = base[g.integers(0, 60, S)].copy()
    X *= 1 + np.where(g.random((S, 1)) < 0.5, 1e-9, 1e-4) * (g.standard_normal((S, N)) + 1j * g.standard_normal((S, N)))
    status = np.where(g.random(S) < 0.85, 0, 2).astype(np.int32)
    U, mult, real, rep = hc.solutions(X, status)
    A, mA = orc.dedup(X[status == 0])
    assert U.shape == A.shape and np.array_equal(U, A) and np.array_equal(mult, mA)
    assert np.array_equal(real, orc.is_real(A))
    assert np.all(rep[status != 0] == -1) and np.all(rep[status == 0] >= 0)
    assert hc.solutions(X[:0])[0].shape == (0, N)   # empty instance


def test_monodromy_matching_goes_through_hc_solutions(hc):
    """monodromy._new_points (R11 matching of loop endpoints against the known set) is the library's
    hc_solutions: points within the tolerance of a known point or of an earlier new point are not new."""
    from paper_2112_03444_b200.monodromy import _new_points
    g = rng.gen(9)
    known = g.standard_normal((20, 4)) + 1j * g.standard_normal((20, 4))
    fresh = g.standard_normal((3, 4)) + 1j * g.standard_normal((3, 4))
    X = np.concatenate([known[[4, 7]] * (1 + 1e-9), fresh[[0]], fresh[[0]] * (1 + 1e-10), fresh[[1]],
                        known[[2]] * (1 + 1e-3)])
    assert _new_points(known, X, 1e-6) == [2, 4, 5]
    assert _new_points(known[:0], X[:2], 1e-6) == [0, 1]
    assert _new_points(known, X[:0], 1e-6) == []


@pytest.mark.parametrize("n", [3, 7, 14, 16, 18])
def test_tracker_sass_one_loop_copy_and_bulk_staging(n):
    """The built tracker kernels (sm_100a SASS, cuobjdump): one copy of the tracking loop per kernel
    (one work-queue atomic + one endgame-list atomic: a loop-invariant branch in the loop once made
    the compiler unswitch it and compile the evaluation + elimination twice), the
    tables staged by bulk async copies (UBLKCP, north_star), at most a couple of local-memory
    instructions for N = 18 (no spilled rows)."""
    import glob
    import subprocess
    objs = glob.glob(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2112_03444_b200",
                                  "build", "*", f"kernels_tracker_n{n}.cu.o"))
    if not objs:
        pytest.skip("library not built")
    sass = subprocess.run(["cuobjdump", "-sass", max(objs, key=os.path.getmtime)], capture_output=True, text=True).stdout
    funcs = re.split(r"\n\s*Function : ", sass)
    tracks = [f for f in funcs if f.startswith(f"_ZN3hcb15hc_track_kernelILi{n}E")]
    assert tracks, "no tracker kernel in the object"
    for f in tracks:
        assert len(re.findall(r"ATOMG\.E\.ADD\.64", f)) == 2, f.split("\n")[0]
        assert len(re.findall(r"UBLKCP", f)) >= 2, f.split("\n")[0]
        if n == 18:
            assert len(re.findall(r"\b(?:LDL|STL)\b", f)) <= 4
