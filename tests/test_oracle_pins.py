"""Pins of the CPU oracle (oracle/) against things other than itself (CPU-only, `-m "not gpu"`).

Each test names what pins it: a library routine (numpy), a closed form, finite
differences, a textbook or paper root count, or planted ground truth.
"""
import numpy as np
import pytest

from hc_inputs import rng, systems
from hc_inputs.evalpoly import eval_poly


def crandn(g, *shape):
    return (g.standard_normal(shape) + 1j * g.standard_normal(shape)) / np.sqrt(2)


SYSTEMS = {
    "katsura-6": lambda: systems.katsura(6),
    "cyclic-5": lambda: systems.cyclic(5),
    "4-view": lambda: systems.nview_triangulation(4),
    "trifocal": lambda: systems.trifocal_unknown_f(),
    "5pt-relpose": lambda: systems.fivepoint_relpose_depth(),
    "univ-param": lambda: systems.univariate_param(5),
}


# ---------------------------------------------------------------- linear solve

def test_lu_matches_numpy_solve(orc):
    """Library pin: textbook LU+2 triangular solves vs numpy.linalg.solve (LAPACK zgesv), N=1..32."""
    g = rng.gen(123)
    for trial in range(300):
        n = 1 + trial % 32
        A = crandn(g, n, n) + np.eye(n) * (1.0 + g.random())
        b = crandn(g, n)
        x, sing = orc.lu_solve(A, b)
        assert not sing
        xr = np.linalg.solve(A, b)
        assert np.max(np.abs(x - xr)) <= 1e-12 * max(1.0, np.max(np.abs(xr))) * np.linalg.cond(A)
        # backward-error bound
        r = np.max(np.abs(A @ x - b))
        assert r <= 1e-10 * (np.max(np.abs(A).sum(1)) * np.max(np.abs(x)) + np.max(np.abs(b)))


def test_lu_needs_pivoting(orc):
    """Closed form: zero leading pivot forces a row swap; A = [[0,1],[2,0]], b = [3,4] -> x = [2,3]."""
    x, sing = orc.lu_solve(np.array([[0, 1], [2, 0]], complex), np.array([3, 4], complex))
    assert not sing and np.allclose(x, [2, 3], atol=0, rtol=1e-15)


def test_lu_singular_flagged(orc):
    """Rank-deficient matrices are flagged, never solved silently (R9)."""
    g = rng.gen(5)
    for n in (2, 7, 18, 32):
        A = crandn(g, n, n)
        A[-1] = A[0] * (0.3 - 0.2j)  # dependent row
        _, sing = orc.lu_solve(A, crandn(g, n))
        assert sing
    _, sing = orc.lu_solve(np.zeros((3, 3), complex), np.ones(3, complex))
    assert sing
    A = np.eye(3, dtype=complex)
    A[1, 1] = np.nan
    _, sing = orc.lu_solve(A, np.ones(3, complex))
    assert sing


# ---------------------------------------------------------------- evaluation

@pytest.mark.parametrize("name", list(SYSTEMS))
def test_F_matches_defining_sum(orc, name):
    """F(x; p) from the descriptor == direct sum over the source polynomial's terms."""
    d = SYSTEMS[name]()
    g = rng.gen(7)
    for _ in range(5):
        x = crandn(g, d.n_vars)
        p = crandn(g, d.n_params)
        F = orc.eval_F(d, p, x)
        ref = np.array([eval_poly(f, x, p) for f in d.polys])
        assert np.max(np.abs(F - ref)) <= 1e-12 * (1 + np.max(np.abs(ref)))


@pytest.mark.parametrize("name", list(SYSTEMS))
def test_JF_matches_central_differences(orc, name):
    """J_F vs central finite differences of F: relative error < 1e-6 with h = 1e-6."""
    d = SYSTEMS[name]()
    g = rng.gen(11)
    h = 1e-6
    for _ in range(3):
        x = crandn(g, d.n_vars)
        p = crandn(g, d.n_params)
        J = orc.eval_JF(d, p, x)
        for v in range(d.n_vars):
            e = np.zeros(d.n_vars, complex)
            e[v] = h
            fd = (orc.eval_F(d, p, x + e) - orc.eval_F(d, p, x - e)) / (2 * h)
            assert np.max(np.abs(J[:, v] - fd)) <= 1e-6 * (1 + np.max(np.abs(fd)))


def test_td_homotopy_endpoints_and_Ht(orc):
    """Eq. 1 endpoints: H(x,0) = gamma G(x) with G_i = x_i^d_i - 1, H(x,1) = F(x); H_t vs central FD in t
    (S:176-198).  G is checked against numpy's power, F against the defining sum."""
    d = systems.katsura(4)
    gam = rng.gamma(3)
    hom = orc.td_homotopy(d, gam)
    g = rng.gen(2)
    deg = np.array(d.degrees())
    for _ in range(4):
        x = crandn(g, d.n_vars)
        H0, _, _ = hom.eval(x, 0.0)
        assert np.allclose(H0, gam * (np.power(x, deg) - 1), rtol=1e-14, atol=1e-14)
        H1, Hx1, _ = hom.eval(x, 1.0)
        F = np.array([eval_poly(f, x) for f in d.polys])
        assert np.allclose(H1, F, rtol=1e-13, atol=1e-13)
        assert np.allclose(Hx1, orc.eval_JF(d, np.zeros(0), x), rtol=1e-13, atol=1e-13)
        t = g.random()
        _, _, Ht = hom.eval(x, t)
        hh = 1e-6
        fd = (hom.eval(x, t + hh)[0] - hom.eval(x, t - hh)[0]) / (2 * hh)
        assert np.max(np.abs(Ht - fd)) <= 1e-6 * (1 + np.max(np.abs(fd)))
        _, _, Ht2 = hom.eval(x, 1 - t)
        assert np.allclose(Ht, Ht2, rtol=1e-13, atol=1e-13)  # straight-line TD: H_t independent of t


@pytest.mark.parametrize("name", ["4-view", "trifocal", "univ-param"])
def test_ph_homotopy_endpoints_and_Ht(orc, name):
    """PH (R3): H(x,0) = F(x;p0), H(x,1) = F(x;p1); H_t vs central FD in t (exactness not assumed)."""
    d = SYSTEMS[name]()
    g = rng.gen(13)
    p0, p1 = crandn(g, d.n_params), crandn(g, d.n_params)
    hom = orc.ph_homotopy(d, p0, p1)
    x = crandn(g, d.n_vars)
    F0 = np.array([eval_poly(f, x, p0) for f in d.polys])
    F1 = np.array([eval_poly(f, x, p1) for f in d.polys])
    assert np.allclose(hom.eval(x, 0.0)[0], F0, rtol=1e-12, atol=1e-12)
    assert np.allclose(hom.eval(x, 1.0)[0], F1, rtol=1e-12, atol=1e-12)
    for t in (0.1, 0.5, 0.93):
        hh = 1e-5
        fd = (hom.eval(x, t + hh)[0] - hom.eval(x, t - hh)[0]) / (2 * hh)
        Ht = hom.eval(x, t)[2]
        assert np.max(np.abs(Ht - fd)) <= 1e-7 * (1 + np.max(np.abs(fd)))


# ---------------------------------------------------------------- predictor / corrector

def _line_homotopy(orc):
    """F(x; p) = x - p with p0 = 1, p1 = 2: H = x - (1 + t), exact path x(t) = 1 + t."""
    from hc_inputs.poly import var_p, var_x
    f = var_x(1, 1, 0) - var_p(1, 1, 0)
    d = systems.from_polys([f], "line")
    return orc.ph_homotopy(d, np.array([1.0]), np.array([2.0]))


def test_predictor_exact_on_linear_path(orc):
    """Closed form: Euler from (x=1, t=0, dt=0.5) gives 1.5 exactly; RK4 equals Euler."""
    hom = _line_homotopy(orc)
    for pred in (0, 1):
        st = orc.default_settings()
        st.predictor = pred
        xp, fail = orc.predict(hom, np.array([1.0 + 0j]), 0.0, 0.5, st)
        assert not fail and xp[0] == 1.5


def _quintic_path_homotopy(orc):
    """F(x; p) = x - p^5 with p0 = 1, p1 = 2: p(t) = 1 + t, exact path x(t) = (1 + t)^5, Davidenko
    rhs dx/dt = 5 (1 + t)^4 depends on t only."""
    from hc_inputs.poly import var_p, var_x
    f = var_x(1, 1, 0) - var_p(1, 1, 0) ** 5
    d = systems.from_polys([f], "quintic-path")
    return orc.ph_homotopy(d, np.array([1.0]), np.array([2.0]))


def test_rk4_is_simpson_on_t_only_ode(orc):
    """Closed form pinning RK4's stage times and weights (classical RK4): when dx/dt = f(t),
    one RK4 step is Simpson's rule h/6 (f(t) + 4 f(t + h/2) + f(t + h)), whose error for the quartic
    f = 5 (1+t)^4 is exactly h^5 f''''/2880 = h^5 / 24 (f'''' = 120).  Euler (Eq. 4) gives
    x + 5h, error (1+h)^5 - 1 - 5h = 10h^2 + 10h^3 + 5h^4 + h^5.  A wrong stage time (e.g. k2 at t)
    or weight breaks the h^5/24 identity at the first digit."""
    hom = _quintic_path_homotopy(orc)
    for h in (0.2, 0.1, 0.05):
        st = orc.default_settings()
        xp, fail = orc.predict(hom, np.array([1.0 + 0j]), 0.0, h, st)
        assert not fail
        err = xp[0].real - (1 + h) ** 5
        assert abs(xp[0].imag) == 0.0
        assert abs(err - h ** 5 / 24) <= 1e-6 * h ** 5 / 24 + 1e-14, (h, err, h ** 5 / 24)   # + rounding of (1+h)^5
        st.predictor = 1
        xe, fail = orc.predict(hom, np.array([1.0 + 0j]), 0.0, h, st)
        assert not fail and abs(xe[0].real - (1 + 5 * h)) <= 1e-15
    # from t0 = 0.3 (the stage times are t0 + {0, h/2, h/2, h}): error h^5/24 again
    xp, _ = orc.predict(hom, np.array([1.3 ** 5 + 0j]), 0.3, 0.1)
    assert abs((xp[0].real - 1.4 ** 5) - 1e-5 / 24) <= 1e-6 * 1e-5 / 24 + 1e-14


def test_rk4_fourth_order_on_x_dependent_ode(orc):
    """Order pin for the x-dependent stages: H = x^2 - (1 + t) (univariate_param(2), p0 = (-1, 0, 1),
    p1 = (-2, 0, 1)); the exact path from x(0) = 1 is sqrt(1 + t) and dx/dt = 1/(2x).  A one-step
    method of order q has local error C h^(q+1), so halving h divides the error by ~2^(q+1): RK4
    (q = 4) -> ~32, Euler (q = 1) -> ~4.  Wrong stage points (x + h/2 k1 etc.) or weights drop the
    order and fail the ratio window."""
    d = systems.univariate_param(2)
    hom = orc.ph_homotopy(d, np.array([-1.0, 0, 1]), np.array([-2.0, 0, 1]))

    def err(h, pred):
        st = orc.default_settings()
        st.predictor = pred
        xp, fail = orc.predict(hom, np.array([1.0 + 0j]), 0.0, h, st)
        assert not fail
        return abs(xp[0] - np.sqrt(1 + h))
    for pred, lo, hi in ((0, 25.0, 40.0), (1, 3.5, 4.5)):
        e = [err(h, pred) for h in (0.2, 0.1, 0.05)]
        for a, b in zip(e, e[1:]):
            assert lo <= a / b <= hi, (pred, e)


def test_endpoint_residuals_by_hand(orc):
    """Reading R10 pinned by hand.  F1 = 2x^2 - 3y + 1, F2 = (1+i)xy - 4 at (x, y) = (1+i, 2):
    x^2 = 2i, so F1 = -5 + 4i, |F1| = sqrt(41), sum |c||m| = 2*2 + 3*2 + 1 = 11;
    F2 = (1+i)(1+i)2 - 4 = -4 + 4i, |F2| = 4 sqrt(2), sum |c||m| = sqrt(2)*2sqrt(2) + 4 = 8.
    r = max(sqrt(41), 4 sqrt(2)) = sqrt(41); r_rel = max(sqrt(41)/11, sqrt(2)/2) = sqrt(2)/2.
    Checked for the total-degree target (F alone) and for a parameter homotopy whose t = 1
    coefficients are p1 (p0 random: it must not enter)."""
    from hc_inputs.poly import const, var_p, var_x
    x, y = var_x(2, 0, 0), var_x(2, 0, 1)
    d = systems.from_polys([2 * x * x - 3 * y + 1, (1 + 1j) * x * y - 4], "resid-2x2")
    pt = np.array([1 + 1j, 2])
    for hom in (orc.td_homotopy(d, rng.gamma(0)),):
        r, rr = orc.endpoint_residual(hom, pt)
        assert abs(r - np.sqrt(41)) <= 1e-14 and abs(rr - np.sqrt(2) / 2) <= 1e-15
    P = 5
    xp, yp = var_x(2, P, 0), var_x(2, P, 1)
    pp = [var_p(2, P, q) for q in range(P)]
    dp = systems.from_polys([pp[0] * xp * xp + pp[1] * yp + pp[2], pp[3] * xp * yp + pp[4]], "resid-2x2-p")
    p1 = np.array([2, -3, 1, 1 + 1j, -4], complex)
    p0 = crandn(rng.gen(3), P)
    r, rr = orc.endpoint_residual(orc.ph_homotopy(dp, p0, p1), pt)
    assert abs(r - np.sqrt(41)) <= 1e-14 and abs(rr - np.sqrt(2) / 2) <= 1e-15
    # a row whose terms all vanish: r_rel = 0 when F_i = 0, and the zero-denominator rule
    r, rr = orc.endpoint_residual(orc.td_homotopy(d, rng.gamma(0)), np.array([0.5 + 0.5j, 0]))
    # F2 = -4 (its monomial vanishes): |F2| / |−4| = 1
    assert abs(rr - 1.0) <= 1e-15
    del const


def test_newton_quadratic_contraction(orc):
    """Closed form: Newton on x^2 - 4 from 2 + 1e-3: one step error ~ e^2/(2*2) = 2.5e-7 < 1e-5."""
    d = systems.univariate([-4, 0, 1])
    hom = orc.td_homotopy(d, 1.0)
    x, code = orc.newton(hom, np.array([2.001 + 0j]), 1.0, 1, 1e-300)
    assert abs(x[0] - 2) < 1e-5
    assert abs(abs(x[0] - 2) - 1e-6 / 4.002) < 1e-12   # exact one-step error e^2 / (2 x0)
    x2, code = orc.newton(hom, np.array([2.001 + 0j]), 1.0, 3, 1e-12)
    assert code == 1 and abs(x2[0] - 2) < 1e-15


def test_track_linear_path(orc):
    """Whole tracker on the exact path x(t) = 1 + t: converges to 2."""
    hom = _line_homotopy(orc)
    res = orc.track(hom, np.array([[1.0 + 0j]]), p1s=np.array([[2.0 + 0j]]))
    assert res.status[0, 0] == orc.CONVERGED
    assert abs(res.x[0, 0, 0] - 2) < 1e-14


# ---------------------------------------------------------------- start system (R2)

def test_td_start_roots_of_unity(orc):
    """Closed form: prod(d) distinct points with x_i^{d_i} = 1 (north_star), exact quarter turns."""
    deg = [1, 2, 3, 4, 5]
    X = orc.td_start(deg)
    assert X.shape == (120, 5)
    assert np.max(np.abs(np.power(X, deg) - 1)) <= 1e-14
    keys = {tuple(np.round(r, 9)) for r in X}
    assert len(keys) == 120
    X4 = orc.td_start([4])
    assert X4[1, 0] == 1j and X4[2, 0] == -1 and X4[3, 0] == -1j


# ---------------------------------------------------------------- whole tracker

def test_univariate_matches_companion_eigenvalues(orc):
    """Library pin: TD endpoints of a random degree-d polynomial = numpy.roots within 1e-8."""
    g = rng.gen(21)
    for d in (2, 3, 5, 8):
        c = crandn(g, d + 1)
        desc = systems.univariate(c)
        hom = orc.td_homotopy(desc, rng.gamma(d))
        res = orc.track(hom, orc.td_start([d]))
        assert np.all(res.status == orc.CONVERGED)
        got = res.x[0, :, 0]
        ref = np.roots(c[::-1])
        ok, ua, ub = orc.match_sets(got[:, None], ref[:, None], tol=1e-8)
        assert ok, (d, ua, ub)


def test_td_x2_plus_1(orc):
    """Closed form: F = x^2 + 1 -> both tracks reach +-i."""
    hom = orc.td_homotopy(systems.univariate([1, 0, 1]), rng.gamma(0))
    res = orc.track(hom, orc.td_start([2]))
    got = np.sort_complex(res.x[0, :, 0])
    assert np.all(res.status == orc.CONVERGED)
    assert np.allclose(got, [-1j, 1j], atol=1e-12)


def test_katsura6_all_64(orc):
    """Textbook count: katsura-6 has 2^6 = 64 finite roots = Bezout number: all 64 tracks converge,
    distinct, residual < 1e-10, and (1,0,...,0) is among them (SURVEY.md §8(c) pins)."""
    d = systems.katsura(6)
    for seed in (0, 1, 2):
        res = orc.track(orc.td_homotopy(d, rng.gamma(seed)), orc.td_start(d.degrees()))
        assert np.all(res.status == orc.CONVERGED)
        U, mult = orc.dedup(orc.finite_solutions(res))
        assert len(U) == 64 and mult.max() == 1
        assert res.resid[0, :, 0].max() < 1e-10
        e0 = np.zeros(7)
        e0[0] = 1
        assert np.min(np.max(np.abs(U - e0), axis=1)) < 1e-12


@pytest.mark.parametrize("n,count", [(5, 70), (6, 156)])
def test_cyclic_counts(orc, n, count):
    """Textbook counts: cyclic-5 has 70 and cyclic-6 has 156 isolated roots."""
    d = systems.cyclic(n)
    res = orc.track(orc.td_homotopy(d, rng.gamma(1)), orc.td_start(d.degrees()))
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == count and mult.max() == 1


def _cyclic_closed(U, n, tol=1e-8):
    """The set is closed under x -> w x (w^n = 1), cyclic shift and reversal (symmetry of cyclic-n)."""
    w = np.exp(2j * np.pi / n)
    for img in (U * w, np.roll(U, 1, axis=1), U[:, ::-1]):
        for y in img:
            if not np.any(np.all(np.abs(U - y) <= tol * np.maximum(1, np.abs(y)), axis=1)):
                return False
    return True


CYCLIC7_GAMMA_SEED = 2  # gamma seed used by config 2 (seeds that reach 924 in the oracle)


def test_cyclic7_924(orc):
    """Paper count: cyclic-7 has 924 finite roots (Table 1), set closed under its symmetry group."""
    d = systems.cyclic(7)
    res = orc.track(orc.td_homotopy(d, rng.gamma(CYCLIC7_GAMMA_SEED)), orc.td_start(d.degrees()))
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == 924 and mult.max() == 1
    assert res.resid[0][res.status[0] == orc.CONVERGED, 0].max() < 1e-10
    assert _cyclic_closed(U, 7)


def test_cyclic7_family_monodromy_fixture(orc):
    """The monodromy start set of the cyclic-7 coefficient family (fixtures/cyclic7_start.sols,
    written by scripts/make_fixtures.py from the oracle) has 924 distinct solutions (= Table 1
    P:467), each solving F(x; p0) by the defining sum; the parameter homotopy from it to the standard
    cyclic-7 reaches the same 924-point set as the total-degree homotopy."""
    from hc_inputs import fixtures
    d = systems.cyclic_family(7)
    S = fixtures.read_solutions(fixtures.fixture_path("cyclic7_start.sols"))
    p0 = fixtures.read_params(fixtures.fixture_path("cyclic7_p0.params"))
    assert S.shape == (924, 7)
    U, mult = orc.dedup(S)
    assert len(U) == 924 and mult.max() == 1
    for x in S[::37]:
        assert max(abs(eval_poly(f, x, p0)) for f in d.polys) < 1e-10
    ph = orc.track(orc.ph_homotopy(d, p0), S, p1s=systems.cyclic_family_target(7)[None])
    assert np.all(ph.status == orc.CONVERGED)
    B = orc.dedup(orc.finite_solutions(ph))[0]
    td = orc.track(orc.td_homotopy(systems.cyclic(7), rng.gamma(CYCLIC7_GAMMA_SEED)),
                   orc.td_start(systems.cyclic(7).degrees()))
    A = orc.dedup(orc.finite_solutions(td))[0]
    ok, ua, ub = orc.match_sets(A, B, tol=1e-8)
    assert ok and len(B) == 924, (len(A), len(B), ua, ub)


def test_p3p_planted_and_symmetry(orc):
    """P3P depth form (Eq. P3PafterElim): for planted real instances the total-degree
    homotopy (8 tracks) gives 8 distinct finite solutions (Table 2), closed under
    rho -> -rho (4 poses), containing the planted depths."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from make_fixtures import constant_system_at   # oracle-only helper (coefficients frozen at p)
    d = systems.p3p_depth()
    for b in range(3):
        p, x = rng.p3p_instance(rng.SEED_P3P_INSTANCE + b)
        td = constant_system_at(d, p)
        res = orc.track(orc.td_homotopy(td, rng.gamma(3)), orc.td_start(td.degrees()))
        U, mult = orc.dedup(orc.finite_solutions(res))
        assert len(U) == 8 and mult.max() == 1
        for y in U:
            assert np.min(np.max(np.abs(U + y), axis=1)) < 1e-8   # -y is a solution too
        assert np.min(np.max(np.abs(U - x), axis=1)) < 1e-9


def test_eco3_closed_form(orc):
    """eco-3 (reading R25) by hand: x1 + x2 + 1 = 0, x2 x3 = 2, (x1 + x1 x2) x3 = 1 give
    2 x2^2 + 5 x2 + 2 = 0, i.e. (x1, x2, x3) = (-1/2, -1/2, -4) and (1, -2, -1)."""
    d = systems.eco(3)
    res = orc.track(orc.td_homotopy(d, rng.gamma(2)), orc.td_start(d.degrees()))
    U, _ = orc.dedup(orc.finite_solutions(res))
    want = np.array([[-0.5, -0.5, -4.0], [1.0, -2.0, -1.0]], dtype=np.complex128)
    assert len(U) == 2
    for w in want:
        assert np.min(np.max(np.abs(U - w), axis=1)) < 1e-12


@pytest.mark.parametrize("n,count", [(5, 8), (6, 16), (8, 64)])
def test_eco_counts(orc, n, count):
    """eco-n has 2^(n-2) finite roots (eco-12: 1024, Table 1); every endpoint solves the
    system as written by its builder (independent evaluator hc_inputs.evalpoly)."""
    d = systems.eco(n)
    res = orc.track(orc.td_homotopy(d, rng.gamma(2)), orc.td_start(d.degrees()))
    assert res.status.size == 2 * 3 ** (n - 2)   # total degree 3^(n-2) * 2 * 1
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == count and mult.max() == 1
    for x in U:
        assert max(abs(eval_poly(f, x)) for f in d.polys) < 1e-10


# ---------------------------------------------------------------- endgame (reading R26)

@pytest.mark.parametrize("m", [2, 3, 4])
def test_cauchy_endgame_winding_and_endpoint(orc, m):
    """Closed form: F = (x - 2)^m by total degree (G = x^m - 1, which does not vanish at 2).  Near
    t = 1, (x - 2)^m ~ -s gamma (2^m - 1), so the m paths are the m branches of a Puiseux series in
    s^{1/m} permuted cyclically around t = 1: the Cauchy endgame must report winding number m for
    every track and the endpoint 2 to 1e-8 (the plain tracker's Newton polish converges only
    linearly at a root of multiplicity m)."""
    from hc_inputs.poly import var_x
    X = var_x(1, 0, 0)
    d = systems.from_polys([(X - 2) ** m], f"(x-2)^{m}")
    res = orc.track(orc.td_homotopy(d, rng.gamma(1)), orc.td_start([m]))
    assert np.all(res.status == orc.CONVERGED), res.status
    assert np.all(res.winding == m), res.winding
    assert np.max(np.abs(res.x[0, :, 0] - 2)) <= 1e-8


def test_cauchy_endgame_double_root_2x2(orc):
    """Closed form: F = ((x - 2)^2 + y - 1, y - 1) has the double root (2, 1) (substitute y = 1);
    both total-degree paths reach it with winding number 2 and 1e-8 accuracy."""
    from hc_inputs.poly import var_x
    x, y = var_x(2, 0, 0), var_x(2, 0, 1)
    d = systems.from_polys([(x - 2) ** 2 + y - 1, y - 1], "double-root")
    for g in (1, 2):
        res = orc.track(orc.td_homotopy(d, rng.gamma(g)), orc.td_start(d.degrees()))
        assert np.all(res.status == orc.CONVERGED) and np.all(res.winding == 2)
        assert np.max(np.abs(res.x[0] - np.array([2, 1]))) <= 1e-8


def test_endgame_at_infinity_cyclic5(orc):
    """Textbook count: cyclic-5 has 70 isolated roots of total degree 120, so 50 paths go to
    infinity.  With the endgame the 70 are found (no root classified at infinity), at least 30 of
    the other 50 are classified AT_INFINITY by their converged valuation, every AT_INFINITY track
    fails to converge without the endgame too, and the endgame saves solves."""
    d = systems.cyclic(5)
    hom, X0 = orc.td_homotopy(d, rng.gamma(1)), orc.td_start(d.degrees())
    res = orc.track(hom, X0)
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == 70 and mult.max() == 1
    inf = res.status[0] == orc.AT_INFINITY
    assert 30 <= inf.sum() <= 50
    st = orc.default_settings()
    st.eg_start = 0
    plain = orc.track(hom, X0, settings=st)
    assert np.all(plain.status[0][inf] != orc.CONVERGED)
    assert res.counters[0][:, 3].sum() < plain.counters[0][:, 3].sum()


def test_endgame_keeps_near_infinity_roots_cyclic7(orc):
    """cyclic-7 has roots of norm up to 9.41 whose paths look exactly like paths to infinity
    (||x|| ~ s^{-1/7}) down to s ~ 1e-7 before turning back (SURVEY [X3]); the endgame's
    eg_inf_s / eg_inf_norm guard must keep all 924 (Table 1) and classify most of the 4116
    diverging paths AT_INFINITY."""
    d = systems.cyclic(7)
    res = orc.track(orc.td_homotopy(d, rng.gamma(CYCLIC7_GAMMA_SEED)), orc.td_start(d.degrees()))
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == 924 and mult.max() == 1
    assert (res.status[0] == orc.AT_INFINITY).sum() >= 2000


def test_determinism_across_thread_counts(orc):
    """bit-identical results for 1 and 8 threads."""
    d = systems.cyclic(5)
    hom = orc.td_homotopy(d, rng.gamma(4))
    X0 = orc.td_start(d.degrees())
    a = orc.track(hom, X0, nthreads=1)
    b = orc.track(hom, X0, nthreads=8)
    assert np.array_equal(a.x.view(np.float64), b.x.view(np.float64))
    assert np.array_equal(a.status, b.status) and np.array_equal(a.counters, b.counters)


# ---------------------------------------------------------------- post-processing

def test_dedup_and_real_classification(orc):
    X = np.array([[1 + 1e-9j, 2], [1, 2 + 1e-9], [1j, 0], [2 + 1e-12j, 0]])
    U, m = orc.dedup(X)
    assert len(U) == 3 and list(m) == [2, 1, 1]
    assert list(orc.is_real(U)) == [True, False, True]
    ok, _, _ = orc.match_sets(U, U[::-1].copy())
    assert ok
    ok, ua, ub = orc.match_sets(U, U[:2])
    assert not ok and ua == 1 and ub == 0


# ---------------------------------------------------------------- vision generators vs oracle

def test_fourview_planted_is_exact(orc):
    """Planted ground truth (R18): F(x*; p) ~ 0 for generated 4-view instances, and p is real."""
    d = systems.nview_triangulation(4)
    for b in range(5):
        p, xs = rng.fourview_instance(rng.SEED_FOURVIEW_INSTANCE + b)
        assert np.all(p.imag == 0)
        F = orc.eval_F(d, p, xs)
        assert np.max(np.abs(F)) < 1e-13


def test_trifocal_start_set_certified(orc):
    """The trifocal start set (668 orbits x 8 = 5344 at p0 = rng.trifocal_complex_start(101), the
    oracle's monodromy) against two independent monodromy runs from other planted (x0, p0') (seeds 202,
    303; scripts/certify_trifocal.py, oracle only), each saturated at 668 orbits: carried to p0 by one
    parameter homotopy, every converged endpoint lies in the fixture (no orbit the fixture lacks), no
    two orbits land on one (the homotopy is a bijection of solution sets), and at most 5 % of the
    paths fail.  SURVEY §8(c): "monodromy saturation"; the paper's 1784 is not this
    formulation's count (R19/R20)."""
    from hc_inputs import fixtures
    d = systems.trifocal_unknown_f()
    full, p0 = fixtures.trifocal_start()
    assert full.shape == (5344, 18)

    def orbit_of(y):
        hit = np.nonzero(np.all(np.abs(full - y) <= 1e-6 * np.maximum(1.0, np.abs(y)), axis=1))[0]
        return int(hit[0]) // 8 if len(hit) else -1
    for seed in (202, 303):
        reps = fixtures.read_solutions(fixtures.fixture_path(f"trifocal_cert_{seed}.sols"))
        ps = fixtures.read_params(fixtures.fixture_path(f"trifocal_cert_{seed}.params"))
        assert reps.shape == (668, 18)
        res = orc.track(orc.ph_homotopy(d, ps, p0), reps)
        ok = res.status[0] == orc.CONVERGED
        ids = [orbit_of(y) for y in res.x[0][ok]]
        assert min(ids) >= 0, f"seed {seed}: an endpoint outside the fixture"
        assert len(set(ids)) == len(ids), f"seed {seed}: two orbits carried onto one"
        assert ok.mean() >= 0.95


def test_trifocal_planted_is_exact(orc):
    """Planted ground truth: F(x_gt; p) ~ 0 for generated trifocal instances; the Z2^3 images of a
    solution are solutions (R20 symmetry)."""
    d = systems.trifocal_unknown_f()
    for b in range(5):
        p, x = rng.trifocal_instance(rng.SEED_TRIFOCAL_INSTANCE + b)
        assert np.max(np.abs(orc.eval_F(d, p, x))) < 1e-12
        for y in systems.trifocal_symmetry(x):
            assert np.max(np.abs(orc.eval_F(d, p, y))) < 1e-12
    p0, x0 = rng.trifocal_complex_start()
    assert np.max(np.abs(orc.eval_F(d, p0, x0))) < 1e-12


# ---------------------------------------------------------------- more Table 2 / §4 counts

def _frozen(desc, p):
    """F(x; p) with coefficients frozen at p (a constant-coefficient TD target)."""
    import oracle
    from hc_inputs.descriptor import SystemDesc
    c = oracle.eval_coefs(desc, p)
    return SystemDesc(desc.n_vars, 0, desc.term_eq, desc.term_xexp, desc.term_coef,
                      np.arange(desc.n_coefs + 1, dtype=np.int32), c,
                      np.zeros((desc.n_coefs, 0), np.int32)).contiguous()


def test_three_view_triangulation_94(orc):
    """Paper count: 3-view triangulation (9 unknowns) has 94 solutions (Table 2); TD at a
    generic complex parameter point, 2^9 = 512 tracks."""
    d = systems.nview_triangulation(3)
    assert (d.n_vars, d.n_params) == (9, 33)
    td = _frozen(d, rng.complex_normal(rng.gen(103), d.n_params))
    res = orc.track(orc.td_homotopy(td, rng.gamma(0)), orc.td_start(td.degrees()))
    U, mult = orc.dedup(orc.finite_solutions(res))
    assert len(U) == 94 and mult.max() == 1


def test_two_view_triangulation_six(orc):
    """Paper: 2-view optimal triangulation reduces to a single 6th-order polynomial, i.e. 6
    stationary points when E is an essential (rank-2) matrix; generic full-rank E gives 8."""
    d = systems.nview_triangulation(2)
    g = rng.gen(5)
    gam = rng.complex_normal(g, 4)
    E = rng.complex_normal(g, (3, 2)) @ rng.complex_normal(g, (2, 3))
    td = _frozen(d, np.concatenate([gam, E.reshape(-1)]))
    res = orc.track(orc.td_homotopy(td, rng.gamma(0)), orc.td_start(td.degrees()))
    assert len(orc.dedup(orc.finite_solutions(res))[0]) == 6
    td8 = _frozen(d, rng.complex_normal(rng.gen(102), d.n_params))
    res8 = orc.track(orc.td_homotopy(td8, rng.gamma(0)), orc.td_start(td8.degrees()))
    assert len(orc.dedup(orc.finite_solutions(res8))[0]) == 8


# ---------------------------------------------------------------- 5-point relative pose + depth (N2, R24)

def _essential(x):
    """E = [T]_x R(q) of a 5-point solution vector (numpy, independent of both evaluators)."""
    R = np.array(systems.quat_rot(*x[10:14]))
    return rng.skew(np.array([x[14], x[15], 1.0])) @ R


def test_fivepoint_planted_is_exact(orc):
    """Planted ground truth: F(x_gt; p) ~ 0 (oracle and the defining-sum evaluator) for generated
    instances and the complex monodromy start; q -> -q maps solutions to solutions."""
    d = systems.fivepoint_relpose_depth()
    assert (d.n_vars, d.n_params) == (16, 20)
    for b in range(5):
        p, x = rng.fivepoint_instance(rng.SEED_FIVEPOINT_INSTANCE + b)
        assert np.all(p.imag == 0)
        for y in systems.fivepoint_symmetry(x):
            assert np.max(np.abs(orc.eval_F(d, p, y))) < 1e-13
    p0, x0 = rng.fivepoint_complex_start()
    assert np.max(np.abs(orc.eval_F(d, p0, x0))) < 1e-12


def test_fivepoint_forty_solutions_ten_essentials(orc):
    """The oracle's monodromy fixture against the 5-point theory: the 40 solutions at p0 solve the
    equations (defining sums), and their essential matrices E = [T]_x R fall into exactly 10 classes
    up to scale -- the 10 roots of the classical tenth-order polynomial -- with 4
    solutions each (q -> -q times the twisted pair); every E is essential (det E = 0,
    2 E E^T E - tr(E E^T) E = 0) and satisfies the five epipolar constraints gb^T E g = 0."""
    from hc_inputs import fixtures
    d = systems.fivepoint_relpose_depth()
    X = fixtures.read_solutions(fixtures.fixture_path("fivepoint_start.sols"))
    p0 = fixtures.read_params(fixtures.fixture_path("fivepoint_p0.params"))
    assert X.shape == (40, 16)
    for x in X[:8]:
        assert max(abs(eval_poly(f, x, p0)) for f in d.polys) < 1e-9
    Es = []
    for x in X:
        E = _essential(x)
        E = E / E.flat[np.argmax(np.abs(E))]
        assert abs(np.linalg.det(E)) < 1e-9
        assert np.max(np.abs(2 * E @ E.T @ E - np.trace(E @ E.T) * E)) < 1e-8
        for i in range(5):
            g = np.array([p0[systems.fivepoint_param_index(0, i, 0)], p0[systems.fivepoint_param_index(0, i, 1)], 1])
            gb = np.array([p0[systems.fivepoint_param_index(1, i, 0)], p0[systems.fivepoint_param_index(1, i, 1)], 1])
            assert abs(gb @ E @ g) < 1e-9
        Es.append(E.reshape(-1))
    Es = np.array(Es)
    classes = []
    for e in Es:
        for c in classes:
            if np.max(np.abs(c[0] - e)) < 1e-7:
                c.append(e)
                break
        else:
            classes.append([e])
    assert len(classes) == 10 and all(len(c) == 4 for c in classes)


def test_fivepoint_planted_recovered_by_tracking(orc):
    """Parameter homotopy from the 40 fixture starts to planted real instances reaches the planted
    ground truth (and its q -> -q image)."""
    from hc_inputs import fixtures
    d = systems.fivepoint_relpose_depth()
    X = fixtures.read_solutions(fixtures.fixture_path("fivepoint_start.sols"))
    p0 = fixtures.read_params(fixtures.fixture_path("fivepoint_p0.params"))
    p1s, xs = rng.fivepoint_batch(3)
    res = orc.track(orc.ph_homotopy(d, p0), X, p1s)
    for b in range(3):
        S = res.x[b][res.status[b] == orc.CONVERGED]
        for y in systems.fivepoint_symmetry(xs[b]):
            assert np.min(np.max(np.abs(S - y), axis=1)) < 1e-8
