"""Polynomial systems of the paper's benchmarks and vision problems, as descriptors.

Only formulations: each builder writes F(x; p) down (§4, Table 1,
SURVEY.md §8(c) readings R16-R20) and expands it with `hc_inputs.poly`.
"""
from __future__ import annotations

import itertools

from .descriptor import SystemDesc, desc_from_equations
from .poly import Poly, const, var_p, var_x


# ---------------------------------------------------------------------------
# Polynomial benchmarks (Table 1) and textbook systems
# ---------------------------------------------------------------------------

def katsura(n: int) -> SystemDesc:
    """katsura-n: n+1 unknowns x_0..x_n (BASELINE.json configs[0]; textbook family).

    sum_{l=-n}^{n} x_|l| x_|m-l| - x_m = 0  (m = 0..n-1),   x_0 + 2 sum_{l>=1} x_l - 1 = 0.
    Bezout number 2^n equals its root count (all finite, SURVEY.md §8(c) pins).
    """
    N = n + 1
    X = [var_x(N, 0, i) for i in range(N)]

    def xa(k):
        k = abs(k)
        return X[k] if k <= n else None

    eqs = []
    for m in range(n):
        f = const(N, 0, 0)
        for l in range(-n, n + 1):
            a, b = xa(l), xa(m - l)
            if a is not None and b is not None:
                f = f + a * b
        eqs.append(f - X[m])
    lin = X[0] - 1
    for l in range(1, N):
        lin = lin + 2 * X[l]
    eqs.append(lin)
    return desc_from_equations(eqs, name=f"katsura-{n}", var_names=[f"x{i}" for i in range(N)])


def cyclic(n: int) -> SystemDesc:
    """cyclic-n (Table 1, cited [backelin1991we]; standard definition SPEC).

    f_k = sum_{i=0}^{n-1} prod_{j=0}^{k-1} x_{(i+j) mod n}  (k = 1..n-1),   f_n = x_0 x_1 ... x_{n-1} - 1.
    """
    X = [var_x(n, 0, i) for i in range(n)]
    eqs = []
    for k in range(1, n):
        f = const(n, 0, 0)
        for i in range(n):
            m = const(n, 0, 1)
            for j in range(k):
                m = m * X[(i + j) % n]
            f = f + m
        eqs.append(f)
    m = const(n, 0, 1)
    for i in range(n):
        m = m * X[i]
    eqs.append(m - 1)
    return desc_from_equations(eqs, name=f"cyclic-{n}", var_names=[f"x{i}" for i in range(n)])


def coefficient_family(base: SystemDesc, name: str = "") -> SystemDesc:
    """The family of `base` (a system with constant coefficients) with a free coefficient per term:
    the same monomial support, term q of base's flattened term list multiplied by parameter p_q
    (the paper's monodromy-start + parameter-homotopy workflow, applied to its
    Table 1 benchmarks).  `base` itself is the member family_target(base)."""
    n, T = base.n_vars, base.n_terms
    eqs = [const(n, T, 0) for _ in range(n)]
    for q in range(T):
        i = int(base.term_eq[q])
        m = var_p(n, T, q)
        for v in range(n):
            for _ in range(int(base.term_xexp[q, v])):
                m = m * var_x(n, T, v)
        eqs[i] = eqs[i] + m
    return desc_from_equations(eqs, name=name or f"{base.name}-family", var_names=base.var_names)


def family_target(base: SystemDesc):
    """Parameters of coefficient_family(base) that give `base`."""
    import numpy as np
    return np.array([complex(base.coef_w[base.coef_ptr[base.term_coef[q]]]) for q in range(base.n_terms)])


def cyclic_family(n: int) -> SystemDesc:
    """cyclic-n coefficient family (Table 1); the standard cyclic-n is cyclic_family_target(n)."""
    return coefficient_family(cyclic(n), name=f"cyclic-{n}-family")


def cyclic_family_target(n: int):
    return family_target(cyclic(n))


def eco(n: int) -> SystemDesc:
    """eco-n (Table 1: eco-12, 12 unknowns, 1024 solutions; the paper cites the
    benchmark without writing it down -- standard economics-modelling family, reading R25):

    f_k = (x_k + sum_{i=1}^{n-k-1} x_i x_{i+k}) x_n - k   (k = 1..n-1),   f_n = x_1 + ... + x_{n-1} + 1.
    Degrees 3 (k <= n-2), 2 (k = n-1), 1: total degree 2 * 3^(n-2) (eco-12: 118,098 tracks); the
    family has 2^(n-2) finite solutions (eco-12: 1024 = Table 1).
    """
    X = [var_x(n, 0, i) for i in range(n)]   # X[i] = x_{i+1}
    eqs = []
    for k in range(1, n):
        inner = X[k - 1]
        for i in range(1, n - k):
            inner = inner + X[i - 1] * X[i + k - 1]
        eqs.append(inner * X[n - 1] - k)
    lin = const(n, 0, 1)
    for i in range(n - 1):
        lin = lin + X[i]
    eqs.append(lin)
    return desc_from_equations(eqs, name=f"eco-{n}", var_names=[f"x{i + 1}" for i in range(n)])


def univariate(coeffs) -> SystemDesc:
    """f(x) = sum_k coeffs[k] x^k  (one equation, one unknown; test system)."""
    X = var_x(1, 0, 0)
    f = const(1, 0, 0)
    for k, c in enumerate(coeffs):
        if c != 0:
            f = f + complex(c) * X ** k
    return desc_from_equations([f], name=f"univariate-{len(coeffs) - 1}", var_names=["x"])


def univariate_param(deg: int) -> SystemDesc:
    """f(x; p) = sum_{k=0}^{deg} p_k x^k: a parameter homotopy family for tests (P = deg+1)."""
    P = deg + 1
    X = var_x(1, P, 0)
    f = const(1, P, 0)
    for k in range(P):
        f = f + var_p(1, P, k) * X ** k
    return desc_from_equations([f], name=f"univariate-param-{deg}", var_names=["x"])


def from_polys(eqs: list[Poly], name: str = "") -> SystemDesc:
    return desc_from_equations(eqs, name=name)


# ---------------------------------------------------------------------------
# N-view triangulation, all pairs (reading R17)
# ---------------------------------------------------------------------------

def nview_pairs(nv: int):
    return [(i, j) for i in range(nv) for j in range(i + 1, nv)]


def nview_triangulation(nv: int = 4) -> SystemDesc:
    """Stationarity system of L = sum_k (u_k^2+v_k^2) + sum_{i<j} lambda_ij c_ij (reading R17).

    c_ij = (gamma_j - dgamma_j)^T E_ij (gamma_i - dgamma_i), gamma_k = (xi_k, eta_k, 1),
    dgamma_k = (u_k, v_k, 0).
    Unknowns x = (u_1, v_1, ..., u_nv, v_nv, lambda_ij for i<j): 2nv + nv(nv-1)/2 (14 for nv=4).
    Parameters p = (xi_1, eta_1, ..., xi_nv, eta_nv, vec(E_ij) row-major per pair): 2nv + 9*pairs (62 for nv=4).
    Equation order: dL/du_1, dL/dv_1, ..., dL/dv_nv, then c_ij in pair order.
    """
    pairs = nview_pairs(nv)
    n = 2 * nv + len(pairs)
    P = 2 * nv + 9 * len(pairs)
    X = [var_x(n, P, i) for i in range(n)]
    Pv = [var_p(n, P, q) for q in range(P)]
    one = const(n, P, 1)
    zero = const(n, P, 0)

    def gvec(k):  # gamma_k - dgamma_k
        return [Pv[2 * k] - X[2 * k], Pv[2 * k + 1] - X[2 * k + 1], one]

    L = zero
    for k in range(nv):
        L = L + X[2 * k] * X[2 * k] + X[2 * k + 1] * X[2 * k + 1]
    cons = []
    for pi, (i, j) in enumerate(pairs):
        a, b = gvec(j), gvec(i)
        E = [[Pv[2 * nv + 9 * pi + 3 * r + s] for s in range(3)] for r in range(3)]
        c = zero
        for r in range(3):
            for s in range(3):
                c = c + a[r] * E[r][s] * b[s]
        cons.append(c)
        L = L + X[2 * nv + pi] * c
    eqs = [L.diff_x(v) for v in range(2 * nv)] + cons
    names = [f"{c}{k + 1}" for k in range(nv) for c in ("u", "v")] + [f"l{i + 1}{j + 1}" for i, j in pairs]
    return desc_from_equations(eqs, name=f"{nv}-view-triangulation", var_names=names)


# ---------------------------------------------------------------------------
# Trifocal relative pose with a common unknown focal length (PAPER.md P:330-351,
# readings R19/R20)
# ---------------------------------------------------------------------------

TRIFOCAL_VARS = ["f", "a12", "b12", "c12", "d12", "a13", "b13", "c13", "d13",
                 "T12x", "T12y", "T12z", "T13x", "T13y", "T13z", "l2", "l3", "l4"]


def quat_rot(a, b, c, d):
    """R(q) for q=(a,b,c,d); a rotation when a^2+b^2+c^2+d^2 = 1."""
    return [[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
            [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
            [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]]


def trifocal_param_index(view: int, point: int, coord: int) -> int:
    """p index of image coordinate `coord` (0: xi, 1: eta) of `point` (0..3) in `view` (0..2)."""
    return 8 * view + 2 * point + coord


def trifocal_unknown_f() -> SystemDesc:
    """18x18 trifocal pose with unknown focal length (reading R19/R20).

    With r_v = f K^{-1} gamma_v = (xi_v, eta_v, f) and lambda = depth/f, P:334-335 reads
    lambda_v r_v = lambda R_1v r_1 + T_1v.  Eliminating lambda_v by the third row:
        xi_v (lambda R r_1 + T)_3 - f (lambda R r_1 + T)_1 = 0,
        eta_v (lambda R r_1 + T)_3 - f (lambda R r_1 + T)_2 = 0,   v = 2, 3; four points,
    plus q12.q12 = 1, q13.q13 = 1.  Scale fixed by lambda of point 1 = 1 (R20).
    Unknowns TRIFOCAL_VARS (18); parameters: 24 image coordinates, trifocal_param_index order.
    """
    n, P = 18, 24
    X = [var_x(n, P, i) for i in range(n)]
    Pv = [var_p(n, P, q) for q in range(P)]
    one = const(n, P, 1)
    f = X[0]
    q = {2: X[1:5], 3: X[5:9]}
    T = {2: X[9:12], 3: X[12:15]}
    lam = [one, X[15], X[16], X[17]]
    eqs = []
    for v in (2, 3):
        R = quat_rot(*q[v])
        for k in range(4):
            r1 = [Pv[trifocal_param_index(0, k, 0)], Pv[trifocal_param_index(0, k, 1)], f]
            w = []
            for row in range(3):
                s = R[row][0] * r1[0] + R[row][1] * r1[1] + R[row][2] * r1[2]
                w.append(lam[k] * s + T[v][row])
            xi = Pv[trifocal_param_index(v - 1, k, 0)]
            eta = Pv[trifocal_param_index(v - 1, k, 1)]
            eqs.append(xi * w[2] - f * w[0])
            eqs.append(eta * w[2] - f * w[1])
    for v in (2, 3):
        a, b, c, d = q[v]
        eqs.append(a * a + b * b + c * c + d * d - 1)
    return desc_from_equations(eqs, name="trifocal-unknown-f", var_names=TRIFOCAL_VARS)


def trifocal_symmetry(x):
    """The Z_2^3 action on trifocal solutions (SURVEY.md §8(c) R20 symmetry note).

    Yields the 8 images of one solution vector x (length 18, any array-like of complex):
    sigma_1: q12 -> -q12, sigma_2: q13 -> -q13, tau: conjugation by diag(1,1,-1).
    """
    import numpy as np
    x = np.asarray(x, dtype=np.complex128)
    out = []
    for s1, s2, tau in itertools.product((1, -1), (1, -1), (False, True)):
        y = x.copy()
        y[1:5] *= s1
        y[5:9] *= s2
        if tau:
            y[0] = -y[0]
            for base in (1, 5):
                y[base + 1] = -y[base + 1]
                y[base + 2] = -y[base + 2]
            y[11] = -y[11]
            y[14] = -y[14]
        out.append(y)
    return out


# ---------------------------------------------------------------------------
# Five-point relative pose with depth reconstruction (Table 2 P:492;
# reading R24)
# ---------------------------------------------------------------------------

FIVEPOINT_VARS = ([f"rho{i + 1}" for i in range(5)] + [f"rhob{i + 1}" for i in range(5)]
                  + ["a", "b", "c", "d", "tx", "ty"])


def fivepoint_param_index(view: int, point: int, coord: int) -> int:
    """p index of image coordinate `coord` (0: u, 1: v) of `point` (0..4) in `view` (0: gamma, 1: gamma-bar)."""
    return 10 * view + 2 * point + coord


def fivepoint_relpose_depth() -> SystemDesc:
    """16x16 relative pose + depth reconstruction (reading R24).

    rhob_i gammab_i = R(q) rho_i gamma_i + T for five correspondences gamma_i = (u_i, v_i, 1),
    gammab_i = (ub_i, vb_i, 1) (the 15 equations of, row by row), plus q.q = 1 (P:207:
    "quaternions which involves 4 unknowns with one equation").  The scale is fixed by T_z = 1,
    T = (tx, ty, 1) (the 2-parameter T-hat of P:207).  Unknowns FIVEPOINT_VARS (16);
    parameters: 20 image coordinates in fivepoint_param_index order.
    """
    n, P = 16, 20
    X = [var_x(n, P, i) for i in range(n)]
    Pv = [var_p(n, P, q) for q in range(P)]
    one = const(n, P, 1)
    rho, rhob = X[0:5], X[5:10]
    a, b, c, d = X[10:14]
    T = [X[14], X[15], one]
    R = quat_rot(a, b, c, d)
    eqs = []
    for i in range(5):
        g = [Pv[fivepoint_param_index(0, i, 0)], Pv[fivepoint_param_index(0, i, 1)], one]
        gb = [Pv[fivepoint_param_index(1, i, 0)], Pv[fivepoint_param_index(1, i, 1)], one]
        for row in range(3):
            Rg = R[row][0] * g[0] + R[row][1] * g[1] + R[row][2] * g[2]
            eqs.append(rhob[i] * gb[row] - rho[i] * Rg - T[row])
    eqs.append(a * a + b * b + c * c + d * d - 1)
    return desc_from_equations(eqs, name="5pt-relpose-depth", var_names=FIVEPOINT_VARS)


def fivepoint_symmetry(x):
    """q -> -q leaves R(q) and hence every equation unchanged: the two images of a solution."""
    import numpy as np
    x = np.asarray(x, dtype=np.complex128)
    y = x.copy()
    y[10:14] = -y[10:14]
    return [x, y]


# ---------------------------------------------------------------------------
# P3P absolute pose, depth form (PAPER.md Eq. P3PafterElim; Table 2: 3 unknowns,
# 8 solutions)
# ---------------------------------------------------------------------------

P3P_VARS = ["rho1", "rho2", "rho3"]


def p3p_param_index(kind: int, point: int, coord: int) -> int:
    """kind 0: image point gamma_i = (u_i, v_i, 1), coord 0..1 -> 0..5; kind 1: world point Gamma_i,
    coord 0..2 -> 6..14."""
    return 2 * point + coord if kind == 0 else 6 + 3 * point + coord


def p3p_depth() -> SystemDesc:
    """(Gamma_j - Gamma_1)^T (Gamma_k - Gamma_1) = (rho_j gamma_j - rho_1 gamma_1)^T (rho_k gamma_k - rho_1 gamma_1)
    for (j, k) = (2, 2), (3, 3), (2, 3): three quadratics in the depths rho_1..3 with
    gamma_i = (u_i, v_i, 1) (calibrated image points) and the world points Gamma_i as parameters
    (p3p_param_index).  Bezout number 8 = the 8 solutions of Table 2 P:512 (4 poses x rho -> -rho,
    P:242)."""
    n, P = 3, 15
    X = [var_x(n, P, i) for i in range(n)]
    Pv = [var_p(n, P, q) for q in range(P)]
    one = const(n, P, 1)
    gam = [[Pv[p3p_param_index(0, i, 0)], Pv[p3p_param_index(0, i, 1)], one] for i in range(3)]
    Gam = [[Pv[p3p_param_index(1, i, c)] for c in range(3)] for i in range(3)]
    def dotp(a, b):
        return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]
    D = [[Gam[j][c] - Gam[0][c] for c in range(3)] for j in range(3)]
    V = [[X[j] * gam[j][c] - X[0] * gam[0][c] for c in range(3)] for j in range(3)]
    eqs = [dotp(D[j], D[k]) - dotp(V[j], V[k]) for j, k in ((1, 1), (2, 2), (1, 2))]
    return desc_from_equations(eqs, name="p3p-depth", var_names=P3P_VARS)

