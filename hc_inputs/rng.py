"""Seeded synthetic inputs (SURVEY.md §8(c) R22, §8(d) "Concrete synthetic inputs").

numpy PCG64 with documented seed bases.  Everything here is input data: gamma,
random complex parameter points, and planted geometric instances.  None of it
evaluates the homotopy.
"""
from __future__ import annotations

import numpy as np

from . import systems

# seed bases (R22)
SEED_FOURVIEW_INSTANCE = 3_000_000
SEED_FOURVIEW_P0 = 7
SEED_TRIFOCAL_INSTANCE = 4_000_000
SEED_TRIFOCAL_SWEEP = 5_000_000
SEED_TRIFOCAL_MONODROMY = 101   # (round 1: 11, whose monodromy set lacked 2 orbits; scripts/certify_trifocal.py)


def gen(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def gamma(seed: int) -> complex:
    """gamma = exp(2 pi i theta), theta ~ U[0,1) from PCG64(seed) (reading R1)."""
    th = gen(seed).random()
    return complex(np.cos(2 * np.pi * th), np.sin(2 * np.pi * th))


def complex_normal(g: np.random.Generator, size) -> np.ndarray:
    """(N(0,1) + i N(0,1)) / sqrt(2)."""
    return (g.standard_normal(size) + 1j * g.standard_normal(size)) / np.sqrt(2.0)


def random_rotation(g: np.random.Generator, lo=0.1, hi=0.5):
    """Rotation by an angle in [lo, hi] rad about a uniformly random axis; also its unit quaternion."""
    ax = g.standard_normal(3)
    ax /= np.linalg.norm(ax)
    th = g.uniform(lo, hi)
    q = np.concatenate([[np.cos(th / 2)], np.sin(th / 2) * ax])
    a, b, c, d = q
    R = np.array([[a * a + b * b - c * c - d * d, 2 * (b * c - a * d), 2 * (b * d + a * c)],
                  [2 * (b * c + a * d), a * a - b * b + c * c - d * d, 2 * (c * d - a * b)],
                  [2 * (b * d - a * c), 2 * (c * d + a * b), a * a - b * b - c * c + d * d]])
    return R, q


def skew(t):
    return np.array([[0, -t[2], t[1]], [t[2], 0, -t[0]], [-t[1], t[0], 0]])


# ---------------------------------------------------------------------------
# 4-view triangulation (config 3)
# ---------------------------------------------------------------------------

def fourview_linear_in_E(x: np.ndarray, gam: np.ndarray, nv: int = 4):
    """F(x; gamma, E) = A vec(E) + b for fixed (x, gamma): the N-view system is affine in E.

    Closed form of the equations written in systems.nview_triangulation (same order),
    used only to plant an exact solution (min-norm correction of E, reading R18).
    gam: [nv, 2] image coordinates (xi, eta).
    """
    pairs = systems.nview_pairs(nv)
    n = 2 * nv + len(pairs)
    A = np.zeros((n, 9 * len(pairs)), dtype=np.complex128)
    b = np.zeros(n, dtype=np.complex128)
    u = x[0:2 * nv:2]
    v = x[1:2 * nv:2]
    lam = x[2 * nv:]

    def g(k):
        return np.array([gam[k, 0] - u[k], gam[k, 1] - v[k], 1.0])

    for k in range(nv):
        b[2 * k] = 2 * u[k]
        b[2 * k + 1] = 2 * v[k]
    for pi, (i, j) in enumerate(pairs):
        a_, b_ = g(j), g(i)
        base = 9 * pi
        for r in range(3):
            for s in range(3):
                col = base + 3 * r + s
                A[2 * nv + pi, col] += a_[r] * b_[s]            # c_ij
                # d c_ij / d u_i = -sum_r a_r E[r,0] ; d/dv_i = -sum_r a_r E[r,1]
                if s == 0:
                    A[2 * i, col] += -lam[pi] * a_[r]
                if s == 1:
                    A[2 * i + 1, col] += -lam[pi] * a_[r]
                # d c_ij / d u_j = -sum_s E[0,s] b_s ; d/dv_j = -sum_s E[1,s] b_s
                if r == 0:
                    A[2 * j, col] += -lam[pi] * b_[s]
                if r == 1:
                    A[2 * j + 1, col] += -lam[pi] * b_[s]
    return A, b


def fourview_instance(seed: int, nv: int = 4):
    """Planted real 4-view instance (SURVEY.md §8(d) config 3 recipe).

    Camera 1 = [I|0]; cameras 2..nv rotated 0.1-0.5 rad about random axes, centres N(0, 0.5^2);
    point (0,0,5) + N(0, 0.5^2); normalised image coords + N(0, 1e-3^2);
    E_ij = [t_ij]x R_ij (unit t) + N(0, 0.01^2) (pose noise, reading R18);
    planted x* = (dgamma ~ N(0, 1e-3^2), lambda ~ N(0, 0.05^2)), made exact by the min-norm dE.
    Returns (p [P] complex, x_star [n] complex).
    """
    g = gen(seed)
    Rs, ts = [np.eye(3)], [np.zeros(3)]
    for _ in range(1, nv):
        R, _q = random_rotation(g)
        C = g.normal(0, 0.5, 3)
        Rs.append(R)
        ts.append(-R @ C)
    Xw = np.array([0.0, 0.0, 5.0]) + g.normal(0, 0.5, 3)
    gam = np.zeros((nv, 2))
    for k in range(nv):
        Xc = Rs[k] @ Xw + ts[k]
        gam[k] = Xc[:2] / Xc[2] + g.normal(0, 1e-3, 2)
    pairs = systems.nview_pairs(nv)
    Evec = []
    for (i, j) in pairs:
        Rij = Rs[j] @ Rs[i].T
        tij = ts[j] - Rij @ ts[i]
        tij = tij / np.linalg.norm(tij)
        E = skew(tij) @ Rij + g.normal(0, 0.01, (3, 3))
        Evec.append(E.reshape(-1))
    Evec = np.concatenate(Evec)
    n = 2 * nv + len(pairs)
    xs = np.zeros(n)
    xs[:2 * nv] = g.normal(0, 1e-3, 2 * nv)
    xs[2 * nv:] = g.normal(0, 0.05, len(pairs))
    A, b = fourview_linear_in_E(xs.astype(np.complex128), gam, nv)
    r = A @ Evec + b
    dE, *_ = np.linalg.lstsq(A.real, -r.real, rcond=None)
    Evec = Evec + dE
    p = np.concatenate([gam.reshape(-1), Evec]).astype(np.complex128)
    return p, xs.astype(np.complex128)


def fourview_p0(seed: int = SEED_FOURVIEW_P0, nv: int = 4) -> np.ndarray:
    """Generic complex start parameters for the 4-view PH (reading R3): complex Gaussian, P = 62."""
    P = 2 * nv + 9 * len(systems.nview_pairs(nv))
    return complex_normal(gen(seed), P)


def fourview_batch(n_instances: int, base: int = SEED_FOURVIEW_INSTANCE):
    ps, xs = zip(*(fourview_instance(base + b) for b in range(n_instances)))
    return np.stack(ps), np.stack(xs)


# ---------------------------------------------------------------------------
# Trifocal pose with unknown focal length (configs 4, 5)
# ---------------------------------------------------------------------------

def trifocal_project(x: np.ndarray, view1: np.ndarray) -> np.ndarray:
    """Image coords of views 2, 3 that make x an exact solution, given view-1 coords [4, 2].

    x in systems.TRIFOCAL_VARS order; closed form xi_v = f w_1 / w_3, eta_v = f w_2 / w_3 with
    w = lambda R r_1 + T (reading R19).  Returns p [24].
    """
    f = x[0]
    q = {2: x[1:5], 3: x[5:9]}
    T = {2: x[9:12], 3: x[12:15]}
    lam = np.concatenate([[1.0], x[15:18]])
    p = np.zeros(24, dtype=np.result_type(x, view1, np.complex128))
    for k in range(4):
        p[systems.trifocal_param_index(0, k, 0)] = view1[k, 0]
        p[systems.trifocal_param_index(0, k, 1)] = view1[k, 1]
    for v in (2, 3):
        R = np.array(systems.quat_rot(*q[v]))
        for k in range(4):
            r1 = np.array([view1[k, 0], view1[k, 1], f])
            w = lam[k] * (R @ r1) + T[v]
            p[systems.trifocal_param_index(v - 1, k, 0)] = f * w[0] / w[2]
            p[systems.trifocal_param_index(v - 1, k, 1)] = f * w[1] / w[2]
    return p


def trifocal_instance(seed: int):
    """Planted real trifocal instance (SURVEY.md §8(d) config 4 recipe).

    3 cameras, common f ~ U[0.8, 1.2] (units of 1000 px); rotations 0.1-0.5 rad; T ~ N(0,1);
    4 points with depth 4-6 in front of all cameras; xi, eta = f X/Z, noise-free.
    Returns (p [24] complex, x_gt [18] complex) with lambda_1 = 1 scaling (R20).
    """
    g = gen(seed)
    while True:
        f = g.uniform(0.8, 1.2)
        R2, q2 = random_rotation(g)
        R3, q3 = random_rotation(g)
        T2, T3 = g.normal(0, 1, 3), g.normal(0, 1, 3)
        Z = g.uniform(4, 6, 4)
        dirs = g.uniform(-0.3, 0.3, (4, 2))
        Xw = np.stack([np.array([dirs[k, 0] * Z[k], dirs[k, 1] * Z[k], Z[k]]) for k in range(4)])
        ok = True
        for R, T in ((R2, T2), (R3, T3)):
            Zc = (Xw @ R.T + T)[:, 2]
            ok &= bool(np.all(Zc > 1.0))
        if ok:
            break
    view1 = f * Xw[:, :2] / Xw[:, 2:3]
    # lambda = depth / f ; scale so lambda of point 1 is 1: lambda_k = Z_k / Z_0, T' = T f / Z_0
    lam = Z / Z[0]
    x = np.concatenate([[f], q2, q3, T2 * f / Z[0], T3 * f / Z[0], lam[1:]]).astype(np.complex128)
    p = trifocal_project(x, view1.astype(np.complex128))
    return p, x


def trifocal_batch(n_instances: int, base: int = SEED_TRIFOCAL_INSTANCE):
    ps, xs = zip(*(trifocal_instance(base + b) for b in range(n_instances)))
    return np.stack(ps), np.stack(xs)


def trifocal_complex_start(seed: int = SEED_TRIFOCAL_MONODROMY):
    """Planted generic complex (x0, p0) for monodromy (SURVEY.md [X6]):
    random complex x0 with q normalised by the complex square root of q.q, random complex view-1
    coordinates, views 2-3 from the closed form."""
    g = gen(seed)
    x = complex_normal(g, 18)
    for base in (1, 5):
        qq = np.sum(x[base:base + 4] ** 2)
        x[base:base + 4] /= np.sqrt(qq)
    view1 = complex_normal(g, (4, 2))
    return trifocal_project(x, view1), x


def fourview_complex_start(seed: int = 23, nv: int = 4):
    """Planted generic complex (x0, p0) for 4-view monodromy: complex random x0 and image points,
    E chosen as the min-norm complex solution of the (affine in E) system F(x0; gamma, E) = 0
    plus a random complex component in its null space."""
    g = gen(seed)
    pairs = systems.nview_pairs(nv)
    n = 2 * nv + len(pairs)
    x0 = complex_normal(g, n)
    gam = complex_normal(g, (nv, 2))
    A, b = fourview_linear_in_E(x0, gam, nv)
    E0, *_ = np.linalg.lstsq(A, -b, rcond=None)
    # add a generic null-space component so p0 is not the minimum-norm (special) point
    _, _, Vh = np.linalg.svd(A)
    null = Vh[A.shape[0]:].conj().T
    E = E0 + null @ complex_normal(g, null.shape[1])
    return np.concatenate([gam.reshape(-1), E]).astype(np.complex128), x0


# ---------------------------------------------------------------------------
# Five-point relative pose + depth (N2 workload, reading R24)
# ---------------------------------------------------------------------------

SEED_FIVEPOINT_INSTANCE = 6_000_000
SEED_FIVEPOINT_MONODROMY = 13
SEED_CYCLIC_MONODROMY = 17
SEED_P3P_INSTANCE = 7_000_000
SEED_P3P_P0 = 31


def fivepoint_project(x: np.ndarray, gam: np.ndarray) -> np.ndarray:
    """Second-view coordinates that make x an exact solution, given the first view gam [5, 2]:
    W = rho_i R(q) gamma_i + T, rhob_i = W_z, gammab_i = W / W_z.  Returns (p [20], x with rhob set)."""
    x = np.array(x, dtype=np.result_type(x, gam, np.complex128))
    R = np.array(systems.quat_rot(*x[10:14]))
    T = np.array([x[14], x[15], 1.0])
    p = np.zeros(20, dtype=x.dtype)
    for i in range(5):
        g = np.array([gam[i, 0], gam[i, 1], 1.0])
        W = x[i] * (R @ g) + T
        x[5 + i] = W[2]
        p[systems.fivepoint_param_index(0, i, 0)] = gam[i, 0]
        p[systems.fivepoint_param_index(0, i, 1)] = gam[i, 1]
        p[systems.fivepoint_param_index(1, i, 0)] = W[0] / W[2]
        p[systems.fivepoint_param_index(1, i, 1)] = W[1] / W[2]
    return p, x


def fivepoint_instance(seed: int):
    """Planted real 5-point instance: rotation 0.1-0.5 rad, T = (tx, ty, 1) with tx, ty ~ N(0, 0.5),
    five points at depth 3-6 in front of both cameras, normalised image coordinates |u|, |v| <= 0.4.
    Returns (p [20] complex, x_gt [16] complex)."""
    g = gen(seed)
    while True:
        _, q = random_rotation(g)
        t = g.normal(0, 0.5, 2)
        rho = g.uniform(3, 6, 5)
        gam = g.uniform(-0.4, 0.4, (5, 2))
        x = np.concatenate([rho, np.zeros(5), q, t]).astype(np.complex128)
        p, x = fivepoint_project(x, gam.astype(np.complex128))
        if np.all(x[5:10].real > 1.0):
            return p, x


def fivepoint_batch(n_instances: int, base: int = SEED_FIVEPOINT_INSTANCE):
    ps, xs = zip(*(fivepoint_instance(base + b) for b in range(n_instances)))
    return np.stack(ps), np.stack(xs)


def family_start(d, seed: int):
    """Planted generic complex (p0, x0) of a coefficient family (systems.coefficient_family): x0 and
    p complex Gaussian, then the first term's parameter of every equation is set so that x0 solves
    it (each equation is linear in its parameters)."""
    n = d.n_vars
    g = gen(seed)
    x0 = complex_normal(g, n)
    p = complex_normal(g, d.n_params)
    mono = np.prod(x0[None, :] ** d.term_xexp, axis=1)          # term q's monomial at x0
    coef_param = [int(np.nonzero(d.coef_pexp[d.coef_ptr[c]])[0][0]) for c in d.term_coef]
    for i in range(n):
        qs = [q for q in range(d.n_terms) if d.term_eq[q] == i]
        rest = sum(p[coef_param[q]] * mono[q] for q in qs[1:])
        p[coef_param[qs[0]]] = -rest / mono[qs[0]]
    return p, x0


def cyclic_family_start(n: int = 7, seed: int = SEED_CYCLIC_MONODROMY):
    from .systems import cyclic_family
    return family_start(cyclic_family(n), seed)


def fivepoint_complex_start(seed: int = SEED_FIVEPOINT_MONODROMY):
    """Planted generic complex (x0, p0) for monodromy: complex depths, T, first-view points and q
    normalised by the complex square root of q.q; the second view from the closed form."""
    g = gen(seed)
    x = complex_normal(g, 16)
    x[10:14] /= np.sqrt(np.sum(x[10:14] ** 2))
    gam = complex_normal(g, (5, 2))
    p, x = fivepoint_project(x, gam)
    return p, x


def p3p_instance(seed: int):
    """Planted real P3P instance: camera [I | 0]; world points Gamma_i = rho_i gamma_i with
    depths rho_i ~ U[3, 6] and calibrated image points |u|, |v| <= 0.4, then moved to a world frame
    by a random rotation (0.1-0.5 rad) and translation N(0, 1) (the equations only see distances
    and dot products of the Gamma differences, so the frame does not matter).
    Returns (p [15] complex, x_gt [3] complex = the depths)."""
    from .systems import p3p_param_index
    g = gen(seed)
    rho = g.uniform(3, 6, 3)
    uv = g.uniform(-0.4, 0.4, (3, 2))
    Rw, _ = random_rotation(g)
    tw = g.normal(0, 1, 3)
    p = np.zeros(15, np.complex128)
    for i in range(3):
        gam = np.array([uv[i, 0], uv[i, 1], 1.0])
        Gam = Rw @ (rho[i] * gam) + tw
        p[p3p_param_index(0, i, 0)], p[p3p_param_index(0, i, 1)] = uv[i]
        for c in range(3):
            p[p3p_param_index(1, i, c)] = Gam[c]
    return p, rho.astype(np.complex128)


def p3p_batch(n_instances: int, base: int = SEED_P3P_INSTANCE):
    P, X = zip(*(p3p_instance(base + b) for b in range(n_instances)))
    return np.stack(P), np.stack(X)


def p3p_p0(seed: int = SEED_P3P_P0) -> np.ndarray:
    """Generic complex start parameters for the P3P parameter homotopy."""
    return complex_normal(gen(seed), 15)

