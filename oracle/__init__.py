"""CPU oracle for batched HC path tracking (ctypes binding of oracle/hc_oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product path
(paper_2112_03444_b200/) never imports it, and it never imports the product.

Every function follows PAPER.md §3 (Eq. 1-6) and the SURVEY.md §8(c) readings
R1-R13; see hc_oracle.c for per-function citations.  Pins live in
tests/test_oracle_*.py.  "parity unpinned" items are listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, fields

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# ORACLE_SO: a prebuilt variant (e.g. the ASan/UBSan build of scripts/sanitize_host.sh)
_SO = os.environ.get("ORACLE_SO") or os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "hc_oracle.c"), os.path.join(_HERE, "hc_oracle.h")]

CONVERGED, DIVERGED, STEP_UNDERFLOW, MAX_STEPS, SINGULAR, NONFINITE, AT_INFINITY = range(7)
STATUS_NAMES = ["CONVERGED", "DIVERGED", "STEP_UNDERFLOW", "MAX_STEPS", "SINGULAR", "NONFINITE", "AT_INFINITY"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (plain C99, -O2, no fast-math, no FMA contraction)."""
    if os.environ.get("ORACLE_SO"):
        return _SO
    stale = force or not os.path.exists(_SO) or any(os.path.getmtime(s) > os.path.getmtime(_SO) for s in _SRC)
    if stale:
        cmd = ["gcc", "-std=gnu99", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
               "-Wall", "-Wno-maybe-uninitialized", "-o", _SO, _SRC[0], "-lm", "-lpthread"]
        subprocess.run(cmd, check=True)
    return _SO


class _Sys(C.Structure):
    _fields_ = [("n", C.c_int32), ("P", C.c_int32), ("nterms", C.c_int32), ("ncoef", C.c_int32),
                ("term_eq", C.c_void_p), ("term_xexp", C.c_void_p), ("term_coef", C.c_void_p),
                ("coef_ptr", C.c_void_p), ("coef_w", C.c_void_p), ("coef_pexp", C.c_void_p)]


class _Hom(C.Structure):
    _fields_ = [("kind", C.c_int32), ("sys", C.c_void_p), ("deg", C.c_void_p),
                ("gamma", C.c_double * 2), ("p0", C.c_void_p), ("p1", C.c_void_p)]


class _Settings(C.Structure):
    _fields_ = [("predictor", C.c_int32), ("dt_init", C.c_double), ("dt_min", C.c_double),
                ("dt_max", C.c_double), ("grow_after", C.c_int32), ("grow", C.c_double),
                ("shrink", C.c_double), ("max_newton", C.c_int32), ("newton_tol", C.c_double),
                ("max_steps", C.c_int32), ("inf_norm", C.c_double), ("end_newton", C.c_int32),
                ("end_tol", C.c_double), ("res_abs", C.c_double), ("res_rel", C.c_double),
                ("pivot_rel", C.c_double), ("eg_start", C.c_double), ("eg_inf_mu", C.c_double),
                ("eg_sing_mu", C.c_double), ("eg_stab", C.c_double), ("eg_inf_s", C.c_double), ("eg_inf_norm", C.c_double), ("eg_samples", C.c_int32), ("eg_max_winding", C.c_int32),
                ("eg_max_radii", C.c_int32), ("eg_tol", C.c_double)]


@dataclass
class Settings:
    """Tracker settings.  Defaults come from orc_settings_default."""
    predictor: int = 0
    dt_init: float = 0.01
    dt_min: float = 1e-14
    dt_max: float = 0.1
    grow_after: int = 4
    grow: float = 2.0
    shrink: float = 0.5
    max_newton: int = 3
    newton_tol: float = 1e-8
    max_steps: int = 10000
    inf_norm: float = 1e14
    end_newton: int = 3
    end_tol: float = 1e-12
    res_abs: float = 1e-10
    res_rel: float = 1e-12
    pivot_rel: float = 1e-14
    eg_start: float = 0.1          # endgame (reading R26); 0 disables it
    eg_inf_mu: float = -0.05
    eg_sing_mu: float = 0.75
    eg_stab: float = 0.02
    eg_inf_s: float = 1e-12
    eg_inf_norm: float = 1e5
    eg_samples: int = 16
    eg_max_winding: int = 8
    eg_max_radii: int = 12
    eg_tol: float = 1e-10

    def _c(self) -> _Settings:
        s = _Settings()
        for f in fields(self):
            setattr(s, f.name, getattr(self, f.name))
        return s


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = C.CDLL(_SO)
        L.orc_settings_default.argtypes = [C.POINTER(_Settings)]
        L.orc_eval_coefs.argtypes = [C.POINTER(_Sys), C.c_void_p, C.c_void_p]
        L.orc_eval_F.argtypes = [C.POINTER(_Sys), C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_eval_JF.argtypes = [C.POINTER(_Sys), C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_eval_H.argtypes = [C.POINTER(_Hom), C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        L.orc_lu_solve.argtypes = [C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_double]
        L.orc_lu_solve.restype = C.c_int
        L.orc_td_start.argtypes = [C.c_int, C.c_void_p, C.c_void_p]
        L.orc_td_start.restype = C.c_int64
        L.orc_track.argtypes = [C.POINTER(_Hom), C.c_void_p, C.c_int64, C.c_void_p, C.c_int64,
                                C.POINTER(_Settings), C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                C.c_void_p]
        L.orc_predict.argtypes = [C.POINTER(_Hom), C.POINTER(_Settings), C.c_void_p, C.c_double, C.c_double,
                                  C.c_void_p]
        L.orc_predict.restype = C.c_int
        L.orc_newton.argtypes = [C.POINTER(_Hom), C.POINTER(_Settings), C.c_void_p, C.c_double, C.c_int,
                                 C.c_double]
        L.orc_newton.restype = C.c_int
        L.orc_endpoint_residual.argtypes = [C.POINTER(_Hom), C.c_void_p, C.c_void_p, C.c_void_p]
        _lib = L
    return _lib


def default_settings() -> Settings:
    s = _Settings()
    lib().orc_settings_default(C.byref(s))
    return Settings(**{f.name: getattr(s, f.name) for f in fields(Settings)})


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class _SysHold:
    """Keeps the numpy arrays behind an orc_sys alive."""

    def __init__(self, desc):
        self.desc = desc.contiguous()
        d = self.desc
        self.s = _Sys(d.n_vars, d.n_params, d.n_terms, d.n_coefs, _ptr(d.term_eq), _ptr(d.term_xexp),
                      _ptr(d.term_coef), _ptr(d.coef_ptr), _ptr(d.coef_w), _ptr(d.coef_pexp))


def _c128(a, shape=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.complex128))
    return a if shape is None else a.reshape(shape)


class Homotopy:
    """H(x,t): total degree (TD, Eq. 1 + gamma) or parameter homotopy (PH, R3)."""

    def __init__(self, desc, kind: str, gamma: complex = 1.0, p0=None, p1=None):
        self._sys = _SysHold(desc)
        self.n = desc.n_vars
        self.kind = kind
        self.deg = np.ascontiguousarray(np.array(desc.degrees(), dtype=np.int32))
        self.p0 = _c128(p0) if p0 is not None else None
        self.p1 = _c128(p1) if p1 is not None else None
        self.h = _Hom()
        self.h.kind = 0 if kind == "td" else 1
        self.h.sys = C.cast(C.pointer(self._sys.s), C.c_void_p)
        self.h.deg = _ptr(self.deg)
        self.h.gamma[0], self.h.gamma[1] = complex(gamma).real, complex(gamma).imag
        self.h.p0 = _ptr(self.p0) if self.p0 is not None else None
        self.h.p1 = _ptr(self.p1) if self.p1 is not None else None

    def eval(self, x, t: float):
        """(H [n], ∂H/∂x [n, n], ∂H/∂t [n]) at (x, t)."""
        x = _c128(x)
        n = self.n
        H = np.zeros(n, np.complex128)
        Hx = np.zeros((n, n), np.complex128)
        Ht = np.zeros(n, np.complex128)
        lib().orc_eval_H(C.byref(self.h), _ptr(x), float(t), _ptr(H), _ptr(Hx), _ptr(Ht))
        return H, Hx, Ht


def predict(hom: "Homotopy", x, t: float, dt: float, settings: "Settings | None" = None):
    """One predictor step (RK4 P:175 / Euler Eq. 4).  Returns (x*, failed)."""
    st = (settings or default_settings())._c()
    x = _c128(x)
    xp = np.zeros_like(x)
    r = lib().orc_predict(C.byref(hom.h), C.byref(st), _ptr(x), float(t), float(dt), _ptr(xp))
    return xp, bool(r)


def newton(hom: "Homotopy", x, t: float, iters: int, tol: float, settings: "Settings | None" = None):
    """Newton at fixed t (Eq. 6).  Returns (x, code) with code 1 converged, 0 not, -1 singular."""
    st = (settings or default_settings())._c()
    x = _c128(x).copy()
    r = lib().orc_newton(C.byref(hom.h), C.byref(st), _ptr(x), float(t), int(iters), float(tol))
    return x, r


def endpoint_residual(hom: "Homotopy", x):
    """Reading R10 at t = 1: (r = ||F||_inf, r_rel = max_i |F_i| / sum_k |c_ik| |m_k(x)|)."""
    x = _c128(x)
    r, rr = C.c_double(), C.c_double()
    lib().orc_endpoint_residual(C.byref(hom.h), _ptr(x), C.byref(r), C.byref(rr))
    return r.value, rr.value


def td_homotopy(desc, gamma: complex) -> Homotopy:
    return Homotopy(desc, "td", gamma=gamma)


def ph_homotopy(desc, p0, p1=None) -> Homotopy:
    return Homotopy(desc, "ph", p0=p0, p1=p1 if p1 is not None else p0)


def eval_coefs(desc, p) -> np.ndarray:
    h = _SysHold(desc)
    p = _c128(p)
    c = np.zeros(desc.n_coefs, np.complex128)
    lib().orc_eval_coefs(C.byref(h.s), _ptr(p), _ptr(c))
    return c


def eval_F(desc, p, x) -> np.ndarray:
    h = _SysHold(desc)
    p, x = _c128(p), _c128(x)
    F = np.zeros(desc.n_vars, np.complex128)
    lib().orc_eval_F(C.byref(h.s), _ptr(p), _ptr(x), _ptr(F))
    return F


def eval_JF(desc, p, x) -> np.ndarray:
    h = _SysHold(desc)
    p, x = _c128(p), _c128(x)
    J = np.zeros((desc.n_vars, desc.n_vars), np.complex128)
    lib().orc_eval_JF(C.byref(h.s), _ptr(p), _ptr(x), _ptr(J))
    return J


def lu_solve(A, b, pivot_rel: float = 1e-14):
    """Returns (x, singular)."""
    A, b = _c128(A), _c128(b)
    n = b.shape[0]
    x = np.zeros(n, np.complex128)
    r = lib().orc_lu_solve(n, _ptr(A), _ptr(b), _ptr(x), pivot_rel)
    return x, bool(r)


def td_start(degrees) -> np.ndarray:
    deg = np.ascontiguousarray(np.array(degrees, dtype=np.int32))
    total = lib().orc_td_start(len(deg), _ptr(deg), None)
    x = np.zeros((total, len(deg)), np.complex128)
    lib().orc_td_start(len(deg), _ptr(deg), _ptr(x))
    return x


@dataclass
class TrackResult:
    x: np.ndarray         # [B, S, n] complex128
    status: np.ndarray    # [B, S] int32
    counters: np.ndarray  # [B, S, 4] int32: steps, rejections, newton iterations, linear solves
    resid: np.ndarray     # [B, S, 2] float64: ||F||_inf, relative (backward-error) residual
    winding: np.ndarray   # [B, S] int32: Cauchy endgame winding number (0: not used)


def nthreads_default() -> int:
    return int(os.environ.get("HC_THREADS", os.cpu_count() or 1))


def track(hom: Homotopy, start_x, p1s=None, settings: Settings | None = None, nthreads: int | None = None) -> TrackResult:
    """Track every start point through H for each instance (PH: rows of p1s; TD: one instance)."""
    st = (settings or default_settings())._c()
    start_x = _c128(start_x)
    S, n = start_x.shape
    if hom.kind == "ph":
        p1s = _c128(p1s if p1s is not None else hom.p1[None, :])
        p1s = p1s.reshape(-1, hom.p0.shape[0])
        B = p1s.shape[0]
    else:
        B = 1
    x = np.zeros((B, S, n), np.complex128)
    status = np.zeros((B, S), np.int32)
    ctr = np.zeros((B, S, 4), np.int32)
    resid = np.zeros((B, S, 2), np.float64)
    wind = np.zeros((B, S), np.int32)
    lib().orc_track(C.byref(hom.h), _ptr(p1s) if hom.kind == "ph" else None, B, _ptr(start_x), S, C.byref(st),
                    int(nthreads or nthreads_default()), _ptr(x), _ptr(status), _ptr(ctr), _ptr(resid), _ptr(wind))
    return TrackResult(x, status, ctr, resid, wind)


# ---------------------------------------------------------------------------------------
# Host post-processing (reading R11 dedup, R12 real classification, R21 matching)
# ---------------------------------------------------------------------------------------

def finite_solutions(res: TrackResult, b: int = 0) -> np.ndarray:
    """Endpoints with status CONVERGED for instance b, in track order."""
    return res.x[b][res.status[b] == CONVERGED]


def dedup(X: np.ndarray, tol: float = 1e-6):
    """Greedy dedup in track order (R11): y merges into an earlier kept x when
    |x_i - y_i| <= tol * max(1, |x_i|) for all i.  Returns (unique [U, n], multiplicity [U])."""
    keep, mult = [], []
    for y in X:
        for u, x in enumerate(keep):
            if np.all(np.abs(x - y) <= tol * np.maximum(1.0, np.abs(x))):
                mult[u] += 1
                break
        else:
            keep.append(y)
            mult.append(1)
    n = X.shape[1] if X.ndim == 2 else 0
    return (np.array(keep).reshape(-1, n), np.array(mult, dtype=np.int64))


def is_real(X: np.ndarray, tol: float = 1e-6) -> np.ndarray:
    """R12: max_i |Im x_i| <= tol * max(1, |x_i|)."""
    return np.all(np.abs(X.imag) <= tol * np.maximum(1.0, np.abs(X)), axis=1)


def match_sets(A: np.ndarray, B: np.ndarray, tol: float = 1e-8):
    """R21: |A| == |B| and every a has a b with |a_i - b_i| <= tol max(1, |a_i|) for all i, and vice
    versa.  Returns (ok, n_unmatched_A, n_unmatched_B)."""
    def unmatched(P, Q):
        cnt = 0
        for a in P:
            if Q.shape[0] == 0 or not np.any(np.all(np.abs(Q - a) <= tol * np.maximum(1.0, np.abs(a)), axis=1)):
                cnt += 1
        return cnt
    ua, ub = unmatched(A, B), unmatched(B, A)
    return (A.shape[0] == B.shape[0] and ua == 0 and ub == 0), ua, ub
