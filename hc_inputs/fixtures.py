"""Fixture file I/O (SPEC.md S:100 solution format; start-parameter files).

Solution file: line 1 `<numVars> <numSols>`, then per solution numVars lines `<re> <im>`.
Parameter file: line 1 `<numParams>`, then numParams lines `<re> <im>`.
Values are written with repr() (17 significant digits), so files round-trip exactly.
"""
from __future__ import annotations

import os

import numpy as np

FIXTURE_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "fixtures")


def write_solutions(path: str, X: np.ndarray, header_comment: str = "") -> None:
    X = np.asarray(X, dtype=np.complex128)
    S, n = X.shape
    with open(path, "w") as fh:
        if header_comment:
            for line in header_comment.splitlines():
                fh.write(f"# {line}\n")
        fh.write(f"{n} {S}\n")
        for s in range(S):
            for v in range(n):
                fh.write(f"{float(X[s, v].real)!r} {float(X[s, v].imag)!r}\n")


def read_solutions(path: str) -> np.ndarray:
    vals = []
    with open(path) as fh:
        lines = [ln.split("#", 1)[0].strip() for ln in fh]
    lines = [ln for ln in lines if ln]
    n, S = (int(a) for a in lines[0].split())
    for ln in lines[1:1 + n * S]:
        re, im = ln.split()
        vals.append(complex(float(re), float(im)))
    return np.array(vals, dtype=np.complex128).reshape(S, n)


def write_params(path: str, p: np.ndarray, header_comment: str = "") -> None:
    p = np.asarray(p, dtype=np.complex128).reshape(-1)
    with open(path, "w") as fh:
        if header_comment:
            for line in header_comment.splitlines():
                fh.write(f"# {line}\n")
        fh.write(f"{p.shape[0]}\n")
        for z in p:
            fh.write(f"{float(z.real)!r} {float(z.imag)!r}\n")


def read_params(path: str) -> np.ndarray:
    with open(path) as fh:
        lines = [ln.split("#", 1)[0].strip() for ln in fh]
    lines = [ln for ln in lines if ln]
    P = int(lines[0])
    out = []
    for ln in lines[1:1 + P]:
        re, im = ln.split()
        out.append(complex(float(re), float(im)))
    return np.array(out, dtype=np.complex128)


def fixture_path(name: str) -> str:
    return os.path.join(FIXTURE_DIR, name)


def have_fixture(name: str) -> bool:
    return os.path.exists(fixture_path(name))


def trifocal_start():
    """(start solutions [S, 18], p0 [24]) of the trifocal fixture: the orbit representatives written by
    scripts/make_fixtures.py expanded by the Z2^3 symmetry in the same order the script used."""
    from . import systems
    reps = read_solutions(fixture_path("trifocal_reps.sols"))
    full = np.concatenate([np.array(systems.trifocal_symmetry(r)) for r in reps])
    return full, read_params(fixture_path("trifocal_p0.params"))
