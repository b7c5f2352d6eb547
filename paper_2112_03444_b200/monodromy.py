"""Monodromy solver on the GPU tracker ("start systems ... generated with
monodromy").

From one known solution x0 of F(x; p0) = 0, repeatedly track every known solution around a loop of
parameter homotopies p0 -> p1 -> p2 -> p0 with random complex p1, p2 (each segment a batched
hc_track_batch call on the fused kernel); endpoints back at p0 that are new are added.  Stops when
`stall_loops` consecutive loops add nothing (or `target` solutions are known).  An optional
`symmetry(x) -> list of solutions` (a group action that commutes with the homotopy, e.g.
hc_inputs.systems.trifocal_symmetry) lets only one representative per orbit be tracked.

Host orchestration only: every path is tracked by libhc.so; deduplication (reading R11) is the
library's host post-processing (hc_solutions: greedy matching in order against the known points).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import hc


@dataclass
class MonodromyResult:
    solutions: np.ndarray                 # [n, N] complex128 at p0 (orbits expanded)
    representatives: np.ndarray           # [m, N] tracked representatives
    loops: int
    tracks: int                           # paths tracked in total
    history: list = field(default_factory=list)   # known count after each loop


def _new_points(known: np.ndarray, X: np.ndarray, tol: float) -> list:
    """Indices of the rows of X that match neither a known point nor an earlier row of X (reading
    R11, through hc_solutions on [known; X]: a row is new when it is kept as its own representative)."""
    if X.shape[0] == 0:
        return []
    n = known.shape[0]
    _, _, _, rep = hc.solutions(np.concatenate([known, X]) if n else X, None, tol=tol)
    return [i for i in range(X.shape[0]) if rep[n + i] == n + i]


def monodromy_solve(system: "hc.System", x0, p0, *, symmetry=None, max_loops: int = 60, stall_loops: int = 4,
                    target: int | None = None, seed: int = 0, settings=None, tol: float = 1e-6,
                    param_scale: float = 1.0) -> MonodromyResult:
    """Monodromy from (x0, p0); `system` must be a parameter-homotopy hc.System (P > 0)."""
    import torch
    P = system.P
    assert P > 0, "monodromy needs a parametrised system"
    x0 = np.asarray(x0, dtype=np.complex128).reshape(1, -1)
    p0 = np.asarray(p0, dtype=np.complex128).reshape(P)
    g = np.random.Generator(np.random.PCG64(seed))
    orbit = (lambda y: [y]) if symmetry is None else symmetry
    reps = [x0[0]]
    known = np.array(orbit(x0[0]), dtype=np.complex128)
    dev = torch.device("cuda", system.device)
    st = settings or hc.hc_tracker_settings_default()
    stall, tracks, hist = 0, 0, []
    loop = 0
    for loop in range(max_loops):
        p1 = (g.standard_normal(P) + 1j * g.standard_normal(P)) * (param_scale / np.sqrt(2))
        p2 = (g.standard_normal(P) + 1j * g.standard_normal(P)) * (param_scale / np.sqrt(2))
        X = np.array(reps)
        for pa, pb in ((p0, p1), (p1, p2), (p2, p0)):
            if X.shape[0] == 0:
                break
            res = hc.track_batch(system, torch.from_numpy(X).to(dev), torch.from_numpy(pa).to(dev),
                                 torch.from_numpy(pb[None]).to(dev), st=st)
            res.wait()
            tracks += X.shape[0]
            ok = res.status.cpu().numpy()[0] == hc.HC_CONVERGED
            X = res.x.cpu().numpy()[0][ok]
            res.close()
        new = 0
        added = np.zeros((0, known.shape[1]), dtype=np.complex128)   # orbits added in this loop
        for i in _new_points(known, X, tol):
            y = X[i]
            if added.shape[0] and not _new_points(added, y[None], tol):
                continue   # in the orbit of a point added earlier in this loop
            reps.append(y)
            orb = np.array(orbit(y), dtype=np.complex128)
            known = np.concatenate([known, orb])
            added = np.concatenate([added, orb])
            new += 1
        hist.append(int(known.shape[0]))
        stall = stall + 1 if new == 0 else 0
        if stall >= stall_loops or (target is not None and known.shape[0] >= target):
            break
    return MonodromyResult(known, np.array(reps), loop + 1, tracks, hist)
