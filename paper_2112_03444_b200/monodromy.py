"""Monodromy solver on the GPU tracker ("start systems ... generated with
monodromy").

From one known solution x0 of F(x; p0) = 0, repeatedly track every known solution around a loop of
parameter homotopies p0 -> p1 -> p2 -> p0 with random complex p1, p2 (each segment a batched
hc_track_batch call on the fused kernel); endpoints back at p0 that are new are added.  Stops when
`stall_loops` consecutive loops add nothing (or `target` solutions are known).  An optional
`symmetry(x) -> list of solutions` (a group action that commutes with the homotopy, e.g.
hc_inputs.systems.trifocal_symmetry) lets only one representative per orbit be tracked.

Host orchestration only: every path is tracked by libhc.so; deduplication (reading R11) is host
post-processing.
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


def _contains(S: np.ndarray, y: np.ndarray, tol: float) -> bool:
    if S.shape[0] == 0:
        return False
    return bool(np.any(np.all(np.abs(S - y) <= tol * np.maximum(1.0, np.abs(y)), axis=1)))


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
        for y in X:
            if not _contains(known, y, tol):
                reps.append(y)
                known = np.concatenate([known, np.array(orbit(y), dtype=np.complex128)])
                new += 1
        hist.append(int(known.shape[0]))
        stall = stall + 1 if new == 0 else 0
        if stall >= stall_loops or (target is not None and known.shape[0] >= target):
            break
    return MonodromyResult(known, np.array(reps), loop + 1, tracks, hist)
