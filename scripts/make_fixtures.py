"""Generate start-solution fixtures with the CPU oracle ONLY (tests/golden-style provenance).

  python scripts/make_fixtures.py fourview   # 4-view TD solve at generic complex p0 -> 296 starts
  python scripts/make_fixtures.py trifocal   # trifocal monodromy from a planted (x0, p0)
  python scripts/make_fixtures.py fivepoint  # 5-point relpose + depth monodromy (reading R24)
  python scripts/make_fixtures.py eco12      # eco-12 TD solve (118,098 tracks) -> the oracle's finite set
  python scripts/make_fixtures.py cyclic7    # cyclic-7 coefficient-family monodromy (Table 1: 924)
  python scripts/make_fixtures.py p3p        # P3P depth form: TD at a generic p0 -> 8 starts (Table 2)

This script imports only `oracle` and `hc_inputs`; the CUDA path never writes fixtures
(prompt rule ③: no stored value comes from the CUDA path).  Start systems of the paper's
vision problems come from monodromy; for 4-view the total-degree solve is small
enough (2^14 = 16384 tracks) to do directly.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from hc_inputs import fixtures, rng, systems  # noqa: E402
from hc_inputs.descriptor import SystemDesc  # noqa: E402

FOURVIEW_TD_GAMMA_SEED = 0


def constant_system_at(desc, p):
    """The system F(x; p) with its coefficient expressions frozen at p (a TD target)."""
    c = oracle.eval_coefs(desc, p)
    return SystemDesc(desc.n_vars, 0, desc.term_eq, desc.term_xexp, desc.term_coef,
                      np.arange(desc.n_coefs + 1, dtype=np.int32), c,
                      np.zeros((desc.n_coefs, 0), np.int32), name=desc.name + "@p0").contiguous()


def make_fourview():
    d = systems.nview_triangulation(4)
    p0 = rng.fourview_p0()
    td = constant_system_at(d, p0)
    t0 = time.time()
    res = oracle.track(oracle.td_homotopy(td, rng.gamma(FOURVIEW_TD_GAMMA_SEED)), oracle.td_start(td.degrees()))
    U, mult = oracle.dedup(oracle.finite_solutions(res))
    print(f"4-view TD: {len(U)} distinct finite of {res.status.size} tracks, max mult {mult.max()}, "
          f"{time.time() - t0:.1f} s", flush=True)
    hdr = (f"4-view triangulation start solutions at p0 = rng.fourview_p0() (seed {rng.SEED_FOURVIEW_P0}).\n"
           f"Written by scripts/make_fixtures.py (oracle only): TD homotopy, gamma seed {FOURVIEW_TD_GAMMA_SEED},\n"
           f"{res.status.size} tracks -> {len(U)} distinct finite solutions (PAPER.md Table 2 P:490: 296).")
    fixtures.write_solutions(fixtures.fixture_path("fourview_start.sols"), U, hdr)
    fixtures.write_params(fixtures.fixture_path("fourview_p0.params"), p0, hdr)


def _orbit(x):
    return systems.trifocal_symmetry(x)


def _contains(S, y, tol=1e-6):
    if S.shape[0] == 0:
        return False
    return bool(np.any(np.all(np.abs(S - y) <= tol * np.maximum(1.0, np.abs(y)), axis=1)))


def _monodromy(d, p0, x0, orbit, seed, max_loops, stall_loops, label):
    """Monodromy ("monodromy module", SURVEY.md [X6]) with a solution symmetry `orbit`:
    only one representative per orbit is tracked; endpoints are expanded by the group."""
    reps = [x0]
    full = np.array(orbit(x0))
    g = rng.gen(seed + 1)
    stall = 0
    t0 = time.time()
    loop = 0
    for loop in range(max_loops):
        p1 = rng.complex_normal(g, d.n_params)
        p2 = rng.complex_normal(g, d.n_params)
        X = np.array(reps)
        alive = np.arange(len(reps))
        for pa, pb in ((p0, p1), (p1, p2), (p2, p0)):
            res = oracle.track(oracle.ph_homotopy(d, pa, pb), X)
            ok = res.status[0] == oracle.CONVERGED
            X = res.x[0][ok]
            alive = alive[ok]
        new = 0
        for y in X:
            if not _contains(full, y):
                reps.append(y)
                full = np.concatenate([full, np.array(orbit(y))])
                new += 1
        stall = stall + 1 if new == 0 else 0
        print(f"{label} loop {loop}: tracked {len(alive)}/{len(reps) - new} survived, +{new} orbits -> "
              f"{len(reps)} orbits = {full.shape[0]} solutions ({time.time() - t0:.0f} s)", flush=True)
        if stall >= stall_loops:
            break
    return reps, full, loop + 1


def make_trifocal(max_loops: int = 60, stall_loops: int = 4, seed: int = rng.SEED_TRIFOCAL_MONODROMY):
    """Trifocal monodromy with the Z2^3 symmetry of R20."""
    d = systems.trifocal_unknown_f()
    p0, x0 = rng.trifocal_complex_start(seed)
    reps, full, loops = _monodromy(d, p0, x0, _orbit, seed, max_loops, stall_loops, "trifocal")
    hdr = (f"trifocal unknown-f start solutions at the planted complex p0 = rng.trifocal_complex_start({seed}).\n"
           f"Written by scripts/make_fixtures.py (oracle only): symmetry-aware monodromy, {loops} loops,\n"
           f"{len(reps)} orbits x 8 = {full.shape[0]} solutions (PAPER.md Table 2 P:488 reports 1784).")
    # the full start set is trifocal_reps.sols expanded by the symmetry (hc_inputs.fixtures.trifocal_start)
    fixtures.write_solutions(fixtures.fixture_path("trifocal_reps.sols"), np.array(reps), hdr)
    fixtures.write_params(fixtures.fixture_path("trifocal_p0.params"), p0, hdr)


def make_fivepoint(max_loops: int = 40, stall_loops: int = 5, seed: int = rng.SEED_FIVEPOINT_MONODROMY):
    """5-point relative pose + depth (reading R24) monodromy with the q -> -q symmetry."""
    d = systems.fivepoint_relpose_depth()
    p0, x0 = rng.fivepoint_complex_start(seed)
    reps, full, loops = _monodromy(d, p0, x0, systems.fivepoint_symmetry, seed, max_loops, stall_loops, "5pt")
    hdr = (f"5-point relative pose + depth start solutions at the planted complex p0 = rng.fivepoint_complex_start({seed}).\n"
           f"Written by scripts/make_fixtures.py (oracle only): symmetry-aware monodromy, {loops} loops,\n"
           f"{len(reps)} orbits x 2 = {full.shape[0]} solutions (PAPER.md Table 2 P:492 reports 160; reading R24).")
    fixtures.write_solutions(fixtures.fixture_path("fivepoint_start.sols"), full, hdr)
    fixtures.write_params(fixtures.fixture_path("fivepoint_p0.params"), p0, hdr)


ECO12_GAMMA_SEED = 2
P3P_TD_GAMMA_SEED = 3


def make_eco12():
    """The oracle's finite solution set of eco-12 (Table 1: 1024 solutions, reading R25),
    the expected set of tests/test_gpu_parity.py::test_eco12_table1_count (the oracle needs
    minutes for the 118,098 total-degree tracks, so the set is stored)."""
    d = systems.eco(12)
    t0 = time.time()
    res = oracle.track(oracle.td_homotopy(d, rng.gamma(ECO12_GAMMA_SEED)), oracle.td_start(d.degrees()))
    U, mult = oracle.dedup(oracle.finite_solutions(res))
    st = np.bincount(res.status.reshape(-1), minlength=6)
    print(f"eco-12 TD: {len(U)} distinct finite of {res.status.size} tracks (statuses {st.tolist()}), "
          f"max mult {mult.max()}, {time.time() - t0:.1f} s", flush=True)
    hdr = (f"eco-12 finite solutions (PAPER.md Table 1 P:469: 1024), reading R25 (standard eco-n).\n"
           f"Written by scripts/make_fixtures.py (oracle only): TD homotopy, gamma seed {ECO12_GAMMA_SEED},\n"
           f"{res.status.size} tracks -> {len(U)} distinct finite solutions; statuses {st.tolist()}.")
    fixtures.write_solutions(fixtures.fixture_path("eco12_solutions.sols"), U, hdr)


def make_p3p():
    """P3P depth form (Eq. P3PafterElim): total-degree solve (2^3 = 8 tracks) at the
    generic complex p0 = rng.p3p_p0() -> the 8 start solutions (Table 2: 8)."""
    d = systems.p3p_depth()
    p0 = rng.p3p_p0()
    td = constant_system_at(d, p0)
    res = oracle.track(oracle.td_homotopy(td, rng.gamma(P3P_TD_GAMMA_SEED)), oracle.td_start(td.degrees()))
    U, mult = oracle.dedup(oracle.finite_solutions(res))
    print(f"P3P TD at p0: {len(U)} distinct finite of {res.status.size} tracks", flush=True)
    hdr = (f"P3P depth-form start solutions at p0 = rng.p3p_p0() (seed {rng.SEED_P3P_P0}).\n"
           f"Written by scripts/make_fixtures.py (oracle only): TD homotopy, gamma seed {P3P_TD_GAMMA_SEED},\n"
           f"{res.status.size} tracks -> {len(U)} distinct finite solutions (PAPER.md Table 2 P:512: 8).")
    fixtures.write_solutions(fixtures.fixture_path("p3p_start.sols"), U, hdr)
    fixtures.write_params(fixtures.fixture_path("p3p_p0.params"), p0, hdr)


def make_cyclic7(max_loops: int = 60, stall_loops: int = 4, seed: int = rng.SEED_CYCLIC_MONODROMY):
    """Monodromy start set of the cyclic-7 coefficient family (systems.cyclic_family) at a planted
    generic complex p0: the paper's start-system workflow (monodromy) for its Table 1
    benchmark (cyclic-7: 924 solutions)."""
    d = systems.cyclic_family(7)
    p0, x0 = rng.cyclic_family_start(7, seed)
    reps, full, loops = _monodromy(d, p0, x0, lambda x: [x], seed, max_loops, stall_loops, "cyclic7")
    hdr = (f"cyclic-7 coefficient family start solutions at the planted complex p0 = rng.cyclic_family_start(7, {seed}).\n"
           f"Written by scripts/make_fixtures.py (oracle only): monodromy, {loops} loops,\n"
           f"{full.shape[0]} solutions (PAPER.md Table 1 P:467: cyclic-7 has 924).")
    fixtures.write_solutions(fixtures.fixture_path("cyclic7_start.sols"), full, hdr)
    fixtures.write_params(fixtures.fixture_path("cyclic7_p0.params"), p0, hdr)


if __name__ == "__main__":
    oracle.build()
    what = sys.argv[1:] or ["fourview", "trifocal", "fivepoint"]
    if "fourview" in what:
        make_fourview()
    if "trifocal" in what:
        make_trifocal()
    if "fivepoint" in what:
        make_fivepoint()
    if "eco12" in what:
        make_eco12()
    if "cyclic7" in what:
        make_cyclic7()
    if "p3p" in what:
        make_p3p()
