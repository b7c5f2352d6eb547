"""Certify the trifocal start set (fixtures/trifocal_reps.sols: 668 orbits x 8 = 5344 solutions at
p0 = rng.trifocal_complex_start(101)) with independent monodromy runs -- oracle only (no CUDA path).

  python scripts/certify_trifocal.py [seed ...]        (default seeds 101 202 303)

For every seed: the oracle's symmetry-aware monodromy (scripts/make_fixtures._monodromy: loops
p0 -> p1 -> p2 -> p0 with random complex p1, p2; Z2^3 orbit representatives; stop after 4 loops
without a new orbit) from the planted generic (x0, p0') = rng.trifocal_complex_start(seed) writes
fixtures/trifocal_cert_<seed>.sols (its representatives at p0') and .params (p0'); then the
representatives are carried to the fixture's p0 by one parameter homotopy p0' -> p0 and every
endpoint (with its symmetry images) is looked up in the fixture.  Seeds 101, 202, 303 all saturate at
668 orbits, and the homotopies between their sets are bijective up to failed paths (failed = unhit);
the round-1 fixture (seed 11, kept as trifocal_cert_11.*) had 666 and, carried to p0, leaves two
more orbits unhit than it has failed paths.  The fixture is seed 101's run (== make_fixtures.py
trifocal); tests/test_oracle_pins.py::test_trifocal_start_set_certified repeats the transfers of seeds
202 and 303 and fails if one finds an orbit the fixture lacks or maps two orbits onto one.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "scripts"))

import oracle  # noqa: E402
from hc_inputs import fixtures, rng, systems  # noqa: E402
from make_fixtures import _monodromy  # noqa: E402


def transfer(d, p_from, p_to, reps):
    """Parameter homotopy p_from -> p_to of the representatives; the CONVERGED endpoints."""
    res = oracle.track(oracle.ph_homotopy(d, p_from, p_to), reps)
    return res.x[0][res.status[0] == oracle.CONVERGED], res.status[0]


def orbit_ids(full, X, tol=1e-6):
    """Index (in the fixture's orbit numbering) of each point of X, -1 when absent."""
    out = []
    for y in X:
        hit = np.nonzero(np.all(np.abs(full - y) <= tol * np.maximum(1.0, np.abs(y)), axis=1))[0]
        out.append(int(hit[0]) // 8 if len(hit) else -1)
    return np.array(out)


def main(seeds):
    oracle.build()
    d = systems.trifocal_unknown_f()
    full, p0 = fixtures.trifocal_start()
    for seed in seeds:
        t0 = time.time()
        p0s, x0s = rng.trifocal_complex_start(seed)
        reps, fs, loops = _monodromy(d, p0s, x0s, systems.trifocal_symmetry, seed, 60, 4, f"cert {seed}")
        hdr = (f"trifocal independent monodromy run for the start-set certificate, planted (x0, p0') =\n"
               f"rng.trifocal_complex_start({seed}); written by scripts/certify_trifocal.py (oracle only):\n"
               f"{loops} loops, {len(reps)} orbits x 8 = {fs.shape[0]} solutions at p0'.")
        fixtures.write_solutions(fixtures.fixture_path(f"trifocal_cert_{seed}.sols"), np.array(reps), hdr)
        fixtures.write_params(fixtures.fixture_path(f"trifocal_cert_{seed}.params"), p0s, hdr)
        X, st = transfer(d, p0s, p0, np.array(reps))
        ids = orbit_ids(full, X)
        print(f"seed {seed}: {len(reps)} orbits by monodromy ({loops} loops, {time.time() - t0:.0f} s); "
              f"transferred to the fixture's p0: {len(X)} converged ({np.bincount(st, minlength=7).tolist()}), "
              f"{len(set(ids[ids >= 0]))} distinct fixture orbits hit, {int((ids < 0).sum())} endpoints NOT in the "
              f"fixture", flush=True)




if __name__ == "__main__":
    main([int(a) for a in sys.argv[1:]] or [101, 202, 303])
