"""GPU monodromy solver timings: wall time of `monodromy_solve` (every path tracked by
libhc.so) from the planted generic starts to saturation, per workload; one JSON line each.

  python scripts/bench_monodromy.py [cyclic7 fivepoint fourview trifocal]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from hc_inputs import rng, systems  # noqa: E402
from paper_2112_03444_b200 import hc  # noqa: E402
from paper_2112_03444_b200.monodromy import monodromy_solve  # noqa: E402


def case(name):
    if name == "cyclic7":
        d = systems.cyclic_family(7)
        p0, x0 = rng.cyclic_family_start(7)
        return d, p0, x0, None, "Table 1 P:467: 924"
    if name == "fivepoint":
        d = systems.fivepoint_relpose_depth()
        p0, x0 = rng.fivepoint_complex_start()
        return d, p0, x0, systems.fivepoint_symmetry, "reading R24: 40 (paper 160)"
    if name == "fourview":
        d = systems.nview_triangulation(4)
        p0, x0 = rng.fourview_complex_start()
        return d, p0, x0, None, "Table 2 P:490: 296"
    if name == "trifocal":
        d = systems.trifocal_unknown_f()
        p0, x0 = rng.trifocal_complex_start()
        return d, p0, x0, systems.trifocal_symmetry, "R19/R20: 5344 = 668 orbits x 8 (paper 1784)"
    raise SystemExit(name)


def main():
    names = sys.argv[1:] or ["cyclic7", "fivepoint", "fourview", "trifocal"]
    for name in names:
        d, p0, x0, sym, note = case(name)
        s = hc.System(d, device=0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        res = monodromy_solve(s, x0, p0, symmetry=sym, seed=3, stall_loops=4)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(json.dumps({"workload": f"{name} monodromy (GPU)", "solutions": int(res.solutions.shape[0]),
                          "expected": note, "loops": res.loops, "wall_s": dt,
                          "tracks": int(res.tracks)}), flush=True)


if __name__ == "__main__":
    main()
