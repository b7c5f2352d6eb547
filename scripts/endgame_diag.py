"""Diagnostics of the GPU endgame (reading R26) on the closed-form pins and small benchmarks:
statuses, windings, counters and resid per track, GPU next to the oracle.  Run on a GPU box; with
an HCB_EG_DEBUG=1 build (HC_LIB_PATH) resid[1] of a fallen-back track holds the failure reason
(1 step budget, 2 no closure within eg_max_winding, 3 radii exhausted, 4 arc step underflow,
5 no step at the start, 6 estimate not a root, 7 radial step underflow)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
from hc_inputs import rng, systems  # noqa: E402
from hc_inputs.poly import var_x  # noqa: E402
from paper_2112_03444_b200 import hc  # noqa: E402

oracle.build()


def run(name, d, g):
    s = hc.System.total_degree_homotopy(d, device=0)
    p0, p1 = s.td_params(rng.gamma(g))
    X0 = s.td_start()
    res = hc.track_batch(s, torch.from_numpy(X0).cuda(), torch.from_numpy(p0).cuda(), torch.from_numpy(p1).cuda()[None])
    res.wait()
    ref = oracle.track(oracle.td_homotopy(d, rng.gamma(g)), oracle.td_start(d.degrees()))
    st, w = res.status.cpu().numpy()[0], res.winding.cpu().numpy()[0]
    print(f"== {name}: gpu statuses {np.bincount(st, minlength=7).tolist()} oracle {np.bincount(ref.status[0], minlength=7).tolist()}")
    print(f"   gpu windings {np.bincount(w).tolist()} oracle {np.bincount(ref.winding[0]).tolist()}")
    if len(st) <= 8:
        print("   gpu x", np.round(res.x.cpu().numpy()[0], 6).tolist())
        print("   gpu ctr", res.counters.cpu().numpy()[0].tolist(), "resid", res.resid.cpu().numpy()[0].tolist())
        print("   orc ctr", ref.counters[0].tolist())
    U = oracle.dedup(oracle.finite_solutions(ref))[0]
    G = oracle.dedup(res.x.cpu().numpy()[0][st == 0])[0]
    ok, ua, ub = oracle.match_sets(U, G, tol=1e-8)
    print(f"   sets: oracle {len(U)} gpu {len(G)} match {ok} ({ua}/{ub})")
    lost = np.nonzero((ref.status[0] == 0) & (st != 0))[0]
    if len(lost):
        print("   oracle-converged tracks the gpu lost:", len(lost), "gpu statuses", np.bincount(st[lost], minlength=7).tolist())


X = var_x(1, 0, 0)
for m in (2, 3, 4):
    run(f"(x-2)^{m}", systems.from_polys([(X - 2) ** m], "p"), 1)
x, y = var_x(2, 0, 0), var_x(2, 0, 1)
run("double root", systems.from_polys([(x - 2) ** 2 + y - 1, y - 1], "dr"), 2)
run("cyclic-5", systems.cyclic(5), 1)
run("eco-8", systems.eco(8), 2)
run("cyclic-7", systems.cyclic(7), 2)
