"""Small workloads of every kernel path for compute-sanitizer (memcheck / racecheck / synccheck):
TD katsura-6 in both lane layouts, 4-view (2 instances, both layouts), P3P (16 instances),
trifocal (first 64 starts of one instance), 5-point (2 instances), batched zgesv n = 7 and 18.
Each case checks its own result loosely (the point is the sanitizer's report).

  compute-sanitizer --tool racecheck python scripts/sanitize_cases.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from hc_inputs import fixtures, rng, systems  # noqa: E402
from paper_2112_03444_b200 import hc  # noqa: E402


def cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def ph(d, S, p0, p1s):
    s = hc.System(d, device=0)
    r = hc.track_batch(s, cuda(S), cuda(p0), cuda(np.atleast_2d(p1s)))
    r.wait()
    return r


def main():
    for lanes in ("wide", "narrow"):
        os.environ["HC_LANES"] = lanes
        s = hc.System.total_degree_homotopy(systems.katsura(6), device=0)
        p0, p1 = s.td_params(rng.gamma(0))
        r = hc.track_batch(s, cuda(s.td_start()), cuda(p0), cuda(p1)[None])
        r.wait()
        print("katsura-6", lanes, int((r.status == 0).sum()), "converged", flush=True)
        d = systems.nview_triangulation(4)
        S = fixtures.read_solutions(fixtures.fixture_path("fourview_start.sols"))
        p0 = fixtures.read_params(fixtures.fixture_path("fourview_p0.params"))
        p1s, _ = rng.fourview_batch(2)
        r = ph(d, S, p0, p1s)
        print("4-view", lanes, int((r.status == 0).sum()), "converged", flush=True)
    os.environ.pop("HC_LANES")
    d = systems.p3p_depth()
    r = ph(d, fixtures.read_solutions(fixtures.fixture_path("p3p_start.sols")),
           fixtures.read_params(fixtures.fixture_path("p3p_p0.params")), rng.p3p_batch(16)[0])
    print("P3P", int((r.status == 0).sum()), "converged", flush=True)
    start, p0 = fixtures.trifocal_start()
    p1, _ = rng.trifocal_instance(rng.SEED_TRIFOCAL_INSTANCE)
    r = ph(systems.trifocal_unknown_f(), start[:64], p0, p1)
    print("trifocal", int((r.status == 0).sum()), "converged of 64", flush=True)
    d = systems.fivepoint_relpose_depth()
    r = ph(d, fixtures.read_solutions(fixtures.fixture_path("fivepoint_start.sols")),
           fixtures.read_params(fixtures.fixture_path("fivepoint_p0.params")), rng.fivepoint_batch(2)[0])
    print("5-point", int((r.status == 0).sum()), "converged", flush=True)
    g = np.random.default_rng(0)
    for n in (7, 18):
        A = g.standard_normal((64, n, n)) + 1j * g.standard_normal((64, n, n))
        b = g.standard_normal((64, n)) + 1j * g.standard_normal((64, n))
        x, info = hc.batched_zgesv(cuda(A), cuda(b))
        err = np.abs(np.einsum("bij,bj->bi", A, x.cpu().numpy()) - b).max()
        print("zgesv", n, "max residual", err, flush=True)


if __name__ == "__main__":
    main()
