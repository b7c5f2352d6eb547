"""Diagnostics: GPU vs oracle statuses for eco-10 (narrow layout) and trifocal instance 777 alone
and inside the 1024-instance batch (stale per-slot state would show only in the batch)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import oracle  # noqa: E402
from hc_inputs import fixtures, rng, systems  # noqa: E402
from paper_2112_03444_b200 import hc  # noqa: E402

oracle.build()
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731

d = systems.eco(10)
s = hc.System.total_degree_homotopy(d, device=0)
p0, p1 = s.td_params(rng.gamma(2))
X0 = s.td_start()
res = hc.track_batch(s, cu(X0), cu(p0), cu(p1)[None])
res.wait()
ref = oracle.track(oracle.td_homotopy(d, rng.gamma(2)), oracle.td_start(d.degrees()))
st = res.status.cpu().numpy()[0]
print("eco-10 gpu", np.bincount(st, minlength=8).tolist(), "oracle", np.bincount(ref.status[0], minlength=8).tolist(), res.launch())
bad = np.nonzero(st != ref.status[0])[0]
print(" mismatching tracks", len(bad), "first", bad[:10].tolist())
for k in bad[:6]:
    print("  ", k, "gpu", st[k], res.counters.cpu().numpy()[0][k].tolist(), res.resid.cpu().numpy()[0][k].tolist(),
          "orc", ref.status[0][k], ref.counters[0][k].tolist())
res2 = hc.track_batch(s, cu(X0), cu(p0), cu(p1)[None], st=hc.settings(eg_start=0.0))
res2.wait()
print("eco-10 gpu, endgame off", np.bincount(res2.status.cpu().numpy()[0], minlength=8).tolist())

d = systems.trifocal_unknown_f()
start, p0 = fixtures.trifocal_start()
p1s, xg = rng.trifocal_batch(1024)
s = hc.System(d, device=0)
for name, P in (("alone", p1s[777:778]), ("batch", p1s)):
    r = hc.track_batch(s, cu(start), cu(p0), cu(P))
    r.wait()
    b = 0 if name == "alone" else 777
    stt = r.status.cpu().numpy()[b]
    print("trifocal 777", name, np.bincount(stt, minlength=8).tolist(), "windings", np.bincount(r.winding.cpu().numpy()[b]).tolist())
    if name == "batch":
        allst = r.status.cpu().numpy()
        conv = (allst == 0).mean(1)
        print("  converged fraction by instance: min", conv.min(), "argmin", int(conv.argmin()), "first bad", np.nonzero(conv < 0.9)[0][:20].tolist())
        print("  statuses of the whole batch", np.bincount(allst.ravel(), minlength=8).tolist())
