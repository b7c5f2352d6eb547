import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
from hc_inputs import rng, systems
from paper_2112_03444_b200 import hc
cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
d = systems.eco(10)
s = hc.System.total_degree_homotopy(d, device=0)
p0, p1 = s.td_params(rng.gamma(2))
X0 = s.td_start()
res = hc.track_batch(s, cu(X0), cu(p0), cu(p1)[None])
res.wait()
st = res.status.cpu().numpy()[0]
print(os.environ.get("HC_LIB_PATH"), "eco-10", np.bincount(st, minlength=8).tolist(), "first-step failures", int((res.counters.cpu().numpy()[0][:, 2] == 0).sum()))
