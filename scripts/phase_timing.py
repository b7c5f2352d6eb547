"""Per-phase cycle breakdown of the tracker kernel (experiment build HCB_VARIANT=timing).

HC_LIB_PATH=paper_2112_03444_b200/lib_timing/libhc.so python scripts/phase_timing.py [config] [instances]
Prints, per warp-iteration (one eval + solve per slot), the average cycles of each phase.
python scripts/phase_timing.py --print a.json b.json   summarises saved outputs.
"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2112_03444_b200 import _lib, hc  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "--print":
    for f in sys.argv[2:]:
        try:
            d = json.load(open(f))
        except Exception:
            continue
        print(f, round(d["cycles_per_iteration"]), d["launch"], d["tracker_ms"])
        for k, v in d["phases"].items():
            print("   %-28s %8.0f %5.1f%%" % (k, v["cycles_per_iter"], 100 * v["share"]))
    sys.exit(0)
cfg = sys.argv[1] if len(sys.argv) > 1 else "trifocal"
B = int(sys.argv[2]) if len(sys.argv) > 2 else 64
d, start, p0, p1s, _, _ = bench.make_workload(cfg, 0, B)
s = hc.System(d, device=0)
res = hc.track_batch(s, start, p0, p1s)
res.wait()
out = (C.c_ulonglong * 8)()
_lib.check(_lib.lib().hc_debug_phase_cycles(res.handle, out), "hc_debug_phase_cycles")
v = np.array(list(out), dtype=np.float64)
it = v[7]
names = ["coefficients (Horner)", "monomial program", "op list", "row load", "elimination + solve",
         "reductions + state machine"]
tot = v[6] + v[5]
print(json.dumps({"config": cfg, "instances": B, "warp_iterations": it, "cycles_per_iteration": tot / it,
                  "phases": {n: {"cycles_per_iter": v[i] / it, "share": v[i] / tot} for i, n in enumerate(names)},
                  "launch": res.launch(), "tracker_ms": res.elapsed_ms()[2]}, indent=1))
