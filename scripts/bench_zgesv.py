"""Fig. 3 re-run: batched small complex linear solves,
1000 matrices of size n x n, n = 4..20 (and up to 32), complex FP64 on B200.

Compares the fused in-register LU + solve on [A | b] (hc_batched_zgesv, one sub-warp per system)
with torch.linalg.solve on the same batch (cuSOLVER/cuBLAS batched getrf + getrs: the library
baseline of the figure).  Device time by CUDA events, median of 50 repeats after warm-up;
prints one JSON line per n.  Also checks every solution against numpy (LAPACK zgesv).
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2112_03444_b200 import hc  # noqa: E402


def time_ms(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def lu_flops(n):
    f = sum(j * (6 + 8 * (j + 1)) for j in range(n))
    return f + 8 * n * (n - 1) // 2 + 6 * n


def main():
    batch = int(os.environ.get("BATCH", 1000))
    g = np.random.Generator(np.random.PCG64(2112))
    for n in list(range(4, 21)) + [24, 28, 32]:
        A = (g.standard_normal((batch, n, n)) + 1j * g.standard_normal((batch, n, n))) + 2 * np.eye(n)
        b = g.standard_normal((batch, n)) + 1j * g.standard_normal((batch, n))
        dA, db = torch.from_numpy(A).cuda(), torch.from_numpy(b).cuda()
        x, info = hc.batched_zgesv(dA, db)
        torch.cuda.synchronize()
        ref = np.linalg.solve(A, b[..., None])[..., 0]
        err = float(np.max(np.abs(x.cpu().numpy() - ref) / np.maximum(1, np.abs(ref).max(1, keepdims=True))))
        t_ours = time_ms(lambda: hc.batched_zgesv(dA, db))
        t_lib = time_ms(lambda: torch.linalg.solve(dA, db[..., None]))
        fl = lu_flops(n) * batch
        print(json.dumps({"n": n, "batch": batch, "ours_ms": t_ours, "torch_linalg_solve_ms": t_lib,
                          "speedup_vs_library": t_lib / t_ours, "ours_gflops": fl / t_ours / 1e6,
                          "max_rel_err_vs_lapack": err, "all_ok": bool((info == 0).all().item())}), flush=True)


if __name__ == "__main__":
    main()
