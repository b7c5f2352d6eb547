"""Fig. 3 re-run: batched small complex linear solves in
complex FP64 on B200, the fused in-register LU + solve on [A | b] (hc_batched_zgesv, one sub-warp per
system) against the library the paper compares with -- cuBLAS batched LU + solve called directly
(cublasZgetrfBatched + cublasZgetrsBatched, tools/cublas_zgesv.cu) -- and, for context, against
torch.linalg.solve.

  python scripts/bench_zgesv.py            (Fig. 3 shape: batch 1000, n = 4..20 and 24, 28, 32;
                                            then a batch sweep 1e3 .. 1e6 at n = 4, 8, 16, 20, 32)

Device time by CUDA events, median of the repeats after warm-up (cuBLAS: getrf + getrs between
events, the input copies outside).  Every solution of the 1000-batch is checked against numpy
(LAPACK zgesv); the sweep checks ours against cuBLAS.  One JSON line per (n, batch).
"""
import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2112_03444_b200 import hc  # noqa: E402

CUBLAS_SO = os.path.join(ROOT, "tools", "libcublas_zgesv.so")


def cublas_lib():
    src = os.path.join(ROOT, "tools", "cublas_zgesv.cu")
    if not os.path.exists(CUBLAS_SO) or os.path.getmtime(CUBLAS_SO) < os.path.getmtime(src):
        subprocess.run(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                        "-Xcompiler", "-fPIC", "-o", CUBLAS_SO, src, "-lcublas"], check=True)
    lib = C.CDLL(CUBLAS_SO)
    lib.cublas_zgesv_time.argtypes = [C.c_int, C.c_longlong, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int,
                                      C.POINTER(C.c_float), C.POINTER(C.c_int)]
    lib.cublas_zgesv_time.restype = C.c_int
    return lib


def time_ms(fn, reps=30):
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


def run(lib, n, batch, check_lapack):
    torch.manual_seed(2112 + n)
    dA = torch.randn((batch, n, n), dtype=torch.complex128, device="cuda") + 2 * torch.eye(n, device="cuda")
    db = torch.randn((batch, n), dtype=torch.complex128, device="cuda")
    x, info = hc.batched_zgesv(dA, db)
    torch.cuda.synchronize()
    reps = 30 if batch <= 100000 else 10
    t_ours = time_ms(lambda: hc.batched_zgesv(dA, db), reps)
    xc = torch.empty_like(db)
    ms, nz = C.c_float(), C.c_int()
    rc = lib.cublas_zgesv_time(n, batch, dA.data_ptr(), db.data_ptr(), xc.data_ptr(), reps, C.byref(ms), C.byref(nz))
    assert rc == 0, rc
    line = {"n": n, "batch": batch, "ours_ms": t_ours, "cublas_getrf_getrs_ms": ms.value,
            "speedup_vs_cublas": ms.value / t_ours, "ours_gflops": lu_flops(n) * batch / t_ours / 1e6,
            "max_rel_diff_vs_cublas": float(((x - xc).abs().amax(1) / xc.abs().amax(1).clamp(min=1)).max().item()),
            "all_ok": bool((info == 0).all().item()) and nz.value == 0}
    if check_lapack:
        A, b = dA.cpu().numpy(), db.cpu().numpy()
        ref = np.linalg.solve(A, b[..., None])[..., 0]
        line["max_rel_err_vs_lapack"] = float(np.max(np.abs(x.cpu().numpy() - ref) /
                                                    np.maximum(1, np.abs(ref).max(1, keepdims=True))))
        line["torch_linalg_solve_ms"] = time_ms(lambda: torch.linalg.solve(dA, db[..., None]), reps)
    print(json.dumps(line), flush=True)


def main():
    lib = cublas_lib()
    for n in list(range(4, 21)) + [24, 28, 32]:
        run(lib, n, 1000, True)
    for n in (4, 8, 16, 20, 32):
        for batch in (10000, 100000, 1000000):
            run(lib, n, batch, False)


if __name__ == "__main__":
    main()
