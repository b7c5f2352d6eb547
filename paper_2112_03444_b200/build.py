"""Build libhc.so (the C-ABI library of include/hc.h) in-tree for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo, one object per translation unit
(the tracker is instantiated once per N = 1..32 in its own unit so they compile in parallel),
static cudart, output paper_2112_03444_b200/lib/libhc.so.  Incremental: an object is rebuilt
when its source or any header is newer; objects live in a directory keyed by a hash of the
compiler flags (variant defines included), so changing HCB_DEFINES never reuses a stale object.
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
# HCB_VARIANT=timing builds an experiment library with per-phase cycle counters (-DHCB_PHASE_TIMING)
# into lib_timing/, HCB_VARIANT=hybrid one with the hybrid 16-lane layout for N = 17, 18 into
# lib_hybrid/ (load either with HC_LIB_PATH); the product library is the default variant.
VARIANT = os.environ.get("HCB_VARIANT", "")
LIBDIR = os.path.join(PKG, "lib" + ("_" + VARIANT if VARIANT else ""))
LIB = os.path.join(LIBDIR, "libhc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I" + INCLUDE, "-I" + CSRC]
if VARIANT == "timing":
    FLAGS = FLAGS + ["-DHCB_PHASE_TIMING"]
elif VARIANT == "hybrid":   # experiment: 16-lane hybrid layout for N = 17, 18 (csrc/hc_internal.h)
    FLAGS = FLAGS + ["-DHCB_HYBRID_LAYOUT=1"]
# any variant may add preprocessor switches for A/B experiments, e.g.
# HCB_VARIANT=w16 HCB_DEFINES="HCB_MAXW_MID=16" (see the #ifndef switches in kernels/tracker.cuh)
FLAGS = FLAGS + ["-D" + d for d in os.environ.get("HCB_DEFINES", "").split()] if VARIANT else FLAGS
# HCB_HOST_FLAGS: extra g++ flags for the host translation units only (e.g. the sanitizer build,
# scripts/sanitize_host.sh)
HOST_FLAGS = os.environ.get("HCB_HOST_FLAGS", "").split() if VARIANT else []
BUILD = os.path.join(PKG, "build" + ("_" + VARIANT if VARIANT else ""),
                     hashlib.sha1(" ".join(ARCH + [f for f in FLAGS if not f.startswith("-I")] + HOST_FLAGS).encode()).hexdigest()[:10])


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "kernels", "*.cu")) + glob.glob(os.path.join(CSRC, "host", "*.cpp")))


def headers():
    return (glob.glob(os.path.join(CSRC, "**", "*.h"), recursive=True)
            + glob.glob(os.path.join(CSRC, "**", "*.cuh"), recursive=True)
            + [os.path.join(INCLUDE, "hc.h")])


def _obj(src):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    return os.path.join(BUILD, rel + ".o")


def _compile(src, hdr_mtime, verbose):
    obj = _obj(src)
    if os.path.exists(obj) and os.path.getmtime(obj) >= max(os.path.getmtime(src), hdr_mtime):
        return obj, False
    lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
    host = [] if src.endswith(".cu") else [a for f in HOST_FLAGS for a in ("-Xcompiler", f)]
    cmd = [NVCC] + ARCH + FLAGS + host + lang + ["-c", src, "-o", obj]
    if verbose:
        print(" ".join(cmd), flush=True)
    p = subprocess.run(cmd, capture_output=True, text=True)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{p.stdout}\n{p.stderr}")
    return obj, True


def build(verbose: bool = False, jobs: int | None = None) -> str:
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    hdr_mtime = max(os.path.getmtime(h) for h in headers())
    srcs = sources()
    with ThreadPoolExecutor(max_workers=jobs or os.cpu_count() or 4) as ex:
        results = list(ex.map(lambda s: _compile(s, hdr_mtime, verbose), srcs))
    objs = [o for o, _ in results]
    changed = any(c for _, c in results)
    if changed or not os.path.exists(LIB) or os.path.getmtime(LIB) < max(os.path.getmtime(o) for o in objs):
        cmd = ([NVCC] + ARCH + ["-shared", "-cudart", "static", "-o", LIB] + objs + ["-lpthread", "-ldl", "-lrt"]
               + [a for f in HOST_FLAGS for a in ("-Xcompiler", f)])
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
