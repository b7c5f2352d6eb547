"""Python surface of the C ABI (include/hc.h): argument marshalling only.

Every step of the path (compile, coefficient prologue, evaluation, LU, RK4, Newton, step
control, classification) runs in libhc.so; PyTorch provides device memory and streams.
Names mirror the C entry points; `System`, `track_batch` and `track_batch_host` are thin
conveniences over hc_system_create / hc_track_batch / hc_result_*.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib as L
from ._lib import (HC_AT_INFINITY, HC_CONVERGED, HC_DIVERGED, HC_EULER, HC_MAX_STEPS, HC_MEM_DEVICE,  # noqa: F401
                   HC_MEM_HOST, HC_LAYOUT_AUTO, HC_LAYOUT_THROUGHPUT, HC_LAYOUT_WIDE,
                   HC_NONFINITE, HC_RK4, HC_SINGULAR, HC_STEP_UNDERFLOW, STATUS_NAMES, HCError, check)


def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _c128(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None and a.size else None


class _Desc:
    """hc_system_desc view over numpy arrays (kept alive by this object)."""

    def __init__(self, d):
        self.arrs = dict(term_eq=_i32(d.term_eq), term_xexp=_i32(d.term_xexp), term_coef=_i32(d.term_coef),
                         coef_ptr=_i32(d.coef_ptr), coef_w=_c128(d.coef_w), coef_pexp=_i32(d.coef_pexp))
        a = self.arrs
        self.c = L.hc_system_desc(int(d.n_vars), int(d.n_params), int(a["term_eq"].shape[0]), _ptr(a["term_eq"]),
                                  _ptr(a["term_xexp"]), _ptr(a["term_coef"]), int(a["coef_ptr"].shape[0] - 1),
                                  _ptr(a["coef_ptr"]), _ptr(a["coef_w"]), _ptr(a["coef_pexp"]))


def hc_tracker_settings_default() -> L.hc_tracker_settings:
    s = L.hc_tracker_settings()
    check(L.lib().hc_tracker_settings_default(C.byref(s)), "hc_tracker_settings_default")
    return s


def settings(**kw) -> L.hc_tracker_settings:
    """Default settings (SURVEY.md §8(c) readings) with overrides, e.g. settings(max_steps=400)."""
    s = hc_tracker_settings_default()
    for k, v in kw.items():
        if not hasattr(s, k):
            raise AttributeError(f"unknown tracker setting {k!r}")
        setattr(s, k, v)
    return s


def hc_system_compile_info(desc) -> dict:
    """Host-only compile of a descriptor; returns hc_system_info as a dict (no GPU needed)."""
    d = _Desc(desc)
    info = L.hc_system_info()
    check(L.lib().hc_system_compile_info(C.byref(d.c), C.byref(info)), "hc_system_compile_info")
    return info.as_dict()


def hc_system_compile_tables(desc):
    """Host-only: the compiled evaluation tables (layouts in csrc/hc_internal.h).

    Returns (ops [Q, L, 2] uint32, mono_prog [n_monos - N - 1] uint32, slot_map [n_coef_slots, 2] int32,
    entry_map [N, N + 1] int16, info)."""
    info = hc_system_compile_info(desc)
    Q, Ln = info["op_steps"], info["lanes_per_track"]
    ops = np.zeros((Q, Ln, 2), np.uint32)
    prog = np.zeros(max(0, info["n_monos"] - info["n_vars"] - 1), np.uint32)
    smap = np.zeros((info["n_coef_slots"], 2), np.int32)
    N = info["n_vars"]
    emap = np.zeros((N, N + 1), np.int16)
    d = _Desc(desc)
    check(L.lib().hc_system_compile_tables(C.byref(d.c), _ptr(ops), _ptr(prog), _ptr(smap), _ptr(emap)),
          "hc_system_compile_tables")
    return ops, prog, smap, emap, info


class System:
    """An hc_system handle (compiled tables resident on `device`)."""

    def __init__(self, desc, device: int | None = None, total_degree: bool = False):
        import torch
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.desc = desc
        d = _Desc(desc)
        h = C.c_void_p()
        fn = L.lib().hc_system_create_total_degree if total_degree else L.lib().hc_system_create
        check(fn(C.byref(d.c), self.device, C.byref(h)), fn.__name__)
        self.h = h
        self.total_degree = total_degree
        info = L.hc_system_info()
        check(L.lib().hc_system_info_get(self.h, C.byref(info)), "hc_system_info_get")
        self.info = info.as_dict()
        self.N = self.info["n_vars"]
        self.P = self.info["n_params"]

    @classmethod
    def total_degree_homotopy(cls, target_desc, device: int | None = None) -> "System":
        return cls(target_desc, device, total_degree=True)

    def td_params(self, gamma: complex):
        """(p0, p1) making the PH equal H = (1-t) gamma G + t F (hc_total_degree_params)."""
        p0 = np.zeros(self.P, np.complex128)
        p1 = np.zeros(self.P, np.complex128)
        g = L.hc_complex(complex(gamma).real, complex(gamma).imag)
        check(L.lib().hc_total_degree_params(self.h, g, _ptr(p0), _ptr(p1)), "hc_total_degree_params")
        return p0, p1

    def td_start(self) -> np.ndarray:
        cnt = L.lib().hc_total_degree_count(self.h)
        if cnt < 0:
            raise HCError(L.HC_E_TOO_LARGE, "hc_total_degree_count", "not a TD system or too many tracks")
        x = np.zeros((cnt, self.N), np.complex128)
        check(L.lib().hc_total_degree_start(self.h, _ptr(x)), "hc_total_degree_start")
        return x

    def close(self):
        if getattr(self, "h", None):
            L.lib().hc_system_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


@dataclass
class BatchResult:
    x: object          # [B, S, N] complex128
    status: object     # [B, S] int32
    counters: object   # [B, S, 4] int32: steps, rejections, newton iterations, solves
    resid: object      # [B, S, 2] float64
    handle: object = None
    winding: object = None   # [B, S] int32: Cauchy endgame winding number (0: not used), or None

    def elapsed_ms(self):
        """(total, prologue, tracker) device ms from the CUDA events on the batch stream."""
        a, b, c = C.c_float(), C.c_float(), C.c_float()
        check(L.lib().hc_result_elapsed_ms(self.handle, C.byref(a), C.byref(b), C.byref(c)), "hc_result_elapsed_ms")
        return a.value, b.value, c.value

    def wait(self):
        check(L.lib().hc_result_wait(self.handle), "hc_result_wait")

    def launch(self) -> dict:
        """Tracker launch configuration (hc_result_launch)."""
        a, b, c, d = C.c_int32(), C.c_int32(), C.c_int32(), C.c_int64()
        check(L.lib().hc_result_launch(self.handle, C.byref(a), C.byref(b), C.byref(c), C.byref(d)), "hc_result_launch")
        return {"lanes_per_track": a.value, "warps_per_cta": b.value, "ctas": c.value, "smem_per_cta": d.value}

    def close(self):
        if self.handle:
            L.lib().hc_result_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def track_batch(system: System, start_x, p0=None, p1=None, st: L.hc_tracker_settings | None = None,
                stream=None, out=None) -> BatchResult:
    """Enqueue one batch on the current (or given) CUDA stream; all tensors on system.device.

    start_x [S, N] complex128, p0 [P], p1 [B, P] (torch tensors on the device).
    Returns BatchResult with device tensors; call .wait() / .elapsed_ms() before reading.
    """
    import torch
    dev = torch.device("cuda", system.device)
    start_x = torch.as_tensor(start_x, dtype=torch.complex128, device=dev).contiguous()
    S, N = start_x.shape
    assert N == system.N, f"start_x has {N} columns, system has N={system.N}"
    if system.P > 0:
        p0 = torch.as_tensor(p0, dtype=torch.complex128, device=dev).contiguous().reshape(system.P)
        p1 = torch.as_tensor(p1, dtype=torch.complex128, device=dev).contiguous().reshape(-1, system.P)
        B = p1.shape[0]
    else:
        B = 1 if p1 is None else int(torch.as_tensor(p1).reshape(-1, 1).shape[0])
    wind = None
    if out is None:
        x = torch.empty((B, S, N), dtype=torch.complex128, device=dev)
        status = torch.empty((B, S), dtype=torch.int32, device=dev)
        ctr = torch.empty((B, S, 4), dtype=torch.int32, device=dev)
        resid = torch.empty((B, S, 2), dtype=torch.float64, device=dev)
        wind = torch.empty((B, S), dtype=torch.int32, device=dev)
    else:
        x, status, ctr, resid = out[:4]
        wind = out[4] if len(out) > 4 else None
        # the kernel writes B*S*N values through raw pointers: a wrong buffer would be an
        # out-of-bounds device write, so every output is checked before the launch
        for name, tns, shape, dtype in (("x", x, (B, S, N), torch.complex128), ("status", status, (B, S), torch.int32),
                                        ("counters", ctr, (B, S, 4), torch.int32),
                                        ("resid", resid, (B, S, 2), torch.float64)) + (
                                            (("winding", wind, (B, S), torch.int32),) if wind is not None else ()):
            if (tuple(tns.shape) != shape or tns.dtype != dtype or not tns.is_contiguous() or tns.device != dev):
                raise ValueError(f"out[{name}] must be a contiguous {dtype} tensor of shape {shape} on {dev}, "
                                 f"got {tns.dtype} {tuple(tns.shape)} on {tns.device}")
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    b = L.hc_batch(B, S, start_x.data_ptr(), p0.data_ptr() if system.P else None,
                   p1.data_ptr() if system.P else None, x.data_ptr(), status.data_ptr(), ctr.data_ptr(),
                   resid.data_ptr(), HC_MEM_DEVICE, stream.cuda_stream, wind.data_ptr() if wind is not None else None)
    h = C.c_void_p()
    check(L.lib().hc_track_batch(system.h, C.byref(st or hc_tracker_settings_default()), C.byref(b), C.byref(h)),
          "hc_track_batch")
    res = BatchResult(x, status, ctr, resid, h, wind)
    res._keep = (start_x, p0, p1, system)   # the system must outlive the result
    return res


def track_batch_host(system: System, start_x, p0=None, p1=None, st: L.hc_tracker_settings | None = None,
                     stream=None, out=None) -> BatchResult:
    """End-to-end call with HOST buffers (HC_MEM_HOST): the library copies inputs to the device,
    tracks, copies results back and returns when done.  numpy in, numpy out (`out` may supply
    preallocated, e.g. pinned, output arrays (x, status, counters, resid))."""
    start_x = _c128(start_x)
    S, N = start_x.shape
    if system.P > 0:
        p0 = _c128(p0).reshape(system.P)
        p1 = _c128(p1).reshape(-1, system.P)
        B = p1.shape[0]
    else:
        B = 1
    wind = None
    if out is None:
        x = np.empty((B, S, N), np.complex128)
        status = np.empty((B, S), np.int32)
        ctr = np.empty((B, S, 4), np.int32)
        resid = np.empty((B, S, 2), np.float64)
        wind = np.empty((B, S), np.int32)
    else:
        x, status, ctr, resid = out[:4]
        wind = out[4] if len(out) > 4 else None
        for name, a, shape, dtype in (("x", x, (B, S, N), np.complex128), ("status", status, (B, S), np.int32),
                                      ("counters", ctr, (B, S, 4), np.int32), ("resid", resid, (B, S, 2), np.float64)) + (
                                          (("winding", wind, (B, S), np.int32),) if wind is not None else ()):
            if a.shape != shape or a.dtype != dtype or not a.flags.c_contiguous:
                raise ValueError(f"out[{name}] must be a C-contiguous {np.dtype(dtype).name} array of shape {shape}, "
                                 f"got {a.dtype} {a.shape}")
    sp = stream.cuda_stream if stream is not None else None
    b = L.hc_batch(B, S, _ptr(start_x), _ptr(p0) if system.P else None, _ptr(p1) if system.P else None, _ptr(x),
                   _ptr(status), _ptr(ctr), _ptr(resid), HC_MEM_HOST, sp, _ptr(wind) if wind is not None else None)
    h = C.c_void_p()
    check(L.lib().hc_track_batch(system.h, C.byref(st or hc_tracker_settings_default()), C.byref(b), C.byref(h)),
          "hc_track_batch")
    res = BatchResult(x, status, ctr, resid, h, wind)
    res._keep = (system,)
    return res


def batched_zgesv(A, b, pivot_rel: float = 1e-14, stream=None):
    """Fused batched LU + solve on device tensors A [batch, n, n], b [batch, n] complex128.
    Returns (x [batch, n], info [batch] int32: 0 ok, 1 singular)."""
    import torch
    A = A.contiguous()
    b = b.contiguous()
    batch, n, _ = A.shape
    x = torch.empty((batch, n), dtype=torch.complex128, device=A.device)
    info = torch.empty((batch,), dtype=torch.int32, device=A.device)
    if stream is None:
        stream = torch.cuda.current_stream(A.device)
    check(L.lib().hc_batched_zgesv(n, batch, A.data_ptr(), b.data_ptr(), x.data_ptr(), info.data_ptr(),
                                   float(pivot_rel), stream.cuda_stream), "hc_batched_zgesv")
    return x, info


def solutions(x, status=None, tol: float = 1e-6, real_tol: float = 1e-6):
    """Endpoint post-processing of one instance (hc_solutions; readings R11, R12): greedy dedup in
    track order of the CONVERGED endpoints and real classification.  x [S, N] complex128 and
    status [S] (host arrays or tensors).  Returns (unique [U, N], multiplicity [U], is_real [U] bool,
    rep [S] int64: kept track each track merged into, -1 if not converged)."""
    X = _c128(x.cpu().numpy() if hasattr(x, "cpu") else x)
    S, N = X.shape
    st = None if status is None else _i32(status.cpu().numpy() if hasattr(status, "cpu") else status)
    rep = np.zeros(S, np.int64)
    real = np.zeros(S, np.int32)
    nu = C.c_int64()
    check(L.lib().hc_solutions(_ptr(X), _ptr(st), S, N, float(tol), float(real_tol), _ptr(rep), _ptr(real),
                               C.byref(nu)), "hc_solutions")
    kept = np.nonzero(rep == np.arange(S))[0]
    mult = np.array([np.sum(rep == k) for k in kept], dtype=np.int64)
    return X[kept], mult, real[kept].astype(bool), rep


def fp64_peak_probe(device: int = 0) -> float:
    """Measured FP64 DFMA throughput of `device` in TFLOP/s (hc_fp64_peak_probe)."""
    v = C.c_double()
    check(L.lib().hc_fp64_peak_probe(int(device), C.byref(v)), "hc_fp64_peak_probe")
    return v.value


def version() -> str:
    return L.lib().hc_version().decode()
