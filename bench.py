"""Benchmark: device-timed tracks/s and instances/s of the fused B200 HC tracker.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config trifocal|fourview|fivepoint|p3p|cyclic7|cyclic7ph|katsura6|eco12]
                  [--instances B | --total-instances T] [--impl ours|reference] [--no-e2e] [--no-cpu-baseline]

One "step" = one pass of the whole hot path (coefficient prologue + fused tracker: every
§8(a) row a2-a10) over one batch.  Default workload: trifocal pose with unknown focal length,
parameter homotopy from the oracle-generated start fixture (S = 5344 start solutions) to
B = 1024 planted synthetic instances per GPU (BASELINE.json configs[3]; at 8 GPUs the job is
configs[4], 8192 instances) -> weak scaling; `--total-instances 8192` runs configs[4] as a fixed
job split over the GPUs (strong scaling).  Under torchrun each rank owns its own
instance block (no collective on the data path); solutions are gathered to rank 0 with NCCL
after the timed region (timed separately, `gather_ms`).

--impl reference times the CPU oracle (oracle/, test infrastructure) on the host cores on a
bounded sample of the same workload (this run has no reference implementation to install).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

BASELINE = json.load(open(os.path.join(ROOT, "BASELINE.json")))
METRIC = BASELINE["metric"]
SM_MAX_MHZ = 1965.0
FP64_DFMA_PER_CLK_PER_SM = 64   # B200 FP64 vector: 64 DFMA/clk/SM


# ------------------------------------------------------------------------------ workloads

def instance_range(args, rank: int, world: int) -> tuple[int, int]:
    """Global instance block [lo, hi) of this rank (paper_2112_03444_b200.distributed.shard_range):
    weak scaling gives every rank --instances instances (the job grows with the GPU count), strong
    scaling splits --total-instances (configs[4]: 8192) into balanced contiguous blocks."""
    from paper_2112_03444_b200.distributed import shard_range
    if args.total_instances:
        return shard_range(args.total_instances, rank, world)
    return shard_range(args.instances * world, rank, world)


def make_workload(name: str, lo: int, hi: int):
    """Seeded synthetic inputs (hc_inputs) for the global instances [lo, hi): (desc, start_x, p0, p1s,
    settings overrides, meta); instance b is generated from seed base + b whichever rank owns it."""
    from hc_inputs import fixtures, rng, systems
    B = hi - lo
    if name == "trifocal":
        d = systems.trifocal_unknown_f()
        start, p0 = fixtures.trifocal_start()
        p1s = np.stack([rng.trifocal_instance(rng.SEED_TRIFOCAL_INSTANCE + b)[0] for b in range(lo, hi)])
        meta = {"workload": f"trifocal rel. pose unknown f (18x18, Table 2 P:488) PH, S={start.shape[0]} starts "
                            f"(oracle monodromy fixture) x {B} planted instances per GPU (configs[3]; "
                            f"configs[4] = 8192 instances at 8 GPUs)"}
        return d, start, p0, p1s, {}, meta
    if name == "fourview":
        d = systems.nview_triangulation(4)
        start = fixtures.read_solutions(fixtures.fixture_path("fourview_start.sols"))
        p0 = fixtures.read_params(fixtures.fixture_path("fourview_p0.params"))
        p1s = np.stack([rng.fourview_instance(rng.SEED_FOURVIEW_INSTANCE + b)[0] for b in range(lo, hi)])
        meta = {"workload": f"4-view triangulation (14x14, Table 2 P:490) PH, S=296 x {B} planted instances "
                            f"per GPU (configs[2])"}
        return d, start, p0, p1s, {}, meta
    if name == "fivepoint":
        d = systems.fivepoint_relpose_depth()
        start = fixtures.read_solutions(fixtures.fixture_path("fivepoint_start.sols"))
        p0 = fixtures.read_params(fixtures.fixture_path("fivepoint_p0.params"))
        p1s = np.stack([rng.fivepoint_instance(rng.SEED_FIVEPOINT_INSTANCE + b)[0] for b in range(lo, hi)])
        meta = {"workload": f"5-point rel. pose + depth (16x16, Table 2 P:492; reading R24) PH, S=40 x {B} "
                            f"planted instances per GPU (SURVEY N2)"}
        return d, start, p0, p1s, {}, meta
    if name == "p3p":
        d = systems.p3p_depth()
        start = fixtures.read_solutions(fixtures.fixture_path("p3p_start.sols"))
        p0 = fixtures.read_params(fixtures.fixture_path("p3p_p0.params"))
        p1s = np.stack([rng.p3p_instance(rng.SEED_P3P_INSTANCE + b)[0] for b in range(lo, hi)])
        meta = {"workload": f"P3P absolute pose, depth form (3x3, Eq. P3PafterElim P:260-273, Table 2 P:512) PH, "
                            f"S={start.shape[0]} x {B} planted instances per GPU (SURVEY N2)"}
        return d, start, p0, p1s, {}, meta
    if name == "cyclic7ph":
        d = systems.cyclic_family(7)
        start = fixtures.read_solutions(fixtures.fixture_path("cyclic7_start.sols"))
        p0 = fixtures.read_params(fixtures.fixture_path("cyclic7_p0.params"))
        p1s = systems.cyclic_family_target(7)[None]   # one instance: the standard cyclic-7 (Table 1)
        meta = {"workload": f"cyclic-7 parameter homotopy from the oracle monodromy start (S={start.shape[0]}, "
                            f"coefficient family) to the standard cyclic-7, single instance (configs[1] system, "
                            f"the paper's monodromy-start workflow P:478)"}
        return d, start, p0, p1s, {}, meta
    if name in ("cyclic7", "katsura6", "eco12"):
        d = {"cyclic7": lambda: systems.cyclic(7), "katsura6": lambda: systems.katsura(6),
             "eco12": lambda: systems.eco(12)}[name]()
        which = {"cyclic7": "configs[1]", "katsura6": "configs[0]", "eco12": "Table 1 P:469, SURVEY N2"}[name]
        meta = {"workload": f"{d.name} total-degree homotopy, gamma seed 2, single instance ({which})"}
        return d, None, None, None, {}, meta
    raise SystemExit(f"unknown config {name}")


# ------------------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.p = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.idx), "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "samples": len(sm),
                "reasons": sorted(reasons)}


# ------------------------------------------------------------------------------ oracle (cpu)

def oracle_sample(name: str, budget_s: float, nthreads: int | None = None):
    """Time the CPU oracle (as it stands) on a bounded, unbiased sample of the workload, sized to
    ~budget_s.  Parameter homotopies: the same number of start solutions, drawn without replacement
    by a seeded permutation, from each of up to 64 instances spread evenly over the 1024-instance
    batch (the trifocal start set is ordered by symmetry orbit and instances differ in difficulty,
    so neither a prefix of one instance nor the first instances is representative); single-instance
    workloads: the whole solve, repeated to fill the budget.  Returns (tracks/s, cores, description)."""
    import oracle
    nthreads = nthreads or oracle.nthreads_default()
    if name in ("cyclic7", "katsura6", "eco12"):
        d, _, _, _, _, _ = make_workload(name, 0, 1)
        from hc_inputs import rng
        hom = oracle.td_homotopy(d, rng.gamma(2))
        start = oracle.td_start(d.degrees())
        # estimate the whole solve's time from an evenly strided probe first (eco-12 on one thread
        # would take ~15 min), then time the whole solve only when it fits the budget
        probe = min(start.shape[0], 16 * nthreads)
        pidx = np.linspace(0, start.shape[0] - 1, probe).astype(np.int64)
        t = time.perf_counter()
        oracle.track(hom, start[pidx], nthreads=nthreads)
        d1 = (time.perf_counter() - t) * start.shape[0] / probe
        if d1 <= budget_s:
            t = time.perf_counter()
            oracle.track(hom, start, nthreads=nthreads)
            d1 = time.perf_counter() - t
        reps = int(min(1000, max(1, budget_s / max(d1, 1e-4))))
        if d1 > budget_s:   # eco-12 (118,098 tracks): a strided subset
            m = max(nthreads * 4, int(start.shape[0] * budget_s / d1))
            idx = np.linspace(0, start.shape[0] - 1, m).astype(np.int64)
            t = time.perf_counter()
            oracle.track(hom, start[idx], nthreads=nthreads)
            dt = time.perf_counter() - t
            return m / dt, nthreads, f"{m} of {start.shape[0]} tracks, evenly strided ({dt:.1f} s, {nthreads} threads)"
        t = time.perf_counter()
        for _ in range(reps):
            oracle.track(hom, start, nthreads=nthreads)
        dt = time.perf_counter() - t
        return start.shape[0] * reps / dt, nthreads, (f"all {start.shape[0]} tracks, {reps} repetitions "
                                                      f"({dt:.1f} s, {nthreads} threads)")
    n_batch = 1 if name == "cyclic7ph" else 1024
    k = min(64, n_batch)
    inst = np.unique(np.linspace(0, n_batch - 1, k).astype(np.int64))
    d, start, p0, _, _, _ = make_workload(name, 0, 1)
    from hc_inputs import rng
    if name == "cyclic7ph":
        from hc_inputs import systems
        p1s = systems.cyclic_family_target(7)[None]
    else:
        p1s = np.concatenate([make_workload(name, int(b), int(b) + 1)[3] for b in inst])
    hom = oracle.ph_homotopy(d, p0)
    S = start.shape[0]
    perm = rng.gen(20261017).permutation(S)
    probe = perm[:max(4, min(S, 2 * nthreads // len(inst) + 2))]
    t = time.perf_counter()
    oracle.track(hom, start[probe], p1s=p1s, nthreads=nthreads)
    per_track = (time.perf_counter() - t) / (len(probe) * len(inst))
    m = int(min(S, max(len(probe), budget_s / max(per_track * len(inst), 1e-9))))
    reps = 1
    if m == S:
        reps = int(min(100, max(1, budget_s / max(per_track * len(inst) * S, 1e-9))))
    t = time.perf_counter()
    for _ in range(reps):
        oracle.track(hom, start[perm[:m]], p1s=p1s, nthreads=nthreads)
    dt = time.perf_counter() - t
    what = (f"{m} of {S} start solutions (seeded permutation) x {len(inst)} instances spread over the "
            f"{n_batch}-instance batch" + (f", {reps} repetitions" if reps > 1 else ""))
    return m * len(inst) * reps / dt, nthreads, f"{what} ({dt:.1f} s, {nthreads} threads)"


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores, same config/metric/unit."""
    rank = int(os.environ.get("RANK", 0))
    if rank != 0:
        return
    steps = []
    for i in range(args.warmup + args.steps):
        v, cores, sample = oracle_sample(args.config, args.ref_step_s)
        if i >= args.warmup:
            steps.append((v, sample))
    vals = [v for v, _ in steps]
    value = statistics.median(vals)
    _, _, _, _, _, meta = make_workload(args.config, 0, 1)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "tracks/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c128 (fp64)", "data": "synthetic",
            "config": {"workload": meta["workload"], "sample": steps[-1][1]},
            "cpu_baseline": {"value": value, "unit": "tracks/s", "cores": cores, "kind": "oracle",
                             "sample": steps[-1][1]},
            "e2e": {"value": value, "unit": "tracks/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)


# ------------------------------------------------------------------------------ our arm

def traffic_bytes(config: str, B: int, S: int):
    """DRAM bytes (read + write) per launch of the tracker kernel for this exact workload, as
    captured by ncu (dram__bytes_read.sum + dram__bytes_write.sum) and recorded in
    profiles/traffic.json by scripts/record_traffic.py; None when no capture of this shape exists."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "traffic.json")))
    except (OSError, ValueError):
        return None
    e = rec.get(f"{config}:{B}x{S}")
    return None if e is None else e.get("bytes")


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2112_03444_b200 import hc
    from paper_2112_03444_b200.distributed import env_rank_world, gather_to_rank0

    rank, local_rank, world = env_rank_world()
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ or args.gather
    if distributed:
        dist.init_process_group("nccl", device_id=dev, init_method=None if "MASTER_ADDR" in os.environ
                                else "tcp://127.0.0.1:29533", world_size=world, rank=rank)

    def barrier():
        if distributed:
            dist.barrier(device_ids=[local_rank])

    lo, hi = instance_range(args, rank, world)
    B = hi - lo
    d, start, p0, p1s, _, meta = make_workload(args.config, lo, hi)
    if p1s is not None:
        B = p1s.shape[0]   # single-instance workloads fix their own batch
    if start is None:
        from hc_inputs import rng
        sysh = hc.System.total_degree_homotopy(d, device=local_rank)
        p0, p1 = sysh.td_params(rng.gamma(2))
        p1s = p1[None]
        start = sysh.td_start()
        B = 1
    else:
        sysh = hc.System(d, device=local_rank)
    S, N = start.shape
    info = sysh.info
    st = hc.hc_tracker_settings_default()
    if args.config in ("trifocal", "fourview", "fivepoint", "p3p"):   # sharded multi-instance job: pinned layout
        from paper_2112_03444_b200.distributed import sharded_settings
        st = sharded_settings(st)
    x_start = torch.from_numpy(start).to(dev)
    t_p0 = torch.from_numpy(np.ascontiguousarray(p0)).to(dev)
    t_p1 = torch.from_numpy(np.ascontiguousarray(p1s)).to(dev)
    out = (torch.empty((B, S, N), dtype=torch.complex128, device=dev),
           torch.empty((B, S), dtype=torch.int32, device=dev),
           torch.empty((B, S, 4), dtype=torch.int32, device=dev),
           torch.empty((B, S, 2), dtype=torch.float64, device=dev),
           torch.empty((B, S), dtype=torch.int32, device=dev))   # Cauchy endgame winding numbers
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)   # 256 MB > 126 MB L2
    # --flush-clean (traffic measurements only): a second 256 MB buffer read after the write flush
    # evicts the flush's dirty lines before the kernel, so the kernel's DRAM counters see only its own
    # write-backs
    flush_rd = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev) if args.flush_clean else None
    stream = torch.cuda.current_stream(dev)

    def step():
        flush.fill_(1.0)   # L2 flush between steps (outside our kernels)
        if flush_rd is not None:
            flush_rd.sum()
        return hc.track_batch(sysh, x_start, t_p0, t_p1, st=st, stream=stream, out=out)

    # warm-up: the same hot path on the first `warmup_instances` instances of the batch (module load,
    # shared-memory carve-out, stream-ordered allocator pool), then the timed full-batch steps
    wb = max(1, min(B, args.warmup_instances))
    for _ in range(args.warmup):
        flush.fill_(1.0)
        hc.track_batch(sysh, x_start, t_p0, t_p1[:wb], st=st, stream=stream,
                       out=tuple(o[:wb] for o in out)).wait()
    # ---- the FP64 peak measured in-process, on this GPU, with its clock (the roofline denominator
    #      beside the derived 148 x 64 DFMA/clk x 2 x 1965 MHz) ----
    pclk = ClockSampler(local_rank)
    pclk.start()
    time.sleep(0.3)
    peak_meas = hc.fp64_peak_probe(local_rank)
    peak_ck = pclk.stop()
    clocks = ClockSampler(local_rank)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    e0.record(stream)
    results = []
    for i in range(args.steps):
        ev[i].record(stream)
        results.append(step())
    ev[-1].record(stream)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    ck = clocks.stop()
    elapsed = e0.elapsed_time(e1)
    t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    if distributed:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    elapsed_max = float(t.item())
    step_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(args.steps)]   # this rank, per step
    launch = results[0].launch()
    per_launch = [r.elapsed_ms() for r in results]   # (total, prologue, tracker) events on the launch stream
    tracker_ms = statistics.mean(p[2] for p in per_launch)
    prologue_ms = statistics.mean(p[1] for p in per_launch)
    endgame_ms = statistics.mean(p[0] - p[1] - p[2] for p in per_launch)   # Cauchy endgame (+ its prologue)
    ctr = out[2]
    solves = int(ctr[..., 3].sum().item())
    # our kernels per step: coefficient prologue + tracker, + the Cauchy endgame kernel when the endgame
    # is on, + its own prologue when its layout (wide for N <= 16) differs from the tracker's
    # (abi.cpp hc_track_batch)
    wide = launch["lanes_per_track"] == 32 and N <= 16
    eg_on = st.eg_start > 0
    n_launch = 2 + (1 if eg_on else 0) + (1 if eg_on and (N <= 16) != wide else 0)
    status = out[1]
    flops = solves * info["flops_solve"]
    converged = int((status == hc.HC_CONVERGED).sum().item())
    status_counts = torch.bincount(status.reshape(-1).to(torch.int64), minlength=7).tolist()
    eg_tracks = int((results[0].winding > 0).sum().item()) if results[0].winding is not None else None
    for r in results:
        r.close()

    B_all = B
    if distributed:   # uneven strong-scaling shards: count what every rank processed
        tb = torch.tensor([B], dtype=torch.int64, device=dev)
        dist.all_reduce(tb)
        B_all = int(tb.item())
    tracks_total = B_all * S * args.steps
    value = tracks_total / (elapsed_max / 1e3)
    sm_mhz = ck.get("sm_mhz") or SM_MAX_MHZ
    peak_max = 148 * FP64_DFMA_PER_CLK_PER_SM * 2 * SM_MAX_MHZ * 1e6 / 1e12
    achieved = flops / (tracker_ms / 1e3) / 1e12

    # ---- gather solutions to rank 0 (NCCL), timed separately ----
    gather_ms = None
    if distributed:
        barrier()
        torch.cuda.synchronize()
        g0 = time.perf_counter()
        gather_to_rank0(list(out[:4]))
        torch.cuda.synchronize()
        gather_ms = (time.perf_counter() - g0) * 1e3

    # ---- end to end through the C ABI with host buffers (pinned), H2D + D2H inside ----
    e2e = None
    if not args.no_e2e:
        pin = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True).numpy()   # noqa: E731
        hx = pin((B, S, N), torch.complex128)
        hs = pin((B, S), torch.int32)
        hcn = pin((B, S, 4), torch.int32)
        hr = pin((B, S, 2), torch.float64)
        hstart = pin((S, N), torch.complex128)
        hstart[:] = start
        hp0 = pin(p0.shape, torch.complex128)
        hp0[:] = p0
        hp1 = pin(np.shape(p1s), torch.complex128)
        hp1[:] = p1s
        barrier()
        k = max(1, min(args.steps, args.e2e_steps))
        w0 = time.perf_counter()
        for _ in range(k):
            hc.track_batch_host(sysh, hstart, hp0, hp1, st=st, out=(hx, hs, hcn, hr)).close()
        w = time.perf_counter() - w0
        tw = torch.tensor([w], dtype=torch.float64, device=dev)
        if distributed:
            dist.all_reduce(tw, op=dist.ReduceOp.MAX)
        h2d = hstart.nbytes + hp0.nbytes + hp1.nbytes
        d2h = hx.nbytes + hs.nbytes + hcn.nbytes + hr.nbytes
        e2e = {"value": B_all * S * k / float(tw.item()), "unit": "tracks/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "steps": k, "timing": "wall clock around synchronous hc_track_batch "
               "(HC_MEM_HOST, pinned buffers), max over ranks"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        v, cores, sample = oracle_sample(args.config, args.cpu_budget_s)
        cpu = {"value": v, "unit": "tracks/s", "cores": cores, "kind": "oracle", "sample": sample}
        if args.config in ("katsura6", "cyclic7", "cyclic7ph", "eco12"):   # benchmarks also on 1 thread
            v1, _, sample1 = oracle_sample(args.config, min(args.cpu_budget_s, 5.0), nthreads=1)
            cpu["single_thread"] = {"value": v1, "unit": "tracks/s", "cores": 1, "sample": sample1}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "tracks/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.total_instances else "weak", "vs_baseline": None, "dtype": "c128 (fp64)",
            "data": "synthetic", "instances_per_sec": B_all * args.steps / (elapsed_max / 1e3),
            "config": {"workload": meta["workload"], "instances_per_gpu": B, "instances_total": B_all,
                       "instance_block_rank0": [lo, hi], "tracks_per_instance": S,
                       "N": N, "l2": "256 MB buffer written between steps (flush)", "parallelism": f"dp{world}",
                       "warmup_instances": wb,
                       "launch": launch},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak_max, "unit": "TFLOP/s",
                         "frac": achieved / peak_max, "traffic": traffic_bytes(args.config, B, S),
                         "kernel": "hcb::hc_track_kernel<%d>" % N,
                         "peak_note": "FP64 vector: 148 SM x 64 DFMA/clk x 2 x 1965 MHz (derived, DESIGN.md); "
                                      "frac at the measured median clock: %.3f" %
                                      (achieved / (peak_max * sm_mhz / SM_MAX_MHZ)),
                         "peak_measured": peak_meas, "frac_of_measured": achieved / peak_meas,
                         "peak_measured_clocks": peak_ck,
                         "peak_measured_note": "hc_fp64_peak_probe (8 independent DFMA chains per thread, "
                                               "2048 threads/SM) run in this process before the timed region",
                         "flops_per_launch": flops,
                         "tracker_ms_per_launch": tracker_ms, "prologue_ms_per_launch": prologue_ms,
                         "endgame_ms_per_launch": endgame_ms},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": n_launch * args.steps,
            "gpu_launches_per_step": n_launch,
            "clocks": ck, "converged_fraction": converged / (B * S), "gather_ms": gather_ms,
            "status_counts": dict(zip(hc.STATUS_NAMES, status_counts)), "cauchy_endgame_tracks": eg_tracks,
            "solves_per_track": solves / (B * S),
            "step_ms": {"median": statistics.median(step_ms), "p10": float(np.percentile(step_ms, 10)),
                        "p90": float(np.percentile(step_ms, 90)), "n": len(step_ms)},
        }
        emit(line)
    if distributed:
        dist.destroy_process_group()


_JSON_OUT = None


def emit(line):
    """Print the one JSON line on the process's original stdout (everything else -- e.g. NCCL's
    version banner at communicator init -- goes to stderr, so the line is the only stdout output)."""
    out = _JSON_OUT or sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def main():
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")   # the original stdout, for the JSON line only
    os.dup2(2, 1)                           # fd 1 -> stderr for libraries writing to stdout
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="trifocal", choices=["trifocal", "fourview", "fivepoint", "p3p", "cyclic7", "cyclic7ph", "katsura6", "eco12"])
    ap.add_argument("--instances", type=int, default=1024, help="instances per GPU (weak scaling)")
    ap.add_argument("--total-instances", type=int, default=0,
                    help="fixed total instances split over the GPUs (strong scaling, e.g. configs[4]: 8192)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--warmup-instances", type=int, default=16)
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gather", action="store_true", help="init NCCL and run the final gather even on 1 GPU")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--flush-clean", action="store_true", help="(traffic measurements) read a second buffer after the L2 flush")
    ap.add_argument("--cpu-budget-s", type=float, default=15.0)
    ap.add_argument("--ref-step-s", type=float, default=10.0)
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
