"""Capture the tracker kernel's DRAM traffic per launch with ncu for one bench workload.

  python scripts/record_traffic.py <config> <instances> [out.json] [--dram-only]

Runs `bench.py --config C --instances B --steps 1 --warmup 3` under
`ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum` plus the FP64
thread-instruction counts (executed FLOP = 2 DFMA + DMUL + DADD), restricted to the
first full-batch launch of hc_track_kernel (the 3 warm-up launches are skipped), and merges
{"<config>:<B>x<S>": {"bytes": read + write, ...}} into out.json (default gpurun_out/traffic.json;
the committed copy is profiles/traffic.json, read by bench.py for roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    dram_only = "--dram-only" in sys.argv   # one replay pass (the SASS counters instrument the kernel: slow)
    cfg, B = args[0], int(args[1])
    out = args[2] if len(args) > 2 else os.path.join(ROOT, "gpurun_out", "traffic.json")
    metrics = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]
    if not dram_only:
        metrics += ["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
                    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
                    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
    cmd = ["ncu", "--metrics", ",".join(metrics),
           "--clock-control", "none", "-k", "regex:hc_track_kernel", "--launch-skip", "3", "-c", "1", "--csv",
           sys.executable, os.path.join(ROOT, "bench.py"), "--config", cfg, "--instances", str(B), "--steps", "1",
           "--warmup", "3", "--no-cpu-baseline", "--no-e2e", "--flush-clean"]
    p = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
    txt = p.stdout
    bench_line = None
    rows = []
    for line in txt.splitlines():
        if line.startswith("{"):
            bench_line = json.loads(line)
        elif line.startswith('"'):
            rows.append(line)
    vals = {}
    kernel = None
    for r in csv.DictReader(io.StringIO("\n".join(rows))):
        name, unit, v = r["Metric Name"], r["Metric Unit"], float(r["Metric Value"].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
                 "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
                 "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0,
                 "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "Tinst": 1e12}.get(unit, 1.0)
        vals[name] = v * scale
        kernel = r["Kernel Name"]
    if bench_line is None or "dram__bytes_read.sum" not in vals:
        sys.stderr.write(p.stdout[-3000:] + p.stderr[-3000:])
        raise SystemExit("ncu capture failed")
    S = bench_line["config"]["tracks_per_instance"]
    key = f"{cfg}:{B}x{S}"
    rec = json.load(open(out)) if os.path.exists(out) else {}
    rec[key] = {"bytes": vals["dram__bytes_read.sum"] + vals["dram__bytes_write.sum"],
                "read": vals["dram__bytes_read.sum"], "write": vals["dram__bytes_write.sum"],
                "kernel_s_under_ncu": vals.get("gpu__time_duration.sum"), "kernel": kernel,
                "tracks": B * S,
                "fp64_flops_executed": 2 * vals.get("smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", 0)
                + vals.get("smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", 0)
                + vals.get("smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", 0),
                "flops_algorithmic": bench_line["roofline"]["flops_per_launch"],
                "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum "
                                          "(scripts/record_traffic.py), first full-batch launch, the L2 flush's dirty lines "
                                          "evicted before it (bench --flush-clean)"}
    os.makedirs(os.path.dirname(out), exist_ok=True)
    json.dump(rec, open(out, "w"), indent=1)
    print(key, rec[key])


if __name__ == "__main__":
    main()
