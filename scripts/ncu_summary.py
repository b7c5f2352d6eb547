"""Summarise an ncu report: key SOL / occupancy / stall metrics + per-source-line instruction and
stall shares of the tracker kernel.  usage: python scripts/ncu_summary.py <report.ncu-rep> [top]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Elapsed Cycles", "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread",
        "Theoretical Occupancy", "Achieved Occupancy", "Achieved Active Warps Per SM", "No Eligible",
        "Eligible Warps Per Scheduler", "Warp Cycles Per Issued Instruction", "L1/TEX Hit Rate",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem", "Executed Instructions",
        "Compute (SM) Throughput", "DRAM Throughput", "Avg. Not Predicated Off Threads Per Warp"]
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
iname, iunit, ival = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
for r in rows[1:]:
    if len(r) > ival and r[iname] in want:
        print(f"{r[iname]:45s} {r[ival]:>16s} {r[iunit]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.sum", "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
            "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum", "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "local_load", "launch__registers_per_thread"]:
    for i, h in enumerate(rr[0]):
        if key in h:
            print(f"{h:70s} {rr[2][i]:>16s} {rr[1][i]}")
# warp-state (stall reason) breakdown from the PC sampler: share of samples per reason
stall = []
for i, h in enumerate(rr[0]):
    if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
        try:
            stall.append((float(rr[2][i].replace(",", "")), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
        except ValueError:
            pass
tot_st = sum(v for v, _ in stall)
if tot_st > 0:
    print("\nstall reasons (PC sampling, share of samples)")
    for v, n in sorted(stall, reverse=True)[:12]:
        print(f"  {n:28s} {100 * v / tot_st:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[2]
iE, iS = hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
lines, ti, ts = [], 0, 0
for r in rows[3:]:
    if r and r[0]:
        try:
            ie, s = int(r[iE]), int(r[iS])
        except (ValueError, IndexError):
            continue
        lines.append((ie, s, r[0], r[1][:100]))
        ti += ie
        ts += s
lines.sort(reverse=True)
print(f"\nper source line: instructions executed (total {ti}) / stall samples (total {ts})")
for ie, s, ln, t in lines[:top]:
    print(f"{100 * ie / ti:5.1f}% inst {100 * s / ts:5.1f}% stall  L{ln}: {t}")
