"""SASS-level stall attribution of the tracker kernel from an ncu report (captured with
--import-source on, -lineinfo build): splits the kernel's instructions into the elimination (the
address range of the arg-max REDUX instructions, i.e. lu_rows) and the rest (evaluation, state
machine), and prints per region and per opcode the share of warp-stall samples, of executed
instructions, and the dominant stall reasons.

  python scripts/ncu_sass_regions.py <report.ncu-rep> [top_opcodes]
"""
import collections
import csv
import io
import subprocess
import sys


def load(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = next(r for r in rows if "Address" in r and "Source" in r)
    ix = {h: i for i, h in enumerate(hdr)}
    stall_keys = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    recs = []
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) < len(hdr):
            continue
        try:
            addr = int(r[ix["Address"]], 16)
        except ValueError:
            continue

        def f(k):
            try:
                return float(r[ix[k]] or 0)
            except ValueError:
                return 0.0
        rec = {"addr": addr, "src": r[ix["Source"]], "samp": f("Warp Stall Sampling (All Samples)"),
               "ex": f("Instructions Executed")}
        rec.update({k: f(k) for k in stall_keys})
        recs.append(rec)
    return recs, stall_keys


def opcode(src):
    t = src.split()
    return (t[1] if t and t[0].startswith("@") and len(t) > 1 else (t[0] if t else "?"))


def main():
    recs, sk = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 12
    tot = sum(x["samp"] for x in recs) or 1.0
    totex = sum(x["ex"] for x in recs) or 1.0
    red = [x["addr"] for x in recs if "CREDUX" in x["src"] or "REDUX" in x["src"]]
    lo, hi = (min(red), max(red)) if red else (0, -1)
    region = lambda a: "elimination (lu_rows)" if lo - 0x200 <= a <= hi + 0x400 else "evaluation + state machine"
    print(f"instructions {len(recs)}, stall samples {tot:.0f}, executed {totex:.3e}")
    for g in ("elimination (lu_rows)", "evaluation + state machine"):
        xs = [x for x in recs if region(x["addr"]) == g]
        s = sum(x["samp"] for x in xs) or 1.0
        st = sorted(((k[6:], sum(x[k] for x in xs) / s) for k in sk), key=lambda kv: -kv[1])
        print(f"\n== {g}: {100 * s / tot:.1f}% of samples, {100 * sum(x['ex'] for x in xs) / totex:.1f}% of executed "
              f"instructions; stalls: " + ", ".join(f"{k} {100 * v:.0f}%" for k, v in st if v > 0.03))
        op = collections.defaultdict(lambda: collections.Counter())
        for x in xs:
            c = op[opcode(x["src"])]
            c["samp"] += x["samp"]
            c["ex"] += x["ex"]
            c["n"] += 1
            for k in sk:
                c[k] += x[k]
        for o, c in sorted(op.items(), key=lambda kv: -kv[1]["samp"])[:top]:
            ss = max(c["samp"], 1.0)
            why = ", ".join(f"{k[6:]} {100 * c[k] / ss:.0f}%" for k in sk if c[k] / ss > 0.1)
            print(f"  {o:18s} static {int(c['n']):5d}  samples {100 * c['samp'] / tot:5.1f}%  executed "
                  f"{100 * c['ex'] / totex:5.1f}%  ({why})")


if __name__ == "__main__":
    main()
