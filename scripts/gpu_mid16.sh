# A/B: CTA size for N = 15, 16 (16-lane tracks) after the per-segment REDUX: 16 warps (default) vs 12
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in lib lib_m16w12 lib lib_m16w12; do for c in "fivepoint 16384 3"; do set -- $c
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MID16', '$L', '$1', round(d['step_ms']['median'],3), round(d['roofline']['frac'],4), d['config']['launch'])"
done; done | tee gpurun_out/mid16_ab.log
