# A/B of the per-segment REDUX on 8-lane tracks (throughput layout forced: HC_LANES=narrow)
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in lib_noseg lib lib_noseg lib; do for c in "cyclic7 1 20" "cyclic7ph 1 20" "katsura6 1 20"; do set -- $c
  HC_LANES=narrow HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 300 python bench.py --config $1 --instances $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG8N', '$L', '$1', round(d['step_ms']['median'],3), d['config']['launch']['lanes_per_track'])"
done; done | tee gpurun_out/seg8_narrow_ab.log
