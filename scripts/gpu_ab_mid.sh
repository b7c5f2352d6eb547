for L in lib lib_w16 lib lib_w16; do
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 2 \
    --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ABMID', '$L', round(d['step_ms']['median'],2), round(d['roofline']['frac'],4), d['config']['launch'])"
done | tee gpurun_out/ab_mid.log
timeout 300 python bench.py --total-instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_total64.json 2>&1; cut -c1-200 gpurun_out/bench_total64.json | tail -1
