# verification of the 8/16-lane REDUX commits: full GPU suite, smoke, A/B against the butterfly build
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for L in lib_noseg lib lib_noseg lib; do for c in "fourview 1024 3" "fivepoint 16384 2" "eco12 1 3" "p3p 65536 3" "cyclic7 1 5" "katsura6 1 10"; do set -- $c
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG', '$L', '$1', round(d['step_ms']['median'],3), round(d['roofline']['frac'],4))"
done; done | tee gpurun_out/seg_ab.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json | cut -c1-600
