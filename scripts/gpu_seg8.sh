python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
for L in lib_prev lib lib_prev lib; do for c in "fourview 1024 3" "fivepoint 16384 2" "eco12 1 3" "p3p 65536 3"; do set -- $c
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG8', '$L', '$1', round(d['step_ms']['median'],2), round(d['roofline']['frac'],4))"
done; done | tee gpurun_out/seg8_ab.log
for L in lib_noseg lib_prev lib; do for mode in narrow wide; do for c in "cyclic7 1 10" "katsura6 1 10"; do set -- $c
  HC_LANES=$mode HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 300 python bench.py --config $1 --instances $2 --steps $3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG8TD', '$L', '$mode', '$1', round(d['step_ms']['median'],3))"
done; done; done | tee -a gpurun_out/seg8_ab.log
