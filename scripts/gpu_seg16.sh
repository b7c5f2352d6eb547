python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "fourview or fivepoint or eco or lane or three_view or two_view or shape or large_n or zgesv" > gpurun_out/pytest_seg16.log 2>&1; tail -2 gpurun_out/pytest_seg16.log
for L in lib_noseg lib lib_noseg lib; do for c in "fourview 1024 3" "fivepoint 16384 2" "eco12 1 3"; do set -- $c
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 2 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG16', '$L', '$1', round(d['step_ms']['median'],2), round(d['roofline']['frac'],4))"
done; done | tee gpurun_out/seg16_ab.log
