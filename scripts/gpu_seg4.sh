# A/B: REDUX arg-max / segment max also for 4-lane tracks (HCB_SEG4_REDUX) vs the butterfly
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
HC_LIB_PATH=paper_2112_03444_b200/lib_seg4/libhc.so timeout 600 python -m pytest tests -m gpu -q -k "zgesv or p3p or two_view or univariate" > gpurun_out/pytest_seg4.log 2>&1; tail -2 gpurun_out/pytest_seg4.log
for L in lib lib_seg4 lib lib_seg4; do for c in "p3p 65536 10"; do set -- $c
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SEG4', '$L', '$1', round(d['step_ms']['median'],3), round(d['roofline']['frac'],4), d['config']['launch'])"
done; done | tee gpurun_out/seg4_ab.log
