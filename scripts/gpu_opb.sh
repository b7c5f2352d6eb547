python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for L in lib lib_opb8 lib lib_opb8; do
  HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 \
    --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('OPB', '$L', round(d['ms_per_step'],1), round(d['roofline']['frac'],4))"
done | tee gpurun_out/opb.log
