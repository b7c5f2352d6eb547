# A/B of CTA shapes for N <= 14 (4-view, eco-12, P3P) across prebuilt variant libraries.
for L in "$@"; do
  for cfg in "fourview 1024 3" "eco12 1 3" "p3p 65536 3"; do
    set -- $cfg
    HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps $3 --warmup 2 \
      --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ABLOW', '$L', '$1', round(d['step_ms']['median'],2), round(d['roofline']['frac'],4), d['config']['launch'])"
  done
done | tee -a gpurun_out/ab_low.log
