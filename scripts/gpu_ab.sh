# A/B of prebuilt variant libraries (lib_<name>/libhc.so): trifocal x64 and 4-view x1024 step times.
# usage: bash scripts/gpu_ab.sh lib lib_nopipe ...
for L in "$@"; do
  for cfg in "trifocal 64" "fourview 1024"; do
    set -- $cfg
    HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 600 python bench.py --config $1 --instances $2 --steps 1 --warmup 1 \
      --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('AB', '$L', '$1', round(d['ms_per_step'],1), round(d['roofline']['frac'],4), d['config']['launch'])"
  done
done | tee -a gpurun_out/ab.log
