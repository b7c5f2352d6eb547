# Session-2 evidence run: GPU tests, per-config bench lines (configs 1-3 + 5-point), traffic capture,
# ncu --set full of config 1 (katsura-6 in full).
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config katsura6 --steps 20 --warmup 3 > gpurun_out/bench_katsura6.json 2> gpurun_out/bench_katsura6.err
timeout 600 python bench.py --config cyclic7 --steps 20 --warmup 3 > gpurun_out/bench_cyclic7.json 2> gpurun_out/bench_cyclic7.err
timeout 600 python bench.py --config fourview --steps 5 --warmup 3 > gpurun_out/bench_fourview.json 2> gpurun_out/bench_fourview.err
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 5 --warmup 3 > gpurun_out/bench_fivepoint.json 2> gpurun_out/bench_fivepoint.err
for c in "katsura6 1" "cyclic7 1" "fourview 1024" "fivepoint 16384" "trifocal 1024"; do
  timeout 900 python scripts/record_traffic.py $c gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_katsura6 python bench.py --config katsura6 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_katsura6.log 2>&1
cat gpurun_out/bench_*.json gpurun_out/traffic.log
