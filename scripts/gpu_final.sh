# Final evidence for round 1: GPU tests, smoke, official bench line + reference arm, every bench
# config, launch list, ncu --set full (trifocal 16 instances; cyclic-7 PH in the wide layout).
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 300 python bench.py --config katsura6 --steps 20 --warmup 3 > gpurun_out/bench_katsura6.json 2> gpurun_out/bench_katsura6.err
timeout 300 python bench.py --config cyclic7 --steps 20 --warmup 3 > gpurun_out/bench_cyclic7.json 2> gpurun_out/bench_cyclic7.err
timeout 300 python bench.py --config cyclic7ph --steps 20 --warmup 3 > gpurun_out/bench_cyclic7ph.json 2> gpurun_out/bench_cyclic7ph.err
timeout 600 python bench.py --config eco12 --steps 5 --warmup 3 > gpurun_out/bench_eco12.json 2> gpurun_out/bench_eco12.err
timeout 600 python bench.py --config fourview --steps 5 --warmup 3 > gpurun_out/bench_fourview.json 2> gpurun_out/bench_fourview.err
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 3 > gpurun_out/bench_fivepoint.json 2> gpurun_out/bench_fivepoint.err
timeout 600 python bench.py --config p3p --instances 65536 --steps 5 --warmup 3 > gpurun_out/bench_p3p.json 2> gpurun_out/bench_p3p.err
timeout 300 python bench.py --config p3p --instances 1 --steps 20 --warmup 3 > gpurun_out/bench_p3p_1.json 2> gpurun_out/bench_p3p_1.err
for c in "katsura6 1" "cyclic7ph 1" "p3p 1"; do timeout 300 python scripts/record_traffic.py $c gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_under_ncu.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_trifocal16 python bench.py --instances 16 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_trifocal16.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_cyclic7ph python bench.py --config cyclic7ph --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cyclic7ph.log 2>&1
cat gpurun_out/bench_default.json
