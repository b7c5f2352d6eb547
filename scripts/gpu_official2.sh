# Round-end evidence with the final kernel: GPU tests, smoke, official bench line + reference arm,
# per-config bench lines, launch list, ncu --set full of trifocal (4 instances) and katsura-6 (full),
# DRAM traffic of eco-12.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
for L in lib_r152w13 lib_r144w14; do HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 300 python bench.py --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ab_$L.json 2> gpurun_out/ab_$L.err; done
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 300 python bench.py --config katsura6 --steps 20 --warmup 3 > gpurun_out/bench_katsura6.json 2> gpurun_out/bench_katsura6.err
timeout 600 python bench.py --config cyclic7 --steps 20 --warmup 3 > gpurun_out/bench_cyclic7.json 2> gpurun_out/bench_cyclic7.err
timeout 600 python bench.py --config eco12 --steps 5 --warmup 3 > gpurun_out/bench_eco12.json 2> gpurun_out/bench_eco12.err
timeout 600 python bench.py --config fourview --steps 5 --warmup 3 > gpurun_out/bench_fourview.json 2> gpurun_out/bench_fourview.err
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 3 > gpurun_out/bench_fivepoint.json 2> gpurun_out/bench_fivepoint.err
timeout 600 python scripts/record_traffic.py eco12 1 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_trifocal python bench.py --instances 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_trifocal.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_katsura6 python bench.py --config katsura6 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_katsura6.log 2>&1
cat gpurun_out/bench_default.json gpurun_out/bench_reference.json
