# bench lines + dram traffic + ncu --set full of the kernels the 8/16-lane REDUX change affects
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
cp profiles/traffic.json gpurun_out/traffic.json
for c in "fourview 1024" "fivepoint 16384" "eco12 1"; do timeout 600 python scripts/record_traffic.py $c gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1; done
timeout 600 python bench.py --config eco12 --steps 5 --warmup 3 > gpurun_out/bench_eco12.json 2> gpurun_out/bench_eco12.err
timeout 600 python bench.py --config fourview --steps 5 --warmup 3 > gpurun_out/bench_fourview.json 2> gpurun_out/bench_fourview.err
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 3 > gpurun_out/bench_fivepoint.json 2> gpurun_out/bench_fivepoint.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_fourview64 python bench.py --config fourview --instances 64 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fourview64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_fivepoint1024 python bench.py --config fivepoint --instances 1024 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fivepoint1024.log 2>&1
tail -1 gpurun_out/ncu_fourview64.log gpurun_out/ncu_fivepoint1024.log
for f in eco12 fourview fivepoint; do cut -c1-300 gpurun_out/bench_$f.json; done
