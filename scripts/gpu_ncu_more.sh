python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_fourview64 python bench.py --config fourview --instances 64 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fourview64.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_fivepoint1024 python bench.py --config fivepoint --instances 1024 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fivepoint1024.log 2>&1
tail -1 gpurun_out/ncu_fourview64.log gpurun_out/ncu_fivepoint1024.log
