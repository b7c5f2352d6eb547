python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_p3p1 python bench.py --config p3p --instances 1 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_p3p1.log 2>&1
tail -2 gpurun_out/ncu_p3p1.log
