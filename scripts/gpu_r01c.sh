set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
bash scripts/gpu_ab.sh lib lib_nopipe lib_w16 lib_w16np
NO_FV=1 bash scripts/gpu_phase.sh
bash scripts/gpu_r01b.sh
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_trifocal python bench.py --instances 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_trifocal.log 2>&1
