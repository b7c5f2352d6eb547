# ncu captures: full set on the tracker kernel (fourview, 64 instances) + launch list of a short bench
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
   -o gpurun_out/prof_fourview python bench.py --config fourview --instances 64 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fourview.log 2>&1
tail -5 gpurun_out/ncu_fourview.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_fourview.csv \
   python bench.py --config fourview --instances 256 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
tail -5 gpurun_out/launches_fourview.csv
