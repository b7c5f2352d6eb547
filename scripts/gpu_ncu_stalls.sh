# Stall-focused ncu capture (few passes) of the tracker kernel at a steadier batch size.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
CFG=${1:-trifocal}; B=${2:-16}; TAG=${3:-stalls}
timeout 1500 ncu --section WarpStateStats --section SchedulerStats --section Occupancy --section LaunchStats \
   --section SourceCounters --section ComputeWorkloadAnalysis --clock-control none --import-source on \
   -k regex:hc_track_kernel -c 1 -o gpurun_out/prof_$TAG python bench.py --config $CFG --instances $B --steps 1 --warmup 0 \
   --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
tail -2 gpurun_out/ncu_$TAG.log
