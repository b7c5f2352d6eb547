# ncu full-set captures of the tracker kernel (usage: bash scripts/gpu_ncu.sh <config> <instances> <tag>)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
CFG=${1:-trifocal}; B=${2:-4}; TAG=${3:-$CFG}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
   -o gpurun_out/prof_$TAG python bench.py --config $CFG --instances $B --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
tail -3 gpurun_out/ncu_$TAG.log
