#!/usr/bin/env bash
# All GPU-box jobs of this repo, run under gpurun from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu.sh <job> [args] ...'
# Jobs (several may be chained in one call: bash scripts/gpu.sh tests bench ...):
#   tests                      build + smoke() + the full `pytest -m gpu` suite
#   bench                      the default bench line, the reference (oracle) arm, torchrun+NCCL gather on 1 GPU
#   launches                   ncu launch list of the default bench command (gpu__time_duration per launch)
#   ncu CFG B TAG              one ncu --set full capture of the tracker kernel (bench --config CFG --instances B)
#   ab NAME=DEFINES ...        A/B of variant libraries built HERE from the committed sources: each NAME is built
#                              with HCB_VARIANT=NAME HCB_DEFINES="DEFINES" (comma-separated defines) into
#                              lib_NAME/; NAME=base is the product library, NAME=@dir a prebuilt dir/libhc.so (e.g. the
#                              previous commit's, built locally into abl/); the AB_CFGS step times
#   phase                      per-phase cycle breakdown (HCB_VARIANT=timing build), trifocal and 4-view
#   sanitize                   compute-sanitizer memcheck / racecheck / synccheck over small cases of every path
#                              (closed on the round-2 GPU pool: "runs under it have left GPUs needing a reset")
#   traffic                    DRAM bytes per launch (ncu) for trifocal and 4-view
#   zgesv                      Fig. 3 re-run (N1): fused batched LU vs cuBLAS getrf/getrsBatched
#   env VAR=VAL ...            the AB_CFGS configs with the product library under each environment setting
#   warps                      trifocal x64 step time at 4, 8, 12 warps per CTA (HC_TRACKER_WARPS; latency hiding)
set -u
mkdir -p gpurun_out
build() { python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1; }
AB_CFGS=${AB_CFGS:-"trifocal:64 fourview:1024"}
build
while [ $# -gt 0 ]; do
  job=$1; shift
  case $job in
    tests)
      timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
      timeout 2400 python -m pytest tests -m gpu -q ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log ;;
    bench)
      nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
      { nproc; lscpu | grep "Model name"; } > gpurun_out/host_cores.txt
      timeout 1500 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
      timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
      timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 \
        bench.py --gpus 1 --instances 64 --warmup 3 --steps 1 --no-cpu-baseline --no-e2e --gather \
        > gpurun_out/bench_torchrun_gather.json 2> gpurun_out/bench_torchrun_gather.err
      cat gpurun_out/bench_default.json gpurun_out/bench_reference.json gpurun_out/bench_torchrun_gather.json ;;
    launches)
      timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
        python bench.py --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1; tail -2 gpurun_out/launches_default.csv ;;
    ncu)
      CFG=$1; B=$2; TAG=$3; shift 3
      timeout 1500 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
        -o gpurun_out/prof_$TAG python bench.py --config $CFG --instances $B --steps 1 --warmup 0 --no-cpu-baseline --no-e2e \
        > gpurun_out/ncu_$TAG.log 2>&1; tail -2 gpurun_out/ncu_$TAG.log ;;
    ab)
      libs=()
      while [ $# -gt 0 ] && [[ $1 == *=* ]]; do
        name=${1%%=*}; defs=${1#*=}; shift
        if [ "$name" = base ]; then libs+=(lib); continue; fi
        if [[ $defs == @* ]]; then libs+=("../${defs#@}"); continue; fi   # NAME=@dir: a prebuilt dir/libhc.so (repo-relative)
        HCB_VARIANT=$name HCB_DEFINES="${defs//,/ }" python paper_2112_03444_b200/build.py > /dev/null || echo "build $name failed"
        libs+=(lib_$name)
      done
      for round in 1 2; do
        for L in "${libs[@]}"; do
          for cfg in $AB_CFGS; do
            c=${cfg%%:*}; b=${cfg#*:}
            HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 900 python bench.py --config $c --instances $b --steps 1 --warmup 1 \
              --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('AB', $round, '$L', '$c', round(d['ms_per_step'],2), round(d['roofline']['frac'],4), round(d['roofline']['tracker_ms_per_launch'],3), d['config']['launch'])"
          done
        done
      done | tee -a gpurun_out/ab.log ;;
    phase)
      HCB_VARIANT=timing python paper_2112_03444_b200/build.py > /dev/null 2>&1
      HC_LIB_PATH=paper_2112_03444_b200/lib_timing/libhc.so timeout 600 python scripts/phase_timing.py trifocal ${TRI_B:-16} > gpurun_out/phase_trifocal.json
      HC_LIB_PATH=paper_2112_03444_b200/lib_timing/libhc.so timeout 600 python scripts/phase_timing.py fourview 256 > gpurun_out/phase_fourview.json
      python scripts/phase_timing.py --print gpurun_out/phase_trifocal.json gpurun_out/phase_fourview.json ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
        echo "== $tool exit $?"; tail -4 gpurun_out/sanitizer_$tool.log
      done ;;
    traffic)
      timeout 900 python scripts/record_traffic.py trifocal ${TRAFFIC_TRI_B:-1024} gpurun_out/traffic.json --dram-only >> gpurun_out/traffic.log 2>&1
      timeout 600 python scripts/record_traffic.py fourview 1024 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
      tail -2 gpurun_out/traffic.log ;;
    traffic_ab)   # DRAM bytes of trifocal x256 with the small per-track outputs / the x output not written
      HCB_VARIANT=out1 HCB_DEFINES="HCB_OUT_EXPERIMENT=1" python paper_2112_03444_b200/build.py > /dev/null
      HCB_VARIANT=out2 HCB_DEFINES="HCB_OUT_EXPERIMENT=2" python paper_2112_03444_b200/build.py > /dev/null
      for v in ${TRAFFIC_LIBS:-lib lib_out1 lib_out2}; do
        HC_LIB_PATH=paper_2112_03444_b200/$v/libhc.so timeout 900 python scripts/record_traffic.py trifocal 256 gpurun_out/traffic_$v.json --dram-only \
          >> gpurun_out/traffic_ab.log 2>&1
        python -c "import json; d=json.load(open('gpurun_out/traffic_$v.json')); v=list(d.values())[0]; print('TRAFFIC', '$v', v['read'] / v['tracks'], v['write'] / v['tracks'])"
      done | tee -a gpurun_out/traffic_ab.log ;;
    zgesv)
      timeout 900 python scripts/bench_zgesv.py > gpurun_out/zgesv_fig3.jsonl 2> gpurun_out/zgesv.err; tail -5 gpurun_out/zgesv_fig3.jsonl ;;
    env)   # env VAR=VALUE ... : the AB_CFGS configs with the product library, once per setting
      kvs=()
      while [ $# -gt 0 ] && [[ $1 == *=* ]]; do kvs+=("$1"); shift; done
      for kv in "${kvs[@]}"; do
        for cfg in $AB_CFGS; do
          c=${cfg%%:*}; b=${cfg#*:}
          env ${kv%%=*}=${kv#*=} timeout 900 python bench.py --config $c --instances $b --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
            2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ENV', '$kv', '$c', round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['roofline']['tracker_ms_per_launch'], d['clocks']['sm_mhz'])"
        done
      done | tee -a gpurun_out/env.log ;;
    warps)
      for w in 4 8 12; do
        HC_TRACKER_WARPS=$w timeout 900 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e \
          2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('WARPS', $w, round(d['ms_per_step'],2), round(d['roofline']['frac'],4), d['config']['launch'])"
      done | tee -a gpurun_out/warps.log ;;
    *) echo "unknown job $job"; exit 2 ;;
  esac
done
