# Round-end style measurement: default bench line, reference arm, torchrun+NCCL gather path on 1 GPU,
# ncu launch list of the default command, one ncu --set full capture of the tracker kernel.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/gpu_info.csv
nproc > gpurun_out/host_cores.txt; lscpu | grep "Model name" >> gpurun_out/host_cores.txt
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 \
    bench.py --gpus 1 --instances 64 --warmup 3 --steps 1 --no-cpu-baseline --no-e2e --gather > gpurun_out/bench_torchrun_gather.json 2> gpurun_out/bench_torchrun_gather.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:hc_track_kernel -c 1 \
    -o gpurun_out/prof_trifocal python bench.py --instances 4 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > gpurun_out/ncu_trifocal.log 2>&1
tail -2 gpurun_out/ncu_trifocal.log
cat gpurun_out/bench_default.json gpurun_out/bench_reference.json gpurun_out/bench_torchrun_gather.json
tail -3 gpurun_out/bench_torchrun_gather.err
