python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29601 \
    bench.py --gpus 1 --instances 64 --warmup 3 --steps 1 --no-cpu-baseline --gather > gpurun_out/bench_torchrun_gather.json 2> gpurun_out/bench_torchrun_gather.err
tail -2 gpurun_out/bench_torchrun_gather.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29602 \
    bench.py --impl reference --gpus 1 --steps 1 --warmup 0 > gpurun_out/bench_torchrun_reference.json 2> gpurun_out/bench_torchrun_reference.err
cat gpurun_out/bench_torchrun_gather.json gpurun_out/bench_torchrun_reference.json
