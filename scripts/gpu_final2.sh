set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 3 > gpurun_out/bench_fivepoint.json 2> gpurun_out/bench_fivepoint.err
timeout 300 python bench.py --config katsura6 --steps 20 --warmup 3 > gpurun_out/bench_katsura6.json 2> gpurun_out/bench_katsura6.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29611 \
    bench.py --gpus 1 --total-instances 64 --warmup 3 --steps 1 --no-cpu-baseline --gather > gpurun_out/bench_torchrun_strong.json 2> gpurun_out/bench_torchrun_strong.err
tail -1 gpurun_out/bench_torchrun_strong.json | cut -c1-300
