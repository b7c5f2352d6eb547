set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "cyclic7 or lane" > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
timeout 300 python bench.py --config cyclic7ph --steps 20 --warmup 3 > gpurun_out/bench_cyclic7ph.json 2> gpurun_out/bench_cyclic7ph.err
HC_LANES=narrow timeout 300 python bench.py --config cyclic7ph --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cyclic7ph_narrow.json 2>&1
timeout 300 python bench.py --config katsura6 --steps 20 --warmup 3 > gpurun_out/bench_katsura6.json 2> gpurun_out/bench_katsura6.err
timeout 300 python bench.py --config cyclic7 --steps 20 --warmup 3 > gpurun_out/bench_cyclic7.json 2> gpurun_out/bench_cyclic7.err
for c in cyclic7ph katsura6 cyclic7; do timeout 300 python scripts/record_traffic.py $c 1 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1; done
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
