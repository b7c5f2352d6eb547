set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "p3p or cyclic7_monodromy" > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
timeout 600 python bench.py --config p3p --instances 65536 --steps 5 --warmup 3 > gpurun_out/bench_p3p.json 2> gpurun_out/bench_p3p.err
timeout 300 python bench.py --config p3p --instances 1 --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_p3p_1.json 2> gpurun_out/bench_p3p_1.err
timeout 600 python scripts/record_traffic.py p3p 65536 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
