set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -q -k "fivepoint" 2>&1 | tail -5
timeout 600 python bench.py --config fivepoint --instances 16384 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_fivepoint.json
cat gpurun_out/bench_fivepoint.json
