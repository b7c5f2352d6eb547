python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "monodromy" > gpurun_out/pytest_mono.log 2>&1; tail -3 gpurun_out/pytest_mono.log
timeout 1200 python scripts/bench_monodromy.py > gpurun_out/bench_monodromy.jsonl 2> gpurun_out/bench_monodromy.err; cat gpurun_out/bench_monodromy.jsonl; tail -3 gpurun_out/bench_monodromy.err
