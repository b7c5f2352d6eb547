python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 1200 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_default_k3.json 2> gpurun_out/bench_default_k3.err
timeout 600 python bench.py --config fourview --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_fourview_k20.json 2> gpurun_out/bench_fourview_k20.err
timeout 600 python bench.py --config p3p --instances 65536 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_p3p_k20.json 2> gpurun_out/bench_p3p_k20.err
for f in default_k3 fourview_k20 p3p_k20; do python -c "import json; d=json.loads(open('gpurun_out/bench_$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['step_ms'], d['roofline']['frac'], d['clocks'])"; done
