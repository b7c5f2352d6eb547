# Lane-layout A/B (throughput vs wide latency layout) on the single-instance TD configs + GPU tests.
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "lane or katsura or cyclic or eco or shape or smoke" > gpurun_out/pytest_lanes.log 2>&1; tail -3 gpurun_out/pytest_lanes.log
for cfg in "katsura6 20" "cyclic7 20" "eco12 3"; do
  set -- $cfg
  for mode in narrow wide; do
    HC_LANES=$mode timeout 600 python bench.py --config $1 --steps $2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
      python -c "import json,sys; d=json.loads(sys.stdin.read()); print('LANES', '$1', '$mode', round(d['step_ms']['median'],3), round(d['roofline']['frac'],4), d['config']['launch'])"
  done
done | tee gpurun_out/lanes_ab.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
