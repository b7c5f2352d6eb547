# dev cycle: build, smoke, GPU tests (fast subset unless FULL=1), exploratory perf lines
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
if [ -n "$FULL" ]; then K=""; else K="-k not(config4_full)"; fi
timeout 900 python -m pytest tests -m gpu -x -q "$K" 2>&1 | tail -15
timeout 300 python bench.py --config cyclic7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config fourview --instances 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
