# quick perf triple (no tests)
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --config cyclic7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config fourview --instances 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e
