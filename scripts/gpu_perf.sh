# exploratory perf sweep (not the official bench line)
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -2
timeout 300 python bench.py --config katsura6 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 300 python bench.py --config cyclic7 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config fourview --instances 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e
timeout 600 python bench.py --config trifocal --instances 64 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e
