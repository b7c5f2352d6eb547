set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for B in 16 256 1024; do timeout 900 python bench.py --config trifocal --instances $B --steps 1 --warmup 1 --no-cpu-baseline --no-e2e; done
