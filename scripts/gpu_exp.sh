set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for W in 16 12 8 4; do HC_TRACKER_WARPS=$W timeout 300 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e; done
