# quick A/B: build, a parity subset, perf lines for 4-view and trifocal
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q -k "fourview or katsura or cyclic or shape" 2>&1 | tail -3
timeout 600 python bench.py --config fourview --instances 1024 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('FOURVIEW', d['ms_per_step'], d['roofline']['frac'])"
timeout 600 python bench.py --config trifocal --instances 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TRIFOCAL', d['ms_per_step'], d['roofline']['frac'])"
