set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "p3p or cyclic7 or katsura or trifocal_ph or fourview_ph" > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
bash scripts/gpu_ab.sh lib_old lib lib_old lib
for L in lib_old lib lib_old lib; do for c in "p3p 1" "cyclic7ph 1" "katsura6 1"; do set -- $c; HC_LIB_PATH=paper_2112_03444_b200/$L/libhc.so timeout 300 python bench.py --config $1 --instances $2 --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('SMALL', '$L', '$1', round(d['step_ms']['median'],4))"; done; done | tee -a gpurun_out/ab.log
