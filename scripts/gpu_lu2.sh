set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q -k "zgesv or katsura or cyclic or trifocal_ph or fivepoint_ph or fourview_ph or shape or lane" > gpurun_out/pytest_quick.log 2>&1; tail -3 gpurun_out/pytest_quick.log
bash scripts/gpu_ab.sh lib_old lib lib_old lib
