set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -x -q -k "katsura or cyclic or fourview_ph or trifocal_ph or fivepoint_ph" > gpurun_out/pytest_gpu_quick.log 2>&1; tail -3 gpurun_out/pytest_gpu_quick.log
bash scripts/gpu_ab.sh lib_base lib lib_base lib
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
