# tied-pivot zgesv test + refreshed repeated-step 4-view line
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
timeout 600 python -m pytest tests -m gpu -q -k "zgesv" > gpurun_out/pytest_zgesv.log 2>&1; tail -3 gpurun_out/pytest_zgesv.log
timeout 600 python bench.py --config fourview --steps 20 --warmup 3 > gpurun_out/bench_fourview_k20.json 2> gpurun_out/bench_fourview_k20.err
cut -c1-300 gpurun_out/bench_fourview_k20.json
