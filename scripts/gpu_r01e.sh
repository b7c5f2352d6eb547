set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
bash scripts/gpu_ab.sh lib lib_r152w13 lib_r144w14 lib_r136w15 lib
