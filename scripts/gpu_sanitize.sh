# compute-sanitizer memcheck / racecheck / synccheck over small cases of every kernel path
set -x
python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
for tool in memcheck racecheck synccheck; do
  timeout 1800 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "== $tool exit $?"; tail -4 gpurun_out/sanitizer_$tool.log
done
bash scripts/gpu_ab_low.sh lib lib_low12 lib_low8 lib
timeout 900 python scripts/record_traffic.py trifocal 1024 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
timeout 600 python scripts/record_traffic.py fourview 1024 gpurun_out/traffic.json >> gpurun_out/traffic.log 2>&1
tail -2 gpurun_out/traffic.log
