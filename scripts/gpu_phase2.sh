export HC_LIB_PATH=paper_2112_03444_b200/lib_timing/libhc.so
for cfg in "p3p 1" "p3p 4096" "cyclic7ph 1" "trifocal 16"; do
  set -- $cfg
  timeout 300 python scripts/phase_timing.py $1 $2 > gpurun_out/phase_$1_$2.json 2> gpurun_out/phase_$1_$2.err
  python -c "
import json
d=json.load(open('gpurun_out/phase_$1_$2.json'))
print('$1 $2', round(d['cycles_per_iteration']), d['launch'], round(d['tracker_ms'],3))
for k,v in d['phases'].items(): print('   %-28s %8.0f %5.1f%%'%(k,v['cycles_per_iter'],100*v['share']))
"
done | tee gpurun_out/phase2.log
