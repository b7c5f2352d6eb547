# per-phase cycle breakdown (experiment build), trifocal and 4-view
set -x
HCB_VARIANT=timing python paper_2112_03444_b200/build.py > /dev/null 2>&1
export HC_LIB_PATH=paper_2112_03444_b200/lib_timing/libhc.so
timeout 300 python scripts/phase_timing.py trifocal ${TRI_B:-32} > gpurun_out/phase_trifocal.json
[ -n "$NO_FV" ] || timeout 300 python scripts/phase_timing.py fourview 256 > gpurun_out/phase_fourview.json
python -c "
import json
for f in ['gpurun_out/phase_trifocal.json','gpurun_out/phase_fourview.json']:
    try: d=json.load(open(f))
    except Exception: continue
    print(f, d['cycles_per_iteration'], d['launch'], d['tracker_ms'])
    for k,v in d['phases'].items(): print('   %-28s %8.0f %5.1f%%'%(k,v['cycles_per_iter'],100*v['share']))
"
