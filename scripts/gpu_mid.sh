python -c "import __graft_entry__ as g; g.build()" 2>&1 | tail -1
HC_LANES=mid timeout 600 python -m pytest tests -m gpu -x -q -k "katsura6_parity or cyclic7_parity or cyclic7_monodromy_ph" > gpurun_out/pytest_mid.log 2>&1; tail -2 gpurun_out/pytest_mid.log
for mode in narrow mid wide mid; do for c in "katsura6 1 20" "cyclic7 1 20" "cyclic7ph 1 20" "p3p 1 20" "p3p 65536 3"; do set -- $c
  HC_LANES=$mode timeout 300 python bench.py --config $1 --instances $2 --steps $3 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.read()); print('MID', '$mode', '$1', '$2', round(d['step_ms']['median'],4), d['config']['launch']['lanes_per_track'])"
done; done | tee gpurun_out/mid_ab.log
