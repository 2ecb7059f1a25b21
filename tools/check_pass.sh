#!/bin/bash
# GPU check of the committed state: parity tests, the default bench line and one
# line per config (fold_m auto) — no profiler.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 400 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for c in c2 c3 c4 c5; do
  timeout 400 python bench.py --config $c --headline-only --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
python - <<'PY'
import json
for c in ['default','c2','c3','c4','c5']:
    try:
        d=json.loads(open('gpurun_out/bench_%s.json'%c).read().strip().splitlines()[-1])
        r=d['roofline']
        print(c, d['config']['workload'], 'm', d['config']['fold_m'], 'value %.1f'%d['value'], 'frac %.3f (%s)'%(r['frac'], r['bound']), 'e2e %.1f'%d['e2e']['value'], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
        for k,v in d.get('configs',{}).items():
            print('   ', k, v.get('workload'), 'best_m', v.get('best_m'), 'value', round(v.get('value',0),1), 'frac', round(v.get('roofline',{}).get('frac',0),3))
    except Exception as e: print(c, 'ERR', e)
PY
