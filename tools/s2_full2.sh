#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for c in c1 c2 c3 c4 c5; do
  timeout 400 python bench.py --config $c --fold-m 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
python - <<'PY'
import json
for c in ['default','c1','c2','c3','c4','c5']:
    try:
        d=json.loads(open('gpurun_out/bench_%s.json'%c).read().strip().splitlines()[-1]); r=d['roofline']
        print(c, d['config']['workload'], 'm', d['config']['fold_m'], 'value %.1f'%d['value'], 'frac %.3f (%s)'%(r['frac'], r['bound']), 'hbm %.3f fma %.3f'%(r['hbm']['frac'], r['fma']['frac']), 'e2e %.1f'%d['e2e']['value'], [(v['fold_m'], round(v['gstencil_s'],1)) for v in d['variants']], d['clocks'].get('sm_mhz'))
    except Exception as e: print(c, 'ERR', e)
PY
