#!/bin/bash
# Full GPU pass for the committed state: parity tests, one bench line per config
# (all fold_m), the default bench line, its ncu launch list and a --set full
# capture of the default's dominant kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for c in c1 c2 c3 c4 c5 c3u; do
  timeout 400 python bench.py --config $c --fold-m 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/profile_sweep.py --config c2 --m 3 --sweeps 2 > gpurun_out/p_c2m3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c2_m3 \
  python tools/profile_sweep.py --config c2 --m 3 --sweeps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
python tools/profile_sweep.py --config c4 --m 2 --sweeps 2 > gpurun_out/p_c4m2.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c4_m2 \
  python tools/profile_sweep.py --config c4 --m 2 --sweeps 2 > gpurun_out/ncu_full_c4.log 2>&1; echo "ncu full c4 rc=$?"
python - <<'PY'
import json
for c in ['default','c1','c2','c3','c4','c5','c3u','reference']:
    try:
        d=json.loads(open('gpurun_out/bench_%s.json'%c).read().strip().splitlines()[-1])
        if c=='reference': print(c, d['value'], d['config']); continue
        r=d['roofline']
        print(c, d['config']['workload'], 'm', d['config']['fold_m'], 'value %.1f'%d['value'], 'frac %.3f (%s)'%(r['frac'], r['bound']), 'hbm %.3f fma %.3f'%(r['hbm']['frac'], r['fma']['frac']), 'e2e %.1f'%d['e2e']['value'], [(v['fold_m'], round(v['gstencil_s'],1)) for v in d['variants']], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))
    except Exception as e: print(c, 'ERR', e)
PY
