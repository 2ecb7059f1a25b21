# Round-2 evidence pass of the committed state: GPU parity, the default bench line, the
# reference arm, the ncu launch list of the default run and --set full captures of the
# dominant kernel of every config.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f_pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/f_pytest_gpu.log
timeout 600 python bench.py > gpurun_out/f_bench_default.json 2> gpurun_out/f_bench_default.err; echo "bench rc=$?"
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/f_bench_reference.json 2> gpurun_out/f_bench_reference.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f_launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/f_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
full() { # name config m stages regex
  python tools/profile_sweep.py --config $2 --m $3 --stages $4 --sweeps 2 > gpurun_out/f_p_$1.log 2>&1 || { echo "$1 plain failed"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$5 -s 1 -c 1 -o gpurun_out/f_prof_$1 \
    python tools/profile_sweep.py --config $2 --m $3 --stages $4 --sweeps 2 > gpurun_out/f_ncu_$1.log 2>&1; echo "$1 ncu rc=$?"
}
full c2_k6_tb2d c2 6 6 tb2d
full c3_k8_tb2d c3 8 8 tb2d
full c4_m2_sweep c4 2 1 sweep_kernel
full c5_m1_sweep c5 1 1 sweep_kernel
python tools/resusage.py > gpurun_out/f_resusage.txt 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/f_bench_default.json').read().strip().splitlines()[-1])
r=d['roofline']
print('C2', d['config']['fold_m'], round(d['value'],1), 'frac', round(r['frac'],3), r['bound'], 'e2e', round(d['e2e']['value'],1), d['clocks'])
for k,v in d.get('configs',{}).items():
    print('  ', k, v.get('best_m'), round(v.get('value',0),1), 'frac', round(v.get('roofline',{}).get('frac',0),3), [(x['fold_m'], round(x['gstencil_s'],1)) for x in v.get('variants',[])])
PY
