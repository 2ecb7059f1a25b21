# tb3d: parity tests, then C4 at the folded m=2 pass and the temporal block K=2,3,4
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb3d.py -q -x > gpurun_out/tb3_pytest.log 2>&1; echo "tb3d pytest rc=$?"; tail -15 gpurun_out/tb3_pytest.log
for c in "2 1" "2 2" "3 3" "4 4"; do set -- $c
  timeout 200 python bench.py --config c4 --fold-m $1 --stages $2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tb3_c4_m$1_s$2.json 2> gpurun_out/tb3_c4_m$1_s$2.err
  python3 -c "
import json
try:
    d=json.loads(open('gpurun_out/tb3_c4_m$1_s$2.json').read().strip().splitlines()[-1]); r=d['roofline']
    print('c4 m=$1 stages=$2', round(d['value'],1), 'hbm', round(r['hbm']['frac'],3), 'fma', round(r['fma']['frac'],3), r.get('kernel'), d['clocks'].get('reasons'))
except Exception as e: print('c4 m=$1 s=$2 ERR', open('gpurun_out/tb3_c4_m$1_s$2.err').read()[-400:])"
done
