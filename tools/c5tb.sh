# 3D box temporal block: parity tests (box), then C5 at m=1 and m=2 (stages 2 = tb3d box), two passes
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_tb3d.py -q -x -k "box" > gpurun_out/c5tb_pytest.log 2>&1; echo "tb3d box pytest rc=$?"; tail -5 gpurun_out/c5tb_pytest.log
for pass in a b; do
for c in "1 0" "2 2"; do set -- $c
  timeout 300 python bench.py --config c5 --fold-m $1 --stages $2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/c5tb_m$1_$pass.json 2> gpurun_out/c5tb_m$1_$pass.err
  python3 -c "
import json
try:
    d=json.loads(open('gpurun_out/c5tb_m$1_$pass.json').read().strip().splitlines()[-1]); r=d['roofline']
    print('c5 m=$1 stages=$2 $pass', round(d['value'],1), 'hbm', round(r['hbm']['frac'],3), 'fma', round(r['fma']['frac'],3), r.get('kernel'), d['clocks'])
except Exception as e: print('c5 m=$1 ERR', open('gpurun_out/c5tb_m$1_$pass.err').read()[-600:])"
done
done
