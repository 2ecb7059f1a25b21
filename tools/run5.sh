timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for c in c2 c3 c4 c5; do timeout 300 python bench.py --config $c --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$c', 'm',d['config']['fold_m'], 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'share %.3f'%r['kernel_share_of_step'], [ (v['fold_m'], round(v['gstencil_s'],1)) for v in d['variants']], d['clocks']['sm_mhz'])"; done
