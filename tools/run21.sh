timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for cfg in "c2 2 1" "c2 4 1" "c2 4 2" "c3 2 1" "c3 4 1" "c3 4 2" "c4 1 1" "c4 2 1" "c4 2 2" "c5 1 1" "c5 2 2"; do set -- $cfg
timeout 300 python bench.py --config $1 --fold-m $2 --stages $3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$1 m$2 s$3', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"; done
