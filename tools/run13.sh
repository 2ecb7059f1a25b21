timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3
for s in 1 2 4; do timeout 300 python bench.py --config c2 --fold-m 4 --stages $s --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('c2 m4 s$s', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"; done
for s in 1 2 4; do timeout 300 python bench.py --config c3 --fold-m 4 --stages $s --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('c3 m4 s$s', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"; done
timeout 300 python bench.py --config c2 --fold-m 2 --stages 2 --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('c2 m2 s2', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"
