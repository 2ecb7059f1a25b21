for lib in tunelibs/*.so; do for c in c4 c5; do for m in 1 2; do STENCIL_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $c --fold-m $m --steps 4 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$lib $c $m', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"; done; done; done
