for lib in tunelibs/lib_old.so tunelibs/lib_new2.so; do for cfg in "c4 1 1" "c4 2 1" "c5 1 1"; do set -- $cfg
STENCIL_B200_LIB=$PWD/$lib timeout 300 python bench.py --config $1 --fold-m $2 --stages $3 --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$lib $1 m$2 s$3', 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'avg_ms %.4f'%r['avg_launch_ms'], d['clocks']['sm_mhz'])"; done; done
