for name in "$@"; do
  if [ "$name" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$name.so; fi
  timeout 120 python bench.py --config c5 --fold-m 1 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/c5_${name}.json 2>gpurun_out/c5_${name}.err
  timeout 120 python bench.py --config c4 --fold-m 2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/c4_${name}.json 2>gpurun_out/c4_${name}.err
done
for f in gpurun_out/c5_*.json gpurun_out/c4_*.json; do python -c "
import json,sys
try:
    d=json.loads(open('$f').read().strip().splitlines()[-1]); r=d['roofline']
    print('$f', round(d['value'],1), 'hbm', round(r['hbm']['frac'],3), 'fma', round(r['fma']['frac'],3), d['clocks'].get('reasons'))
except Exception as e: print('$f ERR', open('$f'.replace('.json','.err')).read()[-200:])
"; done
