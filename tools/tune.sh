#!/bin/bash
# usage: tools/tune.sh "lib1 lib2 ..." "c4:2:0 c5:1:0 ..."   (lib "main" = in-tree library)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for lib in $1; do
  if [ "$lib" = main ]; then L=""; else L="$PWD/tunelibs/lib_$lib.so"; fi
  for cfg in $2; do IFS=: read c m s <<< "$cfg"
    STENCIL_B200_LIB=$L timeout 300 python bench.py --config $c --fold-m $m --stages $s --steps 5 --warmup 3 --no-cpu-baseline 2>gpurun_out/tune_err.log | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
    print('%-5s %s m%s s%s  %8.1f GS/s  hbm %.3f fma %.3f  avg_ms %.4f  mhz %s' % ('$lib','$c','$m','$s', d['value'], r['hbm']['frac'], r['fma']['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz']))
except Exception as e: print('$lib $c m$m s$s FAILED', e)"
  done
done
