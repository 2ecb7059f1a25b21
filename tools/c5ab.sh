# usage: bash tools/c5ab.sh lib...  — box tb3d parity per variant, then C5 m=2 (K=2) A/B passes
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
good=""
for v in "$@"; do
  if STENCIL_B200_LIB=tunelibs/lib_$v.so timeout 300 python -m pytest tests/test_gpu_tb3d.py -q -x -k "box and not fullsize" > gpurun_out/c5ab_$v.log 2>&1; then good="$good $v"; echo "$v tests ok"; else echo "$v tests FAILED"; tail -3 gpurun_out/c5ab_$v.log; fi
done
for pass in a b; do
  for name in main $good; do
    if [ "$name" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$name.so; fi
    timeout 200 python bench.py --config c5 --fold-m 2 --stages 2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/c5ab_${name}_$pass.json 2>/dev/null
    python3 -c "
import json
d=json.loads(open('gpurun_out/c5ab_${name}_$pass.json').read().strip().splitlines()[-1]); print('$name $pass', round(d['value'],1), d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))" 2>/dev/null || echo "$name $pass ERR"
  done
done
