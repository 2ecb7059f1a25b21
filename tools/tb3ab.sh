# usage: bash tools/tb3ab.sh lib...  — tb3d parity per variant (bounded), then C4 K=4 (and K=3) A/B passes
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
good=""
for v in "$@"; do
  if STENCIL_B200_LIB=tunelibs/lib_$v.so timeout 200 python -m pytest tests/test_gpu_tb3d.py -q -x ${TB3_TESTK:+-k "$TB3_TESTK"} > gpurun_out/tb3ab_$v.log 2>&1; then good="$good $v"; echo "$v tests ok"; else echo "$v tests FAILED"; tail -3 gpurun_out/tb3ab_$v.log; fi
done
for pass in a b; do
  for name in main $good; do
    if [ "$name" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$name.so; fi
    for K in ${TB3_KS:-4 3}; do
      timeout 200 python bench.py --config c4 --fold-m $K --stages $K --steps 5 --headline-only --no-cpu-baseline > gpurun_out/t3_${name}_k${K}_$pass.json 2>/dev/null
      python3 -c "
import json
d=json.loads(open('gpurun_out/t3_${name}_k${K}_$pass.json').read().strip().splitlines()[-1]); print('$name K=$K $pass', round(d['value'],1), d['clocks'].get('reasons'))" 2>/dev/null || echo "$name K=$K $pass ERR"
    done
  done
done
