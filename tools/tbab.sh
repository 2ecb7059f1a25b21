# usage: bash tools/tbab.sh lib...  — tb2d parity tests per variant (bounded), then A/B passes of
# the variants whose tests passed against the in-tree library
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
good=""
for v in "$@"; do
  if STENCIL_B200_LIB=tunelibs/lib_$v.so timeout 120 python -m pytest tests/test_gpu_tb.py -q -x > gpurun_out/tbab_$v.log 2>&1; then good="$good $v"; echo "$v tests ok"; else echo "$v tests FAILED"; tail -3 gpurun_out/tbab_$v.log; fi
done
[ -z "$good" ] && exit 0
bash tools/tbtune.sh -p a main $good > /dev/null
bash tools/tbtune.sh -p b $(echo $good | tr ' ' '\n' | tac) main
