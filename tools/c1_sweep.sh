cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "0 0" "16 128" "16 64" "0 34" "0 26"; do set -- $v
  if [ $1 = 0 ]; then unset STENCIL_1D_V; else export STENCIL_1D_V=$1; fi
  if [ $2 = 0 ]; then unset STENCIL_1D_HMAX; else export STENCIL_1D_HMAX=$2; fi
  timeout 300 python bench.py --config c1 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('V=$1 HMAX=$2', round(d['value'],1), d['ms_per_step'], d['roofline']['launches'])"
done
