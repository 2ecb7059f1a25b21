cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "1d or dyadic or edge" 2>&1 | tail -2
for v in "8 64" "8 50" "8 34" "16 128" "16 64" "8 100"; do set -- $v
  echo "V=$1 HMAX=$2"; STENCIL_1D_V=$1 STENCIL_1D_HMAX=$2 bash tools/tune.sh main "c1:1:0 c1:2:0"; done
bash tools/s2_prof3.sh "c2m4s2 main c2 4 2" "c3m4s2r r2 c3 4 2"
