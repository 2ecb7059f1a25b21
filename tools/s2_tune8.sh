cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -2
for v in w1 w2; do STENCIL_B200_LIB=$PWD/tunelibs/lib_$v.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "2d or dyadic or edge" 2>&1 | tail -1; done
bash tools/tune.sh "main w1 w2 w3 w4" "c2:4:2 c2:2:0 c2:4:0 c3:2:0 c3:4:2 c3:4:0"
