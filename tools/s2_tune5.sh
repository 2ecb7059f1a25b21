cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash tools/tune.sh "main p2 p2a" "c2:4:0 c2:4:2 c2:2:0 c3:2:0 c3:4:2"
bash tools/tune.sh "main p3 p3c t3c b1" "c4:2:0 c4:1:0 c5:1:0 c5:2:0"
