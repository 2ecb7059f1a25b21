cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
bash tools/tune.sh "main t3b t3c t3d t3e" "c4:2:0 c4:1:0 c4:2:2 c5:1:0 c5:2:0 c5:2:1"
bash tools/tune.sh "main t2a t2b" "c2:4:0 c2:2:0 c2:4:2 c3:2:0 c3:4:0 c3:4:2"
bash tools/tune.sh "main" "c1:1:0 c1:2:0"
