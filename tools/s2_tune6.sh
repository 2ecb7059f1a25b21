cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/tune.sh "main n3 n3p n2 n4" "c2:4:2 c2:2:0 c3:2:0 c3:4:2"
bash tools/tune.sh "main h1" "c2:4:0 c3:4:0"
bash tools/tune.sh "q3 q4" "c4:2:0 c4:1:0 c5:1:0 c5:2:0"
