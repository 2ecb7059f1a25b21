cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
./tools/lat_probe
bash tools/tune.sh "v1 v2 v3 n4 v4" "c2:4:2 c2:2:0 c2:4:0 c3:4:2 c3:4:0"
