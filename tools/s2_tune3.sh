cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/tune.sh "main r2 r2a" "c2:4:0 c2:4:2 c2:2:0 c3:2:0 c3:4:2 c3:4:4"
bash tools/tune.sh "r3 r3c" "c4:2:0 c4:1:0 c5:1:0 c5:2:0"
python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/p_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:onchip1d -c 1 -o gpurun_out/prof_c1_m2b \
    python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/ncu_c1.log 2>&1; echo "c1 ncu rc=$?"
