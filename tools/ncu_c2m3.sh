cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
python tools/profile_sweep.py --config c2 --m 3 --sweeps 2 > gpurun_out/p_c2m3.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c2_m3 \
  python tools/profile_sweep.py --config c2 --m 3 --sweeps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
