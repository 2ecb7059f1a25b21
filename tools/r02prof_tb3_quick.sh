# one --set full capture of the C4 temporal block (K = 4) for source-level analysis
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 400 ncu --set full --import-source on --clock-control none -k regex:tb3d -s 3 -c 1 -o gpurun_out/r02_c4_tb3 python bench.py --config c4 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1; echo "c4 full rc=$?"
