# ncu evidence for the 3D box temporal block (C5, fold_m = 2 as K = 2 single steps per round trip)
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python bench.py --config c5 --headline-only --no-cpu-baseline > gpurun_out/r02_c5k2_bench.json 2> gpurun_out/r02_c5k2_bench.err; echo "c5 k2 bench rc=$?"
timeout 400 ncu --set full --import-source on --clock-control none -k regex:tb3d -s 3 -c 1 -o gpurun_out/r02_c5_tb3 python bench.py --config c5 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c5k2.log 2>&1; echo "c5 k2 full rc=$?"
ls -la gpurun_out/r02_c5*
