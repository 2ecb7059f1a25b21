# ncu evidence for the 3D temporal block (C4, K = fold_m = 4) and the C5 pass:
# launch list of the C4 bench command, one full capture of each top kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
timeout 300 python bench.py --config c4 --headline-only --no-cpu-baseline > gpurun_out/r02_c4_bench.json 2> gpurun_out/r02_c4_bench.err; echo "c4 bench rc=$?"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_c4_launches.csv python bench.py --config c4 --steps 2 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c4_launch.log 2>&1; echo "launch list rc=$?"
timeout 400 ncu --set full --import-source on --clock-control none -k regex:tb3d -s 3 -c 1 -o gpurun_out/r02_c4_tb3 python bench.py --config c4 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/r02_ncu_c4.log 2>&1; echo "c4 full rc=$?"
ls -la gpurun_out/r02_c4*
