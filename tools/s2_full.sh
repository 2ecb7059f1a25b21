#!/bin/bash
# Round-1 (session 2) full GPU pass: parity tests, bench lines for every config,
# the default bench's ncu launch list and one --set full capture of its top kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
for c in c1 c3 c4 c5; do
  timeout 400 python bench.py --config $c --fold-m 0 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "bench $c rc=$?"
done
timeout 300 python bench.py --config c2 --fold-m 0 --no-cpu-baseline > gpurun_out/bench_c2_all.json 2> gpurun_out/bench_c2_all.err; echo "bench c2 all rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_c2.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
python tools/profile_sweep.py --config c2 --m 4 --sweeps 2 > gpurun_out/p_c2m4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c2_m4 \
  python tools/profile_sweep.py --config c2 --m 4 --sweeps 2 > gpurun_out/ncu_full.log 2>&1; echo "ncu full rc=$?"
