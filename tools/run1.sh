set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
./tools/fma_peak > gpurun_out/fma_peak.json 2>&1; cat gpurun_out/fma_peak.json
for c in c2 c1 c3 c4 c5; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo "rc=$?"; cat gpurun_out/bench_$c.json | head -c 3000; echo; tail -3 gpurun_out/bench_$c.err
done
