timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
python bench.py > gpurun_out/bench_plain.json 2> gpurun_out/bench_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv python bench.py > gpurun_out/bench_ncu.log 2>&1
echo "ncu1 rc=$?"
python tools/profile_sweep.py --config c2 --m 2 --sweeps 2 > gpurun_out/p2_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 1 -o gpurun_out/prof_c2_m2_r1 python tools/profile_sweep.py --config c2 --m 2 --sweeps 2 > gpurun_out/ncu_c2.log 2>&1
echo "ncu2 rc=$?"
cat gpurun_out/bench_plain.json
for c in c1 c3 c4 c5; do timeout 300 python bench.py --config $c --fold-m 0 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$c.json 2>&1; tail -c 600 gpurun_out/bench_$c.json; echo; done
