python tools/profile_sweep.py --config c2 --m 2 --sweeps 3 > gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_c2_m2 python tools/profile_sweep.py --config c2 --m 2 --sweeps 3 > gpurun_out/ncu_c2.log 2>&1
echo "ncu rc=$?"
for m in 4; do for s in 1 2; do timeout 300 python bench.py --config c2 --fold-m $m --stages $s --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print($m,$s,d['value'], d['roofline']['hbm'], d['roofline']['fma'])"; done; done
for s in 1 2; do timeout 300 python bench.py --config c3 --fold-m 4 --stages $s --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('c3',$s,d['value'], d['roofline']['hbm'], d['roofline']['fma'])"; done
