python tools/profile_sweep.py --config c4 --m 2 --sweeps 2 > gpurun_out/p4_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 1 -o gpurun_out/prof_c4_m2 python tools/profile_sweep.py --config c4 --m 2 --sweeps 2 > gpurun_out/ncu_c4.log 2>&1
echo "ncu rc=$?"
for c in c2 c4; do timeout 300 python bench.py --config $c --fold-m 2 --steps 5 --warmup 2 --no-cpu-baseline 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.readlines()[-1]); r=d['roofline']
print('$c', 'm',d['config']['fold_m'], 'value %.1f'%d['value'], 'hbm %.3f'%r['hbm']['frac'], 'fma %.3f'%r['fma']['frac'], 'share %.3f'%r['kernel_share_of_step'], r['avg_launch_ms'])"; done
