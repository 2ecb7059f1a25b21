python tools/profile_sweep.py --config c2 --m 2 --stages 2 --sweeps 2 > gpurun_out/p_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 1 -o gpurun_out/prof_c2_m2s2 python tools/profile_sweep.py --config c2 --m 2 --stages 2 --sweeps 2 > gpurun_out/ncu.log 2>&1
echo "ncu rc=$?"
