for v in new2; do
STENCIL_B200_LIB=$PWD/tunelibs/lib_$v.so python tools/profile_sweep.py --config c4 --m 1 --sweeps 2 > gpurun_out/p_$v.log 2>&1 && \
STENCIL_B200_LIB=$PWD/tunelibs/lib_$v.so ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 0 -c 1 -o gpurun_out/prof_c4m1_$v python tools/profile_sweep.py --config c4 --m 1 --sweeps 2 > gpurun_out/ncu_$v.log 2>&1
echo "$v rc=$?"
done
