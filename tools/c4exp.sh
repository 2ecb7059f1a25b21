cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/c4tune.sh main D E F main E
for n in main D E F; do
  if [ $n = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$n.so; fi
  timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:sweep_kernel -s 2 -c 1 python tools/profile_sweep.py --config c4 --m 2 --sweeps 3 > gpurun_out/c4ncu_$n.log 2>&1
  grep -E "dram__|gpu__time|lts__|warps_active" gpurun_out/c4ncu_$n.log | sed "s/^/$n /"
done
