cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
prof() { # name lib config m stages
  L=""; [ "$2" != main ] && L="$PWD/tunelibs/lib_$2.so"
  STENCIL_B200_LIB=$L python tools/profile_sweep.py --config $3 --m $4 --stages $5 --sweeps 2 > gpurun_out/p_$1.log 2>&1 || { echo "$1 plain failed"; return; }
  STENCIL_B200_LIB=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 1 -c 1 -o gpurun_out/prof_$1 \
    python tools/profile_sweep.py --config $3 --m $4 --stages $5 --sweeps 2 > gpurun_out/ncu_$1.log 2>&1; echo "$1 ncu rc=$?"
}
prof t3c_c4m2 t3c c4 2 0
prof c3m4s2 main c3 4 2
prof c3m4s4 main c3 4 4
prof c2m4s2 main c2 4 2
