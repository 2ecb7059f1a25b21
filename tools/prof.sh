cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
prof() { # name lib config m stages regex
  L=""; [ "$2" != main ] && L="$PWD/tunelibs/lib_$2.so"
  STENCIL_B200_LIB=$L python tools/profile_sweep.py --config $3 --m $4 --stages $5 --sweeps 2 > gpurun_out/p_$1.log 2>&1 || { echo "$1 plain failed"; return; }
  STENCIL_B200_LIB=$L timeout 600 ncu --set full --clock-control none --import-source on -k regex:${6:-sweep_kernel} -s 1 -c 1 -o gpurun_out/prof_$1 \
    python tools/profile_sweep.py --config $3 --m $4 --stages $5 --sweeps 2 > gpurun_out/ncu_$1.log 2>&1; echo "$1 ncu rc=$?"
}
for a in "$@"; do prof $a; done
bash tools/tune.sh main "c1:2:0 c1:1:0"
