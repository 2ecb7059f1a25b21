#!/bin/bash
# ncu --set full of the sweep kernel for the weak variants (C4 m=2, C3 m=4, C5 m=2) and the 1D kernel.
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
prof() { # name config m stages kernel-regex
  python tools/profile_sweep.py --config $2 --m $3 --stages $4 --sweeps 2 > gpurun_out/p_$1.log 2>&1 || { echo "$1 plain failed"; return; }
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$5 -s 1 -c 1 -o gpurun_out/prof_$1 \
    python tools/profile_sweep.py --config $2 --m $3 --stages $4 --sweeps 2 > gpurun_out/ncu_$1.log 2>&1; echo "$1 ncu rc=$?"
}
prof c4_m2 c4 2 0 sweep_kernel
prof c3_m4 c3 4 0 sweep_kernel
prof c5_m2 c5 2 0 sweep_kernel
prof c5_m1 c5 1 0 sweep_kernel
python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/p_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:onchip1d -c 1 -o gpurun_out/prof_c1_m2 \
    python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/ncu_c1.log 2>&1; echo "c1 ncu rc=$?"
