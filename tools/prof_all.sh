#!/bin/bash
# ncu --set full of the dominant kernel of C3 (m=2), C5 (m=1) and C1 (m=2).
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
bash tools/prof.sh "c3m2 main c3 2 0" "c5m1 main c5 1 0"
python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/p_c1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:onchip1d -c 1 -o gpurun_out/prof_c1m2 \
    python tools/profile_sweep.py --config c1 --m 2 --sweeps 50 > gpurun_out/ncu_c1.log 2>&1; echo "c1 ncu rc=$?"
