# A/B of tb2d variants + one ncu --set full of the in-tree C2 K=8 temporal block
cd "${GRAFT_REPO_ROOT:-/root/repo}"; mkdir -p gpurun_out
for v in "$@"; do STENCIL_B200_LIB=tunelibs/lib_$v.so timeout 300 python -m pytest tests/test_gpu_tb.py -q -x 2>&1 | tail -1 | sed "s/^/$v tests: /"; done
bash tools/tbtune.sh -p a main "$@" > /dev/null
bash tools/tbtune.sh -p b "$@" main
python tools/profile_sweep.py --config c2 --m 8 --stages 8 --sweeps 2 > gpurun_out/p_tb.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tb2d -s 1 -c 1 -o gpurun_out/prof_tb_c2 \
  python tools/profile_sweep.py --config c2 --m 8 --stages 8 --sweeps 2 > gpurun_out/ncu_tb.log 2>&1; echo "ncu rc=$?"
