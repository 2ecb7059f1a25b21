export STENCIL_B200_LIB=tunelibs/lib_probe.so
CUDA_LAUNCH_BLOCKING=1 timeout 60 python -u tools/tb_debug.py crash > gpurun_out/tb_crash.log 2>&1
grep -E "case|ok|Error" gpurun_out/tb_crash.log | tail -3
timeout 60 python -u tools/tb_debug.py probe 8 > gpurun_out/tb_probe8.log 2>&1; cat gpurun_out/tb_probe8.log
unset STENCIL_B200_LIB
timeout 300 python -m pytest tests/test_gpu_tb.py -q -x > gpurun_out/pytest_tb.log 2>&1; tail -n 3 gpurun_out/pytest_tb.log
for K in 4 6 8; do timeout 120 python bench.py --config c2 --fold-m $K --stages $K --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tb_c2_k$K.json 2>gpurun_out/tb_c2_k$K.err; done
for K in 4 8; do timeout 120 python bench.py --config c3 --fold-m $K --stages $K --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tb_c3_k$K.json 2>gpurun_out/tb_c3_k$K.err; done
python tools/tbsum.py
