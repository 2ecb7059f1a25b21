set -x
python -m pytest tests/test_gpu_tb.py -q > gpurun_out/pytest_tb.log 2>&1
tail -n 40 gpurun_out/pytest_tb.log
for K in 4 6 8; do python bench.py --config c2 --fold-m $K --stages $K --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tb_c2_k$K.json 2>gpurun_out/tb_c2_k$K.err; done
for K in 4 8; do python bench.py --config c3 --fold-m $K --stages $K --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tb_c3_k$K.json 2>gpurun_out/tb_c3_k$K.err; done
python - <<'PY'
import json,glob
for f in sorted(glob.glob("gpurun_out/tb_c*_k*.json")):
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
        print(f, round(d["value"],1), "frac", round(d["roofline"]["frac"],3), d["roofline"]["bound"], "fma", round(d["roofline"]["fma"]["frac"],3), "clk", d["clocks"].get("sm_mhz"))
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json",".err")).read()[-500:])
PY
ncu --set full --import-source on -k regex:tb2d -s 2 -c 1 -o gpurun_out/prof_tb_c2_k8 python bench.py --config c2 --fold-m 8 --stages 8 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/ncu_tb_c2.log 2>&1
ncu --set full --import-source on -k regex:tb2d -s 2 -c 1 -o gpurun_out/prof_tb_c3_k4 python bench.py --config c3 --fold-m 4 --stages 4 --steps 1 --warmup 1 --headline-only --no-cpu-baseline > gpurun_out/ncu_tb_c3.log 2>&1
tail -n 3 gpurun_out/ncu_tb_c2.log
