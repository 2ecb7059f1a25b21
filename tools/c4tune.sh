for name in "$@"; do
  if [ "$name" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$name.so; fi
  timeout 120 python bench.py --config c4 --fold-m 2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/c4_${name}.json 2>gpurun_out/c4_${name}.err
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/c4_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f.split("/")[-1], round(d["value"], 1), "hbm", round(r["hbm"]["frac"], 3), "fma", round(r["fma"]["frac"], 3), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", open(f.replace(".json", ".err")).read()[-300:])
PY
