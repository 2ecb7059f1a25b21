# usage: bash tools/tbtune.sh [-p PASS] lib1 lib2 ...   (tunelibs/lib_<name>.so; "main" = in-tree library)
# Measures C2 K=8, C3 K=8 and C2 K=6 with each library; repeat with another -p
# label to interleave A/B passes inside one call.
pass=a; if [ "$1" = -p ]; then pass=$2; shift 2; fi
for name in "$@"; do
  if [ "$name" = main ]; then unset STENCIL_B200_LIB; else export STENCIL_B200_LIB=tunelibs/lib_$name.so; fi
  for cfg in ${TB_CFGS:-"c2 8" "c3 8" "c2 6"}; do set -- ${cfg/:/ }
    timeout 120 python bench.py --config $1 --fold-m $2 --stages $2 --steps 5 --headline-only --no-cpu-baseline > gpurun_out/tt_${name}_$1_k$2_$pass.json 2>gpurun_out/tt_${name}_$1_k$2_$pass.err
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/tt_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f.split("/")[-1], round(d["value"], 1), "hbm", round(r["hbm"]["frac"], 3), "fma", round(r["fma"]["frac"], 3), d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", open(f.replace(".json", ".err")).read()[-200:])
PY
