# fold_m scan for the 2D configs: folded pass (stages=1) vs temporal block (stages=m)
for cfg in c2 c3; do
  for m in 2 3 4 5 6 7 8; do
    for s in 1 $m; do
      timeout 120 python bench.py --config $cfg --fold-m $m --stages $s --steps 3 --headline-only --no-cpu-baseline > gpurun_out/ms_${cfg}_m${m}_s${s}.json 2>/dev/null
    done
  done
done
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/ms_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1]); r = d["roofline"]
        print(f.split("/")[-1], round(d["value"], 1), "hbm", round(r["hbm"]["frac"], 3), "fma", round(r["fma"]["frac"], 3))
    except Exception as e:
        print(f, "ERR")
PY
