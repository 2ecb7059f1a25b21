import glob
import json
for f in sorted(glob.glob("gpurun_out/tb_c*_k*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = d["roofline"]
        print(f, round(d["value"], 1), "frac", round(r["frac"], 3), r["bound"], "hbm", round(r["hbm"]["frac"], 3),
              "fma", round(r["fma"]["frac"], 3), "clk", d["clocks"].get("sm_mhz"), d["clocks"].get("reasons"))
    except Exception as e:
        print(f, "ERR", e, open(f.replace(".json", ".err")).read()[-300:])
