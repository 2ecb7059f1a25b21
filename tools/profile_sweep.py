"""Run a few sweeps of one config/variant (for ncu captures of single kernels)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
from bench import CONFIGS  # noqa: E402
from paper_2103_09235_b200 import Plan  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--m", type=int, default=2)
ap.add_argument("--stages", type=int, default=0)
ap.add_argument("--sweeps", type=int, default=3)
a = ap.parse_args()
cfg = CONFIGS[a.config]
nd = len(cfg["dims"])
k = {(1, "star"): 3, (2, "star"): 5, (2, "box"): 9, (3, "star"): 7, (3, "box"): 27}[(nd, cfg["shape"])]
from bench import config_weights  # noqa: E402
plan = Plan(cfg["dims"], 1, cfg["shape"], config_weights(cfg, k), cfg["dtype"])
x, y, w = plan.empty(), plan.empty(), plan.empty()
plan.fill_random(x, 2)
plan.run(x, y, a.m * a.sweeps, a.m, w, a.stages)
torch.cuda.synchronize()
print("ok", a.config, a.m, a.stages, plan.last_launches)
