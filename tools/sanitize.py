"""Small runs of every kernel family for compute-sanitizer (memcheck / racecheck /
synccheck): 2D/3D folded, multi-stage, band, counterparts, PERIODIC, radius 2,
1D, emulated dist with both exchanges."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
from paper_2103_09235_b200 import Plan  # noqa: E402


def case(dims, shape, dtype, T, m, stages=0, r=1, boundary="fixed", w=None):
    nd = len(dims)
    offs = oracle.taps(nd, r, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1) if w is None else w
    p = Plan(dims, r, shape, w, dtype, boundary=boundary)
    a, b, ws = p.empty(), p.empty(), p.empty()
    p.fill_random(a, 2)
    p.run(a, b, T, m, workspace=ws, stages=stages)
    return p


case((40, 300), "star", "f64", 6, 2)
case((40, 300), "box", "f32", 8, 4, 2)
case((40, 300), "star", "f64", 8, 4)
case((12, 20, 70), "star", "f64", 4, 2)
case((12, 20, 70), "box", "f64", 4, 2, 2)
case((40, 300), "box", "f64", 8, 4, w=[1.0 / 9] * 9)           # counterparts
case((40, 300), "box", "f64", 6, 2, boundary="periodic")
case((12, 20, 70), "star", "f32", 4, 2, boundary="periodic")
case((40, 300), "star", "f64", 4, 2, r=2)
case((3000,), "star", "f64", 37, 2)
p = Plan((48, 300), 1, "box", synth.weights(9, 1), "f64")
for exch in ("copies", "peer"):
    G, halo = 2, 2
    ins, outs, wss = [], [], []
    for g in range(G):
        L = p.layout_dist(g, G, halo)
        t = p.empty(layout=L)
        p.fill_random_dist(g, G, halo, t, 2)
        ins.append(t)
        outs.append(p.empty(layout=L))
        wss.append(p.empty(layout=L))
    p.run_dist_emulated(ins, outs, 6, 2, halo, wss, exchange=exch)
torch.cuda.synchronize()
print("sanitize cases ok")
