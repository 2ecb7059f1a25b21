"""Ad-hoc: fp32 3D plans, folded / stepwise passes vs the 3D temporal block (GStencil/s)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
from paper_2103_09235_b200 import Plan

def bench(dims, shape, T, m, stages, n=3):
    k = 7 if shape == "star" else 27
    plan = Plan(dims, 1, shape, synth.weights(k, 1), "f32")
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, m, workspace=ws, stages=stages)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        plan.run(a, b, T, m, workspace=ws, stages=stages)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    pts = 1
    for d in dims:
        pts *= d
    print("%s %s f32 T=%d m=%d stages=%d variant=%s: %.1f GStencil/s" % (dims, shape, T, m, stages, plan.variant(m), pts * T / ms / 1e6), flush=True)

for m, s in [(1, 0), (2, 0), (2, 2), (3, 3), (4, 4)]:
    bench((512, 512, 512), "star", 96, m, s)
for m, s in [(1, 0), (2, 0), (2, 2)]:
    bench((384, 768, 768), "box", 96, m, s)
