"""Parity through every path of the dynamic schedule, and a
whole-frame closed-form check at the full BASELINE sizes.

1. Whole-frame parity vs the fp64 oracle, element by element, on mid-size
   grids where the persistent CTAs must claim chunks, GRAB never-started
   segments (grid capped with stencil_plan_set_schedule's max_ctas) and
   STEAL the upper half of other segments (small chunk / min_steal).  The
   kernels count successful grabs and steals (stencil_plan_sched_stats) and
   each test asserts both happened.

2. Full size (BASELINE configs C2-C5, the fold_m bench.py times): the input is
   an affine field u0(p) = b + a . p on the whole padded frame, ring included.
   With weights summing to 1, one step maps it to u0(p) + a . mu with
   mu = sum_j w_j o_j (the drift of the stencil; exact algebra of
   P:64's weighted sum), so after T steps every point farther than T r from a
   FIXED face holds b + a . (p + T mu).  That checks EVERY deep-interior output
   of the full-size launch (97 % of C2's points), whatever segment, chunk or
   steal produced it; the near-face points are covered by
   test_gpu_fullsize.py's cone-exact samples.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-11, "f32": 2e-5}


def _plan(dims, shape, dtype, w, r=1):
    from paper_2103_09235_b200 import Plan
    return Plan(dims, r, shape, w, dtype)


SCHED_CASES = [
    # dims, shape, dtype, T, m
    ((2048, 3072), "star", "f64", 24, 2),
    ((2048, 3072), "star", "f64", 24, 3),
    ((2048, 3072), "star", "f64", 24, 4),
    ((1024, 4100), "box", "f32", 12, 2),
    ((96, 192, 256), "star", "f64", 8, 1),
    ((96, 192, 256), "star", "f64", 8, 2),
    ((64, 128, 128), "box", "f64", 6, 1),
    ((64, 128, 128), "box", "f64", 6, 2),
]


@pytest.mark.parametrize("dims,shape,dtype,T,m", SCHED_CASES)
@pytest.mark.parametrize("max_ctas", [10, 0])
def test_schedule_paths_whole_frame(dims, shape, dtype, T, m, max_ctas):
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = _plan(dims, shape, dtype, w)
    plan.set_schedule(chunk=4, min_steal=8, max_ctas=max_ctas)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, 1, 1, workspace=ws)          # allocate the schedule scratch
    torch.cuda.synchronize()
    plan.sched_stats(reset=True)
    plan.run(a, b, T, m, workspace=ws, stages=1)   # the folded pass: the dynamic-schedule kernel
    torch.cuda.synchronize()
    grabs, steals = plan.sched_stats()
    got = plan.frame_view(b).cpu().double().numpy()
    err = float(np.max(np.abs(got - ref)))
    assert err <= TOL[dtype] * float(np.max(np.abs(u0))), err
    if max_ctas:
        assert grabs > 0 and steals > 0, (grabs, steals)


FULL = {
    "c2": ((8192, 8192), "star", "f64", 200, 3),
    "c3": ((16384, 16384), "box", "f32", 200, 2),
    "c4": ((512, 512, 512), "star", "f64", 100, 2),
    "c5": ((384, 768, 768), "box", "f64", 100, 1),
}


@pytest.mark.parametrize("key", ["c2", "c3", "c4", "c5"])
def test_fullsize_affine_whole_interior(key):
    dims, shape, dtype, T, m = FULL[key]
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    mu = [sum(wj * o[a] for o, wj in zip(offs, w)) for a in range(nd)]
    plan = _plan(dims, shape, dtype, w)
    L = plan.layout
    a_coef = [0.5 / (n + 2) for n in dims]      # values in [0.1, 1.1]
    b0 = 0.1
    dev = torch.device("cuda")
    buf = plan.empty()
    buf.zero_()
    fr = plan.frame_view(buf)
    # affine field on the padded frame (interior coordinate of frame index i is i - r)
    field = torch.full(L.frame, b0, dtype=torch.float64, device=dev)
    for ax in range(nd):
        shp = [1] * nd
        shp[ax] = L.frame[ax]
        field += a_coef[ax] * (torch.arange(L.frame[ax], dtype=torch.float64, device=dev) - 1).reshape(shp)
    fr.copy_(field.to(plan.torch_dtype))
    out, ws = plan.empty(), plan.empty()
    plan.run(buf, out, 1, 1, workspace=ws)      # allocate the schedule scratch
    torch.cuda.synchronize()
    plan.sched_stats(reset=True)
    plan.run(buf, out, T, m, workspace=ws)
    torch.cuda.synchronize()
    grabs, steals = plan.sched_stats()
    if key == "c4":   # 128 columns for 148 persistent CTAs: 20 start by stealing
        assert steals > 0, (grabs, steals)
    inner = tuple(slice(T + 1, n + 1 - T) for n in dims)   # frame coords: interior p at distance >= T
    expect = field[inner] + T * sum(a_coef[ax] * mu[ax] for ax in range(nd))
    got = plan.frame_view(out)[inner].double()
    err = float((got - expect).abs().max())
    assert err <= TOL[dtype] * 1.1 * 4, (key, err)
    # the frozen ring is untouched
    assert torch.equal(plan.frame_view(out)[(slice(0, 1),) + (slice(None),) * (nd - 1)],
                       fr[(slice(0, 1),) + (slice(None),) * (nd - 1)])


def test_schedule_is_graph_capture_safe():
    """a captured 2D run replays correctly any number of times and
    interleaved with eager runs of the same plan (the schedule scratch is
    zeroed around every captured sweep)."""
    dims, shape, dtype, T, m = (512, 700), "star", "f64", 7, 2
    offs = oracle.taps(2, 1, oracle.STAR)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = _plan(dims, shape, dtype, w)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.run(a, b, T, m, workspace=ws)       # eager first (scratch allocation)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        plan.run(a, b, T, m, workspace=ws, stream=s)
    tol = TOL[dtype] * float(np.max(np.abs(u0)))
    for it in range(5):
        b.zero_()
        g.replay()
        if it % 2:
            plan.run(a, ws, 1, 1)                   # eager runs in between (epochs advance)
        torch.cuda.synchronize()
        got = plan.frame_view(b).cpu().double().numpy()
        assert float(np.max(np.abs(got - ref))) <= tol, it
