"""Full-size parity at BASELINE.json's configs, in the launch configuration
bench.py times (stencil_run with the config's fold_m set, auto stages, on the
full grid), against the oracle on sampled outputs.

The oracle cannot run 16384^2 x 200 steps in seconds, so each sampled output
box is computed exactly on its dependency cone (oracle.run_window: the same
per-point arithmetic as a full-domain run, pinned bit-identical by
tests/test_oracle_pins.py::test_window_is_bit_identical).  Samples cover the
corners and faces (the stepwise band), the band edge and the deep interior.
The 1D config is compared in full.  Multi-GPU: the slab-decomposed algorithm
(emulated ranks on this GPU) is bitwise equal to one GPU at full size.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

CONFIGS = {
    "c1": ((100000,), "star", "f64", 100, (1, 2)),
    "c2": ((8192, 8192), "star", "f64", 200, (1, 2, 3, 4)),
    "c3": ((16384, 16384), "box", "f32", 200, (1, 2, 4)),
    "c4": ((512, 512, 512), "star", "f64", 100, (1, 2)),
    "c5": ((384, 768, 768), "box", "f64", 100, (1, 2)),
}
TOL = {"f64": 1e-11, "f32": 2e-5}


def samples(dims):
    nd = len(dims)
    if nd == 2:
        n0, n1 = dims
        return [((0, 0), (3, 3)), ((0, n1 // 2), (2, n1 // 2 + 3)), ((2, 2), (5, 6)),
                ((n0 // 2 - 1, n1 // 2 - 2), (n0 // 2 + 2, n1 // 2 + 2)), ((n0 - 3, n1 - 3), (n0, n1)),
                ((n0 // 3, 1), (n0 // 3 + 2, 4))]
    n0, n1, n2 = dims
    return [((0, 0, 0), (2, 2, 3)), ((n0 // 2, 0, n2 // 2), (n0 // 2 + 2, 2, n2 // 2 + 2)),
            ((n0 - 2, n1 // 2, n2 - 2), (n0, n1 // 2 + 2, n2))]


@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4", "c5"])
def test_fullsize_sampled(key):
    from paper_2103_09235_b200 import Plan
    dims, shape, dtype, T, ms = CONFIGS[key]
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), synth.DEFAULT_SEED_W)
    plan = Plan(dims, 1, shape, w, dtype)
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, synth.DEFAULT_SEED_U)
    if nd == 1:
        ref = oracle.run(dims, 1, offs, w, synth.u0_frame(dims, 1, 2), T)
        refs = [((0,), dims, ref[1:-1])]
    else:
        refs = []
        for lo, hi in samples(dims):
            r = oracle.run_window(dims, 1, offs, w, T, lo, hi,
                                  lambda l, h: synth.u0_block(dims, 1, l, h, synth.DEFAULT_SEED_U))
            refs.append((lo, hi, r))
    for m in ms:
        plan.run(a, b, T, m, workspace=ws)
        torch.cuda.synchronize()
        inter = plan.interior_view(b)
        for lo, hi, r in refs:
            got = inter[tuple(slice(l, h) for l, h in zip(lo, hi))].cpu().double().numpy()
            err = float(np.max(np.abs(got - r)))
            assert err <= TOL[dtype], (key, m, lo, err)


@pytest.mark.parametrize("key,G,m,exchange", [("c3", 4, 2, "copies"), ("c4", 2, 2, "copies"), ("c2", 8, 4, "copies"),
                                              ("c3", 4, 2, "peer"), ("c4", 4, 2, "peer"), ("c2", 8, 4, "peer")])
def test_fullsize_dist_emulated_bitwise(key, G, m, exchange):
    from paper_2103_09235_b200 import Plan
    dims, shape, dtype, T, _ = CONFIGS[key]
    nd = len(dims)
    k = len(oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX))
    plan = Plan(dims, 1, shape, synth.weights(k, 1), dtype)
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, m, workspace=ws)
    single = plan.interior_view(b)
    halo = m
    ins, outs, wss, Ls = [], [], [], []
    for g in range(G):
        L = plan.layout_dist(g, G, halo)
        Ls.append(L)
        t = plan.empty(layout=L)
        plan.fill_random_dist(g, G, halo, t, 2)
        ins.append(t)
        outs.append(plan.empty(layout=L))
        wss.append(plan.empty(layout=L))
    plan.run_dist_emulated(ins, outs, T, m, halo, wss, exchange=exchange)
    torch.cuda.synchronize()
    per = dims[0] // G
    for g in range(G):
        assert torch.equal(plan.interior_view(outs[g], Ls[g]), single[g * per:(g + 1) * per]), g
