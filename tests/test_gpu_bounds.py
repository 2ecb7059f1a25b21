"""Memory-safety checks of our own (compute-sanitizer is not available on the
GPU pool): every kernel family runs on buffers carved out of one larger
allocation whose guard regions (before, between and after the buffers) hold a
canary pattern; afterwards the guards and `in` must be bit-identical, and the
alignment pads of `out` (never part of the frame) must still hold the canary
that `in` carried there."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

GUARD = 1 << 16   # bytes of guard around each buffer (multiple of 128)
CANARY = -1234.5


def _carve(plan, layout, n):
    """n buffers of `layout` inside one allocation, GUARD bytes apart."""
    es = layout.elem_bytes
    nb = (layout.bytes + 127) // 128 * 128
    g = GUARD // es
    per = nb // es
    big = torch.full((g + n * (per + g),), CANARY, dtype=plan.torch_dtype, device="cuda")
    bufs = [big[g + i * (per + g): g + i * (per + g) + layout.numel] for i in range(n)]
    return big, bufs, g, per


def _guards_ok(big, g, per, n):
    host = big.cpu().numpy()
    idx = np.zeros(host.size, dtype=bool)
    idx[:g] = True
    for i in range(n):
        s = g + i * (per + g)
        idx[s + per: s + per + g] = True
    return bool(np.all(host[idx] == CANARY))


CASES = [
    dict(dims=(40, 300), shape="star", dtype="f64", T=6, m=2),
    dict(dims=(40, 300), shape="box", dtype="f32", T=8, m=4, stages=2),
    dict(dims=(40, 301), shape="star", dtype="f64", T=8, m=4),
    dict(dims=(12, 20, 70), shape="star", dtype="f64", T=4, m=2),
    dict(dims=(12, 20, 70), shape="box", dtype="f64", T=4, m=2, stages=2),
    dict(dims=(40, 300), shape="box", dtype="f64", T=8, m=4, w=[1.0 / 9] * 9),
    dict(dims=(40, 300), shape="box", dtype="f64", T=6, m=2, boundary="periodic"),
    dict(dims=(12, 20, 70), shape="star", dtype="f32", T=4, m=2, boundary="periodic"),
    dict(dims=(40, 300), shape="star", dtype="f64", T=4, m=2, r=2),
    dict(dims=(3000,), shape="star", dtype="f64", T=37, m=2),
    dict(dims=(3001,), shape="star", dtype="f32", T=9, m=2, boundary="periodic"),
]


@pytest.mark.parametrize("c", CASES, ids=lambda c: "%s-%s-%s-m%d-%s" % (
    "x".join(map(str, c["dims"])), c["shape"], c["dtype"], c["m"], c.get("boundary", "fixed")))
def test_no_writes_outside_the_frame(c):
    from paper_2103_09235_b200 import Plan
    dims, r = c["dims"], c.get("r", 1)
    nd = len(dims)
    offs = oracle.taps(nd, r, oracle.STAR if c["shape"] == "star" else oracle.BOX)
    w = c.get("w") or synth.weights(len(offs), 1)
    plan = Plan(dims, r, c["shape"], w, c["dtype"], boundary=c.get("boundary", "fixed"))
    L = plan.layout
    big, (a, b, ws), g, per = _carve(plan, L, 3)
    plan.frame_view(a).copy_(torch.from_numpy(synth.u0_frame(dims, r, 2)).to(plan.torch_dtype))
    a_before = a.clone()
    plan.run(a, b, c["T"], c["m"], workspace=ws, stages=c.get("stages", 0))
    torch.cuda.synchronize()
    assert _guards_ok(big, g, per, 3), "write outside the buffers"
    assert torch.equal(a, a_before), "`in` was written"
    inside = torch.zeros(L.numel, dtype=torch.bool)
    plan.frame_view(inside, L).fill_(True)
    if c.get("boundary", "fixed") == "periodic":   # ghosts beyond the frame are refilled: only check allocation pads
        return
    pads = ~inside.numpy()
    got = b.cpu().numpy()[pads]
    assert np.all(got == a_before.cpu().numpy()[pads]), "pads of `out` changed"


@pytest.mark.parametrize("exchange", ["copies", "peer"])
def test_dist_emulated_no_writes_outside(exchange):
    from paper_2103_09235_b200 import Plan
    plan = Plan((48, 300), 1, "box", synth.weights(9, 1), "f64")
    G, halo = 3, 2
    Ls = [plan.layout_dist(gr, G, halo) for gr in range(G)]
    big, bufs, g, per = _carve(plan, Ls[0], 3 * G)
    ins, outs, wss = bufs[0::3], bufs[1::3], bufs[2::3]
    for gr in range(G):
        plan.fill_random_dist(gr, G, halo, ins[gr], 2)
    plan.run_dist_emulated(ins, outs, 6, 2, halo, wss, exchange=exchange)
    torch.cuda.synchronize()
    assert _guards_ok(big, g, per, 3 * G)
