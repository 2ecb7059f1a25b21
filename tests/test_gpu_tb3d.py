"""Parity of the 3D temporal block (csrc/tb3d.cuh; SURVEY §8 a6 + NEXT-1 in
3D): K = fold_m single steps of the radius-1 fp64 star per HBM round trip
(stencil_run_ex(..., fold_m=K, stages=K)) against the fp64 oracle.

* element by element over the whole padded frame, K = 2, 3, 4, ragged extents
  (several tiles in y and x, partial last tiles, z-segments, thin domains),
  T with and without remainder;
* dyadic inputs: bit-exact (the frozen ring cells re-read from `src` must
  reproduce u0 exactly at every level);
* the dist decomposition (emulated ranks, NCCL-schedule copies and fused peer
  stores) bitwise equal to one GPU;
* no write outside the frame (canary guards);
* full size (C4, 512^3 fp64, K = 4, T = 100): cone-exact samples at faces,
  edges and corners plus the closed-form affine check of the deep interior.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_bounds import _carve, _guards_ok

pytestmark = pytest.mark.gpu

TOL = 1e-11


def _plan(dims, w):
    from paper_2103_09235_b200 import Plan
    return Plan(dims, 1, "star", w, "f64")


def _run(dims, T, K, u0=None, w=None):
    offs = oracle.taps(3, 1, oracle.STAR)
    if w is None:
        w = synth.weights(len(offs), 1)
    if u0 is None:
        u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = _plan(dims, w)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    return plan.frame_view(b).cpu().double().numpy(), ref, u0


@pytest.mark.parametrize("K", [2, 3, 4])
@pytest.mark.parametrize("dims", [(20, 33, 90), (37, 70, 150), (9, 5, 61), (3, 130, 20), (1, 1, 1), (64, 49, 57)])
def test_tb3d_parity(K, dims):
    T = 2 * K + 1   # two blocks + a remainder step
    got, ref, u0 = _run(dims, T, K)
    err = float(np.max(np.abs(got - ref)))
    assert err <= TOL * float(np.max(np.abs(u0))), err


@pytest.mark.parametrize("K,T", [(4, 4), (4, 12), (3, 9), (2, 6)])
def test_tb3d_parity_multiple(K, T):
    got, ref, u0 = _run((41, 77, 130), T, K)
    err = float(np.max(np.abs(got - ref)))
    assert err <= TOL * float(np.max(np.abs(u0))), err


@pytest.mark.parametrize("K,dims,T", [(4, (24, 40, 100), 8), (3, (13, 37, 70), 6), (2, (8, 9, 10), 4),
                                      (4, (2, 66, 3), 4)])
def test_tb3d_dyadic_bitwise(K, dims, T):
    w = synth.dyadic_weights(7, seed=5, denom_bits=3)   # k/8: exact for 8 + 3T <= 53 bits
    u0 = synth.dyadic_field(tuple(n + 2 for n in dims), seed=6)
    got, ref, _ = _run(dims, T, K, u0=u0, w=w)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("exchange", ["copies", "peer"])
@pytest.mark.parametrize("dims,K,G,T", [((48, 40, 100), 4, 4, 9), ((30, 70, 64), 3, 3, 7), ((16, 20, 30), 2, 2, 5)])
def test_tb3d_dist_emulated_bitwise(exchange, dims, K, G, T):
    plan = _plan(dims, synth.weights(7, 1))
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    single = plan.interior_view(b)
    ins, outs, wss, Ls = [], [], [], []
    for g in range(G):
        L = plan.layout_dist(g, G, K)
        Ls.append(L)
        t = plan.empty(layout=L)
        plan.fill_random_dist(g, G, K, t, 2)
        ins.append(t)
        outs.append(plan.empty(layout=L))
        wss.append(plan.empty(layout=L))
    plan.run_dist_emulated(ins, outs, T, K, K, wss, stages=K, exchange=exchange)
    torch.cuda.synchronize()
    per = dims[0] // G
    for g in range(G):
        assert torch.equal(plan.interior_view(outs[g], Ls[g]), single[g * per:(g + 1) * per]), g


@pytest.mark.parametrize("dims,K", [((20, 40, 100), 4), ((7, 70, 65), 3)])
def test_tb3d_no_writes_outside(dims, K):
    plan = _plan(dims, synth.weights(7, 1))
    L = plan.layout
    big, (a, b, ws), g, per = _carve(plan, L, 3)
    plan.frame_view(a).copy_(torch.from_numpy(synth.u0_frame(dims, 1, 2)).to(plan.torch_dtype))
    a_before = a.clone()
    plan.run(a, b, 2 * K + 1, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    assert _guards_ok(big, g, per, 3)
    assert torch.equal(a, a_before)
    inside = torch.zeros(L.numel, dtype=torch.bool)
    plan.frame_view(inside, L).fill_(True)
    pads = ~inside.numpy()
    assert np.all(b.cpu().numpy()[pads] == a_before.cpu().numpy()[pads])


def _samples(n):
    z, y, x = n
    return [((0, 0, 0), (2, 2, 3)), ((z - 2, y - 2, x - 3), (z, y, x)), ((0, y // 2, x // 2), (2, y // 2 + 2, x // 2 + 3)),
            ((z // 2, 0, x - 3), (z // 2 + 2, 2, x)), ((z // 2, y // 2, 0), (z // 2 + 2, y // 2 + 2, 3)),
            ((z // 3, y - 2, x // 3), (z // 3 + 2, y, x // 3 + 2)),
            # tile seams of the 64 x 32 tiles (56 x 24 outputs at K = 4)
            ((z // 2, 23, 55), (z // 2 + 2, 26, 58)), ((z - 2, 47, 111), (z, 50, 114))]


def test_tb3d_fullsize_c4():
    """C4 (512^3 fp64, T = 100) at K = 4, the bench's launch configuration."""
    dims, T, K = (512, 512, 512), 100, 4
    offs = oracle.taps(3, 1, oracle.STAR)
    w = synth.weights(len(offs), 1)
    plan = _plan(dims, w)
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    inter = plan.interior_view(b)
    for lo, hi in _samples(dims):
        r = oracle.run_window(dims, 1, offs, w, T, lo, hi, lambda l, h: synth.u0_block(dims, 1, l, h, 2))
        got = inter[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].cpu().double().numpy()
        assert float(np.max(np.abs(got - r))) <= TOL, (lo, hi)
    # affine field: the whole deep interior against its closed form u0 + T a.mu
    mu = [sum(wj * o[ax] for o, wj in zip(offs, w)) for ax in range(3)]
    L = plan.layout
    coef = [0.5 / (n + 2) for n in dims]
    field = torch.full(L.frame, 0.1, dtype=torch.float64, device="cuda")
    for ax in range(3):
        shp = [1, 1, 1]
        shp[ax] = L.frame[ax]
        field += coef[ax] * (torch.arange(L.frame[ax], dtype=torch.float64, device="cuda") - 1).reshape(shp)
    plan.frame_view(a).copy_(field)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    inner = tuple(slice(T + 1, n + 1 - T) for n in dims)
    expect = field[inner] + T * sum(c * m for c, m in zip(coef, mu))
    err = float((plan.frame_view(b)[inner] - expect).abs().max())
    assert err <= TOL * 4.4, err


# ------------------------------------------------------------------ 3D27P box, K = 2
def _run_box(dims, T, u0=None, w=None, K=2):
    from paper_2103_09235_b200 import Plan
    offs = oracle.taps(3, 1, oracle.BOX)
    if w is None:
        w = synth.weights(len(offs), 1)
    if u0 is None:
        u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = Plan(dims, 1, "box", w, "f64")
    assert tuple(plan.variant(K))[:2] == (1, K)   # the stepwise evaluation: K single steps per round trip
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    return plan.frame_view(b).cpu().double().numpy(), ref, u0


@pytest.mark.parametrize("T", [2, 5, 8])
@pytest.mark.parametrize("dims", [(20, 33, 90), (37, 70, 150), (9, 5, 61), (3, 130, 20), (1, 1, 1), (64, 49, 57)])
def test_tb3d_box_parity(T, dims):
    got, ref, u0 = _run_box(dims, T)
    err = float(np.max(np.abs(got - ref)))
    assert err <= TOL * float(np.max(np.abs(u0))), err


@pytest.mark.parametrize("dims,T", [((24, 40, 100), 6), ((8, 9, 10), 4), ((2, 66, 3), 4)])
def test_tb3d_box_dyadic_bitwise(dims, T):
    """Asymmetric dyadic weights: any transposed or mirrored tap of the 27 changes the bits."""
    w = synth.dyadic_weights(27, seed=5, denom_bits=5)   # k/32: exact for 8 + 5T <= 53 bits
    u0 = synth.dyadic_field(tuple(n + 2 for n in dims), seed=6)
    got, ref, _ = _run_box(dims, T, u0=u0, w=w)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("exchange", ["copies", "peer"])
@pytest.mark.parametrize("dims,G,T", [((48, 40, 100), 4, 9), ((16, 20, 30), 2, 5)])
def test_tb3d_box_dist_emulated_bitwise(exchange, dims, G, T):
    from paper_2103_09235_b200 import Plan
    K = 2
    plan = Plan(dims, 1, "box", synth.weights(27, 1), "f64")
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    single = plan.interior_view(b)
    ins, outs, wss, Ls = [], [], [], []
    for g in range(G):
        L = plan.layout_dist(g, G, K)
        Ls.append(L)
        t = plan.empty(layout=L)
        plan.fill_random_dist(g, G, K, t, 2)
        ins.append(t)
        outs.append(plan.empty(layout=L))
        wss.append(plan.empty(layout=L))
    plan.run_dist_emulated(ins, outs, T, K, K, wss, stages=K, exchange=exchange)
    torch.cuda.synchronize()
    per = dims[0] // G
    for g in range(G):
        assert torch.equal(plan.interior_view(outs[g], Ls[g]), single[g * per:(g + 1) * per]), g


def test_tb3d_box_no_writes_outside():
    from paper_2103_09235_b200 import Plan
    dims, K = (20, 40, 100), 2
    plan = Plan(dims, 1, "box", synth.weights(27, 1), "f64")
    L = plan.layout
    big, (a, b, ws), g, per = _carve(plan, L, 3)
    plan.frame_view(a).copy_(torch.from_numpy(synth.u0_frame(dims, 1, 2)).to(plan.torch_dtype))
    a_before = a.clone()
    plan.run(a, b, 2 * K + 1, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    assert _guards_ok(big, g, per, 3)
    assert torch.equal(a, a_before)


def test_tb3d_box_fullsize_c5():
    """C5 (768 x 768 x 384 fp64 3D27P, T = 100) at K = 2 (BASELINE fold_m = 2): cone-exact
    samples at faces, edges, corners and tile seams."""
    from paper_2103_09235_b200 import Plan
    dims, T, K = (384, 768, 768), 100, 2
    offs = oracle.taps(3, 1, oracle.BOX)
    w = synth.weights(len(offs), 1)
    plan = Plan(dims, 1, "box", w, "f64")
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    inter = plan.interior_view(b)
    z, y, x = dims
    samples = [((0, 0, 0), (2, 2, 2)), ((z - 2, y - 2, x - 2), (z, y, x)), ((z // 2, 0, x - 2), (z // 2 + 1, 2, x)),
               ((z // 2, 51, 59), (z // 2 + 1, 53, 61)), ((z - 1, 103, 119), (z, 105, 121)),   # 60 x 52 outputs per tile
               ((127, 727, 719), (129, 729, 721))]                                            # a z-segment seam, last tile row
    for lo, hi in samples:
        r = oracle.run_window(dims, 1, offs, w, T, lo, hi, lambda l, h: synth.u0_block(dims, 1, l, h, 2))
        got = inter[lo[0]:hi[0], lo[1]:hi[1], lo[2]:hi[2]].cpu().double().numpy()
        assert float(np.max(np.abs(got - r))) <= TOL, (lo, hi)


# ------------------------------------------------------------------ fp32 (star K = 2..4, box K = 2)
@pytest.mark.parametrize("shape,K", [("star", 2), ("star", 3), ("star", 4), ("box", 2)])
@pytest.mark.parametrize("dims", [(20, 33, 90), (37, 70, 300), (9, 5, 61), (1, 1, 1), (64, 49, 257)])
def test_tb3d_f32_parity(shape, K, dims):
    from paper_2103_09235_b200 import Plan
    offs = oracle.taps(3, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, 1, 2)
    T = 2 * K + 1
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = Plan(dims, 1, shape, w, "f32")
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    got = plan.frame_view(b).cpu().double().numpy()
    err = float(np.max(np.abs(got - ref)))
    assert err <= 2e-5 * float(np.max(np.abs(u0))), err


@pytest.mark.parametrize("shape,K,G", [("star", 4, 4), ("box", 2, 2)])
def test_tb3d_f32_dist_emulated_bitwise(shape, K, G):
    from paper_2103_09235_b200 import Plan
    dims, T = (48, 40, 200), 2 * K + 1
    plan = Plan(dims, 1, shape, synth.weights(7 if shape == "star" else 27, 1), "f32")
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    single = plan.interior_view(b)
    ins, outs, wss, Ls = [], [], [], []
    for g in range(G):
        L = plan.layout_dist(g, G, K)
        Ls.append(L)
        t = plan.empty(layout=L)
        plan.fill_random_dist(g, G, K, t, 2)
        ins.append(t)
        outs.append(plan.empty(layout=L))
        wss.append(plan.empty(layout=L))
    plan.run_dist_emulated(ins, outs, T, K, K, wss, stages=K, exchange="peer")
    torch.cuda.synchronize()
    per = dims[0] // G
    for g in range(G):
        assert torch.equal(plan.interior_view(outs[g], Ls[g]), single[g * per:(g + 1) * per]), g
