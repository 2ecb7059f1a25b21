"""Parity of the 2D temporal block (csrc/tb2d.cuh; SURVEY §8 a6 + NEXT-1):
K = fold_m single steps per HBM round trip (stencil_run_ex(..., fold_m=K,
stages=K)) against the fp64 oracle.

* element by element over the whole padded frame, every K = 2..8, star and
  box, fp64 and fp32, ragged extents (several strips and segments, partial
  last strip, segments not dividing the rows), T with and without remainder;
* dyadic inputs: bit-exact (the frozen ring rows/columns re-read from shared
  memory must reproduce u0 exactly);
* the dist decomposition (emulated ranks, NCCL-schedule copies and fused peer
  stores) bitwise equal to one GPU;
* no write outside the frame (canary guards);
* full size (C2 fp64 K=8, C3 fp32 K=8): cone-exact samples near every face
  and corner plus the closed-form affine check of the whole deep interior.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_bounds import _carve, _guards_ok

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-11, "f32": 2e-5}


def _plan(dims, shape, dtype, w):
    from paper_2103_09235_b200 import Plan
    return Plan(dims, 1, shape, w, dtype)


def _run(dims, shape, dtype, T, K, u0=None, w=None):
    offs = oracle.taps(2, 1, oracle.STAR if shape == "star" else oracle.BOX)
    if w is None:
        w = synth.weights(len(offs), 1)
    if u0 is None:
        u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = _plan(dims, shape, dtype, w)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    return plan.frame_view(b).cpu().double().numpy(), ref, u0


@pytest.mark.parametrize("K", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("dims", [(70, 523), (301, 1100), (9, 40)])
def test_tb_parity(K, shape, dtype, dims):
    T = 3 * K + (1 if dims[0] % 2 else 0)      # with and without a remainder sweep
    got, ref, u0 = _run(dims, shape, dtype, T, K)
    err = float(np.max(np.abs(got - ref)))
    assert err <= TOL[dtype] * float(np.max(np.abs(u0))), err


@pytest.mark.parametrize("K,shape,dims,T", [(4, "star", (40, 300), 4), (4, "box", (40, 300), 11),
                                            (8, "star", (33, 250), 8), (3, "box", (20, 129), 9),
                                            (8, "box", (5, 7), 8), (2, "star", (1, 1), 6), (5, "star", (70, 270), 10)])
def test_tb_dyadic_bitwise(K, shape, dims, T):
    k = len(oracle.taps(2, 1, oracle.STAR if shape == "star" else oracle.BOX))
    w = synth.dyadic_weights(k, seed=5, denom_bits=4)   # k/16: exact for 8 + 4T <= 53 bits
    u0 = synth.dyadic_field(tuple(n + 2 for n in dims), seed=6)
    got, ref, _ = _run(dims, shape, "f64", T, K, u0=u0, w=w)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("exchange", ["copies", "peer"])
@pytest.mark.parametrize("dims,shape,dtype,K,G,T", [((64, 700), "star", "f64", 4, 4, 9), ((96, 1100), "box", "f32", 8, 3, 17),
                                                    ((48, 300), "star", "f64", 8, 2, 17),
                                                    # the bench's N > 1 configuration: fold 6 with T mod 6 = 2
                                                    ((72, 1030), "star", "f64", 6, 3, 20)])
def test_tb_dist_emulated_bitwise(exchange, dims, shape, dtype, K, G, T):
    k = len(oracle.taps(2, 1, oracle.STAR if shape == "star" else oracle.BOX))
    plan = _plan(dims, shape, dtype, synth.weights(k, 1))
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


@pytest.mark.parametrize("dims,shape,dtype,K", [((40, 300), "star", "f64", 8), ((40, 301), "box", "f32", 4),
                                                ((7, 1030), "star", "f32", 6)])
def test_tb_no_writes_outside(dims, shape, dtype, K):
    k = len(oracle.taps(2, 1, oracle.STAR if shape == "star" else oracle.BOX))
    plan = _plan(dims, shape, dtype, synth.weights(k, 1))
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


# the bench's launch configurations: C2 at fold 6 (its default, 33 blocks + one folded
# lambda^(2) sweep) and 8, C3 at fold 8
FULL = {"c2": ((8192, 8192), "star", "f64", 200, 6), "c2k8": ((8192, 8192), "star", "f64", 200, 8),
        "c3": ((16384, 16384), "box", "f32", 200, 8)}


def _samples(n0, n1):
    return [((0, 0), (3, 3)), ((0, n1 // 2), (2, n1 // 2 + 3)), ((3, 5), (6, 9)), ((n0 - 3, n1 - 3), (n0, n1)),
            ((n0 // 2 - 1, 0), (n0 // 2 + 2, 3)), ((n0 // 2, n1 - 2), (n0 // 2 + 2, n1)),
            ((n0 // 3, n1 // 3), (n0 // 3 + 3, n1 // 3 + 3)), ((n0 - 2, 7), (n0, 10))]


@pytest.mark.parametrize("key", ["c2", "c2k8", "c3"])
def test_tb_fullsize(key):
    dims, shape, dtype, T, K = FULL[key]
    offs = oracle.taps(2, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    plan = _plan(dims, shape, dtype, w)
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    inter = plan.interior_view(b)
    for lo, hi in _samples(*dims):
        r = oracle.run_window(dims, 1, offs, w, T, lo, hi, lambda l, h: synth.u0_block(dims, 1, l, h, 2))
        got = inter[lo[0]:hi[0], lo[1]:hi[1]].cpu().double().numpy()
        assert float(np.max(np.abs(got - r))) <= TOL[dtype], (lo, hi)
    # affine field: the whole deep interior against its closed form
    mu = [sum(wj * o[ax] for o, wj in zip(offs, w)) for ax in range(2)]
    L = plan.layout
    coef = [0.5 / (n + 2) for n in dims]
    field = torch.full(L.frame, 0.1, dtype=torch.float64, device="cuda")
    for ax in range(2):
        shp = [1, 1]
        shp[ax] = L.frame[ax]
        field += coef[ax] * (torch.arange(L.frame[ax], dtype=torch.float64, device="cuda") - 1).reshape(shp)
    plan.frame_view(a).copy_(field.to(plan.torch_dtype))
    plan.run(a, b, T, K, workspace=ws, stages=K)
    torch.cuda.synchronize()
    inner = tuple(slice(T + 1, n + 1 - T) for n in dims)
    expect = field[inner] + T * (coef[0] * mu[0] + coef[1] * mu[1])
    err = float((plan.frame_view(b)[inner].double() - expect).abs().max())
    assert err <= TOL[dtype] * 4.4, err
