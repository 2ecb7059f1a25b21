"""PERIODIC boundary on the GPU: the CUDA path against
the fp64 oracle's PERIODIC mode (interior, element by element) and against the
closed form of a Fourier mode (independent of the oracle): with
u0 = cos(theta . x), theta = 2 pi k / N, T steps give Re(sigma(theta)^T e^{i theta . x})
where sigma(theta) = sum_j w_j e^{i theta . o_j} (Eq.2's folded weights are the
T-fold convolution, whose symbol is sigma^T)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-11, "f32": 2e-5}


def _interior(a, r=1):
    return a[tuple(slice(r, -r) for _ in range(a.ndim))]


def run_periodic(dims, shape, dtype, T, m, stages, u0=None, w=None, r=1):
    from paper_2103_09235_b200 import Plan
    nd = len(dims)
    offs = oracle.taps(nd, r, oracle.STAR if shape == "star" else oracle.BOX)
    if w is None:
        w = synth.weights(len(offs), 1)
    if u0 is None:
        u0 = synth.u0_frame(dims, r, 2)
    plan = Plan(dims, r, shape, w, dtype, boundary="periodic")
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, m, workspace=ws, stages=stages)
    torch.cuda.synchronize()
    got = plan.frame_view(b).cpu().double().numpy()
    ref = oracle.run(dims, r, offs, w, u0, T, boundary=oracle.PERIODIC)
    return got, ref, u0, plan, b, offs, w


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("m,stages", [(1, 1), (2, 1), (4, 1), (2, 2), (4, 2)])
@pytest.mark.parametrize("T", [5, 8])
def test_periodic_parity_2d(dtype, shape, m, stages, T):
    got, ref, u0, _, _, _, _ = run_periodic((70, 523), shape, dtype, T, m, stages)
    err = np.max(np.abs(_interior(got) - _interior(ref)))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("m,stages", [(1, 1), (2, 1), (2, 2)])
def test_periodic_parity_3d(dtype, shape, m, stages):
    got, ref, u0, _, _, _, _ = run_periodic((19, 37, 75), shape, dtype, 5, m, stages)
    err = np.max(np.abs(_interior(got) - _interior(ref)))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("n,T,m", [(1000, 37, 1), (1000, 37, 2), (100000, 100, 2), (333, 9, 4)])
def test_periodic_parity_1d(n, T, m):
    got, ref, u0, _, _, _, _ = run_periodic((n,), "star", "f64", T, m, 0)
    assert np.max(np.abs(_interior(got) - _interior(ref))) <= 1e-11 * np.max(np.abs(u0))


@pytest.mark.parametrize("dims,shape,m,T", [((40, 300), "box", 2, 6), ((40, 300), "star", 4, 7),
                                            ((12, 20, 70), "star", 2, 5), ((12, 20, 70), "box", 1, 3),
                                            ((333,), "star", 2, 7)])
def test_periodic_dyadic_bitwise(dims, shape, m, T):
    """Dyadic weights (j/64) and field (multiples of 2^-8): with T <= 7 every
    partial sum needs at most 8 + 6T <= 50 significant bits, so it is exact in
    fp64 and folded, stepwise and any accumulation order agree with the
    oracle bit for bit."""
    nd = len(dims)
    k = len(oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX))
    w = synth.dyadic_weights(k, seed=5)
    u0 = synth.dyadic_field(tuple(n + 2 for n in dims), seed=6)
    got, ref, _, _, _, _, _ = run_periodic(dims, shape, "f64", T, m, 0, u0=u0, w=w)
    assert np.array_equal(_interior(got), _interior(ref))


@pytest.mark.parametrize("dims,shape,kvec", [((64, 96), "box", (3, 5)), ((16, 24, 40), "star", (1, 2, 3)),
                                             ((256,), "star", (7,))])
@pytest.mark.parametrize("m", [1, 2])
def test_periodic_fourier_mode_closed_form(dims, shape, kvec, m):
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 3)
    theta = [2 * np.pi * kk / n for kk, n in zip(kvec, dims)]
    grids = np.meshgrid(*[np.arange(-1, n + 1) for n in dims], indexing="ij")
    phase = sum(t * g for t, g in zip(theta, grids))
    u0 = np.cos(phase)
    T = 6
    got, _, _, _, _, _, _ = run_periodic(dims, shape, "f64", T, m, 0, u0=u0, w=w)
    sigma = sum(wj * np.exp(1j * sum(t * o for t, o in zip(theta, oj))) for wj, oj in zip(w, offs))
    want = np.real(sigma ** T * np.exp(1j * phase))
    assert np.max(np.abs(_interior(got) - _interior(want))) <= 1e-12


def test_periodic_ghosts_hold_wrapped_interior():
    dims = (30, 50)
    got, _, _, plan, b, _, _ = run_periodic(dims, "box", "f64", 4, 2, 0)
    L = plan.layout
    full = b.cpu().double().numpy().reshape(L.extent[0], L.stride[0])
    G = 8
    oy, ox = L.origin
    inter = full[oy:oy + 30, ox:ox + 50]
    ext = full[oy - G:oy + 30 + G, ox - G:ox + 50 + G]
    assert np.array_equal(ext, np.pad(inter, G, mode="wrap"))
