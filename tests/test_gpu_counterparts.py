"""Counterpart evaluation on the GPU (vertical/horizontal
folding Eq.4-6, counterpart reuse Eq.7): low-rank folded
weights (the paper's uniform 2D9P; separable weights) evaluated through
rank-1 counterparts must match the fp64 oracle and the dense folded pass."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-11, "f32": 2e-5}


def _run(dims, w, dtype, T, m, counterparts=True, boundary="fixed"):
    from paper_2103_09235_b200 import Plan
    plan = Plan(dims, 1, "box", w, dtype, boundary=boundary)
    plan.set_counterparts(counterparts)
    u0 = synth.u0_frame(dims, 1, 2)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, m, workspace=ws)
    torch.cuda.synchronize()
    return plan.frame_view(b).cpu().double().numpy(), u0, plan


def _weights(kind):
    if kind == "uniform":
        return np.full(9, 1.0 / 9.0)
    rng = np.random.default_rng(11)
    return np.outer(rng.uniform(0.5, 1.5, 3), rng.uniform(0.5, 1.5, 3)).ravel() / 9.0


@pytest.mark.parametrize("kind", ["uniform", "separable"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("m,T", [(2, 6), (2, 7), (4, 8), (4, 9)])
def test_counterpart_parity(kind, dtype, m, T):
    dims = (70, 523)
    w = _weights(kind)
    got, u0, plan = _run(dims, w, dtype, T, m)
    assert plan.variant(m)[2] == 1                       # the counterpart pass ran
    offs = oracle.taps(2, 1, oracle.BOX)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    assert np.max(np.abs(got - ref)) <= TOL[dtype] * np.max(np.abs(u0))
    dense, _, _ = _run(dims, w, dtype, T, m, counterparts=False)
    assert np.max(np.abs(got - dense)) <= TOL[dtype] * np.max(np.abs(u0))


@pytest.mark.parametrize("m", [2, 4])
def test_counterpart_periodic(m):
    dims = (48, 300)
    w = _weights("uniform")
    got, u0, _ = _run(dims, w, "f64", 8, m, boundary="periodic")
    ref = oracle.run(dims, 1, oracle.taps(2, 1, oracle.BOX), w, u0, 8, boundary=oracle.PERIODIC)
    assert np.max(np.abs(got[1:-1, 1:-1] - ref[1:-1, 1:-1])) <= 1e-11 * np.max(np.abs(u0))
