"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 CPU oracle on the
same seeded inputs, element by element over the whole padded frame, at sizes
that span several tiles and ragged tails.  Tolerances (BASELINE.json
north_star): max|d| <= 1e-11 max|u0| (fp64), <= 2e-5 max|u0| (fp32)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

TOL = {"f64": 1e-11, "f32": 2e-5}


def _plan(dims, shape, dtype, w):
    from paper_2103_09235_b200 import Plan
    return Plan(dims, 1, shape, w, dtype)


def run_case(dims, shape, dtype, T, m, stages, seed_w=1, seed_u=2, u0=None, w=None):
    nd = len(dims)
    sh = oracle.STAR if shape == "star" else oracle.BOX
    offs = oracle.taps(nd, 1, sh)
    if w is None:
        w = synth.weights(len(offs), seed_w)
    if u0 is None:
        u0 = synth.u0_frame(dims, 1, seed_u)
    ref = oracle.run(dims, 1, offs, w, u0, T)
    plan = _plan(dims, shape, dtype, w)
    a = plan.from_frame(u0)
    b = plan.empty()
    ws = plan.empty()
    plan.run(a, b, T, m, workspace=ws, stages=stages)
    torch.cuda.synchronize()
    got = plan.frame_view(b).cpu().double().numpy()
    # `in` is never written
    assert np.array_equal(plan.frame_view(a).cpu().double().numpy(),
                          u0.astype(np.float64 if dtype == "f64" else np.float32).astype(np.float64))
    return got, ref, u0, plan


CASES_2D = [(m, s) for (m, s) in [(1, 1), (2, 1), (3, 1), (4, 1), (2, 2), (4, 2), (4, 4)]]


@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("m,stages", CASES_2D)
@pytest.mark.parametrize("T", [7, 8])
def test_parity_2d(shape, dtype, m, stages, T):
    dims = (70, 523)
    got, ref, u0, _ = run_case(dims, shape, dtype, T, m, stages)
    err = np.max(np.abs(got - ref))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("shape", ["star", "box"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("m,stages", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("T", [5, 6])
def test_parity_3d(shape, dtype, m, stages, T):
    dims = (19, 37, 75)
    got, ref, u0, _ = run_case(dims, shape, dtype, T, m, stages)
    err = np.max(np.abs(got - ref))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("n,T,m,stages", [(1000, 37, 1, 1), (1000, 37, 2, 1), (1000, 37, 2, 2),
                                          (100000, 100, 1, 1), (100000, 100, 2, 1), (100000, 100, 4, 1),
                                          (5000, 300, 2, 1), (50, 9, 4, 1)])
def test_parity_1d(dtype, n, T, m, stages):
    got, ref, u0, _ = run_case((n,), "star", dtype, T, m, stages)
    err = np.max(np.abs(got - ref))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("dims,shape,m,stages,T", [
    ((40, 300), "box", 1, 1, 6), ((40, 300), "box", 2, 1, 6), ((40, 300), "box", 4, 1, 7),
    ((40, 300), "star", 4, 2, 7), ((40, 300), "star", 4, 4, 5), ((12, 20, 70), "box", 2, 1, 6),
    ((12, 20, 70), "star", 2, 2, 7), ((333,), "star", 2, 1, 7)])
def test_exact_dyadic_bitwise(dims, shape, m, stages, T):
    """Dyadic weights and field: every partial sum is exact in fp64, so the GPU
    (any accumulation order, folded or stepwise, band included) must equal
    the oracle bit for bit."""
    nd = len(dims)
    k = len(oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX))
    w = synth.dyadic_weights(k, seed=5)
    u0 = synth.dyadic_field(tuple(n + 2 for n in dims), seed=6)
    got, ref, _, _ = run_case(dims, shape, "f64", T, m, stages, u0=u0, w=w)
    assert np.array_equal(got, ref)


@pytest.mark.parametrize("dims,shape,m,T", [((3, 5), "box", 4, 9), ((2, 3, 4), "star", 2, 5),
                                            ((1, 50), "star", 2, 6), ((50, 1), "box", 4, 8),
                                            ((1, 1, 9), "box", 2, 4), ((7, 9), "star", 4, 1),
                                            ((6, 200), "star", 2, 0), ((1,), "star", 2, 5)])
def test_edge_cases(dims, shape, m, T):
    got, ref, u0, _ = run_case(dims, shape, "f64", T, m, 0)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(u0))


def test_device_generator_matches_host_generator():
    for dims, shape in [((37, 301), "star"), ((9, 17, 70), "box"), ((777,), "star")]:
        k = len(oracle.taps(len(dims), 1, oracle.STAR if shape == "star" else oracle.BOX))
        for dt in ("f64", "f32"):
            plan = _plan(dims, shape, dt, synth.weights(k, 1))
            buf = plan.empty()
            plan.fill_random(buf, 2)
            torch.cuda.synchronize()
            got = plan.frame_view(buf).cpu().numpy()
            ref = synth.u0_frame(dims, 1, 2).astype(got.dtype)
            assert np.array_equal(got, ref)


def test_dist_generator_and_layout():
    dims = (64, 20, 40)
    plan = _plan(dims, "star", "f64", synth.weights(7, 1))
    G, halo = 4, 2
    for g in range(G):
        L = plan.layout_dist(g, G, halo)
        buf = plan.empty(layout=L)
        plan.fill_random_dist(g, G, halo, buf, 2)
        torch.cuda.synchronize()
        # local planes [-1, n+1) on axis 0 map to global padded rows g*16 + ...
        lo = L.global_offset0
        full = synth.u0_frame(dims, 1, 2)
        for zl in range(-1, L.interior[0] + 1):
            zg = lo + zl
            if zg < -1 or zg > dims[0]:
                continue
            plane = buf.as_strided((dims[1] + 2, dims[2] + 2), L.stride[1:],
                                   (L.origin[0] + zl) * L.stride[0] + (L.origin[1] - 1) * L.stride[1] + L.origin[2] - 1)
            assert np.array_equal(plane.cpu().numpy(), full[zg + 1])


@pytest.mark.parametrize("exchange", ["copies", "peer"])
@pytest.mark.parametrize("dims,shape,dtype,m,stages,T,G", [
    ((64, 300), "box", "f32", 2, 1, 9, 2), ((64, 300), "box", "f32", 4, 2, 9, 4),
    ((48, 20, 70), "star", "f64", 2, 1, 7, 4), ((48, 20, 70), "box", "f64", 2, 2, 6, 2),
    ((64, 300), "star", "f64", 1, 1, 5, 8), ((24, 20, 70), "star", "f64", 2, 1, 8, 4)])
def test_dist_emulated_bitwise_equals_single(dims, shape, dtype, m, stages, T, G, exchange):
    """The slab-decomposed algorithm (all ranks on this GPU, the same kernels and
    boxes as stencil_run_dist) is bitwise equal to 1 GPU and within tolerance of
    the oracle -- with the NCCL path's schedule (exchange by D2D copies) and with
    the fused peer stores of NEXT-2 (the sweep kernel writes the neighbours'
    ghost planes itself; band blocks included)."""
    nd = len(dims)
    k = len(oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX))
    w = synth.weights(k, 1)
    plan = _plan(dims, shape, dtype, w)
    a = plan.empty()
    plan.fill_random(a, 2)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, m, workspace=ws, stages=stages)
    halo = max(m, 2)
    ins, outs, wss, Ls = [], [], [], []
    for g in range(G):
        L = plan.layout_dist(g, G, halo)
        Ls.append(L)
        t = plan.empty(layout=L)
        plan.fill_random_dist(g, G, halo, t, 2)
        ins.append(t)
        outs.append(plan.empty(layout=L))
        wss.append(plan.empty(layout=L))
    plan.run_dist_emulated(ins, outs, T, m, halo, wss, stages=stages, exchange=exchange)
    torch.cuda.synchronize()
    single = plan.interior_view(b).cpu().numpy()
    per = dims[0] // G
    for g in range(G):
        loc = plan.interior_view(outs[g], Ls[g]).cpu().numpy()
        assert np.array_equal(loc, single[g * per:(g + 1) * per]), g
    ref = oracle.run(dims, 1, oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX), w,
                     synth.u0_frame(dims, 1, 2), T)
    err = np.max(np.abs(plan.frame_view(b).cpu().double().numpy() - ref))
    assert err <= TOL[dtype]


def test_errors_and_launch_count():
    from paper_2103_09235_b200 import StencilError
    dims = (64, 64)
    plan = _plan(dims, "star", "f64", synth.weights(5, 1))
    a, b = plan.empty(), plan.empty()
    with pytest.raises(StencilError):
        plan.run(a, a, 4, 1, workspace=b)            # aliasing
    with pytest.raises(StencilError):
        plan.run(a, b, -1, 1, workspace=None)
    with pytest.raises(StencilError):
        plan.run(a, b, 4, -1, workspace=None)        # fold_m < 0 (0 = auto)
    with pytest.raises(StencilError):
        plan.run(a, b, 20, 0, workspace=None)        # auto fold (8): 3 sweeps need a workspace
    with pytest.raises(StencilError):
        plan.run(a, b, 8, 2, workspace=None)         # needs a workspace
    with pytest.raises(StencilError):
        plan.run(a, b, 8, 4, workspace=plan.empty(), stages=3)   # 3 does not divide 4
    plan.fill_random(a, 2)
    plan.run(a, b, 8, 2, workspace=plan.empty())
    torch.cuda.synchronize()
    assert plan.last_launches >= 4 + 1


def run_case_r(dims, r, shape, dtype, T, m, stages, boundary="fixed"):
    """As run_case, for any radius (NEXT-4: higher-order stencils, e.g. 1D5P)."""
    from paper_2103_09235_b200 import Plan
    nd = len(dims)
    offs = oracle.taps(nd, r, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, r, 2)
    bc = oracle.PERIODIC if boundary == "periodic" else oracle.FIXED
    ref = oracle.run(dims, r, offs, w, u0, T, boundary=bc)
    plan = Plan(dims, r, shape, w, dtype, boundary=boundary)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, T, m, workspace=ws, stages=stages)
    torch.cuda.synchronize()
    got = plan.frame_view(b).cpu().double().numpy()
    if boundary == "periodic":
        sl = tuple(slice(r, -r) for _ in dims)
        got, ref = got[sl], ref[sl]
    return got, ref, u0


@pytest.mark.parametrize("dims,shape,m,stages", [
    ((5000,), "star", 1, 1), ((5000,), "star", 2, 1), ((5000,), "star", 4, 1), ((5000,), "star", 2, 2),
    ((60, 301), "star", 1, 1), ((60, 301), "star", 2, 1), ((60, 301), "star", 2, 2),
    ((60, 301), "box", 1, 1), ((60, 301), "box", 2, 1), ((60, 301), "box", 2, 2),
    ((14, 23, 70), "star", 1, 1), ((14, 23, 70), "star", 2, 1), ((14, 23, 70), "star", 2, 2),
    ((14, 23, 70), "box", 1, 1)])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("boundary", ["fixed", "periodic"])
def test_parity_radius2(dims, shape, m, stages, dtype, boundary):
    got, ref, u0 = run_case_r(dims, 2, shape, dtype, 6, m, stages, boundary)
    err = np.max(np.abs(got - ref))
    assert err <= TOL[dtype] * np.max(np.abs(u0)), err


def test_peer_comm_single_rank_api():
    """The fused-exchange C-ABI on one GPU: create a peer comm over the two
    ping-pong buffers, export its IPC records, attach (no neighbours with one
    rank) and run through stencil_run_dist -- equal to stencil_run; a run with
    other buffers than the registered pair is rejected."""
    from paper_2103_09235_b200 import StencilError
    from paper_2103_09235_b200.api import Comm
    dims = (64, 300)
    plan = _plan(dims, "box", "f64", synth.weights(9, 1))
    L = plan.layout_dist(0, 1, 2)
    a = plan.empty(layout=L)
    plan.fill_random_dist(0, 1, 2, a, 2)
    b, ws = plan.empty(layout=L), plan.empty(layout=L)
    comm = Comm.peer(0, 1, b, ws)
    rec = comm.handles()
    assert len(rec) == Comm.PEER_RECORD
    comm.attach([rec])
    plan.run_dist(comm, a, b, 9, 2, 2, ws)
    b2, ws2 = plan.empty(layout=L), plan.empty(layout=L)
    with pytest.raises(StencilError):           # registered pair, swapped roles: one fixed order
        plan.run_dist(comm, a, ws, 1, 1, 2, b)
    with pytest.raises(StencilError):
        plan.halo_exchange(comm, b, 2)          # peer comm: ghosts come from the sweep kernel
    with pytest.raises(StencilError):
        plan.run_dist(comm, a, b2, 9, 2, 2, ws2)
    torch.cuda.synchronize()
    ref, refws = plan.empty(), plan.empty()
    a1 = plan.empty()
    plan.fill_random(a1, 2)
    plan.run(a1, ref, 9, 2, workspace=refws)
    torch.cuda.synchronize()
    assert torch.equal(plan.interior_view(b, L), plan.interior_view(ref))
    comm.close()


@pytest.mark.parametrize("dims,shape,dtype,m", [((70, 523), "star", "f64", 2), ((70, 523), "box", "f32", 2),
                                                ((19, 37, 75), "star", "f64", 2), ((70, 523), "star", "f64", 4)])
def test_fault_injection_is_caught(dims, shape, dtype, m):
    """Perturbing one folded coefficient by 1e-6 (relative to the weights' scale)
    must make the parity check fail: the tests see a wrong lambda^(m)."""
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, 8)
    plan = _plan(dims, shape, dtype, w)
    side = 2 * m + 1
    center = (side ** nd) // 2
    plan.perturb_fold(m, center, 1e-6 if dtype == "f64" else 1e-3)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, 8, m, workspace=ws, stages=1)
    torch.cuda.synchronize()
    err = np.max(np.abs(plan.frame_view(b).cpu().double().numpy() - ref))
    assert err > TOL[dtype] * np.max(np.abs(u0)), err


@pytest.mark.parametrize("r,m,T,boundary", [(4, 8, 17, "fixed"), (3, 6, 13, "fixed"), (3, 6, 13, "periodic"),
                                            (4, 4, 9, "periodic"), (2, 8, 21, "fixed")])
def test_parity_1d_wide_folds(r, m, T, boundary):
    """1D folds of radius m*r > 16 (32 cells per lane) and up to STENCIL_MAX_FOLD."""
    got, ref, u0 = run_case_r((4000,), r, "star", "f64", T, m, 0, boundary)
    assert np.max(np.abs(got - ref)) <= 1e-11 * np.max(np.abs(u0))


@pytest.mark.parametrize("dims,shape,dtype,m", [((70, 523), "star", "f64", 2), ((19, 37, 75), "box", "f32", 2),
                                                ((70, 523), "box", "f64", 4), ((5000,), "star", "f64", 2)])
def test_resume_is_the_semigroup(dims, shape, dtype, m):
    """Checkpoint/resume needs no state beyond the grids: running T1 steps
    and then T2 more from the result equals running T1 + T2 -- bitwise when T1 is a
    multiple of fold_m (the same sweeps run), within tolerance otherwise."""
    nd = len(dims)
    k = len(oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX))
    plan = _plan(dims, shape, dtype, synth.weights(k, 1))
    a, ws = plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    full, mid, res = plan.empty(), plan.empty(), plan.empty()
    plan.run(a, full, 4 * m + 2, m, workspace=ws)
    plan.run(a, mid, 2 * m, m, workspace=ws)
    plan.run(mid, res, 2 * m + 2, m, workspace=ws)
    torch.cuda.synchronize()
    if nd > 1:
        assert torch.equal(plan.frame_view(full), plan.frame_view(res))
    else:   # 1D: which warps take the exact stepwise path depends on the launch's step count
        err = (plan.frame_view(full).double() - plan.frame_view(res).double()).abs().max().item()
        assert err <= TOL[dtype]
    plan.run(a, mid, 2 * m + 1, m, workspace=ws)
    plan.run(mid, res, 2 * m + 1, m, workspace=ws)
    torch.cuda.synchronize()
    err = (plan.frame_view(full).double() - plan.frame_view(res).double()).abs().max().item()
    assert err <= TOL[dtype]


@pytest.mark.parametrize("dims,shape,dtype", [((70, 523), "star", "f64"), ((19, 37, 75), "box", "f64"),
                                              ((1000,), "star", "f64")])
def test_auto_fold_run(dims, shape, dtype):
    """fold_m = 0 runs the plan's auto fold and matches the oracle."""
    nd = len(dims)
    offs = oracle.taps(nd, 1, oracle.STAR if shape == "star" else oracle.BOX)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, 1, 2)
    ref = oracle.run(dims, 1, offs, w, u0, 9)
    plan = _plan(dims, shape, dtype, w)
    a = plan.from_frame(u0)
    b, ws = plan.empty(), plan.empty()
    plan.run(a, b, 9, 0, workspace=ws)
    torch.cuda.synchronize()
    assert np.max(np.abs(plan.frame_view(b).cpu().double().numpy() - ref)) <= TOL[dtype] * np.max(np.abs(u0))


@pytest.mark.parametrize("dims,shape,dtype,T,m", [
    ((70, 523), "star", "f64", 3, 4), ((70, 523), "box", "f32", 7, 4), ((70, 523), "star", "f64", 11, 4),
    ((19, 37, 75), "star", "f64", 3, 4), ((19, 37, 75), "box", "f64", 5, 2), ((19, 37, 75), "star", "f64", 1, 2)])
def test_remainder_sweeps(dims, shape, dtype, T, m):
    """T mod m != 0 (R10): the remainder runs as one sweep of lambda^(T mod m) where
    that fold is compiled (2D: 3 -> lambda^(3)), else as single steps (3D: 3);
    T < m has no full sweep at all (so 3D T=3, m=4 runs although no 3D
    evaluation of fold 4 is compiled)."""
    got, ref, u0, _ = run_case(dims, shape, dtype, T, m, 0)
    assert np.max(np.abs(got - ref)) <= TOL[dtype] * np.max(np.abs(u0))


def test_uncompiled_fold_is_unsupported():
    from paper_2103_09235_b200 import StencilError
    with pytest.raises(StencilError):
        run_case((19, 37, 75), "box", "f64", 7, 4, 0)      # 3D fold 4: not compiled


# The exact boundary band (K-G3) under stress: band boxes cut into
# several ragged blocks along every axis (the 64-cell block cap and the shared-memory
# fit), bands thicker than half an axis (the main region empty along it), and domains
# that are all band.
@pytest.mark.parametrize("dims,shape,dtype,m,T", [
    ((3, 70, 130), "star", "f64", 2, 5), ((70, 3, 130), "box", "f32", 2, 4),
    ((67, 66, 3), "star", "f64", 2, 4), ((2, 40, 41), "box", "f64", 2, 6),
    ((5, 5, 5), "star", "f32", 2, 7), ((4, 600), "star", "f64", 4, 9),
    ((600, 5), "box", "f32", 4, 8), ((130, 300), "box", "f64", 3, 7)])
def test_band_geometry(dims, shape, dtype, m, T):
    got, ref, u0, _ = run_case(dims, shape, dtype, T, m, 1)
    assert np.max(np.abs(got - ref)) <= TOL[dtype] * np.max(np.abs(u0))
