"""CPU-side tests of the C-ABI library: it loads, exports every symbol the
header declares, validates arguments, and its host-side coefficient-folding
generator agrees with the (independently written, pinned) oracle fold.
No compute call here needs a GPU."""
import os
import re
import subprocess

import numpy as np
import pytest

import oracle
import synth
from paper_2103_09235_b200 import _lib
from paper_2103_09235_b200 import Plan, StencilError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stencil_b200.h")


def header_symbols():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(stencil_[a-z_0-9]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = _lib.load()
    syms = header_symbols()
    assert len(syms) >= 20
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    for s in syms:
        assert s in exported, s
        assert hasattr(lib, s)
    # the binding mirrors the header one to one
    assert sorted(_lib.SIGNATURES) == syms


def test_version_and_error_channel():
    lib = _lib.load()
    assert b"sm_100a" in lib.stencil_version()
    with pytest.raises(StencilError) as e:
        Plan((8, 8), 1, "star", [1.0] * 4)      # 2D STAR needs 5 taps
    assert e.value.code == -1 and "canonical tap count 5" in str(e.value)


@pytest.mark.parametrize("bad", [dict(dims=(0, 8)), dict(radius=0), dict(dims=(4, 4, 4, 4))])
def test_plan_create_rejects(bad):
    kw = dict(dims=(8, 8), radius=1, shape="star", coeffs=[0.2] * 5)
    kw.update(bad)
    with pytest.raises((StencilError, KeyError, ValueError)):
        Plan(**kw)


def test_canonical_taps_match_oracle():
    for nd in (1, 2, 3):
        for shape in ("star", "box"):
            k = len(oracle.taps(nd, 1, 0 if shape == "star" else 1))
            p = Plan((5,) * nd, 1, shape, synth.weights(k, 1))
            assert p.taps() == oracle.taps(nd, 1, 0 if shape == "star" else 1)


@pytest.mark.parametrize("nd,shape,m", [(1, "star", 2), (1, "star", 5), (2, "star", 2), (2, "star", 4),
                                        (2, "box", 2), (2, "box", 4), (3, "star", 2), (3, "box", 2),
                                        (2, "star", 3), (1, "star", 8)])
def test_fold_generator_matches_oracle_fold(nd, shape, m):
    sh = 0 if shape == "star" else 1
    offs = oracle.taps(nd, 1, sh)
    w = synth.weights(len(offs), 9)
    p = Plan((7,) * nd, 1, shape, w)
    lib_lam = p.fold_coeffs(m)
    ref = oracle.fold_ref(oracle.dense_from_taps(nd, 1, offs, w), m)
    assert lib_lam.shape == ref.shape
    assert np.max(np.abs(lib_lam - ref)) <= 1e-15 * np.abs(ref).sum()
    assert np.count_nonzero(lib_lam) == np.count_nonzero(ref)


def test_fold_generator_paper_example_exact():
    """Integer weights: exact agreement with the paper's worked example."""
    from conftest import read_golden
    golden = np.array([[float(x) for x in row] for row in read_golden("fold_2d9p_uniform_m2.txt")])
    p = Plan((5, 5), 1, "box", [1.0] * 9)
    assert np.array_equal(p.fold_coeffs(2), golden)
    with pytest.raises(StencilError):
        p.fold_coeffs(0)


def test_layout_alignment_and_views():
    import torch
    for dt, es in (("f64", 8), ("f32", 4)):
        p = Plan((100, 37), 1, "star", synth.weights(5, 1), dtype=dt)
        L = p.layout
        assert L.elem_bytes == es
        assert (L.origin[-1] * es) % 128 == 0          # interior x = 0 is 128-byte aligned
        assert (L.stride[0] * es) % 128 == 0           # row pitch multiple of 128 bytes
        assert L.extent[0] == 102 and L.origin[0] == 1
        buf = p.empty("cpu")
        fr = p.frame_view(buf)
        assert tuple(fr.shape) == (102, 39)
        u0 = synth.u0_frame((100, 37), 1, 2)
        b2 = p.from_frame(u0, "cpu")
        assert np.array_equal(p.frame_view(b2).numpy(), u0.astype(np.float64 if dt == "f64" else np.float32))
        assert torch.count_nonzero(b2) == np.count_nonzero(u0)


def test_dist_layout():
    p = Plan((64, 32, 16), 1, "star", synth.weights(7, 1))
    with pytest.raises(StencilError):
        p.layout_dist(0, 3, 2)          # 64 not divisible by 3
    L0 = p.layout_dist(0, 4, 2)
    L3 = p.layout_dist(3, 4, 2)
    assert L0.interior[0] == 16 and L0.origin[0] == 2 and L0.extent[0] == 20
    assert L3.global_offset0 == 48


def test_periodic_layout_has_ghost_ring():
    """PERIODIC plans (NEXT-4): a ghost ring of STENCIL_MAX_FOLD * r cells on
    every axis (refilled from the wrapped interior after every sweep)."""
    for r in (1, 2):
        k = len(oracle.taps(2, r, oracle.BOX))
        p = Plan((40, 30), r, "box", synth.weights(k, 1), boundary="periodic")
        L = p.layout
        G = 8 * r
        assert L.origin[0] == G and L.extent[0] == 40 + 2 * G
        assert L.origin[1] >= G and L.extent[1] >= L.origin[1] + 30 + G
        assert (L.origin[1] * L.elem_bytes) % 128 == 0
        # the frame view (interior + r-ring) still has the oracle's shape
        assert tuple(p.frame_view(p.empty("cpu")).shape) == (40 + 2 * r, 30 + 2 * r)
    with pytest.raises(StencilError):
        Plan((64, 32), 1, "star", synth.weights(5, 1), boundary="periodic").layout_dist(0, 2, 2)


# ------------------------------------------------------------ counterparts (NEXT-3)
def test_counterparts_paper_example_rank_one():
    """The paper's uniform 2D9P, m = 2: every column of Lambda is a
    multiple of lambda^(1) = {1,2,3,2,1} (the counterparts lambda^(2) = 2 lambda^(1),
    lambda^(3) = 3 lambda^(1)), i.e. Lambda has rank 1 and one counterpart suffices."""
    from conftest import read_golden
    golden = np.array([[float(x) for x in row] for row in read_golden("fold_2d9p_uniform_m2.txt")])
    p = Plan((64, 64), 1, "box", [1.0] * 9)
    rank, a, b = p.fold_rank(2)
    assert rank == 1
    lam1 = np.array([1.0, 2.0, 3.0, 2.0, 1.0])
    # the counterpart's vertical and horizontal weights are both multiples of lambda^(1)
    assert np.allclose(a[0] / a[0][2], lam1 / 3.0, rtol=0, atol=1e-15)
    assert np.allclose(b[0] / b[0][2], lam1 / 3.0, rtol=0, atol=1e-15)
    assert np.allclose(np.outer(a[0], b[0]), golden, rtol=0, atol=1e-13)
    # the plan's profitability choice (GPU Eq.3): 2 W rank = 10 FMAs < |supp| = 25
    assert p.variant(2) == (2, 1, 1)
    assert p.variant(4) == (4, 1, 1)     # 18 < 81


@pytest.mark.parametrize("m", [1, 2, 4])
def test_counterparts_separable_and_full_rank(m):
    rng = np.random.default_rng(7)
    u, v = rng.uniform(0.5, 1.5, 3), rng.uniform(0.5, 1.5, 3)
    w_sep = np.outer(u, v).ravel()                        # separable box weights
    p = Plan((64, 64), 1, "box", w_sep)
    rank, a, b = p.fold_rank(m)
    assert rank == 1
    lam = p.fold_coeffs(m)
    assert np.max(np.abs(np.einsum("ki,kj->ij", a, b) - lam)) <= 1e-14 * np.max(np.abs(lam))
    # rank 2: a sum of two separable kernels
    u2, v2 = rng.uniform(0.5, 1.5, 3), rng.uniform(0.5, 1.5, 3)
    w2 = (np.outer(u, v) + np.outer(u2, v2)).ravel()
    r2, a2, b2 = Plan((64, 64), 1, "box", w2).fold_rank(m)
    lam2 = Plan((64, 64), 1, "box", w2).fold_coeffs(m)
    # (A + B)^{*m} = sum_i C(m,i) A^{*i} B^{*(m-i)}: m + 1 separable terms at most
    assert r2 <= m + 1 and np.allclose(np.einsum("ki,kj->ij", a2, b2), lam2, rtol=0,
                                                      atol=1e-13 * np.max(lam2))
    # generic random weights: full rank, so the dense folded pass is kept
    pr = Plan((64, 64), 1, "box", synth.weights(9, 1))
    assert pr.fold_rank(m)[0] == 2 * m + 1
    assert pr.variant(m)[2] == 0


def test_counterparts_can_be_disabled():
    p = Plan((64, 64), 1, "box", [1.0 / 9] * 9)
    assert p.variant(2)[2] == 1
    p.set_counterparts(False)
    assert p.variant(2)[2] == 0


def test_new_entry_points_validate_arguments():
    """Argument checks of the NEXT-2/3 entry points that need no GPU."""
    import ctypes
    lib = _lib.load()
    p3 = Plan((8, 8, 8), 1, "star", synth.weights(7, 1))
    with pytest.raises(StencilError):
        p3.fold_rank(2)                                  # counterparts are 2D
    p2 = Plan((16, 16), 1, "box", synth.weights(9, 1))
    with pytest.raises(StencilError):
        p2.fold_rank(0)
    with pytest.raises(StencilError):
        p2.variant(0)
    with pytest.raises(StencilError):
        p2.perturb_fold(2, 25, 1.0)                      # 5x5 = 25 entries: index 25 is out of range
    p2.perturb_fold(2, 12, 0.0)                          # in range, no-op
    r = ctypes.c_int()
    assert lib.stencil_plan_variant(p2._h, 2, None, None, None) == -1
    assert lib.stencil_plan_fold_rank(p2._h, 2, None, None, None, 0) == -1
    h = ctypes.c_void_p()
    assert lib.stencil_comm_create_peer(ctypes.byref(h), 0, 2, None, None) == -1
    assert lib.stencil_comm_create_peer(ctypes.byref(h), 2, 2, ctypes.c_void_p(256), ctypes.c_void_p(512)) == -1
    assert lib.stencil_comm_peer_handles(None, ctypes.create_string_buffer(216)) == -1
    assert lib.stencil_comm_peer_attach(None, ctypes.create_string_buffer(216)) == -1
    del r


def test_auto_fold_table():
    """fold_m = 0 (auto): the measured-best fold per family."""
    assert Plan((100,), 1, "star", synth.weights(3, 1)).auto_fold() == 2
    assert Plan((64, 64), 1, "star", synth.weights(5, 1)).auto_fold() == 6             # temporal block (fp64 star)
    assert Plan((64, 64), 1, "star", synth.weights(5, 1), dtype="f32").auto_fold() == 8
    assert Plan((64, 64), 1, "box", synth.weights(9, 1), dtype="f32").auto_fold() == 8
    assert Plan((64, 64), 1, "box", [1.0 / 9] * 9, dtype="f32").auto_fold() == 4      # counterparts
    assert Plan((64, 64), 1, "star", synth.weights(5, 1), boundary="periodic").auto_fold() == 3
    assert Plan((64, 64), 1, "box", synth.weights(9, 1), boundary="periodic").auto_fold() == 2
    # variant policy: temporal block (q = 1, stages = m) for m >= 4 (stars) / m >= 3 (boxes)
    st = Plan((64, 64), 1, "star", synth.weights(5, 1))
    bx = Plan((64, 64), 1, "box", synth.weights(9, 1), dtype="f32")
    assert st.variant(3) == (3, 1, 0) and st.variant(4) == (1, 4, 0) and st.variant(8) == (1, 8, 0)
    assert bx.variant(2) == (2, 1, 0) and bx.variant(3) == (1, 3, 0)
    assert Plan((16, 16, 16), 1, "star", synth.weights(7, 1)).auto_fold() == 4          # temporal block (tb3d)
    f3 = Plan((16, 16, 16), 1, "star", synth.weights(7, 1), dtype="f32")
    assert f3.auto_fold() == 4 and f3.variant(4) == (1, 4, 0) and f3.variant(3) == (3, 1, 0)   # tb3d fp32 from m = 4
    assert Plan((16, 16, 16), 1, "star", synth.weights(7, 1), dtype="f32", boundary="periodic").auto_fold() == 2
    s3 = Plan((16, 16, 16), 1, "star", synth.weights(7, 1))
    assert s3.variant(2) == (2, 1, 0) and s3.variant(3) == (1, 3, 0) and s3.variant(4) == (1, 4, 0)
    b3 = Plan((16, 16, 16), 1, "box", synth.weights(27, 1))
    assert b3.auto_fold() == 2 and b3.variant(2) == (1, 2, 0)                             # temporal block (tb3d box)
    assert Plan((16, 16, 16), 1, "box", synth.weights(27, 1), dtype="f32").auto_fold() == 1
    assert Plan((16, 16, 16), 1, "box", synth.weights(27, 1), boundary="periodic").auto_fold() == 1
