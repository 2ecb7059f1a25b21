"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test pins a part of ``oracle/`` to something other than itself:
matrix powers of the affine step operator (numpy fp64 and exact Fractions on
dyadic inputs), the periodic Fourier-mode closed form, constant fields, the
paper's worked folding example, closed forms of the fold,
impulse responses, and the exactness of the dependency-cone window.
"""
import itertools
import math
from fractions import Fraction

import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden

RNG = np.random.default_rng(12345)


def _interior_index(dims):
    return list(itertools.product(*[range(n) for n in dims]))


def _affine_operator(dims, r, offs, w, u0):
    """Build the (n+1)x(n+1) augmented step matrix from the DEFINITION
    u'[p] = sum_j w_j u[p+o_j] with the ring frozen at u0 (reading R1):
    interior->interior couplings plus a constant column from ring cells."""
    pts = _interior_index(dims)
    pos = {p: i for i, p in enumerate(pts)}
    n = len(pts)
    M = [[0.0] * (n + 1) for _ in range(n + 1)]
    for p in pts:
        i = pos[p]
        for o, wj in zip(offs, w):
            q = tuple(p[a] + o[a] for a in range(len(dims)))
            if q in pos:
                M[i][pos[q]] += wj
            else:  # ring cell: frozen u0 value (padded coords = q + r)
                M[i][n] += wj * u0[tuple(c + r for c in q)]
    M[n][n] = 1.0
    return M, pts


@pytest.mark.parametrize("dims,shape", [((7,), oracle.STAR), ((6, 5), oracle.STAR),
                                        ((6, 5), oracle.BOX), ((3, 4, 5), oracle.STAR),
                                        ((3, 4, 5), oracle.BOX)])
def test_matrix_power_fixed(dims, shape):
    r = 1
    offs = oracle.taps(len(dims), r, shape)
    w = RNG.uniform(0.1, 1.0, len(offs))           # asymmetric, unnormalised
    w = w / w.sum()
    P = tuple(n + 2 * r for n in dims)
    u0 = RNG.uniform(-1, 1, P)
    T = 9
    M, pts = _affine_operator(dims, r, offs, w, u0)
    M = np.array(M)
    v = np.array([u0[tuple(c + r for c in p)] for p in pts] + [1.0])
    vT = np.linalg.matrix_power(M, T) @ v
    got = oracle.run(dims, r, offs, w, u0, T)
    for i, p in enumerate(pts):
        assert abs(got[tuple(c + r for c in p)] - vT[i]) <= 1e-13
    # ring untouched
    mask = np.ones(P, bool)
    mask[tuple(slice(r, r + n) for n in dims)] = False
    assert np.array_equal(got[mask], u0[mask])


@pytest.mark.parametrize("dims,shape,T", [((7,), oracle.STAR, 7), ((6, 6), oracle.BOX, 3),
                                          ((5, 4), oracle.STAR, 5), ((3, 3, 4), oracle.BOX, 2),
                                          ((3, 4, 4), oracle.STAR, 4)])
def test_exact_dyadic_fractions(dims, shape, T):
    """Dyadic weights (k/64, sum exactly 1) and u0 (k/256): every partial sum is
    representable, so fp64 must equal the exact rational result bit for bit."""
    r = 1
    offs = oracle.taps(len(dims), r, shape)
    w = synth.dyadic_weights(len(offs), seed=7)
    P = tuple(n + 2 * r for n in dims)
    u0 = synth.dyadic_field(P, seed=11)
    Mf, pts = _affine_operator(dims, r, offs, [Fraction(x) for x in w],
                               np.vectorize(Fraction, otypes=[object])(u0))
    v = [Fraction(u0[tuple(c + r for c in p)]) for p in pts] + [Fraction(1)]
    for _ in range(T):
        v = [sum((Mf[i][j] * v[j] for j in range(len(v)) if Mf[i][j] != 0), Fraction(0))
             for i in range(len(v))]
    got = oracle.run(dims, r, offs, w, u0, T)
    for i, p in enumerate(pts):
        assert Fraction(got[tuple(c + r for c in p)]) == v[i]


@pytest.mark.parametrize("dims,shape", [((16,), oracle.STAR), ((12, 10), oracle.BOX),
                                        ((12, 10), oracle.STAR), ((6, 8, 10), oracle.STAR),
                                        ((6, 8, 10), oracle.BOX)])
def test_fourier_mode_periodic(dims, shape):
    """u0 = cos/sin(theta . x) with theta = 2 pi k / N; after T periodic steps
    u_T + i v_T = sigma(theta)^T e^{i theta . x}, sigma = sum_j w_j e^{i theta . o_j}."""
    r = 1
    nd = len(dims)
    offs = oracle.taps(nd, r, shape)
    w = RNG.uniform(0.2, 1.0, len(offs))
    w = w / w.sum()
    k = [1 + (a % 2) for a in range(nd)]
    theta = np.array([2 * math.pi * k[a] / dims[a] for a in range(nd)])
    P = tuple(n + 2 * r for n in dims)
    grids = np.meshgrid(*[np.arange(n) - r for n in P], indexing="ij")
    phase = sum(theta[a] * grids[a] for a in range(nd))
    T = 10
    uc = oracle.run(dims, r, offs, w, np.cos(phase), T, oracle.PERIODIC)
    us = oracle.run(dims, r, offs, w, np.sin(phase), T, oracle.PERIODIC)
    sigma = sum(wj * np.exp(1j * float(np.dot(theta, o))) for o, wj in zip(offs, w))
    expect = sigma ** T * np.exp(1j * phase)
    assert np.max(np.abs(uc - expect.real)) < 1e-13
    assert np.max(np.abs(us - expect.imag)) < 1e-13


@pytest.mark.parametrize("nd,shape", [(1, oracle.STAR), (2, oracle.STAR), (2, oracle.BOX),
                                      (3, oracle.STAR), (3, oracle.BOX)])
def test_constant_field(nd, shape):
    dims = [9, 7, 5][:nd]
    r = 1
    offs = oracle.taps(nd, r, shape)
    w = synth.weights(len(offs), 3)
    c = 0.7
    P = tuple(n + 2 * r for n in dims)
    T = 25
    got = oracle.run(dims, r, offs, w, np.full(P, c), T)
    assert np.max(np.abs(got - c)) <= T * (len(offs) + 1) * 2.0 ** -53 * c * 2


def test_canonical_taps():
    assert oracle.taps(2, 1, oracle.STAR) == [(-1, 0), (0, -1), (0, 0), (0, 1), (1, 0)]
    assert oracle.taps(3, 1, oracle.STAR) == [(-1, 0, 0), (0, -1, 0), (0, 0, -1), (0, 0, 0),
                                              (0, 0, 1), (0, 1, 0), (1, 0, 0)]
    assert len(oracle.taps(2, 1, oracle.BOX)) == 9
    assert len(oracle.taps(3, 1, oracle.BOX)) == 27
    assert len(oracle.taps(1, 2, oracle.STAR)) == 5


def test_fold_paper_worked_example():
    """uniform 2D9P, m=2 -> counterparts {1,2,3,2,1} x {1,2,3}."""
    golden = np.array([[float(x) for x in row] for row in read_golden("fold_2d9p_uniform_m2.txt")])
    lam = oracle.fold_ref(np.ones((3, 3)), 2)
    assert np.array_equal(lam, golden)
    # counterpart rows: column t carries lambda^(c-|t|), lambda^(n) = n lambda^(1)
    lam1 = golden[:, 0]
    assert list(lam1) == [1, 2, 3, 2, 1]
    for t in range(-2, 3):
        assert np.array_equal(golden[:, t + 2], (3 - abs(t)) * lam1)


def test_fold_profitability_collects():
    """|C(E)| = 90 for the naive 2-step 2D9P (10 sub-expressions
    of 9 taps), |C(E_Lambda)| = 25 = support of lambda^(2), P = 3.6."""
    g = {row[0]: float(row[1]) for row in read_golden("profitability_2d9p_m2.txt")}
    w = np.ones((3, 3))
    lam = oracle.fold_ref(w, 2)
    support = int(np.count_nonzero(lam))
    # naive: one sub-expression per t+1 point feeding the centre, plus the centre
    naive = (int(np.count_nonzero(oracle.fold_ref(w, 1))) + 1) * 9
    assert naive == g["collect_naive"]
    assert support == g["collect_folded"]
    assert naive / support == pytest.approx(g["profitability"])


def test_fold_1d3p_closed_form():
    a, b, c = 0.3, 0.45, 0.25
    lam = oracle.fold_ref(np.array([a, b, c]), 2)
    assert np.allclose(lam, [a * a, 2 * a * b, b * b + 2 * a * c, 2 * b * c, c * c], rtol=0, atol=1e-16)


@pytest.mark.parametrize("nd,shape,m,support", [
    (1, oracle.STAR, 2, 5), (2, oracle.STAR, 2, 13), (2, oracle.STAR, 4, 41),
    (2, oracle.BOX, 2, 25), (2, oracle.BOX, 4, 81), (3, oracle.STAR, 2, 25),
    (3, oracle.BOX, 2, 125)])
def test_fold_support_and_sum(nd, shape, m, support):
    offs = oracle.taps(nd, 1, shape)
    w = synth.weights(len(offs), 5)
    lam = oracle.fold_ref(oracle.dense_from_taps(nd, 1, offs, w), m)
    assert lam.shape == (2 * m + 1,) * nd
    assert int(np.count_nonzero(lam)) == support
    assert lam.sum() == pytest.approx(w.sum() ** m, abs=1e-14)


def test_fold_semigroup_and_symbol():
    offs = oracle.taps(2, 1, oracle.BOX)
    w = RNG.uniform(0.1, 1.0, len(offs))
    W = oracle.dense_from_taps(2, 1, offs, w)
    l2, l3, l5 = (oracle.fold_ref(W, m) for m in (2, 3, 5))
    assert np.allclose(oracle.convolve_full(l2, l3), l5, rtol=0, atol=1e-13)
    for _ in range(5):
        th = RNG.uniform(-math.pi, math.pi, 2)
        sig = sum(W[i, j] * np.exp(1j * (th[0] * (i - 1) + th[1] * (j - 1)))
                  for i in range(3) for j in range(3))
        sl = sum(l5[i, j] * np.exp(1j * (th[0] * (i - 5) + th[1] * (j - 5)))
                 for i in range(11) for j in range(11))
        assert abs(sl - sig ** 5) < 1e-14 * W.sum() ** 5


def test_impulse_response():
    golden = [float(x) for x in read_golden("impulse_1d3p_uniform_T2.txt")[0]]
    n = 21
    u0 = np.zeros(n + 2)
    u0[1 + 10] = 1.0
    got = oracle.run([n], 1, oracle.taps(1, 1, oracle.STAR), [1.0, 1.0, 1.0], u0, 2)
    assert list(got[1 + 8:1 + 13]) == golden
    # asymmetric weights: response is the MIRRORED T-fold kernel (correlation form)
    w = [0.2, 0.5, 0.3]
    got = oracle.run([n], 1, oracle.taps(1, 1, oracle.STAR), w, u0, 3)
    lam = oracle.fold_ref(np.array(w), 3)
    assert np.allclose(got[1 + 7:1 + 14], lam[::-1], rtol=0, atol=1e-16)
    assert not np.allclose(lam, lam[::-1])


def _apply_dense_once(u0, lam, dims, r, m):
    """Apply a dense (2mr+1)^d map once at interior points (test helper)."""
    nd = len(dims)
    R = m * r
    out = np.array(u0, copy=True)
    for p in _interior_index(dims):
        acc = 0.0
        for idx in itertools.product(*[range(2 * R + 1)] * nd):
            v = lam[idx]
            if v == 0.0:
                continue
            q = tuple(p[a] + r + idx[a] - R for a in range(nd))
            if all(0 <= q[a] < dims[a] + 2 * r for a in range(nd)):
                acc += v * u0[q]
            else:
                acc = float("nan")
        out[tuple(c + r for c in p)] = acc
    return out


@pytest.mark.parametrize("nd,shape,m", [(1, oracle.STAR, 2), (2, oracle.STAR, 2),
                                        (2, oracle.BOX, 4), (3, oracle.STAR, 2)])
def test_fold_equals_steps_away_from_fixed_boundary(nd, shape, m):
    """Reading R2: m stepwise steps == one folded application at distance
    >= (m-1) r from every face; they differ inside that band."""
    r = 1
    dims = [13, 11, 9][:nd]
    offs = oracle.taps(nd, r, shape)
    w = RNG.uniform(0.1, 1.0, len(offs))
    w = w / w.sum()
    P = tuple(n + 2 * r for n in dims)
    u0 = RNG.uniform(0, 1, P)
    step = oracle.run(dims, r, offs, w, u0, m)
    lam = oracle.fold_ref(oracle.dense_from_taps(nd, r, offs, w), m)
    fold = _apply_dense_once(u0, lam, dims, r, m)
    band = (m - 1) * r
    for p in _interior_index(dims):
        q = tuple(c + r for c in p)
        dist = min(min(p[a], dims[a] - 1 - p[a]) for a in range(nd))
        if dist >= band:
            assert abs(step[q] - fold[q]) < 1e-14
        elif dist == 0:
            assert not (abs(step[q] - fold[q]) < 1e-14)


@pytest.mark.parametrize("nd,shape,dims,T", [(2, oracle.STAR, (64, 70), 11),
                                             (3, oracle.BOX, (20, 18, 22), 5)])
def test_window_is_bit_identical(nd, shape, dims, T):
    r = 1
    offs = oracle.taps(nd, r, shape)
    w = synth.weights(len(offs), 1)
    u0 = synth.u0_frame(dims, r, 2)
    full = oracle.run(dims, r, offs, w, u0, T)
    for lo in ([0] * nd, [d // 2 for d in dims], [d - 3 for d in dims]):
        hi = [min(l + 3, d) for l, d in zip(lo, dims)]
        sl = tuple(slice(l + r, h + r) for l, h in zip(lo, hi))
        for cone in (False, True):
            got = oracle.run_window(dims, r, offs, w, T, lo, hi,
                                    lambda a, b: synth.u0_block(dims, r, a, b, 2), cone=cone)
            assert np.array_equal(got, full[sl])


def test_generator_counter_form_is_sequential_splitmix64():
    seq = synth.splitmix64_sequence(2, 50)
    assert np.array_equal(synth.uniform(2, np.arange(50)), seq)
    w = synth.weights(9, 1)
    assert abs(sum(w) - 1.0) < 1e-15 and (w > 0).all()
    u = synth.u0_frame((5, 6), 1, 2)
    assert u.shape == (7, 8)
    assert np.array_equal(u.ravel(), synth.uniform(2, np.arange(56)))


# ---------------------------------------------------------------- radius > 1
# The same four pins at r = 2 (and r = 3, 4 in 1D): the 1D5P workload of
# Table 1 and the radius-2 stencils of NEXT-4.  The ring is r
# wide; every tap reaches at most r cells, so the affine operator, the exact
# rational run and the Fourier closed form are built the same way as for r = 1.

@pytest.mark.parametrize("dims,r,shape", [((9,), 2, oracle.STAR), ((11,), 3, oracle.STAR),
                                          ((12,), 4, oracle.STAR), ((6, 7), 2, oracle.STAR),
                                          ((5, 6), 2, oracle.BOX), ((4, 5, 6), 2, oracle.STAR),
                                          ((3, 4, 5), 2, oracle.BOX)])
def test_matrix_power_fixed_radius(dims, r, shape):
    offs = oracle.taps(len(dims), r, shape)
    assert len(offs) == (2 * len(dims) * r + 1 if shape == oracle.STAR else (2 * r + 1) ** len(dims))
    w = RNG.uniform(0.1, 1.0, len(offs))
    w = w / w.sum()
    P = tuple(n + 2 * r for n in dims)
    u0 = RNG.uniform(-1, 1, P)
    T = 7
    M, pts = _affine_operator(dims, r, offs, w, u0)
    M = np.array(M)
    v = np.array([u0[tuple(c + r for c in p)] for p in pts] + [1.0])
    vT = np.linalg.matrix_power(M, T) @ v
    got = oracle.run(dims, r, offs, w, u0, T)
    for i, p in enumerate(pts):
        assert abs(got[tuple(c + r for c in p)] - vT[i]) <= 1e-13
    mask = np.ones(P, bool)
    mask[tuple(slice(r, r + n) for n in dims)] = False
    assert np.array_equal(got[mask], u0[mask])


@pytest.mark.parametrize("dims,r,shape,T", [((10,), 2, oracle.STAR, 6), ((6, 5), 2, oracle.STAR, 4),
                                            ((5, 5), 2, oracle.BOX, 3), ((3, 4, 4), 2, oracle.STAR, 3)])
def test_exact_dyadic_fractions_radius(dims, r, shape, T):
    """Bitwise equality with exact rational arithmetic at r = 2 (dyadic inputs)."""
    offs = oracle.taps(len(dims), r, shape)
    w = synth.dyadic_weights(len(offs), seed=9)
    P = tuple(n + 2 * r for n in dims)
    u0 = synth.dyadic_field(P, seed=13)
    Mf, pts = _affine_operator(dims, r, offs, [Fraction(x) for x in w],
                               np.vectorize(Fraction, otypes=[object])(u0))
    v = [Fraction(u0[tuple(c + r for c in p)]) for p in pts] + [Fraction(1)]
    for _ in range(T):
        v = [sum((Mf[i][j] * v[j] for j in range(len(v)) if Mf[i][j] != 0), Fraction(0))
             for i in range(len(v))]
    got = oracle.run(dims, r, offs, w, u0, T)
    for i, p in enumerate(pts):
        assert Fraction(got[tuple(c + r for c in p)]) == v[i]


@pytest.mark.parametrize("dims,r,shape", [((20,), 2, oracle.STAR), ((24,), 3, oracle.STAR),
                                          ((12, 14), 2, oracle.STAR), ((10, 12), 2, oracle.BOX),
                                          ((8, 10, 12), 2, oracle.STAR), ((6, 8, 10), 2, oracle.BOX)])
def test_fourier_mode_periodic_radius(dims, r, shape):
    """Periodic Fourier mode at r > 1: the r-wide wrapped ring must carry the
    interior cells r away, or sigma(theta)^T fails."""
    nd = len(dims)
    offs = oracle.taps(nd, r, shape)
    w = RNG.uniform(0.2, 1.0, len(offs))
    w = w / w.sum()
    k = [1 + (a % 2) for a in range(nd)]
    theta = np.array([2 * math.pi * k[a] / dims[a] for a in range(nd)])
    P = tuple(n + 2 * r for n in dims)
    grids = np.meshgrid(*[np.arange(n) - r for n in P], indexing="ij")
    phase = sum(theta[a] * grids[a] for a in range(nd))
    T = 8
    uc = oracle.run(dims, r, offs, w, np.cos(phase), T, oracle.PERIODIC)
    us = oracle.run(dims, r, offs, w, np.sin(phase), T, oracle.PERIODIC)
    sigma = sum(wj * np.exp(1j * float(np.dot(theta, o))) for o, wj in zip(offs, w))
    expect = sigma ** T * np.exp(1j * phase)
    assert np.max(np.abs(uc - expect.real)) < 1e-13
    assert np.max(np.abs(us - expect.imag)) < 1e-13


@pytest.mark.parametrize("nd,r,shape,bc", [(1, 2, oracle.STAR, oracle.FIXED), (1, 4, oracle.STAR, oracle.PERIODIC),
                                           (2, 2, oracle.STAR, oracle.FIXED), (2, 2, oracle.BOX, oracle.PERIODIC),
                                           (3, 2, oracle.STAR, oracle.FIXED), (3, 2, oracle.BOX, oracle.FIXED)])
def test_constant_field_radius(nd, r, shape, bc):
    dims = [9, 7, 6][:nd]
    offs = oracle.taps(nd, r, shape)
    w = synth.weights(len(offs), 3)
    c = 0.7
    P = tuple(n + 2 * r for n in dims)
    T = 20
    got = oracle.run(dims, r, offs, w, np.full(P, c), T, bc)
    assert np.max(np.abs(got - c)) <= T * (len(offs) + 1) * 2.0 ** -53 * c * 2


def test_radius2_fold_equals_steps_away_from_boundary():
    """R2/R8 at r = 2: one application of lambda^(2) (reach 2r) equals two steps
    at distance >= (m-1) r = 2 from every FIXED face, and differs at distance 0."""
    r, m, dims = 2, 2, [14, 13]
    offs = oracle.taps(2, r, oracle.STAR)
    w = RNG.uniform(0.1, 1.0, len(offs))
    w = w / w.sum()
    P = tuple(n + 2 * r for n in dims)
    u0 = RNG.uniform(0, 1, P)
    step = oracle.run(dims, r, offs, w, u0, m)
    lam = oracle.fold_ref(oracle.dense_from_taps(2, r, offs, w), m)
    assert lam.shape == (4 * r + 1,) * 2
    fold = _apply_dense_once(u0, lam, dims, r, m)
    for p in _interior_index(dims):
        q = tuple(c + r for c in p)
        dist = min(min(p[a], dims[a] - 1 - p[a]) for a in range(2))
        if dist >= (m - 1) * r:
            assert abs(step[q] - fold[q]) < 1e-14
        elif dist == 0:
            assert not (abs(step[q] - fold[q]) < 1e-14)
