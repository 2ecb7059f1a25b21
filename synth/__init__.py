"""Seeded synthetic inputs shared by the oracle side and the product side.

This module holds NONE of the method's arithmetic (no stencil, no folding,
no tap enumeration).  It only turns (seed, counter) into numbers, so that the
oracle tests, the GPU parity tests and ``bench.py`` all see the same inputs.

Generator (reading R6; SURVEY.md §8(c) ambiguity #6):

    U(s, i) = (mix64(s + (i + 1) * 0x9E3779B97F4A7C15) >> 11) * 2**-53

which is exactly the i-th output of a sequential splitmix64 seeded with ``s``
(counter form, so every slab / window / rank can generate its own part).

* ``u0`` value at a grid position is ``U(seed_u, i)`` where ``i`` is the
  row-major linear index of the position in the UNALIGNED padded frame
  ``prod(N_a + 2r)`` (interior plus the r-wide ring, slowest axis first).
  Values therefore do not depend on the library's row pitch, on fold_m or on
  the GPU count.
* weights (reading R5): ``w~_j = 0.5 + U(seed_w, j)`` for j in the
  canonical tap order, ``w_j = w~_j / sum(w~)`` with the sum taken
  sequentially in tap order in fp64 — "seeded positive weights normalised to
  sum 1" / "uniform[0.5,1.5] normalised" of BASELINE.json's configs.

The CUDA library carries its own, independent implementation of the same
generator (``stencil_fill_random``); ``tests/test_gpu_parity.py`` checks the
two agree bit for bit.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
DEFAULT_SEED_W = 1
DEFAULT_SEED_U = 2


def _mix64(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def uniform(seed: int, idx: np.ndarray) -> np.ndarray:
    """U(seed, idx) in [0, 1) as float64, elementwise over integer ``idx``."""
    with np.errstate(over="ignore"):
        i = np.asarray(idx, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + (i + np.uint64(1)) * GAMMA
        bits = _mix64(z) >> np.uint64(11)
    return bits.astype(np.float64) * (2.0 ** -53)


def splitmix64_sequence(seed: int, n: int) -> np.ndarray:
    """Sequential splitmix64 (state += gamma; mix) — used by tests to show the
    counter form above is the textbook sequential generator."""
    out = np.empty(n, dtype=np.float64)
    state = seed & 0xFFFFFFFFFFFFFFFF
    for k in range(n):
        state = (state + 0x9E3779B97F4A7C15) & 0xFFFFFFFFFFFFFFFF
        z = state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        z = z ^ (z >> 31)
        out[k] = (z >> 11) * (2.0 ** -53)
    return out


def weights(ntaps: int, seed_w: int = DEFAULT_SEED_W) -> np.ndarray:
    """Seeded positive weights normalised to sum 1 (fp64), in tap order."""
    wt = 0.5 + uniform(seed_w, np.arange(ntaps))
    s = 0.0
    for v in wt:            # sequential, tap order (reading R5)
        s += float(v)
    return np.array([float(v) / s for v in wt], dtype=np.float64)


def padded_extents(dims, r: int):
    return tuple(int(n) + 2 * r for n in dims)


def u0_block(dims, r: int, lo, hi, seed_u: int = DEFAULT_SEED_U) -> np.ndarray:
    """u0 over the padded-frame box [lo, hi) (padded coordinates, 0 = first
    ring cell), fp64, C-order.  The whole frame is ``lo=0, hi=padded``."""
    P = padded_extents(dims, r)
    nd = len(P)
    axes = [np.arange(int(lo[a]), int(hi[a]), dtype=np.int64) for a in range(nd)]
    lin = np.zeros([len(a) for a in axes], dtype=np.int64)
    stride = 1
    for a in reversed(range(nd)):
        shape = [1] * nd
        shape[a] = len(axes[a])
        lin = lin + axes[a].reshape(shape) * stride
        stride *= P[a]
    return uniform(seed_u, lin)


def u0_frame(dims, r: int, seed_u: int = DEFAULT_SEED_U) -> np.ndarray:
    P = padded_extents(dims, r)
    return u0_block(dims, r, [0] * len(P), P, seed_u)


def dyadic_weights(ntaps: int, seed: int, denom_bits: int = 6) -> np.ndarray:
    """Positive weights that are multiples of 2**-denom_bits and sum to exactly 1
    (for exact-arithmetic pins).  Integer partition driven by the generator."""
    D = 1 << denom_bits
    if ntaps > D:
        raise ValueError("too many taps for this denominator")
    raw = 1.0 + uniform(seed, np.arange(ntaps))
    share = np.floor(raw / raw.sum() * (D - ntaps)).astype(np.int64) + 1
    share[int(np.argmax(share))] += D - int(share.sum())
    assert share.sum() == D and (share > 0).all()
    return share.astype(np.float64) / D


def dyadic_field(shape, seed: int, bits: int = 8) -> np.ndarray:
    """Values k * 2**-bits in [0, 1), exactly representable."""
    n = int(np.prod(shape))
    v = np.floor(uniform(seed, np.arange(n)) * (1 << bits)) / (1 << bits)
    return v.reshape(shape)
