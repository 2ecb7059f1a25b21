"""oracle — TEST INFRASTRUCTURE ONLY (see oracle.c header).

Plain fp64 CPU reference for arXiv 2103.09235's time-iterated stencil and its
temporal computation folding.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` leg may import this
package.  It shares no code with ``paper_2103_09235_b200`` and never imports
it (and vice versa).

Functions and the passages they follow:

* ``taps(nd, r, shape)`` — canonical tap offsets (reading R4; STAR /
  BOX as SPEC.md:31-32): offsets in [-r, r]^d, lexicographic, slowest axis
  outermost; STAR keeps offsets with at most one nonzero coordinate.
* ``run(...)`` — T naive steps, PAPER.md:64 (§1) and PAPER.md:410; the loops
  are in ``oracle.c``.
* ``fold_ref(w_dense, m)`` — the folding matrix lambda^(m) of Eq.2
  ("weights are all reassigned based on the m-step
  expansion"): the m-fold self-convolution of the tap map, computed as m-1
  repeated plain dense convolutions (offsets add, no mirroring, because
  composing two correlations adds offsets; reading R3).
* ``run_window(...)`` — the same ``run`` applied to a sub-window of the
  padded frame that contains the dependency cone of an output box; the
  per-point arithmetic is identical, so the box's values are bit-identical to
  a full-domain run (tests pin this).

Pins (tests/test_oracle_pins.py, ``-m "not gpu"``): matrix powers on tiny
grids (numpy fp64 and exact Fractions with dyadic inputs), the periodic
Fourier mode closed form, constant-field invariance, the paper's worked
folding example, 1D3P closed form, sum and semigroup and
symbol identities of the fold, impulse responses.
"""
from __future__ import annotations

import ctypes
import itertools
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

FIXED = 0
PERIODIC = 1
STAR = 0
BOX = 1


def build(force: bool = False) -> str:
    """Compile oracle.c with gcc (-O2 -ffp-contract=off -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp.%d" % os.getpid()
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC",
                               "-shared", "-std=c99", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            lib.oracle_run.restype = ctypes.c_int
            lib.oracle_run.argtypes = [
                ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_int,
                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double), ctypes.c_int,
                ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                ctypes.c_int]
            lib.oracle_run_cone.restype = ctypes.c_int
            lib.oracle_run_cone.argtypes = [
                ctypes.c_int, ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.c_int,
                ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double),
                ctypes.POINTER(ctypes.c_double), ctypes.c_int64, ctypes.POINTER(ctypes.c_int64),
                ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_double), ctypes.c_int]
            lib.oracle_max_threads.restype = ctypes.c_int
            _lib = lib
    return _lib


def max_threads() -> int:
    return int(_load().oracle_max_threads())


def taps(nd: int, r: int, shape: int):
    """Canonical taps: list of offset tuples (slowest axis first)."""
    out = []
    for o in itertools.product(range(-r, r + 1), repeat=nd):
        if shape == STAR and sum(1 for c in o if c != 0) > 1:
            continue
        out.append(tuple(o))
    return out


def dense_from_taps(nd: int, r: int, offs, w) -> np.ndarray:
    """Tap list -> dense (2r+1)^d coefficient array, index [o + r]."""
    D = np.zeros((2 * r + 1,) * nd, dtype=np.float64)
    for o, v in zip(offs, w):
        D[tuple(c + r for c in o)] = v
    return D


def convolve_full(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """Plain full convolution of two dense coefficient maps (offsets add)."""
    nd = a.ndim
    out = np.zeros(tuple(a.shape[k] + b.shape[k] - 1 for k in range(nd)), dtype=np.float64)
    for ia in itertools.product(*[range(s) for s in a.shape]):
        va = a[ia]
        if va == 0.0:
            continue
        for ib in itertools.product(*[range(s) for s in b.shape]):
            vb = b[ib]
            if vb == 0.0:
                continue
            idx = tuple(ia[k] + ib[k] for k in range(nd))
            out[idx] = out[idx] + va * vb
    return out


def fold_ref(w_dense: np.ndarray, m: int) -> np.ndarray:
    """lambda^(m) = w * w * ... * w (m factors), Eq.2 / PAPER.md:335.
    Returns the dense (2mr+1)^d array indexed by [o + m r]."""
    if m < 1:
        raise ValueError("fold_m must be >= 1 (SPEC.md:62)")
    lam = np.array(w_dense, dtype=np.float64)
    for _ in range(m - 1):
        lam = convolve_full(lam, w_dense)
    return lam


def run(dims, r: int, offs, w, u0: np.ndarray, T: int, boundary: int = FIXED,
        nthreads: int = 0) -> np.ndarray:
    """T naive steps on the padded frame ``u0`` (shape prod(dims+2r))."""
    lib = _load()
    nd = len(dims)
    P = tuple(int(n) + 2 * r for n in dims)
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    if u0.shape != P:
        raise ValueError("u0 must be the padded frame %s, got %s" % (P, u0.shape))
    out = np.empty_like(u0)
    d = (ctypes.c_int64 * nd)(*[int(n) for n in dims])
    flat = [int(c) for o in offs for c in o]
    o_arr = (ctypes.c_int * len(flat))(*flat)
    w_arr = np.ascontiguousarray(w, dtype=np.float64)
    rc = lib.oracle_run(nd, d, int(r), len(offs), o_arr,
                        w_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(boundary),
                        u0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(T),
                        out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_run failed (%d)" % rc)
    return out


def window_for(dims, r: int, T: int, lo, hi):
    """Padded-frame window [wlo, whi) that holds the T-step dependency cone of
    the interior output box [lo, hi) (interior coordinates), plus an r-wide
    (artificial or physical) ring.  Clipped to the padded frame."""
    wlo, whi = [], []
    for a, n in enumerate(dims):
        # interior coords -> padded coords: +r
        wlo.append(max(0, int(lo[a]) + r - T * r - r))
        whi.append(min(int(n) + 2 * r, int(hi[a]) + r + T * r + r))
    return wlo, whi


def run_cone(dims, r: int, offs, w, u0: np.ndarray, T: int, blo, bhi, nthreads: int = 0) -> np.ndarray:
    """T FIXED steps updating, at step t, only the points within (T-t) r of the
    interior box [blo, bhi): the box's values equal a full run's bit for bit."""
    lib = _load()
    nd = len(dims)
    u0 = np.ascontiguousarray(u0, dtype=np.float64)
    out = np.empty_like(u0)
    d = (ctypes.c_int64 * nd)(*[int(n) for n in dims])
    flat = [int(c) for o in offs for c in o]
    o_arr = (ctypes.c_int * len(flat))(*flat)
    w_arr = np.ascontiguousarray(w, dtype=np.float64)
    lo = (ctypes.c_int64 * nd)(*[int(v) for v in blo])
    hi = (ctypes.c_int64 * nd)(*[int(v) for v in bhi])
    rc = lib.oracle_run_cone(nd, d, int(r), len(offs), o_arr,
                             w_arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                             u0.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(T), lo, hi,
                             out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), int(nthreads))
    if rc != 0:
        raise ValueError("oracle_run_cone failed (%d)" % rc)
    return out


def run_window(dims, r: int, offs, w, T: int, lo, hi, u0_block_fn, nthreads: int = 0, cone: bool = True):
    """Exact oracle values on the interior box [lo, hi) after T FIXED steps,
    computed on the dependency-cone window only.  ``u0_block_fn(wlo, whi)``
    returns u0 on the padded-frame window.  Returns an array of shape hi-lo."""
    wlo, whi = window_for(dims, r, T, lo, hi)
    block = u0_block_fn(wlo, whi)
    nd = len(dims)
    wdims = [whi[a] - wlo[a] - 2 * r for a in range(nd)]
    blo = [int(lo[a]) + r - wlo[a] - r for a in range(nd)]     # box in window-interior coords
    bhi = [int(hi[a]) + r - wlo[a] - r for a in range(nd)]
    if cone:
        res = run_cone(wdims, r, offs, w, block, T, blo, bhi, nthreads)
    else:
        res = run(wdims, r, offs, w, block, T, FIXED, nthreads)
    sl = tuple(slice(int(lo[a]) + r - wlo[a], int(hi[a]) + r - wlo[a]) for a in range(nd))
    return res[sl]
