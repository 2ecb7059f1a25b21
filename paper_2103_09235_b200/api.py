"""Thin Python binding over the C-ABI (argument marshalling only).

Every step of the path runs in the library's CUDA kernels; PyTorch supplies
device memory, streams and (for multi-GPU) process groups.

    plan = Plan(dims=(8192, 8192), radius=1, shape="star", coeffs=w, dtype="f64")
    a, b, ws = plan.empty(), plan.empty(), plan.empty()
    plan.fill_random(a, seed=2)
    plan.run(a, b, T=200, fold_m=2, workspace=ws)
    u = plan.frame_view(b)          # strided view of the padded frame (N + 2r per axis)
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np
import torch

from ._lib import StencilLayout, check, load

STAR, BOX = 0, 1
F32, F64 = 0, 1
FIXED, PERIODIC = 0, 1
_SHAPES = {"star": STAR, "box": BOX, STAR: STAR, BOX: BOX}
_DTYPES = {"f32": F32, "fp32": F32, "float32": F32, torch.float32: F32,
           "f64": F64, "fp64": F64, "float64": F64, torch.float64: F64, F32: F32, F64: F64}
_BCS = {"fixed": FIXED, "periodic": PERIODIC, FIXED: FIXED, PERIODIC: PERIODIC}


@dataclass(frozen=True)
class Layout:
    ndim: int
    radius: int
    interior: tuple
    extent: tuple
    stride: tuple
    origin: tuple
    elem_bytes: int
    bytes: int
    global_offset0: int

    @property
    def numel(self) -> int:
        return self.bytes // self.elem_bytes

    @property
    def frame(self) -> tuple:
        """Padded-frame extents N_a + 2r (axis 0 of a dist layout: local N + 2r)."""
        return tuple(n + 2 * self.radius for n in self.interior)


def _layout(cl: StencilLayout) -> Layout:
    nd = cl.ndim
    return Layout(nd, cl.radius, tuple(cl.interior[:nd]), tuple(cl.extent[:nd]), tuple(cl.stride[:nd]),
                  tuple(cl.origin[:nd]), cl.elem_bytes, cl.bytes, cl.global_offset0)


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    return int(t)


def _stream(stream) -> Optional[int]:
    if stream is None:
        stream = torch.cuda.current_stream()
    if isinstance(stream, torch.cuda.Stream):
        return stream.cuda_stream
    return int(stream)


class Plan:
    """stencil_plan_create(dims, radius, shape, coeffs, dtype, boundary)."""

    def __init__(self, dims: Sequence[int], radius: int, shape, coeffs, dtype="f64", boundary="fixed"):
        self._lib = load()
        self.dims = tuple(int(d) for d in dims)
        self.ndim = len(self.dims)
        self.radius = int(radius)
        self.shape = _SHAPES[shape]
        self.dtype_code = _DTYPES[dtype]
        self.torch_dtype = torch.float64 if self.dtype_code == F64 else torch.float32
        self.boundary = _BCS[boundary]
        w = np.ascontiguousarray(coeffs, dtype=np.float64)
        self.coeffs = w.copy()
        h = ctypes.c_void_p()
        d = (ctypes.c_int64 * self.ndim)(*self.dims)
        check(self._lib.stencil_plan_create(ctypes.byref(h), self.ndim, d, self.radius, self.shape,
                                            w.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), len(w),
                                            self.dtype_code, self.boundary))
        self._h = h
        cl = StencilLayout()
        check(self._lib.stencil_plan_layout(self._h, ctypes.byref(cl)))
        self.layout = _layout(cl)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            self._lib.stencil_plan_destroy(h)
            self._h = None

    # ---------------------------------------------------------------- host info
    @property
    def ntaps(self) -> int:
        k = ctypes.c_int()
        check(self._lib.stencil_plan_ntaps(self._h, ctypes.byref(k)))
        return k.value

    def taps(self):
        k = self.ntaps
        buf = (ctypes.c_int * (k * self.ndim))()
        check(self._lib.stencil_plan_taps(self._h, buf, k * self.ndim))
        return [tuple(buf[j * self.ndim:(j + 1) * self.ndim]) for j in range(k)]

    def fold_coeffs(self, m: int) -> np.ndarray:
        """lambda^(m) as a dense (2mr+1)^d fp64 array (index o + m r)."""
        side = 2 * m * self.radius + 1
        out = np.zeros((side,) * self.ndim, dtype=np.float64)
        check(self._lib.stencil_plan_fold_coeffs(self._h, int(m), out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                 out.size))
        return out

    def fold_rank(self, m: int):
        """Counterpart decomposition of lambda^(m) (2D): (rank, a, b) with
        lambda^(m)[i, j] = sum_k a[k, i] b[k, j] (stencil_plan_fold_rank)."""
        W = 2 * m * self.radius + 1
        rank = ctypes.c_int()
        a = np.zeros((W, W), dtype=np.float64)
        b = np.zeros((W, W), dtype=np.float64)
        check(self._lib.stencil_plan_fold_rank(self._h, int(m), ctypes.byref(rank),
                                               a.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                               b.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), a.size))
        return rank.value, a[:rank.value].copy(), b[:rank.value].copy()

    def perturb_fold(self, m: int, index: int, delta: float) -> None:
        """Fault injection (tests): lambda^(m)[index] += delta for later runs."""
        check(self._lib.stencil_plan_perturb_fold(self._h, int(m), int(index), float(delta)))

    def auto_fold(self) -> int:
        """The fold_m a run with fold_m = 0 uses (stencil_plan_auto_fold)."""
        m = ctypes.c_int()
        check(self._lib.stencil_plan_auto_fold(self._h, ctypes.byref(m)))
        return m.value

    def set_counterparts(self, enable: bool) -> None:
        check(self._lib.stencil_plan_set_counterparts(self._h, 1 if enable else 0))

    def variant(self, m: int):
        """(q, stages, rank) the plan chooses for fold_m = m (stencil_plan_variant)."""
        q, s, r = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(self._lib.stencil_plan_variant(self._h, int(m), ctypes.byref(q), ctypes.byref(s), ctypes.byref(r)))
        return q.value, s.value, r.value

    def layout_dist(self, rank: int, nranks: int, halo: int) -> Layout:
        cl = StencilLayout()
        check(self._lib.stencil_plan_layout_dist(self._h, rank, nranks, halo, ctypes.byref(cl)))
        return _layout(cl)

    # ---------------------------------------------------------------- buffers
    def empty(self, device="cuda", layout: Optional[Layout] = None, pin_memory=False) -> torch.Tensor:
        L = layout or self.layout
        if device == "cpu":
            return torch.zeros(L.numel, dtype=self.torch_dtype, pin_memory=pin_memory)
        return torch.empty(L.numel, dtype=self.torch_dtype, device=device)

    def frame_view(self, buf: torch.Tensor, layout: Optional[Layout] = None) -> torch.Tensor:
        """Strided view of the padded frame (interior + r-ring) of a buffer."""
        L = layout or self.layout
        r = L.radius
        off = sum((L.origin[a] - r) * L.stride[a] for a in range(L.ndim))
        return buf.as_strided(L.frame, L.stride, buf.storage_offset() + off)

    def interior_view(self, buf: torch.Tensor, layout: Optional[Layout] = None) -> torch.Tensor:
        L = layout or self.layout
        off = sum(L.origin[a] * L.stride[a] for a in range(L.ndim))
        return buf.as_strided(L.interior, L.stride, buf.storage_offset() + off)

    def from_frame(self, frame: np.ndarray, device="cuda") -> torch.Tensor:
        """A buffer in the plan layout holding `frame` (padded frame array); pads = 0."""
        buf = torch.zeros(self.layout.numel, dtype=self.torch_dtype)
        self.frame_view(buf).copy_(torch.from_numpy(np.asarray(frame, dtype=np.float64)).to(self.torch_dtype))
        return buf.to(device) if device != "cpu" else buf

    # ---------------------------------------------------------------- compute
    def fill_random(self, buf: torch.Tensor, seed: int, stream=None):
        check(self._lib.stencil_fill_random(self._h, _ptr(buf), int(seed), _stream(stream)))

    def run(self, inp, out, T: int, fold_m: int = 1, workspace=None, stages: int = 0, stream=None):
        check(self._lib.stencil_run_ex(self._h, _ptr(inp), _ptr(out), int(T), int(fold_m), int(stages),
                                       _ptr(workspace), _stream(stream)))

    def run_host(self, in_host, out_host, T: int, fold_m: int, dev_in, dev_out, workspace=None, stages: int = 0,
                 stream=None):
        check(self._lib.stencil_run_host(self._h, _ptr(in_host), _ptr(out_host), int(T), int(fold_m), int(stages),
                                         _ptr(dev_in), _ptr(dev_out), _ptr(workspace), _stream(stream)))

    def run_host_batch(self, in_hosts, out_hosts, T: int, fold_m: int, dev_sets, stages: int = 0, stream=None):
        """nbatch problems from pinned host buffers, H2D / run / D2H pipelined over
        two device buffer sets dev_sets = [(in, out, ws), (in, out, ws)]
        (stencil_run_host_batch)."""
        n = len(in_hosts)
        if len(out_hosts) != n:
            raise ValueError("in_hosts and out_hosts differ in length")
        arr = ctypes.c_void_p * n
        flat = [_ptr(t) for s in list(dev_sets)[:2] for t in s]
        flat += [None] * (6 - len(flat))
        check(self._lib.stencil_run_host_batch(self._h, n, arr(*[_ptr(t) for t in in_hosts]),
                                               arr(*[_ptr(t) for t in out_hosts]), int(T), int(fold_m), int(stages),
                                               (ctypes.c_void_p * 6)(*flat), _stream(stream)))

    def set_schedule(self, chunk: int = 0, min_steal: int = 0, max_ctas: int = 0) -> None:
        """Schedule granularity of the 2D/3D sweep (tests/tuning; 0 = default)."""
        check(self._lib.stencil_plan_set_schedule(self._h, int(chunk), int(min_steal), int(max_ctas)))

    def sched_stats(self, reset: bool = False):
        """(grabs, steals) counted by the sweep kernels (stencil_plan_sched_stats)."""
        g, s = ctypes.c_int64(), ctypes.c_int64()
        check(self._lib.stencil_plan_sched_stats(self._h, ctypes.byref(g), ctypes.byref(s), 1 if reset else 0))
        return g.value, s.value

    @property
    def last_launches(self) -> int:
        n = ctypes.c_int64()
        check(self._lib.stencil_plan_last_launches(self._h, ctypes.byref(n)))
        return n.value

    # ---------------------------------------------------------------- measurement
    def set_timing(self, enable: bool):
        check(self._lib.stencil_plan_set_timing(self._h, 1 if enable else 0))

    def timing(self, kind: int = 0) -> dict:
        """Event-timed kernel time of the recorded launches of `kind` (0 main
        sweep / 1D kernel, 1 band): ms, launches, algorithmic bytes and FMAs."""
        ms, n, by, fm = ctypes.c_double(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        check(self._lib.stencil_plan_timing(self._h, int(kind), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(by),
                                            ctypes.byref(fm)))
        return {"ms": ms.value, "launches": n.value, "bytes": by.value, "fmas": fm.value}

    def timing_reset(self):
        check(self._lib.stencil_plan_timing_reset(self._h))

    # ---------------------------------------------------------------- multi-GPU
    def fill_random_dist(self, rank, nranks, halo, buf, seed, stream=None):
        check(self._lib.stencil_fill_random_dist(self._h, rank, nranks, halo, _ptr(buf), int(seed), _stream(stream)))

    def run_dist(self, comm: "Comm", inp, out, T, fold_m, halo, workspace=None, stages=0, stream=None):
        check(self._lib.stencil_run_dist(self._h, comm._h, _ptr(inp), _ptr(out), int(T), int(fold_m), int(stages),
                                         int(halo), _ptr(workspace), _stream(stream)))

    def halo_exchange(self, comm: "Comm", buf, halo, stream=None):
        check(self._lib.stencil_halo_exchange(self._h, comm._h, _ptr(buf), int(halo), _stream(stream)))

    def halo_exchange_loopback(self, comm: "Comm", buf, halo, stream=None):
        """Diagnostic: the NCCL exchange with this rank as both neighbours (one-GPU boxes)."""
        check(self._lib.stencil_halo_exchange_loopback(self._h, comm._h, _ptr(buf), int(halo), _stream(stream)))

    def run_dist_emulated(self, ins, outs, T, fold_m, halo, workspaces=None, stages=0, stream=None,
                          exchange="copies"):
        """All ranks in this process on one GPU; exchange = "copies" (the NCCL
        path's schedule with device-to-device copies) or "peer" (fused peer stores)."""
        n = len(ins)
        arr = ctypes.c_void_p * n
        wp = arr(*[_ptr(w) for w in workspaces]) if workspaces is not None else None
        mode = {"copies": 0, "peer": 1}[exchange]
        check(self._lib.stencil_run_dist_emulated(self._h, n, arr(*[_ptr(t) for t in ins]),
                                                  arr(*[_ptr(t) for t in outs]), int(T), int(fold_m), int(stages),
                                                  int(halo), wp, mode, _stream(stream)))


class Comm:
    """NCCL communicator over the slab decomposition (one process per GPU).

    Bootstrap: rank 0 creates the 128-byte unique id, which is broadcast through
    torch.distributed (see paper_2103_09235_b200.dist.make_comm)."""

    def __init__(self, uid: bytes, rank: int, nranks: int):
        self._lib = load()
        h = ctypes.c_void_p()
        check(self._lib.stencil_comm_create(ctypes.byref(h), uid, int(rank), int(nranks)))
        self._h = h
        self.rank, self.nranks = rank, nranks

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(load().stencil_comm_unique_id(buf))
        return buf.raw

    @classmethod
    def peer(cls, rank: int, nranks: int, buf0, buf1) -> "Comm":
        """Fused peer-store exchange (NEXT-2): buf0/buf1 are this rank's
        ping-pong buffers (every run passes buf0 as out and buf1 as workspace).  Attach
        the neighbours with attach(all_records) after an all-gather of
        handles() (paper_2103_09235_b200.dist.make_peer_comm does both)."""
        self = cls.__new__(cls)
        self._lib = load()
        h = ctypes.c_void_p()
        check(self._lib.stencil_comm_create_peer(ctypes.byref(h), int(rank), int(nranks), _ptr(buf0), _ptr(buf1)))
        self._h = h
        self.rank, self.nranks = rank, nranks
        return self

    PEER_RECORD = 3 * 72   # 3 x STENCIL_PEER_HANDLE_BYTES

    def handles(self) -> bytes:
        buf = ctypes.create_string_buffer(self.PEER_RECORD)
        check(self._lib.stencil_comm_peer_handles(self._h, buf))
        return buf.raw

    def attach(self, records) -> None:
        """records: every rank's handles() in rank order."""
        blob = b"".join(records)
        if len(blob) != self.PEER_RECORD * self.nranks:
            raise ValueError("expected %d records of %d bytes" % (self.nranks, self.PEER_RECORD))
        check(self._lib.stencil_comm_peer_attach(self._h, blob))

    def wait(self, stream=None, timeout_ms: int = -1) -> None:
        """Block until `stream` drains, polling the NCCL async error; abort the
        comm and raise on an NCCL failure or after timeout_ms (stencil_comm_wait)."""
        check(self._lib.stencil_comm_wait(self._h, _stream(stream), int(timeout_ms)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.stencil_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
