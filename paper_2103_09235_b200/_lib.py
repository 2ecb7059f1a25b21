"""ctypes loader for libstencil_b200.so (the C-ABI in include/stencil_b200.h).

There is no fallback: if the shared library is missing and cannot be built,
importing the binding raises.
"""
from __future__ import annotations

import ctypes
import os
import threading

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("STENCIL_B200_LIB") or os.path.join(HERE, "libstencil_b200.so")
_lock = threading.Lock()
_lib = None

c_int, c_i64, c_u64, c_vp, c_dp = ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double)


class StencilLayout(ctypes.Structure):
    _fields_ = [("ndim", c_int), ("radius", c_int), ("interior", c_i64 * 3), ("extent", c_i64 * 3),
                ("stride", c_i64 * 3), ("origin", c_i64 * 3), ("elem_bytes", c_i64), ("bytes", c_i64),
                ("global_offset0", c_i64)]


# name -> (restype, argtypes); mirrors include/stencil_b200.h one to one
SIGNATURES = {
    "stencil_plan_create": (c_int, [ctypes.POINTER(c_vp), c_int, ctypes.POINTER(c_i64), c_int, c_int, c_dp, c_int,
                                    c_int, c_int]),
    "stencil_plan_destroy": (c_int, [c_vp]),
    "stencil_plan_layout": (c_int, [c_vp, ctypes.POINTER(StencilLayout)]),
    "stencil_plan_ntaps": (c_int, [c_vp, ctypes.POINTER(c_int)]),
    "stencil_plan_taps": (c_int, [c_vp, ctypes.POINTER(c_int), c_int]),
    "stencil_plan_fold_coeffs": (c_int, [c_vp, c_int, c_dp, c_i64]),
    "stencil_plan_fold_rank": (c_int, [c_vp, c_int, ctypes.POINTER(c_int), c_dp, c_dp, c_i64]),
    "stencil_plan_set_counterparts": (c_int, [c_vp, c_int]),
    "stencil_plan_perturb_fold": (c_int, [c_vp, c_int, c_i64, ctypes.c_double]),
    "stencil_plan_auto_fold": (c_int, [c_vp, ctypes.POINTER(c_int)]),
    "stencil_plan_variant": (c_int, [c_vp, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int),
                                     ctypes.POINTER(c_int)]),
    "stencil_workspace_size": (c_int, [c_vp, ctypes.POINTER(c_i64)]),
    "stencil_fill_random": (c_int, [c_vp, c_vp, c_u64, c_vp]),
    "stencil_run": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_vp, c_vp]),
    "stencil_run_ex": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp]),
    "stencil_run_host": (c_int, [c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_vp, c_vp, c_vp, c_vp]),
    "stencil_run_host_batch": (c_int, [c_vp, c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i64, c_int, c_int,
                                       ctypes.POINTER(c_vp), c_vp]),
    "stencil_plan_last_launches": (c_int, [c_vp, ctypes.POINTER(c_i64)]),
    "stencil_plan_set_schedule": (c_int, [c_vp, c_int, c_int, c_int]),
    "stencil_plan_sched_stats": (c_int, [c_vp, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64), c_int]),
    "stencil_comm_wait": (c_int, [c_vp, c_vp, c_i64]),
    "stencil_plan_set_timing": (c_int, [c_vp, c_int]),
    "stencil_plan_timing": (c_int, [c_vp, c_int, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(c_i64),
                                    ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]),
    "stencil_plan_timing_reset": (c_int, [c_vp]),
    "stencil_comm_unique_id": (c_int, [ctypes.c_char_p]),
    "stencil_comm_create": (c_int, [ctypes.POINTER(c_vp), ctypes.c_char_p, c_int, c_int]),
    "stencil_comm_destroy": (c_int, [c_vp]),
    "stencil_plan_layout_dist": (c_int, [c_vp, c_int, c_int, c_int, ctypes.POINTER(StencilLayout)]),
    "stencil_fill_random_dist": (c_int, [c_vp, c_int, c_int, c_int, c_vp, c_u64, c_vp]),
    "stencil_run_dist": (c_int, [c_vp, c_vp, c_vp, c_vp, c_i64, c_int, c_int, c_int, c_vp, c_vp]),
    "stencil_halo_exchange": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp]),
    "stencil_halo_exchange_loopback": (c_int, [c_vp, c_vp, c_vp, c_int, c_vp]),
    "stencil_run_dist_emulated": (c_int, [c_vp, c_int, ctypes.POINTER(c_vp), ctypes.POINTER(c_vp), c_i64, c_int,
                                          c_int, c_int, ctypes.POINTER(c_vp), c_int, c_vp]),
    "stencil_comm_create_peer": (c_int, [ctypes.POINTER(c_vp), c_int, c_int, c_vp, c_vp]),
    "stencil_comm_peer_handles": (c_int, [c_vp, ctypes.c_char_p]),
    "stencil_comm_peer_attach": (c_int, [c_vp, ctypes.c_char_p]),
    "stencil_last_error": (ctypes.c_char_p, []),
    "stencil_version": (ctypes.c_char_p, []),
}

STATUS = {0: "STENCIL_OK", -1: "STENCIL_EINVAL", -2: "STENCIL_EUNSUPPORTED", -3: "STENCIL_ECUDA",
          -4: "STENCIL_ENCCL", -5: "STENCIL_ENOMEM", -6: "STENCIL_ETIMEOUT"}


class StencilError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__("%s (%d): %s" % (STATUS.get(code, "?"), code, msg))
        self.code = code


def load():
    """Load (building in-tree first if the .so is absent) the C-ABI library."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                from . import build as _build
                _build.build()
            lib = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(rc):
    if rc != 0:
        msg = load().stencil_last_error().decode(errors="replace")
        raise StencilError(rc, msg)
    return rc
