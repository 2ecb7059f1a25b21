"""Debug/probe harness for the 2D temporal block (tuning builds only).

  STENCIL_B200_LIB=tunelibs/lib_probe.so CUDA_LAUNCH_BLOCKING=1 python tools/tb_debug.py crash
  STENCIL_B200_LIB=tunelibs/lib_probe.so python tools/tb_debug.py probe [K]

crash: single sweeps of small cases, one per process-local try, to find a faulting case.
probe: one C2 sweep with per-warp smid/start/end recorded by the kernel (TB_PROBE build).
"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2103_09235_b200 import Plan  # noqa: E402
from paper_2103_09235_b200._lib import load  # noqa: E402


def crash():
    for dims in [(70, 523), (9, 40), (301, 1100), (8192, 8192)]:
        for dtype in ["f64", "f32"]:
            for shape in ["star", "box"]:
                for K in [2, 3, 4, 5, 8]:
                    k = 5 if shape == "star" else 9
                    plan = Plan(dims, 1, shape, synth.weights(k, 1), dtype)
                    a, b = plan.empty(), plan.empty()
                    plan.fill_random(a, 2)
                    torch.cuda.synchronize()
                    print("case", dims, dtype, shape, K, flush=True)
                    plan.run(a, b, K, K, stages=K)
                    torch.cuda.synchronize()
                    print("  ok", flush=True)


def probe(K):
    lib = load()
    fn = lib.stencil_debug_tb_probe
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
    n = 8192
    buf = np.zeros(4 * n, dtype=np.uint64)
    plan = Plan((8192, 8192), 1, "star", synth.weights(5, 1), "f64")
    a, b = plan.empty(), plan.empty()
    plan.fill_random(a, 2)
    plan.run(a, b, K, K, stages=K)
    torch.cuda.synchronize()
    fn(buf.ctypes.data, n, 1)
    plan.run(a, b, K, K, stages=K)
    torch.cuda.synchronize()
    fn(buf.ctypes.data, n, 0)
    r = buf.reshape(n, 4)
    used = r[:, 1] > 0
    r = r[used].astype(np.float64)
    t0 = r[:, 1].min()
    st, en = (r[:, 1] - t0) / 1e3, (r[:, 2] - t0) / 1e3
    dur = en - st
    print("warps", len(r), "start max %.1f us" % st.max(), "end min %.1f max %.1f us" % (en.min(), en.max()))
    print("dur us percentiles", np.percentile(dur, [0, 10, 50, 90, 99, 100]).round(1))
    order = np.argsort(-dur)[:12]
    for i in order:
        print("  warp", int(np.nonzero(used)[0][i]), "sm", int(r[i, 0]), "start %.1f end %.1f rows %d" % (st[i], en[i], r[i, 3]))
    sms = {}
    for i in range(len(r)):
        sms.setdefault(int(r[i, 0]), []).append(i)
    per_sm = sorted((len(v), k) for k, v in sms.items())
    print("SMs used", len(sms), "warps per SM min/max", per_sm[0], per_sm[-1])


if __name__ == "__main__":
    if sys.argv[1] == "crash":
        crash()
    else:
        probe(int(sys.argv[2]) if len(sys.argv) > 2 else 8)
