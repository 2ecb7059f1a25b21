"""Build variant copies of the C-ABI library with different tile macros.

  python tools/tunebuild.py NAME -DSB_3D_VY=4 -DSB_3D_NTY=4 ...

Recompiles the sweep*.cu, run.cu and aux.cu sources with the extra defines (and
STENCIL_TUNING_BUILD, which compiles in the environment tuning knobs), links it with the in-tree objects
of the other sources and writes tunelibs/lib_NAME.so (load it with
STENCIL_B200_LIB=... to measure a variant; tunelibs/ is scratch, git-ignored).
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2103_09235_b200 import build as B  # noqa: E402


def main():
    name, defs = sys.argv[1], sys.argv[2:]
    B.build()
    out = os.path.join(ROOT, "tunelibs")
    os.makedirs(out, exist_ok=True)
    tuned = [f for f in B.SOURCES if f.startswith(("sweep", "tb2d", "tb3d")) or f in ("run.cu", "aux.cu")]
    defs = ["-DSTENCIL_TUNING_BUILD"] + defs   # enables the STENCIL_DEBUG_* / STENCIL_1D_* env knobs
    objs = []
    for src in tuned:
        obj = os.path.join(out, "%s_%s.o" % (src[:-3], name))
        cmd = [B.NVCC] + B.ARCH + B.FLAGS + defs + ["-c", os.path.join(B.CSRC, src), "-o", obj]
        subprocess.run(cmd, check=True)
        objs.append(obj)
    objs += [os.path.join(B.BUILD, s + ".o") for s in B.SOURCES if s not in tuned]
    lib = os.path.join(out, "lib_%s.so" % name)
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
