"""Variant copies of the library that differ only in tb3d_f64.cu's macros.

  python tools/tb3build.py NAME -DTB3_NWY=16 -DTB3_VY=2 ...

Compiles tb3d_f64.cu with the defines (ptxas -v output to tunelibs/NAME.ptxas),
links it with the in-tree objects of every other source and writes
tunelibs/lib_NAME.so (load with STENCIL_B200_LIB=...; tunelibs/ is scratch).
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
    src = os.environ.get("TB3_SRC", "tb3d_f64.cu")   # (TB3_SRC=tb3d_f32.cu for the fp32 unit)
    obj = os.path.join(out, "%s_%s.o" % (src[:-3], name))
    cmd = [B.NVCC] + B.ARCH + B.FLAGS + defs + ["-Xptxas", "-v", "-c", os.path.join(B.CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    open(os.path.join(out, name + ".ptxas"), "w").write(r.stderr)
    if r.returncode:
        sys.exit(r.stderr[-2000:])
    objs = [obj] + [os.path.join(B.BUILD, s + ".o") for s in B.SOURCES if s != src]
    lib = os.path.join(out, "lib_%s.so" % name)
    subprocess.run([B.NVCC] + B.ARCH + ["-shared", "-cudart", "static", "-o", lib] + objs + ["-ldl"], check=True)
    print(lib)


if __name__ == "__main__":
    main()
