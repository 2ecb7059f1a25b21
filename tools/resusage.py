"""Registers / stack (spill) per sweep_kernel config of a built library.

  python tools/resusage.py [lib.so ...]
"""
import re
import subprocess
import sys

libs = sys.argv[1:] or ["paper_2103_09235_b200/libstencil_b200.so"]
for lib in libs:
    out = subprocess.run(["cuobjdump", "--dump-resource-usage", lib], capture_output=True, text=True).stdout
    print("==", lib)
    name = None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        if name and "REG:" in line:
            reg = re.search(r"REG:(\d+)", line).group(1)
            stk = re.search(r"STACK:(\d+)", line).group(1)
            c = re.search(r"CfgI(\w)((?:Li-?\d+E)+)", name)
            if c:
                args = re.findall(r"Li(-?\d+)E", c.group(2))
                names = ["Q", "S", "NTX", "NTY", "VY", "PB", "NSLOT", "VXM", "MINB", "ROT", "PINC"]
                short = "%s nd=%s %s r=%s " % (c.group(1), args[0], "box" if args[1] == "1" else "star", args[2]) + " ".join(
                    "%s=%s" % kv for kv in zip(names, args[3:]))
            else:
                short = re.sub(r"_ZN2sb\d+", "", name)[:60]
            print("  %-90s REG %3s STACK %s" % (short, reg, stk))
            name = None
