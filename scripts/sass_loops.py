#!/usr/bin/env python3
"""Per-loop SASS instruction mix of libxg_gpu.so kernels (static analysis aid).

usage: python scripts/sass_loops.py [lib.so] [name-filter]
Prints, for every backward branch (a loop), the instruction count and opcode
histogram of the loop body -- the per-word issue budget of the fill kernels.
"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_1108_0486_b200/lib/libxg_gpu.so"
filt = sys.argv[2] if len(sys.argv) > 2 else ""
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in txt.split("Function : ")[1:]:
    name = f.split("\n")[0].strip()
    if filt not in name:
        continue
    ins = re.findall(r"/\*([0-9a-f]{4,5})\*/\s+([^;]*);", f)
    for addr, i in ins:
        m = re.search(r"BRA\S*\s+(?:\S+,\s*)?(0x[0-9a-f]+)", i)
        if m and int(m.group(1), 16) < int(addr, 16):
            a0, a1 = int(m.group(1), 16), int(addr, 16)
            body = [x for a, x in ins if a0 <= int(a, 16) <= a1]
            ops = Counter((x.split()[1] if x.startswith("@") else x.split()[0]).split(".")[0]
                          for x in body)
            print(f"{name}\n  loop {a0:#x}-{a1:#x}: {len(body)} instrs  {dict(ops.most_common())}")
