"""Per-kernel registers and spill bytes from the build's ptxas logs (paper_2401_17474_b200/build/*.ptxas.txt).

    python tools/spills.py [--all]
"""
import glob
import os
import re
import sys

BUILD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2401_17474_b200", "build")
show_all = "--all" in sys.argv
for f in sorted(glob.glob(os.path.join(BUILD, "*.ptxas.txt"))):
    cur, spill = None, None
    for line in open(f):
        m = re.search(r"Compiling entry function '([^']+)'", line)
        if m:
            cur = m.group(1)
        m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
        if m:
            spill = (int(m.group(1)), int(m.group(2)))
        m = re.search(r"Used (\d+) registers", line)
        if m and cur and spill is not None:
            if show_all or spill != (0, 0):
                print(f"{os.path.basename(f)[:-14]:10s} regs {m.group(1):>3s} spill st/ld {spill[0]:4d}/{spill[1]:4d}  {cur}")
            cur, spill = None, None
