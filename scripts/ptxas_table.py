"""Registers / spills per kernel from `nvcc -Xptxas -v` output on stdin."""
import re, sys
cur = None
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m and cur:
        spill = int(m.group(1))
    m2 = re.search(r"Used (\d+) registers", line)
    if m2 and cur:
        if not sys.argv[1:] or any(a in cur for a in sys.argv[1:]):
            print(f"{int(m2.group(1)):4d} regs  spill {spill:4d}  {cur[:90]}")
        cur = None
