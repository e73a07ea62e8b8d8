"""Registers / spills per kernel from paper_2110_12952_b200/build.log: python tools/regs.py [regex]"""
import re
import sys

pat = re.compile(sys.argv[1] if len(sys.argv) > 1 else ".")
cur = None
for line in open("paper_2110_12952_b200/build.log"):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur and pat.search(cur):
        print(f"{m.group(1):>4} regs  {cur[:140]}")
        cur = None
