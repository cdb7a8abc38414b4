"""Registers / stack / spills per kernel from an nvcc -Xptxas -v log.
Usage: python tools/ptxas_regs.py build/elimtw/ptxas.log"""
import re, sys
cur = None
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
        k = re.search(r"(k_\w+?)(I.*?E)?E?Ev", name)
        cur = name
        short = re.sub(r"_ZN3etw\d+_GLOBAL__N__\w+?_\d+_\w+?_cu_\w{8}\d+", "", name)
        cur = short[:60]
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        stack, spill = m.groups()
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        print(f"{cur:60s} regs={m.group(1):>4s} stack={stack:>5s} spill={spill}")
        cur = None
