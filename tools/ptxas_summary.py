"""Summarise `nvcc -Xptxas -v` output: one line per kernel with registers,
spills and shared memory (demangled).  Usage: nvcc ... -Xptxas -v 2>&1 | python tools/ptxas_summary.py"""
import re
import subprocess
import sys

cur = None
rows = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(\w+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = int(m.group(1)) + int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
    m = re.search(r"(\d+) bytes smem", line)
    if m:
        rows[cur]["smem"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    r = rows[n]
    d = re.sub(r"qj::|void |\(.*", "", d)
    print(f"{r.get('regs', '?'):>4} regs  spill {r.get('spill', 0):>5}  smem {r.get('smem', 0):>6}  {d}")
