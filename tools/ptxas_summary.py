"""Summarise `nvcc -Xptxas -v` output: kernel, registers, spills, smem."""
import re
import sys

cur = None
rows = {}
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur]["spill"] = f"{m.group(1)}/{m.group(2)}"
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = m.group(1)
pat = sys.argv[2] if len(sys.argv) > 2 else ""
for k, v in rows.items():
    name = re.sub(r"_ZN3dbx\d+_GLOBAL__N__\w+?_cu_\w{8}", "", k)
    if pat and not re.search(pat, name):
        continue
    print(f"{name[:60]:60s} regs={v.get('regs','?'):>4s} spill={v.get('spill','?')}")
