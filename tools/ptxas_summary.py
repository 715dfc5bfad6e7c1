"""Summarise `nvcc -Xptxas -v` output: kernel -> registers, spills (reads stdin)."""
import re
import sys

cur = None
info = {}
for line in sys.stdin:
    m = re.search(r"Compiling entry function '([^']+)'", line)
    if m:
        cur = m.group(1)
        info[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes spill stores", line)
    if m:
        info[cur]["spill"] = int(m.group(1))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        info[cur]["regs"] = int(m.group(1))
pat = sys.argv[1] if len(sys.argv) > 1 else ""
for k, v in info.items():
    if pat in k:
        name = re.sub(r"_ZN2ck(40_GLOBAL__N__\w+?_)?\d+", "", k)[:60]
        print(f"{name:60s} regs={v.get('regs')} spill={v.get('spill')}")
