"""Summarise `nvcc -Xptxas -v` output per kernel: registers, stack, spills.

    nvcc ... -Xptxas -v -c file.cu 2>&1 | python tools/ptxas_table.py [filter]
"""
import re
import subprocess
import sys

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cur = None
rows = {}
for line in sys.stdin:
    m = (re.search(r"Compiling entry function '([^']+)'", line) or
         re.search(r"Function properties for '?([A-Za-z0-9_$.]+)'?", line))
    if m:
        cur = m.group(1)
        rows.setdefault(cur, {})
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        rows[cur].update(stack=int(m.group(1)), st=int(m.group(2)), ld=int(m.group(3)))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
names = list(rows)
dem = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True).stdout.split("\n")
for n, d in zip(names, dem):
    r = rows[n]
    if "regs" not in r or flt not in d:
        continue
    d = re.sub(r"\(uuv::EngineP<(float|double)>.*", "", d).replace("uuv::", "")
    print(f"{r['regs']:4d} regs  stack {r.get('stack',0):4d}  spill st {r.get('st',0):4d} ld {r.get('ld',0):4d}  {d}")
