"""Instruction mix of the innermost sub-step loop of a kernel (from cuobjdump -sass).

    python tools/sass_loop.py <mangled-or-substring> [lib]
The loop is the largest backward-branch region; prints its size and opcode mix.
"""
import re
import subprocess
import sys
from collections import Counter

name = sys.argv[1]
lib = sys.argv[2] if len(sys.argv) > 2 else "paper_2410_14117_b200/_lib/libuuvsim_core.so"
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s*Function : ", out)
sel = [f for f in funcs if f.split("\n", 1)[0].strip() == name] or \
      [f for f in funcs if name in f.split("\n", 1)[0]]
if not sel:
    sys.exit(f"no function matching {name}")
body = sel[0]
ins = []
for l in body.splitlines():
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), re.sub(r"^@!?U?P\w+\s+", "", m.group(2).strip())))
loops = []
for a, t in ins:
    m = re.match(r"BRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((int(m.group(1), 16), a))
print(body.split("\n", 1)[0].strip()[:100], "total", len(ins))
for lo, hi in sorted(loops, key=lambda x: x[0] - x[1])[:3]:   # the three largest loops
    c = Counter(t.split()[0] for a, t in ins if lo <= a <= hi)
    print(f"loop [{lo:#x},{hi:#x}] {sum(c.values())} instructions")
    print("   " + ", ".join(f"{k} {v}" for k, v in c.most_common()))
