"""Instruction mix of every loop of one kernel (SASS of the built library).

    python scripts/loop_census.py <mangled kernel name> [min loop length]
"""
import re
import subprocess
import sys
import os

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1902_09046_b200", "libvexbayes_cuda.so")
name = sys.argv[1]
min_len = int(sys.argv[2]) if len(sys.argv) > 2 else 100
sass = subprocess.run(["cuobjdump", "-sass", "-fun", name, SO], capture_output=True, text=True).stdout
ins, seen = [], set()
for line in sass.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        a = int(m.group(1), 16)
        if a in seen:
            break
        seen.add(a)
        ins.append((a, m.group(2).strip()))
print(name, len(ins), "instructions")
for a, t in ins:
    m = re.search(r"\bBRA(?:\.\w+)*\s+(?:!?\w+,\s*)?(0x[0-9a-f]+)", t)
    if not m or int(m.group(1), 16) > a:
        continue
    lo, hi = int(m.group(1), 16), a
    body = [t2 for a2, t2 in ins if lo <= a2 <= hi]
    if len(body) < min_len:
        continue
    ops = {}
    for t2 in body:
        parts = t2.split()
        op = parts[1] if parts[0].startswith("@") else parts[0]
        ops[op] = ops.get(op, 0) + 1
    print(f"loop 0x{lo:04x}-0x{hi:04x}: {len(body)} instructions")
    print("   ", ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda x: -x[1])))
