"""Where do the register spills of the kernels built under forced launch bounds sit?
For every kernel whose SASS has local-memory traffic (STL / LDL), list each such
instruction with the innermost loop (backward-branch interval) that contains it and
that loop's length in instructions -- a spill outside every loop, or only in an outer
loop that runs a handful of times, is off the hot path.

    python scripts/spill_report.py > profiles/r2_spill_report.txt
"""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SO = os.path.join(ROOT, "paper_1902_09046_b200", "libvexbayes_cuda.so")
sass = subprocess.run(["cuobjdump", "-sass", SO], capture_output=True, text=True).stdout
funcs, cur = {}, None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
demangle = lambda n: subprocess.run(["c++filt", n], capture_output=True, text=True).stdout.strip().split("(")[0]
for name, ins in funcs.items():
    local = [(a, t) for a, t in ins if re.search(r"\b(STL|LDL)\b", t.split()[0] if not t.startswith("@") else t.split()[1])]
    if not local:
        continue
    loops = []   # (target, branch address) of backward branches
    for a, t in ins:
        m = re.search(r"\bBRA(?:\.\w+)*\s+(?:\w+,\s*)?(0x[0-9a-f]+)", t)
        if m and int(m.group(1), 16) <= a:
            loops.append((int(m.group(1), 16), a))
    rows = []
    for a, t in local:
        inner = [l for l in loops if l[0] <= a <= l[1]]
        if inner:
            lo, hi = min(inner, key=lambda l: l[1] - l[0])
            n_in = sum(1 for x, _ in ins if lo <= x <= hi)
            where = f"innermost loop 0x{lo:04x}-0x{hi:04x} ({n_in} instructions, nesting {len(inner)})"
        else:
            n_in, where = 0, "outside every loop"
        rows.append((a, t, n_in, where))
    outside = sum(1 for r in rows if r[2] == 0)
    outer = sum(1 for r in rows if r[2] >= 1000)
    mid = sum(1 for r in rows if 200 <= r[2] < 1000)
    hot = sum(1 for r in rows if 0 < r[2] < 200)
    print(f"{demangle(name)}: {len(ins)} instructions, {len(local)} local-memory instructions: "
          f"{outside} outside every loop, {outer} in loops of >= 1000 instructions (per-iteration "
          f"control flow), {mid} in loops of 200-999, {hot} in loops shorter than 200 instructions")
    if "-v" in sys.argv or hot:
        for a, t, n_in, where in rows:
            if "-v" in sys.argv or 0 < n_in < 200:
                print(f"    0x{a:04x} {t.split('/*')[0][:60]:60s} {where}")
