"""Achieved DRAM GB/s per kernel from an ncu CSV with gpu__time_duration.sum,
dram__bytes_read.sum and dram__bytes_write.sum (profiles/r1_compaction_kernels_1e8.csv)."""
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10 and r[0].isdigit()]
by = {}
for r in rows:
    name = r[4].split("(")[0].replace("void vxb::", "").replace("vxb::", "")
    by.setdefault((r[0], name, r[8]), {})[r[12]] = (float(r[14]), r[13])
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
agg = {}
for (_, name, grid), m in by.items():
    t, rd, wr = (m[k][0] * scale[m[k][1]] for k in ("gpu__time_duration.sum", "dram__bytes_read.sum",
                                                    "dram__bytes_write.sum"))
    agg.setdefault((name, grid), []).append((t, rd, wr))
for (name, grid), v in agg.items():
    t, rd, wr = (sum(x[k] for x in v) / len(v) for k in range(3))
    print(f"{name:34s} grid={grid:>15s} n={len(v):2d} t={t * 1e6:8.1f} us  read={rd / 1e6:8.2f} MB  "
          f"write={wr / 1e6:6.2f} MB  {(rd + wr) / t / 1e9:7.1f} GB/s")
