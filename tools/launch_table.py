#!/usr/bin/env python3
"""Per-kernel table from an ncu launch list with one or more metrics (gpu__time_duration.sum,
dram__bytes_read.sum, dram__bytes_write.sum): count, avg time, DRAM bytes and GB/s."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
h = rows[0]
ki, mi, vi, gi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Grid Size")
d = collections.defaultdict(lambda: collections.defaultdict(list))
for r in rows[1:]:
    d[r[ki].split("(")[0][:44] + " " + r[gi]][r[mi]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v["gpu__time_duration.sum"]) for v in d.values())
for k, v in sorted(d.items(), key=lambda x: -sum(x[1]["gpu__time_duration.sum"])):
    t = v["gpu__time_duration.sum"]
    rb = v.get("dram__bytes_read.sum", [0]); wb = v.get("dram__bytes_write.sum", [0])
    avg = sum(t) / len(t)
    byt = (sum(rb) / len(rb) + sum(wb) / len(wb))
    print(f"{k:58s} n={len(t):4d} share={100 * sum(t) / tot:5.1f}% avg={avg / 1e3:8.2f} us  dram={byt / 1e6:8.1f} MB "
          f"{byt / avg:7.1f} GB/s")
print(f"total us per step {tot / 1e3 / steps:.1f}")
