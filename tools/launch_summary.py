#!/usr/bin/env python3
"""Summarise an ncu launch list (gpu__time_duration.sum per launch) by kernel."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
ki, mi, gi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Grid Size")
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[1:]:
    v = float(r[mi].replace(",", ""))
    name = r[ki].split("(")[0][:56] + " " + r[gi]
    tot[name] += v
    cnt[name] += 1
s = sum(tot.values())
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
for k, v in sorted(tot.items(), key=lambda x: -x[1]):
    print("%-72s n=%4d share=%5.1f%% avg=%8.2f us" % (k, cnt[k], 100 * v / s, v / cnt[k] / 1e3))
print("total us per step %.1f" % (s / 1e3 / steps))
