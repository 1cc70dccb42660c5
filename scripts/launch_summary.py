"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

usage: python scripts/launch_summary.py launches.csv "header note" > profiles/<name>.txt"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 5]
h = rows[0]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
agg = collections.OrderedDict()
for r in rows[1:]:
    k = r[ki].split("(")[0].replace("void ", "").replace("hy::", "").split("<")[0]
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(a[1] for a in agg.values())
print("# " + " ".join(sys.argv[2:]))
print("# kernel  launches  total_us  share")
for k, a in sorted(agg.items(), key=lambda x: -x[1][1]):
    print("%s %d %.0f %.1f%%" % (k, a[0], a[1], 100 * a[1] / tot))
print("# total %.1f ms (ncu: cold-cache, serialised launches)" % (tot / 1e3))
