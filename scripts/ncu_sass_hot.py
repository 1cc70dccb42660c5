"""Summarise an ncu report's SASS source page: top instructions by stall samples,
and the stall reasons of the hottest ones.  usage: ncu_sass_hot.py report [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
h = rows[0]
si = h.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, c in enumerate(h) if c.startswith("stall_")]
data = []
for r in rows[1:]:
    if len(r) < len(h):
        continue
    try:
        data.append((int(r[si]), r[1].strip(), {h[i]: int(r[i]) for i in stall_cols if r[i] not in ("", "0")}, r[0]))
    except ValueError:
        pass
tot = sum(d[0] for d in data)
print("total samples", tot)
agg = {}
for d in data:
    for k, v in d[2].items():
        agg[k] = agg.get(k, 0) + v
print("stall reasons:", ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:10]))
idx = {d[3]: i for i, d in enumerate(data)}
for d in sorted(data, key=lambda x: -x[0])[:N]:
    i = idx[d[3]]
    top = sorted(d[2].items(), key=lambda x: -x[1])[:3]
    print("%5.1f%% %5d  %-60s %s" % (100 * d[0] / tot, i, d[1][:60], " ".join("%s:%d" % (k[6:], v) for k, v in top)))
