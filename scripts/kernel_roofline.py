"""Per-kernel roofline table from an ncu metric list over every launch of a run:

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active \
      --clock-control none --csv --log-file run.csv python <program>

usage: python scripts/kernel_roofline.py run.csv "title" [hbm_gbs]
Per kernel name: launches, total time, DRAM bytes, achieved DRAM GB/s (bytes / time) and
its fraction of the HBM peak, time-weighted DMMA-pipe and FP64-pipe activity."""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, title = sys.argv[1], sys.argv[2]
try:
    peak = float(sys.argv[3])
except (IndexError, ValueError):
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
rows = [r for r in csv.reader(open(path)) if len(r) > 5]
h = rows[0]
ID, KN, MN, MU, MV = (h.index(x) for x in ("ID", "Kernel Name", "Metric Name", "Metric Unit", "Metric Value"))
unit = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1.0}
launch = collections.defaultdict(dict)
names = {}
for r in rows[1:]:
    v = float(r[MV].replace(",", "")) * unit.get(r[MU], 1.0)
    launch[r[ID]][r[MN]] = v
    names[r[ID]] = r[KN].split("(")[0].replace("void ", "").replace("hy::", "").split("<")[0]
agg = collections.OrderedDict()
for i, m in launch.items():
    a = agg.setdefault(names[i], dict(n=0, t=0.0, b=0.0, dm=0.0, fp=0.0))
    t = m.get("gpu__time_duration.sum", 0.0)
    a["n"] += 1
    a["t"] += t
    a["b"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    a["dm"] += t * m.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
    a["fp"] += t * m.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 0.0)
tot = sum(a["t"] for a in agg.values())
print("# %s" % title)
print("# ncu per-launch metrics aggregated per kernel (cold-cache, serialised launches); HBM peak %.0f GB/s" % peak)
print("%-18s %7s %10s %6s %10s %8s %7s %7s %7s" % ("kernel", "launch", "time_ms", "share", "DRAM_GB", "GB/s", "%HBM", "DMMA%", "FP64%"))
for k, a in sorted(agg.items(), key=lambda x: -x[1]["t"]):
    gbs = a["b"] / a["t"] / 1e9 if a["t"] else 0.0
    print("%-18s %7d %10.3f %5.1f%% %10.3f %8.0f %6.1f%% %6.1f%% %6.1f%%" % (
        k, a["n"], a["t"] * 1e3, 100 * a["t"] / tot, a["b"] / 1e9, gbs, 100 * gbs / peak,
        a["dm"] / a["t"] if a["t"] else 0, a["fp"] / a["t"] if a["t"] else 0))
print("# total %.3f ms" % (tot * 1e3))
