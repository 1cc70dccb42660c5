"""Summarise an ncu --set full report (one kernel launch) into profiles/<name>.txt.

usage: python scripts/ncu_summary.py report.ncu-rep name [extra note]"""
import csv
import io
import subprocess
import sys

import os

rep, name = sys.argv[1], sys.argv[2]
note = " ".join(sys.argv[3:])
flt = os.environ.get("NCU_FILTER", "").split()   # e.g. "--kernel-name regex:k_bt_hub --launch-skip 1"
det = subprocess.run(["ncu", "-i", rep, *flt, "--page", "details", "--csv"], capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, *flt, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
want = ["Duration", "Memory Throughput", "DRAM Throughput", "Compute (SM) Throughput", "L1/TEX Hit Rate",
        "L2 Hit Rate", "Issued Warp Per Scheduler", "No Eligible", "Warp Cycles Per Issued Instruction",
        "Block Size", "Grid Size", "Registers Per Thread", "Dynamic Shared Memory Per Block",
        "Theoretical Occupancy", "Achieved Occupancy"]
out = ["# ncu --set full summary: %s (B200, --clock-control none)" % name]
if note:
    out.append("# " + note)
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
kn = hdr.index("Kernel Name")
mi, ui, vi = hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
out.append("kernel = %s" % rows[1][kn])
seen = set()
for r in rows[1:]:
    if len(r) > vi and r[mi] in want and r[mi] not in seen:
        seen.add(r[mi])
        out.append("%s (%s) = %s" % (r[mi], r[ui], r[vi]))
rr = list(csv.reader(io.StringIO(raw)))
h, v = rr[0], rr[2] if len(rr) > 2 else rr[1]
for key in ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
            "lts__t_sector_hit_rate.pct", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"]:
    if key in h:
        i = h.index(key)
        unit = rr[1][i] if len(rr) > 2 else ""
        out.append("%s = %s %s" % (key, v[i], unit))
open("profiles/%s.txt" % name, "w").write("\n".join(out) + "\n")
print("\n".join(out))
