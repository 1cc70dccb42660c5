"""From an ncu --set full report with many launches of one kernel: pick the longest launch and
print its key metrics next to the totals over all launches.

usage: python scripts/ncu_pick_longest.py report.ncu-rep > profiles/<name>.txt"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h, units, rows = rr[0], rr[1], rr[2:]
col = {k: i for i, k in enumerate(h)}


def f(r, k):
    try:
        return float(r[col[k]].replace(",", ""))
    except (KeyError, ValueError):
        return float("nan")


dur = "gpu__time_duration.sum"
scale = {"ns": 1e-6, "us": 1e-3, "ms": 1.0, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}[units[col[dur]]]
keys = [dur, "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__t_sector_hit_rate.pct",
        "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor_subpipe_dmma.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__grid_size", "launch__registers_per_thread", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio"]
tot = sum(f(r, dur) for r in rows) * scale
best = max(rows, key=lambda r: f(r, dur))
print("# %d launches of %s, total %.2f ms (ncu: cold-cache, serialised)" % (len(rows), best[col["Kernel Name"]].split("(")[0], tot))
wd = sum(f(r, dur) * f(r, keys[5]) for r in rows) / sum(f(r, dur) for r in rows)
print("# duration-weighted DMMA pipe activity over all launches: %.1f %%" % wd)
print("# longest launch (ID %s):" % best[col["ID"]])
for k in keys:
    if k in col:
        print("%s = %s %s" % (k, best[col[k]], units[col[k]]))
print("# ten longest launches: ms, DMMA %, warps active %, grid")
for r in sorted(rows, key=lambda r: -f(r, dur))[:10]:
    print("%.3f  %.1f  %.1f  %d" % (f(r, dur) * scale, f(r, keys[5]), f(r, keys[7]), int(f(r, "launch__grid_size"))))
