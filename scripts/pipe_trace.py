"""Task timeline of the batched pipeline kernel (k_bt_pipe2) on c4: needs a library
built with -DHYLU_TRACE (HYLU_LIB_PATH=variants/libhylu_trace.so).  Per task the
kernel records claim / dependencies-ready / end timestamps (%globaltimer); this script
reports where warp time goes (waiting on flags vs running steps), per level."""
import ctypes
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, device, generators as gen, analysis as an_mod, schedule  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

B = int(os.environ.get("B", 4096))
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
vals = np.empty((B, base.A.nnz))
rhs = np.empty((B, 20000))
bv.fill(range(B), vals, rhs, 16)
A0 = base.A.with_values(bv.instance(0)[0])
an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
s = an.symbolic
prior = api.factorize_analysis(an)
br = api.BatchedRefactorizer(prior)
dv = torch.from_numpy(vals).cuda()
dr = torch.from_numpy(rhs).cuda()
for _ in range(3):
    x, npert = br.run(dv, dr, refine=False)
torch.cuda.synchronize()
lib = device.library()
nt = s.nnodes * ((B + 63) // 64)
buf = torch.zeros(nt * 12, dtype=torch.int64, device="cuda")
hbuf = torch.zeros(1 + 8 * 4096, dtype=torch.int64, device="cuda")
lib.hy_debug_hub_trace.argtypes = [ctypes.c_void_p]
lib.hy_debug_hub_trace(ctypes.c_void_p(hbuf.data_ptr()))
lib.hy_debug_pipe_trace.argtypes = [ctypes.c_void_p]
rc = lib.hy_debug_pipe_trace(ctypes.c_void_p(buf.data_ptr()))
assert rc == 0, rc
x, npert = br.run(dv, dr, refine=False)
torch.cuda.synchronize()
lib.hy_debug_pipe_trace(ctypes.c_void_p(0))
lib.hy_debug_hub_trace(ctypes.c_void_p(0))
hb = hbuf.cpu().numpy()
hrec = hb[1:1 + 8 * int(hb[0])].reshape(-1, 8)
for hu in np.unique(hrec[:, 0]):
    hm = hrec[:, 0] == hu
    c = hrec[hm][:, 2:6].astype(np.float64) / 1.965e3   # us at 1965 MHz
    print("hub node %d: %d CTAs  total %.0f us (max %.0f)  init %.0f  levels %.0f  fwd %.0f" % (
        hu, hm.sum(), c[:, 0].mean(), c[:, 0].max(), c[:, 1].mean(), c[:, 2].mean(), c[:, 3].mean()))
t = buf.cpu().numpy().reshape(-1, 12)
t = t[t[:, 0] != 0]
claim, ready, end, tag = t[:, 0], t[:, 1], t[:, 2], t[:, 3]
u = tag >> 32
g = (tag >> 16) & 0xffff
sm = tag & 0xffff
t0 = claim.min()
span = (end.max() - t0) / 1e3
wait = (ready - claim) / 1e3
work = (end - ready) / 1e3
lev = np.asarray(s.level)[u]
pr = schedule.build_programs(an, np.zeros(s.n, np.int64))
steps_row = np.diff(pr.row_ptr)
steps_node = np.add.reduceat(steps_row, np.asarray(s.node_first)[:-1])
cnt_node = np.zeros(s.nnodes)
cons_row = np.repeat(np.arange(s.n), steps_row)
np.add.at(cnt_node, np.asarray(s.node_of)[cons_row], pr.st_cnt)
out = {"tasks": int(len(t)), "span_us": float(span), "warp_slots": int(len(np.unique(sm))) * 16,
       "sum_wait_ms": float(wait.sum() / 1e3), "sum_work_ms": float(work.sum() / 1e3),
       "slot_time_ms": float(span * len(np.unique(sm)) * 16 / 1e3)}
print(json.dumps(out))
print("lev  tasks   wait_us(mean/p50/p99)   work_us(mean/p99)  steps/task  upd/task  us/step  claim window [us]")
for l in range(int(lev.max()) + 1):
    m = lev == l
    if not m.any():
        continue
    st = steps_node[u[m]].mean()
    print("%3d %6d   %8.1f %8.1f %8.1f   %8.1f %8.1f   %7.1f %8.1f  %6.2f   %8.0f..%8.0f" % (
        l, m.sum(), wait[m].mean(), np.median(wait[m]), np.percentile(wait[m], 99), work[m].mean(),
        np.percentile(work[m], 99), st, cnt_node[u[m]].mean(), work[m].mean() / max(st, 1e-9),
        (claim[m].min() - t0) / 1e3, (claim[m].max() - t0) / 1e3))
# phase cycle counters (SM clock): claim->deps ready, node body, fence; inside the body:
# row init (A scatter), multiplier (pivot/target value arrives), update batches, row finalize
cyc = t[:, 4:11].astype(np.float64)
names = ["init", "mult", "upd", "fin", "claim+poll", "body", "fence"]
tot = cyc[:, 4:7].sum()
print("phase shares of task cycles: " + ", ".join("%s %.1f%%" % (n, 100 * cyc[:, k].sum() / tot) for k, n in enumerate(names)))
nst = steps_node[u].astype(np.float64)
nup = cnt_node[u]
m = nst > 0
print("per step: mult %.0f cyc, upd %.0f cyc (%.0f per update); per task: init %.0f, fin %.0f, claim+poll %.0f, fence %.0f" % (
    cyc[m, 1].sum() / nst[m].sum(), cyc[m, 2].sum() / nst[m].sum(), cyc[m, 2].sum() / nup[m].sum(),
    cyc[:, 0].mean(), cyc[:, 3].mean(), cyc[:, 4].mean(), cyc[:, 6].mean()))
for lo, hi in [(0, 1), (1, 3), (3, 6), (6, 10), (10, 20), (20, 40)]:
    mm = (lev >= lo) & (lev < hi)
    ms = mm & m
    print("levels %2d-%2d: tasks %7d  init %6.0f  fin %6.0f  claim+poll %6.0f  fence %6.0f | per step mult %5.0f upd %5.0f" % (
        lo, hi - 1, mm.sum(), cyc[mm, 0].mean(), cyc[mm, 3].mean(), cyc[mm, 4].mean(), cyc[mm, 6].mean(),
        cyc[ms, 1].sum() / max(1, nst[ms].sum()), cyc[ms, 2].sum() / max(1, nst[ms].sum())))
# concurrency over time: tasks working / waiting in 100 buckets
edges = np.linspace(0, span, 51)
print("time_us  working  waiting")
for a, b2 in zip(edges[:-1], edges[1:]):
    mid = t0 + (a + b2) / 2 * 1e3
    print("%8.0f %7d %7d" % ((a + b2) / 2, ((ready <= mid) & (end > mid)).sum(), ((claim <= mid) & (ready > mid)).sum()))
if os.environ.get("TRACE_SAVE"):
    np.save("gpurun_out/pipe_trace.npy", t)
