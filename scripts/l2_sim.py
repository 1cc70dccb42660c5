"""Estimate L2 reuse of the batched pipeline's U-row reads under different task orders.

A read of producer node v's values by consumer task (u, g) hits L2 (approximately)
when the bytes written between the producer task and the consumer task, times
ALPHA (reads share the cache), stay below CAP."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import generators as gen, analysis as an_mod, schedule  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

G = 128
CAP = float(os.environ.get("CAP_MB", "100")) * 2**20
ALPHA = float(os.environ.get("ALPHA", "2"))
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
A0 = base.A.with_values(bv.instance(0)[0])
an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
s = an.symbolic
pr = schedule.build_programs(an, np.zeros(s.n, np.int64))
nn = s.nnodes
W = np.diff(s.colptr)
rows = np.diff(s.node_first)
wbytes = rows * W * 256.0
valoff = np.asarray(s.valoff)
node_of_pos = lambda p: np.searchsorted(valoff, p, side="right") - 1
# reads per consumer node: (producer node, bytes)
row_ptr = pr.row_ptr
cons_row = np.repeat(np.arange(s.n), np.diff(row_ptr))
cons = np.asarray(s.node_of)[cons_row]
prod = node_of_pos(pr.st_src)
rb = (pr.st_cnt + 2) * 256.0
hub = pr.node_hub.astype(bool)
lp = np.asarray(s.level_ptr)
ln = np.asarray(s.level_nodes)
nl = len(lp) - 1
print("nodes", nn, "levels", nl, "hubs", hub.sum(), "read MB/group %.1f" % (rb.sum() / 2**20),
      "write MB/group %.1f" % (wbytes.sum() / 2**20))


def order(skew=1, window=0):
    """task list [(node, group)] in claim order, segment by segment."""
    out = []
    l = 0
    while l < nl:
        l1 = l + 1
        if not hub[ln[lp[l]:lp[l + 1]]].any():
            while l1 < nl and not hub[ln[lp[l1]:lp[l1 + 1]]].any():
                l1 += 1
        hs = [u for u in ln[lp[l]:lp[l + 1]] if hub[u]]
        for g in range(G):
            for u in hs:
                out.append((u, g))
        L = l1 - l
        lev = [[u for u in ln[lp[l + k]:lp[l + k + 1]] if not hub[u]] for k in range(L)]
        groups = range(G)
        wins = [list(groups)] if not window else [list(range(a, min(G, a + window))) for a in range(0, G, window)]
        # windows are laid one after another along the diagonal (window w starts
        # when window w-1 has advanced `stagger` levels)
        cells = []
        for wi, wg in enumerate(wins):
            for gi, g in enumerate(wg):
                for k in range(L):
                    d = skew * gi + k + (wi * (window * skew) if window else 0)
                    cells.append((d, k, g))
        cells.sort()
        for d, k, g in cells:
            for u in lev[k]:
                out.append((u, g))
        l = l1
    return out


def evaluate(tl):
    t = np.array(tl)
    pos = np.empty((nn, G), np.int64)
    pos[t[:, 0], t[:, 1]] = np.arange(len(t))
    cw = np.concatenate([[0], np.cumsum(wbytes[t[:, 0]])])
    hit = 0.0
    tot = 0.0
    for g in range(0, G, 8):
        pc = pos[cons, g]
        pp = pos[prod, g]
        dist = (cw[pc] - cw[pp + 1]) * ALPHA
        h = dist < CAP
        hit += rb[h].sum()
        tot += rb.sum()
    return hit / tot


for name, kw in [("diag skew1", {}), ("diag skew2", {"skew": 2}), ("diag skew4", {"skew": 4}),
                 ("win32", {"window": 32}), ("win16", {"window": 16}), ("win8", {"window": 8})]:
    print("%-12s hit %.3f" % (name, evaluate(order(**kw))), flush=True)
