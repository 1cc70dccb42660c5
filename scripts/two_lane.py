"""Probe: the c4 batch as two half-batches on two handles / two streams (do the
low-occupancy phases of one half (hub, backward solve) overlap the other's
pipeline?).  Prints one JSON line per configuration."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

B = 4096
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
vals = np.empty((B, base.A.nnz))
rhs = np.empty((B, 20000))
bv.fill(range(B), vals, rhs, 16)
A0 = base.A.with_values(bv.instance(0)[0])
dv = torch.from_numpy(vals).cuda()
dr = torch.from_numpy(rhs).cuda()
lanes = []
for _ in range(4):
    an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
    prior = api.factorize_analysis(an)
    lanes.append(api.BatchedRefactorizer(prior))
streams = [torch.cuda.Stream() for _ in range(4)]


def run(nl, split):
    bounds = np.linspace(0, B, nl + 1).astype(int) if split is None else split
    outs = []
    cur = torch.cuda.current_stream()
    for k in range(nl):
        streams[k].wait_stream(cur)
        a, b = bounds[k], bounds[k + 1]
        outs.append(lanes[k].run(dv[a:b], dr[a:b], stream=streams[k], refine=False))
    for k in range(nl):
        cur.wait_stream(streams[k])
    return outs


for nl in (1, 2, 3, 4):
    for _ in range(3):
        run(nl, None)
    ts = []
    for _ in range(8):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        outs = run(nl, None)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    x = torch.cat([o[0] for o in outs])
    print(json.dumps({"lanes": nl, "ms_median": float(np.median(ts)), "per_s": B / float(np.median(ts)) * 1e3,
                      "xsum": float(x.sum().item())}), flush=True)
