"""Batched refactorize+solve time vs batch size (CUDA events)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

Bmax = 8192
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
vals = np.empty((Bmax, base.A.nnz))
rhs = np.empty((Bmax, 20000))
bv.fill(range(Bmax), vals, rhs, 16)
A0 = base.A.with_values(bv.instance(0)[0])
an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
prior = api.factorize_analysis(an)
dv = torch.from_numpy(vals).cuda()
dr = torch.from_numpy(rhs).cuda()
for B in [int(a) for a in sys.argv[1:]] or [512, 1024, 2048, 4096, 8192]:
    br = api.BatchedRefactorizer(prior)
    x = torch.empty((B, 20000), dtype=torch.float64, device="cuda")
    npert = torch.empty(B, dtype=torch.int32, device="cuda")
    for _ in range(2):
        br.run(dv[:B], dr[:B], x, npert)
    ts = []
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        br.run(dv[:B], dr[:B], x, npert)
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    print("B %5d  ms %.3f  inst/s %.0f" % (B, min(ts), B / min(ts) * 1e3), flush=True)
