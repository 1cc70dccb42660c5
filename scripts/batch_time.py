"""Device-resident c4 step time (refactorize+solve over 4096 instances), CUDA events,
median of K steps after W warm-ups.  HYLU_LIB_PATH selects a library variant."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

B = int(os.environ.get("B", 4096))
K = int(os.environ.get("K", 10))
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
vals = np.empty((B, base.A.nnz))
rhs = np.empty((B, 20000))
bv.fill(range(B), vals, rhs, 16)
A0 = base.A.with_values(bv.instance(0)[0])
an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
prior = api.factorize_analysis(an)
br = api.BatchedRefactorizer(prior)
dv = torch.from_numpy(vals).cuda()
dr = torch.from_numpy(rhs).cuda()
for _ in range(3):
    x, npert = br.run(dv, dr, refine=False)
ts = []
for _ in range(K):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    x, npert = br.run(dv, dr, refine=False)
    b.record()
    torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
print(json.dumps({"lib": os.environ.get("HYLU_LIB_PATH", "default"), "B": B, "ms_median": float(np.median(ts)),
                  "ms_min": float(min(ts)), "per_s": B / float(np.median(ts)) * 1e3,
                  "xsum": float(x.sum().item())}), flush=True)
