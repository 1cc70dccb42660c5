"""Time one batched refactorize+solve pass (c4, 4096 instances) with the library
named by HYLU_LIB_PATH (kernel build variants): median / min of 7 after 2 warm-ups."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix  # noqa: E402

B = 4096
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
x = torch.empty((B, 20000), dtype=torch.float64, device="cuda")
npert = torch.empty(B, dtype=torch.int32, device="cuda")
for _ in range(2):
    br.run(dv, dr, x, npert)
ts = []
for _ in range(7):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    br.run(dv, dr, x, npert)
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e))
xh = x[:3].cpu().numpy()
res = max(np.linalg.norm(refmatrix.spmv(A0.with_values(vals[b]), xh[b]) - rhs[b]) / np.linalg.norm(rhs[b])
          for b in range(3))
print("%-28s ms %.3f (min %.3f)  inst/s %.0f  res %.1e" % (os.path.basename(os.environ.get("HYLU_LIB_PATH", "default")),
      np.median(ts), min(ts), B / min(ts) * 1e3, res), flush=True)
