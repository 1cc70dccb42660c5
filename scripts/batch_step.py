"""One batched refactorize+solve step (for ncu launch lists / captures)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
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
for _ in range(reps):
    x, npert = br.run(dv, dr)
torch.cuda.synchronize()
print("ok", float(x[0, :4].sum()))
