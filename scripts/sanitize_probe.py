"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one batched refactorize+solve over a 64-instance c4-recipe batch with hub rows
(k_bt_pipe2 dependency flags, k_bt_hub, k_batch_bwd2) and one level fan-in
factorize + solve of small c2/c3-recipe matrices (k_fi_* kernels)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import analysis, api, generators as gen  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

bp = gen.circuit_batch(64, 2000, 2, 200)
an = analysis.analyze(bp.A0, SolverConfig(ordering="amd"))
prior = api.factorize_analysis(an)
X, npert = api.refactorize_solve_batched(bp.values, prior, bp.rhs, hub_steps=20)
for name in ("c2", "c3"):
    p = gen.config(name, "small")
    a2 = analysis.analyze(p.A, SolverConfig(ordering=p.ordering))
    f = api.factorize_analysis(a2)
    x, _ = api.solve(p.A, f, b=p.b)
torch.cuda.synchronize()
print("sanitize probe ok", float(np.abs(X).max()))
