"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck):
one batched refactorize+solve over a 64-instance c4-recipe batch with hub rows
(k_bt_pipe2 dependency flags, k_bt_hub, k_batch_bwd2) and one level fan-in
factorize + solve of small c2/c3-recipe matrices (k_fi_* kernels) in every kernel mode,
the batched refinement of a perturbed instance (masked residual / update kernels) and
the partition-based multi-RHS solve (k_msolve)."""
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
vals = bp.values.copy()
gen.zero_first_pivot(an, vals[5])
X, npert = api.refactorize_solve_batched(vals, prior, bp.rhs, hub_steps=20)
assert npert[5] > 0 and 5 in api.refactorize_solve_batched.last_reports
for name in ("c2", "c3"):
    p = gen.config(name, "small")
    a2 = analysis.analyze(p.A, SolverConfig(ordering=p.ordering, seg_nnz_threshold=2000))
    for mode in (0, 2):
        f = api.factorize_analysis(a2, opts=api.FactorOptions(kernel_override=mode))
        x, _ = api.solve(p.A, f, b=p.b)
    f._ctx.ensure_partition(config=a2.config)
    Xm = api.substitute_multi(f, np.stack([p.b, 2 * p.b]))
torch.cuda.synchronize()
print("sanitize probe ok", float(np.abs(X).max()))
