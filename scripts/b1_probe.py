"""Single-instance refactorize+solve through the batched kernels (B = 1) vs the
level fan-in path, per config (CUDA events, best of 5)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix  # noqa: E402


def timed(fn, reps=5):
    ts = []
    out = None
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        out = fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts), out


for name in sys.argv[1:] or ["c0", "c1"]:
    p = gen.config(name)
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    f = api.factorize_analysis(an)
    dv = torch.from_numpy(np.array(p.A.values)).cuda()
    db = torch.from_numpy(np.array(p.b)).cuda()
    t_fan, _ = timed(lambda: api.substitute(api.refactorize(dv, f), db))
    br = api.BatchedRefactorizer(f)
    dv1, db1 = dv[None].contiguous(), db[None].contiguous()
    t_b1, (x, _) = timed(lambda: br.run(dv1, db1))
    xh = x[0].cpu().numpy()
    res = np.linalg.norm(refmatrix.spmv(p.A, xh) - p.b) / np.linalg.norm(p.b)
    print("%s refactor+solve: fan-in %.3f ms, batched B=1 %.3f ms (residual %.1e)" % (name, t_fan, t_b1, res), flush=True)
