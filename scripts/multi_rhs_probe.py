"""32 right-hand sides per config through each multi-RHS route (partition / levels /
columns): CUDA-event ms (best of 3) and the max residual.  Development probe."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix  # noqa: E402

NR = 32
for name in sys.argv[1:]:
    p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    f = api.factorize_analysis(an)
    B = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, (NR, p.A.n))).cuda()
    out = {"config": name, "auto": api.multi_rhs_method(f)}
    for m in ("partition", "levels", "columns"):
        X = api.substitute_multi(f, B, method=m)
        ts = []
        for _ in range(3):
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            s.record()
            X = api.substitute_multi(f, B, method=m)
            e.record()
            torch.cuda.synchronize()
            ts.append(s.elapsed_time(e))
        Xh = X.cpu().numpy()
        Bh = B.cpu().numpy()
        res = max(float(np.linalg.norm(refmatrix.spmv(p.A, Xh[j]) - Bh[j]) / np.linalg.norm(Bh[j])) for j in (0, NR - 1))
        out[m] = {"ms": min(ts), "residual": res}
    print(json.dumps(out), flush=True)
