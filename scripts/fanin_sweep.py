"""Time the fan-in factorization with the DMMA routing on/off."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

name = sys.argv[1]
p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
dv = torch.from_numpy(np.array(p.A.values)).cuda()
f = api.factorize_analysis(an, dv)
ctx = f._ctx
opt = os.environ.get("SWEEP_OPT", "fanin_dmma")
for v in [int(x) for x in os.environ.get("SWEEP_VALS", "1,0,1").split(",")]:
    ctx.set_option(opt, v)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g = api.factorize_analysis(an, dv)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    err = float((g.values - f.values).abs().max())
    print(name, opt, v, "factor ms %.1f" % min(ts), "GFLOP/s %.0f" % (an.symbolic.flops / min(ts) / 1e6),
          "maxdiff vs first %.2e" % err, flush=True)
