"""Sweep HYLU_SPLIT_SRC (split-K threshold of packed update items)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod, schedule  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

name = sys.argv[1]
p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
dv = torch.from_numpy(np.array(p.A.values)).cuda()
for cap in [int(a) for a in sys.argv[2:]]:
    schedule.SPLIT_SRC = cap
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    api.factorize_analysis(an, dv)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.factorize_analysis(an, dv)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(name, "split_src", cap, "factor ms %.2f" % min(ts), flush=True)
