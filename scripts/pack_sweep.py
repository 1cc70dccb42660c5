"""Sweep the fan-in packing criterion (HYLU_PACK_M / HYLU_PACK_N)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

name = sys.argv[1]
p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
dv = torch.from_numpy(np.array(p.A.values)).cuda()
base = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
for spec in sys.argv[2:]:
    m, n = spec.split(",")
    os.environ["HYLU_PACK_M"], os.environ["HYLU_PACK_N"] = m, n
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    f = api.factorize_analysis(an, dv)
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        api.factorize_analysis(an, dv)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(name, "pack m<%s n>=%s" % (m, n), "factor ms %.1f" % min(ts), flush=True)
