"""One factorize (+ optional solve) of a named config (ncu launch lists)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

name = sys.argv[1]
solve = len(sys.argv) > 2 and sys.argv[2] == "solve"
p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
dv = torch.from_numpy(np.array(p.A.values)).cuda()
f = api.factorize_analysis(an, dv)
if solve:
    x = api.substitute(f, torch.from_numpy(np.array(p.b)).cuda())
torch.cuda.synchronize()
print("ok")
