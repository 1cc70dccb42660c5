"""Sweep the fan-in deadline-merge caps (HYLU_MERGE_ROWS / HYLU_MERGE_RECS)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

name = sys.argv[1]
p = gen.fem27(int(name[3:])) if name.startswith("c3k") else gen.config(name)
dv = torch.from_numpy(np.array(p.A.values)).cuda()
ref = None
for spec in sys.argv[2:]:
    rows, recs = spec.split(",")
    os.environ["HYLU_MERGE_ROWS"], os.environ["HYLU_MERGE_RECS"] = rows, recs
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    t0 = time.perf_counter()
    f = api.factorize_analysis(an, dv)
    tp = time.perf_counter() - t0
    ts = []
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g = api.factorize_analysis(an, dv)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if ref is None:
        ref = g.values.clone()
    err = float((g.values - ref).abs().max() / ref.abs().max())
    print(name, "merge rows<=%s recs<=%s" % (rows, recs), "items", len(an.symbolic._fanin_plan.up_t),
          "factor ms %.1f" % min(ts), "first-call %.1fs" % tp, "reldiff %.1e" % err, flush=True)
