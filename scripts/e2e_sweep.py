"""e2e (host pinned buffers, chunked H2D / compute / D2H) timing for chunk layouts."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402

B = 4096
base = gen.circuit(20000, 3, 2000, gen.SEEDS["c4"])
bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
vals = np.empty((B, base.A.nnz))
rhs = np.empty((B, 20000))
bv.fill(range(B), vals, rhs, 16)
A0 = base.A.with_values(bv.instance(0)[0])
an = an_mod.analyze(A0, SolverConfig(ordering="amd"))
prior = api.factorize_analysis(an)
br = api.BatchedRefactorizer(prior)
h_vals = torch.from_numpy(vals).pin_memory()
h_rhs = torch.from_numpy(rhs).pin_memory()
h_x = torch.empty((B, 20000), dtype=torch.float64).pin_memory()
h_np = torch.empty(B, dtype=torch.int32).pin_memory()
layouts = {
    "u8": dict(chunks=8), "u4": dict(chunks=4), "u2": dict(chunks=2), "u3": dict(chunks=3),
    "p8": dict(chunks=8, pipelined=True), "p6": dict(chunks=6, pipelined=True),
    "p4": dict(chunks=4, pipelined=True), "p3": dict(chunks=3, pipelined=True),
    "p2": dict(chunks=2, pipelined=True),
}
K = 5
for name in (sys.argv[1:] or layouts):
    kw = layouts[name]
    for _ in range(2):
        br.run_host(h_vals, h_rhs, h_x, h_np, **kw)
    br.host_wait()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(K):
        br.run_host(h_vals, h_rhs, h_x, h_np, **kw)
    br.host_wait()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / K
    print("%-4s ms/step %.2f  inst/s %.0f" % (name, ms, B / ms * 1e3), flush=True)
