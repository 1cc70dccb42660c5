"""c3 literal recipe at fem27(K): device factors per update-kernel variant against
the oracle; where is the largest difference (node, row offset, column position)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix  # noqa: E402
from oracle import numeric as on  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 16
p = gen.fem27(k, recipe="literal")
an = an_mod.analyze(p.A, SolverConfig(ordering="nd"))
s = an.symbolic
ref = on.factorize(an, threads=16)
f = api.factorize_analysis(an)
ctx = f._ctx
amax = np.abs(ref.values).max()
for tc in (5, 4, 2, 0):
    ctx.set_option("fanin_tc", tc)
    g = api.factorize_analysis(an)
    v = g.host_values()
    d = np.abs(v - ref.values)
    i = int(np.argmax(d))
    u = int(np.searchsorted(s.valoff, i, side="right") - 1)
    W = int(s.colptr[u + 1] - s.colptr[u])
    t, q = divmod(i - int(s.valoff[u]), W)
    x, _ = api.solve(p.A, g, b=p.b)
    res = float(np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b))
    # relative to the node's own magnitude
    blk = ref.values[s.valoff[u]:s.valoff[u + 1]]
    print(json.dumps({"tc": tc, "max_abs": float(d.max()), "rel_global": float(d.max() / max(1, amax)),
                      "amax": float(amax), "node": u, "node_rows": int(s.node_first[u + 1] - s.node_first[u]),
                      "W": W, "t": int(t), "q": int(q), "nl": int(s.nl[u]), "ref_val": float(ref.values[i]),
                      "node_amax": float(np.abs(blk).max()), "level": int(s.level[u]), "nlev": int(len(s.level_ptr) - 1),
                      "inner_perm_equal": bool(np.array_equal(g.host_inner_perm(), ref.inner_perm)),
                      "frac_gt_1e-11": float((d > 1e-11 * max(1, amax)).mean()), "residual": res}), flush=True)
