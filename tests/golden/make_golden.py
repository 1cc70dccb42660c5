"""Generate tests/golden/*.npz — run in the build container (needs /root/reference).

For small seeded versions of the five configs this records, from the reference's
own shipped host code (polylu._matching.max_weight_match, polylu._amd
.amd_permutation, imported from /root/reference/pkg/src): row_perm, dr, dc and the
fill-reducing permutation; plus the symbolic statistics and, from the oracle
(pinned by tests/test_oracle_spec.py against SPEC's known answers), the factor
values, inner_perm and solution.  The GPU box has no /root/reference: the tests
compare against these files.

    PYTHONPATH=/root/repo python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
os.environ["POLYLU_PATH"] = "/root/reference/pkg/src"

from paper_2509_07690_b200 import analysis, generators as gen  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig  # noqa: E402
from oracle import numeric as on  # noqa: E402

CASES = {
    "c0": lambda: gen.lap2d(10),
    "c1": lambda: gen.circuit(600, 1, 60),
    "c2": lambda: gen.convdiff3d(6),
    "c3": lambda: gen.fem27(3),
    "c4": lambda: gen.circuit_batch(3, 600, 1, 60),
}


def main():
    import polylu.matrix as pm
    assert pm.__file__.startswith("/root/reference"), pm.__file__
    for name, make in CASES.items():
        p = make()
        A = p.A0 if name == "c4" else p.A
        b = p.rhs[0] if name == "c4" else p.b
        an = analysis.analyze(A, SolverConfig(ordering=p.ordering))
        s = an.symbolic
        f = on.factorize(an)
        x, _ = on.solve(an, f, b)
        out = dict(row_ptr=A.row_ptr, col_idx=A.col_idx, values=A.values, b=b,
                   row_perm=an.pivot_scale.row_perm, dr=an.pivot_scale.dr, dc=an.pivot_scale.dc,
                   perm=an.ordering.perm, node_first=s.node_first, cols=s.cols,
                   flops=s.flops, fill_nnz=s.fill_nnz, kernel_mode=int(s.kernel_mode),
                   F=f.values, inner_perm=f.inner_perm, x=x)
        if name == "c4":
            out["batch_values"] = p.values
            out["batch_rhs"] = p.rhs
        np.savez_compressed(os.path.join(HERE, "%s.npz" % name), **out)
        print(name, A.n, A.nnz, s.fill_nnz, s.kernel_mode.name)


if __name__ == "__main__":
    main()
