"""Pin the METIS nested-dissection permutations of the full-size c2 / c3 configs.

Nested dissection is outside the reference: the oracle and the
device path both factor the permutation ``preprocess.nd_order`` returns.  This
script (run in the build container) stores that permutation for c2 (convdiff3d(64))
and c3 (fem27(48)) as compressed int32 arrays; ``tests/test_golden.py`` recomputes
it and requires the identical array, so a different METIS build or a generator
change cannot silently move the full-size parity tests to another ordering.

    PYTHONPATH=. python tests/golden/make_nd.py
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_2509_07690_b200 import generators as gen, preprocess as pp  # noqa: E402


def nd_perm(p):
    ps = pp.static_pivot(p.A)
    ap, ai = pp.pivoted_sym_pattern(p.A, ps)
    return pp.nd_order(ap, ai).perm


def main():
    for name, p in (("c2_64", gen.convdiff3d(64)), ("c3_48", gen.fem27(48))):
        perm = nd_perm(p)
        np.savez_compressed(os.path.join(HERE, "nd_%s.npz" % name), perm=perm.astype(np.int32),
                            n=p.A.n, nnz=p.A.nnz)
        print(name, p.A.n, perm[:5])


if __name__ == "__main__":
    main()
