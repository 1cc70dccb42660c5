"""Partition-based substitution (Fig. 3): the
host partition against SPEC's build_partition examples and invariants, and the
device launch lists (through their CPU interpreter) against the oracle.  CPU only;
the device parity is in test_gpu_parity.py::test_solve_multi_*."""
import numpy as np
import pytest

from paper_2509_07690_b200 import analysis as an_mod
from paper_2509_07690_b200 import generators as gen
from paper_2509_07690_b200 import partition as pt
from paper_2509_07690_b200._ref import SolverConfig, SparseMatrixCSR
from oracle import numeric as on


def _an(dense, ordering="natural"):
    A = SparseMatrixCSR.from_dense(np.asarray(dense, float))
    return an_mod.analyze(A, SolverConfig(ordering=ordering))


def test_diagonal_single_bulk_segment():
    """diagonal matrix -> single segment, fully bulk, no rectangular blocks."""
    an = _an(np.diag(np.arange(1.0, 41.0)))
    p = pt.build_partition(an.symbolic, threads=4)
    assert p.nsegments == 1 and len(p.cut_points) == 0 and p.bulk_segment
    assert p.rect_l_nnz.sum() == 0 and p.rect_u_nnz.sum() == 0


def test_tridiagonal_one_chain():
    """tridiagonal -> one long chain solved sequentially, no cuts."""
    n = 50
    T = np.diag(np.full(n, 4.0)) + np.diag(np.full(n - 1, -1.0), 1) + np.diag(np.full(n - 1, -1.5), -1)
    an = _an(T)
    p = pt.build_partition(an.symbolic, threads=4)
    assert len(p.cut_points) == 0 and p.nsegments == 1 and not p.bulk_segment
    assert p.sequential[0]


def test_block_arrow_cut_at_tail_and_balanced_ranges():
    """many independent leading blocks + dense tail -> the cut lands on
    the block/tail boundary and the coupling block's row ranges balance its
    nonzeros within one row."""
    rng = np.random.default_rng(7)
    nb, bs, tail = 24, 3, 20
    n = nb * bs + tail
    M = np.zeros((n, n))
    for k in range(nb):
        s = slice(k * bs, (k + 1) * bs)
        M[s, s] = rng.uniform(-1, 1, (bs, bs)) + 4 * np.eye(bs)
    M[nb * bs:, :] = rng.uniform(-1, 1, (tail, n)) * (rng.uniform(0, 1, (tail, n)) < 0.5)
    M[:, nb * bs:] += (rng.uniform(-1, 1, (n, tail)) * (rng.uniform(0, 1, (n, tail)) < 0.3))
    M[nb * bs:, nb * bs:] += 8 * np.eye(tail)
    M += np.diag(np.full(n, 6.0))
    an = _an(M)
    s = an.symbolic
    threads = 4
    p = pt.build_partition(s, threads=threads, config=SolverConfig(seg_nnz_threshold=10 ** 9))
    assert p.bulk_segment
    assert list(p.cut_points) == [nb * bs]
    assert p.rect_l_nnz[1] > 0
    r = p.rect_l_ranges[1]
    cl, _ = pt._split_counts(s, int(p.seg_rows[1]), int(p.seg_rows[2]))
    per = [int(cl[r[t] - r[0]:r[t + 1] - r[0]].sum()) for t in range(threads)]
    assert sum(per) == p.rect_l_nnz[1]
    assert max(per) - min(per) <= 2 * int(cl.max())


@pytest.mark.parametrize("name,thr", [("c0", 300), ("c1", 2000), ("c2", 20000), ("c3", 20000)])
def test_partition_covers_rows_and_applies_every_entry_once(name, thr):
    """segments cover [0, n) exactly and disjointly; the device launch
    lists (CPU interpreter) apply every stored L/U entry exactly once per
    substitution and reproduce the oracle's solution."""
    p_ = gen.config(name, "small")
    an = an_mod.analyze(p_.A, SolverConfig(ordering=p_.ordering))
    s = an.symbolic
    part = pt.build_partition(s, threads=8, config=SolverConfig(seg_nnz_threshold=thr))
    assert part.seg_rows[0] == 0 and part.seg_rows[-1] == s.n
    assert np.all(np.diff(part.seg_rows) > 0)
    assert part.nsegments >= 2
    fac = on.factorize(an)
    rng = np.random.default_rng(3)
    B = rng.uniform(-1, 1, (3, s.n))
    # b-hat per oracle conventions, then the launch lists in place
    Y = np.empty((s.n, 3))
    for j in range(3):
        Y[:, j] = _bhat(an, fac, B[j])
    hits = pt.solve_cpu(s, fac.values, part, Y)
    # every stored entry applied exactly once (L entries + U entries + each pivot)
    want = np.zeros(len(fac.values), np.int64)
    for u in range(s.nnodes):
        W = int(s.colptr[u + 1] - s.colptr[u])
        for t in range(int(s.node_first[u + 1] - s.node_first[u])):
            want[s.valoff[u] + t * W: s.valoff[u] + (t + 1) * W] = 1
    assert np.array_equal(hits, want)
    for j in range(3):
        x = np.empty(s.n)
        x[an.ordering.perm] = an.pivot_scale.dc[an.ordering.perm] * Y[:, j]
        xo = on.substitute(an, fac, B[j])
        assert np.abs(x - xo).max() <= 1e-12 * max(1.0, np.abs(xo).max())


def _bhat(an, fac, b):
    s = an.symbolic
    y = np.empty(s.n)
    for u in range(s.nnodes):
        r = int(s.node_first[u])
        for t in range(int(s.node_first[u + 1]) - r):
            src = r + int(fac.inner_perm[r + t]) if s.node_kind[u] == 1 else r + t
            a = int(an.vmap.mrow_src[src])
            y[r + t] = an.pivot_scale.dr[a] * b[a]
    return y
