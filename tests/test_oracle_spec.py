"""Pin the CPU oracle (oracle/numeric.py) and the shared host symbolic against every
known-answer example of the reference SPEC for this path, plus the SPEC's dense
property oracles.  CPU only."""
import numpy as np
import pytest

from paper_2509_07690_b200 import analysis as an_mod
from paper_2509_07690_b200 import generators as gen
from paper_2509_07690_b200 import preprocess as pp
from paper_2509_07690_b200._ref import KernelMode, SolverConfig, SparseMatrixCSR, errors
from paper_2509_07690_b200._ref import matrix as refmatrix
from paper_2509_07690_b200.symbolic import select_kernel, symbolic_from_pattern
from oracle import dense as od
from oracle import numeric as on


def _analyze(A, ordering="natural", mode=None, cfg=None):
    cfg = cfg or SolverConfig(ordering=ordering)
    return an_mod.analyze(A, cfg, kernel_override=mode)


def _csr(dense):
    return SparseMatrixCSR.from_dense(np.asarray(dense, float))


# ---------------------------------------------------------------- pivot_perturb
@pytest.mark.parametrize("p,expect,fired", [(0.0, 1e-8, True), (-1e-12, -1e-8, True), (0.5, 0.5, False)])
def test_pivot_perturb_examples(p, expect, fired):
    v, f = on._perturb.py_func(p, 1e-8 * 1.0)
    assert v == expect and f == fired


# ---------------------------------------------------------------- select_kernel
def test_select_kernel_examples():
    assert select_kernel(1e6, 100, 0.0) == KernelMode.ROWROW
    assert select_kernel(100 * 1000, 1000, 0.8) == KernelMode.SUPSUP
    assert select_kernel(20 * 1000, 1000, 0.5) == KernelMode.SUPROW
    assert select_kernel(20 * 1000, 1000, 0.5, override="rowrow") == KernelMode.ROWROW


# ---------------------------------------------------------------- symbolic
def _sym_dense(mask):
    mask = np.asarray(mask, bool)
    n = mask.shape[0]
    mp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    mc = np.concatenate([np.flatnonzero(mask[i]) for i in range(n)]).astype(np.int64)
    return symbolic_from_pattern(n, mp, mc)


def test_symbolic_tridiagonal_n5():
    m = np.eye(5, dtype=bool) | np.eye(5, k=1, dtype=bool) | np.eye(5, k=-1, dtype=bool)
    s = _sym_dense(m)
    assert s.exact_l_nnz == 4 and s.exact_u_nnz == 9 and s.fill_nnz == 13


def test_symbolic_arrow_hub_first_full_fill():
    m = np.eye(4, dtype=bool)
    m[0, :] = True
    m[:, 0] = True
    assert _sym_dense(m).fill_nnz == 16


def test_symbolic_dense3_flops():
    assert _sym_dense(np.ones((3, 3), bool)).flops == 13


def test_supernodes_examples():
    s = _sym_dense(np.ones((4, 4), bool))
    assert s.nnodes == 1 and s.node_kind[0] == 1 and s.node_rows[0] == 4
    s = _sym_dense(np.eye(6, dtype=bool))
    assert s.supernode_count == 0 and s.nnodes == 6
    m = np.zeros((6, 6), bool)
    m[:3, :3] = True
    m[3:, 3:] = True
    s = _sym_dense(m)
    assert s.supernode_count == 2 and list(s.node_rows) == [3, 3]


def test_task_graph_and_levels_examples():
    # L entries {(1,0),(2,0),(3,1),(3,2)} -> deps 1<-{0}, 2<-{0}, 3<-{1,2}; levels [[0],[1,2],[3]]
    m = np.eye(4, dtype=bool)
    for i, j in [(1, 0), (2, 0), (3, 1), (3, 2)]:
        m[i, j] = True
    cfg = SolverConfig(min_supernode_rows=5)   # keep all rows standalone
    n = 4
    mp = np.concatenate([[0], np.cumsum(m.sum(1))]).astype(np.int64)
    mc = np.concatenate([np.flatnonzero(m[i]) for i in range(n)]).astype(np.int64)
    s = symbolic_from_pattern(n, mp, mc, cfg)
    assert [list(s.node_deps(u)) for u in range(4)] == [[], [0], [0], [1, 2]]
    assert s.levels == [[0], [1, 2], [3]]


def test_levels_diagonal_and_chain():
    s = _sym_dense(np.eye(5, dtype=bool))
    assert s.levels == [[0, 1, 2, 3, 4]]
    m = np.eye(5, dtype=bool) | np.eye(5, k=-1, dtype=bool)
    s = symbolic_from_pattern(5, *[np.asarray(x, np.int64) for x in (
        np.concatenate([[0], np.cumsum(m.sum(1))]),
        np.concatenate([np.flatnonzero(m[i]) for i in range(5)]))],
        SolverConfig(min_supernode_rows=9))
    assert len(s.levels) == 5 and s.bulk_level_cutoff == 0


@pytest.mark.parametrize("seed", range(40))
def test_symbolic_matches_dense_symbolic_oracle(seed):
    """SPEC.md:228 / acceptance 6: pattern = no-cancellation dense elimination, n <= 32."""
    rng = np.random.default_rng(seed)
    n = int(rng.integers(2, 33))
    mask = rng.random((n, n)) < rng.uniform(0.05, 0.4)
    np.fill_diagonal(mask, True)
    L, U = od.dense_symbolic(mask)
    for method in ("general",) + (("symmetric",) if np.array_equal(mask, mask.T) else ()):
        s = symbolic_from_pattern(n, np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64),
                                  np.concatenate([np.flatnonzero(mask[i]) for i in range(n)]).astype(np.int64),
                                  method=method)
        assert s.exact_l_nnz == int(L.sum()) and s.exact_u_nnz == int(U.sum())
        assert s.flops == od.dense_flops(L, U)
        for i in range(n):
            lc, uc = s.row_patterns(i)
            assert set(np.flatnonzero(U[i])) <= set(uc.tolist()) | set(lc.tolist())


@pytest.mark.parametrize("seed", range(10))
def test_symmetric_and_general_symbolic_agree(seed):
    rng = np.random.default_rng(100 + seed)
    n = int(rng.integers(5, 60))
    mask = rng.random((n, n)) < 0.1
    mask = mask | mask.T
    np.fill_diagonal(mask, True)
    mp = np.concatenate([[0], np.cumsum(mask.sum(1))]).astype(np.int64)
    mc = np.concatenate([np.flatnonzero(mask[i]) for i in range(n)]).astype(np.int64)
    a = symbolic_from_pattern(n, mp, mc, method="general")
    b = symbolic_from_pattern(n, mp, mc, method="symmetric")
    assert np.array_equal(a.cols, b.cols) and np.array_equal(a.node_first, b.node_first)
    assert a.flops == b.flops and a.fill_nnz == b.fill_nnz


def test_zero_diagonal_raises():
    m = np.array([[1, 1], [1, 0]], bool)
    with pytest.raises(errors.ZeroDiagonal):
        _sym_dense(m)


# ---------------------------------------------------------------- factorize
def test_factorize_identity():
    A = SparseMatrixCSR.identity(4)
    an = _analyze(A)
    f = on.factorize(an)
    assert np.allclose(f.values, 1.0) and not f.perturbed


def test_factorize_2x2_reconstruction():
    A = _csr([[4.0, 3.0], [6.0, 3.0]])
    an = _analyze(A)
    f = on.factorize(an)
    L, U, src = od.factors_dense(an, f.values, f.inner_perm)
    M = od.m_dense(an)
    assert np.allclose(L @ U, M[src], atol=1e-15)


def test_factorize_2x2_literal_without_scaling():
    """[[4,3],[6,3]] natural order, no scaling -> L(1,0)=1.5, U = {4, 3, -1.5}."""
    A = _csr([[4.0, 3.0], [6.0, 3.0]])
    an = _analyze(A, cfg=SolverConfig(ordering="natural", min_supernode_rows=3))
    an.vmap.scale[:] = 1.0
    an.vmap.mrow_src[:] = np.arange(2)
    an.ordering.perm[:] = np.arange(2)
    f = on.factorize(an)
    L, U, _ = od.factors_dense(an, f.values, f.inner_perm)
    assert L[1, 0] == 1.5 and U[0, 0] == 4 and U[0, 1] == 3 and U[1, 1] == -1.5


def test_factorize_swap_matrix_no_perturbation():
    A = _csr([[0.0, 1.0], [1.0, 0.0]])
    an = _analyze(A)
    assert list(an.pivot_scale.row_perm) == [1, 0]
    f = on.factorize(an)
    assert not f.perturbed


# ---------------------------------------------------------------- update primitives
def test_rowrow_zero_multiplier_keeps_workspace():
    F = np.array([0.0, 5.0, 7.0, 2.0, 3.0])
    pos_of = np.full(10, -1, np.int64)
    pos_of[[1, 2, 3]] = [0, 1, 2]
    cols = np.array([1, 2, 3], np.int64)
    # target row at F[0:3] = [0(L at col1), 5, 7]; source row j=1 stored at F[3:5] ([2, 3] diag first)
    F2 = F.copy()
    on._rowrow.py_func(F2, 0, pos_of, 1, F2, 3, 0, 2, np.array([1, 2], np.int64), 0)
    assert F2[0] == 0.0 and np.array_equal(F2[1:], F[1:])


def test_internal_factorize_swap_cases():
    """Block [[0,1],[1,0]] -> step 0 swaps; diag(3,5) -> identity.
    Both blocks keep their explicit zeros, so the 2x2 pattern is full
    and the two rows form one supernode on which internal_factorize runs."""
    for blk, expect in (([[0.0, 1.0], [1.0, 0.0]], [1, 0]), ([[3.0, 0.0], [0.0, 5.0]], [0, 1])):
        A = SparseMatrixCSR.from_dense(np.array(blk), keep_zeros=True)
        an = _analyze(A, mode=None)
        an.vmap.scale[:] = 1.0
        an.vmap.mrow_src[:] = np.arange(2)
        an.ordering.perm[:] = np.arange(2)
        s = an.symbolic
        assert s.supernode_count == 1 and s.node_kind[0] == 1
        f = on.factorize(an)
        assert list(f.inner_perm) == expect
        assert not f.perturbed
        L, U, src = od.factors_dense(an, f.values, f.inner_perm)
        assert np.array_equal(L @ U, np.array(blk)[src])


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_cross_mode_agreement(mode):
    """Acceptance 3: factors under ROWROW/SUPROW/SUPSUP agree within 1e-12."""
    p = gen.lap2d(10)
    base = on.factorize(_analyze(p.A, "amd", 0))
    f = on.factorize(_analyze(p.A, "amd", mode))
    assert np.abs(f.values - base.values).max() <= 1e-12 * max(1, np.abs(base.values).max())


# ---------------------------------------------------------------- refactorize
def test_refactorize_bitwise_on_unchanged_values():
    p = gen.lap2d(12)
    an = _analyze(p.A, "amd")
    f0 = on.factorize(an)
    f1 = on.factorize(an, prior=f0)
    assert np.array_equal(f0.values, f1.values)


def test_refactorize_scaled_values_halves_solution():
    p = gen.lap2d(12)
    an = _analyze(p.A, "amd")
    f0 = on.factorize(an)
    x0, _ = on.solve(an, f0, p.b)
    A2 = p.A.with_values(2 * p.A.values)
    f2 = on.factorize(an, A2.values, prior=f0)
    x2, _ = on.solve(an, f2, p.b, A=A2)
    assert np.allclose(x2, x0 / 2, rtol=1e-14, atol=0)


def test_refactorize_zero_pivot_triggers_perturbation_and_refinement():
    A = _csr([[2.0, 1.0, 0.0], [1.0, 2.0, 1.0], [0.0, 1.0, 2.0]])
    an = _analyze(A)
    f0 = on.factorize(an)
    v = A.values.copy()
    v[0] = 0.5                        # makes the first pivot tiny after elimination below
    A2 = A.with_values(v)
    vals = A.values.copy()
    vals[0] = 1e-30
    A3 = A.with_values(vals)
    f3 = on.factorize(an, A3.values, prior=f0)
    assert f3.perturbed
    b = np.array([1.0, 2.0, 3.0])
    x, rep = on.solve(an, f3, b, A=A3)
    assert rep["iterations"] >= 1
    assert refmatrix.backward_error(A3, x, b) <= 1e-13
    del A2


# ---------------------------------------------------------------- solve
def test_solve_examples():
    A = SparseMatrixCSR.identity(3)
    an = _analyze(A)
    x, rep = on.solve(an, on.factorize(an), np.array([1.0, 2.0, 3.0]))
    assert np.array_equal(x, [1, 2, 3]) and rep["iterations"] == 0
    A = _csr([[2.0, 0.0], [0.0, 4.0]])
    an = _analyze(A)
    x, _ = on.solve(an, on.factorize(an), np.array([2.0, 4.0]))
    assert np.allclose(x, [1, 1])


@pytest.mark.parametrize("seed", range(60))
def test_oracle_equivalence_random(seed):
    """Acceptance 1/2: dense-oracle solve <= 1e-8 and reconstruction <= 64·eps·n·max|M|."""
    rng = np.random.default_rng(1000 + seed)
    n = int(rng.integers(2, 65))
    dens = rng.uniform(0.05, 1.0)
    D = np.where(rng.random((n, n)) < dens, rng.standard_normal((n, n)), 0.0)
    D[np.arange(n), rng.permutation(n)] += rng.uniform(1, 2, n) * rng.choice([-1, 1], n)
    if np.linalg.cond(D) > 1e8:
        pytest.skip("ill-conditioned sample")
    A = _csr(D)
    an = _analyze(A, "amd")
    f = on.factorize(an)
    b = rng.uniform(-1, 1, n)
    x, _ = on.solve(an, f, b)
    xd = np.linalg.solve(D, b)
    assert np.abs(x - xd).max() <= 1e-8 * max(1.0, np.abs(xd).max())
    if not f.perturbed:
        L, U, src = od.factors_dense(an, f.values, f.inner_perm)
        M = od.m_dense(an)
        assert np.abs(L @ U - M[src]).max() <= 64 * np.finfo(float).eps * n * np.abs(M).max()


def test_inner_perm_selects_block_maximum():
    """step t picks an in-block maximum, |block[p_t][t]| >= |block[r][t]|
    for r in t..s-1.  In the final factors that is: every in-block multiplier
    L(r, t) = block[r][t] / block[p_t][t] (r > t, same supernode) has |.| <= 1, and
    a non-trivial inner_perm occurs (the recipe is not diagonally dominant)."""
    p = gen.fem27(3, recipe="literal")
    an = _analyze(p.A, "amd", 2)
    f = on.factorize(an)
    s = an.symbolic
    assert s.supernode_count > 0
    assert not f.perturbed
    L, U, src = od.factors_dense(an, f.values, f.inner_perm)
    M = od.m_dense(an)
    assert np.abs(L @ U - M[src]).max() <= 1e-12 * np.abs(M).max()
    worst, checked, swapped = 0.0, 0, 0
    for u in range(s.nnodes):
        if s.node_kind[u] != 1:
            continue
        r, e = int(s.node_first[u]), int(s.node_first[u + 1])
        blk = L[r:e, r:e]
        worst = max(worst, float(np.abs(np.tril(blk, -1)).max()))
        checked += 1
        swapped += int(np.any(f.inner_perm[r:e] != np.arange(e - r)))
    assert checked > 0 and swapped > 0
    assert worst <= 1.0
def test_tridiagonal_1e5_zero_fill_rowrow_fast():
    """Acceptance 6 (host part): tridiagonal n=100000 → zero fill, ROWROW, oracle solve."""
    import time
    p = gen.tridiag(100000)
    t0 = time.perf_counter()
    an = _analyze(p.A, "amd")
    s = an.symbolic
    assert s.fill_nnz == p.A.nnz and s.kernel_mode == KernelMode.ROWROW
    f = on.factorize(an)
    x, _ = on.solve(an, f, p.b)
    assert refmatrix.backward_error(p.A, x, p.b) <= 1e-12
    assert time.perf_counter() - t0 < 60


def test_laplacian_250_supernodal():
    """Acceptance 7 (selection part): 250^2 5-point Laplacian picks a supernodal mode."""
    p = gen.lap2d(250)
    an = _analyze(p.A, "amd")
    assert an.symbolic.kernel_mode in (KernelMode.SUPROW, KernelMode.SUPSUP)


def test_static_pivot_examples():
    ps = pp.static_pivot(_csr([[0.0, 3.0], [2.0, 0.0]]))
    assert list(ps.row_perm) == [1, 0]
    ps = pp.static_pivot(_csr([[2.0, 0.0], [0.0, 0.5]]))
    assert list(ps.row_perm) == [0, 1]
