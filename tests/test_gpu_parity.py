"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs (SURVEY §8(c) bars: bit-exact symbolic/permutations, L/U within
1e-11 relative, ||Ax-b||/||b|| <= 1e-10)."""
import numpy as np
import pytest

from paper_2509_07690_b200 import generators as gen
from paper_2509_07690_b200 import analysis as an_mod
from paper_2509_07690_b200 import api
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix

pytestmark = pytest.mark.gpu

LU_RTOL = 1e-11
RES_TOL = 1e-10


def _oracle():
    from oracle import numeric
    return numeric


def _rel(a, b):
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def _analysis(name, mode=None):
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering), kernel_override=mode)
    return p, an


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
@pytest.mark.parametrize("mode", [None, 0, 1, 2])
def test_factorize_matches_oracle(name, mode):
    p, an = _analysis(name, mode)
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm), "inner_perm differs"
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    assert len(f.perturbed) == len(ref.perturbed)
    x, rep = api.solve(p.A, f, b=p.b)
    res = np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b)
    assert res <= RES_TOL
    xo, _ = on.solve(an, ref, p.b)
    assert _rel(x, xo) <= 1e-9


@pytest.mark.parametrize("name", ["c0", "c2", "c3"])
@pytest.mark.parametrize("mode", [1, 2])
def test_wide_rows_on_slab_path(name, mode, monkeypatch):
    """Row/slab path in SUP modes with standalone rows routed to the column-slab
    kernel (tiny threshold, tiny slabs)."""
    monkeypatch.setenv("HYLU_WIDE_ROW", "4")
    monkeypatch.setenv("HYLU_PATH", "rows")
    p, an = _analysis(name, mode)
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL
    f2 = api.refactorize(p.A, f)
    assert np.array_equal(f2.host_values(), f.host_values())


@pytest.mark.parametrize("name", ["c0", "c1", "c3"])
def test_refactorize_matches_oracle(name):
    p, an = _analysis(name)
    on = _oracle()
    f0 = api.factorize_analysis(an)
    rng = np.random.default_rng(5)
    v2 = p.A.values * (1.0 + rng.uniform(-0.05, 0.05, p.A.nnz))
    A2 = p.A.with_values(v2)
    ref0 = on.factorize(an)
    ref2 = on.factorize(an, v2, prior=ref0)
    f2 = api.refactorize(A2, f0)
    assert _rel(f2.host_values(), ref2.values) <= LU_RTOL
    # unchanged values -> bitwise identical to factorize (acceptance 8)
    f1 = api.refactorize(p.A, f0)
    assert np.array_equal(f1.host_values(), f0.host_values())


@pytest.mark.parametrize("hub_steps", [384, 6])
def test_batched_matches_oracle(hub_steps):
    bp = gen.circuit_batch(40, 2000, 2, 200)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    on = _oracle()
    prior = api.factorize_analysis(an)
    oprior = on.factorize(an)
    X, npert = api.refactorize_solve_batched(bp.values, prior, bp.rhs, hub_steps=hub_steps)
    Xo, npo = on.refactor_solve_batch(an, oprior, bp.values, bp.rhs)
    assert _rel(X, Xo) <= 1e-9
    assert np.array_equal(npert, npo)
    for b in range(bp.values.shape[0]):
        A = bp.A0.with_values(bp.values[b])
        res = np.linalg.norm(refmatrix.spmv(A, X[b]) - bp.rhs[b]) / np.linalg.norm(bp.rhs[b])
        assert res <= RES_TOL


def test_batched_factor_values_match_oracle():
    bp = gen.circuit_batch(33, 2000, 2, 200)   # a partial last group
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    on = _oracle()
    prior = api.factorize_analysis(an)
    oprior = on.factorize(an)
    br = api.BatchedRefactorizer(prior, hub_steps=20)
    import torch
    dv = torch.from_numpy(bp.values).cuda()
    dr = torch.from_numpy(bp.rhs).cuda()
    br.run(dv, dr)
    for b in (0, 17, 32):
        ref = on.factorize(an, bp.values[b], prior=oprior)
        got = br.factor_values(b).cpu().numpy()
        assert _rel(got, ref.values) <= LU_RTOL


@pytest.mark.parametrize("name", ["c1", "c0", "c3"])
def test_single_path_hub_rows(name, monkeypatch):
    """ROWROW row path with standalone rows above a tiny step threshold routed to the
    single-instance pull kernel (k_hub1)."""
    monkeypatch.setenv("HYLU_HUB_STEPS", "6")
    p, an = _analysis(name, 0)
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    f2 = api.refactorize(p.A, f)
    assert np.array_equal(f2.host_values(), f.host_values())
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL


@pytest.mark.parametrize("name", ["c1", "c0"])
def test_rowrow_on_fanin_path(name, monkeypatch):
    """ROWROW-mode analysis executed by the level fan-in kernels (supernode sources
    applied as blocks: same values up to summation order)."""
    monkeypatch.setenv("HYLU_PATH", "fanin")
    p, an = _analysis(name, 0)
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL


@pytest.mark.parametrize("name", ["c1", "c2", "c0"])
def test_fanin_warp_kernels_and_split_k(name, monkeypatch):
    """Every small multiplier block / small-target update on the warp-per-item
    kernels (threshold forced to 1) and heavy packed items split-K at a low
    threshold: factors still match the oracle."""
    from paper_2509_07690_b200 import schedule
    monkeypatch.setenv("HYLU_OPTIONS", "fanin_warp_min=1")
    monkeypatch.setattr(schedule, "SPLIT_SRC", 2)
    monkeypatch.setattr(schedule, "SPLIT_REL", 1.0)
    p, an = _analysis(name, None)
    plan = schedule.build_fanin_plan(an.symbolic)
    an.symbolic._fanin_plan = plan
    assert len(plan.part_n) > 0
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL


@pytest.mark.parametrize("name", ["c0", "c1", "c3"])
def test_device_backward_error_is_the_references(name):
    """hy_residual reproduces matrix.py's backward_error bit for bit."""
    p, an = _analysis(name, None)
    f = api.factorize_analysis(an)
    x, _ = api.solve(p.A, f, b=p.b)
    rng = np.random.default_rng(7)
    for xx in (x, x * (1 + 1e-9 * rng.standard_normal(x.shape)), np.zeros_like(x)):
        assert api.backward_error(p.A, f, xx, p.b) == refmatrix.backward_error(p.A, xx, p.b)


def _perturbed_case():
    """c0 small refactorized with the M diagonal of a few rows without L entries
    (first pivots of their elimination) set to ~0: the prior pivoting and scaling
    are reused, so those pivots are tiny, perturbation fires and the
    solve refines."""
    p, an = _analysis("c0", None)
    f0 = api.factorize_analysis(an)
    s = an.symbolic
    ps, order = an.pivot_scale, an.ordering
    rows = [int(s.node_first[u]) for u in range(s.nnodes)
            if s.node_kind[u] == 0 and s.nl[u] == 0][:3]
    assert rows
    v = np.array(p.A.values)
    rp, ci = p.A.row_ptr, p.A.col_idx
    for k in rows:
        c = int(order.perm[k])                       # column of M's pivot k
        r = int(ps.row_perm[c])                      # original row matched to it
        d = rp[r] + int(np.flatnonzero(ci[rp[r]:rp[r + 1]] == c)[0])
        v[d] = 1e-300
    A = p.A.with_values(v)
    f = api.refactorize(A, f0)
    return A, f, np.asarray(p.b)


def test_device_refinement_matches_host_loop():
    """The device refinement loop takes the same steps as the
    host formulation with the reference's spmv / backward_error: same iteration
    count, bitwise-equal backward errors and solution."""
    A, f, b = _perturbed_case()
    assert f.perturbed
    x, rep = api.solve(A, f, b=b)
    cfg = SolverConfig()
    xh = api.substitute(f, b).cpu().numpy()
    errs = [refmatrix.backward_error(A, xh, b)]
    it, conv = 0, errs[-1] <= cfg.refine_tolerance
    while not conv and it < cfg.max_refine_iters:
        r = b - refmatrix.spmv(A, xh)
        xn = xh + api.substitute(f, r).cpu().numpy()
        e = refmatrix.backward_error(A, xn, b)
        it += 1
        if e > cfg.refine_stagnation_factor * errs[-1]:
            if e < errs[-1]:
                xh, errs = xn, errs + [e]
            break
        xh, errs = xn, errs + [e]
        conv = e <= cfg.refine_tolerance
    assert rep.iterations == it and rep.converged == conv
    assert rep.backward_errors == errs
    assert np.array_equal(x, xh)
    assert rep.iterations >= 1


@pytest.mark.parametrize("pipelined", [False, True])
def test_batched_host_buffers_match_device_path(pipelined):
    """Public host-buffer call (chunked H2D / compute / D2H): equal to the device
    path, also when consecutive pipelined calls overlap (per-chunk buffer reuse)."""
    import torch
    bp = gen.circuit_batch(100, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    prior = api.factorize_analysis(an)
    br = api.BatchedRefactorizer(prior)
    B = bp.values.shape[0]
    xs_dev = []
    for k in range(3):   # three different inputs: scaled rhs per call
        dv = torch.from_numpy(bp.values).cuda()
        dr = torch.from_numpy(bp.rhs * (k + 1)).cuda()
        x, _ = br.run(dv, dr)
        xs_dev.append(x.cpu().numpy())
    h_vals = torch.from_numpy(bp.values).pin_memory()
    outs = []
    for k in range(3):
        h_rhs = torch.from_numpy(bp.rhs * (k + 1)).pin_memory()
        h_x = torch.empty((B, bp.rhs.shape[1]), dtype=torch.float64).pin_memory()
        br.run_host(h_vals, h_rhs, h_x, chunks=3, pipelined=pipelined)
        outs.append((h_rhs, h_x))
    br.host_wait()
    torch.cuda.synchronize()
    for k in range(3):
        assert np.array_equal(outs[k][1].numpy(), xs_dev[k])


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_full_size_factor_matches_oracle(name):
    """BASELINE configs at their full size (c0 n=4096, c1 n=200000): inner_perm equal,
    L/U within 1e-11, refactorize on unchanged values bitwise equal, residual bound."""
    p = gen.config(name)
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    f2 = api.refactorize(p.A, f)
    assert np.array_equal(f2.host_values(), f.host_values())
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL


def test_batched_full_n_matches_oracle():
    """c4 recipe at its full per-instance size (n = 20000, 3 hubs of 2000 entries) on
    a 40-instance batch (a partial last group): factor values of sampled instances
    within 1e-11 of the oracle's refactorize, solutions within 1e-9, perturbation
    counts equal."""
    import torch
    bp = gen.circuit_batch(40)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    on = _oracle()
    prior = api.factorize_analysis(an)
    oprior = on.factorize(an)
    br = api.BatchedRefactorizer(prior)
    x, npert = br.run(torch.from_numpy(bp.values).cuda(), torch.from_numpy(bp.rhs).cuda())
    Xo, npo = on.refactor_solve_batch(an, oprior, bp.values, bp.rhs)
    assert _rel(x.cpu().numpy(), Xo) <= 1e-9
    assert np.array_equal(npert.cpu().numpy(), npo)
    for b in (0, 33, 39):
        ref = on.factorize(an, bp.values[b], prior=oprior)
        assert _rel(br.factor_values(b).cpu().numpy(), ref.values) <= LU_RTOL


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_update_kernel_variants(name):
    """Sup-sup update kernels: the per-source DMMA kernel (fanin_tc=2) is bitwise equal
    to the FFMA kernel (DMMA chains its four products per element in k order); the
    K-concatenated DMMA kernels (default fanin_tc=5: packed items too; 4: packed items
    on the FFMA packing kernel) differ only by summation order."""
    p, an = _analysis(name)
    on = _oracle()
    ref = on.factorize(an)
    f4 = api.factorize_analysis(an)
    ctx = f4._ctx
    try:
        ctx.set_option("fanin_tc", 0)
        f0 = api.factorize_analysis(an)
        ctx.set_option("fanin_tc", 2)
        f2 = api.factorize_analysis(an)
        ctx.set_option("fanin_tc", 4)
        f4b = api.factorize_analysis(an)
    finally:
        ctx.set_option("fanin_tc", 5)
    v0, v2, v4, v4b = f0.host_values(), f2.host_values(), f4.host_values(), f4b.host_values()
    assert np.array_equal(v2, v0)
    assert _rel(v4, v0) <= 1e-12 and _rel(v4b, v0) <= 1e-12
    assert _rel(v4, ref.values) <= LU_RTOL


def test_api_errors_and_tiny_systems():
    """Error convention (polylu.errors) and degenerate sizes through the device path."""
    from paper_2509_07690_b200._ref import errors, SparseMatrixCSR
    # n = 1
    A1 = SparseMatrixCSR(1, np.array([0, 1]), np.array([0]), np.array([4.0]))
    an1 = an_mod.analyze(A1, SolverConfig(ordering="amd"))
    f1 = api.factorize_analysis(an1)
    x1, _ = api.solve(A1, f1, b=np.array([2.0]))
    assert abs(x1[0] - 0.5) <= 1e-15
    # diagonal matrix: no fill, exact solve
    n = 50
    D = SparseMatrixCSR(n, np.arange(n + 1), np.arange(n), np.arange(1.0, n + 1))
    anD = an_mod.analyze(D, SolverConfig(ordering="amd"))
    fD = api.factorize_analysis(anD)
    xD, _ = api.solve(D, fD, b=np.ones(n))
    assert np.allclose(xD, 1.0 / np.arange(1.0, n + 1), rtol=0, atol=1e-15)
    # refactorize with a different pattern -> PatternMismatch
    p, an = _analysis("c0")
    f = api.factorize_analysis(an)
    A = p.A
    rp, ci, va = np.asarray(A.row_ptr), np.asarray(A.col_idx), np.asarray(A.values)
    drop = next(k for k in range(rp[0], rp[1]) if ci[k] != 0)      # an off-diagonal of row 0
    keep = np.ones(len(ci), bool)
    keep[drop] = False
    rp2 = rp.copy()
    rp2[1:] -= 1
    bad = SparseMatrixCSR(A.n, rp2, ci[keep], va[keep])
    with pytest.raises(errors.PatternMismatch):
        api.refactorize(bad, f)
    # rhs of the wrong length -> DimensionMismatch
    with pytest.raises(errors.DimensionMismatch):
        api.solve(A, f, b=np.ones(A.n + 1))


def test_single_call_batched_abi_matches_two_phase():
    """hy_refactorize_solve_batched (one C call) equals refactorize_batched +
    solve_batched bit for bit, including a batch of one instance."""
    import torch
    from paper_2509_07690_b200.device import check
    bp = gen.circuit_batch(36, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    prior = api.factorize_analysis(an)
    br = api.BatchedRefactorizer(prior)
    ctx = br.ctx
    for B in (36, 1):
        dv = torch.from_numpy(bp.values[:B].copy()).cuda()
        dr = torch.from_numpy(bp.rhs[:B].copy()).cuda()
        x2, n2 = br.run(dv, dr)
        x1 = torch.empty_like(x2)
        n1 = torch.empty_like(n2)
        check(ctx.lib.hy_refactorize_solve_batched(ctx.h, B, dv.data_ptr(), dr.data_ptr(), x1.data_ptr(),
                                                   1e-8, prior._desc, n1.data_ptr(), ctx.stream_handle(None)))
        torch.cuda.synchronize()
        assert torch.equal(x1, x2) and torch.equal(n1, n2)
        A = bp.A0.with_values(bp.values[0])
        xh = x1[0].cpu().numpy()
        assert np.linalg.norm(refmatrix.spmv(A, xh) - bp.rhs[0]) / np.linalg.norm(bp.rhs[0]) <= RES_TOL


def test_c3_literal_recipe_matches_oracle():
    """c3 read literally (every 3x3 block XᵀX + 3I, not diagonally dominant): static
    pivoting moves most rows and the pivoted pattern is unsymmetric; the device
    factors still match the oracle and the solve meets the residual bound."""
    p = gen.fem27(5, recipe="literal")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    assert not np.array_equal(np.asarray(an.pivot_scale.row_perm), np.arange(p.A.n))
    on = _oracle()
    ref = on.factorize(an)
    f = api.factorize_analysis(an)
    assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
    assert _rel(f.host_values(), ref.values) <= LU_RTOL
    x, _ = api.solve(p.A, f, b=p.b)
    assert np.linalg.norm(refmatrix.spmv(p.A, x) - p.b) / np.linalg.norm(p.b) <= RES_TOL


def test_cli_solve_report(tmp_path):
    """SPEC.md cli example: `solve --matrix lap.mtx --repeat K --report out.json` gives a
    SolveReport JSON with K repeat entries and a small final backward error; the
    identity example gives x = b with backward error 0."""
    import json
    from paper_2509_07690_b200 import cli
    p = gen.config("c0", "small")
    mtx = tmp_path / "lap.mtx"
    A = p.A
    rp, ci, va = np.asarray(A.row_ptr), np.asarray(A.col_idx), np.asarray(A.values)
    lines = ["%%MatrixMarket matrix coordinate real general", "%d %d %d" % (A.n, A.n, A.nnz)]
    for i in range(A.n):
        for k in range(rp[i], rp[i + 1]):
            lines.append("%d %d %r" % (i + 1, ci[k] + 1, float(va[k])))
    mtx.write_text("\n".join(lines) + "\n")
    out = tmp_path / "out.json"
    assert cli.main(["--matrix", str(mtx), "--repeat", "3", "--perturb-values", "0.01",
                     "--rhs", "random:3", "--report", str(out)]) == 0
    r = json.loads(out.read_text())
    assert len(r["repeat_times_seconds"]) == 3 and r["n"] == p.A.n
    assert r["backward_error_final"] <= 1e-13
    assert set(r["phase_times_seconds"]) == {"preprocess", "factorize", "solve"}
    eye = tmp_path / "id2.mtx"
    eye.write_text("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2 1.0\n")
    out2 = tmp_path / "id.json"
    assert cli.main(["--matrix", str(eye), "--report", str(out2)]) == 0
    assert json.loads(out2.read_text())["backward_error_final"] == 0.0


def test_device_random_corpus_acceptance():
    """SPEC acceptance 1-3 on the device path: random matrices n in [2, 64], density
    in [0.05, 1] (condition <= 1e8): solve within 1e-8 of a dense solve, factors
    within 1e-11 of the oracle's, and the three kernel modes agree within 1e-12."""
    from paper_2509_07690_b200._ref import SparseMatrixCSR
    on = _oracle()
    done = 0
    for seed in range(40):
        rng = np.random.default_rng(5000 + seed)
        n = int(rng.integers(2, 65))
        dens = rng.uniform(0.05, 1.0)
        D = np.where(rng.random((n, n)) < dens, rng.standard_normal((n, n)), 0.0)
        D[np.arange(n), rng.permutation(n)] += rng.uniform(1, 2, n) * rng.choice([-1, 1], n)
        if np.linalg.cond(D) > 1e8:
            continue
        A = SparseMatrixCSR.from_dense(D)
        b = rng.uniform(-1, 1, n)
        xd = np.linalg.solve(D, b)
        vals = []
        for mode in (0, 1, 2):
            an = an_mod.analyze(A, SolverConfig(ordering="amd"), kernel_override=mode)
            f = api.factorize_analysis(an)
            ref = on.factorize(an)
            assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
            assert _rel(f.host_values(), ref.values) <= LU_RTOL
            x, _ = api.solve(A, f, b=b)
            assert np.abs(x - xd).max() <= 1e-8 * max(1.0, np.abs(xd).max())
            vals.append(f.host_values())
        assert _rel(vals[1], vals[0]) <= 1e-12 and _rel(vals[2], vals[0]) <= 1e-12
        done += 1
    assert done >= 20


def test_device_tridiagonal_and_laplacian_acceptance():
    """SPEC acceptance 6/7 on the device: tridiagonal n = 100000 (zero fill, ROWROW,
    backward error <= 1e-12) and the 250 x 250 5-point Laplacian (supernodal mode,
    backward error <= 1e-12)."""
    from paper_2509_07690_b200._ref import KernelMode
    p = gen.tridiag(100000)
    an = an_mod.analyze(p.A, SolverConfig(ordering="amd"))
    assert an.symbolic.fill_nnz == p.A.nnz and an.symbolic.kernel_mode == KernelMode.ROWROW
    f = api.factorize_analysis(an)
    x, _ = api.solve(p.A, f, b=p.b)
    assert refmatrix.backward_error(p.A, x, p.b) <= 1e-12
    p = gen.lap2d(250)
    an = an_mod.analyze(p.A, SolverConfig(ordering="amd"))
    assert an.symbolic.kernel_mode in (KernelMode.SUPROW, KernelMode.SUPSUP)
    f = api.factorize_analysis(an)
    x, _ = api.solve(p.A, f, b=p.b)
    assert refmatrix.backward_error(p.A, x, p.b) <= 1e-12


def test_zero_pivot_without_perturbation_raises_numeric_breakdown():
    """errors.NumericBreakdown (errors.py:60) only when perturbation is disabled
    (perturbation_epsilon = 0) and a pivot is exactly zero."""
    from paper_2509_07690_b200._ref import errors
    p, an = _analysis("c0", None)
    f0 = api.factorize_analysis(an)
    s = an.symbolic
    ps, order = an.pivot_scale, an.ordering
    k = next(int(s.node_first[u]) for u in range(s.nnodes) if s.node_kind[u] == 0 and s.nl[u] == 0)
    v = np.array(p.A.values)
    rp, ci = p.A.row_ptr, p.A.col_idx
    c = int(order.perm[k])
    r = int(ps.row_perm[c])
    v[rp[r] + int(np.flatnonzero(ci[rp[r]:rp[r + 1]] == c)[0])] = 0.0
    A = p.A.with_values(v)
    with pytest.raises(errors.NumericBreakdown):
        api.refactorize(A, f0, api.FactorOptions(perturbation_epsilon=0.0))
    f = api.refactorize(A, f0)                      # default eps: perturbed, no error
    assert len(f.perturbed) >= 1


def _gpu_shard_worker(rank, world, port, q):
    import os
    import torch
    import torch.distributed as dist
    from paper_2509_07690_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)   # gather only, off the data path
    try:
        total = 96
        bp = gen.circuit_batch(total, 2000, 2, 200)
        an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
        prior = api.factorize_analysis(an)
        br = api.BatchedRefactorizer(prior)
        lo, hi = sharding.shard_range(total, rank, world)
        x, npert = br.run(torch.from_numpy(bp.values[lo:hi]).cuda(), torch.from_numpy(bp.rhs[lo:hi]).cuda())
        X = sharding.gather_shards(x.cpu().numpy(), total, dist)
        NP = sharding.gather_shards(npert.cpu().numpy(), total, dist)
        if rank == 0:
            x1, n1 = br.run(torch.from_numpy(bp.values).cuda(), torch.from_numpy(bp.rhs).cuda())
            q.put((bool(np.array_equal(X, x1.cpu().numpy())), bool(np.array_equal(NP, n1.cpu().numpy()))))
    except Exception as e:          # report instead of hanging the parent
        q.put(("error", repr(e)))
    dist.destroy_process_group()


def test_sharded_batch_two_processes_bitwise():
    """SURVEY §8(e) on one device: two independent processes each refactorize+solve
    their contiguous shard (no collective on the data path; a gloo gather off the
    clock), and the gathered x / perturbation counts equal a one-process run bit for
    bit (per instance the arithmetic does not depend on its group or lane)."""
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_gpu_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(600)
    res = q.get(timeout=5)
    assert res == (True, True), res


def _perturbed_batch():
    bp = gen.circuit_batch(40, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    vals = bp.values.copy()
    for b in (3, 33):                      # one in each group of 32
        gen.zero_first_pivot(an, vals[b])
    return bp, an, vals


def test_batched_refinement_of_perturbed_instances():
    """SPEC.md:492 on the batched path: instances whose pivots were perturbed are
    refined on the device (masked batched residual / substitution / update) and
    match the oracle's refined solutions; the others are untouched."""
    import torch
    bp, an, vals = _perturbed_batch()
    on = _oracle()
    prior = api.factorize_analysis(an)
    oprior = on.factorize(an)
    reps_o = {}
    Xo, npo = on.refactor_solve_batch(an, oprior, vals, bp.rhs, reports=reps_o)
    assert sorted(reps_o) == [3, 33]
    X, npert = api.refactorize_solve_batched(vals, prior, bp.rhs)
    reps = api.refactorize_solve_batched.last_reports
    assert np.array_equal(npert, npo)
    assert sorted(reps) == [3, 33]
    for b in (3, 33):
        assert reps[b].converged and reps[b].iterations >= 1
        assert reps[b].backward_errors[-1] <= 1e-13
        assert abs(reps[b].iterations - reps_o[b]["iterations"]) <= 1
    assert _rel(X, Xo) <= 1e-9
    # without refinement the perturbed instances are far off; the rest identical
    br = api.BatchedRefactorizer(prior)
    dv = torch.from_numpy(vals).cuda()
    dr = torch.from_numpy(bp.rhs).cuda()
    x0, _ = br.run(dv, dr, refine=False)
    x0 = x0.cpu().numpy()
    keep = [b for b in range(len(vals)) if b not in (3, 33)]
    assert np.array_equal(x0[keep], X[keep])
    A3 = bp.A0.with_values(vals[3])
    assert refmatrix.backward_error(A3, x0[3], bp.rhs[3]) > 1e-13


@pytest.mark.parametrize("pipelined", [False, True])
def test_batched_host_buffers_refine_perturbed_instances(pipelined):
    import torch
    bp, an, vals = _perturbed_batch()
    prior = api.factorize_analysis(an)
    X, _ = api.refactorize_solve_batched(vals, prior, bp.rhs)
    br = api.BatchedRefactorizer(prior)
    h_vals = torch.from_numpy(vals).pin_memory()
    h_rhs = torch.from_numpy(bp.rhs).pin_memory()
    h_x = torch.empty(bp.rhs.shape, dtype=torch.float64).pin_memory()
    h_np = torch.empty(len(vals), dtype=torch.int32).pin_memory()
    br.run_host(h_vals, h_rhs, h_x, h_np, chunks=2, pipelined=pipelined)
    br.host_wait()
    torch.cuda.synchronize()
    assert sorted(br.reports) == [3, 33]
    assert _rel(h_x.numpy(), X) <= 1e-12


@pytest.mark.parametrize("name", ["c0", "c2", "c3"])
def test_kernel_override_at_factorize_routes_the_device(name):
    """FactorOptions.kernel_override at factorize time sets the
    device dispatch: ROWROW runs the row-row operation order,
    SUPROW / SUPSUP the block order (bitwise the same on the device, as in the
    oracle); every mode matches the oracle of that mode and the modes agree within
    SPEC's 1e-12."""
    from paper_2509_07690_b200._ref import KernelMode
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    on = _oracle()
    fv = {}
    for m in (2, 0, 1):
        f = api.factorize_analysis(an, opts=api.FactorOptions(kernel_override=m))
        assert int(f.kernel_mode) == m
        ref = on.factorize(an, mode=m)
        assert np.array_equal(f.host_inner_perm(), ref.inner_perm)
        assert _rel(f.host_values(), ref.values) <= LU_RTOL
        r = f.routing()
        assert r["kernel_mode"] == KernelMode(m).name
        assert r["update_order"].startswith("row-row") == (m == 0)
        fv[m] = f.host_values()
        # refactorize keeps the prior's mode: bitwise equal on unchanged values
        f2 = api.refactorize(p.A, f)
        assert int(f2.kernel_mode) == m and np.array_equal(f2.host_values(), fv[m])
    assert np.array_equal(fv[1], fv[2])
    assert an.symbolic.supernode_count > 0
    assert not np.array_equal(fv[0], fv[2]), "ROWROW must run the row-row order"
    assert _rel(fv[0], fv[2]) <= 1e-12
    # the default (no override) is the analysis' mode
    f = api.factorize_analysis(an)
    assert f.kernel_mode == an.symbolic.kernel_mode


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
@pytest.mark.parametrize("nrhs,method", [(1, "partition"), (37, "partition"), (5, "levels")])
def test_solve_multi_matches_oracle(name, nrhs, method):
    """Partition-based multi-RHS substitution (Fig. 3) on the device
    against the oracle's substitution on the same (device) factors, per right-hand
    side, with a forced multi-segment partition."""
    from oracle.numeric import OracleFactors
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    on = _oracle()
    f = api.factorize_analysis(an)
    ctx = f._ctx
    part = ctx.ensure_partition(config=SolverConfig(seg_nnz_threshold=max(500, an.symbolic.stored_values // 12)))
    assert part.seg_rows[-1] == an.symbolic.n and part.nsegments >= 2
    rng = np.random.default_rng(11)
    B = rng.uniform(-1, 1, (nrhs, p.A.n))
    X = api.substitute_multi(f, B, method=method).cpu().numpy()
    fo = OracleFactors(f.host_values(), f.host_inner_perm(), [], f.anorm)
    for j in range(nrhs):
        xo = on.substitute(an, fo, B[j])
        assert _rel(X[j], xo) <= 1e-13
    xs = api.substitute(f, B[0]).cpu().numpy()
    assert _rel(X[0], xs) <= 1e-13
    for j in range(min(nrhs, 3)):
        res = np.linalg.norm(refmatrix.spmv(p.A, X[j]) - B[j]) / np.linalg.norm(B[j])
        assert res <= RES_TOL


def test_solve_multi_small_segments_and_refinement():
    """Many small segments (sequential triangles, balanced rectangular ranges) and the
    automatic refinement of solve_multi on a perturbed factorization."""
    from paper_2509_07690_b200 import partition as pt
    bp = gen.circuit_batch(2, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd", seg_nnz_threshold=500))
    vals = bp.values[1].copy()
    gen.zero_first_pivot(an, vals)
    A1 = bp.A0.with_values(vals)
    f = api.factorize(A1, an.pivot_scale, an.ordering, an.symbolic)
    assert f.perturbed
    part = f._ctx.ensure_partition(config=an.config)
    assert part.nsegments > 4 and part.sequential.any()
    rng = np.random.default_rng(5)
    B = rng.uniform(-1, 1, (4, 1500))
    X, reps = api.solve_multi(A1, f, B)
    for j in range(4):
        assert reps[j].converged
        assert refmatrix.backward_error(A1, X[j], B[j]) <= 1e-13
        xj, _ = api.solve(A1, f, b=B[j])
        assert _rel(X[j], xj) <= 1e-12


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_launch_options_do_not_change_results(name):
    """Launch-level options are scheduling only: factors and solutions are bitwise
    equal with programmatic dependent launch, CUDA graphs, the two-stream phase
    overlap and the thread-per-node kernel for single-row nodes switched off; the batched path likewise for PDL, the pair-workspace
    width and the pipeline's claim order (diagonal / level-major)."""
    import torch
    p, an = _analysis(name)
    f = api.factorize_analysis(an)
    ctx = f._ctx
    b = torch.from_numpy(np.asarray(p.b, np.float64)).cuda()
    x = api.substitute(f, b)
    try:
        for opt in ("pdl", "graphs", "fanin_overlap", "lu1_kernel"):
            ctx.set_option(opt, 0)
            g = api.factorize_analysis(an)
            assert torch.equal(g.values, f.values), opt
            assert torch.equal(api.substitute(g, b), x), opt
            ctx.set_option(opt, 1)
        # refactorize with and without the L-part panel tiles (no-ops there): bitwise equal
        r1 = api.refactorize(p.A, f)
        ctx.set_option("refactor_panels", 0)
        r0 = api.refactorize(p.A, f)
        ctx.set_option("refactor_panels", 1)
        assert torch.equal(r0.values, r1.values) and torch.equal(r1.values, f.values)
    finally:
        for opt in ("pdl", "graphs", "fanin_overlap", "lu1_kernel"):
            ctx.set_option(opt, 1)
    if name == "c1":
        bp = gen.circuit_batch(70, 2000, 2, 200)
        an4 = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
        prior = api.factorize_analysis(an4)
        br = api.BatchedRefactorizer(prior)
        dv = torch.from_numpy(bp.values).cuda()
        dr = torch.from_numpy(bp.rhs).cuda()
        x0, _ = br.run(dv, dr)
        x0 = x0.clone()
        c4 = br.ctx
        try:
            for opt, val in (("pdl", 0), ("pipe_ws", 16), ("pipe_ws", 2), ("pipe_order", 0), ("pipe_order", 4)):
                c4.set_option(opt, val)
                x1, _ = br.run(dv, dr)
                assert torch.equal(x1, x0), (opt, val)
        finally:
            c4.set_option("pdl", 1)
            c4.set_option("pipe_ws", 6)
            c4.set_option("pipe_order", 1)


def test_batched_edge_sizes_match_oracle():
    """Ragged batches: one instance, one short of a group, exactly one group pair, one past
    it — each against the oracle on the same instances; an empty batch and mismatched
    shapes are rejected (ABI: batch size outside [1, 65535])."""
    from paper_2509_07690_b200._ref import errors
    from paper_2509_07690_b200.device import DeviceError
    bp = gen.circuit_batch(65, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    on = _oracle()
    prior = api.factorize_analysis(an)
    oprior = on.factorize(an)
    Xo, npo = on.refactor_solve_batch(an, oprior, bp.values, bp.rhs)
    for B in (1, 31, 64, 65):
        X, npert = api.refactorize_solve_batched(bp.values[:B], prior, bp.rhs[:B])
        assert X.shape == (B, bp.A0.n)
        assert _rel(X, Xo[:B]) <= 1e-9
        assert np.array_equal(npert, npo[:B])
    with pytest.raises(DeviceError):
        api.refactorize_solve_batched(bp.values[:0], prior, bp.rhs[:0])
    with pytest.raises(errors.DimensionMismatch):
        api.refactorize_solve_batched(bp.values[:4], prior, bp.rhs[:3])
    with pytest.raises(errors.DimensionMismatch):
        api.refactorize_solve_batched(bp.values[:4, :-1], prior, bp.rhs[:4])
