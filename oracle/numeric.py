"""CPU restatement of SPEC's numeric module and triangular solve
 — TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Executor: sequential in pivot (node) order — the ``threads=1`` instance of
``run_pipeline`` ("single worker → equivalent to sequential
processing in pivot order").  Storage: the node layout of
``paper_2509_07690_b200.symbolic`` (shared with the device).

Interpretive choices, identical on the device:

1. sup-row / sup-sup triangular solve uses the source's *upper, non-unit*
   diagonal block, x = w_b·U_bb⁻¹ (forced by SPEC.md:303's equivalence clause),
   evaluated in axpy order (t ascending), then the panel GEMV
   w[c] -= Σ_t x_t·U(t,c) with t ascending.  ``update_sup_by_sup``
    is the blocked form of the same loop nest, so on a supernode
   target SUPROW and SUPSUP give identical arithmetic here.
2. Dispatch: ``kernel_mode`` is the maximum tier.  A standalone
   source always uses row-row; a supernode source uses row-row over its rows in
   ROWROW mode and the sup-row/sup-sup block update otherwise.  Supernodes and
   ``internal_factorize`` exist in every mode.
3. Every pivot (standalone rows included) passes through ``pivot_perturb``;
   the perturbation log records (factor row index, original pivot).
4. ``anorm`` = max|M| of the values being factorized; refactorize
   reuses the prior factors' anorm together with the rest of the prior
   artifacts ("reuses PivotScale ... Ordering ... inner_perm").
5. Internal LU: step t takes the first row with the maximum |·| in
   column t over rows t..s-1 of the block (ties → lowest index), swaps whole
   stored rows (L union included), perturbs, then eliminates right-looking; per
   entry this is the same operation sequence as up-looking, so refactorize with
   the prior ``inner_perm`` pre-applied at scatter time is bitwise identical to
   factorize on unchanged values (acceptance 8).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numba import njit, prange

STANDALONE_ROW = 0
SUPERNODE = 1
ROWROW, SUPROW, SUPSUP = 0, 1, 2


@njit(cache=True, inline="always")
def _perturb(p, thr):
    """pivot_perturb: |p| < eps·anorm → sign(p)·eps·anorm (sign(0)=+)."""
    if abs(p) < thr:
        if p < 0.0:
            return -thr, True
        return thr, True
    return p, False


@njit(cache=True, inline="always")
def _rowrow(F, R, pos_of, j, F_src, sbase, sdiag, sW, scols, sc0):
    """update_row_by_row: target row at F[R:], source row j whose
    stored values are F_src[sbase : sbase+sW] with its diagonal at position sdiag."""
    pj = R + pos_of[j]
    l = F[pj] / F_src[sbase + sdiag]
    F[pj] = l
    if l != 0.0:
        for q in range(sdiag + 1, sW):
            F[R + pos_of[scols[sc0 + q]]] -= l * F_src[sbase + q]


@njit(cache=True)
def _suprow(F, R, pos_of, vfirst, vs, vbase, vW, vnl, cols, vc0, x):
    """update_row_by_sup for one target row at F[R:]."""
    for t in range(vs):
        p = pos_of[vfirst + t]
        x[t] = F[R + p] if p >= 0 else 0.0
    for t in range(vs):                      # x = w_b · U_bb^-1, axpy order
        rowt = vbase + t * vW + vnl
        xt = x[t] / F[rowt + t]
        x[t] = xt
        if xt != 0.0:
            for t2 in range(t + 1, vs):
                x[t2] -= xt * F[rowt + t2]
    for t in range(vs):
        p = pos_of[vfirst + t]
        if p >= 0:
            F[R + p] = x[t]
    for q in range(vnl + vs, vW):           # GEMV over the source's U panel
        acc = 0.0
        for t in range(vs):
            acc += x[t] * F[vbase + t * vW + q]
        F[R + pos_of[cols[vc0 + q]]] -= acc


@njit(cache=True)
def factorize_kernel(n, first, kind, colptr, cols, nl, valoff, dptr, deps, node_of, mode,
                     a_ptr, a_val, mrow_src, colpos, scale, F, iperm, refactor, thr):
    """factorize / refactorize over all nodes in pivot order.

    Returns (perturbed rows, original pivots, breakdown row or -1)."""
    nn = len(kind)
    pos_of = np.full(n, -1, np.int64)
    smax = 1
    for u in range(nn):
        smax = max(smax, first[u + 1] - first[u])
    x = np.empty(smax)
    inv = np.empty(smax, np.int64)
    prow_l = []
    pval_l = []
    breakdown = -1
    for u in range(nn):
        r = first[u]
        s = first[u + 1] - r
        c0 = colptr[u]
        W = colptr[u + 1] - c0
        L = nl[u]
        base = valoff[u]
        issn = kind[u] == SUPERNODE
        # ---- scatter M rows (inner_perm pre-applied on refactorize)
        F[base:base + s * W] = 0.0
        for t in range(s):
            inv[t] = t
        if issn:
            if refactor:
                for p in range(s):
                    inv[iperm[r + p]] = p
            else:
                for p in range(s):
                    iperm[r + p] = p
        for t in range(s):
            a = mrow_src[r + t]
            R = base + inv[t] * W
            for e in range(a_ptr[a], a_ptr[a + 1]):
                F[R + colpos[e]] = a_val[e] * scale[e]
        for q in range(W):
            pos_of[cols[c0 + q]] = q
        # ---- external updates, sources ascending
        for di in range(dptr[u], dptr[u + 1]):
            v = deps[di]
            vfirst = first[v]
            vs = first[v + 1] - vfirst
            vc0 = colptr[v]
            vW = colptr[v + 1] - vc0
            vnl = nl[v]
            vbase = valoff[v]
            if kind[v] == STANDALONE_ROW or mode == ROWROW:
                for tj in range(vs):
                    j = vfirst + tj
                    if pos_of[j] < 0:
                        continue
                    for t in range(s):
                        _rowrow(F, base + t * W, pos_of, j, F, vbase + tj * vW, vnl + tj, vW,
                                cols, vc0)
            else:
                for t in range(s):
                    _suprow(F, base + t * W, pos_of, vfirst, vs, vbase, vW, vnl, cols, vc0, x)
        # ---- pivots
        if not issn:
            piv = F[base + L]
            newp, fired = _perturb(piv, thr)
            if fired:
                prow_l.append(r)
                pval_l.append(piv)
            if thr == 0.0 and piv == 0.0 and breakdown < 0:
                breakdown = r
            F[base + L] = newp
        else:
            # internal_factorize: LU of the s x (s + panel) part,
            # row pivoting restricted to the diagonal block
            for t in range(s):
                Rt = base + t * W
                if not refactor:
                    p = t
                    best = abs(F[Rt + L + t])
                    for q in range(t + 1, s):
                        vq = abs(F[base + q * W + L + t])
                        if vq > best:
                            best = vq
                            p = q
                    if p != t:
                        Rp = base + p * W
                        for c in range(W):
                            tmp = F[Rt + c]
                            F[Rt + c] = F[Rp + c]
                            F[Rp + c] = tmp
                        tmpi = iperm[r + t]
                        iperm[r + t] = iperm[r + p]
                        iperm[r + p] = tmpi
                piv = F[Rt + L + t]
                newp, fired = _perturb(piv, thr)
                if fired:
                    prow_l.append(r + t)
                    pval_l.append(piv)
                if thr == 0.0 and piv == 0.0 and breakdown < 0:
                    breakdown = r + t
                F[Rt + L + t] = newp
                for q in range(t + 1, s):
                    Rq = base + q * W
                    l = F[Rq + L + t] / newp
                    F[Rq + L + t] = l
                    if l != 0.0:
                        for c in range(L + t + 1, W):
                            F[Rq + c] -= l * F[Rt + c]
        for q in range(W):
            pos_of[cols[c0 + q]] = -1
    prow = np.empty(len(prow_l), np.int64)
    pval = np.empty(len(pval_l))
    for k in range(len(prow_l)):
        prow[k] = prow_l[k]
        pval[k] = pval_l[k]
    return prow, pval, breakdown


@njit(cache=True, inline="always")
def _internal_lu(F, iperm, r, s, W, L, base, refactor, thr, pflag, pval, bdflag):
    """internal_factorize of one supernode, as in factorize_kernel."""
    for t in range(s):
        Rt = base + t * W
        if not refactor:
            p = t
            best = abs(F[Rt + L + t])
            for q in range(t + 1, s):
                vq = abs(F[base + q * W + L + t])
                if vq > best:
                    best = vq
                    p = q
            if p != t:
                Rp = base + p * W
                for c in range(W):
                    tmp = F[Rt + c]
                    F[Rt + c] = F[Rp + c]
                    F[Rp + c] = tmp
                tmpi = iperm[r + t]
                iperm[r + t] = iperm[r + p]
                iperm[r + p] = tmpi
        piv = F[Rt + L + t]
        newp, fired = _perturb(piv, thr)
        if fired:
            pflag[r + t] = 1
            pval[r + t] = piv
        if thr == 0.0 and piv == 0.0:
            bdflag[r + t] = 1
        F[Rt + L + t] = newp
        for q in range(t + 1, s):
            Rq = base + q * W
            l = F[Rq + L + t] / newp
            F[Rq + L + t] = l
            if l != 0.0:
                for c in range(L + t + 1, W):
                    F[Rq + c] -= l * F[Rt + c]


@njit(cache=True, parallel=True)
def factorize_levels_kernel(n, first, kind, colptr, cols, nl, valoff, dptr, deps, node_of, mode,
                            a_ptr, a_val, mrow_src, colpos, scale, F, iperm, refactor, thr,
                            level_ptr, level_nodes, nthreads, pflag, pval, bdflag):
    """The same computation as ``factorize_kernel`` executed level by level
    (SPEC.md:397-405 ``run_bulk``: the nodes of a level depend only on earlier
    levels).  Phase 1 runs one task per (node, row) on ``nthreads`` threads: scatter
    of the row's M values, then every dependency update of that row in ascending
    source order — per row exactly the operation sequence of the sequential loop
    (row-row and sup-row updates of a target row read only final source rows and
    write only that row).  Phase 2 runs the pivots / internal LU per node.  The
    result is therefore bitwise identical to the sequential executor (tested).
    Perturbations and breakdowns are flagged per factor row."""
    smax = 1
    for u in range(len(kind)):
        smax = max(smax, first[u + 1] - first[u])
    pos_all = np.full((nthreads, n), -1, np.int64)
    x_all = np.empty((nthreads, smax))
    cur_all = np.full(nthreads, -1, np.int64)
    nlev = len(level_ptr) - 1
    for lev in range(nlev):
        l0 = level_ptr[lev]
        l1 = level_ptr[lev + 1]
        cnt = l1 - l0
        rp = np.empty(cnt + 1, np.int64)
        rp[0] = 0
        for k in range(cnt):
            u = level_nodes[l0 + k]
            rp[k + 1] = rp[k] + first[u + 1] - first[u]
        nitems = rp[cnt]
        for T in prange(nthreads):
            pos_of = pos_all[T]
            x = x_all[T]
            k = 0
            for it in range(T, nitems, nthreads):
                while rp[k + 1] <= it:
                    k += 1
                u = level_nodes[l0 + k]
                prow = it - rp[k]
                r = first[u]
                c0 = colptr[u]
                W = colptr[u + 1] - c0
                base = valoff[u]
                issn = kind[u] == SUPERNODE
                if cur_all[T] != u:
                    if cur_all[T] >= 0:
                        pu = cur_all[T]
                        for q in range(colptr[pu], colptr[pu + 1]):
                            pos_of[cols[q]] = -1
                    for q in range(W):
                        pos_of[cols[c0 + q]] = q
                    cur_all[T] = u
                # scatter: destination row prow receives M row t with inv[t] == prow
                t = prow
                if issn:
                    if refactor:
                        t = iperm[r + prow]
                    else:
                        iperm[r + prow] = prow
                R = base + prow * W
                for c in range(W):
                    F[R + c] = 0.0
                a = mrow_src[r + t]
                for e in range(a_ptr[a], a_ptr[a + 1]):
                    F[R + colpos[e]] = a_val[e] * scale[e]
                for di in range(dptr[u], dptr[u + 1]):
                    v = deps[di]
                    vfirst = first[v]
                    vs = first[v + 1] - vfirst
                    vc0 = colptr[v]
                    vW = colptr[v + 1] - vc0
                    vnl = nl[v]
                    vbase = valoff[v]
                    if kind[v] == STANDALONE_ROW or mode == ROWROW:
                        for tj in range(vs):
                            j = vfirst + tj
                            if pos_of[j] < 0:
                                continue
                            _rowrow(F, R, pos_of, j, F, vbase + tj * vW, vnl + tj, vW, cols, vc0)
                    else:
                        _suprow(F, R, pos_of, vfirst, vs, vbase, vW, vnl, cols, vc0, x)
        for k in prange(cnt):
            u = level_nodes[l0 + k]
            r = first[u]
            s = first[u + 1] - r
            W = colptr[u + 1] - colptr[u]
            L = nl[u]
            base = valoff[u]
            if kind[u] != SUPERNODE:
                piv = F[base + L]
                newp, fired = _perturb(piv, thr)
                if fired:
                    pflag[r] = 1
                    pval[r] = piv
                if thr == 0.0 and piv == 0.0:
                    bdflag[r] = 1
                F[base + L] = newp
            else:
                _internal_lu(F, iperm, r, s, W, L, base, refactor, thr, pflag, pval, bdflag)


@njit(cache=True)
def anorm_kernel(a_val, scale):
    m = 0.0
    for e in range(len(a_val)):
        v = abs(a_val[e] * scale[e])
        if v > m:
            m = v
    return m


@njit(cache=True)
def solve_kernel(n, first, kind, colptr, cols, nl, valoff, F, iperm, mrow_src, dr, dc, perm, b, x):
    """solve without refinement: b̂ = P_inner·P·Dr·b, L y = b̂ (unit L,
    rows ascending), U z = y (rows descending), x = Dc·Q·z."""
    nn = len(kind)
    y = np.empty(n)
    for u in range(nn):
        r = first[u]
        for t in range(first[u + 1] - r):
            src = r + iperm[r + t] if kind[u] == SUPERNODE else r + t
            a = mrow_src[src]
            y[r + t] = dr[a] * b[a]
    for u in range(nn):                                  # forward_substitution
        r = first[u]
        c0 = colptr[u]
        W = colptr[u + 1] - c0
        for t in range(first[u + 1] - r):
            R = valoff[u] + t * W
            acc = y[r + t]
            for p in range(nl[u] + t):
                acc -= F[R + p] * y[cols[c0 + p]]
            y[r + t] = acc
    for u in range(nn - 1, -1, -1):                      # backward_substitution
        r = first[u]
        c0 = colptr[u]
        W = colptr[u + 1] - c0
        for t in range(first[u + 1] - r - 1, -1, -1):
            R = valoff[u] + t * W
            d = nl[u] + t
            acc = y[r + t]
            for p in range(d + 1, W):
                acc -= F[R + p] * y[cols[c0 + p]]
            y[r + t] = acc / F[R + d]
    for k in range(n):
        x[perm[k]] = dc[perm[k]] * y[k]


# --------------------------------------------------------------------------- Python API
@dataclass
class OracleFactors:
    """NumericFactors in node layout."""
    values: np.ndarray           # float64[stored]
    inner_perm: np.ndarray       # int64[n] (block-relative, 0 for standalone rows)
    perturbed: list              # [(factor row, original pivot)]
    anorm: float
    breakdown: int = -1
    extra: dict = field(default_factory=dict)


def _sym_args(an):
    s = an.symbolic
    return (s.n, s.node_first, s.node_kind, s.colptr, s.cols.astype(np.int64), s.nl, s.valoff,
            s.dep_ptr, s.deps.astype(np.int64), s.node_of)


def factorize(an, values=None, eps=1e-8, mode=None, prior=None, threads=1):
    """Oracle factorize (prior=None) or refactorize (prior = OracleFactors).

    ``threads=1``: the sequential executor (pivot order).  ``threads>1``:
    the level-parallel executor ``factorize_levels_kernel`` on that many threads —
    bitwise the same factors (tests/test_oracle_spec.py::test_parallel_oracle_is_bitwise_sequential)."""
    if threads and threads > 1:
        return _factorize_par(an, values, eps, mode, prior, int(threads))
    s = an.symbolic
    vals = np.ascontiguousarray(an.A.values if values is None else values, np.float64)
    vm = an.vmap
    F = np.empty(s.stored_values)
    if prior is None:
        iperm = np.zeros(s.n, np.int64)
        anorm = anorm_kernel(vals, vm.scale)
    else:
        iperm = prior.inner_perm.copy()
        anorm = prior.anorm
    m = int(s.kernel_mode if mode is None else mode)
    prow, pval, bd = factorize_kernel(*_sym_args(an), m, an.A.row_ptr, vals, vm.mrow_src,
                                      vm.colpos.astype(np.int64), vm.scale, F, iperm,
                                      prior is not None, eps * anorm)
    return OracleFactors(F, iperm, list(zip(prow.tolist(), pval.tolist())), anorm, bd)


def _factorize_par(an, values, eps, mode, prior, threads):
    import numba
    s = an.symbolic
    vals = np.ascontiguousarray(an.A.values if values is None else values, np.float64)
    vm = an.vmap
    F = np.empty(s.stored_values)
    if prior is None:
        iperm = np.zeros(s.n, np.int64)
        anorm = anorm_kernel(vals, vm.scale)
    else:
        iperm = prior.inner_perm.copy()
        anorm = prior.anorm
    m = int(s.kernel_mode if mode is None else mode)
    pflag = np.zeros(s.n, np.int8)
    pval = np.zeros(s.n)
    bdflag = np.zeros(s.n, np.int8)
    old = numba.get_num_threads()
    numba.set_num_threads(min(threads, numba.config.NUMBA_NUM_THREADS))
    try:
        factorize_levels_kernel(*_sym_args(an), m, an.A.row_ptr, vals, vm.mrow_src,
                                vm.colpos.astype(np.int64), vm.scale, F, iperm, prior is not None,
                                eps * anorm, s.level_ptr.astype(np.int64),
                                s.level_nodes.astype(np.int64), numba.get_num_threads(), pflag, pval,
                                bdflag)
    finally:
        numba.set_num_threads(old)
    rows = np.flatnonzero(pflag)
    bd = np.flatnonzero(bdflag)
    return OracleFactors(F, iperm, list(zip(rows.tolist(), pval[rows].tolist())), anorm,
                         int(bd[0]) if len(bd) else -1)


def substitute(an, fac, b):
    s = an.symbolic
    x = np.empty(s.n)
    solve_kernel(s.n, s.node_first, s.node_kind, s.colptr, s.cols.astype(np.int64), s.nl,
                 s.valoff, fac.values, fac.inner_perm, an.vmap.mrow_src, an.pivot_scale.dr,
                 an.pivot_scale.dc, an.ordering.perm, np.ascontiguousarray(b, np.float64), x)
    return x


def solve(an, fac, b, A=None, cfg=None):
    """solve + automatic iterative_refinement when perturbation fired."""
    from paper_2509_07690_b200._ref import matrix as refmatrix, SolverConfig
    cfg = cfg or an.config or SolverConfig()
    A = A or an.A
    x = substitute(an, fac, b)
    report = {"iterations": 0, "backward_errors": [], "converged": True}
    if fac.perturbed:
        x, report = refine(an, fac, A, b, x, cfg)
    return x, report


def refine(an, fac, A, b, x, cfg):
    """iterative_refinement (constants SPEC.md:516 / config.py:52-54)."""
    from paper_2509_07690_b200._ref import matrix as refmatrix
    errs = [refmatrix.backward_error(A, x, b)]
    it = 0
    converged = errs[-1] <= cfg.refine_tolerance
    while not converged and it < cfg.max_refine_iters:
        r = b - refmatrix.spmv(A, x)
        xn = x + substitute(an, fac, r)
        e = refmatrix.backward_error(A, xn, b)
        it += 1
        if e > cfg.refine_stagnation_factor * errs[-1]:
            if e < errs[-1]:
                x = xn
                errs.append(e)
            break
        x = xn
        errs.append(e)
        converged = e <= cfg.refine_tolerance
    return x, {"iterations": it, "backward_errors": errs, "converged": bool(converged)}


@njit(cache=True, parallel=True)
def batch_refactor_solve(n, first, kind, colptr, cols, nl, valoff, dptr, deps, node_of, mode,
                         a_ptr, vals, mrow_src, colpos, scale, iperm0, thr, dr, dc, perm, rhs, X,
                         npert):
    """CPU baseline for c4: refactorize + solve for every instance (instances in parallel)."""
    B = vals.shape[0]
    for b in prange(B):
        F = np.empty(valoff[len(kind)])
        ip = iperm0.copy()
        prow, pval, bd = factorize_kernel(n, first, kind, colptr, cols, nl, valoff, dptr, deps,
                                          node_of, mode, a_ptr, vals[b], mrow_src, colpos, scale,
                                          F, ip, True, thr)
        npert[b] = len(prow)
        solve_kernel(n, first, kind, colptr, cols, nl, valoff, F, ip, mrow_src, dr, dc, perm,
                     rhs[b], X[b])


def refactor_solve_batch(an, prior, values, rhs, mode=None, refine_perturbed=True, cfg=None,
                         reports=None):
    """refactorize + solve per instance.  With
    ``refine_perturbed`` every instance whose perturbation log is non-empty gets the
    automatic iterative_refinement of SPEC.md:492,499-507 (``refine`` on that
    instance's factors and matrix); ``reports`` (a dict) receives them."""
    s = an.symbolic
    B = values.shape[0]
    X = np.empty((B, s.n))
    npert = np.zeros(B, np.int64)
    m = int(s.kernel_mode if mode is None else mode)
    batch_refactor_solve(*_sym_args(an), m, an.A.row_ptr, np.ascontiguousarray(values),
                         an.vmap.mrow_src, an.vmap.colpos.astype(np.int64), an.vmap.scale,
                         prior.inner_perm, 1e-8 * prior.anorm, an.pivot_scale.dr,
                         an.pivot_scale.dc, an.ordering.perm, np.ascontiguousarray(rhs), X, npert)
    if refine_perturbed:
        from paper_2509_07690_b200._ref import SolverConfig
        cfg = cfg or an.config or SolverConfig()
        for b in np.flatnonzero(npert > 0):
            fac = factorize(an, values=values[b], mode=mode, prior=prior)
            Ab = an.A.with_values(np.ascontiguousarray(values[b]))
            X[b], rep = refine(an, fac, Ab, np.ascontiguousarray(rhs[b], np.float64), X[b].copy(), cfg)
            if reports is not None:
                reports[int(b)] = rep
    return X, npert
