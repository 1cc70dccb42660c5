"""Public API mirroring the reference's SPEC entry points (drop-in surface).

| SPEC operation                                     | here                               |
|----------------------------------------------------|------------------------------------|
| static_pivot(A) -> PivotScale        SPEC.md:155   | ``static_pivot`` (reference code)  |
| amd_order(pattern) -> Ordering       SPEC.md:165   | ``amd_order`` (reference code)     |
| symbolic_factorize(A, ps, ord)       SPEC.md:175   | ``symbolic_factorize``             |
| factorize(A, ps, ord, sym, opts)     SPEC.md:280   | ``factorize``  (device)            |
| refactorize(A_new, prior, opts)      SPEC.md:340   | ``refactorize`` (device)           |
| solve(A, factors, ps, ord, b, thr)   SPEC.md:489   | ``solve`` (device substitution +   |
|                                                    |  automatic refinement)|
| (BASELINE config 4, no SPEC name)                  | ``refactorize_solve_batched``      |

``analyze`` (not a reference name) = static_pivot → ordering → symbolic_factorize.
Errors are the reference's own classes (``polylu.errors``).  The device path has
no CPU fallback: without a CUDA device or the built library these raise.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import preprocess as _pp
from ._ref import KernelMode, SolverConfig, errors
from .analysis import Analysis, analyze, value_map
from .symbolic import SymbolicStructure, symbolic_from_pattern

static_pivot = _pp.static_pivot
PivotScale = _pp.PivotScale
Ordering = _pp.Ordering


def amd_order(ap, ai):
    return _pp.amd_order(ap, ai)


def symbolic_factorize(A, ps, order, config=None, kernel_override=None, threads=1):
    """SPEC.md:175-183 (+ detect_supernodes, select_kernel, build_task_graph, levels)."""
    mp, mc, _ = _pp.m_pattern(A, ps, order)
    return symbolic_from_pattern(A.n, mp, mc, config, kernel_override, threads)


@dataclass
class FactorOptions:
    """SPEC.md:273-276.  ``threads`` has no effect on the device (kept for the API);
    ``device`` selects the GPU."""
    kernel_override: object = None
    perturbation_epsilon: float = 1e-8
    threads: int = 1
    pivot_tolerance: object = None
    device: int = 0

    def __post_init__(self):
        if not (0.0 <= self.perturbation_epsilon < 1.0):
            raise ValueError("perturbation_epsilon must lie in [0, 1)")


@dataclass
class RefinementReport:
    """SPEC.md:454-457."""
    iterations: int = 0
    backward_errors: list = field(default_factory=list)
    converged: bool = True


@dataclass
class NumericFactors:
    """SPEC.md:266-271, resident on the device in node layout."""
    symbolic: SymbolicStructure
    values: object            # torch.float64 CUDA tensor [stored]
    inner_perm: object        # torch.int32 CUDA tensor [n]
    anorm: float
    perturbed: list
    _bufs: dict = field(repr=False, default=None)
    _desc: object = field(repr=False, default=None)
    _ctx: object = field(repr=False, default=None)
    kernel_mode: object = None   # the mode (maximum tier) this factorization ran with

    def routing(self):
        """Device dispatch of this factorization: see
        ``schedule.device_routing``."""
        from .schedule import device_routing
        return device_routing(self.symbolic, self.kernel_mode)

    def host_values(self):
        return self.values.cpu().numpy()

    def host_inner_perm(self):
        return self.inner_perm.cpu().numpy().astype(np.int64)

    def l_values(self):
        """Per-row L values aligned with ``symbolic.l_pattern()`` (SPEC layout view)."""
        return [v for v, _ in self._row_views()]

    def u_values(self):
        return [v for _, v in self._row_views()]

    def _row_views(self):
        s = self.symbolic
        F = self.host_values()
        out = []
        for i in range(s.n):
            u = int(s.node_of[i])
            t = i - int(s.node_first[u])
            W = int(s.colptr[u + 1] - s.colptr[u])
            d = int(s.nl[u]) + t
            row = F[s.valoff[u] + t * W: s.valoff[u] + (t + 1) * W]
            out.append((row[:d], row[d:]))
        return out


# --------------------------------------------------------------------------- contexts
def _context(an, device=0):
    ctxs = an.__dict__.setdefault("_device_ctx", {})
    if device not in ctxs:
        from .device import DeviceContext
        ctxs[device] = DeviceContext(an, device)
    return ctxs[device]


def _analysis_for(A, ps, order, sym, config=None):
    an = getattr(sym, "_analysis", None)
    if an is None or an.pivot_scale is not ps or an.ordering is not order:
        vm = value_map(A, ps, order, sym)
        an = Analysis(A, ps, order, sym, vm, config or SolverConfig(), {})
        sym._analysis = an
    return an


def _check_pattern(an, A):
    if A.n != an.A.n:
        raise errors.DimensionMismatch("matrix dimension %d differs from analyzed %d" % (A.n, an.A.n))
    if (A.nnz != an.A.nnz or not np.array_equal(A.row_ptr, an.A.row_ptr)
            or not np.array_equal(A.col_idx, an.A.col_idx)):
        raise errors.PatternMismatch("refactorization input pattern differs from the analyzed pattern")


def _apply_mode(ctx, an, opts):
    """FactorOptions.kernel_override ("an explicit user override always
    wins"): the mode (maximum tier) of this call, set on the handle
    before the launch; None = the analysis' kernel_mode.  Returns the mode."""
    from .device import check
    mode = opts.kernel_override
    if mode is None:
        mode = an.symbolic.kernel_mode
    else:
        mode = KernelMode.parse(mode) if isinstance(mode, str) else KernelMode(mode)
    check(ctx.lib.hy_set_kernel_mode(ctx.h, int(mode)))
    return mode


def _device_values(ctx, vals, what="values"):
    """Matrix values as a contiguous float64 tensor on the context's device (a torch
    tensor is checked, not converted: its data_ptr goes to the C ABI as is)."""
    import torch
    if isinstance(vals, torch.Tensor):
        if vals.dtype != torch.float64 or vals.device != ctx.device or vals.dim() != 1 \
                or vals.numel() != ctx.nnz or not vals.is_contiguous():
            raise errors.DimensionMismatch(
                "%s must be a contiguous float64 tensor of length %d on %s" % (what, ctx.nnz, ctx.device))
        return vals
    v = np.array(vals, np.float64, copy=True)
    if v.shape != (ctx.nnz,):
        raise errors.DimensionMismatch("%s must have length %d" % (what, ctx.nnz))
    return torch.from_numpy(v).to(ctx.device)


def _enter_stream(ctx, stream, tensors):
    """Order a launch on ``stream`` after the current stream (where the buffers were
    allocated and zeroed) and tell the caching allocator the buffers are in use
    there.  Returns the current stream if it differs from ``stream``, else None."""
    import torch
    if stream is None:
        return None
    cur = torch.cuda.current_stream(ctx.device)
    if stream == cur:
        return None
    stream.wait_stream(cur)
    for t in tensors:
        t.record_stream(stream)
    return cur


def _leave_stream(cur, stream):
    """Order the current stream (status reads in _finish) after the launch."""
    if cur is not None:
        cur.wait_stream(stream)


def _finish(ctx, an, bufs, desc, check_breakdown=True):
    st = bufs["status"].cpu().numpy()
    npert = int(st[0])
    if check_breakdown and st[1] != 0:
        raise errors.NumericBreakdown("zero pivot at factor row %d with perturbation disabled"
                                      % (int(st[1]) - 1))
    k = min(npert, int(desc.pert_cap))
    rows = bufs["pert_rows"][:k].cpu().numpy()
    vals = bufs["pert_vals"][:k].cpu().numpy()
    o = np.argsort(rows, kind="stable")
    pert = list(zip(rows[o].tolist(), vals[o].tolist()))
    anorm = float(bufs["anorm"].cpu().item())
    return NumericFactors(an.symbolic, bufs["values"], bufs["inner_perm"], anorm, pert,
                          bufs, desc, ctx, KernelMode(int(desc.kernel_mode)))


def factorize_analysis(an, values=None, opts=None, stream=None):
    """factorize on an ``Analysis`` (values default to the analyzed A's)."""
    import torch
    opts = opts or FactorOptions()
    ctx = _context(an, opts.device)
    _apply_mode(ctx, an, opts)
    d_vals = _device_values(ctx, an.A.values if values is None else values)
    bufs, desc = ctx.alloc_factors()
    from .device import check
    cur = _enter_stream(ctx, stream, [d_vals, *bufs.values()])
    check(ctx.lib.hy_factorize(ctx.h, d_vals.data_ptr(), float(opts.perturbation_epsilon),
                               desc, ctx.stream_handle(stream)))
    _leave_stream(cur, stream)
    return _finish(ctx, an, bufs, desc)


def factorize(A, ps, order=None, sym=None, opts=None):
    """SPEC.md:280-288.  Also accepts ``factorize(analysis, opts=...)``."""
    if isinstance(A, Analysis):
        return factorize_analysis(A, None, ps if isinstance(ps, FactorOptions) else opts)
    an = _analysis_for(A, ps, order, sym)
    if A is not an.A:
        _check_pattern(an, A)
    return factorize_analysis(an, A.values, opts)


def refactorize(A_new, prior, opts=None, stream=None):
    """reuse PivotScale, Ordering, symbolic, schedule, inner_perm, anorm."""
    import torch
    from .device import check
    opts = opts or FactorOptions()
    ctx = prior._ctx
    an = ctx.analysis
    if isinstance(A_new, torch.Tensor):
        d_vals = _device_values(ctx, A_new, "refactorization values")
    else:
        _check_pattern(an, A_new)
        d_vals = _device_values(ctx, A_new.values)
    if opts.kernel_override is None:
        opts = FactorOptions(prior.kernel_mode, opts.perturbation_epsilon, opts.threads,
                             opts.pivot_tolerance, opts.device)
    _apply_mode(ctx, an, opts)
    bufs, desc = ctx.alloc_factors()
    cur = _enter_stream(ctx, stream, [d_vals, prior.values, prior.inner_perm, *bufs.values()])
    check(ctx.lib.hy_refactorize(ctx.h, d_vals.data_ptr(), float(opts.perturbation_epsilon),
                                 prior._desc, desc, ctx.stream_handle(stream)))
    _leave_stream(cur, stream)
    return _finish(ctx, an, bufs, desc)


def substitute(factors, b, stream=None):
    """Forward/backward substitution with scaling and permutations (no refinement)."""
    import torch
    from .device import check
    ctx = factors._ctx
    d_b = b if isinstance(b, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(b, np.float64)).to(ctx.device)
    if d_b.shape != (ctx.n,):
        raise errors.DimensionMismatch("b must have length %d" % ctx.n)
    d_x = torch.empty(ctx.n, dtype=torch.float64, device=ctx.device)
    check(ctx.lib.hy_solve(ctx.h, factors._desc, d_b.data_ptr(), d_x.data_ptr(),
                           ctx.stream_handle(stream)))
    return d_x


def multi_rhs_method(factors):
    """Route of ``substitute_multi(method="auto")``: the level-scheduled multi-RHS
    solve ("levels": warp per standalone row, CTA per wide row, CTA per supernode with
    its off-block panel on DMMA).  Measured on one B200 with 32 right-hand sides
    (``scripts/multi_rhs_probe.py``): c0 1.04 ms levels / 10.4 ms partition / 16.1 ms
    as 32 single solves; c1 5.2 / 18.3 / 19.3 ms; c2 243 / 9521 / 785 ms; c3 (k=32)
    145 / 6119 / 468 ms.  The partition solve of SPEC.md:461-487 ("partition") stays
    selectable: it is the reference's method, and one warp per row range is the GPU
    form of its per-thread row ranges."""
    return "levels"


def substitute_multi(factors, B, stream=None, method="auto"):
    """Forward/backward substitution for many right-hand sides at once.  ``method``:
    "partition" — the partition-based device solve (Fig. 3;
    ``partition.py``, ``hy_solve_multi``); "levels" — the level-scheduled multi-RHS
    solve (``partition.device_launches_levels``: warp per standalone row, CTA per wide
    row, CTA per supernode with its off-block panel on DMMA); "columns" — one
    ``hy_solve`` per right-hand side; "auto" — ``multi_rhs_method``.  B is [nrhs, n]
    (numpy or a CUDA float64 tensor); returns X [nrhs, n] on the device."""
    import torch
    from .device import check
    ctx = factors._ctx
    d_B = B if isinstance(B, torch.Tensor) else torch.from_numpy(
        np.ascontiguousarray(B, np.float64)).to(ctx.device)
    if d_B.dim() == 1:
        d_B = d_B.reshape(1, -1)
    if d_B.dim() != 2 or d_B.shape[1] != ctx.n or d_B.dtype != torch.float64 or d_B.device != ctx.device:
        raise errors.DimensionMismatch("B must be a float64 [nrhs, %d] array" % ctx.n)
    d_B = d_B.contiguous()
    d_X = torch.empty_like(d_B)
    if method == "auto":
        method = multi_rhs_method(factors)
    sh = ctx.stream_handle(stream)
    if method == "columns":
        for j in range(d_B.shape[0]):
            check(ctx.lib.hy_solve(ctx.h, factors._desc, d_B[j].data_ptr(), d_X[j].data_ptr(), sh))
        return d_X
    if method == "levels":
        ctx.ensure_partition(method="levels")
    elif method == "partition":
        if getattr(ctx, "_partition_key", ("levels",)) == ("levels",):   # else: the uploaded one
            ctx.ensure_partition()
    else:
        raise ValueError("method must be auto, partition, levels or columns")
    check(ctx.lib.hy_solve_multi(ctx.h, factors._desc, d_B.shape[0], d_B.data_ptr(), d_X.data_ptr(), sh))
    return d_X


def solve_multi(A, factors, B, config=None):
    """solve for the rows of B [nrhs, n] at once: partition-based
    substitution, then the automatic refinement of SPEC.md:492 per right-hand side
    when perturbation fired.  Returns (X [nrhs, n] numpy, [RefinementReport])."""
    import torch
    B = np.ascontiguousarray(B, np.float64)
    if B.ndim != 2 or B.shape[1] != A.n:
        raise errors.DimensionMismatch("B must have shape [nrhs, %d]" % A.n)
    X = substitute_multi(factors, B)
    reports = [RefinementReport() for _ in range(B.shape[0])]
    if factors.perturbed:
        ctx = factors._ctx
        for j in range(B.shape[0]):
            d_b = torch.from_numpy(B[j].copy()).to(ctx.device)
            xj, reports[j] = iterative_refinement(A, factors, d_b, X[j].clone(), config)
            X[j] = xj
    return X.cpu().numpy(), reports


def solve(A, factors, ps=None, order=None, b=None, threads=1, config=None):
    """SPEC.md:489-497 (+ automatic iterative_refinement when perturbation fired,
    SPEC.md:499-507, on the device: residual and backward error in original
    coordinates, bitwise the reference's matrix.py row loops)."""
    import torch
    b = np.ascontiguousarray(b, np.float64)
    if b.shape != (A.n,):
        raise errors.DimensionMismatch("b must have length %d" % A.n)
    ctx = factors._ctx
    d_b = torch.from_numpy(b.copy()).to(ctx.device)
    d_x = substitute(factors, d_b)
    report = RefinementReport()
    if factors.perturbed:
        d_x, report = iterative_refinement(A, factors, d_b, d_x, config)
    return d_x.cpu().numpy(), report


def backward_error(A, factors, x, b):
    """Componentwise backward error (matrix.py:303-310) computed on the device."""
    import torch
    from .device import check
    ctx = factors._ctx
    ctx.ensure_matrix(A)
    dev = ctx.device
    d_a = torch.from_numpy(np.array(A.values, np.float64, copy=True)).to(dev)
    d_x = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.array(x, np.float64, copy=True)).to(dev)
    d_b = b if isinstance(b, torch.Tensor) else torch.from_numpy(np.array(b, np.float64, copy=True)).to(dev)
    berr = torch.zeros(1, dtype=torch.float64, device=dev)
    check(ctx.lib.hy_residual(ctx.h, d_a.data_ptr(), d_x.data_ptr(), d_b.data_ptr(), None,
                              berr.data_ptr(), ctx.stream_handle(None)))
    return float(berr.item())


def iterative_refinement(A, factors, d_b, d_x, config=None):
    """SPEC.md:499-507 on the device: r = b - A x, stop at backward error <=
    refine_tolerance, after max_refine_iters, or when the error fails to drop by
    refine_stagnation_factor; else x += solve(r).  One fused residual/backward-error
    pass per iteration; only the scalar backward error crosses to the host."""
    import torch
    from .device import check
    cfg = config or SolverConfig()
    ctx = factors._ctx
    ctx.ensure_matrix(A)
    dev = ctx.device
    sh = ctx.stream_handle(None)
    d_a = torch.from_numpy(np.array(A.values, np.float64, copy=True)).to(dev)
    r = torch.empty_like(d_x)
    berr = torch.zeros(1, dtype=torch.float64, device=dev)

    def resid(x):
        check(ctx.lib.hy_residual(ctx.h, d_a.data_ptr(), x.data_ptr(), d_b.data_ptr(), r.data_ptr(),
                                  berr.data_ptr(), sh))
        return float(berr.item())

    x = d_x
    errs = [resid(x)]
    it = 0
    converged = errs[-1] <= cfg.refine_tolerance
    while not converged and it < cfg.max_refine_iters:
        dx = substitute(factors, r)
        xn = x.clone()
        check(ctx.lib.hy_axpy(ctx.h, xn.data_ptr(), dx.data_ptr(), sh))
        e = resid(xn)
        it += 1
        if e > cfg.refine_stagnation_factor * errs[-1]:
            if e < errs[-1]:
                x = xn
                errs.append(e)
            break
        x = xn
        errs.append(e)
        converged = e <= cfg.refine_tolerance
    return x, RefinementReport(it, errs, bool(converged))


class BatchedRefactorizer:
    """B x [refactorize → solve] sharing one symbolic structure on one GPU
    (BASELINE config 4).  Reuses ``prior``'s inner_perm and anorm."""

    def __init__(self, prior, eps=1e-8, hub_steps=None):
        from .schedule import HUB_STEPS, build_programs
        self.prior = prior
        self.ctx = prior._ctx
        self.eps = eps
        self.programs = build_programs(self.ctx.analysis, prior.host_inner_perm(),
                                       HUB_STEPS if hub_steps is None else hub_steps)
        self.ctx.upload_programs(self.programs)

    def run(self, d_vals, d_rhs, d_x=None, d_npert=None, stream=None, refine=True, config=None):
        """Refactorize + solve B instances (device buffers).  ``refine=True`` (SPEC.md:492:
        refinement runs automatically when perturbation fired): waits for the batch,
        and instances with a nonzero perturbation count get ``refine``; their reports
        land in ``self.reports`` ({instance: RefinementReport}).  ``refine=False``
        keeps the call asynchronous; the caller then checks ``d_npert`` and calls
        ``refine`` before the next batched call on this handle."""
        import torch
        from .device import check
        B = d_vals.shape[0]
        if d_vals.shape[1] != self.ctx.nnz or d_rhs.shape != (B, self.ctx.n):
            raise errors.DimensionMismatch("batched values/rhs shapes do not match the analysis")
        if d_x is None:
            d_x = torch.empty((B, self.ctx.n), dtype=torch.float64, device=self.ctx.device)
        if d_npert is None:
            d_npert = torch.empty(B, dtype=torch.int32, device=self.ctx.device)
        sh = self.ctx.stream_handle(stream)
        check(self.ctx.lib.hy_refactorize_batched(
            self.ctx.h, B, d_vals.data_ptr(), float(self.eps), self.prior._desc, d_npert.data_ptr(),
            d_rhs.data_ptr(), sh))
        check(self.ctx.lib.hy_solve_batched(self.ctx.h, B, None, d_x.data_ptr(), sh))
        self.reports = {}
        if refine:
            self.reports = self.refine(d_vals, d_rhs, d_x, d_npert, config, stream)
        return d_x, d_npert

    def refine(self, d_vals, d_rhs, d_x, d_npert, config=None, stream=None):
        """iterative_refinement for every instance of the batch just
        factorized on this handle whose perturbation count is nonzero, on the device:
        per iteration one masked batched residual + backward error pass
        (``hy_residual_batched``, bitwise the reference's matrix.py loops per
        instance), one batched substitution with the residuals as right-hand sides
        (``hy_solve_batched``), one masked x + dx; per-instance stop rules as the
        single-instance loop (tolerance, max iterations, stagnation).  Only the B
        backward errors cross to the host per iteration.  Returns
        {instance: RefinementReport}; ``d_x`` is updated in place."""
        import torch
        from .device import check
        cfg = config or SolverConfig()
        ctx = self.ctx
        dev = ctx.device
        B = d_vals.shape[0]
        st = stream or torch.cuda.current_stream(dev)
        st.synchronize()
        npert = d_npert.cpu().numpy()
        todo = np.flatnonzero(npert > 0)
        if len(todo) == 0:
            return {}
        ctx.ensure_matrix(ctx.analysis.A)
        sh = ctx.stream_handle(st)
        lib = ctx.lib
        with torch.cuda.stream(st):
            r = torch.zeros_like(d_x)
            dx = torch.zeros_like(d_x)
            xn = torch.empty_like(d_x)
            berr = torch.zeros(B, dtype=torch.float64, device=dev)
            mask_h = np.zeros(B, np.int32)
            mask = torch.zeros(B, dtype=torch.int32, device=dev)

        def set_mask(idx):
            mask_h[:] = 0
            mask_h[idx] = 1
            mask.copy_(torch.from_numpy(mask_h))

        def resid(x):
            check(lib.hy_residual_batched(ctx.h, B, d_vals.data_ptr(), x.data_ptr(), d_rhs.data_ptr(),
                                          r.data_ptr(), berr.data_ptr(), mask.data_ptr(), sh))
            return berr.cpu().numpy()

        with torch.cuda.stream(st):
            set_mask(todo)
            e0 = resid(d_x)
            errs = {int(b): [float(e0[b])] for b in todo}
            iters = {int(b): 0 for b in todo}
            conv = {int(b): bool(e0[b] <= cfg.refine_tolerance) for b in todo}
            active = [int(b) for b in todo if not conv[int(b)]]
            while active:
                set_mask(active)
                check(lib.hy_solve_batched(ctx.h, B, r.data_ptr(), dx.data_ptr(), sh))
                check(lib.hy_axpy_batched(ctx.h, B, xn.data_ptr(), d_x.data_ptr(), dx.data_ptr(),
                                          mask.data_ptr(), sh))
                e = resid(xn)
                accept, nxt = [], []
                for b in active:
                    eb, last = float(e[b]), errs[b][-1]
                    iters[b] += 1
                    if eb > cfg.refine_stagnation_factor * last:
                        if eb < last:
                            accept.append(b)
                            errs[b].append(eb)
                        continue
                    accept.append(b)
                    errs[b].append(eb)
                    conv[b] = eb <= cfg.refine_tolerance
                    if not conv[b] and iters[b] < cfg.max_refine_iters:
                        nxt.append(b)
                if accept:
                    set_mask(accept)
                    check(lib.hy_axpy_batched(ctx.h, B, d_x.data_ptr(), xn.data_ptr(), None,
                                              mask.data_ptr(), sh))
                # a continuing instance was accepted: r already holds b - A x_new
                active = nxt
            st.synchronize()
        return {b: RefinementReport(iters[b], errs[b], bool(conv[b])) for b in errs}

    def run_host(self, h_vals, h_rhs, h_x, h_npert=None, chunks=8, sizes=None, pipelined=False,
                 refine=True):
        """Host buffers in, host buffers out, copies overlapped with compute.

        The batch is cut into ``chunks`` contiguous slabs (multiples of 32
        instances); chunk k's values/rhs go H2D on a copy stream while chunk k-1
        is refactorized+solved on the compute stream and chunk k-2's solutions go
        D2H on a third stream.  ``h_*`` should be pinned torch CPU tensors.
        ``sizes`` (optional) gives explicit chunk sizes instead.

        ``pipelined=False``: the caller's current stream waits for the last D2H
        (results are ready in stream order).  ``pipelined=True`` (streaming use):
        the call returns without that wait, so the next call's H2D copies start
        while this call's last chunks still compute — each chunk's device buffers
        are reused only after their previous compute / D2H finished (per-chunk
        events).  Call ``host_wait()`` before reading ``h_x``.

        ``refine`` (needs ``h_npert``): perturbed instances are refined once the
        copies are done — at the end of the call (``pipelined=False``) or in
        ``host_wait()`` (``pipelined=True``); see ``_fixup_host``."""
        import torch
        B = h_vals.shape[0]
        dev = self.ctx.device
        if sizes is None:
            per = ((B + chunks - 1) // chunks + 31) // 32 * 32
            sizes = [min(per, B - a) for a in range(0, B, per)]
        bounds, a = [], 0
        for c in sizes:
            if a >= B:
                break
            bounds.append((a, min(B, a + int(c))))
            a += int(c)
        if a < B:
            bounds.append((a, B))
        key = (B, tuple(bounds))
        if getattr(self, "_host_key", None) != key:
            if getattr(self, "_host_key", None) is not None:
                torch.cuda.synchronize(dev)
            self._host_key = key
            self._streams = [torch.cuda.Stream(dev) for _ in range(3)]
            self._dbufs = []
            for a, b in bounds:
                self._dbufs.append((torch.empty((b - a, self.ctx.nnz), dtype=torch.float64, device=dev),
                                    torch.empty((b - a, self.ctx.n), dtype=torch.float64, device=dev),
                                    torch.empty((b - a, self.ctx.n), dtype=torch.float64, device=dev),
                                    torch.empty(b - a, dtype=torch.int32, device=dev)))
            self._ev_cmp = [None] * len(bounds)   # compute of chunk k done (dv/dr free)
            self._ev_out = [None] * len(bounds)   # D2H of chunk k done (dx/dn free)
        s_in, s_cmp, s_out = self._streams
        cur = torch.cuda.current_stream(dev)
        s_in.wait_stream(cur)
        for k, ((a, b), (dv, dr, dx, dn)) in enumerate(zip(bounds, self._dbufs)):
            with torch.cuda.stream(s_in):
                if self._ev_cmp[k] is not None:
                    s_in.wait_event(self._ev_cmp[k])
                dv.copy_(h_vals[a:b], non_blocking=True)
                dr.copy_(h_rhs[a:b], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(s_in)
            s_cmp.wait_event(ev_in)
            if self._ev_out[k] is not None:
                s_cmp.wait_event(self._ev_out[k])
            self.run(dv, dr, dx, dn, s_cmp, refine=False)
            ev_c = torch.cuda.Event()
            ev_c.record(s_cmp)
            self._ev_cmp[k] = ev_c
            s_out.wait_event(ev_c)
            with torch.cuda.stream(s_out):
                h_x[a:b].copy_(dx, non_blocking=True)
                if h_npert is not None:
                    h_npert[a:b].copy_(dn, non_blocking=True)
                ev_o = torch.cuda.Event()
                ev_o.record(s_out)
                self._ev_out[k] = ev_o
        self._pending = (h_vals, h_rhs, h_x, h_npert) if (refine and h_npert is not None) else None
        if not pipelined:
            cur.wait_stream(s_out)
            self._fixup_host()
        return h_x, h_npert

    def _fixup_host(self):
        """Automatic refinement for run_host: once the copies are done,
        instances whose perturbation count is nonzero are refactorized again as one
        sub-batch on the device and refined (``run(..., refine=True)``); their
        solutions replace the rows of ``h_x``.  Reports go to ``self.reports``."""
        import torch
        pend, self._pending = getattr(self, "_pending", None), None
        self.reports = {}
        if pend is None:
            return
        h_vals, h_rhs, h_x, h_npert = pend
        self._streams[2].synchronize()
        idx = np.flatnonzero(h_npert.numpy() > 0)
        if len(idx) == 0:
            return
        dev = self.ctx.device
        ti = torch.from_numpy(idx)
        dv = h_vals[ti].to(dev)
        dr = h_rhs[ti].to(dev)
        dx, _ = self.run(dv, dr)
        h_x[ti] = dx.cpu()
        self.reports = {int(idx[k]): rep for k, rep in self.reports.items()}

    def host_wait(self, stream=None):
        """Make ``stream`` (default: current) wait for every pending run_host copy.  If
        the last run_host call asked for refinement (``h_npert`` given), this first
        waits for its copies and refines the perturbed instances (``_fixup_host``)."""
        import torch
        if getattr(self, "_pending", None) is not None:
            self._fixup_host()
        if getattr(self, "_streams", None):
            (stream or torch.cuda.current_stream(self.ctx.device)).wait_stream(self._streams[2])

    def factor_values(self, b, stream=None):
        import torch
        from .device import check
        out = torch.empty(self.ctx.stored, dtype=torch.float64, device=self.ctx.device)
        check(self.ctx.lib.hy_batched_factor_values(self.ctx.h, b, out.data_ptr(),
                                                    self.ctx.stream_handle(stream)))
        return out


def refactorize_solve_batched(values, prior, rhs, opts=None, hub_steps=None):
    """Host-facing batched call: values [B, nnz], rhs [B, n] (numpy or CUDA tensors)
    → (x [B, n] numpy, perturbation counts [B]).  Perturbed instances are refined
    automatically; their RefinementReports are left in
    ``refactorize_solve_batched.last_reports`` ({instance: report})."""
    import torch
    opts = opts or FactorOptions()
    br = BatchedRefactorizer(prior, opts.perturbation_epsilon, hub_steps)
    dev = br.ctx.device
    dv = values if isinstance(values, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(values)).to(dev)
    dr = rhs if isinstance(rhs, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(rhs)).to(dev)
    x, npert = br.run(dv, dr, refine=True)
    refactorize_solve_batched.last_reports = br.reports
    return x.cpu().numpy(), npert.cpu().numpy()
