"""Symbolic factorization, supernode detection, kernel selection, task graph and
levels — the host half of the hot path, uploaded once.

The reference ships none of these operations; this is a from-SPEC
implementation shared by the CPU oracle and the device path, so symbolic
structure, supernode partition and ``kernel_mode`` are bit-identical on both by
construction.  Interpretive choices are recorded here:

* flops / fill_nnz are counted on the exact pre-union pattern (App. B #3):
  flops = Σ_k [2·|L(:,k) below|·|U(k,:) right| + |L(:,k) below|],
  fill_nnz = nnz(L strictly lower) + nnz(U incl. diagonal).
* Supernode = maximal run of consecutive rows with U(i+1,:) = U(i,:) \\ {i}
  (SPEC.md:188); runs longer than ``max_supernode_rows`` are cut into chunks of
  exactly ``max_supernode_rows`` from the top, the last chunk holding the rest;
  any run/chunk shorter than ``min_supernode_rows`` becomes standalone rows.
* Within-supernode L union: every row of a supernode stores the
  union of the rows' L columns left of the block, plus the dense diagonal block.

Node storage layout (shared with the device):
every node u owns one ascending column list ``ncols[colptr[u]:colptr[u+1]]`` of
width W_u and a dense row-major value block of ``rows_u x W_u`` doubles at
``valoff[u]``.  For a standalone row the list is L(i,:) ++ U(i,:) with the
diagonal at position ``nl[u]``; for a supernode it is Lunion ++ block ++ panel,
so row t of the block has its diagonal at position ``nl[u] + t``.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numba import njit, prange

from ._ref import KernelMode, SolverConfig, errors

STANDALONE_ROW = 0
SUPERNODE = 1


# --------------------------------------------------------------------------- symbolic kernels
@njit(cache=True)
def _has_full_diag(n, mp, mc):
    for i in range(n):
        ok = False
        for t in range(mp[i], mp[i + 1]):
            if mc[t] == i:
                ok = True
                break
        if not ok:
            return i
    return -1


@njit(cache=True)
def _general_symbolic(n, mp, mc):
    """Row-by-row Gilbert–Peierls reach: L(i,:) = columns j<i reachable
    from M(i,<i) through U rows; U(i,:) = M(i,>=i) ∪ ⋃_{j∈L(i,:)} U(j,>j).

    Returns exact (lp, li, up, ui); U rows list the diagonal first."""
    cap_l = max(16, 2 * (mp[n] - n) + 16)
    cap_u = max(16, 2 * mp[n] + 16)
    lp = np.zeros(n + 1, np.int64)
    up = np.zeros(n + 1, np.int64)
    li = np.empty(cap_l, np.int32)
    ui = np.empty(cap_u, np.int32)
    mark = np.full(n, -1, np.int64)
    work = np.empty(n, np.int64)
    lbuf = np.empty(n, np.int32)
    ubuf = np.empty(n, np.int32)
    for i in range(n):
        nw = 0
        nl = 0
        nu = 0
        for t in range(mp[i], mp[i + 1]):
            k = mc[t]
            mark[k] = i
            if k < i:
                work[nw] = k
                nw += 1
            else:
                ubuf[nu] = k
                nu += 1
        while nw > 0:
            nw -= 1
            j = work[nw]
            lbuf[nl] = j
            nl += 1
            for t in range(up[j] + 1, up[j + 1]):
                k = ui[t]
                if mark[k] != i:
                    mark[k] = i
                    if k < i:
                        work[nw] = k
                        nw += 1
                    else:
                        ubuf[nu] = k
                        nu += 1
        ls = np.sort(lbuf[:nl])
        us = np.sort(ubuf[:nu])
        if lp[i] + nl > cap_l:
            cap_l = max(2 * cap_l, lp[i] + nl)
            tmp = np.empty(cap_l, np.int32)
            tmp[:lp[i]] = li[:lp[i]]
            li = tmp
        if up[i] + nu > cap_u:
            cap_u = max(2 * cap_u, up[i] + nu)
            tmp = np.empty(cap_u, np.int32)
            tmp[:up[i]] = ui[:up[i]]
            ui = tmp
        li[lp[i]:lp[i] + nl] = ls
        ui[up[i]:up[i] + nu] = us
        lp[i + 1] = lp[i] + nl
        up[i + 1] = up[i] + nu
    return lp, li[:lp[n]].copy(), up, ui[:up[n]].copy()


@njit(cache=True)
def _general_symbolic_chains(n, mp, mc):
    """Same result as ``_general_symbolic`` (exact L/U patterns, bit for bit), with
    the reach accelerated by U-nesting chains: rows h..e form a chain when
    U(r+1,:) = U(r,:) minus {r} for h <= r < e, so for every row r of a chain
    U(r,>r) = {r+1..e} ∪ U(e,>e).  Within the reach of row i each chain's tail row
    U(e,>e) is therefore scanned once, and the chain's rows above the lowest visited
    one are added as a range, instead of scanning U(r,>r) for every visited r —
    the cost drops from Σ_{j∈L(i,:)} |U(j,>j)| (the flop count) to about the
    output size.  (a supernodal form of the Gilbert–Peierls reach.)"""
    cap_l = max(16, 2 * (mp[n] - n) + 16)
    cap_u = max(16, 2 * mp[n] + 16)
    lp = np.zeros(n + 1, np.int64)
    up = np.zeros(n + 1, np.int64)
    li = np.empty(cap_l, np.int32)
    ui = np.empty(cap_u, np.int32)
    mark = np.full(n, -1, np.int64)
    work = np.empty(n, np.int64)
    lbuf = np.empty(n, np.int32)
    ubuf = np.empty(n, np.int32)
    head = np.empty(n, np.int64)       # chain head of each processed row
    tail = np.empty(n, np.int64)       # chain tail (indexed by head)
    cseen = np.full(n, -1, np.int64)   # per head: row i whose reach visited the chain
    cmin = np.empty(n, np.int64)       # per head: lowest chain row visited in that reach
    for i in range(n):
        nw = 0
        nl = 0
        nu = 0
        for t in range(mp[i], mp[i + 1]):
            k = mc[t]
            mark[k] = i
            if k < i:
                work[nw] = k
                nw += 1
            else:
                ubuf[nu] = k
                nu += 1
        while nw > 0:
            nw -= 1
            j = work[nw]
            lbuf[nl] = j
            nl += 1
            h = head[j]
            e = tail[h]
            if cseen[h] != i:
                cseen[h] = i
                cmin[h] = e
                # the tail's off-diagonal U entries
                for t in range(up[e] + 1, up[e + 1]):
                    k = ui[t]
                    if mark[k] != i:
                        mark[k] = i
                        if k < i:
                            work[nw] = k
                            nw += 1
                        else:
                            ubuf[nu] = k
                            nu += 1
            if j < cmin[h]:
                # chain rows j+1 .. cmin-1 (rows up to the tail are columns of U(j,>j));
                # the row cmin itself is already marked (it was visited or is the tail,
                # whose own U row above covers the rest)
                for k in range(j + 1, cmin[h] + 1):
                    if mark[k] != i:
                        mark[k] = i
                        if k < i:
                            work[nw] = k
                            nw += 1
                        else:
                            ubuf[nu] = k
                            nu += 1
                cmin[h] = j
        ls = np.sort(lbuf[:nl])
        us = np.sort(ubuf[:nu])
        if lp[i] + nl > cap_l:
            cap_l = max(2 * cap_l, lp[i] + nl)
            tmp = np.empty(cap_l, np.int32)
            tmp[:lp[i]] = li[:lp[i]]
            li = tmp
        if up[i] + nu > cap_u:
            cap_u = max(2 * cap_u, up[i] + nu)
            tmp = np.empty(cap_u, np.int32)
            tmp[:up[i]] = ui[:up[i]]
            ui = tmp
        li[lp[i]:lp[i] + nl] = ls
        ui[up[i]:up[i] + nu] = us
        lp[i + 1] = lp[i] + nl
        up[i + 1] = up[i] + nu
        # chain membership: row i extends row i-1's chain when U(i,:) = U(i-1,:) minus {i-1}
        ext = False
        if i > 0 and up[i] - up[i - 1] == nu + 1 and ui[up[i - 1]] == i - 1:
            ext = True
            for t in range(nu):
                if ui[up[i - 1] + 1 + t] != ui[up[i] + t]:
                    ext = False
                    break
        if ext:
            h = head[i - 1]
            head[i] = h
            tail[h] = i
        else:
            head[i] = i
            tail[i] = i
            cseen[i] = -1
    return lp, li[:lp[n]].copy(), up, ui[:up[n]].copy()


@njit(cache=True)
def _etree(n, mp, mc):
    """Elimination tree of a structurally symmetric pattern (Liu, path compression)."""
    parent = np.full(n, -1, np.int64)
    anc = np.full(n, -1, np.int64)
    for i in range(n):
        for t in range(mp[i], mp[i + 1]):
            k = mc[t]
            if k >= i:
                continue
            r = k
            while anc[r] != -1 and anc[r] != i:
                nxt = anc[r]
                anc[r] = i
                r = nxt
            if anc[r] == -1:
                anc[r] = i
                parent[r] = i
    return parent


@njit(cache=True, parallel=True)
def _row_subtrees(n, mp, mc, parent, nthreads):
    """L(i,:) = row subtree of i in the etree (symmetric patterns); exact, sorted.

    Rows are independent given the etree: two passes (count, fill) over rows dealt
    round-robin to ``nthreads`` workers, each with its own mark array (marker = the
    row being walked).  Output is independent of the thread count."""
    cnt = np.zeros(n + 1, np.int64)
    marks = np.full((nthreads, n), -1, np.int64)
    for T in prange(nthreads):
        mark = marks[T]
        for i in range(T, n, nthreads):
            mark[i] = i
            c = 0
            for t in range(mp[i], mp[i + 1]):
                j = mc[t]
                while j < i and mark[j] != i:
                    mark[j] = i
                    c += 1
                    j = parent[j]
            cnt[i + 1] = c
    lp = np.cumsum(cnt)
    li = np.empty(lp[n], np.int32)
    for T in prange(nthreads):
        mark = marks[T]
        mark[:] = -1
        for i in range(T, n, nthreads):
            mark[i] = i
            c = lp[i]
            for t in range(mp[i], mp[i + 1]):
                j = mc[t]
                while j < i and mark[j] != i:
                    mark[j] = i
                    li[c] = j
                    c += 1
                    j = parent[j]
            li[lp[i]:c] = np.sort(li[lp[i]:c])
    return lp, li


@njit(cache=True)
def _u_from_l(n, lp, li):
    """U(j,:) = {j} ∪ {i : j ∈ L(i,:)} (symmetric case), ascending."""
    cnt = np.ones(n + 1, np.int64)
    cnt[0] = 0
    for t in range(lp[n]):
        cnt[li[t] + 1] += 1
    up = np.cumsum(cnt)
    ui = np.empty(up[n], np.int32)
    fill = up[:n].copy()
    for j in range(n):
        ui[fill[j]] = j
        fill[j] += 1
    for i in range(n):
        for t in range(lp[i], lp[i + 1]):
            j = li[t]
            ui[fill[j]] = i
            fill[j] += 1
    return up, ui


@njit(cache=True)
def _flops_fill(n, lp, li, up):
    colcnt = np.zeros(n, np.int64)
    for t in range(lp[n]):
        colcnt[li[t]] += 1
    flops = 0.0
    for k in range(n):
        lk = colcnt[k]
        uk = up[k + 1] - up[k] - 1
        flops += 2.0 * lk * uk + lk
    return flops, lp[n] + up[n]


@njit(cache=True)
def _nested(up, ui, i):
    """U(i+1,:) == U(i,:) \\ {i}."""
    a0, a1 = up[i] + 1, up[i + 1]
    b0, b1 = up[i + 1], up[i + 2]
    if a1 - a0 != b1 - b0:
        return False
    for t in range(a1 - a0):
        if ui[a0 + t] != ui[b0 + t]:
            return False
    return True


@njit(cache=True)
def _partition(n, up, ui, smin, smax):
    """Node boundaries (node_first[nn+1]) and kinds per the detect_supernodes rule."""
    first = np.empty(n + 1, np.int64)
    kind = np.empty(n, np.int8)
    nn = 0
    i = 0
    while i < n:
        j = i
        while j + 1 < n and _nested(up, ui, j):
            j += 1
        run = j - i + 1
        s = i
        while s <= j:
            c = min(smax, j - s + 1)
            if c >= smin and c >= 2:
                first[nn] = s
                kind[nn] = SUPERNODE
                nn += 1
                s += c
            else:
                for r in range(s, s + c):
                    first[nn] = r
                    kind[nn] = STANDALONE_ROW
                    nn += 1
                s += c
        i = j + 1
    first[nn] = n
    return first[:nn + 1].copy(), kind[:nn].copy()


@njit(cache=True)
def _node_cols(n, nn, first, kind, lp, li, up, ui):
    """Per-node ascending column lists (Lunion ++ block ++ panel / L ++ U) and nl."""
    colptr = np.zeros(nn + 1, np.int64)
    nl = np.zeros(nn, np.int64)
    mark = np.full(n, -1, np.int64)
    # pass 1: widths
    for u in range(nn):
        r = first[u]
        s = first[u + 1] - r
        if kind[u] == STANDALONE_ROW:
            nl[u] = lp[r + 1] - lp[r]
            colptr[u + 1] = nl[u] + up[r + 1] - up[r]
        else:
            c = 0
            for t in range(r, r + s):
                for q in range(lp[t], lp[t + 1]):
                    j = li[q]
                    if j < r and mark[j] != u:
                        mark[j] = u
                        c += 1
            nl[u] = c
            colptr[u + 1] = c + (up[r + 1] - up[r])
    for u in range(nn):
        colptr[u + 1] += colptr[u]
    cols = np.empty(colptr[nn], np.int32)
    mark[:] = -1
    for u in range(nn):
        r = first[u]
        s = first[u + 1] - r
        o = colptr[u]
        if kind[u] == STANDALONE_ROW:
            k = lp[r + 1] - lp[r]
            cols[o:o + k] = li[lp[r]:lp[r + 1]]
            cols[o + k:colptr[u + 1]] = ui[up[r]:up[r + 1]]
        else:
            c = o
            for t in range(r, r + s):
                for q in range(lp[t], lp[t + 1]):
                    j = li[q]
                    if j < r and mark[j] != u:
                        mark[j] = u
                        cols[c] = j
                        c += 1
            cols[o:c] = np.sort(cols[o:c])
            cols[c:colptr[u + 1]] = ui[up[r]:up[r + 1]]
    return colptr, cols, nl


@njit(cache=True)
def _deps_levels(n, nn, first, colptr, cols, nl, kind):
    """build_task_graph + compute_levels over the
    stored (union) pattern, and backward-solve levels over U(:, beyond node)."""
    node_of = np.empty(n, np.int64)
    for u in range(nn):
        for r in range(first[u], first[u + 1]):
            node_of[r] = u
    dcnt = np.zeros(nn + 1, np.int64)
    for u in range(nn):
        last = -1
        for q in range(colptr[u], colptr[u] + nl[u]):
            v = node_of[cols[q]]
            if v != last:
                dcnt[u + 1] += 1
                last = v
    dptr = np.cumsum(dcnt)
    deps = np.empty(dptr[nn], np.int32)
    level = np.zeros(nn, np.int64)
    for u in range(nn):
        last = -1
        c = dptr[u]
        lv = 0
        for q in range(colptr[u], colptr[u] + nl[u]):
            v = node_of[cols[q]]
            if v != last:
                deps[c] = v
                c += 1
                last = v
                if level[v] + 1 > lv:
                    lv = level[v] + 1
        level[u] = lv
    # backward solve: node u needs nodes owning its columns right of its last row
    ulevel = np.zeros(nn, np.int64)
    for u in range(nn - 1, -1, -1):
        lastrow = first[u + 1] - 1
        lv = 0
        start = colptr[u] + nl[u]
        for q in range(start, colptr[u + 1]):
            k = cols[q]
            if k > lastrow:
                v = node_of[k]
                if ulevel[v] + 1 > lv:
                    lv = ulevel[v] + 1
        ulevel[u] = lv
    return node_of, dptr, deps, level, ulevel


def _level_sets(level):
    order = np.argsort(level, kind="stable")
    nlev = int(level.max()) + 1 if len(level) else 0
    ptr = np.zeros(nlev + 1, np.int64)
    np.add.at(ptr[1:], level, 1)
    np.cumsum(ptr, out=ptr)
    return ptr, order.astype(np.int32)


def select_kernel(flops, fill_nnz, rho, cfg=None, override=None):
    """ROWROW if ρ < kernel_rho_min or q < kernel_q_rowrow; SUPROW if
    q < kernel_q_suprow; else SUPSUP.  An explicit override always wins."""
    if override is not None:
        return KernelMode(override) if not isinstance(override, str) else KernelMode.parse(override)
    cfg = cfg or SolverConfig()
    q = flops / fill_nnz if fill_nnz else 0.0
    if rho < cfg.kernel_rho_min or q < cfg.kernel_q_rowrow:
        return KernelMode.ROWROW
    if q < cfg.kernel_q_suprow:
        return KernelMode.SUPROW
    return KernelMode.SUPSUP


# --------------------------------------------------------------------------- structure
@dataclass
class SymbolicStructure:
    """SPEC.md:139-151 in node-compressed form (see module docstring).

    ``l_pattern`` / ``u_pattern`` of SPEC are available per row through
    ``row_patterns(i)`` / ``l_pattern()`` / ``u_pattern()`` (derived, union L)."""
    n: int
    node_first: np.ndarray      # int64[nn+1]
    node_kind: np.ndarray       # int8[nn]
    colptr: np.ndarray          # int64[nn+1]
    cols: np.ndarray            # int32[colptr[-1]]
    nl: np.ndarray              # int64[nn]   L-part width (Lunion / L(i,:))
    node_of: np.ndarray         # int64[n]
    dep_ptr: np.ndarray         # int64[nn+1]
    deps: np.ndarray            # int32[...], ascending per node
    level: np.ndarray           # int64[nn]
    level_ptr: np.ndarray       # int64[nlev+1]
    level_nodes: np.ndarray     # int32[nn], ascending within each level
    ulevel: np.ndarray          # backward-solve levels
    ulevel_ptr: np.ndarray
    ulevel_nodes: np.ndarray
    flops: float
    fill_nnz: int
    rho: float
    kernel_mode: KernelMode
    auto_mode: KernelMode
    bulk_level_cutoff: int
    exact_l_nnz: int
    exact_u_nnz: int
    # value layout
    valoff: np.ndarray = field(default=None)   # int64[nn+1]
    mp: np.ndarray = field(default=None, repr=False)   # M pattern (for PatternMismatch checks)
    mc: np.ndarray = field(default=None, repr=False)

    @property
    def nnodes(self):
        return len(self.node_kind)

    @property
    def node_rows(self):
        return np.diff(self.node_first)

    @property
    def width(self):
        return np.diff(self.colptr)

    @property
    def supernode_count(self):
        return int((self.node_kind == SUPERNODE).sum())

    @property
    def standalone_row_count(self):
        return int((self.node_rows[self.node_kind == STANDALONE_ROW]).sum())

    @property
    def stored_values(self):
        return int(self.valoff[-1])

    @property
    def levels(self):
        return [self.level_nodes[self.level_ptr[k]:self.level_ptr[k + 1]].tolist()
                for k in range(len(self.level_ptr) - 1)]

    def node_deps(self, u):
        return self.deps[self.dep_ptr[u]:self.dep_ptr[u + 1]]

    def node_cols(self, u):
        return self.cols[self.colptr[u]:self.colptr[u + 1]]

    def row_patterns(self, i):
        """(L columns, U columns) of factor row i as stored (L union in supernodes)."""
        u = int(self.node_of[i])
        c = self.node_cols(u)
        d = int(self.nl[u]) + (i - int(self.node_first[u]))
        return c[:d], c[d:]

    def l_pattern(self):
        return [self.row_patterns(i)[0] for i in range(self.n)]

    def u_pattern(self):
        return [self.row_patterns(i)[1] for i in range(self.n)]


def _host_threads():
    import numba
    return max(1, int(numba.config.NUMBA_NUM_THREADS))


def symbolic_from_pattern(n, mp, mc, cfg=None, kernel_override=None, threads=1, method="auto"):
    """symbolic_factorize on the permuted pattern M.

    ``method``: 'general' (row reach), 'symmetric' (etree row subtrees; only valid
    for structurally symmetric M) or 'auto'."""
    cfg = cfg or SolverConfig()
    mp = np.ascontiguousarray(mp, np.int64)
    mc = np.ascontiguousarray(mc, np.int64)
    bad = _has_full_diag(n, mp, mc)
    if bad >= 0:
        raise errors.ZeroDiagonal("row %d of the permuted matrix has no diagonal entry" % bad)
    if method == "auto":
        method = "symmetric" if _pattern_symmetric(n, mp, mc) else "general"
    if method == "symmetric":
        parent = _etree(n, mp, mc)
        lp, li = _row_subtrees(n, mp, mc, parent, _host_threads())
        up, ui = _u_from_l(n, lp, li)
    else:
        lp, li, up, ui = _general_symbolic_chains(n, mp, mc)
    flops, fill = _flops_fill(n, lp, li, up)
    first, kind = _partition(n, up, ui, int(cfg.min_supernode_rows), int(cfg.max_supernode_rows))
    nn = len(kind)
    colptr, cols, nl = _node_cols(n, nn, first, kind, lp, li, up, ui)
    del li, ui
    node_of, dptr, deps, level, ulevel = _deps_levels(n, nn, first, colptr, cols, nl, kind)
    lptr, lnodes = _level_sets(level)
    uptr, unodes = _level_sets(ulevel)
    rows = np.diff(first)
    rho = float(rows[kind == SUPERNODE].sum()) / n
    auto = select_kernel(flops, fill, rho, cfg)
    mode = select_kernel(flops, fill, rho, cfg, kernel_override) if kernel_override is not None else auto
    thr = int(cfg.bulk_width_factor) * max(1, int(threads))
    widths = np.diff(lptr)
    small = np.flatnonzero(widths < thr)
    cutoff = int(small[0]) if len(small) else len(widths)
    valoff = np.zeros(nn + 1, np.int64)
    np.cumsum(rows * np.diff(colptr), out=valoff[1:])
    return SymbolicStructure(
        n=n, node_first=first, node_kind=kind, colptr=colptr, cols=cols, nl=nl, node_of=node_of,
        dep_ptr=dptr, deps=deps, level=level, level_ptr=lptr, level_nodes=lnodes,
        ulevel=ulevel, ulevel_ptr=uptr, ulevel_nodes=unodes, flops=float(flops), fill_nnz=int(fill),
        rho=rho, kernel_mode=mode, auto_mode=auto, bulk_level_cutoff=cutoff,
        exact_l_nnz=int(lp[n]), exact_u_nnz=int(up[n]), valoff=valoff, mp=mp, mc=mc)


def _pattern_symmetric(n, mp, mc):
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(mp))
    a = np.sort(rows * n + mc)
    b = np.sort(mc * n + rows)
    return bool(np.array_equal(a, b))
