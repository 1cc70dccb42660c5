"""Partition-based triangular solve (the paper's Fig. 3) for many
right-hand sides at once — SURVEY §8(f) rank 4.

``build_partition`` follows SPEC's [OP] build_partition:

* the first cut point is the row where the bulk levels end: one past the last row
  of any node whose level is below ``bulk_level_cutoff`` (levels narrower than
  ``bulk_width_factor x threads`` run in pipeline mode); the leading
  segment [0, cut0) is solved "bulk-sequential";
* the remaining rows are cut at node boundaries (every node of the narrow pipeline
  levels is its own level boundary) whenever a segment's stored L+U entries would
  exceed ``seg_nnz_threshold`` (``SolverConfig.seg_threshold``, config.py:55-58);
* a segment's triangular part (its entries whose columns lie inside the segment)
  with fewer than ``small_tri_threshold`` entries is flagged sequential;
* the rectangular blocks — L entries of a segment's rows in columns before it
  (forward) and U entries in columns after it (backward) — get ``threads`` row
  ranges that balance their entries greedily by prefix sums, ties to the lower
  thread index.

Entries are the stored node-layout entries (the union-padded supernode panels the
device reads), so "every nonzero of L (resp. U) is applied exactly once per
substitution" is checked over exactly what the kernels touch.

On the device (``solve_multi``) the rectangular blocks are sparse-times-dense
products over the ``nrhs`` columns (one warp per balanced row range, lanes over the
right-hand sides), the triangular parts run one launch per level present in the
segment (warp per node) or, when flagged sequential, one warp walks the segment's
nodes in order.  Forward rows subtract their entries in column order (rectangular
prefix, then the triangle) with separate multiply and subtract, which is the
oracle's forward loop operation for operation.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._ref import SolverConfig


@dataclass
class SolvePartition:
    """SPEC.md:447-451 (SolvePartition)."""
    n: int
    threads: int
    cut_points: np.ndarray     # ascending interior row cuts (strictly inside (0, n))
    seg_rows: np.ndarray       # int64[nseg+1]: segment k = rows [seg_rows[k], seg_rows[k+1])
    seg_nodes: np.ndarray      # int64[nseg+1]: the same boundaries as node indices
    bulk_segment: bool         # segment 0 is the bulk-sequential leading segment
    sequential: np.ndarray     # bool[nseg]: triangular part below small_tri_threshold
    tri_nnz: np.ndarray        # int64[nseg]: stored entries inside the segment's triangle (L+U)
    rect_l_nnz: np.ndarray     # int64[nseg]: L entries left of the segment
    rect_u_nnz: np.ndarray     # int64[nseg]: U entries right of the segment
    rect_l_ranges: list        # per segment: int64[threads+1] row bounds (balanced L rect entries)
    rect_u_ranges: list        # per segment: int64[threads+1] row bounds (balanced U rect entries)

    @property
    def nsegments(self):
        return len(self.seg_rows) - 1


def _row_counts(sym):
    """Per factor row: stored L entries (before the diagonal) and U entries after it."""
    s = sym
    rows = np.diff(s.node_first)
    W = np.diff(s.colptr)
    node = s.node_of
    t = np.arange(s.n) - s.node_first[node]
    nl = s.nl[node] + t
    nu = W[node] - nl - 1
    return nl.astype(np.int64), nu.astype(np.int64), rows


def _split_counts(sym, lo, hi):
    """For rows [lo, hi): L entries with column < lo and U entries with column >= hi."""
    s = sym
    out_l = np.zeros(hi - lo, np.int64)
    out_u = np.zeros(hi - lo, np.int64)
    for i in range(lo, hi):
        u = int(s.node_of[i])
        t = i - int(s.node_first[u])
        c0 = int(s.colptr[u])
        W = int(s.colptr[u + 1]) - c0
        d = int(s.nl[u]) + t
        cols = s.cols[c0:c0 + W]
        out_l[i - lo] = int(np.searchsorted(cols[:d], lo, "left"))
        out_u[i - lo] = W - int(np.searchsorted(cols[d + 1:], hi, "left")) - (d + 1)
    return out_l, out_u


def balanced_ranges(counts, threads):
    """Row ranges of ``threads`` parts with equal entry totals, greedily by prefix
    sums (part t ends at the first row whose prefix reaches (t+1)/threads of the
    total; ties go to the lower part): int64[threads+1] bounds."""
    counts = np.asarray(counts, np.int64)
    m = len(counts)
    pre = np.concatenate([[0], np.cumsum(counts)])
    total = int(pre[-1])
    b = np.zeros(threads + 1, np.int64)
    b[threads] = m
    for t in range(1, threads):
        target = (total * t + threads - 1) // threads
        b[t] = min(m, max(int(b[t - 1]), int(np.searchsorted(pre, target, "left"))))
    return b


def build_partition(sym, threads=1, config=None):
    """SPEC.md:461-469 (see module docstring)."""
    cfg = config or SolverConfig()
    s = sym
    n = s.n
    threads = max(1, int(threads))
    nl, nu, rows = _row_counts(s)
    nnz_total = int(nl.sum() + nu.sum() + n)
    seg_thr = cfg.seg_threshold(nnz_total, threads)
    width = np.diff(s.level_ptr)
    narrow = np.flatnonzero(width < cfg.bulk_width_factor * threads)
    cutoff = int(narrow[0]) if len(narrow) else len(width)
    bulk_nodes = np.flatnonzero(s.level < cutoff)
    cut0 = int(s.node_first[bulk_nodes.max() + 1]) if len(bulk_nodes) else 0
    node_bounds = [0]
    if 0 < cut0 < n:
        node_bounds.append(int(s.node_of[cut0]))
    bulk = cut0 > 0
    # remaining rows: cut at node boundaries when the segment would exceed seg_thr
    row_nnz = nl + nu + 1
    node_nnz = np.add.reduceat(row_nnz, s.node_first[:-1]) if s.nnodes else np.zeros(0, np.int64)
    u0 = int(s.node_of[cut0]) if cut0 < n else s.nnodes
    acc = 0
    for u in range(u0, s.nnodes):
        w = int(node_nnz[u])
        if acc > 0 and acc + w > seg_thr:
            node_bounds.append(u)
            acc = 0
        acc += w
    node_bounds.append(s.nnodes)
    node_bounds = np.unique(np.asarray(node_bounds, np.int64))
    seg_rows = s.node_first[node_bounds].astype(np.int64)
    nseg = len(seg_rows) - 1
    tri = np.zeros(nseg, np.int64)
    rl = np.zeros(nseg, np.int64)
    ru = np.zeros(nseg, np.int64)
    lr, ur = [], []
    for k in range(nseg):
        lo, hi = int(seg_rows[k]), int(seg_rows[k + 1])
        cl, cu = _split_counts(s, lo, hi)
        rl[k], ru[k] = int(cl.sum()), int(cu.sum())
        tri[k] = int(nl[lo:hi].sum() + nu[lo:hi].sum()) - rl[k] - ru[k]
        lr.append(balanced_ranges(cl, threads) + lo)
        ur.append(balanced_ranges(cu, threads) + lo)
    seq = tri < cfg.small_tri_threshold
    if bulk:
        seq[0] = False
    return SolvePartition(n, threads, seg_rows[1:-1].copy(), seg_rows, node_bounds, bulk, seq, tri,
                          rl, ru, lr, ur)


def device_launches(sym, part):
    """Launch lists of the device multi-RHS solve.  Per direction a list of
    (kind, seq, lo, hi, item offset, item count): kind 0 = rectangular block (items:
    row-range pairs, one warp each, entries with column < lo (forward) / >= hi
    (backward)), kind 1 = triangular level (items: nodes; entries with column in
    [lo, hi)); seq = 1: one warp walks all items in order.  Returns
    (fwd launches int64[k,6], bwd launches int64[k,6], items int32[*])."""
    s = sym
    items = []
    fwd, bwd = [], []

    def add(lst, kind, seq, lo, hi, arr):
        off = sum(len(a) for a in items)
        arr = np.asarray(arr, np.int32)
        items.append(arr)
        lst.append((kind, seq, lo, hi, off, len(arr) // (2 if kind == 0 else 1)))

    def rect(lst, ranges):
        pairs = [(int(ranges[t]), int(ranges[t + 1])) for t in range(len(ranges) - 1)
                 if ranges[t + 1] > ranges[t]]
        return np.asarray(pairs, np.int32).reshape(-1)

    for k in range(part.nsegments):
        lo, hi = int(part.seg_rows[k]), int(part.seg_rows[k + 1])
        u0, u1 = int(part.seg_nodes[k]), int(part.seg_nodes[k + 1])
        if part.rect_l_nnz[k]:
            add(fwd, 0, 0, lo, hi, rect(fwd, part.rect_l_ranges[k]))
        nodes = np.arange(u0, u1)
        if part.sequential[k]:
            add(fwd, 1, 1, lo, hi, nodes)
        else:
            lv = s.level[u0:u1]
            for L in np.unique(lv):
                add(fwd, 1, 0, lo, hi, nodes[lv == L])
    for k in range(part.nsegments - 1, -1, -1):
        lo, hi = int(part.seg_rows[k]), int(part.seg_rows[k + 1])
        u0, u1 = int(part.seg_nodes[k]), int(part.seg_nodes[k + 1])
        if part.rect_u_nnz[k]:
            add(bwd, 0, 0, lo, hi, rect(bwd, part.rect_u_ranges[k]))
        nodes = np.arange(u0, u1)
        if part.sequential[k]:
            add(bwd, 1, 1, lo, hi, nodes[::-1])
        else:
            lv = s.ulevel[u0:u1]
            for L in np.unique(lv):
                add(bwd, 1, 0, lo, hi, nodes[lv == L])
    it = np.concatenate(items).astype(np.int32) if items else np.zeros(0, np.int32)
    return (np.asarray(fwd, np.int64).reshape(-1, 6), np.asarray(bwd, np.int64).reshape(-1, 6), it)


def device_launches_levels(sym, long_row=64):
    """Launch lists (same format as ``device_launches``) of the level-scheduled
    multi-RHS substitution for supernodal factors: per forward level (``sym.level``)
    and backward level (``sym.ulevel``) one launch per node class — standalone rows
    with at most ``long_row`` off-diagonal entries in the direction (kind 1, warp per
    row), wider standalone rows (kind 3, CTA per row, entries split over 8 warps),
    supernodes (kind 4, CTA per supernode: off-block panel on DMMA, then the in-block
    triangle); lo / hi = [0, n) (every entry)."""
    s = sym
    n = s.n
    kind = np.asarray(s.node_kind)
    W = np.diff(s.colptr)
    items, fwd, bwd = [], [], []

    def add(lst, k, arr):
        if len(arr) == 0:
            return
        off = sum(len(a) for a in items)
        items.append(np.asarray(arr, np.int32))
        lst.append((k, 0, 0, n, off, len(arr)))

    for lst, lev_ptr, lev_nodes, fwd_dir in ((fwd, s.level_ptr, s.level_nodes, True),
                                           (bwd, s.ulevel_ptr, s.ulevel_nodes, False)):
        for lv in range(len(lev_ptr) - 1):
            nodes = np.asarray(lev_nodes[lev_ptr[lv]:lev_ptr[lv + 1]], np.int64)
            if not len(nodes):
                continue
            sn = kind[nodes] == 1
            width = np.asarray(s.nl)[nodes] if fwd_dir else W[nodes] - np.asarray(s.nl)[nodes] - 1
            wide = (~sn) & (width > long_row)
            add(lst, 1, nodes[(~sn) & ~wide])
            add(lst, 3, nodes[wide])
            add(lst, 4, nodes[sn])
    it = np.concatenate(items).astype(np.int32) if items else np.zeros(0, np.int32)
    return (np.asarray(fwd, np.int64).reshape(-1, 6), np.asarray(bwd, np.int64).reshape(-1, 6), it)


def solve_cpu(sym, F, part, Y, direction_both=True):
    """CPU interpreter of the device launch lists (test infrastructure helper for the
    coverage property): applies the forward then backward substitution to the
    columns of Y ([n, nrhs], already b-hat) in place and returns per-entry
    application counts (stored positions), so every entry can be checked to be
    applied exactly once."""
    s = sym
    fwd, bwd, items = device_launches(s, part)
    hits = np.zeros(len(F), np.int64)

    def row_apply(i, clo, chi, forward, finish):
        u = int(s.node_of[i])
        t = i - int(s.node_first[u])
        c0 = int(s.colptr[u])
        W = int(s.colptr[u + 1]) - c0
        d = int(s.nl[u]) + t
        base = int(s.valoff[u]) + t * W
        rng = range(0, d) if forward else range(d + 1, W)
        acc = Y[i].copy()
        for p in rng:
            c = int(s.cols[c0 + p])
            if clo <= c < chi:
                acc -= F[base + p] * Y[c]
                hits[base + p] += 1
        if finish and not forward:
            acc = acc / F[base + d]
            hits[base + d] += 1
        Y[i] = acc

    for lst, forward in ((fwd, True), (bwd, False)):
        for kind, seq, lo, hi, off, cnt in lst:
            if kind == 0:
                for q in range(cnt):
                    r0, r1 = int(items[off + 2 * q]), int(items[off + 2 * q + 1])
                    for i in range(r0, r1):
                        if forward:
                            row_apply(i, 0, lo, True, False)
                        else:
                            row_apply(i, hi, s.n, False, False)
            else:
                for q in range(cnt):
                    u = int(items[off + q])
                    r, e = int(s.node_first[u]), int(s.node_first[u + 1])
                    order = range(r, e) if forward else range(e - 1, r - 1, -1)
                    for i in order:
                        if forward:
                            row_apply(i, lo, hi, True, False)
                        else:
                            row_apply(i, lo, hi, False, True)
    return hits
