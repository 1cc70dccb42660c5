"""``analyze`` = static_pivot → ordering → symbolic_factorize.

``analyze`` is not a reference name; it is the composition of the
three SPEC preprocessing operations and returns the SPEC types plus the value map
the device needs to scatter A into factor storage.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
from numba import njit

from . import preprocess as pp
from ._ref import SolverConfig, errors
from .symbolic import SymbolicStructure, symbolic_from_pattern


@dataclass
class ValueMap:
    """Where each A entry lands in node storage (identity inner permutation).

    M row i takes A row ``mrow_src[i]``; the entries of that row, in A's CSR order,
    go to column position ``colpos[e]`` of the node owning row i, scaled by
    ``scale[e] = dr[a]·dc[c]``.  Indexed by the A entry e."""
    mrow_src: np.ndarray   # int64[n]
    colpos: np.ndarray     # int32[nnz]
    scale: np.ndarray      # float64[nnz]


@dataclass
class Analysis:
    A: object
    pivot_scale: pp.PivotScale
    ordering: pp.Ordering
    symbolic: SymbolicStructure
    vmap: ValueMap
    config: SolverConfig
    times: dict


@njit(cache=True)
def _colpos(n, a_ptr, a_col, mrow_src, mcol_of, node_of, colptr, cols):
    """Binary-search each A entry's M column in its node's column list."""
    out = np.empty(a_ptr[n], np.int32)
    for i in range(n):
        a = mrow_src[i]
        u = node_of[i]
        lo0 = colptr[u]
        hi0 = colptr[u + 1]
        for e in range(a_ptr[a], a_ptr[a + 1]):
            k = mcol_of[a_col[e]]
            lo = lo0
            hi = hi0
            while lo < hi:
                mid = (lo + hi) >> 1
                if cols[mid] < k:
                    lo = mid + 1
                else:
                    hi = mid
            if lo >= hi0 or cols[lo] != k:
                return out, e
            out[e] = lo - lo0
    return out, -1


def value_map(A, ps, order, sym):
    mrow_src, mcol_of, scale = pp.permuted_rows(A, ps, order)
    colpos, bad = _colpos(A.n, A.row_ptr, A.col_idx, mrow_src, mcol_of, sym.node_of,
                          sym.colptr, sym.cols)
    if bad >= 0:
        raise errors.CycleDetected("internal: A entry %d missing from symbolic pattern" % bad)
    return ValueMap(mrow_src, colpos, scale)


def analyze(A, config=None, kernel_override=None, threads=1, symbolic_method="auto"):
    """static_pivot → ordering (amd | natural | user perm | 'nd') → symbolic."""
    import time
    cfg = config or SolverConfig()
    t = {}
    t0 = time.perf_counter()
    ps = pp.static_pivot(A)
    t["static_pivot"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    order = pp.resolve_ordering(A, ps, cfg)
    t["ordering"] = time.perf_counter() - t0
    t0 = time.perf_counter()
    mp, mc, _ = pp.m_pattern(A, ps, order)
    sym = symbolic_from_pattern(A.n, mp, mc, cfg, kernel_override, threads, symbolic_method)
    vm = value_map(A, ps, order, sym)
    t["symbolic"] = time.perf_counter() - t0
    return Analysis(A, ps, order, sym, vm, cfg, t)
