"""Host preprocessing: static pivoting, fill-reducing ordering, and the permuted
pattern M = P·(Dr·A·Dc)·Q that symbolic factorization and the device consume.

Static pivoting and AMD are the reference's own shipped code
(``polylu._matching.max_weight_match`` at ``_matching.py:169``,
``polylu._amd.amd_permutation`` at ``_amd.py:334``); this module only wraps them in
the SPEC types ``PivotScale`` / ``Ordering`` (``SPEC.md:127-137``) and the SPEC
operations ``static_pivot`` (``SPEC.md:155``) and ``amd_order`` (``SPEC.md:165``).
Nested dissection (configs c2/c3) is outside the reference (``SPEC.md:12,235``):
``nd_order`` calls METIS_NodeND from the CUDA toolkit through a C shim and is fed
to the pipeline as a user permutation (``config.py:46-47,69-77``).

Conventions (shared by symbolic, oracle and device):
  * ``row_perm[j]`` = original row matched to column j (``_matching.py:172``).
  * ``perm[k]`` = index placed at position k (``_amd.py:337-338``).
  * M[i, k] = dr[a]·A[a, c]·dc[c] with a = row_perm[perm[i]], c = perm[k].
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _ref
from ._ref import errors

_LIBDIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib")


@dataclass(frozen=True)
class PivotScale:
    """SPEC.md:127-132."""
    row_perm: np.ndarray   # int64[n]
    dr: np.ndarray         # float64[n], indexed by original row
    dc: np.ndarray         # float64[n], indexed by original column


@dataclass(frozen=True)
class Ordering:
    """SPEC.md:134-137."""
    perm: np.ndarray
    inverse_perm: np.ndarray


def static_pivot(A):
    """reference ``max_weight_match`` (``_matching.py:169-209``)."""
    row_perm, dr, dc, unmatched = _ref.matching.max_weight_match(A.n, A.row_ptr, A.col_idx, A.values)
    if len(unmatched):
        raise errors.StructurallySingular(unmatched.tolist())
    return PivotScale(np.asarray(row_perm, np.int64), np.asarray(dr), np.asarray(dc))


def pivoted_sym_pattern(A, ps):
    """Strictly off-diagonal structural pattern of |PA| + |PA|ᵀ.

    Built structurally so explicitly stored zeros stay in the pattern.
    Returns CSR (ap, ai) with ascending columns."""
    n = A.n
    inv_rp = np.empty(n, np.int64)
    inv_rp[ps.row_perm] = np.arange(n)
    rows = np.repeat(inv_rp, np.diff(A.row_ptr))     # PA row of each entry
    cols = A.col_idx
    off = rows != cols
    r = np.concatenate([rows[off], cols[off]])
    c = np.concatenate([cols[off], rows[off]])
    key = np.unique(r * n + c)
    r, c = key // n, key % n
    ap = np.zeros(n + 1, np.int64)
    np.add.at(ap[1:], r, 1)
    np.cumsum(ap, out=ap)
    return ap, c.astype(np.int64)


def amd_order(ap, ai):
    """reference ``amd_permutation`` (``_amd.py:334-373``)."""
    n = len(ap) - 1
    perm = _ref.amd.amd_permutation(n, ap, ai)
    return _ordering(perm)


def _ordering(perm):
    perm = np.asarray(perm, np.int64)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    return Ordering(perm, inv)


def _metis_lib():
    path = os.path.join(_LIBDIR, "libhymetis.so")
    if not os.path.exists(path):
        from . import build as _build
        _build.build_metis()
    lib = ctypes.CDLL(path)
    p = ctypes.POINTER(ctypes.c_int64)
    lib.hy_metis_nodend.argtypes = [ctypes.c_int64, p, p, p, p]
    lib.hy_metis_nodend.restype = ctypes.c_int
    return lib


def nd_order(ap, ai):
    """METIS_NodeND (default options) on the symmetric off-diagonal pattern.

    Not in the reference; its output is pinned by caching/passing the same array to
    oracle and device."""
    n = len(ap) - 1
    xadj = np.ascontiguousarray(ap, np.int64).copy()
    adj = np.ascontiguousarray(ai, np.int64).copy()
    perm = np.empty(n, np.int64)
    iperm = np.empty(n, np.int64)
    p = ctypes.POINTER(ctypes.c_int64)
    st = _metis_lib().hy_metis_nodend(n, xadj.ctypes.data_as(p), adj.ctypes.data_as(p),
                                      perm.ctypes.data_as(p), iperm.ctypes.data_as(p))
    if st != 1:
        raise RuntimeError("METIS_NodeND failed with status %d" % st)
    return _ordering(perm)


def resolve_ordering(A, ps, cfg):
    """Apply ``SolverConfig.ordering`` (``config.py:69-77``): 'amd' | 'natural' | user
    permutation; additionally 'nd' (METIS) for the c2/c3 configs."""
    if isinstance(cfg.ordering, str) and cfg.ordering.lower() == "nd":
        ap, ai = pivoted_sym_pattern(A, ps)
        return nd_order(ap, ai)
    kind, perm = cfg.resolve_ordering_spec()
    if kind == "natural":
        return _ordering(np.arange(A.n))
    if kind == "user":
        if perm.shape != (A.n,) or not np.array_equal(np.sort(perm), np.arange(A.n)):
            raise errors.DimensionMismatch("user ordering is not a permutation of [0, n)")
        return _ordering(perm)
    ap, ai = pivoted_sym_pattern(A, ps)
    return amd_order(ap, ai)


def permuted_rows(A, ps, order):
    """Maps for M = P·(Dr·A·Dc)·Q.

    Returns (mrow_src, mcol_of, scale) where M row i is original row
    ``mrow_src[i] = row_perm[perm[i]]``, original column c lands at M column
    ``mcol_of[c] = inverse_perm[c]``, and ``scale[e] = dr[row(e)]·dc[col(e)]`` per A entry."""
    mrow_src = ps.row_perm[order.perm]
    mcol_of = order.inverse_perm
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    scale = ps.dr[rows] * ps.dc[A.col_idx]
    return mrow_src, mcol_of, scale


def m_pattern(A, ps, order):
    """CSR pattern of M (rows in M order, columns ascending in M indices), int64.

    Also returns ``src_entry[t]``: the A entry index that M-pattern slot t came from."""
    n = A.n
    mrow_src, mcol_of, _ = permuted_rows(A, ps, order)
    lens = np.diff(A.row_ptr)[mrow_src]
    mp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=mp[1:])
    # gather A entries row by row in M order
    starts = A.row_ptr[mrow_src]
    ent = np.repeat(starts - mp[:-1], lens) + np.arange(mp[-1])
    cols = mcol_of[A.col_idx[ent]]
    rows = np.repeat(np.arange(n), lens)
    o = np.lexsort((cols, rows))
    return mp, cols[o].astype(np.int64), ent[o].astype(np.int64)
