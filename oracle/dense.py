"""Dense oracles for the SPEC property tests — TEST INFRASTRUCTURE ONLY.

* ``dense_symbolic`` — SPEC.md:228: run dense elimination marking every touched
  position nonzero (no cancellation); gives the exact L/U patterns of M.
* ``reconstruct`` — assemble L (unit) and U from node-layout factors, with the
  row order P* (inner_perm ∘ static/ordering permutation), for SPEC.md:270/353.
* ``dense_solve`` — LAPACK partial-pivoting solve (numpy) for SPEC.md:354/597.
"""

from __future__ import annotations

import numpy as np


def m_dense(an, values=None):
    """Dense M = P·(Dr·A·Dc)·Q in M coordinates."""
    A = an.A
    vals = A.values if values is None else values
    n = A.n
    rows = np.repeat(np.arange(n), np.diff(A.row_ptr))
    inv_src = np.empty(n, np.int64)
    inv_src[an.vmap.mrow_src] = np.arange(n)
    M = np.zeros((n, n))
    M[inv_src[rows], an.ordering.inverse_perm[A.col_idx]] = vals * an.vmap.scale
    return M


def dense_symbolic(mask):
    """Boolean no-cancellation LU pattern of a square boolean mask (diagonal assumed)."""
    P = np.array(mask, dtype=bool)
    n = P.shape[0]
    for k in range(n):
        below = np.flatnonzero(P[k + 1:, k]) + k + 1
        right = np.flatnonzero(P[k, k + 1:]) + k + 1
        if len(below) and len(right):
            P[np.ix_(below, right)] = True
    return np.tril(P, -1), np.triu(P)


def dense_flops(L, U):
    n = L.shape[0]
    f = 0
    for k in range(n):
        lk = int(L[k + 1:, k].sum())
        uk = int(U[k, k + 1:].sum())
        f += 2 * lk * uk + lk
    return f


def factors_dense(an, values, inner_perm):
    """(Lunit, U, row_src) from node-layout values: factor row i holds M row row_src[i]."""
    s = an.symbolic
    n = s.n
    Ld = np.eye(n)
    Ud = np.zeros((n, n))
    row_src = np.arange(n)
    for u in range(s.nnodes):
        r = int(s.node_first[u])
        rows = int(s.node_first[u + 1]) - r
        c = s.node_cols(u)
        W = len(c)
        blk = values[s.valoff[u]:s.valoff[u] + rows * W].reshape(rows, W)
        for t in range(rows):
            i = r + t
            d = int(s.nl[u]) + t
            Ld[i, c[:d]] = blk[t, :d]
            Ud[i, c[d:]] = blk[t, d:]
            if s.node_kind[u] == 1:
                row_src[i] = r + int(inner_perm[i])
    return Ld, Ud, row_src


def dense_solve(A, b):
    return np.linalg.solve(A.to_dense(), b)
