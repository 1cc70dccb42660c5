"""Seeded synthetic inputs for the five BASELINE configs.

The reference publishes no fixture matrices (its paper benchmarks SuiteSparse,
absent here); these seeded generators stand in with the shapes, sizes and value
distributions BASELINE.json names.  Every generator takes a size parameter so
tests can run the same recipe at small scale.  Draw order is part of the recipe
and is documented per generator; all randomness is ``numpy.random.default_rng``.

Configs (BASELINE.json ``configs[0..4]``):

* c0 ``lap2d(64)``         2-D 5-point Laplacian, unsymmetric perturbation, AMD.
* c1 ``circuit(200000)``   power-law (Zipf 2.5) local couplings + dense-ish hubs, AMD.
* c2 ``convdiff3d(64)``    7-point convection-diffusion, upwind c=0.3, METIS ND.
* c3 ``fem27(48)``         27-point node graph x 3 dof, "dominant" block recipe
  (off-diagonal blocks -0.1*B, diagonal blocks B+81I, B=XᵀX/3),
  METIS ND.
* c4 ``circuit_batch``     c1 recipe at n=20000 with 3 hubs; per-instance value
  perturbation x(1+U[-0.2,0.2]) and diagonal reset to 1.1x row abs-sum.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
from numba import njit

from ._ref import SparseMatrixCSR

SEEDS = {"c0": 20240, "c1": 20241, "c2": 20242, "c3": 20243, "c4": 20244}


@dataclass
class Problem:
    name: str
    A: SparseMatrixCSR
    b: np.ndarray
    ordering: str = "amd"           # "amd" | "nd" | "natural"
    meta: dict = field(default_factory=dict)


@dataclass
class BatchProblem:
    name: str
    A0: SparseMatrixCSR             # instance 0 (analyzed once)
    values: np.ndarray              # [B, nnz] float64, same pattern as A0
    rhs: np.ndarray                 # [B, n]
    ordering: str = "amd"
    meta: dict = field(default_factory=dict)


def _csr(n, rows, cols, vals):
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    row_ptr = np.zeros(n + 1, dtype=np.int64)
    np.add.at(row_ptr[1:], rows, 1)
    np.cumsum(row_ptr, out=row_ptr)
    return row_ptr, cols.astype(np.int64), vals.astype(np.float64)


# --------------------------------------------------------------------------- c0
def lap2d(k=64, seed=SEEDS["c0"]):
    """2-D 5-point Laplacian on a k x k grid (Dirichlet truncation).

    Draw order: s~U[0,0.1] per row (diagonal 4+s), then u~U[-0.1,0.1] per
    stored off-diagonal in CSR order (value -(1+u)), then b~U[-1,1].
    """
    n = k * k
    rng = np.random.default_rng(seed)
    idx = np.arange(n)
    x, y = idx % k, idx // k
    rows, cols = [idx], [idx]
    for dx, dy in ((1, 0), (-1, 0), (0, 1), (0, -1)):
        ok = (x + dx >= 0) & (x + dx < k) & (y + dy >= 0) & (y + dy < k)
        rows.append(idx[ok])
        cols.append(idx[ok] + dx + k * dy)
    rows = np.concatenate(rows)
    cols = np.concatenate(cols)
    row_ptr, col_idx, _ = _csr(n, rows, cols, np.zeros(len(rows)))
    vals = np.empty(len(col_idx))
    diag = col_idx == np.repeat(idx, np.diff(row_ptr))
    s = rng.uniform(0.0, 0.1, n)
    u = rng.uniform(-0.1, 0.1, int((~diag).sum()))
    vals[diag] = 4.0 + s
    vals[~diag] = -(1.0 + u)
    b = rng.uniform(-1.0, 1.0, n)
    return Problem("c0_lap2d_%d" % k, SparseMatrixCSR(n, row_ptr, col_idx, vals), b, "amd",
                   {"k": k, "seed": seed})


# --------------------------------------------------------------------------- c1 / c4
@njit(cache=True)
def _dedupe_rows(n, cand, kwant):
    """Per row keep the first kwant[i] distinct candidates != i (in draw order)."""
    m = cand.shape[1]
    cnt = np.zeros(n, np.int64)
    out = np.empty((n, 6), np.int64)
    for i in range(n):
        c = 0
        for t in range(m):
            j = cand[i, t]
            if j == i:
                continue
            dup = False
            for q in range(c):
                if out[i, q] == j:
                    dup = True
                    break
            if dup:
                continue
            out[i, c] = j
            c += 1
            if c == kwant[i]:
                break
        cnt[i] = c
    return out, cnt


def circuit_pattern(n, n_hubs, hub_nnz, rng):
    """Row/col arrays of the circuit-like pattern (diagonal included).

    Per row: k~U{1..6}; 48 candidate draws d~Zipf(2.5) (capped at n-1), sign +-1
    (p=1/2), j=i+sign*d reflected at the borders; the first k distinct j != i are
    kept (a row keeps fewer if its 48 draws do not hold k distinct columns).
    Then n_hubs hub rows and n_hubs hub columns (distinct, uniform), each with
    hub_nnz uniform-random distinct partners.  Columns are local and heavy-tailed
    on purpose (uniform placement makes an expander graph).
    """
    m = 48
    kwant = rng.integers(1, 7, size=n)
    d = np.minimum(rng.zipf(2.5, size=(n, m)), n - 1)
    sign = np.where(rng.random((n, m)) < 0.5, -1, 1)
    j = np.arange(n)[:, None] + sign * d
    j = np.where(j < 0, -j, j)
    j = np.where(j >= n, 2 * (n - 1) - j, j)
    out, cnt = _dedupe_rows(n, j.astype(np.int64), kwant)
    keep = np.arange(6)[None, :] < cnt[:, None]
    rows = [np.repeat(np.arange(n), cnt), np.arange(n)]
    cols = [out[keep], np.arange(n)]
    hub_rows = rng.choice(n, n_hubs, replace=False)
    hub_cols = rng.choice(n, n_hubs, replace=False)
    for h in hub_rows:
        c = rng.choice(n, hub_nnz, replace=False)
        rows.append(np.full(hub_nnz, h))
        cols.append(c)
    for h in hub_cols:
        r = rng.choice(n, hub_nnz, replace=False)
        rows.append(r)
        cols.append(np.full(hub_nnz, h))
    rows = np.concatenate(rows).astype(np.int64)
    cols = np.concatenate(cols).astype(np.int64)
    key = np.unique(rows * n + cols)
    return key // n, key % n, {"hub_rows": hub_rows, "hub_cols": hub_cols}


def _dominant_diag(n, row_ptr, col_idx, offvals):
    """Insert diagonal = 1.1 x row abs-sum of the off-diagonals (1.0 if empty)."""
    rows = np.repeat(np.arange(n), np.diff(row_ptr))
    diag = col_idx == rows
    vals = np.empty(len(col_idx))
    vals[~diag] = offvals
    rs = np.bincount(rows[~diag], weights=np.abs(offvals), minlength=n)
    vals[diag] = np.where(rs > 0, 1.1 * rs, 1.0)
    return vals, diag


def circuit(n=200000, n_hubs=5, hub_nnz=2000, seed=SEEDS["c1"]):
    """c1: draw order = pattern (see circuit_pattern), off-diagonals U[-1,1] in CSR
    order, diagonal = 1.1 x row abs-sum, then b~U[-1,1]."""
    rng = np.random.default_rng(seed)
    rows, cols, hubs = circuit_pattern(n, n_hubs, hub_nnz, rng)
    row_ptr, col_idx, _ = _csr(n, rows, cols, np.zeros(len(rows)))
    ndiag = int((col_idx != np.repeat(np.arange(n), np.diff(row_ptr))).sum())
    off = rng.uniform(-1.0, 1.0, ndiag)
    vals, _ = _dominant_diag(n, row_ptr, col_idx, off)
    b = rng.uniform(-1.0, 1.0, n)
    return Problem("c1_circuit_%d" % n, SparseMatrixCSR(n, row_ptr, col_idx, vals), b, "amd",
                   {"n": n, "hubs": n_hubs, "hub_nnz": hub_nnz, "seed": seed})


class BatchValues:
    """Per-instance values/rhs of the c4 batch (pattern work done once).

    Instance b: rng = default_rng(seed + 1 + b); off-diagonals x (1+U[-0.2,0.2])
    (CSR order), diagonal reset to 1.1 x row abs-sum (1.0 for an empty row), then
    rhs~U[-1,1] from the same stream."""

    def __init__(self, A0, seed):
        n = A0.n
        self.n, self.nnz, self.seed = n, A0.nnz, seed
        rows = np.repeat(np.arange(n), np.diff(A0.row_ptr))
        self.diag = A0.col_idx == rows
        self.off_rows = rows[~self.diag]
        self.base_off = np.asarray(A0.values)[~self.diag]

    def instance(self, b, vals_out=None, rhs_out=None):
        rng = np.random.default_rng(self.seed + 1 + b)
        off = self.base_off * (1.0 + rng.uniform(-0.2, 0.2, len(self.base_off)))
        vals = np.empty(self.nnz) if vals_out is None else vals_out
        vals[~self.diag] = off
        rs = np.bincount(self.off_rows, weights=np.abs(off), minlength=self.n)
        vals[self.diag] = np.where(rs > 0, 1.1 * rs, 1.0)
        rhs = rng.uniform(-1.0, 1.0, self.n) if rhs_out is None else rhs_out
        if rhs_out is not None:
            rhs[:] = rng.uniform(-1.0, 1.0, self.n)
        return vals, rhs

    def fill(self, indices, vals, rhs, threads=8):
        """Generate instances ``indices`` into vals[len, nnz] / rhs[len, n] (threaded)."""
        from concurrent.futures import ThreadPoolExecutor
        idx = list(indices)

        def work(t):
            self.instance(idx[t], vals[t], rhs[t])

        with ThreadPoolExecutor(max(1, threads)) as ex:
            list(ex.map(work, range(len(idx))))


def circuit_batch(batch=4096, n=20000, n_hubs=3, hub_nnz=2000, seed=SEEDS["c4"], instances=None,
                  threads=8):
    """c4: base pattern/values = circuit(n, n_hubs, hub_nnz, seed); instance b per
    ``BatchValues``; ``A0`` carries instance 0's values (analyzed once).
    ``instances`` restricts generation to a subset of indices."""
    base = circuit(n, n_hubs, hub_nnz, seed)
    gen = BatchValues(base.A, seed)
    idx = list(range(batch)) if instances is None else list(instances)
    vals = np.empty((len(idx), base.A.nnz))
    rhs = np.empty((len(idx), n))
    gen.fill(idx, vals, rhs, threads)
    v0 = vals[idx.index(0)] if 0 in idx else gen.instance(0)[0]
    A0 = base.A.with_values(v0)
    return BatchProblem("c4_batch_%dx%d" % (len(idx), n), A0, vals, rhs, "amd",
                        {"n": n, "batch": batch, "instances": idx, "seed": seed, "gen": gen})


# --------------------------------------------------------------------------- c2
def convdiff3d(k=64, c=0.3, seed=SEEDS["c2"]):
    """c2: 7-point 3-D convection-diffusion on k^3 (x fastest), Dirichlet truncation.

    Diagonal 6, -1 per neighbour; d = normalize(N(0, I3)) (the only draw, then
    b~U[-1,1]); for each axis a: diagonal += c|d_a| and the upwind neighbour
    i - sign(d_a) e_a (if inside the grid) -= c|d_a|.  An M-matrix.
    """
    rng = np.random.default_rng(seed)
    d = rng.normal(size=3)
    d /= np.linalg.norm(d)
    n = k ** 3
    idx = np.arange(n)
    x, y, z = idx % k, (idx // k) % k, idx // (k * k)
    coord = (x, y, z)
    stride = (1, k, k * k)
    rows, cols, vals = [idx], [idx], [np.full(n, 6.0 + c * np.abs(d).sum())]
    for a in range(3):
        up = -int(np.sign(d[a])) if d[a] != 0 else 0
        for s in (1, -1):
            ok = (coord[a] + s >= 0) & (coord[a] + s < k)
            v = np.full(int(ok.sum()), -1.0)
            if s == up:
                v -= c * abs(d[a])
            rows.append(idx[ok])
            cols.append(idx[ok] + s * stride[a])
            vals.append(v)
    row_ptr, col_idx, values = _csr(n, np.concatenate(rows), np.concatenate(cols),
                                    np.concatenate(vals))
    b = rng.uniform(-1.0, 1.0, n)
    return Problem("c2_convdiff3d_%d" % k, SparseMatrixCSR(n, row_ptr, col_idx, values), b, "nd",
                   {"k": k, "c": c, "dir": d.tolist(), "seed": seed})


# --------------------------------------------------------------------------- c3
def fem27(k=48, dof=3, seed=SEEDS["c3"], recipe="dominant"):
    """c3: 27-point node stencil (incl. self) on k^3 nodes, dof x dof blocks.

    "Dominant" reading of the recipe (recorded in DESIGN.md):
    per stored node pair (p, q) in CSR order, X~N(0,1) dof x dof, B = XᵀX/3;
    block = B + 81 I if p == q else -0.1 B; then every entry x (1+U[-0.05,0.05])
    (all X drawn first, then all U, then b~U[-1,1]).
    ``recipe="literal"``: every block is XᵀX + 3I (BASELINE's text read literally),
    then the same ±5% perturbation — not diagonally dominant, so static pivoting
    moves most rows and the pivoted pattern is unsymmetric.
    """
    rng = np.random.default_rng(seed)
    nn = k ** 3
    idx = np.arange(nn)
    x, y, z = idx % k, (idx // k) % k, idx // (k * k)
    pr, pc = [], []
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                ok = ((x + dx >= 0) & (x + dx < k) & (y + dy >= 0) & (y + dy < k)
                      & (z + dz >= 0) & (z + dz < k))
                pr.append(idx[ok])
                pc.append(idx[ok] + dx + k * dy + k * k * dz)
    pr = np.concatenate(pr)
    pc = np.concatenate(pc)
    order = np.lexsort((pc, pr))
    pr, pc = pr[order], pc[order]
    nb = len(pr)
    X = rng.normal(size=(nb, dof, dof))
    self_ = pr == pc
    if recipe == "literal":
        B = np.einsum("bki,bkj->bij", X, X) + 3.0 * np.eye(dof)
    else:
        B = np.einsum("bki,bkj->bij", X, X) / 3.0
        B[~self_] *= -0.1
        B[self_] += 81.0 * np.eye(dof)
    B *= 1.0 + rng.uniform(-0.05, 0.05, size=B.shape)
    # expand blocks to CSR: row 3p+a has, for each neighbour q ascending, cols 3q+0..dof-1
    n = nn * dof
    cnt_node = np.bincount(pr, minlength=nn)
    node_ptr = np.zeros(nn + 1, np.int64)
    np.cumsum(cnt_node, out=node_ptr[1:])
    row_len = np.repeat(cnt_node * dof, dof)
    row_ptr = np.zeros(n + 1, np.int64)
    np.cumsum(row_len, out=row_ptr[1:])
    # entry order: for node p, for a in dof, for block t in p's blocks, for bcol in dof
    a = np.arange(dof)
    vals = np.empty(row_ptr[-1])
    cols = np.empty(row_ptr[-1], np.int64)
    blk_start = node_ptr[pr]                       # first block of p
    t_in = np.arange(nb) - blk_start               # block index within p's list
    for ai in range(dof):
        base = row_ptr[pr * dof + ai] + t_in * dof
        for bj in range(dof):
            cols[base + bj] = pc * dof + bj
            vals[base + bj] = B[:, ai, bj]
    del a
    b = rng.uniform(-1.0, 1.0, n)
    return Problem("c3_fem27_%dx%d" % (k, dof), SparseMatrixCSR(n, row_ptr, cols, vals), b, "nd",
                   {"k": k, "dof": dof, "seed": seed, "recipe": "dominant"})


# --------------------------------------------------------------------------- misc
def tridiag(n, seed=7):
    rng = np.random.default_rng(seed)
    idx = np.arange(n)
    rows = np.concatenate([idx, idx[1:], idx[:-1]])
    cols = np.concatenate([idx, idx[:-1], idx[1:]])
    row_ptr, col_idx, _ = _csr(n, rows, cols, np.zeros(len(rows)))
    vals = rng.uniform(-1, 1, len(col_idx))
    diag = col_idx == np.repeat(idx, np.diff(row_ptr))
    vals[diag] = 4.0
    return Problem("tridiag_%d" % n, SparseMatrixCSR(n, row_ptr, col_idx, vals),
                   rng.uniform(-1, 1, n), "amd")


def config(name, scale="full"):
    """Return the named BASELINE config.  ``scale='small'`` gives the same recipe at
    a size the CPU oracle finishes in well under a second (parity tests)."""
    small = scale == "small"
    if name == "c0":
        return lap2d(16 if small else 64)
    if name == "c1":
        return circuit(2000, 2, 200) if small else circuit()
    if name == "c2":
        return convdiff3d(10 if small else 64)
    if name == "c3":
        return fem27(5 if small else 48)
    if name == "c4":
        return circuit_batch(8, 2000, 2, 200) if small else circuit_batch()
    raise ValueError(name)


def zero_first_pivot(an, values):
    """Test helper ("new values placing 0 at a previously chosen pivot"):
    zero, in ``values`` (one instance of ``an``'s pattern, modified in place), the A
    entry that lands on the diagonal of the first factor row with an empty L row,
    off-diagonal U entries and a later row depending on it (so A stays nonsingular),
    making that row's pivot exactly 0 so perturbation fires.  Returns the A entry."""
    s = an.symbolic
    vm = an.vmap
    A = an.A
    used = np.zeros(s.nnodes, bool)
    used[s.deps] = True
    for i in range(s.n):
        u = int(s.node_of[i])
        if int(s.node_kind[u]) != 0 or int(s.nl[u]) != 0 or not used[u] or \
                int(s.colptr[u + 1] - s.colptr[u]) < 2:
            continue
        a = int(vm.mrow_src[i])
        for e in range(int(A.row_ptr[a]), int(A.row_ptr[a + 1])):
            if int(vm.colpos[e]) == 0:          # standalone row, no L: diagonal at position 0
                values[e] = 0.0
                return e
    raise ValueError("no standalone row with an empty L row")
