"""Host-built device schedules ("row programs") — uploaded once, shared by every
instance of a batch and by every refactorization.

Up-looking row i applies, for each L position p in ascending
order, the source row j = cols[p]: l = w[p] / U(j,j); w[pos(k)] -= l·U(j,k).  The
program of a factor row lists only the *structurally nonzero* steps (L positions
reached by A's pattern or by an earlier step — union padding inside supernodes
and never-filled positions have l = 0 exactly and are skipped, which leaves every
stored value unchanged) together with the target positions ``rel`` of every
U(j, >j) entry, so the device never searches column lists.

Rows with many steps (circuit hub rows: 7k–27k L entries, but only ~80–90
dependency levels inside the row) get a *pull* program instead: positions are
grouped by intra-row level, and each position gathers its contributions
w[p] = m[p] − Σ_s l_s·U_s(col p) in ascending step order (the same operation
order as the sequential push loop), so a whole CTA works on one row.

Supernode rows use the fixed pivot order of a prior factorization (refactorize
semantics), so programs are built per prior ``inner_perm``.
"""

from __future__ import annotations

from dataclasses import dataclass

import os

import numba
import numpy as np
from numba import njit, prange

HUB_STEPS = 384


@njit(cache=True)
def _programs(n, first, kind, colptr, cols, nl, valoff, node_of, a_ptr, mrow_src, colpos, iperm,
              hub_steps, standalone_only):
    nn = len(kind)
    # upper bounds for allocation: steps <= sum of L widths incl. in-block parts
    max_steps = 0
    for u in range(nn):
        s = first[u + 1] - first[u]
        max_steps += s * nl[u] + s * (s - 1) // 2
    st_p = np.empty(max_steps, np.int32)
    st_j = np.empty(max_steps, np.int32)
    st_src = np.empty(max_steps, np.int64)
    st_cnt = np.empty(max_steps, np.int32)
    st_rel = np.empty(max_steps, np.int64)
    row_ptr = np.zeros(n + 1, np.int64)
    cap_rel = 1 << 20
    rel = np.empty(cap_rel, np.int32)
    nrel = 0
    nst = 0
    pos_of = np.full(n, -1, np.int64)
    nz = np.zeros(1, np.uint8)
    maxW = 0
    for u in range(nn):
        maxW = max(maxW, colptr[u + 1] - colptr[u])
    nz = np.zeros(maxW, np.uint8)
    node_hub = np.zeros(nn, np.uint8)
    for u in range(nn):
        r = first[u]
        s = first[u + 1] - r
        c0 = colptr[u]
        W = colptr[u + 1] - c0
        L = nl[u]
        for q in range(W):
            pos_of[cols[c0 + q]] = q
        for t in range(s):
            i = r + t
            nz[:W] = 0
            src_row = r + iperm[i] if kind[u] == 1 else r
            a = mrow_src[src_row]
            for e in range(a_ptr[a], a_ptr[a + 1]):
                nz[colpos[e]] = 1
            Lt = L + t
            for p in range(Lt):
                if nz[p] == 0:
                    continue
                j = cols[c0 + p]
                v = node_of[j]
                tj = j - first[v]
                vc0 = colptr[v]
                vW = colptr[v + 1] - vc0
                sd = nl[v] + tj
                cnt = vW - sd - 1
                if nrel + cnt > cap_rel:
                    cap_rel = max(2 * cap_rel, nrel + cnt)
                    tmp = np.empty(cap_rel, np.int32)
                    tmp[:nrel] = rel[:nrel]
                    rel = tmp
                st_p[nst] = p
                st_j[nst] = j
                st_src[nst] = valoff[v] + tj * vW + sd
                st_cnt[nst] = cnt
                st_rel[nst] = nrel
                for q in range(sd + 1, vW):
                    tp = pos_of[cols[vc0 + q]]
                    rel[nrel] = tp
                    nz[tp] = 1
                    nrel += 1
                nst += 1
            row_ptr[i + 1] = nst
            if row_ptr[i + 1] - row_ptr[i] > hub_steps and (kind[u] == 0 or not standalone_only):
                node_hub[u] = 1
        for q in range(W):
            pos_of[cols[c0 + q]] = -1
    return (row_ptr, st_p[:nst].copy(), st_j[:nst].copy(), st_src[:nst].copy(),
            st_cnt[:nst].copy(), st_rel[:nst].copy(), rel[:nrel].copy(), node_hub)


@njit(cache=True)
def _pull(n, first, colptr, nl, valoff, a_ptr, mrow_src, colpos, kind, iperm, hub_nodes, row_ptr,
          st_p, st_src, st_cnt, st_rel, rel):
    """Pull programs for every row of the hub nodes.

    Per hub row (in node order): positions grouped by intra-row level; per position
    its contributions (multiplier position, U value offset) in ascending step order
    and its kind: >=0 → L position (divide by the value at that offset),
    -1 → U position, -2 → pivot."""
    nrows = 0
    for k in range(len(hub_nodes)):
        u = hub_nodes[k]
        nrows += first[u + 1] - first[u]
    hrow_lev = np.zeros(nrows + 1, np.int64)      # offsets into lev_ptr
    lev_ptr_l = [np.int64(0)]
    pos_l = []
    div_l = []
    pp_l = [np.int64(0)]
    pred_p_l = []
    pred_u_l = []
    hr = 0
    nlev_tot = 0
    for k in range(len(hub_nodes)):
        u = hub_nodes[k]
        r = first[u]
        s = first[u + 1] - r
        W = colptr[u + 1] - colptr[u]
        L = nl[u]
        for t in range(s):
            i = r + t
            Lt = L + t
            level = np.full(W, -1, np.int64)
            npred = np.zeros(W, np.int64)
            step_at = np.full(W, -1, np.int64)
            src_row = r + iperm[i] if kind[u] == 1 else r
            a = mrow_src[src_row]
            for e in range(a_ptr[a], a_ptr[a + 1]):
                level[colpos[e]] = 0
            for st in range(row_ptr[i], row_ptr[i + 1]):
                p = st_p[st]
                step_at[p] = st
                lp = level[p]
                for q in range(st_cnt[st]):
                    tp = rel[st_rel[st] + q]
                    npred[tp] += 1
                    if lp + 1 > level[tp]:
                        level[tp] = lp + 1
            maxl = level.max()
            # positions by level (structurally nonzero ones only)
            cnt = np.zeros(maxl + 2, np.int64)
            for p in range(W):
                if level[p] >= 0:
                    cnt[level[p] + 1] += 1
            for l in range(maxl + 1):
                cnt[l + 1] += cnt[l]
            order = np.empty(cnt[maxl + 1], np.int64)
            fillp = cnt[:maxl + 1].copy()
            for p in range(W):
                if level[p] >= 0:
                    order[fillp[level[p]]] = p
                    fillp[level[p]] += 1
            # pred lists per position (ascending step order)
            pstart = np.zeros(W + 1, np.int64)
            for p in range(W):
                pstart[p + 1] = pstart[p] + npred[p]
            pp = np.empty(pstart[W], np.int32)
            pu = np.empty(pstart[W], np.int64)
            fill2 = pstart[:W].copy()
            for st in range(row_ptr[i], row_ptr[i + 1]):
                p = st_p[st]
                for q in range(st_cnt[st]):
                    tp = rel[st_rel[st] + q]
                    pp[fill2[tp]] = p
                    pu[fill2[tp]] = st_src[st] + 1 + q
                    fill2[tp] += 1
            for l in range(maxl + 1):
                lev_ptr_l.append(lev_ptr_l[-1] + (cnt[l + 1] - cnt[l]))
            nlev_tot += maxl + 1
            hrow_lev[hr + 1] = nlev_tot
            for x in range(len(order)):
                p = order[x]
                pos_l.append(np.int32(p))
                if p < Lt:
                    div_l.append(st_src[step_at[p]])
                elif p == Lt:
                    div_l.append(np.int64(-2))
                else:
                    div_l.append(np.int64(-1))
                for y in range(pstart[p], pstart[p + 1]):
                    pred_p_l.append(pp[y])
                    pred_u_l.append(pu[y])
                pp_l.append(pp_l[-1] + (pstart[p + 1] - pstart[p]))
            hr += 1
    lev_ptr = np.empty(len(lev_ptr_l), np.int64)
    for x in range(len(lev_ptr_l)):
        lev_ptr[x] = lev_ptr_l[x]
    hpos = np.empty(len(pos_l), np.int32)
    hdiv = np.empty(len(div_l), np.int64)
    for x in range(len(pos_l)):
        hpos[x] = pos_l[x]
        hdiv[x] = div_l[x]
    hpp = np.empty(len(pp_l), np.int64)
    for x in range(len(pp_l)):
        hpp[x] = pp_l[x]
    pred_p = np.empty(len(pred_p_l), np.int32)
    pred_u = np.empty(len(pred_u_l), np.int64)
    for x in range(len(pred_p_l)):
        pred_p[x] = pred_p_l[x]
        pred_u[x] = pred_u_l[x]
    return hrow_lev, lev_ptr, hpos, hdiv, hpp, pred_p, pred_u


@njit(cache=True)
def _chunks(hrow_lev, lev_ptr, hpp, ch):
    """Per intra-row level, split the gather work into items of <= ch contributions.

    Work item: (position x, pred range [y0, y1), slot); slot = -1 → the item holds the
    whole position (finalize directly); slot >= 0 → partial sum into scratch slot.
    Split positions: (x, first slot, slot count), combined in slot order."""
    nlev = len(lev_ptr) - 1
    wi_x_l = []
    wi_y0_l = []
    wi_y1_l = []
    wi_slot_l = []
    sp_x_l = []
    sp_s0_l = []
    sp_n_l = []
    lev_wi = np.zeros(nlev + 1, np.int64)
    lev_sp = np.zeros(nlev + 1, np.int64)
    max_slots = 0
    for lev in range(nlev):
        slot = 0
        for x in range(lev_ptr[lev], lev_ptr[lev + 1]):
            y0 = hpp[x]
            y1 = hpp[x + 1]
            if y1 - y0 <= ch:
                wi_x_l.append(np.int32(x))
                wi_y0_l.append(y0)
                wi_y1_l.append(y1)
                wi_slot_l.append(np.int32(-1))
            else:
                nsl = 0
                y = y0
                while y < y1:
                    wi_x_l.append(np.int32(x))
                    wi_y0_l.append(y)
                    wi_y1_l.append(min(y + ch, y1))
                    wi_slot_l.append(np.int32(slot + nsl))
                    nsl += 1
                    y += ch
                sp_x_l.append(np.int32(x))
                sp_s0_l.append(np.int32(slot))
                sp_n_l.append(np.int32(nsl))
                slot += nsl
        max_slots = max(max_slots, slot)
        lev_wi[lev + 1] = len(wi_x_l)
        lev_sp[lev + 1] = len(sp_x_l)
    nwi = len(wi_x_l)
    wi_x = np.empty(nwi, np.int32)
    wi_y0 = np.empty(nwi, np.int64)
    wi_y1 = np.empty(nwi, np.int64)
    wi_slot = np.empty(nwi, np.int32)
    for k in range(nwi):
        wi_x[k] = wi_x_l[k]
        wi_y0[k] = wi_y0_l[k]
        wi_y1[k] = wi_y1_l[k]
        wi_slot[k] = wi_slot_l[k]
    nsp = len(sp_x_l)
    sp_x = np.empty(nsp, np.int32)
    sp_s0 = np.empty(nsp, np.int32)
    sp_n = np.empty(nsp, np.int32)
    for k in range(nsp):
        sp_x[k] = sp_x_l[k]
        sp_s0[k] = sp_s0_l[k]
        sp_n[k] = sp_n_l[k]
    return lev_wi, wi_x, wi_y0, wi_y1, wi_slot, lev_sp, sp_x, sp_s0, sp_n, max_slots


HUB_LPT = os.environ.get("HYLU_HUB_LPT", "1") != "0"   # probe switch: work items in generation order


def _balance_items(hrow_lev, lev_wi, wi_x, wi_y0, wi_y1, wi_slot):
    """Work items of an intra-row level in longest-first order (by gather rounds of 8 terms):
    the hub kernel's warps claim a level's items one by one, so the order is its schedule
    (longest-processing-time first).  The item holding a level's lowest pred offset stays
    first and, in the last level of a hub row, the one holding the highest stays last: the
    kernel takes a level's pred range from them.  Items are independent within a level (split
    positions combine by slot), so the order changes no result."""
    last_levels = set(int(v) - 1 for v in hrow_lev[1:])
    perm = np.arange(len(wi_x))
    for lev in range(len(lev_wi) - 1):
        a, b = int(lev_wi[lev]), int(lev_wi[lev + 1])
        hi = b - 1 if lev in last_levels else b
        if hi - (a + 1) < 2:
            continue
        rounds = (wi_y1[a + 1:hi] - wi_y0[a + 1:hi] + 7) // 8
        perm[a + 1:hi] = a + 1 + np.argsort(-rounds, kind="stable")
    return wi_x[perm], wi_y0[perm], wi_y1[perm], wi_slot[perm]


JOINT_HUB_ROWS = os.environ.get("HYLU_JOINT_HUB", "1") != "0"


def _joint_hub_rows(hub_nodes, first, colptr, valoff, hrow_lev, lev_ptr, hpos, hdiv, hpp, pred_p,
                    pred_u, merge=True):
    """Merge the per-row pull programs of each hub supernode into one program.

    Row t's levels below its first *cross level* (the first level with a
    contribution or divisor taken from an earlier row of the same node) depend on
    no other row of the node, so level q of all such rows runs as one joint level;
    the remaining levels of each row follow row by row.  Positions (and multiplier
    positions) become node-relative, t*W + p, so one level can span rows.  The whole
    node program is attached to the node's first hub row (the other rows get empty
    level ranges); every row is initialised before the node's first level runs.
    Contribution order per position is unchanged, so the arithmetic is identical.
    merge=False keeps the row-by-row level order (same node-relative form)."""
    n_lev = [0]
    pos, div, pp, pu, hppn = [], [], [], [], [0]
    new_hrow = [0]
    hr = 0
    for u in hub_nodes:
        r, s = int(first[u]), int(first[u + 1] - first[u])
        W = int(colptr[u + 1] - colptr[u])
        lo, hi = int(valoff[u]), int(valoff[u + 1])
        levs = [list(range(int(hrow_lev[hr + t]), int(hrow_lev[hr + t + 1]))) for t in range(s)]
        cut = []
        for t in range(s):
            c = len(levs[t])
            if t > 0:
                for q, l in enumerate(levs[t]):
                    x0, x1 = int(lev_ptr[l]), int(lev_ptr[l + 1])
                    d = hdiv[x0:x1]
                    u_ = pred_u[hpp[x0]:hpp[x1]]
                    if ((d >= lo) & (d < hi)).any() or ((u_ >= lo) & (u_ < hi)).any():
                        c = q
                        break
            cut.append(c if merge else (len(levs[t]) if t == 0 else 0))
        virt = []
        for q in range(max(cut) if cut else 0):
            seg = [(t, levs[t][q]) for t in range(s) if q < cut[t]]
            if seg:
                virt.append(seg)
        for t in range(s):
            for q in range(cut[t], len(levs[t])):
                virt.append([(t, levs[t][q])])
        for seg in virt:
            cnt = 0
            for t, l in seg:
                x0, x1 = int(lev_ptr[l]), int(lev_ptr[l + 1])
                pos.append(hpos[x0:x1].astype(np.int64) + t * W)
                div.append(hdiv[x0:x1])
                y0, y1 = int(hpp[x0]), int(hpp[x1])
                pp.append(pred_p[y0:y1].astype(np.int64) + t * W)
                pu.append(pred_u[y0:y1])
                hppn.append(np.diff(hpp[x0:x1 + 1]))
                cnt += x1 - x0
            n_lev.append(n_lev[-1] + cnt)
        new_hrow.append(new_hrow[-1] + len(virt))
        new_hrow.extend([new_hrow[-1]] * (s - 1))
        hr += s
    cat = lambda xs, dt: np.concatenate(xs).astype(dt) if xs else np.zeros(0, dt)
    hpp_new = np.concatenate([[0], np.cumsum(cat(hppn[1:], np.int64))]).astype(np.int64)
    return (np.asarray(new_hrow, np.int64), np.asarray(n_lev, np.int64), cat(pos, np.int32),
            cat(div, np.int64), hpp_new, cat(pp, np.int32), cat(pu, np.int64))


@dataclass
class RowPrograms:
    row_ptr: np.ndarray     # int64[n+1] steps of factor row i
    st_p: np.ndarray        # int32 multiplier position in the target row
    st_j: np.ndarray        # int32 source row (forward-solve coupling)
    st_src: np.ndarray      # int64 offset of U(j,j) in node storage
    st_cnt: np.ndarray      # int32 number of U(j,>j) entries
    st_rel: np.ndarray      # int64 offset into rel
    rel: np.ndarray         # int32 target positions of U(j,>j) entries
    node_hub: np.ndarray    # uint8[nn]
    hub_nodes: np.ndarray   # int32
    hrow_lev: np.ndarray    # int64[nhubrows+1] -> lev_ptr index
    lev_ptr: np.ndarray     # int64 -> hpos index
    hpos: np.ndarray        # int32 positions in level order
    hdiv: np.ndarray        # int64 per position: diag offset (L), -1 (U), -2 (pivot)
    hpp: np.ndarray         # int64[len(hpos)+1] -> pred index
    pred_p: np.ndarray      # int32
    pred_u: np.ndarray      # int64
    lev_wi: np.ndarray      # int64[nlev+1] work items per intra-row level
    wi_p: np.ndarray        # int32 target position of the work item
    wi_kd: np.ndarray       # int64 finalize kind (hdiv of the position)
    wi_y0: np.ndarray       # int64
    wi_y1: np.ndarray       # int64
    wi_slot: np.ndarray     # int32 (-1 = whole position)
    lev_sp: np.ndarray      # int64[nlev+1] split positions per level
    sp_p: np.ndarray        # int32
    sp_kd: np.ndarray       # int64
    sp_s0: np.ndarray       # int32
    sp_n: np.ndarray        # int32
    max_slots: int
    level_ws: np.ndarray    # int32[nlevels] max width of non-hub nodes per factor level
    node_rec: np.ndarray    # int64[nn, 4]: valoff, dep0, (first | rows<<32), (W | L<<32)
    row_rec: np.ndarray     # int64[n, 4]: step0, a_e0, (nsteps | k<<32), a (original row)

    @property
    def nsteps(self):
        return len(self.st_p)

    def nbytes(self):
        return sum(getattr(self, k).nbytes for k in self.__dataclass_fields__
                   if isinstance(getattr(self, k), np.ndarray))


HUB_CHUNK = int(os.environ.get("HYLU_HUB_CHUNK", "64"))


def build_programs(an, inner_perm, hub_steps=HUB_STEPS, chunk=HUB_CHUNK, standalone_only=False):
    s = an.symbolic
    vm = an.vmap
    ip = np.ascontiguousarray(inner_perm, np.int64)
    (row_ptr, st_p, st_j, st_src, st_cnt, st_rel, rel, node_hub) = _programs(
        s.n, s.node_first, s.node_kind, s.colptr, s.cols, s.nl, s.valoff, s.node_of,
        an.A.row_ptr, vm.mrow_src, vm.colpos, ip, hub_steps, standalone_only)
    hub_nodes = np.flatnonzero(node_hub).astype(np.int32)
    if len(hub_nodes):
        hrow_lev, lev_ptr, hpos, hdiv, hpp, pred_p, pred_u = _pull(
            s.n, s.node_first, s.colptr, s.nl, s.valoff, an.A.row_ptr, vm.mrow_src, vm.colpos,
            s.node_kind, ip, hub_nodes.astype(np.int64), row_ptr, st_p, st_src, st_cnt, st_rel, rel)
        hrow_lev, lev_ptr, hpos, hdiv, hpp, pred_p, pred_u = _joint_hub_rows(
            hub_nodes, s.node_first, s.colptr, s.valoff, hrow_lev, lev_ptr, hpos, hdiv, hpp,
            pred_p, pred_u, JOINT_HUB_ROWS)
    else:
        hrow_lev = np.zeros(1, np.int64)
        lev_ptr = np.zeros(1, np.int64)
        hpos = np.zeros(0, np.int32)
        hdiv = np.zeros(0, np.int64)
        hpp = np.zeros(1, np.int64)
        pred_p = np.zeros(0, np.int32)
        pred_u = np.zeros(0, np.int64)
    (lev_wi, wi_x, wi_y0, wi_y1, wi_slot, lev_sp, sp_x, sp_s0, sp_n,
     max_slots) = _chunks(hrow_lev, lev_ptr, hpp, chunk)
    if HUB_LPT:
        wi_x, wi_y0, wi_y1, wi_slot = _balance_items(hrow_lev, lev_wi, wi_x, wi_y0, wi_y1, wi_slot)
    W = np.diff(s.colptr)
    rows = np.diff(s.node_first)
    ndeps = np.diff(s.dep_ptr)
    node_rec = np.zeros((s.nnodes, 4), np.int64)
    node_rec[:, 0] = s.valoff[:-1]
    node_rec[:, 1] = s.dep_ptr[:-1]
    node_rec[:, 2] = s.node_first[:-1] | (rows.astype(np.int64) << 32)
    node_rec[:, 3] = W | (s.nl.astype(np.int64) << 32)
    del ndeps
    # row records: physical row i of node u holds M row (first + iperm[i]) in supernodes
    first_of = s.node_first[s.node_of]
    src = np.where(s.node_kind[s.node_of] == 1, first_of + ip, np.arange(s.n))
    a = vm.mrow_src[src]
    row_rec = np.zeros((s.n, 4), np.int64)
    row_rec[:, 0] = row_ptr[:-1]
    row_rec[:, 1] = an.A.row_ptr[a]
    k = an.A.row_ptr[a + 1] - an.A.row_ptr[a]
    row_rec[:, 2] = (row_ptr[1:] - row_ptr[:-1]) | (k.astype(np.int64) << 32)
    row_rec[:, 3] = a
    level_ws = np.zeros(len(s.level_ptr) - 1, np.int32)
    for lv in range(len(level_ws)):
        nodes = s.level_nodes[s.level_ptr[lv]:s.level_ptr[lv + 1]]
        nodes = nodes[node_hub[nodes] == 0]
        level_ws[lv] = int(W[nodes].max()) if len(nodes) else 0
    return RowPrograms(row_ptr, st_p, st_j, st_src, st_cnt, st_rel, rel, node_hub, hub_nodes,
                       hrow_lev, lev_ptr, hpos, hdiv, hpp, pred_p, pred_u, lev_wi,
                       hpos[wi_x].astype(np.int32), hdiv[wi_x].astype(np.int64), wi_y0, wi_y1, wi_slot,
                       lev_sp, hpos[sp_x].astype(np.int32), hdiv[sp_x].astype(np.int64), sp_s0, sp_n,
                       int(max_slots), level_ws, node_rec, row_rec)


# --------------------------------------------------------------------------- slab plan
SLAB_BUDGET = 16384      # accumulator doubles per slab CTA (rows x columns), 128 KB
SLAB_COLS = 2048         # column cap per slab


@njit(cache=True)
def _lower_bound(a, lo, hi, key):
    while lo < hi:
        mid = (lo + hi) >> 1
        if a[mid] < key:
            lo = mid + 1
        else:
            hi = mid
    return lo


@njit(cache=True)
def _slab_plan(first, kind, colptr, cols, nl, dptr, deps, node_of, level, budget, cap, slab_node):
    """Column slabs of every supernode target and, per slab, the ascending list of
    source steps that touch it (or whose block it owns).

    A target's L-region slabs never split a source node's columns; the block slab
    starts at the diagonal block.  Item = (dep index k, q0, q1, owner) where
    [q0, q1) is the range of the source's beyond-block columns that land in the slab."""
    nn = len(kind)
    # pass 1: count slabs / items
    sl_node_l = []
    sl_c0_l = []
    sl_c1_l = []
    sl_kind_l = []
    it_ptr_l = [np.int64(0)]
    it_k_l = []
    it_q0_l = []
    it_q1_l = []
    it_own_l = []
    sn_slab0 = np.full(nn, -1, np.int64)
    sn_nslab = np.zeros(nn, np.int64)
    sn_bslab = np.full(nn, -1, np.int64)
    for u in range(nn):
        if slab_node[u] == 0:
            continue
        r = first[u]
        s = first[u + 1] - r
        c0 = colptr[u]
        W = colptr[u + 1] - c0
        L = nl[u]
        sw = budget // s
        if sw > cap:
            sw = cap
        if sw < 64:
            sw = 64
        base = len(sl_node_l)
        sn_slab0[u] = base
        # L-region slabs: pack node runs
        p = 0
        while p < L:
            start = p
            while p < L:
                v = node_of[cols[c0 + p]]
                q = p
                while q < L and node_of[cols[c0 + q]] == v:
                    q += 1
                if q - start > sw and p > start:
                    break
                p = q
                if p - start >= sw:
                    break
            sl_node_l.append(u)
            sl_c0_l.append(start)
            sl_c1_l.append(p)
            sl_kind_l.append(0)
        # block slab + panel slabs
        p = L
        first_u = True
        while p < W:
            e = min(W, p + sw)
            sl_node_l.append(u)
            sl_c0_l.append(p)
            sl_c1_l.append(e)
            if first_u:
                sn_bslab[u] = len(sl_node_l) - 1
                sl_kind_l.append(1)
                first_u = False
            else:
                sl_kind_l.append(2)
            p = e
        ns = len(sl_node_l) - base
        sn_nslab[u] = ns
        # items per slab
        for si in range(base, base + ns):
            a0 = sl_c0_l[si]
            a1 = sl_c1_l[si]
            idlo = cols[c0 + a0]
            idhi = cols[c0 + a1 - 1]
            for k in range(dptr[u + 1] - dptr[u]):
                v = deps[dptr[u] + k]
                vf = first[v]
                vs = first[v + 1] - vf
                vc0 = colptr[v]
                vW = colptr[v + 1] - vc0
                pst = nl[v] + vs          # first beyond-block position in v's list
                # block position of v in the target (owner test)
                pb0 = _lower_bound(cols, c0, c0 + L, vf) - c0
                own = 1 if (pb0 >= a0 and pb0 < a1) else 0
                q0 = _lower_bound(cols, vc0 + pst, vc0 + vW, idlo) - vc0 - pst
                q1 = _lower_bound(cols, vc0 + pst, vc0 + vW, idhi + 1) - vc0 - pst
                if q1 > q0 or own:
                    it_k_l.append(np.int32(k))
                    it_q0_l.append(np.int32(q0))
                    it_q1_l.append(np.int32(q1))
                    it_own_l.append(np.int8(own))
            it_ptr_l.append(np.int64(len(it_k_l)))
    ns = len(sl_node_l)
    sl_node = np.empty(ns, np.int32)
    sl_c0 = np.empty(ns, np.int32)
    sl_c1 = np.empty(ns, np.int32)
    sl_kind = np.empty(ns, np.int8)
    for x in range(ns):
        sl_node[x] = sl_node_l[x]
        sl_c0[x] = sl_c0_l[x]
        sl_c1[x] = sl_c1_l[x]
        sl_kind[x] = sl_kind_l[x]
    it_ptr = np.empty(len(it_ptr_l), np.int64)
    for x in range(len(it_ptr_l)):
        it_ptr[x] = it_ptr_l[x]
    ni = len(it_k_l)
    it_k = np.empty(ni, np.int32)
    it_q0 = np.empty(ni, np.int32)
    it_q1 = np.empty(ni, np.int32)
    it_own = np.empty(ni, np.int8)
    for x in range(ni):
        it_k[x] = it_k_l[x]
        it_q0[x] = it_q0_l[x]
        it_q1[x] = it_q1_l[x]
        it_own[x] = it_own_l[x]
    return sl_node, sl_c0, sl_c1, sl_kind, it_ptr, it_k, it_q0, it_q1, it_own, sn_slab0, sn_nslab, sn_bslab


@dataclass
class SlabPlan:
    sl_node: np.ndarray
    sl_c0: np.ndarray
    sl_c1: np.ndarray
    sl_kind: np.ndarray      # 0 L-region, 1 block (+ first panel part), 2 panel
    it_ptr: np.ndarray
    it_k: np.ndarray
    it_q0: np.ndarray
    it_q1: np.ndarray
    it_own: np.ndarray
    sn_slab0: np.ndarray
    sn_nslab: np.ndarray
    sn_bslab: np.ndarray
    level_slab_ptr: np.ndarray   # slabs grouped by factorization level (slab ids are in level order)

    @property
    def nslabs(self):
        return len(self.sl_node)


WIDE_ROW = 1024


def slab_nodes(sym, wide_row=WIDE_ROW):
    """Nodes processed by the slab kernel: every supernode and, in SUPROW/SUPSUP
    modes, standalone rows wider than ``wide_row`` (their supernode sources are
    sup-row updates, i.e. block updates of a 1-row target)."""
    m = (sym.node_kind == 1).astype(np.uint8)
    if int(sym.kernel_mode) >= 1:
        m |= ((sym.node_kind == 0) & (np.diff(sym.colptr) > wide_row)).astype(np.uint8)
    return m


def build_slab_plan(sym, budget=SLAB_BUDGET, cap=SLAB_COLS, wide_row=WIDE_ROW):
    """Slabs in factorization-level order (so one launch per level covers a
    contiguous slab-id range, targets ascending, slabs ascending within a target)."""
    s = sym
    mask = slab_nodes(s, wide_row)
    (sl_node, sl_c0, sl_c1, sl_kind, it_ptr, it_k, it_q0, it_q1, it_own, sn_slab0, sn_nslab,
     sn_bslab) = _slab_plan(s.node_first, s.node_kind, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps,
                            s.node_of, s.level, budget, cap, mask)
    # reorder slabs by (level, node, slab) — nodes ascending already; stable sort on level
    lev = s.level[sl_node] if len(sl_node) else np.zeros(0, np.int64)
    order = np.argsort(lev, kind="stable")
    inv = np.empty_like(order)
    inv[order] = np.arange(len(order))
    cnt = np.diff(it_ptr)
    new_ptr = np.zeros(len(order) + 1, np.int64)
    np.cumsum(cnt[order], out=new_ptr[1:])
    idx = np.concatenate([np.arange(it_ptr[o], it_ptr[o + 1]) for o in order]) if len(order) else \
        np.zeros(0, np.int64)
    nlev = len(s.level_ptr) - 1
    lptr = np.zeros(nlev + 1, np.int64)
    if len(lev):
        np.add.at(lptr[1:], lev, 1)
    np.cumsum(lptr, out=lptr)
    has = sn_slab0 >= 0
    sn_slab0 = sn_slab0.copy()
    sn_bslab = sn_bslab.copy()
    sn_slab0[has] = inv[sn_slab0[has]]
    sn_bslab[has] = inv[sn_bslab[has]]
    return SlabPlan(sl_node[order], sl_c0[order], sl_c1[order], sl_kind[order], new_ptr,
                    it_k[idx], it_q0[idx], it_q1[idx], it_own[idx], sn_slab0, sn_nslab, sn_bslab,
                    lptr)


@njit(cache=True)
def _dep_block_pos(first, kind, colptr, cols, nl, dptr, deps):
    """Per dependency edge (u, v): position in u's column list of v's first present
    block column, and the per-slab-level shared-memory needs."""
    nd = dptr[len(kind)]
    pb = np.empty(nd, np.int32)
    for u in range(len(kind)):
        c0 = colptr[u]
        L = nl[u]
        for k in range(dptr[u], dptr[u + 1]):
            v = deps[k]
            pb[k] = _lower_bound(cols, c0, c0 + L, first[v]) - c0
    return pb


def slab_level_smem(sym, plan):
    """(Smax, Mmax, SWmax, ACCmax) per level for the slab launch's shared memory."""
    s = sym
    nlev = len(plan.level_slab_ptr) - 1
    out = np.zeros((nlev, 4), np.int64)
    rows = np.diff(s.node_first)
    for lv in range(nlev):
        a, b = plan.level_slab_ptr[lv], plan.level_slab_ptr[lv + 1]
        if a == b:
            continue
        nodes = plan.sl_node[a:b]
        sw = (plan.sl_c1[a:b] - plan.sl_c0[a:b])
        mm = 1
        for u in np.unique(nodes):
            d = s.deps[s.dep_ptr[u]:s.dep_ptr[u + 1]]
            if len(d):
                mm = max(mm, int(rows[d].max()))
        out[lv] = (int(rows[nodes].max()), mm, int(sw.max()), int((rows[nodes] * sw).max()))
    return out


# --------------------------------------------------------------------------- level fan-in plan
FANIN_TILE = 64          # target columns per update tile
PANEL_TILE = 256         # columns per permutation / TRSM tile


@njit(cache=True)
def _fanin_plan(first, kind, colptr, cols, nl, dptr, deps, level, nlev, tw, pw, updates=True):
    """Per level: LU nodes, perm/TRSM tiles, X pairs and update tiles.

    Update item = (target T, tile [c0, c1)) with its source list (dep index k, q0, q1):
    the sources of T that finish at this level and whose beyond-block columns meet
    the tile ([q0, q1) indexes those columns)."""
    nn = len(kind)
    # ---- nodes by level (LU) and perm/TRSM tiles
    lu_cnt = np.zeros(nlev + 1, np.int64)
    for u in range(nn):
        lu_cnt[level[u] + 1] += 1
    lu_ptr = np.cumsum(lu_cnt)
    lu_nodes = np.empty(nn, np.int32)
    fillp = lu_ptr[:-1].copy()
    for u in range(nn):
        lu_nodes[fillp[level[u]]] = u
        fillp[level[u]] += 1
    pt_node_l = []
    pt_c0_l = []
    pt_c1_l = []
    pt_ptr = np.zeros(nlev + 1, np.int64)
    for lv in range(nlev):
        for x in range(lu_ptr[lv], lu_ptr[lv + 1]):
            u = lu_nodes[x]
            s = first[u + 1] - first[u]
            if s < 2:
                continue
            W = colptr[u + 1] - colptr[u]
            L = nl[u]
            c = 0
            while c < L:
                pt_node_l.append(u)
                pt_c0_l.append(c)
                pt_c1_l.append(min(L, c + pw))
                c += pw
            c = L + s
            while c < W:
                pt_node_l.append(u)
                pt_c0_l.append(c)
                pt_c1_l.append(min(W, c + pw))
                c += pw
        pt_ptr[lv + 1] = len(pt_node_l)
    # ---- X pairs: dependency edges grouped by the source's level
    nd = dptr[nn]
    xp_cnt = np.zeros(nlev + 1, np.int64)
    for u in range(nn):
        for k in range(dptr[u], dptr[u + 1]):
            xp_cnt[level[deps[k]] + 1] += 1
    xp_ptr = np.cumsum(xp_cnt)
    xp_edge = np.empty(nd, np.int64)
    xp_tgt = np.empty(nd, np.int32)
    fillx = xp_ptr[:-1].copy()
    for u in range(nn):
        for k in range(dptr[u], dptr[u + 1]):
            lv = level[deps[k]]
            xp_edge[fillx[lv]] = k
            xp_tgt[fillx[lv]] = u
            fillx[lv] += 1
    # ---- update tiles: for each edge (grouped by source level, then target), walk the
    # source's beyond-block columns tile by tile
    up_t_l = []      # target
    up_c0_l = []
    up_c1_l = []
    up_ptr_l = [np.int64(0)]   # per item: range into src lists
    src_k_l = []
    src_q0_l = []
    src_q1_l = []
    lev_up = np.zeros(nlev + 1, np.int64)
    tmp_tile = np.empty(0, np.int64)
    for lv in range(nlev if updates else 0):
        x = xp_ptr[lv]
        while x < xp_ptr[lv + 1]:
            u = xp_tgt[x]
            x1 = x
            while x1 < xp_ptr[lv + 1] and xp_tgt[x1] == u:
                x1 += 1
            # edges x..x1 share target u; gather (tile, k, q0, q1) records
            c0u = colptr[u]
            W = colptr[u + 1] - c0u
            ntile = (W + tw - 1) // tw
            cnt = np.zeros(ntile, np.int64)
            recs_t = []
            recs_k = []
            recs_q0 = []
            recs_q1 = []
            for e in range(x, x1):
                k = xp_edge[e]
                v = deps[k]
                vs = first[v + 1] - first[v]
                vc0 = colptr[v]
                vW = colptr[v + 1] - vc0
                pst = nl[v] + vs
                q = pst
                while q < vW:
                    pos = _lower_bound(cols, c0u, c0u + W, cols[vc0 + q]) - c0u
                    t = pos // tw
                    hi_id = cols[c0u + min(W, (t + 1) * tw) - 1]
                    qe = _lower_bound(cols, vc0 + q, vc0 + vW, hi_id + 1) - vc0
                    recs_t.append(t)
                    recs_k.append(k - dptr[u])
                    recs_q0.append(q - pst)
                    recs_q1.append(qe - pst)
                    cnt[t] += 1
                    q = qe
            # emit items tile-ordered, sources in edge (ascending k) order
            for t in range(ntile):
                if cnt[t] == 0:
                    continue
                up_t_l.append(u)
                up_c0_l.append(t * tw)
                up_c1_l.append(min(W, (t + 1) * tw))
                for z in range(len(recs_t)):
                    if recs_t[z] == t:
                        src_k_l.append(np.int32(recs_k[z]))
                        src_q0_l.append(np.int32(recs_q0[z]))
                        src_q1_l.append(np.int32(recs_q1[z]))
                up_ptr_l.append(np.int64(len(src_k_l)))
            x = x1
        lev_up[lv + 1] = len(up_t_l)
    nu = len(up_t_l)
    up_t = np.empty(nu, np.int32)
    up_c0 = np.empty(nu, np.int32)
    up_c1 = np.empty(nu, np.int32)
    for z in range(nu):
        up_t[z] = up_t_l[z]
        up_c0[z] = up_c0_l[z]
        up_c1[z] = up_c1_l[z]
    up_ptr = np.empty(len(up_ptr_l), np.int64)
    for z in range(len(up_ptr_l)):
        up_ptr[z] = up_ptr_l[z]
    ns = len(src_k_l)
    src_k = np.empty(ns, np.int32)
    src_q0 = np.empty(ns, np.int32)
    src_q1 = np.empty(ns, np.int32)
    for z in range(ns):
        src_k[z] = src_k_l[z]
        src_q0[z] = src_q0_l[z]
        src_q1[z] = src_q1_l[z]
    npt = len(pt_node_l)
    pt_node = np.empty(npt, np.int32)
    pt_c0 = np.empty(npt, np.int32)
    pt_c1 = np.empty(npt, np.int32)
    for z in range(npt):
        pt_node[z] = pt_node_l[z]
        pt_c0[z] = pt_c0_l[z]
        pt_c1[z] = pt_c1_l[z]
    return (lu_ptr, lu_nodes, pt_ptr, pt_node, pt_c0, pt_c1, xp_ptr, xp_edge.astype(np.int64), xp_tgt,
            lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1)


@njit(cache=True)
def _tile_records(cols, first, colptr, nl, deps, dptr, xp_edge, x, x1, u, tw, out_t, out_k, out_q0, out_q1):
    """Walk the beyond-block columns of the sources of edges x..x1 (all into target u)
    tile by tile; fill the record arrays (if given, len > 0) and return the count."""
    c0u = colptr[u]
    W = colptr[u + 1] - c0u
    n = 0
    for e in range(x, x1):
        k = xp_edge[e]
        v = deps[k]
        vs = first[v + 1] - first[v]
        vc0 = colptr[v]
        vW = colptr[v + 1] - vc0
        pst = nl[v] + vs
        q = pst
        while q < vW:
            pos = _lower_bound(cols, c0u, c0u + W, cols[vc0 + q]) - c0u
            t = pos // tw
            hi_id = cols[c0u + min(W, (t + 1) * tw) - 1]
            qe = _lower_bound(cols, vc0 + q, vc0 + vW, hi_id + 1) - vc0
            if len(out_t):
                out_t[n] = t
                out_k[n] = k - dptr[u]
                out_q0[n] = q - pst
                out_q1[n] = qe - pst
            n += 1
            q = qe
    return n


@njit(cache=True, parallel=True)
def _fanin_updates_par(first, colptr, cols, nl, dptr, deps, xp_ptr, xp_edge, xp_tgt, nlev, tw, nth):
    """The update items of _fanin_plan, built in parallel over (level, target) groups:
    pass 1 counts each group's records and distinct tiles, pass 2 fills them at
    prefix-sum offsets (records of a group counting-sorted by tile, edge order kept
    within a tile) — the same arrays as the serial loop.  Per-thread scratch (no
    allocation inside the parallel loops); ``nth`` must cover every thread id of the
    pool (numba.config.NUMBA_NUM_THREADS)."""
    # groups: maximal runs of equal target within a level
    ng = 0
    for lv in range(nlev):
        for x in range(xp_ptr[lv], xp_ptr[lv + 1]):
            if x == xp_ptr[lv] or xp_tgt[x] != xp_tgt[x - 1]:
                ng += 1
    gs = np.empty(ng + 1, np.int64)
    gl = np.empty(ng, np.int64)
    g = 0
    for lv in range(nlev):
        for x in range(xp_ptr[lv], xp_ptr[lv + 1]):
            if x == xp_ptr[lv] or xp_tgt[x] != xp_tgt[x - 1]:
                gs[g] = x
                gl[g] = lv
                g += 1
    gs[ng] = xp_ptr[nlev]
    maxW = 0
    for u in range(len(colptr) - 1):
        maxW = max(maxW, colptr[u + 1] - colptr[u])
    mt = (maxW + tw - 1) // tw + 1
    stamp = np.zeros((nth, mt), np.int64)
    nrec = np.zeros(ng, np.int64)
    nitem = np.zeros(ng, np.int64)
    e0 = np.zeros(0, np.int64)
    e32 = np.zeros(0, np.int32)
    for g in prange(ng):
        th = numba.get_thread_id()
        u = xp_tgt[gs[g]]
        c0u = colptr[u]
        W = colptr[u + 1] - c0u
        n = 0
        ni = 0
        for e in range(gs[g], gs[g + 1]):
            k = xp_edge[e]
            v = deps[k]
            vc0 = colptr[v]
            vW = colptr[v + 1] - vc0
            q = nl[v] + first[v + 1] - first[v]
            while q < vW:
                pos = _lower_bound(cols, c0u, c0u + W, cols[vc0 + q]) - c0u
                t = pos // tw
                hi_id = cols[c0u + min(W, (t + 1) * tw) - 1]
                q = _lower_bound(cols, vc0 + q, vc0 + vW, hi_id + 1) - vc0
                n += 1
                if stamp[th, t] != g + 1:
                    stamp[th, t] = g + 1
                    ni += 1
        nrec[g] = n
        nitem[g] = ni
    roff = np.zeros(ng + 1, np.int64)
    ioff = np.zeros(ng + 1, np.int64)
    maxn = 1
    for g in range(ng):
        roff[g + 1] = roff[g] + nrec[g]
        ioff[g + 1] = ioff[g] + nitem[g]
        maxn = max(maxn, nrec[g])
    NI = ioff[ng]
    NS = roff[ng]
    up_t = np.empty(NI, np.int32)
    up_c0 = np.empty(NI, np.int32)
    up_c1 = np.empty(NI, np.int32)
    up_ptr = np.empty(NI + 1, np.int64)
    up_ptr[NI] = NS
    src_k = np.empty(NS, np.int32)
    src_q0 = np.empty(NS, np.int32)
    src_q1 = np.empty(NS, np.int32)
    srt = np.empty((nth, maxn), np.int64)
    srk = np.empty((nth, maxn), np.int32)
    sr0 = np.empty((nth, maxn), np.int32)
    sr1 = np.empty((nth, maxn), np.int32)
    scnt = np.empty((nth, mt + 1), np.int64)
    for g in prange(ng):
        th = numba.get_thread_id()
        u = xp_tgt[gs[g]]
        W = colptr[u + 1] - colptr[u]
        ntile = (W + tw - 1) // tw
        rt = srt[th]
        rk = srk[th]
        r0 = sr0[th]
        r1 = sr1[th]
        n = _tile_records(cols, first, colptr, nl, deps, dptr, xp_edge, gs[g], gs[g + 1], u, tw, rt, rk, r0, r1)
        cnt = scnt[th]
        for t in range(ntile + 1):
            cnt[t] = 0
        for z in range(n):
            cnt[rt[z] + 1] += 1
        for t in range(ntile):
            cnt[t + 1] += cnt[t]
        base = roff[g]
        it = ioff[g]
        for t in range(ntile):
            if cnt[t + 1] > cnt[t]:
                up_t[it] = u
                up_c0[it] = t * tw
                up_c1[it] = min(W, (t + 1) * tw)
                up_ptr[it] = base + cnt[t]
                it += 1
        for z in range(n):          # stable counting sort by tile (cnt becomes the fill cursor)
            d = base + cnt[rt[z]]
            cnt[rt[z]] += 1
            src_k[d] = rk[z]
            src_q0[d] = r0[z]
            src_q1[d] = r1[z]
    lev_up = np.zeros(nlev + 1, np.int64)
    for g in range(ng):
        lev_up[gl[g] + 1] += nitem[g]
    for lv in range(nlev):
        lev_up[lv + 1] += lev_up[lv]
    return lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1


@dataclass
class FaninPlan:
    lu_ptr: np.ndarray
    lu_nodes: np.ndarray
    pt_ptr: np.ndarray
    pt_node: np.ndarray
    pt_c0: np.ndarray
    pt_c1: np.ndarray
    xp_ptr: np.ndarray
    xp_edge: np.ndarray
    xp_tgt: np.ndarray
    lev_up: np.ndarray
    up_t: np.ndarray
    up_c0: np.ndarray
    up_c1: np.ndarray
    up_ptr: np.ndarray
    src_k: np.ndarray
    src_q0: np.ndarray
    src_q1: np.ndarray
    dep_pb: np.ndarray
    level_smax: np.ndarray     # max target rows among update items of a level
    level_mmax: np.ndarray     # max source rows of a level
    lev_up_big: np.ndarray     # per level: first update item whose target has >= BIG_ROWS rows
    lev_up_reg: np.ndarray     # per level: first item of the per-source (regular) group
    lev_up_rs: np.ndarray      # per level: first regular item for the CTA kernel (before: warp kernel)
    lev_xp_big: np.ndarray     # per level: first multiplier item for the CTA kernel (before: warp kernel)
    lev_hub: np.ndarray        # per level: offsets into hub_list
    hub_list: np.ndarray       # pull-program rows by level (k_hub1)
    up_part: np.ndarray        # per update item: split-K part id, -1 if unsplit
    part_first: np.ndarray     # per part: first part id of its item's group
    part_n: np.ndarray         # per part: parts in its group
    part_off: np.ndarray       # per part: offset (doubles) of its partial tile in the scratch

    @property
    def nlevels(self):
        return len(self.lu_ptr) - 1


@njit(cache=True)
def _fanin_levels(first, colptr, cols, nl, dptr, deps, node_of):
    """Longest-path levels over L edges (v -> u for u's L entries in v's columns) and
    U edges (v -> w when v's beyond-block columns meet w's block): within a fan-in
    level no source updates another source's block columns, and every node's
    updates come from strictly lower levels.  Equal to the L levels for
    structurally symmetric patterns."""
    nn = len(nl)
    lev = np.zeros(nn, np.int64)
    for u in range(nn):                    # nodes in topological (index) order
        for k in range(dptr[u], dptr[u + 1]):
            v = deps[k]
            if lev[v] + 1 > lev[u]:
                lev[u] = lev[v] + 1
        # push U edges forward: owners of u's beyond-block columns
        s = first[u + 1] - first[u]
        c0 = colptr[u]
        last = -1
        for q in range(c0 + nl[u] + s, colptr[u + 1]):
            w = node_of[cols[q]]
            if w != last:
                if lev[u] + 1 > lev[w]:
                    lev[w] = lev[u] + 1
                last = w
    return lev


BIG_ROWS = 32
WARP_ROWS = 4          # update items with targets this small run warp-per-item
XW_ROWS, XW_M = 32, 8  # multiplier blocks this small (target rows, source rows) too


def _split_items(out, rows, nlev, src_rows):
    """Within each level order the update items in four contiguous launch groups:
    0 = many small sources (packed K-slice kernel), 1 = regular with a target of
    <= WARP_ROWS rows (warp-per-item kernel), 2 = regular (per-source FFMA CTA
    kernel), 3 = target >= BIG_ROWS rows (DMMA-eligible; runs the FFMA kernel
    unless DMMA routing is enabled)."""
    (lu_ptr, lu_nodes, pt_ptr, pt_node, pt_c0, pt_c1, xp_ptr, xp_edge, xp_tgt,
     lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1) = out
    nitem = len(up_t)
    lvl = np.repeat(np.arange(nlev), np.diff(lev_up))
    nsrc = np.diff(up_ptr)
    msum = np.add.reduceat(src_rows, up_ptr[:-1]) if len(src_rows) else np.zeros(nitem)
    import os
    pm = float(os.environ.get("HYLU_PACK_M", "4"))
    pn = int(os.environ.get("HYLU_PACK_N", "4"))
    packed = (nsrc >= pn) & (msum < pm * nsrc)
    big = (rows[up_t] >= BIG_ROWS) & ~packed
    small = (rows[up_t] <= WARP_ROWS) & ~packed & ~big
    grp = np.where(packed, 0, np.where(big, 3, np.where(small, 1, 2))).astype(np.int64)
    order = np.lexsort((grp, lvl))
    cnt = np.diff(up_ptr)[order]
    new_ptr = np.zeros(nitem + 1, np.int64)
    np.cumsum(cnt, out=new_ptr[1:])
    gather = np.repeat(up_ptr[:-1][order], cnt) + (np.arange(new_ptr[-1]) - np.repeat(new_ptr[:-1], cnt))
    def cnt_of(k):
        return np.bincount(lvl[grp == k], minlength=nlev) if nitem else np.zeros(nlev, np.int64)
    reg = lev_up[:-1] + cnt_of(0)
    rs = reg + cnt_of(1)
    split = rs + cnt_of(2)
    out = (lu_ptr, lu_nodes, pt_ptr, pt_node, pt_c0, pt_c1, xp_ptr, xp_edge, xp_tgt, lev_up,
           up_t[order], up_c0[order], up_c1[order], new_ptr, src_k[gather], src_q0[gather],
           src_q1[gather])
    return out, split.astype(np.int64), reg.astype(np.int64), rs.astype(np.int64)


SPLIT_SRC = int(os.environ.get("HYLU_SPLIT_SRC", "8"))
SPLIT_REL = float(os.environ.get("HYLU_SPLIT_REL", "4"))
SPLIT_LEVEL_ITEMS = int(os.environ.get("HYLU_SPLIT_LEVEL_ITEMS", "8192"))  # packed items per level


def _split_heavy(out, split, reg, rs, rows, nlev, cap=None):
    """Split-K for packed update items (group 0) with more than `cap` sources: the
    item becomes ceil(nsrc/cap) consecutive parts over contiguous source ranges.
    Each part accumulates its partial product tile; the last part to finish adds
    the partials in part order and updates the target once (deterministic).
    Returns the plan, the shifted group offsets and the part tables."""
    cap = SPLIT_SRC if cap is None else cap
    out = list(out)
    lev_up, up_t, up_c0, up_c1, up_ptr = out[9], out[10], out[11], out[12], out[13]
    nitem = len(up_t)
    nsrc = np.diff(up_ptr)
    lvl = np.repeat(np.arange(nlev), np.diff(lev_up))
    grp0 = np.arange(nitem) < reg[lvl] if nitem else np.zeros(0, bool)
    # only outliers: items far above their level's mean source count set the
    # level's critical path; splitting typical items just adds partial traffic
    g0cnt = np.bincount(lvl[grp0], minlength=nlev)
    g0sum = np.bincount(lvl[grp0], weights=nsrc[grp0], minlength=nlev)
    mean = np.where(g0cnt > 0, g0sum / np.maximum(g0cnt, 1), 0.0)
    outlier = nsrc > SPLIT_REL * mean[lvl] if nitem else np.zeros(0, bool)
    narrow = (g0cnt < SPLIT_LEVEL_ITEMS)[lvl] if nitem else np.zeros(0, bool)
    heavy = grp0 & narrow & outlier & (nsrc > cap) if cap > 0 else np.zeros(nitem, bool)
    npart = np.where(heavy, (nsrc + cap - 1) // max(cap, 1), 1).astype(np.int64)
    empty = (np.full(0, -1, np.int32), np.zeros(0, np.int32), np.zeros(0, np.int32),
             np.zeros(0, np.int64))
    if not heavy.any():
        return tuple(out), split, reg, rs, (np.full(nitem, -1, np.int32),) + empty[1:]
    newstart = np.concatenate([[0], np.cumsum(npart)]).astype(np.int64)
    tot = int(newstart[-1])
    item_of = np.repeat(np.arange(nitem), npart)
    k = np.arange(tot) - newstart[item_of]
    out[10], out[11], out[12] = up_t[item_of], up_c0[item_of], up_c1[item_of]
    starts = up_ptr[:-1][item_of] + k * cap
    out[13] = np.concatenate([starts, [up_ptr[-1]]]).astype(np.int64)
    out[9] = newstart[lev_up]
    split, reg, rs = newstart[split], newstart[reg], newstart[rs]
    # part tables
    is_part = heavy[item_of]
    nparts = int(is_part.sum())
    up_part = np.full(tot, -1, np.int32)
    up_part[is_part] = np.arange(nparts, dtype=np.int32)
    part_n = npart[item_of][is_part].astype(np.int32)
    part_first = (np.arange(nparts) - k[is_part]).astype(np.int32)
    # partial tiles are live only within their level: offsets restart per level
    tile = rows[up_t[item_of][is_part]].astype(np.int64) * FANIN_TILE
    plev = lvl[item_of][is_part]
    csum = np.cumsum(tile) - tile
    lev_base = np.zeros(nlev, np.int64)
    if nparts:
        first_in_lev = np.searchsorted(plev, np.arange(nlev))
        has = first_in_lev < nparts
        lev_base[has] = csum[first_in_lev[has]]
    part_off = (csum - lev_base[plev]).astype(np.int64)
    return tuple(out), split, reg, rs, (up_part, part_first, part_n, part_off)


def _split_xp(out, s, rows, nlev):
    """Within each level put the small multiplier items (target <= XW_ROWS rows,
    <= XW_M source rows) first: they run warp-per-item; the rest run CTA-per-item."""
    out = list(out)
    xp_ptr, xp_edge, xp_tgt = out[6], np.asarray(out[7], np.int64), np.asarray(out[8])
    n = len(xp_tgt)
    big = np.zeros(nlev, np.int64)
    if n:
        v = s.deps[xp_edge]
        tb0 = s.cols[s.colptr[xp_tgt] + np.asarray(_dep_pb_cache(s))[xp_edge]] - s.node_first[v]
        m = rows[v] - tb0
        small = (rows[xp_tgt] <= XW_ROWS) & (m <= XW_M)
        lvl = np.repeat(np.arange(nlev), np.diff(xp_ptr))
        order = np.lexsort((~small, lvl))
        out[7], out[8] = out[7][order], out[8][order]
        big = xp_ptr[:-1] + np.bincount(lvl[small], minlength=nlev)
    else:
        big = np.asarray(xp_ptr[:-1], np.int64).copy()
    return tuple(out), big.astype(np.int64)


def _dep_pb_cache(s):
    pb = getattr(s, "_dep_pb", None)
    if pb is None:
        pb = _dep_block_pos(s.node_first, s.node_kind, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps)
        s._dep_pb = pb
    return pb


def _drop_pull_targets(out, pull, nlev):
    """Take the pull-program rows out of the fan-in plan as targets: no LU, tile,
    multiplier-block or update item has them as target (they are computed whole
    by their pull program at their level, once every source is final); they stay
    sources of later nodes.  Returns the plan and the per-level pull-row lists."""
    (lu_ptr, lu_nodes, pt_ptr, pt_node, pt_c0, pt_c1, xp_ptr, xp_edge, xp_tgt,
     lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1) = out

    def keep_ptr(ptr, keep):
        lvl = np.repeat(np.arange(nlev), np.diff(ptr))
        cnt = np.bincount(lvl[keep], minlength=nlev)
        return np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)

    lu_nodes = np.asarray(lu_nodes)
    k_lu = ~pull[lu_nodes]
    lvl_lu = np.repeat(np.arange(nlev), np.diff(lu_ptr))
    hub_list = lu_nodes[~k_lu].astype(np.int32)
    lev_hub = np.concatenate([[0], np.cumsum(np.bincount(lvl_lu[~k_lu], minlength=nlev))]).astype(np.int64)
    k_pt = ~pull[np.asarray(pt_node)]
    k_xp = ~pull[np.asarray(xp_tgt)]
    k_up = ~pull[np.asarray(up_t)]
    nsrc = np.diff(up_ptr)
    k_src = np.repeat(k_up, nsrc)
    new_up_ptr = np.concatenate([[0], np.cumsum(nsrc[k_up])]).astype(np.int64)
    out = (keep_ptr(lu_ptr, k_lu), lu_nodes[k_lu], keep_ptr(pt_ptr, k_pt), pt_node[k_pt], pt_c0[k_pt],
           pt_c1[k_pt], keep_ptr(xp_ptr, k_xp), xp_edge[k_xp], xp_tgt[k_xp], keep_ptr(lev_up, k_up),
           up_t[k_up], up_c0[k_up], up_c1[k_up], new_up_ptr, src_k[k_src], src_q0[k_src], src_q1[k_src])
    return out, lev_hub, hub_list


def build_fanin_plan(sym, tw=FANIN_TILE, pw=PANEL_TILE, pull=None):
    """pull: optional bool[nnodes] — standalone rows computed by pull programs
    (k_hub1) at their level instead of receiving fan-in updates."""
    s = sym
    flev = _fanin_levels(s.node_first, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps, s.node_of)
    nlev = int(flev.max()) + 1
    out = _fanin_plan(s.node_first, s.node_kind, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps,
                      flev, nlev, tw, pw, False)
    # update items in parallel over (level, target) groups (the serial loop's arrays)
    out = out[:9] + _fanin_updates_par(s.node_first, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps,
                                       out[6], out[7], out[8], nlev, tw, numba.config.NUMBA_NUM_THREADS)
    if pull is not None and pull.any():
        out, lev_hub, hub_list = _drop_pull_targets(out, np.asarray(pull, bool), nlev)
    else:
        lev_hub, hub_list = np.zeros(nlev + 1, np.int64), np.zeros(0, np.int32)
    dep_pb = _dep_pb_cache(s)
    rows = np.diff(s.node_first)
    # source rows per update-source record (rows of v from its first present block row)
    up_ptr, up_t, src_k = out[13], out[10], out[14]
    tgt = np.repeat(up_t.astype(np.int64), np.diff(up_ptr))
    dk = s.dep_ptr[tgt] + src_k
    v = s.deps[dk]
    tb0 = s.cols[s.colptr[tgt] + dep_pb[dk]] - s.node_first[v]
    src_rows = (rows[v] - tb0).astype(np.int64)
    import os
    cap_rows = int(os.environ.get("HYLU_MERGE_ROWS", "0"))
    if cap_rows > 0:
        cap_recs = int(os.environ.get("HYLU_MERGE_RECS", "64"))
        (lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1, src_rows) = _merge_items(
            nlev, flev, s.node_first, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps, s.node_of,
            out[9], out[10], out[11], out[12], out[13], out[14], out[15], out[16], src_rows,
            cap_rows, cap_recs)
        out = out[:9] + (lev_up, up_t, up_c0, up_c1, up_ptr, src_k, src_q0, src_q1)
    out, split, reg, rs = _split_items(out, rows, nlev, src_rows)
    out, split, reg, rs, parts = _split_heavy(out, split, reg, rs, rows, nlev)
    out, xp_big = _split_xp(out, s, rows, nlev)
    lu_ptr, lu_nodes = out[0], out[1]
    lev_up, up_t = out[9], out[10]
    smax = np.ones(nlev, np.int32)
    mmax = np.ones(nlev, np.int32)
    for lv in range(nlev):
        a, b = lev_up[lv], lev_up[lv + 1]
        if b > a:
            smax[lv] = int(rows[up_t[a:b]].max())
        nodes = lu_nodes[lu_ptr[lv]:lu_ptr[lv + 1]]
        if len(nodes):
            mmax[lv] = int(rows[nodes].max())
    return FaninPlan(*out, dep_pb, smax, mmax, split, reg, rs, xp_big, lev_hub, hub_list, *parts)


def fanin_source_records(sym, plan):
    """Per update-source record: (source node v, block position pb0 in the target,
    first present block row tb0) — static, so the device does no metadata chasing."""
    s = sym
    # target of each source record
    cnt = np.diff(plan.up_ptr)
    tgt = np.repeat(plan.up_t.astype(np.int64), cnt)
    dk = s.dep_ptr[tgt] + plan.src_k
    v = s.deps[dk].astype(np.int32)
    pb0 = plan.dep_pb[dk].astype(np.int32)
    tb0 = (s.cols[s.colptr[tgt] + pb0] - s.node_first[v]).astype(np.int32)
    return v, pb0, tb0


@njit(cache=True, parallel=True)
def _kc_maps(first, colptr, cols, nl, valoff, up_t, up_c0, up_c1, up_ptr, src_q0, src_q1, sv, stb):
    nsrc = len(src_q0)
    off = np.zeros(nsrc + 1, np.int64)
    for z in range(nsrc):
        off[z + 1] = off[z] + (src_q1[z] - src_q0[z])
    pos = np.empty(off[nsrc], np.int8)
    vb = np.empty(nsrc, np.int64)
    vW = np.empty(nsrc, np.int32)
    qb = np.empty(nsrc, np.int32)
    mm = np.empty(nsrc, np.int32)
    for it in prange(len(up_t)):   # items own disjoint record ranges
        T = up_t[it]
        t0 = colptr[T] + up_c0[it]
        t1 = colptr[T] + up_c1[it]
        for z in range(up_ptr[it], up_ptr[it + 1]):
            v = sv[z]
            vs = first[v + 1] - first[v]
            q = nl[v] + vs + src_q0[z]
            vb[z] = valoff[v]
            vW[z] = colptr[v + 1] - colptr[v]
            qb[z] = q
            mm[z] = vs - stb[z]
            base = colptr[v] + q
            lo = t0
            for c in range(src_q1[z] - src_q0[z]):
                key = cols[base + c]
                # columns ascend: continue the search from the previous position
                hi = t1
                while lo < hi:
                    mid = (lo + hi) >> 1
                    if cols[mid] < key:
                        lo = mid + 1
                    else:
                        hi = mid
                pos[off[z] + c] = lo - t0
    return off, pos, vb, vW, qb, mm


def kc_source_maps(sym, plan):
    """Per update-source record, host-precomputed for the K-concatenated DMMA kernel:
    the tile position (0..63) of each of its nq columns (int8, records concatenated,
    offsets int64) and the source's value offset / width / first panel column / block
    height — the data the kernel otherwise derives per item with dependent loads and
    binary searches."""
    s = sym
    sv, _, stb = fanin_source_records(s, plan)
    return _kc_maps(np.asarray(s.node_first), np.asarray(s.colptr), np.asarray(s.cols), np.asarray(s.nl),
                    np.asarray(s.valoff), plan.up_t, plan.up_c0, plan.up_c1, plan.up_ptr,
                    plan.src_q0, plan.src_q1, sv, stb)


def executed_update_flops(sym, plan):
    """Flops the fan-in sup-sup / sup-row updates execute on the union-padded node
    panels: Σ over update-source records of 2·s_T·m·nq (target rows × source block
    rows × source columns in the tile).  SURVEY §8(d) asks for this beside the
    algorithmic count (exact pre-union pattern) so the padding gap is visible."""
    v, _, tb0 = fanin_source_records(sym, plan)
    first = np.asarray(sym.node_first)
    rows = np.diff(first)
    cnt = np.diff(plan.up_ptr)
    st = np.repeat(rows[plan.up_t], cnt).astype(np.float64)
    m = (rows[v] - tb0).astype(np.float64)
    nq = (plan.src_q1 - plan.src_q0).astype(np.float64)
    return float(2.0 * np.sum(st * m * nq))


# --------------------------------------------------------------------------- deadline merging
@njit(cache=True)
def _merge_items(nlev, flev, first, colptr, cols, nl, dptr, deps, node_of, lev_up, up_t, up_c0,
                 up_c1, up_ptr, src_k, src_q0, src_q1, src_rows, cap_rows, cap_recs):
    """Re-chunk each (target, tile)'s update records across levels.

    Deadline D of a tile = the first level consuming it: the target's own level if
    the tile reaches the block/panel, and the level of every source block owner
    inside the tile (its multiplier block X is formed there).  Records (sorted by
    source level, then dependency index) are packed into chunks of at most
    cap_rows source rows / cap_recs records; a chunk runs at the level of its last
    source (as early as possible), bumped to the next level if that tile already
    has a chunk there (never beyond D-1, else merged)."""
    nitem = len(up_t)
    # group items by (target, tile) -> key order
    keyT = up_t.astype(np.int64)
    key = keyT * (1 << 20) + up_c0.astype(np.int64)
    order = np.argsort(key, kind="mergesort")
    out_lvl = []
    out_t = []
    out_c0 = []
    out_c1 = []
    out_ptr = [np.int64(0)]
    o_k = []
    o_q0 = []
    o_q1 = []
    o_rows = []
    x = 0
    item_level = np.empty(nitem, np.int64)
    for lv in range(nlev):
        for it in range(lev_up[lv], lev_up[lv + 1]):
            item_level[it] = lv
    while x < nitem:
        it0 = order[x]
        T = up_t[it0]
        c0 = up_c0[it0]
        x1 = x
        while x1 < nitem and up_t[order[x1]] == T and up_c0[order[x1]] == c0:
            x1 += 1
        c1 = up_c1[it0]
        # deadline
        tc0 = colptr[T]
        L = nl[T]
        D = nlev
        if c1 > L:
            D = flev[T]
        hiL = min(c1, L)
        q = c0
        while q < hiL:
            w = node_of[cols[tc0 + q]]
            if flev[w] < D:
                D = flev[w]
            q += 1
        # gather records (items at increasing level; records already in dep order)
        recs_lv = []
        recs_z = []
        for y in range(x, x1):
            it = order[y]
            for z in range(up_ptr[it], up_ptr[it + 1]):
                recs_lv.append(item_level[it])
                recs_z.append(z)
        nr = len(recs_z)
        ro = np.empty(nr, np.int64)
        lvs = np.empty(nr, np.int64)
        for a in range(nr):
            lvs[a] = recs_lv[a]
        idx = np.argsort(lvs, kind="mergesort")
        for a in range(nr):
            ro[a] = recs_z[idx[a]]
        # part A: records whose source level is below the tile deadline are merged
        # into capped chunks run as early as possible (never later than D-1);
        # part B: the rest keep one chunk per source level (always valid).
        last_level = -1
        a = 0
        nA = 0
        while nA < nr and recs_lv[idx[nA]] <= D - 1:
            nA += 1
        while a < nr:
            rows_sum = 0
            b = a
            if a < nA:
                while b < nA and (b - a) < cap_recs and (rows_sum + src_rows[ro[b]] <= cap_rows or b == a):
                    rows_sum += src_rows[ro[b]]
                    b += 1
                lvl = recs_lv[idx[b - 1]]
                if lvl <= last_level:
                    lvl = last_level + 1
                if lvl > D - 1:
                    lvl = D - 1
            else:
                lv0 = recs_lv[idx[a]]
                while b < nr and recs_lv[idx[b]] == lv0:
                    b += 1
                lvl = lv0
            if lvl <= last_level and len(out_t) > 0:
                # same level as this tile's previous chunk: merge into it
                for c in range(a, b):
                    z = ro[c]
                    o_k.append(src_k[z])
                    o_q0.append(src_q0[z])
                    o_q1.append(src_q1[z])
                    o_rows.append(src_rows[z])
                out_ptr[-1] = np.int64(len(o_k))
                a = b
                continue
            out_lvl.append(lvl)
            out_t.append(T)
            out_c0.append(c0)
            out_c1.append(c1)
            for c in range(a, b):
                z = ro[c]
                o_k.append(src_k[z])
                o_q0.append(src_q0[z])
                o_q1.append(src_q1[z])
                o_rows.append(src_rows[z])
            out_ptr.append(np.int64(len(o_k)))
            last_level = lvl
            a = b
        x = x1
    n = len(out_t)
    lv_arr = np.empty(n, np.int64)
    for a in range(n):
        lv_arr[a] = out_lvl[a]
    perm = np.argsort(lv_arr, kind="mergesort")
    new_lev = np.zeros(nlev + 1, np.int64)
    for a in range(n):
        new_lev[lv_arr[a] + 1] += 1
    for l in range(nlev):
        new_lev[l + 1] += new_lev[l]
    nt = np.empty(n, np.int32)
    nc0 = np.empty(n, np.int32)
    nc1 = np.empty(n, np.int32)
    nptr = np.zeros(n + 1, np.int64)
    tot = len(o_k)
    nk = np.empty(tot, np.int32)
    nq0 = np.empty(tot, np.int32)
    nq1 = np.empty(tot, np.int32)
    nrw = np.empty(tot, np.int64)
    pos = 0
    for a in range(n):
        it = perm[a]
        nt[a] = out_t[it]
        nc0[a] = out_c0[it]
        nc1[a] = out_c1[it]
        for z in range(out_ptr[it], out_ptr[it + 1]):
            nk[pos] = o_k[z]
            nq0[pos] = o_q0[z]
            nq1[pos] = o_q1[z]
            nrw[pos] = o_rows[z]
            pos += 1
        nptr[a + 1] = pos
    return new_lev, nt, nc0, nc1, nptr, nk, nq0, nq1, nrw


# --------------------------------------------------------------------------- device dispatch
TIER_NAMES = ("row-row", "sup-row", "sup-sup")


def device_routing(sym, mode=None, warp_min=256):
    """The device's kernel selection for one factorization,
    written down so it can be reported (SolveReport) and tested.

    * ``edges``: dependency edges (target u <- source v) by (target kind, source kind)
      and the tier SPEC assigns them: min(kernel_mode, natural tier), natural =
      row-row for a standalone source, sup-row for a supernode source into a
      standalone target, sup-sup for supernode into supernode.
    * ``update_order``: ROWROW mode runs every update in row-row operation order
      (running target value minus each source row's product, source rows ascending:
      the ``chain`` flag of the update kernels); SUPROW / SUPSUP apply supernode
      sources as blocks (TRSM multiplier block, product summed then subtracted once)
      — on supernode targets SUPROW and SUPSUP are the same arithmetic (oracle note 1).
    * ``kernels``: launches of the level fan-in plan per kernel — multiplier blocks
      (k_fi_x_w warp / k_fi_x CTA TRSM), update items (k_fi_upd_kcp packed DMMA,
      k_fi_upd_w warp GEMV for targets of <= WARP_ROWS rows, k_fi_upd_kc DMMA GEMM),
      split-K parts; the same grouping as run_fanin in csrc/hylu_abi.cu
      (``warp_min`` = option fanin_warp_min)."""
    from .symbolic import KernelMode
    m = int(sym.kernel_mode if mode is None else mode)
    kind = np.asarray(sym.node_kind)
    tgt = np.repeat(np.arange(sym.nnodes), np.diff(sym.dep_ptr))
    src = np.asarray(sym.deps)
    tk, sk = kind[tgt], kind[src]
    natural = np.where(sk == 0, 0, np.where(tk == 0, 1, 2))
    tier = np.minimum(natural, m)
    names = {(0, 0): "row<-row", (0, 1): "row<-sup", (1, 0): "sup<-row", (1, 1): "sup<-sup"}
    edges = {nm: int(np.sum((tk == a) & (sk == b))) for (a, b), nm in names.items()}
    tiers = {TIER_NAMES[t]: int(np.sum(tier == t)) for t in range(3)}
    out = {"kernel_mode": KernelMode(m).name, "edges": edges, "edge_tiers": tiers,
           "update_order": "row-row (chained)" if m == 0 else "block (summed, subtracted once)"}
    plan = getattr(sym, "_fanin_plan", None)
    if plan is not None:
        k = {"k_fi_x_w": 0, "k_fi_x": 0, "k_fi_upd_kcp": 0, "k_fi_upd_w": 0, "k_fi_upd_kc": 0}
        for lv in range(plan.nlevels):
            xp0, xp1, xb = int(plan.xp_ptr[lv]), int(plan.xp_ptr[lv + 1]), int(plan.lev_xp_big[lv])
            if xp1 > xp0:
                xb = xp0 if xb - xp0 < warp_min else xb
                k["k_fi_x_w"] += xb - xp0
                k["k_fi_x"] += xp1 - xb
            u0, u1 = int(plan.lev_up[lv]), int(plan.lev_up[lv + 1])
            if u1 > u0:
                reg, rs = int(plan.lev_up_reg[lv]), int(plan.lev_up_rs[lv])
                rs = reg if rs - reg < warp_min else rs
                k["k_fi_upd_kcp"] += reg - u0
                k["k_fi_upd_w"] += rs - reg
                k["k_fi_upd_kc"] += u1 - rs
        k["split_k_parts"] = int(np.sum(np.asarray(plan.up_part) >= 0))
        out["kernels"] = k
        out["tensor_core_items"] = k["k_fi_upd_kcp"] + k["k_fi_upd_kc"]
    return out
