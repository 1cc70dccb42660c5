// hylu_fanin.cu — level-synchronous fan-in supernodal factorization (SUPROW /
// SUPSUP modes, single instance).
//
// Every node (supernode or standalone row) is a dense rows x W block in node
// layout.  All A values are scattered once (k_fi_scatter).  Then, per level ℓ of
// the elimination DAG:
//   k_fi_lu    — each node finishing at ℓ has received every update: in-block LU
//                with pivoting restricted to the diagonal block
//                and pivot perturbation; standalone rows only
//                perturb their pivot.
//   k_fi_panel — row permutation of the node's other columns and the unit-lower
//                TRSM of its panel (U_panel = L_bb⁻¹ P·panel), tile-parallel.
//   k_fi_x     — for every edge (T, v) with v at level ℓ: the multiplier block
//                X = T[:, blk_v] · U_vv⁻¹ (the sup-row / sup-sup TRSM with the
//                source's upper, non-unit block), in place: these
//                are T's final L values.
//   k_fi_upd   — per (target T, 64-column tile): T[:, tile] -= Σ_v X_{T,v} ·
//                U_v[:, tile] over the level's sources v of T, accumulated in
//                shared memory (K-aggregated across sources) and written once.
// Sources finishing at the same level never touch each other's block columns
// (that would make one depend on the other), so all X blocks of a level are
// independent, and each target column receives its updates in ascending level
// order — the up-looking dependency order.  Supernode sources act as blocks in
// these modes (sup-row for row targets, sup-sup for supernode targets); the
// result differs from per-row application only in summation order.
#include "hylu_common.cuh"

namespace hy {

struct FaninDev {
  const int32_t *lu_nodes;   // nodes by level
  const int32_t *pt_node;    // perm / TRSM tiles
  const int32_t *pt_c0;
  const int32_t *pt_c1;
  const int64_t *xp_edge;    // X pairs: dependency edge index (target given by xp_tgt)
  const int32_t *xp_tgt;
  const int32_t *up_t;       // update items
  const int32_t *up_c0;
  const int32_t *up_c1;
  const int64_t *up_ptr;
  const int32_t *src_k;
  const int32_t *src_q0;
  const int32_t *src_q1;
  const int32_t *dep_pb;
  const int32_t *src_v;      // per source record: source node, block position, first block row
  const int32_t *src_pb;
  const int32_t *src_tb;
  const int32_t *up_part;    // split-K: part id per item (-1: unsplit)
  const int32_t *part_first;
  const int32_t *part_n;
  const int64_t *part_off;
  double *part_scr;          // partial tiles
  int *part_cnt;             // arrivals per split item (indexed by its first part id)
  // host-precomputed per source record (k_fi_upd_kc; null: derived on the device)
  const int64_t *src_poff;   // [nsrc+1] offsets into src_pos
  const int8_t *src_pos;     // tile position of each of the record's columns
  const int64_t *src_vb;     // source node value offset
  const int32_t *src_vW;     // source node width
  const int32_t *src_qb;     // first panel column of the record in the source
  const int32_t *src_m;      // source block rows from the first present one
  const ItemRec *up_rec;     // [items] packed prologue records (k_item_rec)
  const uint64_t *up_mask;   // [items] tile columns any source touches (k_item_mask; needs the maps)
  const XRec *xp_rec;        // [X items] packed records (k_x_rec)
  const NodeItemRec *lu_rec; // [LU items] / [panel items] packed records (k_node_rec)
  const NodeItemRec *pt_rec;
};

constexpr int FI_THREADS = 256;
constexpr int FXLD = 65;

// ---------------------------------------------------------------------------- scatter
// warp per M row: physical row = inverse of the prior inner_perm on refactorize
__device__ __forceinline__ void d_fi_scatter(DevSym S, const CallP *__restrict__ Pd, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  const int warp = (bid * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= S.n) return;
  const int i = warp;
  const int u = S.node_of[i];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  int t = i - r;
  int prow = t;
  if (P.refactor && s > 1) {
    // physical row p holds M row r + iperm[r+p]; find p with iperm[r+p] == t
    const int a0 = lane < s ? P.iperm_prior[r + lane] : -1;
    const int a1 = lane + 32 < s ? P.iperm_prior[r + lane + 32] : -1;
    const unsigned m0 = __ballot_sync(HY_FULL, a0 == t), m1 = __ballot_sync(HY_FULL, a1 == t);
    prow = m0 ? __ffs(m0) - 1 : 32 + __ffs(m1) - 1;
  }
  double *row = P.F + S.valoff[u] + (int64_t)prow * W;
  const int64_t a = S.mrow_src[i];
  for (int64_t e = S.a_ptr[a] + lane; e < S.a_ptr[a + 1]; e += 32) row[S.colpos[e]] = P.A[e] * S.scale[e];
}
__global__ void k_fi_scatter(DevSym S, const CallP *__restrict__ Pd) { d_fi_scatter(S, Pd, blockIdx.x); }

// ---------------------------------------------------------------------------- LU
__device__ __forceinline__ void d_fi_lu(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double lu_dyn[];
  double *B = lu_dyn;                  // [64 * FXLD] (dynamic: fi_lu_smem())
  __shared__ int perm[64];
  const NodeItemRec nr = D.lu_rec[base + bid];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = nr.r, s = nr.s, W = nr.W, L = nr.L;
  double *Pm = P.F + nr.valoff;
  const double thr = P.eps * P.anorm[0];
  if (s == 1) {
    if (tid == 0) {
      const double piv = Pm[L];
      bool fired;
      Pm[L] = perturb(piv, thr, fired);
      log_pivot(P, r, piv, fired, thr);
      P.iperm[r] = 0;
    }
    return;
  }
  for (int idx = tid; idx < s * s; idx += FI_THREADS) {
    const int t = idx / s, a = idx - t * s;
    B[t * FXLD + a] = Pm[(int64_t)t * W + L + a];
  }
  if (tid < s) perm[tid] = tid;
  __syncthreads();
  for (int t = 0; t < s; ++t) {
    if (!P.refactor && warp == 0) {
      double best = -1.0;
      int bi = s;
      for (int q = t + lane; q < s; q += 32) {
        const double av = fabs(B[q * FXLD + t]);
        if (av > best) { best = av; bi = q; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(HY_FULL, best, o);
        const int oi = __shfl_xor_sync(HY_FULL, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (bi != t && bi < s) {
        for (int c = lane; c < s; c += 32) {
          const double tmp = B[t * FXLD + c];
          B[t * FXLD + c] = B[bi * FXLD + c];
          B[bi * FXLD + c] = tmp;
        }
        if (lane == 0) {
          const int tp = perm[t];
          perm[t] = perm[bi];
          perm[bi] = tp;
        }
      }
    }
    // warp 0 (after its own pivot search and swap): perturb the pivot and scale
    // the column, then one barrier; the rank-1 update runs column-per-thread
    // (column tid&63, rows strided by 4), then the second barrier of the step
    if (warp == 0) {
      __syncwarp();
      double pv = B[t * FXLD + t];
      if (lane == 0) {
        bool fired;
        const double piv = pv;
        pv = perturb(piv, thr, fired);
        B[t * FXLD + t] = pv;
        log_pivot(P, r + t, piv, fired, thr);
      }
      pv = __shfl_sync(HY_FULL, pv, 0);
      for (int q = t + 1 + lane; q < s; q += 32) B[q * FXLD + t] /= pv;
    }
    __syncthreads();
    const int c = tid & 63;
    if (c > t && c < s) {
      const double ut = B[t * FXLD + c];
      for (int q = t + 1 + (tid >> 6); q < s; q += FI_THREADS / 64) B[q * FXLD + c] -= B[q * FXLD + t] * ut;
    }
    __syncthreads();
  }
  for (int idx = tid; idx < s * s; idx += FI_THREADS) {
    const int t = idx / s, a = idx - t * s;
    Pm[(int64_t)t * W + L + a] = B[t * FXLD + a];
  }
  if (tid < s) P.iperm[r + tid] = P.refactor ? P.iperm_prior[r + tid] : perm[tid];
}
__global__ void __launch_bounds__(FI_THREADS) k_fi_lu(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base) { d_fi_lu(S, Pd, D, base, blockIdx.x); }

// Single-row nodes of a level: their "LU" is the pivot perturbation (SPEC.md:320-328 with
// s = 1), one thread per node instead of a CTA each (c1's first levels list 10^4-10^5 of them).
__global__ void __launch_bounds__(256) k_fi_lu1(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base,
                                                int count) {
  pdl_wait();
  pdl_launch_dependents();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= count) return;
  const CallP P = *Pd;
  const NodeItemRec nr = D.lu_rec[base + k];
  const int r = nr.r;
  double *Pm = P.F + nr.valoff;
  const int L = nr.L;
  const double thr = P.eps * P.anorm[0];
  const double piv = Pm[L];
  bool fired;
  Pm[L] = perturb(piv, thr, fired);
  log_pivot(P, r, piv, fired, thr);
  P.iperm[r] = 0;
}

// ---------------------------------------------------------------------------- panel
// Tile of node v's columns [c0, c1) outside the block: apply the pivot row
// permutation (factorize only) and, for panel tiles, the unit-lower TRSM.
// Unit-lower TRSM of one panel column (thread `tid`), rows in register blocks of 16:
// a block first takes the updates of every earlier (final) row from shared memory,
// then its own triangle in registers.  Per element the updates are applied in
// ascending t, as in the plain column loop.
__device__ __forceinline__ void panel_trsm_col(double *tl, const double *Lb, int s, int tw, int tid) {
  constexpr int RB = 16;
  for (int q0 = 0; q0 < s; q0 += RB) {
    double x[RB];
#pragma unroll
    for (int q = 0; q < RB; ++q) x[q] = q0 + q < s ? tl[(q0 + q) * tw + tid] : 0.0;
    for (int t = 0; t < q0; ++t) {
      const double xt = tl[t * tw + tid];
#pragma unroll
      for (int q = 0; q < RB; ++q) x[q] -= Lb[(q0 + q) * FXLD + t] * xt;
    }
#pragma unroll
    for (int t = 0; t + 1 < RB; ++t) {
      const double xt = x[t];
#pragma unroll
      for (int q = t + 1; q < RB; ++q) x[q] -= Lb[(q0 + q) * FXLD + q0 + t] * xt;
    }
#pragma unroll
    for (int q = 0; q < RB; ++q)
      if (q0 + q < s) tl[(q0 + q) * tw + tid] = x[q];
  }
}

__device__ __forceinline__ void d_fi_panel(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double tl[];   // s x (c1-c0), stride PANEL
  double *Lb = tl + 64 * 256;                    // [64 * FXLD] after the tile (fi_panel_smem())
  __shared__ int perm[64];
  __shared__ int ident;
  const NodeItemRec nr = D.pt_rec[base + bid];
  const int c0 = nr.c0, c1 = nr.c1;
  const int tw = c1 - c0;
  const int tid = threadIdx.x;
  const int r = nr.r, s = nr.s, W = nr.W, L = nr.L;
  double *Pm = P.F + nr.valoff;
  const bool panel = c0 >= L + s;
  if (tid == 0) ident = 1;
  __syncthreads();
  if (tid < s) {
    perm[tid] = P.refactor ? tid : P.iperm[r + tid];
    if (perm[tid] != tid) ident = 0;
  }
  __syncthreads();
  if (ident && !panel) return;
  if (panel)
    for (int idx = tid; idx < s * s; idx += FI_THREADS) {
      const int t = idx / s, a = idx - t * s;
      Lb[t * FXLD + a] = Pm[(int64_t)t * W + L + a];
    }
  for (int idx = tid; idx < s * tw; idx += FI_THREADS) {
    const int t = idx / tw, c = idx - t * tw;
    tl[idx] = Pm[(int64_t)perm[t] * W + c0 + c];
  }
  __syncthreads();
  if (panel) {
    // unit-lower TRSM, one thread per column (tw <= FI_THREADS), the column held in
    // registers (one shared broadcast load per FMA instead of a shared
    // read-modify-write); no barriers, per-element update sequence (ascending t)
    // unchanged
    if (tid < tw) panel_trsm_col(tl, Lb, s, tw, tid);
    __syncthreads();
  }
  for (int idx = tid; idx < s * tw; idx += FI_THREADS) {
    const int t = idx / tw, c = idx - t * tw;
    Pm[(int64_t)t * W + c0 + c] = tl[idx];
  }
}
__global__ void __launch_bounds__(FI_THREADS) k_fi_panel(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base) { d_fi_panel(S, Pd, D, base, blockIdx.x); }

// ---------------------------------------------------------------------------- X blocks
// X = T[:, pb0 .. pb0+m) · U_bb⁻¹ in place; 4 threads per target row.
__device__ __forceinline__ void d_fi_x(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double xsm[];
  double *Ub = xsm;
  double *Xt = xsm + 64 * FXLD;
  const XRec xr0 = D.xp_rec[base + bid];
  const int tid = threadIdx.x, lane = tid & 31;
  const int s = xr0.s, W = xr0.W, vW = xr0.vW, m = xr0.m;
  const double *vb = P.F + xr0.u_off;   // row a of the source triangle at vb + a * vW, from column tb0
  double *Pm = P.F + xr0.t_off;         // target block (rows t at Pm + t * W)
  // warp per row, lanes over columns (no index divisions); the diagonal's
  // reciprocals are formed once, so the sequential loop multiplies instead of
  // dividing (x_a = w_a * (1/U_aa): within one rounding of the division)
  const int warp = tid >> 5;
  __shared__ double rinv[64];
  for (int a = warp; a < m; a += FI_THREADS / 32) {
    const double *urow = vb + (int64_t)a * vW;
    for (int b2 = lane; b2 < m; b2 += 32) {
      const double u = b2 >= a ? urow[b2] : 0.0;
      Ub[a * FXLD + b2] = u;
      if (b2 == a) rinv[a] = 1.0 / u;
    }
  }
  for (int t = warp; t < s; t += FI_THREADS / 32) {
    const double *xs = Pm + (int64_t)t * W;
    for (int a = lane; a < m; a += 32) Xt[t * FXLD + a] = xs[a];
  }
  __syncthreads();
  {
    // 4 threads per target row; thread qd holds the row's columns qd, qd+4, ... in
    // registers (16 values), so the sequential loop has no shared read-modify-write
    const int t = tid >> 2, qd = tid & 3;
    double *xr = Xt + t * FXLD;
    const bool act = t < s;
    double xi[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) xi[i] = (act && qd + 4 * i < m) ? xr[qd + 4 * i] : 0.0;
#pragma unroll
    for (int a = 0; a < 64; ++a) {
      if (a < m) {
        double x = 0.0;
        if ((a & 3) == qd) {
          x = xi[a >> 2] * rinv[a];
          xi[a >> 2] = x;
        }
        x = __shfl_sync(HY_FULL, x, (lane & ~3) | (a & 3));
        if (x != 0.0) {
#pragma unroll
          for (int i = (a + 1) >> 2; i < 16; ++i) {
            const int b2 = qd + 4 * i;
            if (b2 > a && b2 < m) xi[i] -= x * Ub[a * FXLD + b2];
          }
        }
      }
    }
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (act && qd + 4 * i < m) xr[qd + 4 * i] = xi[i];
  }
  __syncthreads();
  for (int t = warp; t < s; t += FI_THREADS / 32) {
    double *xd = Pm + (int64_t)t * W;
    for (int a = lane; a < m; a += 32) xd[a] = Xt[t * FXLD + a];
  }
}
__global__ void __launch_bounds__(FI_THREADS) k_fi_x(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base) { d_fi_x(S, Pd, D, base, blockIdx.x); }

// Warp-per-item multiplier blocks for small pairs (target <= 32 rows, <= 8 source
// rows): lane = target row, the row's multipliers in registers; per element the
// same operation sequence as k_fi_x (x_a = w_a / U_aa, then w_b -= x_a U_ab for
// b > a, skipped when x_a == 0).
constexpr int XW_M = 8;
__device__ __forceinline__ void d_fi_x_w(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int count, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jj = bid * (FI_THREADS / 32) + warp;
  if (jj >= count) return;
  const XRec xr0 = D.xp_rec[base + jj];
  const int s = xr0.s, W = xr0.W, vW = xr0.vW, m = xr0.m;
  const double *ub = P.F + xr0.u_off;   // row a of the source triangle at ub + a * vW, from column tb0
  double *Pm = P.F + xr0.t_off;
  if (lane >= s) return;
  double *row = Pm + (int64_t)lane * W;
  double xr[XW_M];
#pragma unroll
  for (int a = 0; a < XW_M; ++a) xr[a] = a < m ? row[a] : 0.0;
#pragma unroll
  for (int a = 0; a < XW_M; ++a) {
    if (a < m) {
      const double *ua = ub + (int64_t)a * vW;
      const double x = xr[a] / ua[a];
      xr[a] = x;
      if (x != 0.0)
#pragma unroll
        for (int b2 = a + 1; b2 < XW_M; ++b2)
          if (b2 < m) xr[b2] -= x * ua[b2];
    }
  }
#pragma unroll
  for (int a = 0; a < XW_M; ++a)
    if (a < m) row[a] = xr[a];
}
#ifndef XW_MINB
#define XW_MINB 6   // 40 registers: 48 resident warps/SM for the warp-per-item X kernel (c1 -1 %)
#endif
__global__ void __launch_bounds__(FI_THREADS, XW_MINB) k_fi_x_w(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int count) { d_fi_x_w(S, Pd, D, base, count, blockIdx.x); }

// Warp-per-item tile updates for small targets (<= 4 rows): lanes over the
// source's columns in the tile; per source c = Σ_a X[t][a] U[a][q] (ascending a,
// fused multiply-adds from zero), then the tile position of q gets -= c — the
// per-element sequence of k_fi_upd.  The tile lives in a per-warp shared buffer.
constexpr int UW_ROWS = 4;
constexpr int UW_TILE = 64;   // == FI_TILE
__device__ __forceinline__ void d_fi_upd_w(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int count, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double uw_dyn[];   // [FI_THREADS / 32][UW_ROWS * UW_TILE] (fi_upd_w_smem())
  double (*tile_s)[UW_ROWS * UW_TILE] = reinterpret_cast<double (*)[UW_ROWS * UW_TILE]>(uw_dyn);
  __shared__ int tcol_s[FI_THREADS / 32][UW_TILE];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jj = bid * (FI_THREADS / 32) + warp;
  if (jj >= count) return;
  const int j = base + jj;
  const int T = D.up_t[j];
  const int c0 = D.up_c0[j], c1 = D.up_c1[j];
  const int tw = c1 - c0;
  const int r = (int)S.first[T];
  const int s = (int)(S.first[T + 1] - r);
  const int64_t tc0 = S.colptr[T];
  const int W = (int)(S.colptr[T + 1] - tc0);
  double *Pm = P.F + S.valoff[T];
  double *acc = tile_s[warp];
  int *tcol = tcol_s[warp];
  for (int c = lane; c < tw; c += 32) {
    tcol[c] = S.cols[tc0 + c0 + c];
    for (int t = 0; t < s; ++t) acc[t * UW_TILE + c] = Pm[(int64_t)t * W + c0 + c];
  }
  __syncwarp();
  const bool maps = D.src_pos != nullptr;   // host-precomputed positions / metadata
  const bool chain = P.chain != 0;
  for (int64_t z = D.up_ptr[j]; z < D.up_ptr[j + 1]; ++z) {
    const int q0 = D.src_q0[z];
    const int nq = D.src_q1[z] - q0;
    const int pb0 = D.src_pb[z];
    const int tb0 = D.src_tb[z];
    int vW, m, qbase;
    int64_t vc0 = 0;
    const double *vb;
    if (maps) {
      vW = D.src_vW[z];
      m = D.src_m[z];
      qbase = D.src_qb[z];
      vb = P.F + D.src_vb[z];
    } else {
      const int v = D.src_v[z];
      const int vs = (int)(S.first[v + 1] - S.first[v]);
      vc0 = S.colptr[v];
      vW = (int)(S.colptr[v + 1] - vc0);
      vb = P.F + S.valoff[v];
      m = vs - tb0;
      qbase = S.nl[v] + vs + q0;
    }
    for (int q = lane; q < nq; q += 32) {
      const int pos = maps ? (int)D.src_pos[D.src_poff[z] + q]
                           : lower_bound_i32(tcol, 0, tw, S.cols[vc0 + qbase + q]);
      // sup-row order: c = sum_a x_a u_a, then one subtraction; row-row order (chain):
      // the running target value minus each source row's product in turn
      double c[UW_ROWS];
#pragma unroll
      for (int t = 0; t < UW_ROWS; ++t) c[t] = (chain && t < s) ? acc[t * UW_TILE + pos] : 0.0;
      for (int a = 0; a < m; ++a) {
        const double u = vb[(int64_t)(tb0 + a) * vW + qbase + q];
#pragma unroll
        for (int t = 0; t < UW_ROWS; ++t)
          if (t < s) {
            const double x = Pm[(int64_t)t * W + pb0 + a];
            c[t] = fma(chain ? -x : x, u, c[t]);
          }
      }
#pragma unroll
      for (int t = 0; t < UW_ROWS; ++t)
        if (t < s) acc[t * UW_TILE + pos] = chain ? c[t] : acc[t * UW_TILE + pos] - c[t];
    }
    __syncwarp();
  }
  for (int c = lane; c < tw; c += 32)
    for (int t = 0; t < s; ++t) Pm[(int64_t)t * W + c0 + c] = acc[t * UW_TILE + c];
}
#ifndef UPDW_MINB
#define UPDW_MINB 5   // 48 registers: 40 resident warps/SM for the warp-per-item update kernel (c1 3.67 -> 3.58 ms; 6 / 8 spill and are slower)
#endif
__global__ void __launch_bounds__(FI_THREADS, UPDW_MINB) k_fi_upd_w(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int count) { d_fi_upd_w(S, Pd, D, base, count, blockIdx.x); }

// ---------------------------------------------------------------------------- updates
constexpr int FI_TILE = 64;
static_assert(FI_TILE == UW_TILE, "warp update kernel assumes 64-column tiles");
constexpr int FI_KC = 32;      // K (source rows) chunk staged per pass
constexpr int KLD = FI_KC + 1;

// k_fi_upd's register-tiled product over one staged K chunk: NX row groups and NY
// column groups of 16 (the ones the source and target actually cover).
template <int NX, int NY>
__device__ __forceinline__ void fi_steps(const double *Xs, const double *Ut, int kc, int tr, int tcl,
                                         int s, double (&c4)[4][4]) {
#pragma unroll 4
  for (int a = 0; a < kc; ++a) {
    double xv[NX], uv[NY];
#pragma unroll
    for (int x = 0; x < NX; ++x) xv[x] = (tr + 16 * x < s) ? Xs[(tr + 16 * x) * KLD + a] : 0.0;
#pragma unroll
    for (int y = 0; y < NY; ++y) uv[y] = Ut[a * FXLD + tcl + 16 * y];
#pragma unroll
    for (int x = 0; x < NX; ++x)
#pragma unroll
      for (int y = 0; y < NY; ++y) c4[x][y] = fma(xv[x], uv[y], c4[x][y]);
  }
}

__global__ void __launch_bounds__(FI_THREADS) k_fi_upd(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base,
                                                       int Smax, int Mmax) {
  const CallP P = *Pd;
  extern __shared__ __align__(16) double fs[];
  __shared__ int tcol[FI_TILE];
  __shared__ int spos[FI_TILE];
  const int j = base + blockIdx.x;
  const int T = D.up_t[j];
  const int c0 = D.up_c0[j], c1 = D.up_c1[j];
  const int tw = c1 - c0;
  const int tid = threadIdx.x;
  const int r = (int)S.first[T];
  const int s = (int)(S.first[T + 1] - r);
  const int64_t tc0 = S.colptr[T];
  const int W = (int)(S.colptr[T + 1] - tc0);
  double *Pm = P.F + S.valoff[T];
  double *acc = fs;                          // s x FI_TILE
  double *Xs = acc + (size_t)Smax * FI_TILE; // Smax x KLD
  double *Ut = Xs + (size_t)Smax * KLD;      // FI_KC x FXLD
  (void)Mmax;
  for (int c = tid; c < tw; c += FI_THREADS) tcol[c] = S.cols[tc0 + c0 + c];
  for (int idx = tid; idx < s * FI_TILE; idx += FI_THREADS) {
    const int t = idx / FI_TILE, c = idx - t * FI_TILE;
    acc[idx] = c < tw ? Pm[(int64_t)t * W + c0 + c] : 0.0;
  }
  const int tr = tid >> 4, tcl = tid & 15;
  for (int64_t z = D.up_ptr[j]; z < D.up_ptr[j + 1]; ++z) {
    const int v = D.src_v[z];
    const int q0 = D.src_q0[z];
    const int nq = D.src_q1[z] - q0;
    const int vf = (int)S.first[v];
    const int vs = (int)(S.first[v + 1] - vf);
    const int64_t vc0 = S.colptr[v];
    const int vW = (int)(S.colptr[v + 1] - vc0);
    const int vnl = S.nl[v];
    const double *vb = P.F + S.valoff[v];
    const int pb0 = D.src_pb[z];
    const int tb0 = D.src_tb[z];
    const int m = vs - tb0;
    const int qbase = vnl + vs + q0;
    __syncthreads();
    if (tid < nq) spos[tid] = lower_bound_i32(tcol, 0, tw, S.cols[vc0 + qbase + tid]);
    double c4[4][4];
#pragma unroll
    for (int x = 0; x < 4; ++x)
#pragma unroll
      for (int y = 0; y < 4; ++y) c4[x][y] = 0.0;
    // only the source's columns (nq) and the target's rows (s) are computed: the
    // register tile shrinks to NX row groups x NY column groups of 16
    const int ny = nq <= 16 ? 1 : (nq <= 32 ? 2 : 4);
    const int nx = s <= 16 ? 1 : (s <= 32 ? 2 : 4);
    const int cw = 16 * ny;
    for (int k0 = 0; k0 < m; k0 += FI_KC) {
      const int kc = min(FI_KC, m - k0);
      if (k0) __syncthreads();
      for (int idx = tid; idx < s * kc; idx += FI_THREADS) {
        const int t = idx / kc, a = idx - t * kc;
        Xs[t * KLD + a] = Pm[(int64_t)t * W + pb0 + k0 + a];
      }
      for (int idx = tid; idx < kc * cw; idx += FI_THREADS) {
        const int a = idx / cw, c = idx - a * cw;
        Ut[a * FXLD + c] = c < nq ? vb[(int64_t)(tb0 + k0 + a) * vW + qbase + c] : 0.0;
      }
      __syncthreads();
      switch (nx * 8 + ny) {
        case 9: fi_steps<1, 1>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 10: fi_steps<1, 2>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 12: fi_steps<1, 4>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 17: fi_steps<2, 1>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 18: fi_steps<2, 2>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 20: fi_steps<2, 4>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 33: fi_steps<4, 1>(Xs, Ut, kc, tr, tcl, s, c4); break;
        case 34: fi_steps<4, 2>(Xs, Ut, kc, tr, tcl, s, c4); break;
        default: fi_steps<4, 4>(Xs, Ut, kc, tr, tcl, s, c4); break;
      }
    }
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int t = tr + 16 * x;
      if (t < s) {
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int c = tcl + 16 * y;
          if (c < nq) acc[t * FI_TILE + spos[c]] -= c4[x][y];
        }
      }
    }
  }
  __syncthreads();
  for (int idx = tid; idx < s * FI_TILE; idx += FI_THREADS) {
    const int t = idx / FI_TILE, c = idx - t * FI_TILE;
    if (c < tw) Pm[(int64_t)t * W + c0 + c] = acc[idx];
  }
}

// Sources of an item are packed into K-slices of <= FI_KC source rows: each
// slice's multiplier columns go to Xs and its U rows are scattered into the
// tile's 64-column space of Ut (zeros elsewhere), so one register-tiled GEMM
// handles many small sources per synchronisation round and the whole item is
// accumulated in registers (K-aggregated over all of its sources) before the
// tile is updated once.
__global__ void __launch_bounds__(FI_THREADS) k_fi_upd_pk(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base,
                                                       int Smax, int Mmax) {
  const CallP P = *Pd;
  extern __shared__ __align__(16) double fs[];
  __shared__ int tcol[FI_TILE];
  // slice descriptors of the current batch (built by warp 0)
  __shared__ int sl_n;                 // slices in batch
  __shared__ int sl_koff[FI_KC];       // first K row of the slice in Xs / Ut
  __shared__ int sl_m[FI_KC];          // rows in the slice
  __shared__ int sl_pb[FI_KC];         // target column of the slice's first multiplier
  __shared__ int sl_urow[FI_KC];       // first U row (within v) of the slice
  __shared__ int sl_nq[FI_KC];
  __shared__ int sl_qoff[FI_KC];
  __shared__ int sl_vW[FI_KC];
  __shared__ int64_t sl_vbase[FI_KC];
  __shared__ int64_t sl_vc0[FI_KC];
  __shared__ int64_t s_znext;
  __shared__ int s_anext;
  __shared__ int kmap[FI_KC];          // K row -> slice
  __shared__ int pcache[FI_KC][FI_TILE];  // tile position of each slice column
  const int j = base + blockIdx.x;
  const int T = D.up_t[j];
  const int c0 = D.up_c0[j], c1 = D.up_c1[j];
  const int tw = c1 - c0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int r = (int)S.first[T];
  const int s = (int)(S.first[T + 1] - r);
  const int64_t tc0 = S.colptr[T];
  const int W = (int)(S.colptr[T + 1] - tc0);
  double *Pm = P.F + S.valoff[T];
  double *Xs = fs;                           // Smax x KLD
  double *Ut = Xs + (size_t)Smax * KLD;      // FI_KC x FXLD
  (void)Mmax;
  for (int c = tid; c < tw; c += FI_THREADS) tcol[c] = S.cols[tc0 + c0 + c];
  const int tr = tid >> 4, tcl = tid & 15;
  double c4[4][4];
#pragma unroll
  for (int x = 0; x < 4; ++x)
#pragma unroll
    for (int y = 0; y < 4; ++y) c4[x][y] = 0.0;
  const int64_t z0 = D.up_ptr[j], z1 = D.up_ptr[j + 1];
  int64_t z = z0;
  int a0 = 0;            // first unprocessed row of source z
  while (z < z1) {
    __syncthreads();
    if (warp == 0) {
      // lanes fetch metadata of up to 32 upcoming sources; lane 0 packs the batch
      const int64_t zz = z + lane;
      int m = 0, nq = 0, pb = 0, tb = 0, vW = 0, qoff = 0;
      int64_t vb = 0, vc0 = 0;
      if (zz < z1) {
        const int v = D.src_v[zz];
        const int vf = (int)S.first[v];
        const int vs = (int)(S.first[v + 1] - vf);
        vc0 = S.colptr[v];
        vW = (int)(S.colptr[v + 1] - vc0);
        vb = S.valoff[v];
        pb = D.src_pb[zz];
        tb = D.src_tb[zz];
        m = vs - tb;
        const int q0 = D.src_q0[zz];
        nq = D.src_q1[zz] - q0;
        qoff = S.nl[v] + vs + q0;
      }
      // gather all lanes' metadata to lane-indexed smem, then lane 0 packs
      __shared__ int g_m[32], g_nq[32], g_pb[32], g_tb[32], g_vW[32], g_qoff[32];
      __shared__ int64_t g_vb[32], g_vc0[32];
      g_m[lane] = m; g_nq[lane] = nq; g_pb[lane] = pb; g_tb[lane] = tb; g_vW[lane] = vW;
      g_qoff[lane] = qoff; g_vb[lane] = vb; g_vc0[lane] = vc0;
      __syncwarp();
      if (lane == 0) {
        int k = 0, n = 0;
        int64_t zc = z;
        int ac = a0;
        while (zc < z1 && zc - z < 32 && k < FI_KC) {
          const int jj = (int)(zc - z);
          const int take = min(g_m[jj] - ac, FI_KC - k);
          for (int kk = 0; kk < take; ++kk) kmap[k + kk] = n;
          sl_koff[n] = k;
          sl_m[n] = take;
          sl_pb[n] = g_pb[jj] + ac;
          sl_urow[n] = g_tb[jj] + ac;
          sl_nq[n] = g_nq[jj];
          sl_qoff[n] = g_qoff[jj];
          sl_vW[n] = g_vW[jj];
          sl_vbase[n] = g_vb[jj];
          sl_vc0[n] = g_vc0[jj];
          ++n;
          k += take;
          ac += take;
          if (ac >= g_m[jj]) {
            ++zc;
            ac = 0;
          }
        }
        sl_n = n;
        s_znext = zc;
        s_anext = ac;
      }
    }
    __syncthreads();
    const int nsl = sl_n;
    const int kb = sl_koff[nsl - 1] + sl_m[nsl - 1];
    // Xs columns and zeroed Ut rows of the batch
    for (int idx = tid; idx < s * kb; idx += FI_THREADS) {
      const int t = idx / kb, a = idx - t * kb;
      const int q = kmap[a];
      Xs[t * KLD + a] = Pm[(int64_t)t * W + sl_pb[q] + (a - sl_koff[q])];
    }
    for (int idx = tid; idx < kb * FI_TILE; idx += FI_THREADS) Ut[(idx >> 6) * FXLD + (idx & 63)] = 0.0;
    for (int idx = tid; idx < nsl * FI_TILE; idx += FI_THREADS) {
      const int q = idx >> 6, c = idx & 63;
      if (c < sl_nq[q]) pcache[q][c] = lower_bound_i32(tcol, 0, tw, S.cols[sl_vc0[q] + sl_qoff[q] + c]);
    }
    __syncthreads();
    // scatter each slice's U rows into the tile's column space
    for (int idx = tid; idx < kb * FI_TILE; idx += FI_THREADS) {
      const int a = idx >> 6, c = idx & 63;
      const int q = kmap[a];
      if (c < sl_nq[q]) {
        const int ar = a - sl_koff[q];
        Ut[a * FXLD + pcache[q][c]] = P.F[sl_vbase[q] + (int64_t)(sl_urow[q] + ar) * sl_vW[q] + sl_qoff[q] + c];
      }
    }
    __syncthreads();
    for (int a = 0; a < kb; ++a) {
      double xv[4], uv[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) xv[x] = (tr + 16 * x < s) ? Xs[(tr + 16 * x) * KLD + a] : 0.0;
#pragma unroll
      for (int y = 0; y < 4; ++y) uv[y] = Ut[a * FXLD + tcl + 16 * y];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) c4[x][y] = fma(xv[x], uv[y], c4[x][y]);
    }
    z = s_znext;
    a0 = s_anext;
  }
  const int part = D.up_part ? D.up_part[j] : -1;
  if (part < 0) {
    // one update of the tile: T[:, tile] -= accumulated product
#pragma unroll
    for (int x = 0; x < 4; ++x) {
      const int t = tr + 16 * x;
      if (t < s) {
#pragma unroll
        for (int y = 0; y < 4; ++y) {
          const int c = tcl + 16 * y;
          if (c < tw) Pm[(int64_t)t * W + c0 + c] -= c4[x][y];
        }
      }
    }
    return;
  }
  // split-K part: publish the partial tile; the last part of the item adds the
  // partials in part order and updates the target once
  double *mine = D.part_scr + D.part_off[part];
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int t = tr + 16 * x;
    if (t < s)
#pragma unroll
      for (int y = 0; y < 4; ++y) mine[t * FI_TILE + tcl + 16 * y] = c4[x][y];
  }
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  const int first = D.part_first[part], np = D.part_n[part];
  if (tid == 0) s_last = atomicAdd(D.part_cnt + first, 1) == np - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int idx = tid; idx < s * FI_TILE; idx += FI_THREADS) {
    const int t = idx / FI_TILE, c = idx - t * FI_TILE;
    if (c >= tw) continue;
    double sum = 0.0;
    for (int k = 0; k < np; ++k) sum += __ldcg(D.part_scr + D.part_off[first + k] + t * FI_TILE + c);
    Pm[(int64_t)t * W + c0 + c] -= sum;
  }
  if (tid == 0) D.part_cnt[first] = 0;
}

// ---------------------------------------------------------------------------- updates, DMMA
// k_fi_upd with every per-source contraction on the FP64 tensor cores
// (mma.sync.aligned.m8n8k4 f64 -> SASS DMMA).  Warp tiles: 16 x 32 (4 x 2 warps
// over the 64 x 64 output) when the source covers more than 32 tile columns, else
// 8 x 32 (8 warps over the rows).  Each warp keeps its A fragments (one per 8-row
// block) and B fragments (one per 8-column block) in registers per k-step of 4, so
// a k-step costs 2 + 4 shared loads for 8 DMMAs (0.75 B/FMA vs 6 B/FMA for the 4x2
// FFMA register tile).  Staging is warp-per-row (one 256-byte line per load), no
// index divisions; the shared pitches (36 / 68 doubles) make the fragment loads
// conflict-free.  Per output element DMMA applies its four products as chained
// FMAs in k order, so the result equals k_fi_upd's bit for bit (tested).
constexpr int TC_XLD = 36;
constexpr int TC_ULD = 68;
size_t fi_upd_tc_smem(int smax) {
  return ((size_t)smax * FI_TILE + (size_t)smax * TC_XLD + (size_t)FI_KC * TC_ULD) * sizeof(double);
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(FI_THREADS, 3) k_fi_upd_tc(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base,
                                                          int Smax) {
  const CallP P = *Pd;
  extern __shared__ __align__(16) double fs[];
  __shared__ int tcol[FI_TILE];
  __shared__ int spos[FI_TILE];
  const int j = base + blockIdx.x;
  const int T = D.up_t[j];
  const int c0 = D.up_c0[j], c1 = D.up_c1[j];
  const int tw = c1 - c0;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, lr = lane >> 2;
  const int r = (int)S.first[T];
  const int s = (int)(S.first[T + 1] - r);
  const int64_t tc0 = S.colptr[T];
  const int W = (int)(S.colptr[T + 1] - tc0);
  double *Pm = P.F + S.valoff[T];
  double *acc = fs;                             // s x FI_TILE
  double *Xs = acc + (size_t)Smax * FI_TILE;    // Smax x TC_XLD
  double *Ut = Xs + (size_t)Smax * TC_XLD;      // FI_KC x TC_ULD
  for (int c = tid; c < tw; c += FI_THREADS) tcol[c] = S.cols[tc0 + c0 + c];
  for (int t = warp; t < s; t += FI_THREADS / 32) {
    const double *src = Pm + (int64_t)t * W + c0;
    acc[t * FI_TILE + lane] = lane < tw ? src[lane] : 0.0;
    acc[t * FI_TILE + lane + 32] = lane + 32 < tw ? src[lane + 32] : 0.0;
  }
  for (int64_t z = D.up_ptr[j]; z < D.up_ptr[j + 1]; ++z) {
    const int v = D.src_v[z];
    const int q0 = D.src_q0[z];
    const int nq = D.src_q1[z] - q0;
    const int vf = (int)S.first[v];
    const int vs = (int)(S.first[v + 1] - vf);
    const int64_t vc0 = S.colptr[v];
    const int vW = (int)(S.colptr[v + 1] - vc0);
    const double *vb = P.F + S.valoff[v];
    const int pb0 = D.src_pb[z];
    const int tb0 = D.src_tb[z];
    const int m = vs - tb0;
    const int qbase = S.nl[v] + vs + q0;
    const int ncw = (nq + 7) & ~7;
    // warp tile
    const bool wide = nq > 32;
    const int wr0 = wide ? (warp >> 1) * 16 : warp * 8;
    const int wc0 = wide ? (warp & 1) * 32 : 0;
    const int nrb = wide ? 2 : 1;
    double d[2][4][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) d[a][b][0] = d[a][b][1] = 0.0;
    bool ra[2], ca[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) ra[a] = a < nrb && wr0 + 8 * a < s;
#pragma unroll
    for (int b = 0; b < 4; ++b) ca[b] = wc0 + 8 * b < nq;
    __syncthreads();
    if (tid < nq) spos[tid] = lower_bound_i32(tcol, 0, tw, S.cols[vc0 + qbase + tid]);
    for (int k0 = 0; k0 < m; k0 += FI_KC) {
      const int kc = min(FI_KC, m - k0);
      const int kc4 = (kc + 3) & ~3;
      if (k0) __syncthreads();
      for (int t = warp; t < s; t += FI_THREADS / 32)
        if (lane < kc4) Xs[t * TC_XLD + lane] = lane < kc ? Pm[(int64_t)t * W + pb0 + k0 + lane] : 0.0;
      for (int a = warp; a < kc4; a += FI_THREADS / 32) {
        const double *urow = vb + (int64_t)(tb0 + k0 + a) * vW + qbase;
        const bool ok = a < kc;
        if (lane < ncw) Ut[a * TC_ULD + lane] = (ok && lane < nq) ? urow[lane] : 0.0;
        if (lane + 32 < ncw) Ut[a * TC_ULD + lane + 32] = (ok && lane + 32 < nq) ? urow[lane + 32] : 0.0;
      }
      __syncthreads();
      if (ra[0]) {
        for (int k = 0; k < kc4; k += 4) {
          double av[2], bv[4];
#pragma unroll
          for (int a = 0; a < 2; ++a) av[a] = ra[a] ? Xs[(wr0 + 8 * a + lr) * TC_XLD + k + kq] : 0.0;
#pragma unroll
          for (int b = 0; b < 4; ++b) bv[b] = ca[b] ? Ut[(k + kq) * TC_ULD + wc0 + 8 * b + lr] : 0.0;
#pragma unroll
          for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b)
              if (ra[a] && ca[b]) dmma884(d[a][b], av[a], bv[b]);
        }
      }
    }
    // scatter-subtract into the staged tile (row lr of each 8-row block, columns
    // 2*kq, 2*kq+1 of each 8-column block)
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int t = wr0 + 8 * a + lr;
      if (!ra[a] || t >= s) continue;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = wc0 + 8 * b + 2 * kq + e;
          if (ca[b] && c < nq) acc[t * FI_TILE + spos[c]] -= d[a][b][e];
        }
    }
  }
  __syncthreads();
  for (int t = warp; t < s; t += FI_THREADS / 32) {
    double *dst = Pm + (int64_t)t * W + c0;
    if (lane < tw) dst[lane] = acc[t * FI_TILE + lane];
    if (lane + 32 < tw) dst[lane + 32] = acc[t * FI_TILE + lane + 32];
  }
}

// ---------------------------------------------------------------------------- updates, K-concatenated DMMA
// One CTA per update item (target T, 64-column tile).  The K dimension is the
// concatenation of the item's sources' block rows, in chunks of <= FI_KC rows that
// never straddle a source; each chunk's U rows are scattered into the tile's
// 64-column space (cp.async with zero-fill for the columns the source does not
// cover), so the whole item is ONE register-resident GEMM
//     T[:, tile] -= X_item (s x K) * U_item (K x 64)
// on DMMA (mma.sync.m8n8k4 f64), warp tile 16 x 32, A/B fragments loaded once per
// k-step of 4 (2 + 4 shared loads per 8 DMMAs).  Chunk i+1 is in flight (cp.async,
// double-buffered) while chunk i is multiplied; the source -> tile column maps of a
// batch of sources are computed once up front (one parallel binary-search pass),
// so no per-source round trip or barrier sits between the tensor-core steps.  The
// target tile is read-modify-written once, straight from the accumulator
// fragments.  Summation order per element: all sources' products chained in
// ascending (source, row) order, then one subtraction — the packed kernel's order.

constexpr int KC_ULD = 68;
// Tile knobs, re-swept on the round-2 final kernels (factor ms, c2 / c3 k=32; defaults 286.9 / 107.3):
// KC_MINB 2: 324.5 / 118.1, 4: 315.2 / 115.8 (spills); KC_CHUNK 16: 297.0 / 115.0; KC_BIG 8: 288.1 / 107.4,
// 32: 286.9 / 107.2; KC_NSB 8: 289.5 / 107.7, 32: 288.6 / 107.6 (profiles/r02_kc_knob_sweep_final.txt).
#ifndef KC_NSB_DEF
#define KC_NSB_DEF 16
#endif
constexpr int KC_NSB = KC_NSB_DEF;     // sources per column-map batch (multi-batch path: > KC_NSB sources)
#ifndef KC_CHUNK_DEF
#define KC_CHUNK_DEF 32
#endif
#ifndef KC_MINB_DEF
#define KC_MINB_DEF 3
#endif
constexpr int KC_K = KC_CHUNK_DEF;   // K rows per chunk (<= 32: one lane per X column)
#ifndef KC_BIG_DEF
#define KC_BIG_DEF 16
#endif
constexpr int KC_BIG = KC_BIG_DEF;   // sources with at least this many rows get their own chunks
constexpr int KC_XLD = KC_K + 4;     // pitches == 4 (mod 16) doubles: conflict-free fragments
// one pipeline stage: an X chunk then a U chunk; it also holds the s x 64 target tile
// prefetched for the epilogue
constexpr int KC_STAGE = (64 * KC_XLD + KC_K * KC_ULD) > 64 * 64 ? (64 * KC_XLD + KC_K * KC_ULD) : 64 * 64;
size_t fi_upd_kc_smem() {
  return 2 * (size_t)KC_STAGE * sizeof(double) + (size_t)KC_NSB * 64;
}

__device__ __forceinline__ void kc_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void kc_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void kc_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async8z(double *smem_dst, const double *gsrc, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  const int n = ok ? 8 : 0;   // src-size 0: the 8 bytes are zero-filled, nothing is read
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(gsrc), "r"(n) : "memory");
}

// DMMA without `volatile`: the compiler may schedule the fragment loads of the next
// k-step across the MMAs
__device__ __forceinline__ void dmma884s(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// One staged K chunk of a warp's 16 (or 8) x 32 output tile.  Full tiles (every
// 8-row and 8-column block live: the bulk of the c2/c3 work) run a predicate-free
// loop; partial ones skip dead blocks warp-uniformly.  CHAIN negates the multipliers
// (row-row operation order, see k_fi_upd_kc).
template <bool CHAIN, int NA>
__device__ __forceinline__ void kc_chunk_full(const double *X, const double *U, int kc4, int wr0, int wc0,
                                              int lr, int kq, double (&d)[2][4][2]) {
#pragma unroll 2
  for (int k = 0; k < kc4; k += 4) {
    double av[NA], bv[4];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      av[a] = X[(wr0 + 8 * a + lr) * KC_XLD + k + kq];
      if (CHAIN) av[a] = -av[a];
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = U[(k + kq) * KC_ULD + wc0 + 8 * b + lr];
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) dmma884s(d[a][b], av[a], bv[b]);
  }
}

template <bool CHAIN>
__device__ __forceinline__ void kc_chunk(const double *X, const double *U, int kc4, int wr0, int wc0, int lr,
                                         int kq, const bool (&ra)[2], const bool (&cb)[4], unsigned bm,
                                         double (&d)[2][4][2]) {
  if (!ra[0] || !(bm & 15u)) return;
  if (cb[0] && cb[1] && cb[2] && cb[3]) {
    if (ra[1]) kc_chunk_full<CHAIN, 2>(X, U, kc4, wr0, wc0, lr, kq, d);
    else kc_chunk_full<CHAIN, 1>(X, U, kc4, wr0, wc0, lr, kq, d);
    return;
  }
  for (int k = 0; k < kc4; k += 4) {
    double av[2], bv[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      av[a] = ra[a] ? X[(wr0 + 8 * a + lr) * KC_XLD + k + kq] : 0.0;
      if (CHAIN) av[a] = -av[a];
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) bv[b] = cb[b] ? U[(k + kq) * KC_ULD + wc0 + 8 * b + lr] : 0.0;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (ra[a] && cb[b]) dmma884s(d[a][b], av[a], bv[b]);
  }
}

template <bool CHAIN>
__device__ __forceinline__ void d_fi_upd_kc(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double fs[];
  __shared__ int tcol[FI_TILE];
  __shared__ int8_t cidx[FI_TILE];     // tile column -> compact column (-1: untouched)
  __shared__ int8_t ucol[FI_TILE];     // compact column -> tile column
  __shared__ int s_nu;
  __shared__ int64_t s_vb[KC_NSB];
  __shared__ int s_vW[KC_NSB], s_qb[KC_NSB], s_pb[KC_NSB], s_tb[KC_NSB], s_m[KC_NSB];
  __shared__ unsigned s_bm[KC_NSB];   // 8-column blocks (compact space) a source touches
  const int j = base + bid;
  const ItemRec ir = D.up_rec[j];
  const int c0 = ir.c0;
  const int tw = ir.tw;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, lr = lane >> 2;
  const int s = ir.s;
  const int W = ir.W;
  double *Pm = P.F + ir.valoff;
  constexpr int KC_BUF = KC_STAGE;
  int8_t *inv = reinterpret_cast<int8_t *>(fs + 2 * KC_BUF);   // [KC_NSB][64] source col -> compact col
  const int64_t zb = ir.zb, ze = ir.zb + ir.nz;
  const bool compact = ze - zb <= KC_NSB;
  if (!D.src_pos || !compact) {   // the tile's column indices, for the column-map searches
    const int64_t tc0 = S.colptr[D.up_t[j]];
    for (int c = tid; c < tw; c += FI_THREADS) tcol[c] = S.cols[tc0 + c0 + c];
  }
  if (compact && D.src_pos && D.up_mask) {
    // the item's touched tile columns are a precomputed 64-bit mask: a source
    // column's compact index is the popcount of the mask below its tile position,
    // so the maps and 8-column block masks are built in one pass, one barrier
    const uint64_t mask = D.up_mask[j];
    if (warp == 0) {
      for (int c = lane; c < 64; c += 32)
        if ((mask >> c) & 1ull) ucol[__popcll(mask & ((1ull << c) - 1ull))] = (int8_t)c;
      if (lane == 0) s_nu = __popcll(mask);
    }
    for (int k = warp; k < (int)(ze - zb); k += FI_THREADS / 32) {
      const int64_t z = zb + k;
      const int nq = D.src_q1[z] - D.src_q0[z];
      if (lane == 0) {
        s_vb[k] = D.src_vb[z];
        s_vW[k] = D.src_vW[z];
        s_qb[k] = D.src_qb[z];
        s_pb[k] = D.src_pb[z];
        s_tb[k] = D.src_tb[z];
        s_m[k] = D.src_m[z];
      }
      const int8_t *pz = D.src_pos + D.src_poff[z];
      int cp0 = -1, cp1 = -1;
      if (lane < nq) cp0 = __popcll(mask & ((1ull << pz[lane]) - 1ull));
      if (lane + 32 < nq) cp1 = __popcll(mask & ((1ull << pz[lane + 32]) - 1ull));
      inv[k * 64 + lane] = -1;
      inv[k * 64 + lane + 32] = -1;
      __syncwarp();
      unsigned bits = 0;
      if (cp0 >= 0) { inv[k * 64 + cp0] = (int8_t)lane; bits |= 1u << (cp0 >> 3); }
      if (cp1 >= 0) { inv[k * 64 + cp1] = (int8_t)(lane + 32); bits |= 1u << (cp1 >> 3); }
      bits = __reduce_or_sync(HY_FULL, bits);
      if (lane == 0) s_bm[k] = bits;
    }
  } else {
  if (tid < FI_TILE) cidx[tid] = compact ? -1 : (int8_t)tid;
  __syncthreads();
  if (compact) {
    // tile columns any source touches -> compact column space [0, nu); the source
    // column maps are written with compact indices (inv doubles as scratch for the
    // tile positions first)
    for (int k = warp; k < (int)(ze - zb); k += FI_THREADS / 32) {
      const int64_t z = zb + k;
      const int nq = D.src_q1[z] - D.src_q0[z];
      if (D.src_pos) {
        // host-precomputed: metadata and the tile position of every source column
        // (one round of independent loads, no binary search)
        if (lane == 0) {
          s_vb[k] = D.src_vb[z];
          s_vW[k] = D.src_vW[z];
          s_qb[k] = D.src_qb[z];
          s_pb[k] = D.src_pb[z];
          s_tb[k] = D.src_tb[z];
          s_m[k] = D.src_m[z];
        }
        const int8_t *pz = D.src_pos + D.src_poff[z];
        for (int c = lane; c < 64; c += 32) {
          int pos = -1;
          if (c < nq) {
            pos = pz[c];
            cidx[pos] = 1;
          }
          inv[k * 64 + c] = (int8_t)pos;
        }
        continue;
      }
      const int v = D.src_v[z];
      const int vs = (int)(S.first[v + 1] - S.first[v]);
      const int64_t vcol = S.colptr[v];
      const int qb = S.nl[v] + vs + D.src_q0[z];
      const int64_t vc = vcol + qb;
      if (lane == 0) {   // per-source metadata for the chunk loop (single batch)
        const int tb0 = D.src_tb[z];
        s_vb[k] = S.valoff[v];
        s_vW[k] = (int)(S.colptr[v + 1] - vcol);
        s_qb[k] = qb;
        s_pb[k] = D.src_pb[z];
        s_tb[k] = tb0;
        s_m[k] = vs - tb0;
      }
      for (int c = lane; c < 64; c += 32) {
        int pos = -1;
        if (c < nq) {
          pos = lower_bound_i32(tcol, 0, tw, S.cols[vc + c]);
          cidx[pos] = 1;
        }
        inv[k * 64 + c] = (int8_t)pos;
      }
    }
    __syncthreads();
    if (warp == 0) {
      const bool t0 = cidx[lane] == 1, t1 = cidx[lane + 32] == 1;
      const unsigned m0 = __ballot_sync(HY_FULL, t0), m1 = __ballot_sync(HY_FULL, t1);
      const int below = __popc(m0 & ((1u << lane) - 1));
      const int i0 = below, i1 = __popc(m0) + __popc(m1 & ((1u << lane) - 1));
      cidx[lane] = t0 ? (int8_t)i0 : -1;
      cidx[lane + 32] = t1 ? (int8_t)i1 : -1;
      if (t0) ucol[i0] = (int8_t)lane;
      if (t1) ucol[i1] = (int8_t)(lane + 32);
      if (lane == 0) s_nu = __popc(m0) + __popc(m1);
    }
    __syncthreads();
    // inv[k][tile pos] -> inv[k][compact col] = source col
    for (int k = warp; k < (int)(ze - zb); k += FI_THREADS / 32) {
      const int p0 = inv[k * 64 + lane], p1 = inv[k * 64 + lane + 32];
      __syncwarp();
      inv[k * 64 + lane] = -1;
      inv[k * 64 + lane + 32] = -1;
      __syncwarp();
      if (p0 >= 0) inv[k * 64 + cidx[p0]] = (int8_t)lane;
      if (p1 >= 0) inv[k * 64 + cidx[p1]] = (int8_t)(lane + 32);
      __syncwarp();
      // compact 8-column blocks this source has entries in
      const unsigned m0 = __ballot_sync(HY_FULL, inv[k * 64 + lane] >= 0);
      const unsigned m1 = __ballot_sync(HY_FULL, inv[k * 64 + lane + 32] >= 0);
      if (lane == 0) {
        unsigned bm = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if ((m0 >> (8 * b)) & 0xffu) bm |= 1u << b;
          if ((m1 >> (8 * b)) & 0xffu) bm |= 1u << (b + 4);
        }
        s_bm[k] = bm;
      }
    }
  } else {
    if (tid < FI_TILE) ucol[tid] = (int8_t)tid;
    if (tid == 0) s_nu = tw;
  }
  }   // compact column space
  __syncthreads();
  const int nu = s_nu;
  // warp tiles over the s x nu product: 8 x 32 (8 warps over the rows) when the
  // item touches <= 32 columns, else 16 x 32 (4 x 2 warps)
  const bool narrow = nu <= 32;
  const int wr0 = narrow ? warp * 8 : (warp >> 1) * 16;
  const int wc0 = narrow ? 0 : (warp & 1) * 32;
  bool ra[2], ca[4];
  ra[0] = wr0 < s;
  ra[1] = !narrow && wr0 + 8 < s;
#pragma unroll
  for (int b = 0; b < 4; ++b) ca[b] = wc0 + 8 * b < nu;
  // row-row order (chain): the accumulators start at the target's values and the
  // multipliers enter negated, so DMMA's chained FMAs subtract every source row's
  // product from the running value in (source, row) order; else they start at 0
  // and the sum is subtracted once in the epilogue
  const bool chain = CHAIN;
  double d[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = wr0 + 8 * a + lr, c = wc0 + 8 * b + 2 * kq + e;
        d[a][b][e] = (chain && ra[a] && t < s && ca[b] && c < nu) ? Pm[(int64_t)t * W + c0 + ucol[c]] : 0.0;
      }

  for (int64_t zb0 = zb; zb0 < ze; zb0 += KC_NSB) {
    const int nsb = (int)(ze - zb0 < KC_NSB ? ze - zb0 : KC_NSB);
    const bool last_batch = zb0 + KC_NSB >= ze;
    if (zb0 != zb) __syncthreads();   // previous batch's chunks consumed
    if (!compact && tid < nsb) {
      const int64_t z = zb0 + tid;
      const int v = D.src_v[z];
      const int vs = (int)(S.first[v + 1] - S.first[v]);
      const int tb0 = D.src_tb[z];
      s_vb[tid] = S.valoff[v];
      s_vW[tid] = (int)(S.colptr[v + 1] - S.colptr[v]);
      s_qb[tid] = S.nl[v] + vs + D.src_q0[z];
      s_pb[tid] = D.src_pb[z];
      s_tb[tid] = tb0;
      s_m[tid] = vs - tb0;
    }
    if (!compact) {
      for (int q = tid; q < nsb * 64; q += FI_THREADS) inv[q] = -1;
      __syncthreads();
      for (int k = warp; k < nsb; k += FI_THREADS / 32) {
        const int64_t z = zb0 + k;
        const int v = D.src_v[z];
        const int nq = D.src_q1[z] - D.src_q0[z];
        const int64_t vc = S.colptr[v] + s_qb[k];
        for (int c = lane; c < nq; c += 32) inv[k * 64 + lower_bound_i32(tcol, 0, tw, S.cols[vc + c])] = (int8_t)c;
      }
      __syncthreads();
    }
    // per source: the compact 8-column blocks it has entries in (its other blocks of
    // U are zero: those DMMAs are skipped, warp-uniformly); the compact path computed
    // them with the column maps
    for (int k = warp; k < nsb && !compact; k += FI_THREADS / 32) {
      const unsigned m0 = __ballot_sync(HY_FULL, inv[k * 64 + lane] >= 0);
      const unsigned m1 = __ballot_sync(HY_FULL, inv[k * 64 + lane + 32] >= 0);
      if (lane == 0) {
        unsigned bm = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if ((m0 >> (8 * b)) & 0xffu) bm |= 1u << b;
          if ((m1 >> (8 * b)) & 0xffu) bm |= 1u << (b + 4);
        }
        s_bm[k] = bm;
      }
    }
    if (!compact) __syncthreads();   // (compact: published by the barrier after the maps)
    auto issue = [&](int k, int k0, int buf) {
      const int kc = min(KC_K, s_m[k] - k0);
      const double *xs = Pm + s_pb[k] + k0;
      double *X = fs + buf * KC_BUF;
      if (lane < KC_K)
        for (int t = warp; t < s; t += FI_THREADS / 32)
          cp_async8z(X + t * KC_XLD + lane, xs + (int64_t)t * W + (lane < kc ? lane : 0), lane < kc);
      const double *ub = P.F + s_vb[k] + (int64_t)(s_tb[k] + k0) * s_vW[k] + s_qb[k];
      double *U = X + 64 * KC_XLD;
      const int i0 = inv[k * 64 + lane], i1 = inv[k * 64 + lane + 32];
      const bool w1 = lane + 32 < nu;   // compact columns beyond nu are never read
      for (int a = warp; a < KC_K; a += FI_THREADS / 32) {
        const double *ur = ub + (int64_t)(a < kc ? a : 0) * s_vW[k];
        cp_async8z(U + a * KC_ULD + lane, ur + (i0 >= 0 ? i0 : 0), a < kc && i0 >= 0);
        if (w1) cp_async8z(U + a * KC_ULD + lane + 32, ur + (i1 >= 0 ? i1 : 0), a < kc && i1 >= 0);
      }
    };
    int ck = 0, ck0 = 0, buf = 0;       // chunk being computed
    issue(0, 0, 0);
    kc_commit();
    for (;;) {
      int nk = ck, nk0 = ck0 + KC_K;
      if (nk0 >= s_m[nk]) { ++nk; nk0 = 0; }
      const bool more = nk < nsb;
      if (more) {
        issue(nk, nk0, buf ^ 1);
      } else if (last_batch) {
        // the target's touched tile values, into the free stage, for the epilogue
        double *Tv = fs + (buf ^ 1) * KC_BUF;
        for (int t = warp; t < s; t += FI_THREADS / 32) {
          const double *prow = Pm + (int64_t)t * W + c0;
          if (lane < nu) cp_async8z(Tv + t * 64 + lane, prow + ucol[lane], true);
          if (lane + 32 < nu) cp_async8z(Tv + t * 64 + lane + 32, prow + ucol[lane + 32], true);
        }
      }
      kc_commit();
      kc_wait1();
      __syncthreads();
      const int kc = min(KC_K, s_m[ck] - ck0);
      const int kc4 = (kc + 3) & ~3;
      const double *X = fs + buf * KC_BUF, *U = X + 64 * KC_XLD;
      const unsigned bm = s_bm[ck] >> (wc0 >> 3);
      bool cb[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) cb[b] = ca[b] && ((bm >> b) & 1u);
      kc_chunk<CHAIN>(X, U, kc4, wr0, wc0, lr, kq, ra, cb, bm, d);
      if (!more) break;
      __syncthreads();   // buffer `buf` free for the chunk after next
      ck = nk; ck0 = nk0; buf ^= 1;
    }
    if (last_batch) {
      kc_wait0();
      __syncthreads();
      // T[:, tile] -= product (row lr of each 8-row block, compact columns 2*kq, 2*kq+1)
      const double *Tv = fs + (buf ^ 1) * KC_BUF;
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int t = wr0 + 8 * a + lr;
        if (!ra[a] || t >= s) continue;
        double *prow = Pm + (int64_t)t * W + c0;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = wc0 + 8 * b + 2 * kq + e;
            if (ca[b] && c < nu) prow[ucol[c]] = chain ? d[a][b][e] : Tv[t * 64 + c] - d[a][b][e];
          }
      }
    }
  }
}
template <bool CHAIN>
__global__ void __launch_bounds__(FI_THREADS, KC_MINB_DEF) k_fi_upd_kc(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base) { d_fi_upd_kc<CHAIN>(S, Pd, D, base, blockIdx.x); }

// k_fi_upd_kcp: k_fi_upd_kc for the packed items (many small sources): chunks hold
// up to KC_K rows of consecutive sources (sources of >= KC_BIG rows still get their
// own chunks), so a synchronisation round covers several sources; split-K parts of
// outlier items publish partial tiles (tile column space) and the last part adds
// them in part order.  Replaces k_fi_upd_pk (fanin_tc=5): c2 350 -> 340 ms.
template <bool CHAIN>
__device__ __forceinline__ void d_fi_upd_kcp(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base, int bid) {
  pdl_wait();
  pdl_launch_dependents();
  const CallP P = *Pd;
  extern __shared__ __align__(16) double fs[];
  __shared__ int tcol[FI_TILE];
  __shared__ int8_t cidx[FI_TILE];     // tile column -> compact column (-1: untouched)
  __shared__ int8_t ucol[FI_TILE];     // compact column -> tile column
  __shared__ int s_nu;
  __shared__ int64_t s_vb[KC_NSB];
  __shared__ int s_vW[KC_NSB], s_qb[KC_NSB], s_pb[KC_NSB], s_tb[KC_NSB], s_m[KC_NSB];
  __shared__ int s_koff[KC_NSB + 1];   // first K row of each source of the batch
  __shared__ unsigned s_bm[KC_NSB];    // 8-column blocks (compact space) a source touches
  __shared__ int8_t ksrc[KC_NSB * 64]; // K row -> source of the batch
  __shared__ int s_cst[KC_NSB * 64 / 4 + KC_NSB + 2];   // chunk start rows (+ end)
  __shared__ int s_nch;
  const int j = base + bid;
  const ItemRec ir = D.up_rec[j];
  const int c0 = ir.c0;
  const int tw = ir.tw;
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31, kq = lane & 3, lr = lane >> 2;
  const int s = ir.s;
  const int W = ir.W;
  double *Pm = P.F + ir.valoff;
  constexpr int KC_BUF = KC_STAGE;
  int8_t *inv = reinterpret_cast<int8_t *>(fs + 2 * KC_BUF);   // [KC_NSB][64] source col -> compact col
  const int part = D.up_part ? D.up_part[j] : -1;               // split-K part (packed items)
  const int64_t zb = ir.zb, ze = ir.zb + ir.nz;
  // split-K parts publish whole tiles: no column compaction for them
  const bool compact = ze - zb <= KC_NSB && part < 0;
  if (!D.src_pos || !compact) {   // the tile's column indices, for the column-map searches
    const int64_t tc0 = S.colptr[D.up_t[j]];
    for (int c = tid; c < tw; c += FI_THREADS) tcol[c] = S.cols[tc0 + c0 + c];
  }
  if (tid < FI_TILE) cidx[tid] = compact ? -1 : (int8_t)tid;
  __syncthreads();
  // per-source metadata and column maps of a batch of <= KC_NSB sources; `pos`
  // mode (compact first pass) stores tile positions and marks touched columns
  auto source_maps = [&](int64_t zb0, int nsb, bool pos) {
    for (int k = warp; k < nsb; k += FI_THREADS / 32) {
      const int64_t z = zb0 + k;
      const int nq = D.src_q1[z] - D.src_q0[z];
      if (D.src_pos) {   // host-precomputed maps (hy_upload_fanin_maps)
        if (lane == 0) {
          s_vb[k] = D.src_vb[z];
          s_vW[k] = D.src_vW[z];
          s_qb[k] = D.src_qb[z];
          s_pb[k] = D.src_pb[z];
          s_tb[k] = D.src_tb[z];
          s_m[k] = D.src_m[z];
        }
        const int8_t *pz = D.src_pos + D.src_poff[z];
        for (int c = lane; c < 64; c += 32) {
          int p = -1;
          if (c < nq) {
            p = pz[c];
            if (pos) cidx[p] = 1;
          }
          inv[k * 64 + c] = (int8_t)p;
        }
        continue;
      }
      const int v = D.src_v[z];
      const int vs = (int)(S.first[v + 1] - S.first[v]);
      const int64_t vcol = S.colptr[v];
      const int qb = S.nl[v] + vs + D.src_q0[z];
      const int64_t vc = vcol + qb;
      const int tb0 = D.src_tb[z];
      if (lane == 0) {
        s_vb[k] = S.valoff[v];
        s_vW[k] = (int)(S.colptr[v + 1] - vcol);
        s_qb[k] = qb;
        s_pb[k] = D.src_pb[z];
        s_tb[k] = tb0;
        s_m[k] = vs - tb0;
      }
      for (int c = lane; c < 64; c += 32) {
        int p = -1;
        if (c < nq) {
          p = lower_bound_i32(tcol, 0, tw, S.cols[vc + c]);
          if (pos) cidx[p] = 1;
        }
        inv[k * 64 + c] = (int8_t)p;   // tile position of source column c
      }
    }
  };
  // tile positions -> compact columns (inv[k][compact col] = source col), block masks
  auto remap = [&](int nsb) {
    for (int k = warp; k < nsb; k += FI_THREADS / 32) {
      const int p0 = inv[k * 64 + lane], p1 = inv[k * 64 + lane + 32];
      __syncwarp();
      inv[k * 64 + lane] = -1;
      inv[k * 64 + lane + 32] = -1;
      __syncwarp();
      if (p0 >= 0) inv[k * 64 + cidx[p0]] = (int8_t)lane;
      if (p1 >= 0) inv[k * 64 + cidx[p1]] = (int8_t)(lane + 32);
      __syncwarp();
      const unsigned m0 = __ballot_sync(HY_FULL, inv[k * 64 + lane] >= 0);
      const unsigned m1 = __ballot_sync(HY_FULL, inv[k * 64 + lane + 32] >= 0);
      if (lane == 0) {
        unsigned bm = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          if ((m0 >> (8 * b)) & 0xffu) bm |= 1u << b;
          if ((m1 >> (8 * b)) & 0xffu) bm |= 1u << (b + 4);
        }
        s_bm[k] = bm;
      }
    }
  };
  // K layout of a batch: sources' rows concatenated (koff prefix sums, row -> source)
  auto k_layout = [&](int nsb) {
    if (warp == 0) {
      int m = lane < nsb ? s_m[lane] : 0;
      int incl = m;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(HY_FULL, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane < nsb) s_koff[lane] = incl - m;
      if (lane == nsb - 1) s_koff[nsb] = incl;
      __syncwarp();
      if (lane == 0) {
        // chunk boundaries: sources of >= KC_BIG rows start a chunk and are cut in
        // KC_K-row pieces (no straddling: their 8-column block masks stay tight);
        // smaller sources are packed together up to KC_K rows
        int nch = 0, open = -1;
        for (int k = 0; k < nsb; ++k) {
          const int off = s_koff[k], mk = s_m[k];
          if (mk >= KC_BIG) {
            if (open >= 0) { s_cst[nch++] = open; open = -1; }
            for (int q = 0; q < mk; q += KC_K) s_cst[nch++] = off + q;
          } else if (mk > 0) {
            if (open >= 0 && off + mk - open > KC_K) { s_cst[nch++] = open; open = -1; }
            if (open < 0) open = off;
          }
        }
        if (open >= 0) s_cst[nch++] = open;
        s_cst[nch] = s_koff[nsb];
        s_nch = nch;
      }
    }
    __syncthreads();
    for (int k = warp; k < nsb; k += FI_THREADS / 32)
      for (int rr = lane; rr < s_m[k]; rr += 32) ksrc[s_koff[k] + rr] = (int8_t)k;
  };
  if (compact) {
    const int nsb = (int)(ze - zb);
    source_maps(zb, nsb, true);
    __syncthreads();
    if (warp == 0) {
      const bool t0 = cidx[lane] == 1, t1 = cidx[lane + 32] == 1;
      const unsigned m0 = __ballot_sync(HY_FULL, t0), m1 = __ballot_sync(HY_FULL, t1);
      const int i0 = __popc(m0 & ((1u << lane) - 1)), i1 = __popc(m0) + __popc(m1 & ((1u << lane) - 1));
      cidx[lane] = t0 ? (int8_t)i0 : -1;
      cidx[lane + 32] = t1 ? (int8_t)i1 : -1;
      if (t0) ucol[i0] = (int8_t)lane;
      if (t1) ucol[i1] = (int8_t)(lane + 32);
      if (lane == 0) s_nu = __popc(m0) + __popc(m1);
    }
    __syncthreads();
    remap(nsb);
  } else {
    if (tid < FI_TILE) ucol[tid] = (int8_t)tid;
    if (tid == 0) s_nu = tw;
  }
  __syncthreads();
  const int nu = s_nu;
  // warp tiles over the s x nu product: 8 x 32 (8 warps over the rows) when the
  // item touches <= 32 columns, else 16 x 32 (4 x 2 warps)
  const bool narrow = nu <= 32;
  const int wr0 = narrow ? warp * 8 : (warp >> 1) * 16;
  const int wc0 = narrow ? 0 : (warp & 1) * 32;
  bool ra[2], ca[4];
  ra[0] = wr0 < s;
  ra[1] = !narrow && wr0 + 8 < s;
#pragma unroll
  for (int b = 0; b < 4; ++b) ca[b] = wc0 + 8 * b < nu;
  // row-row order (chain): the accumulators start at the target's values and the
  // multipliers enter negated, so DMMA's chained FMAs subtract every source row's
  // product from the running value in (source, row) order; else they start at 0
  // and the sum is subtracted once in the epilogue
  const bool chain = CHAIN && part < 0;
  double d[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int t = wr0 + 8 * a + lr, c = wc0 + 8 * b + 2 * kq + e;
        d[a][b][e] = (chain && ra[a] && t < s && ca[b] && c < nu) ? Pm[(int64_t)t * W + c0 + ucol[c]] : 0.0;
      }

  int buf = 0;
  for (int64_t zb0 = zb; zb0 < ze; zb0 += KC_NSB) {
    const int nsb = (int)(ze - zb0 < KC_NSB ? ze - zb0 : KC_NSB);
    const bool last_batch = zb0 + KC_NSB >= ze;
    if (!compact) {
      if (zb0 != zb) __syncthreads();   // previous batch's chunks consumed
      source_maps(zb0, nsb, false);
      __syncthreads();
      remap(nsb);   // identity compact space: stores source col by tile position
    }
    k_layout(nsb);
    __syncthreads();
    const int nch = s_nch;
    // chunk ch = K rows [s_cst[ch], s_cst[ch+1]) of the batch, any number of sources
    auto issue = [&](int ch, int bf) {
      double *X = fs + bf * KC_BUF;
      double *U = X + 64 * KC_XLD;
      const int a0 = s_cst[ch], a1 = s_cst[ch + 1];
      if (lane < KC_K) {
        const int ga = a0 + lane;
        const bool ok = ga < a1;
        const int k = ok ? ksrc[ga] : 0;
        const int col = ok ? s_pb[k] + ga - s_koff[k] : 0;
        for (int t = warp; t < s; t += FI_THREADS / 32)
          cp_async8z(X + t * KC_XLD + lane, Pm + (int64_t)t * W + col, ok);
      }
      const bool w1 = lane + 32 < nu;   // compact columns beyond nu are never read
      for (int a = warp; a < KC_K; a += FI_THREADS / 32) {
        const int ga = a0 + a;
        const bool ok = ga < a1;
        const int k = ok ? ksrc[ga] : 0;
        const double *ur = P.F + s_vb[k] + (int64_t)(s_tb[k] + (ok ? ga - s_koff[k] : 0)) * s_vW[k] + s_qb[k];
        const int i0 = inv[k * 64 + lane], i1 = inv[k * 64 + lane + 32];
        cp_async8z(U + a * KC_ULD + lane, ur + (i0 >= 0 ? i0 : 0), ok && i0 >= 0);
        if (w1) cp_async8z(U + a * KC_ULD + lane + 32, ur + (i1 >= 0 ? i1 : 0), ok && i1 >= 0);
      }
    };
    auto prefetch_tile = [&](int bf) {   // the target's touched tile values, for the epilogue
      double *Tv = fs + bf * KC_BUF;
      for (int t = warp; t < s; t += FI_THREADS / 32) {
        const double *prow = Pm + (int64_t)t * W + c0;
        if (lane < nu) cp_async8z(Tv + t * 64 + lane, prow + ucol[lane], true);
        if (lane + 32 < nu) cp_async8z(Tv + t * 64 + lane + 32, prow + ucol[lane + 32], true);
      }
    };
    if (nch > 0) issue(0, buf);
    else if (last_batch && part < 0) prefetch_tile(buf ^ 1);
    kc_commit();
    for (int ch = 0; ch < nch; ++ch) {
      const bool more = ch + 1 < nch;
      if (more) {
        issue(ch + 1, buf ^ 1);
      } else if (last_batch && part < 0) {
        prefetch_tile(buf ^ 1);   // into the free stage
      }
      kc_commit();
      kc_wait1();
      __syncthreads();
      const int a0 = s_cst[ch];
      const int rows = s_cst[ch + 1] - a0;
      const int kc4 = (rows + 3) & ~3;
      // 8-column blocks any source of this chunk touches
      unsigned bmc = 0;
      for (int k = ksrc[a0]; k <= ksrc[a0 + rows - 1]; ++k) bmc |= s_bm[k];
      const double *X = fs + buf * KC_BUF, *U = X + 64 * KC_XLD;
      const unsigned bm = bmc >> (wc0 >> 3);
      bool cb[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) cb[b] = ca[b] && ((bm >> b) & 1u);
      if (chain) kc_chunk<true>(X, U, kc4, wr0, wc0, lr, kq, ra, cb, bm, d);   // split-K parts: sums
      else kc_chunk<false>(X, U, kc4, wr0, wc0, lr, kq, ra, cb, bm, d);
      if (more) {
        __syncthreads();   // buffer `buf` free for the chunk after next
        buf ^= 1;
      }
    }
    if (!last_batch) {
      __syncthreads();
      buf ^= 1;   // the next batch starts in the other stage
    }
  }
  kc_wait0();
  __syncthreads();
  if (part < 0) {
    // T[:, tile] -= product (row lr of each 8-row block, compact columns 2*kq, 2*kq+1)
    const double *Tv = fs + (buf ^ 1) * KC_BUF;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int t = wr0 + 8 * a + lr;
      if (!ra[a] || t >= s) continue;
      double *prow = Pm + (int64_t)t * W + c0;
#pragma unroll
      for (int b = 0; b < 4; ++b)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int c = wc0 + 8 * b + 2 * kq + e;
          if (ca[b] && c < nu) prow[ucol[c]] = chain ? d[a][b][e] : Tv[t * 64 + c] - d[a][b][e];
        }
    }
    return;
  }
  // split-K part (tile column space): publish the partial tile; the last part of the
  // item adds the partials in part order and updates the target once
  double *mine = D.part_scr + D.part_off[part];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
    const int t = wr0 + 8 * a + lr;
    if (!ra[a] || t >= s) continue;
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = wc0 + 8 * b + 2 * kq + e;
        if (ca[b] && c < tw) mine[t * FI_TILE + c] = d[a][b][e];
      }
  }
  __threadfence();
  __syncthreads();
  __shared__ int s_last;
  const int first = D.part_first[part], np = D.part_n[part];
  if (tid == 0) s_last = atomicAdd(D.part_cnt + first, 1) == np - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  for (int idx = tid; idx < s * FI_TILE; idx += FI_THREADS) {
    const int t = idx / FI_TILE, c = idx - t * FI_TILE;
    if (c >= tw) continue;
    double sum = 0.0;
    for (int k = 0; k < np; ++k) sum += __ldcg(D.part_scr + D.part_off[first + k] + t * FI_TILE + c);
    Pm[(int64_t)t * W + c0 + c] -= sum;
  }
  if (tid == 0) D.part_cnt[first] = 0;
}
template <bool CHAIN>
__global__ void __launch_bounds__(FI_THREADS, KC_MINB_DEF) k_fi_upd_kcp(DevSym S, const CallP *__restrict__ Pd, FaninDev D, int base) { d_fi_upd_kcp<CHAIN>(S, Pd, D, base, blockIdx.x); }


size_t fi_lu_smem() { return (size_t)64 * FXLD * sizeof(double); }
size_t fi_panel_smem() { return (size_t)(64 * 256 + 64 * FXLD) * sizeof(double); }
size_t fi_upd_w_smem() { return (size_t)(FI_THREADS / 32) * UW_ROWS * UW_TILE * sizeof(double); }

__global__ void k_item_mask(FaninDev D, int64_t nitems, uint64_t *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nitems;
       j += (int64_t)gridDim.x * blockDim.x) {
    uint64_t m = 0;
    for (int64_t z = D.up_ptr[j]; z < D.up_ptr[j + 1]; ++z) {
      const int8_t *pz = D.src_pos + D.src_poff[z];
      const int nq = D.src_q1[z] - D.src_q0[z];
      for (int c = 0; c < nq; ++c) m |= 1ull << pz[c];
    }
    out[j] = m;
  }
}

__global__ void k_node_rec(DevSym S, const int32_t *nodes, const int32_t *c0, const int32_t *c1, int64_t nitems,
                           NodeItemRec *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nitems;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int u = nodes[j];
    NodeItemRec r;
    r.valoff = S.valoff[u];
    r.r = (int32_t)S.first[u];
    r.s = (int32_t)(S.first[u + 1] - S.first[u]);
    r.W = (int32_t)(S.colptr[u + 1] - S.colptr[u]);
    r.L = S.nl[u];
    r.c0 = c0 ? c0[j] : 0;
    r.c1 = c1 ? c1[j] : 0;
    out[j] = r;
  }
}

__global__ void k_x_rec(DevSym S, FaninDev D, int64_t nitems, XRec *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nitems;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t dk = D.xp_edge[j];
    const int T = D.xp_tgt[j];
    const int v = S.deps[dk];
    const int64_t tc0 = S.colptr[T];
    const int vf = (int)S.first[v];
    const int vW = (int)(S.colptr[v + 1] - S.colptr[v]);
    const int pb0 = D.dep_pb[dk];
    const int tb0 = S.cols[tc0 + pb0] - vf;
    XRec r;
    r.t_off = S.valoff[T] + pb0;
    r.u_off = S.valoff[v] + (int64_t)tb0 * vW + S.nl[v] + tb0;
    r.W = (int32_t)(S.colptr[T + 1] - tc0);
    r.vW = vW;
    r.s = (int16_t)(S.first[T + 1] - S.first[T]);
    r.m = (int16_t)((int)(S.first[v + 1] - vf) - tb0);
    r.pad = 0;
    out[j] = r;
  }
}

__global__ void k_item_rec(DevSym S, FaninDev D, int64_t nitems, ItemRec *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < nitems;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int T = D.up_t[j];
    ItemRec r;
    r.valoff = S.valoff[T];
    r.zb = D.up_ptr[j];
    r.nz = (int32_t)(D.up_ptr[j + 1] - r.zb);
    r.W = (int32_t)(S.colptr[T + 1] - S.colptr[T]);
    r.s = (int16_t)(S.first[T + 1] - S.first[T]);
    r.c0 = D.up_c0[j];
    r.tw = (int16_t)(D.up_c1[j] - D.up_c0[j]);
    out[j] = r;
  }
}

template __global__ void k_fi_upd_kc<false>(DevSym, const CallP *, FaninDev, int);
template __global__ void k_fi_upd_kc<true>(DevSym, const CallP *, FaninDev, int);
template __global__ void k_fi_upd_kcp<false>(DevSym, const CallP *, FaninDev, int);
template __global__ void k_fi_upd_kcp<true>(DevSym, const CallP *, FaninDev, int);

size_t fi_upd_smem(int Smax, int Mmax) {
  (void)Mmax;
  // k_fi_upd uses Xs + Ut only; the DMMA variant also keeps an accumulator tile
  return ((size_t)Smax * FI_TILE + (size_t)Smax * KLD + (size_t)FI_KC * FXLD) * sizeof(double);
}

}  // namespace hy
