// hylu_batch.cu — batched same-pattern refactorization + solve (BASELINE config 4).
//
// B instances share one symbolic structure.  Factor values are stored
// instance-interleaved in groups of 32: value p of instance b lives at
//   BF[((b/32) * stored + p) * 32 + (b%32)]
// so one warp processes one (node, group) task with lane = instance: every lane
// runs the same up-looking row-row loop over the same pattern,
// every value access is one coalesced 256-byte line, and all index work is
// warp-uniform.  Refactorize semantics: the prior inner_perm is
// pre-applied at scatter time, no pivot search, perturbation active against the
// prior anorm.  Supernode rows are processed up-looking in their fixed pivot order,
// which per entry is the same operation sequence as external updates followed by
// internal_factorize (see oracle/numeric.py note 5).
#include "hylu_common.cuh"

namespace hy {

constexpr int BW = 4;          // warps per block (row kernel)
constexpr int WS = 32;         // rows with W <= WS keep their accumulator in shared memory
constexpr int HUB_THREADS = 256;

// ---------------------------------------------------------------------------
// Row kernel: one warp per (non-hub node, group of 32 instances), lane = instance.
// Executes the node's row programs (structural steps only, precomputed target
// positions), fuses the forward substitution y_i = b̂_i − Σ_s l_s y_{j_s}.
__global__ void __launch_bounds__(BW * 32) k_bt_rows(DevSym S, BatchP P, DevProg R,
                                                     const int32_t *nodes, int count, int G,
                                                     const double *rhs, double *Y) {
  __shared__ double wsm[BW][WS * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * BW + warp;
  if (task >= (int64_t)count * G) return;
  const int u = nodes[task / G];
  const int g = (int)(task % G);
  const int64_t b = (int64_t)g * 32 + lane;
  const bool live = b < P.B;
  const int nlive = (int)(P.B - (int64_t)g * 32 < 32 ? P.B - (int64_t)g * 32 : 32);
  const double thr = P.eps * P.anorm[0];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  const int L = S.nl[u];
  double *gb0 = P.BF + (int64_t)g * P.stored * 32;  // group base (no lane offset)
  const double *gb = gb0 + lane;
  double *yb = Y + (int64_t)g * S.n * 32 + lane;
  const double *Ab = P.A + (int64_t)g * 32 * S.nnz;
  const bool inSm = W <= WS;
  for (int t = 0; t < s; ++t) {
    const int i = r + t;
    double *w0 = inSm ? wsm[warp] : gb0 + (S.valoff[u] + (int64_t)t * W) * 32;
    double *w = w0 + lane;
    for (int q = 0; q < W; ++q) w[q * 32] = 0.0;
    const int srow = S.kind[u] ? r + P.iperm[i] : r;
    const int64_t a = S.mrow_src[srow];
    const int64_t e0 = S.a_ptr[a];
    const int k = (int)(S.a_ptr[a + 1] - e0);
    __syncwarp();
    for (int idx = lane; idx < nlive * k; idx += 32) {
      const int inst = idx / k, e = idx - inst * k;
      w0[S.colpos[e0 + e] * 32 + inst] = Ab[(int64_t)inst * S.nnz + e0 + e] * S.scale[e0 + e];
    }
    double yacc = (live && rhs) ? S.dr[a] * rhs[b * S.n + a] : 0.0;
    __syncwarp();
    const int64_t s0 = R.row_ptr[i], s1 = R.row_ptr[i + 1];
    for (int64_t st = s0; st < s1; ++st) {
      const int p = R.st_p[st];
      const int64_t src = R.st_src[st];
      const int cnt = R.st_cnt[st];
      const int32_t *rl = R.rel + R.st_rel[st];
      const double d = gb[src * 32];
      const double yj = yb[(int64_t)R.st_j[st] * 32];
      const double l = w[p * 32] / d;
      w[p * 32] = l;
      yacc -= l * yj;
      const double *us = gb + (src + 1) * 32;
      int q = 0;
      for (; q + 4 <= cnt; q += 4) {
        const int t0 = rl[q], t1 = rl[q + 1], t2 = rl[q + 2], t3 = rl[q + 3];
        const double u0 = us[(q + 0) * 32], u1 = us[(q + 1) * 32];
        const double u2 = us[(q + 2) * 32], u3 = us[(q + 3) * 32];
        w[t0 * 32] -= l * u0;
        w[t1 * 32] -= l * u1;
        w[t2 * 32] -= l * u2;
        w[t3 * 32] -= l * u3;
      }
      for (; q < cnt; ++q) w[rl[q] * 32] -= l * us[q * 32];
    }
    const int Lt = L + t;
    const double piv = w[Lt * 32];
    bool fired;
    w[Lt * 32] = perturb(piv, thr, fired);
    if (fired && live) atomicAdd(&P.npert[b], 1);
    yb[(int64_t)i * 32] = yacc;
    if (inSm) {
      double *dst = gb0 + (S.valoff[u] + (int64_t)t * W) * 32 + lane;
      for (int q = 0; q < W; ++q) dst[q * 32] = w[q * 32];
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// Hub kernel: one CTA per (hub node, group).  Pull programs: positions of a row are
// processed level by level (intra-row dependency levels); each position gathers
// its contributions in ascending step order.  Forward substitution fused with a
// fixed-order cross-warp reduction.
__global__ void __launch_bounds__(HUB_THREADS) k_bt_hub(DevSym S, BatchP P, DevProg R,
                                                        const int32_t *nodes, int count, int G,
                                                        const double *rhs, double *Y) {
  __shared__ double red[HUB_THREADS / 32][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = HUB_THREADS / 32;
  const int task = blockIdx.x;
  const int u = nodes[task / G];
  const int g = task % G;
  const int64_t b = (int64_t)g * 32 + lane;
  const bool live = b < P.B;
  const int nlive = (int)(P.B - (int64_t)g * 32 < 32 ? P.B - (int64_t)g * 32 : 32);
  const double thr = P.eps * P.anorm[0];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  double *gb0 = P.BF + (int64_t)g * P.stored * 32;
  const double *gb = gb0 + lane;
  double *yb = Y + (int64_t)g * S.n * 32 + lane;
  const double *Ab = P.A + (int64_t)g * 32 * S.nnz;
  const int hr0 = R.hub_base[u];
  for (int t = 0; t < s; ++t) {
    const int i = r + t;
    double *w0 = gb0 + (S.valoff[u] + (int64_t)t * W) * 32;
    double *w = w0 + lane;
    for (int q = threadIdx.x; q < W * 32; q += HUB_THREADS) w0[q] = 0.0;
    __syncthreads();
    const int srow = S.kind[u] ? r + P.iperm[i] : r;
    const int64_t a = S.mrow_src[srow];
    const int64_t e0 = S.a_ptr[a];
    const int k = (int)(S.a_ptr[a + 1] - e0);
    for (int idx = threadIdx.x; idx < nlive * k; idx += HUB_THREADS) {
      const int inst = idx / k, e = idx - inst * k;
      w0[S.colpos[e0 + e] * 32 + inst] = Ab[(int64_t)inst * S.nnz + e0 + e] * S.scale[e0 + e];
    }
    __syncthreads();
    const int hr = hr0 + t;
    for (int64_t lev = R.hrow_lev[hr]; lev < R.hrow_lev[hr + 1]; ++lev) {
      for (int64_t x = R.lev_ptr[lev] + warp; x < R.lev_ptr[lev + 1]; x += nw) {
        const int p = R.hpos[x];
        double acc = w[p * 32];
        const int64_t y0 = R.hpp[x], y1 = R.hpp[x + 1];
        int64_t y = y0;
        for (; y + 4 <= y1; y += 4) {
          const double l0 = w[R.pred_p[y] * 32], l1 = w[R.pred_p[y + 1] * 32];
          const double l2 = w[R.pred_p[y + 2] * 32], l3 = w[R.pred_p[y + 3] * 32];
          const double v0 = gb[R.pred_u[y] * 32], v1 = gb[R.pred_u[y + 1] * 32];
          const double v2 = gb[R.pred_u[y + 2] * 32], v3 = gb[R.pred_u[y + 3] * 32];
          acc -= l0 * v0;
          acc -= l1 * v1;
          acc -= l2 * v2;
          acc -= l3 * v3;
        }
        for (; y < y1; ++y) acc -= w[R.pred_p[y] * 32] * gb[R.pred_u[y] * 32];
        const int64_t kd = R.hdiv[x];
        if (kd >= 0) {
          acc = acc / gb[kd * 32];
        } else if (kd == -2) {
          bool fired;
          const double piv = acc;
          acc = perturb(piv, thr, fired);
          if (fired && live) atomicAdd(&P.npert[b], 1);
        }
        w[p * 32] = acc;
      }
      __syncthreads();
    }
    // forward substitution for row i: y_i = b̂_i − Σ_s l_s y_{j_s}
    double part = 0.0;
    for (int64_t st = R.row_ptr[i] + warp; st < R.row_ptr[i + 1]; st += nw)
      part += w[R.st_p[st] * 32] * yb[(int64_t)R.st_j[st] * 32];
    red[warp][lane] = part;
    __syncthreads();
    if (warp == 0) {
      double yacc = (live && rhs) ? S.dr[a] * rhs[b * S.n + a] : 0.0;
      for (int k2 = 0; k2 < nw; ++k2) yacc -= red[k2][lane];
      yb[(int64_t)i * 32] = yacc;
    }
    __syncthreads();
  }
}

// rhs [B][n] -> interleaved b_hat [G][n][32]: b_hat[i] = dr[a] b[a], a = source row of factor row i
__global__ void k_batch_bhat(DevSym S, const int32_t *iperm, const double *rhs, double *Y, int64_t B) {
  __shared__ double tile[32][33];
  const int g = blockIdx.y;
  const int i0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;  // 32 x 8 threads
  for (int ii = wy; ii < 32; ii += 8) {
    const int inst = ii;
    const int64_t b = (int64_t)g * 32 + inst;
    const int row = i0 + lane;
    double v = 0.0;
    if (row < S.n && b < B) {
      const int u = S.node_of[row];
      int src = row;
      if (S.kind[u] == 1) src = (int)S.first[u] + iperm[row];
      const int64_t a = S.mrow_src[src];
      v = S.dr[a] * rhs[b * S.n + a];
    }
    tile[inst][lane] = v;
  }
  __syncthreads();
  for (int ii = wy; ii < 32; ii += 8) {
    const int row = i0 + ii;
    if (row < S.n) Y[((int64_t)g * S.n + row) * 32 + lane] = tile[lane][ii];
  }
}

// interleaved z [G][n][32] -> x [B][n]: x[perm[k]] = dc[perm[k]] z[k]
__global__ void k_batch_xout(DevSym S, const double *Y, double *X, int64_t B) {
  __shared__ double tile[32][33];
  const int g = blockIdx.y;
  const int k0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  for (int kk = wy; kk < 32; kk += 8) {
    const int k = k0 + kk;
    tile[kk][lane] = k < S.n ? Y[((int64_t)g * S.n + k) * 32 + lane] : 0.0;
  }
  __syncthreads();
  for (int ii = wy; ii < 32; ii += 8) {
    const int64_t b = (int64_t)g * 32 + ii;
    const int k = k0 + lane;
    if (k < S.n && b < B) {
      const int64_t c = S.perm[k];
      X[b * S.n + c] = S.dc[c] * tile[lane][ii];
    }
  }
}

// unfused forward substitution (when the batch was refactorized without a rhs)
__global__ void __launch_bounds__(BW * 32) k_batch_fwd(DevSym S, const double *BF, int64_t stored,
                                                       const int32_t *nodes, int count, int G,
                                                       double *Y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * BW + warp;
  if (task >= (int64_t)count * G) return;
  const int u = nodes[task / G];
  const int g = (int)(task % G);
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *gbase = BF + (int64_t)g * stored * 32 + lane;
  double *y = Y + (int64_t)g * S.n * 32 + lane;
  const int32_t *cc = S.cols + c0;
  for (int t = 0; t < s; ++t) {
    const double *row = gbase + (S.valoff[u] + (int64_t)t * W) * 32;
    double acc = y[(int64_t)(r + t) * 32];
    for (int p = 0; p < L + t; ++p) acc -= row[(int64_t)p * 32] * y[(int64_t)cc[p] * 32];
    y[(int64_t)(r + t) * 32] = acc;
  }
}

__global__ void __launch_bounds__(BW * 32) k_batch_bwd(DevSym S, const double *BF, int64_t stored,
                                                       const int32_t *nodes, int count, int G,
                                                       double *Y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * BW + warp;
  if (task >= (int64_t)count * G) return;
  const int u = nodes[task / G];
  const int g = (int)(task % G);
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *gbase = BF + (int64_t)g * stored * 32 + lane;
  double *y = Y + (int64_t)g * S.n * 32 + lane;
  const int32_t *cc = S.cols + c0;
  for (int t = s - 1; t >= 0; --t) {
    const double *row = gbase + (S.valoff[u] + (int64_t)t * W) * 32;
    const int d = L + t;
    double acc = y[(int64_t)(r + t) * 32];
    for (int p = d + 1; p < W; ++p) acc -= row[(int64_t)p * 32] * y[(int64_t)cc[p] * 32];
    y[(int64_t)(r + t) * 32] = acc / row[(int64_t)d * 32];
  }
}

// de-interleave one instance's factor values into node layout
__global__ void k_batch_extract(const double *BF, int64_t stored, int64_t b, double *out) {
  const int64_t g = b / 32, lane = b % 32;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < stored;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = BF[(g * stored + p) * 32 + lane];
}

}  // namespace hy
