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

constexpr int BW = 4;          // warps per block
constexpr int BCAP = 1024;     // target columns cached in shared memory


__global__ void __launch_bounds__(BW * 32) k_batch_factor(DevSym S, BatchP P, const int32_t *nodes,
                                                          int count, int G) {
  __shared__ int32_t tcs[BW][BCAP];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * BW + warp;
  if (task >= (int64_t)count * G) return;
  const int u = nodes[task / G];
  const int g = (int)(task % G);
  const int64_t b = (int64_t)g * 32 + lane;
  const bool live = b < P.B;
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const bool inSm = W <= BCAP;
  const int32_t *tc = inSm ? tcs[warp] : S.cols + c0;
  if (inSm)
    for (int q = lane; q < W; q += 32) tcs[warp][q] = S.cols[c0 + q];
  double *gbase = P.BF + (int64_t)g * P.stored * 32;
  const double *Ab = P.A + (int64_t)g * 32 * S.nnz;
  const double thr = P.eps * P.anorm[0];
  const int nlive = (int)(P.B - (int64_t)g * 32 < 32 ? P.B - (int64_t)g * 32 : 32);
  __syncwarp();
  for (int t = 0; t < s; ++t) {
    double *w = gbase + (S.valoff[u] + (int64_t)t * W) * 32;
    for (int q = 0; q < W; ++q) w[(int64_t)q * 32 + lane] = 0.0;
    // scatter M row (r + iperm[r+t]) for the 32 instances: lanes over (instance, entry)
    const int src = (s > 1) ? r + P.iperm[r + t] : r;
    const int64_t a = S.mrow_src[src];
    const int64_t e0 = S.a_ptr[a];
    const int k = (int)(S.a_ptr[a + 1] - e0);
    __syncwarp();
    for (int idx = lane; idx < nlive * k; idx += 32) {
      const int inst = idx / k, e = idx - inst * k;
      w[(int64_t)S.colpos[e0 + e] * 32 + inst] = Ab[(int64_t)inst * S.nnz + e0 + e] * S.scale[e0 + e];
    }
    __syncwarp();
    const int Lt = L + t;
    for (int p = 0; p < Lt; ++p) {
      const int j = tc[p];
      const int v = S.node_of[j];
      const int tj = j - (int)S.first[v];
      const int64_t vc0 = S.colptr[v];
      const int vW = (int)(S.colptr[v + 1] - vc0);
      const int sd = S.nl[v] + tj;
      const double *srow = gbase + (S.valoff[v] + (int64_t)tj * vW) * 32 + lane;
      const int32_t *vc = S.cols + vc0;
      const double l = w[(int64_t)p * 32 + lane] / srow[(int64_t)sd * 32];
      w[(int64_t)p * 32 + lane] = l;
      if (__any_sync(HY_FULL, l != 0.0)) {
        int pos = p + 1;
        for (int q = sd + 1; q < vW; ++q) {
          const int kc = vc[q];
          pos = lower_bound_i32(tc, pos, W, kc);  // source columns ascend: search forward
          w[(int64_t)pos * 32 + lane] -= l * srow[(int64_t)q * 32];
        }
      }
    }
    // pivot
    double *dp = w + (int64_t)Lt * 32 + lane;
    const double piv = *dp;
    bool fired;
    *dp = perturb(piv, thr, fired);
    if (fired && live) atomicAdd(&P.npert[b], 1);
    __syncwarp();
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
