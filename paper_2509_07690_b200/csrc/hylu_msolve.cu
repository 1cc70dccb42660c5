// hylu_msolve.cu — partition-based forward/backward substitution for many right-hand
// sides at once (the paper's Fig. 3).
//
// The host partition (paper_2509_07690_b200/partition.py) cuts the rows into
// segments; per segment the rectangular block (L entries left of it / U entries
// right of it) is a sparse x dense product over the nrhs columns, split into
// nonzero-balanced row ranges (one warp each), and the triangular part runs one
// launch per level present in the segment (warp per node) or, when it is small,
// one warp walking the segment's nodes in order.  Y is [n][nrhs] (the right-hand
// sides of a row contiguous): lane = right-hand side, so every gathered y row is
// one coalesced line and every factor entry is a warp-uniform broadcast.
// Forward rows subtract their entries in column order (rectangular prefix, then
// the triangle) with separate multiply and subtract: the oracle's forward loop
// (oracle/numeric.py solve_kernel) operation for operation.
#include "hylu_common.cuh"

namespace hy {

constexpr int MS_WARPS = 4;

__device__ __forceinline__ int ms_lower_bound(const int32_t *a, int lo, int hi, int key) {
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < key) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// One factor row i against the right-hand sides: forward uses L entries p in [0, d)
// whose column lies in [clo, chi); backward uses U entries p in (d, W) in that
// column range and, if finish, divides by the pivot.
__device__ __forceinline__ void ms_row(const DevSym &S, const double *__restrict__ F, int i, int clo,
                                       int chi, bool fwd, bool finish, double *Y, int nrhs,
                                       int lane) {
  const int u = S.node_of[i];
  const int t = i - (int)S.first[u];
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int d = S.nl[u] + t;
  const double *row = F + S.valoff[u] + (int64_t)t * W;
  const int32_t *cc = S.cols + c0;
  int p0, p1;
  if (fwd) {
    p0 = ms_lower_bound(cc, 0, d, clo);
    p1 = ms_lower_bound(cc, p0, d, chi);
  } else {
    p0 = ms_lower_bound(cc, d + 1, W, clo);
    p1 = ms_lower_bound(cc, p0, W, chi);
  }
  const double piv = finish ? row[d] : 1.0;
  for (int j0 = 0; j0 < nrhs; j0 += 32) {
    const int j = j0 + lane;
    const bool ok = j < nrhs;
    double acc = ok ? Y[(int64_t)i * nrhs + j] : 0.0;
    int p = p0;
    for (; p + 4 <= p1; p += 4) {
      double f[4], y[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        f[e] = __ldg(row + p + e);
        y[e] = ok ? Y[(int64_t)__ldg(cc + p + e) * nrhs + j] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) acc = __dsub_rn(acc, __dmul_rn(f[e], y[e]));
    }
    for (; p < p1; ++p) {
      const double y = ok ? Y[(int64_t)__ldg(cc + p) * nrhs + j] : 0.0;
      acc = __dsub_rn(acc, __dmul_rn(__ldg(row + p), y));
    }
    if (finish) acc = __ddiv_rn(acc, piv);
    if (ok) Y[(int64_t)i * nrhs + j] = acc;
  }
}

// kind 0: rectangular block, items = row-range pairs; kind 1: triangular level,
// items = nodes; seq: one warp walks every item in order.
__global__ void __launch_bounds__(MS_WARPS * 32) k_msolve(DevSym S, const double *__restrict__ F, int kind,
                                                          int seq, int lo, int hi, const int32_t *items,
                                                          int count, int fwd, double *Y, int nrhs) {
  const int lane = threadIdx.x & 31;
  const int w = blockIdx.x * MS_WARPS + (threadIdx.x >> 5);
  int q0 = w, q1 = w + 1;
  if (seq) {
    if (w != 0) return;
    q1 = count;
  }
  if (q0 >= count) return;
  for (int q = q0; q < q1; ++q) {
    if (kind == 0) {
      const int r0 = items[2 * q], r1 = items[2 * q + 1];
      for (int i = r0; i < r1; ++i)
        if (fwd) ms_row(S, F, i, 0, lo, true, false, Y, nrhs, lane);
        else ms_row(S, F, i, hi, (int)S.n, false, false, Y, nrhs, lane);
    } else {
      const int u = items[q];
      const int r = (int)S.first[u], e = (int)S.first[u + 1];
      if (fwd)
        for (int i = r; i < e; ++i) ms_row(S, F, i, lo, hi, true, false, Y, nrhs, lane);
      else
        for (int i = e - 1; i >= r; --i) ms_row(S, F, i, lo, hi, false, true, Y, nrhs, lane);
    }
    if (seq) __syncwarp();
  }
}

// B [nrhs][n] -> Y [n][nrhs]: Y[i][j] = dr[a] B[j][a], a = source row of factor row i
// (b̂ = P_inner P Dr b)
__global__ void k_mbhat(DevSym S, const int32_t *iperm, const double *B, double *Y, int nrhs) {
  const int64_t total = (int64_t)S.n * nrhs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int i = (int)(q / nrhs), j = (int)(q - (int64_t)i * nrhs);
    const int u = S.node_of[i];
    int src = i;
    if (S.kind[u] == 1) src = (int)S.first[u] + iperm[i];
    const int64_t a = S.mrow_src[src];
    Y[q] = S.dr[a] * B[(int64_t)j * S.n + a];
  }
}

// Y [n][nrhs] -> X [nrhs][n]: x[perm[k]] = dc[perm[k]] z[k]
__global__ void k_mxout(DevSym S, const double *Y, double *X, int nrhs) {
  const int64_t total = (int64_t)S.n * nrhs;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < total;
       q += (int64_t)gridDim.x * blockDim.x) {
    const int k = (int)(q / nrhs), j = (int)(q - (int64_t)k * nrhs);
    const int64_t c = S.perm[k];
    X[(int64_t)j * S.n + c] = S.dc[c] * Y[q];
  }
}


// ---------------------------------------------------------------------------- level-scheduled
// Multi-RHS substitution by levels for supernodal factors (kinds 3 / 4 of the launch
// lists; the partition's warp-per-row form serialises wide panels).  grid.y = chunks
// of 32 right-hand sides.
__device__ __forceinline__ void ms_dmma(double (&d)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(d[0]), "+d"(d[1])
      : "d"(a), "d"(b));
}

// kind 3: one standalone row with a wide off-diagonal part: 8 warps take contiguous
// slices of its entries (lanes = right-hand sides), partial sums combined in warp
// order; backward rows divide by the pivot.
__global__ void __launch_bounds__(256) k_msolve_long(DevSym S, const double *__restrict__ F,
                                                     const int32_t *items, int fwd, double *Y, int nrhs) {
  __shared__ double red[8][32];
  const int u = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n0 = blockIdx.y * 32, j = n0 + lane;
  const bool ok = j < nrhs;
  const int i = (int)S.first[u];
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int d = S.nl[u];
  const double *row = F + S.valoff[u];
  const int32_t *cc = S.cols + c0;
  const int p0 = fwd ? 0 : d + 1, p1 = fwd ? d : W;
  const int per = (p1 - p0 + 7) / 8;
  const int q0 = p0 + warp * per, q1 = min(p1, q0 + per);
  double acc = 0.0;
  int p = q0;
  for (; p + 4 <= q1; p += 4) {
    double f[4], y[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      f[e] = __ldg(row + p + e);
      y[e] = ok ? Y[(int64_t)__ldg(cc + p + e) * nrhs + j] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < 4; ++e) acc = fma(f[e], y[e], acc);
  }
  for (; p < q1; ++p) acc = fma(__ldg(row + p), ok ? Y[(int64_t)__ldg(cc + p) * nrhs + j] : 0.0, acc);
  red[warp][lane] = acc;
  __syncthreads();
  if (warp == 0 && ok) {
    double v = Y[(int64_t)i * nrhs + j];
    for (int w = 0; w < 8; ++w) v -= red[w][lane];
    if (!fwd) v /= row[d];
    Y[(int64_t)i * nrhs + j] = v;
  }
}

// kind 4: one supernode: its off-block panel times the gathered solution rows on
// DMMA — 16 warps: warp w takes rows 16(w&3)..+15 and the (w>>2)-th quarter of the
// off-block columns, all 32 right-hand sides of the chunk; the four column quarters'
// products are subtracted in quarter order (deterministic) — then the in-block
// triangular solve (unit lower forward / upper with pivots backward) by warp 0,
// lane = right-hand side.
constexpr int SN_KS = 4;
__global__ void __launch_bounds__(128 * SN_KS) k_msolve_sn(DevSym S, const double *__restrict__ F,
                                                          const int32_t *items, int fwd, double *Y, int nrhs) {
  __shared__ double Yb[64][33];
  const int u = items[blockIdx.x];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, kq = lane & 3, lr = lane >> 2;
  const int wr = warp & 3, ks = warp >> 2;
  const int n0 = blockIdx.y * 32;
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *Fu = F + S.valoff[u];
  const int32_t *cc = S.cols + c0;
  const int kb0 = fwd ? 0 : L + s, kb1 = fwd ? L : W;
  const int per = ((kb1 - kb0 + SN_KS - 1) / SN_KS + 3) & ~3;
  const int k0 = kb0 + ks * per, k1 = min(kb1, k0 + per);
  const int r0 = wr * 16 + lr, r1 = r0 + 8;
  const bool a0 = r0 < s, a1 = r1 < s;
  double d[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) d[a][b][0] = d[a][b][1] = 0.0;
  if (wr * 16 < s) {
    bool nb[4];
#pragma unroll
    for (int b = 0; b < 4; ++b) nb[b] = n0 + 8 * b + lr < nrhs;
#pragma unroll 4
    for (int k = k0; k < k1; k += 4) {
      const int kk = k + kq;
      const bool kin = kk < k1;
      const int col = kin ? __ldg(cc + kk) : 0;
      const double x0 = (a0 && kin) ? __ldg(Fu + (int64_t)r0 * W + kk) : 0.0;
      const double x1 = (a1 && kin) ? __ldg(Fu + (int64_t)r1 * W + kk) : 0.0;
      const double *yr = Y + (int64_t)col * nrhs + n0 + lr;
      double bv[4];
#pragma unroll
      for (int b = 0; b < 4; ++b) bv[b] = (kin && nb[b]) ? yr[8 * b] : 0.0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        ms_dmma(d[0][b], x0, bv[b]);
        ms_dmma(d[1][b], x1, bv[b]);
      }
    }
  }
  // y_t := y_t - (panel product)_t, the column quarters in order, into shared memory
  for (int q = 0; q < SN_KS; ++q) {
    if (ks == q) {
#pragma unroll
      for (int a = 0; a < 2; ++a) {
        const int t = wr * 16 + 8 * a + lr;
        if (t >= s) continue;
#pragma unroll
        for (int b = 0; b < 4; ++b)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * b + 2 * kq + e, j = n0 + c;
            const double prev = q == 0 ? (j < nrhs ? Y[(int64_t)(r + t) * nrhs + j] : 0.0) : Yb[t][c];
            Yb[t][c] = prev - d[a][b][e];
          }
      }
    }
    __syncthreads();
  }
  if (warp == 0) {
    const double *blk = Fu + L;   // row t of the diagonal block at blk + t * W
    if (fwd) {
      for (int t = 1; t < s; ++t) {
        double acc = Yb[t][lane];
        for (int q = 0; q < t; ++q) acc -= __ldg(blk + (int64_t)t * W + q) * Yb[q][lane];
        Yb[t][lane] = acc;
        __syncwarp();
      }
    } else {
      for (int t = s - 1; t >= 0; --t) {
        double acc = Yb[t][lane];
        for (int q = t + 1; q < s; ++q) acc -= __ldg(blk + (int64_t)t * W + q) * Yb[q][lane];
        Yb[t][lane] = acc / __ldg(blk + (int64_t)t * W + t);
        __syncwarp();
      }
    }
  }
  __syncthreads();
  for (int idx = threadIdx.x; idx < s * 32; idx += 128 * SN_KS) {
    const int t = idx >> 5, c = idx & 31, j = n0 + c;
    if (j < nrhs) Y[(int64_t)(r + t) * nrhs + j] = Yb[t][c];
  }
}

}  // namespace hy
