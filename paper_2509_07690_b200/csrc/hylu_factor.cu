// hylu_factor.cu — single-instance numeric factorization and triangular solve
// kernels for sm_100a (one factorization per GPU).
//
// Execution: the elimination DAG is level-scheduled (SPEC.md:215-223 levels; the
// bulk mode of SPEC.md:397-405 on the device).  Per level two kernels run:
//   k_rows  — one warp per standalone-row node: scatter its M row into a
//             shared-memory accumulator, apply row-row and
//             sup-row updates in ascending source order, perturb
//             the pivot, write the row once.
//   k_sn    — one CTA per supernode node: scatter, external updates (row-row per
//             source row in ROWROW mode, TRSM + GEMM otherwise),
//             then the in-supernode dense LU with block-restricted pivoting
//             (SPEC.md:320-328).
// Solve: per-level forward (unit L) and backward (U) substitution kernels.
#include "hylu_common.cuh"

namespace hy {

// ============================================================================ anorm
__global__ void k_anorm(const double *__restrict__ A, const double *__restrict__ scale, int64_t nnz,
                        double *out) {
  double m = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[e] * scale[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(HY_FULL, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(out, m);
}

// ============================================================================ per-call setup
// The per-call parameters live in device memory (one CallP per handle) so that the
// launch sequence of a factorization is a fixed CUDA graph: k_call_set writes the
// call's CallP (stream-ordered, from its by-value argument), the graph's first
// kernels clear / seed the outputs through it.
__global__ void k_call_set(CallP *dst, CallP src) { *dst = src; }
__global__ void k_ptr_set(const double **dst, const double *src) { *dst = src; }

// status[0..3] = 0; factorize: inner_perm = 0, anorm = 0; refactorize: inner_perm =
// prior inner_perm, anorm = prior anorm; zero_f: F[0:stored) = 0 (level fan-in).
__global__ void k_call_prep(const CallP *__restrict__ Pd, int n, int64_t stored, int zero_f) {
  const CallP P = *Pd;
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t nth = (int64_t)gridDim.x * blockDim.x;
  if (tid < 4) P.status[tid] = 0;
  if (tid == 0) *const_cast<double *>(P.anorm) = P.refactor ? *P.anorm_prior : 0.0;
  for (int64_t i = tid; i < n; i += nth) P.iperm[i] = P.refactor ? P.iperm_prior[i] : 0;
  if (zero_f && (reinterpret_cast<uintptr_t>(P.F) & 15)) {
    for (int64_t i = tid; i < stored; i += nth) P.F[i] = 0.0;
  } else if (zero_f) {
    double2 *F2 = reinterpret_cast<double2 *>(P.F);
    const int64_t h = stored >> 1;
    for (int64_t i = tid; i < h; i += nth) F2[i] = make_double2(0.0, 0.0);
    if ((stored & 1) && tid == 0) P.F[stored - 1] = 0.0;
  }
}

// anorm = max |A·scale| (factorize only; refactorize keeps the prior anorm)
__global__ void k_anorm_p(const CallP *__restrict__ Pd, const double *__restrict__ scale, int64_t nnz) {
  if (Pd->refactor) return;
  const double *A = Pd->A;
  double m = 0.0;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < nnz;
       e += (int64_t)gridDim.x * blockDim.x)
    m = fmax(m, fabs(A[e] * scale[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(HY_FULL, m, o));
  if ((threadIdx.x & 31) == 0 && m > 0.0) atomic_max_nonneg(const_cast<double *>(Pd->anorm), m);
}

// ============================================================================ rows
constexpr int RW_WARPS = 4;
constexpr int CAPW = 512;

struct RowSmem {
  double w[CAPW];
  int32_t c[CAPW];
  double x[64];
};

__device__ void row_task(const DevSym &S, const CallP &P, int u, RowSmem &sm, int lane) {
  const int64_t i = S.first[u];
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  double *F = P.F;
  double *Fu = F + S.valoff[u];
  const bool inSm = W <= CAPW;
  double *w = inSm ? sm.w : Fu;
  const int32_t *tc = inSm ? sm.c : S.cols + c0;
  for (int q = lane; q < W; q += 32) {
    w[q] = 0.0;
    if (inSm) sm.c[q] = S.cols[c0 + q];
  }
  __syncwarp();
  {
    const int64_t a = S.mrow_src[i];
    for (int64_t e = S.a_ptr[a] + lane; e < S.a_ptr[a + 1]; e += 32)
      w[S.colpos[e]] = P.A[e] * S.scale[e];
  }
  __syncwarp();
  int p = 0;
  while (p < L) {
    const int j = tc[p];
    const int v = S.node_of[j];
    const int vf = (int)S.first[v];
    const int64_t vc0 = S.colptr[v];
    const int vW = (int)(S.colptr[v + 1] - vc0);
    const int vnl = S.nl[v];
    const int32_t *vc = S.cols + vc0;
    const double *vb = F + S.valoff[v];
    if (S.kind[v] == 0 || S.mode == 0) {
      // ---- row-row: source row j
      const int tj = j - vf;
      const double *srow = vb + (int64_t)tj * vW;
      const int sd = vnl + tj;
      const double l = w[p] / srow[sd];
      __syncwarp();
      if (lane == 0) w[p] = l;
      if (l != 0.0) {
        for (int q = sd + 1 + lane; q < vW; q += 32) {
          const int pos = lower_bound_i32(tc, p + 1, W, vc[q]);
          w[pos] -= l * srow[q];
        }
      }
      __syncwarp();
      p++;
    } else {
      // ---- sup-row: TRSV with the source's upper block, then GEMV over its panel
      const int vs = (int)(S.first[v + 1] - vf);
      const int t0 = j - vf;
      const int m = vs - t0;
      for (int t = lane; t < vs; t += 32) sm.x[t] = (t >= t0) ? w[p + t - t0] : 0.0;
      __syncwarp();
      for (int t = t0; t < vs; ++t) {
        const double *ur = vb + (int64_t)t * vW + vnl;
        const double xt = sm.x[t] / ur[t];
        __syncwarp();
        if (lane == 0) sm.x[t] = xt;
        if (xt != 0.0)
          for (int t2 = t + 1 + lane; t2 < vs; t2 += 32) sm.x[t2] -= xt * ur[t2];
        __syncwarp();
      }
      for (int t = t0 + lane; t < vs; t += 32) w[p + t - t0] = sm.x[t];
      for (int q = vnl + vs + lane; q < vW; q += 32) {
        double acc = 0.0;
        for (int t = t0; t < vs; ++t) acc += sm.x[t] * vb[(int64_t)t * vW + q];
        const int pos = lower_bound_i32(tc, p + m, W, vc[q]);
        w[pos] -= acc;
      }
      __syncwarp();
      p += m;
    }
  }
  if (lane == 0) {
    const double piv = w[L];
    const double thr = P.eps * P.anorm[0];
    bool fired;
    w[L] = perturb(piv, thr, fired);
    log_pivot(P, i, piv, fired, thr);
  }
  __syncwarp();
  if (inSm)
    for (int q = lane; q < W; q += 32) Fu[q] = w[q];
}

__global__ void __launch_bounds__(RW_WARPS * 32) k_rows(DevSym S, const CallP *__restrict__ Pd, const int32_t *nodes,
                                                        int count) {
  const CallP P = *Pd;
  __shared__ RowSmem sm[RW_WARPS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * RW_WARPS + warp;
  if (idx >= count) return;
  row_task(S, P, nodes[idx], sm[warp], lane);
}

// ============================================================================ supernodes
constexpr int SN_THREADS = 256;
constexpr int SMAX = 64;
constexpr int LDX = SMAX + 1;
constexpr int TILE = 64;
constexpr int CAPC = 8192;
constexpr int SPOS = 2048;

struct SnSmem {
  double X[SMAX * LDX];   // multipliers / diagonal block LU
  double U[SMAX * LDX];   // source diagonal block
  double T[SMAX * LDX];   // GEMM / panel tile
  int32_t spos[SPOS];
  int32_t tcols[CAPC];
  double lm[SMAX];
  int32_t perm[SMAX];
  int32_t pinv[SMAX];
  int32_t piv_row;
};

// positions of source columns vc[qa..qa+cnt) in the target column list tc[lo..W), -1 if absent
__device__ __forceinline__ void map_cols(const int32_t *vc, int qa, int cnt, const int32_t *tc,
                                         int lo, int W, int32_t *out) {
  for (int q = threadIdx.x; q < cnt; q += blockDim.x) {
    const int k = vc[qa + q];
    const int pos = lower_bound_i32(tc, lo, W, k);
    out[q] = (pos < W && tc[pos] == k) ? pos : -1;
  }
}

__global__ void __launch_bounds__(SN_THREADS, 1) k_sn(DevSym S, const CallP *__restrict__ Pd, const int32_t *nodes) {
  const CallP P = *Pd;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  SnSmem &sm = *reinterpret_cast<SnSmem *>(smem_raw);
  const int u = nodes[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = SN_THREADS / 32;
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  double *F = P.F;
  double *Pm = F + S.valoff[u];
  const bool colsSm = W <= CAPC;
  const int32_t *tc = colsSm ? sm.tcols : S.cols + c0;
  const double thr = P.eps * P.anorm[0];

  if (colsSm)
    for (int q = tid; q < W; q += SN_THREADS) sm.tcols[q] = S.cols[c0 + q];
  if (tid < s) {
    if (P.refactor) {
      const int t = P.iperm_prior[r + tid];
      sm.pinv[t] = tid;
      P.iperm[r + tid] = t;
    } else {
      sm.pinv[tid] = tid;
    }
  }
  for (int64_t q = tid; q < (int64_t)s * W; q += SN_THREADS) Pm[q] = 0.0;
  __syncthreads();
  for (int t = warp; t < s; t += nwarps) {
    const int64_t a = S.mrow_src[r + t];
    double *row = Pm + (int64_t)sm.pinv[t] * W;
    for (int64_t e = S.a_ptr[a] + lane; e < S.a_ptr[a + 1]; e += 32)
      row[S.colpos[e]] = P.A[e] * S.scale[e];
  }
  __syncthreads();

  // ------------------------------------------------------------ external updates
  for (int64_t di = S.dptr[u]; di < S.dptr[u + 1]; ++di) {
    const int v = S.deps[di];
    const int vf = (int)S.first[v];
    const int vs = (int)(S.first[v + 1] - vf);
    const int64_t vc0 = S.colptr[v];
    const int vW = (int)(S.colptr[v + 1] - vc0);
    const int vnl = S.nl[v];
    const int32_t *vc = S.cols + vc0;
    const double *vb = F + S.valoff[v];
    if (S.kind[v] == 0 || S.mode == 0) {
      for (int tj = 0; tj < vs; ++tj) {
        const int j = vf + tj;
        const int pj = lower_bound_i32(tc, 0, L, j);
        if (pj >= L || tc[pj] != j) continue;  // uniform
        const double *srow = vb + (int64_t)tj * vW;
        const int sd = vnl + tj;
        if (tid < s) {
          const double l = Pm[(int64_t)tid * W + pj] / srow[sd];
          Pm[(int64_t)tid * W + pj] = l;
          sm.lm[tid] = l;
        }
        for (int qa = sd + 1; qa < vW; qa += SPOS) {
          const int cnt = min(SPOS, vW - qa);
          __syncthreads();
          map_cols(vc, qa, cnt, tc, pj + 1, W, sm.spos);
          __syncthreads();
          for (int idx = tid; idx < s * cnt; idx += SN_THREADS) {
            const int t = idx / cnt, q = idx - t * cnt;
            const double l = sm.lm[t];
            if (l != 0.0) Pm[(int64_t)t * W + sm.spos[q]] -= l * srow[qa + q];
          }
        }
        __syncthreads();
      }
    } else {
      // block update: X = W_b U_bb^-1 (TRSM), W_panel -= X U_panel (GEMM)
      __syncthreads();
      map_cols(vc, vnl, vs, tc, 0, W, sm.spos);
      __syncthreads();
      for (int idx = tid; idx < s * vs; idx += SN_THREADS) {
        const int t = idx / vs, tt = idx - t * vs;
        const int ps = sm.spos[tt];
        sm.X[t * LDX + tt] = ps >= 0 ? Pm[(int64_t)t * W + ps] : 0.0;
      }
      for (int idx = tid; idx < vs * vs; idx += SN_THREADS) {
        const int tt = idx / vs, t2 = idx - tt * vs;
        sm.U[tt * LDX + t2] = t2 >= tt ? vb[(int64_t)tt * vW + vnl + t2] : 0.0;
      }
      __syncthreads();
      for (int tt = 0; tt < vs; ++tt) {
        if (tid < s) sm.X[tid * LDX + tt] /= sm.U[tt * LDX + tt];
        __syncthreads();
        const int rem = vs - tt - 1;
        for (int idx = tid; idx < s * rem; idx += SN_THREADS) {
          const int t = idx / rem, t2 = tt + 1 + idx - t * rem;
          sm.X[t * LDX + t2] -= sm.X[t * LDX + tt] * sm.U[tt * LDX + t2];
        }
        __syncthreads();
      }
      for (int idx = tid; idx < s * vs; idx += SN_THREADS) {
        const int t = idx / vs, tt = idx - t * vs;
        const int ps = sm.spos[tt];
        if (ps >= 0) Pm[(int64_t)t * W + ps] = sm.X[t * LDX + tt];
      }
      // GEMM over the source panel, 64-column tiles, 4x4 outputs per thread
      const int tr = tid >> 4, tcl = tid & 15;
      for (int qa = vnl + vs; qa < vW; qa += TILE) {
        const int nq = min(TILE, vW - qa);
        __syncthreads();
        for (int idx = tid; idx < vs * TILE; idx += SN_THREADS) {
          const int tt = idx / TILE, c = idx - tt * TILE;
          sm.T[tt * LDX + c] = c < nq ? vb[(int64_t)tt * vW + qa + c] : 0.0;
        }
        map_cols(vc, qa, nq, tc, 0, W, sm.spos);
        __syncthreads();
        double acc[4][4];
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
        for (int tt = 0; tt < vs; ++tt) {
          double xv[4], tv[4];
#pragma unroll
          for (int a = 0; a < 4; ++a) xv[a] = sm.X[(tr + 16 * a) * LDX + tt];
#pragma unroll
          for (int b = 0; b < 4; ++b) tv[b] = sm.T[tt * LDX + tcl + 16 * b];
#pragma unroll
          for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 4; ++b) acc[a][b] = fma(xv[a], tv[b], acc[a][b]);
        }
#pragma unroll
        for (int a = 0; a < 4; ++a) {
          const int t = tr + 16 * a;
          if (t < s) {
#pragma unroll
            for (int b = 0; b < 4; ++b) {
              const int c = tcl + 16 * b;
              if (c < nq) Pm[(int64_t)t * W + sm.spos[c]] -= acc[a][b];
            }
          }
        }
      }
      __syncthreads();
    }
  }

  // ------------------------------------------------------------ internal LU
  __syncthreads();
  for (int idx = tid; idx < s * s; idx += SN_THREADS) {
    const int t = idx / s, tt = idx - t * s;
    sm.X[t * LDX + tt] = Pm[(int64_t)t * W + L + tt];
  }
  if (tid < s) sm.perm[tid] = tid;
  __syncthreads();
  for (int t = 0; t < s; ++t) {
    if (!P.refactor && warp == 0) {
      // pivot search over rows t..s-1 of column t: max |.|, lowest index on ties
      double best = -1.0;
      int bi = s;
      for (int q = t + lane; q < s; q += 32) {
        const double a = fabs(sm.X[q * LDX + t]);
        if (a > best) { best = a; bi = q; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(HY_FULL, best, o);
        const int oi = __shfl_xor_sync(HY_FULL, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (bi != t && bi < s) {
        for (int c = lane; c < s; c += 32) {
          const double tmp = sm.X[t * LDX + c];
          sm.X[t * LDX + c] = sm.X[bi * LDX + c];
          sm.X[bi * LDX + c] = tmp;
        }
        if (lane == 0) {
          const int tp = sm.perm[t];
          sm.perm[t] = sm.perm[bi];
          sm.perm[bi] = tp;
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      const double piv = sm.X[t * LDX + t];
      bool fired;
      sm.X[t * LDX + t] = perturb(piv, thr, fired);
      log_pivot(P, r + t, piv, fired, thr);
    }
    __syncthreads();
    const double pv = sm.X[t * LDX + t];
    for (int q = t + 1 + tid; q < s; q += SN_THREADS) sm.X[q * LDX + t] /= pv;
    __syncthreads();
    const int rem = s - t - 1;
    for (int idx = tid; idx < rem * rem; idx += SN_THREADS) {
      const int q = t + 1 + idx / rem, c = t + 1 + idx % rem;
      sm.X[q * LDX + c] -= sm.X[q * LDX + t] * sm.X[t * LDX + c];
    }
    __syncthreads();
  }
  // permute the L-union part by tiles (in place, tile read fully before written)
  for (int ca = 0; ca < L; ca += TILE) {
    const int nq = min(TILE, L - ca);
    for (int idx = tid; idx < s * nq; idx += SN_THREADS) {
      const int t = idx / nq, c = idx - t * nq;
      sm.T[t * LDX + c] = Pm[(int64_t)sm.perm[t] * W + ca + c];
    }
    __syncthreads();
    for (int idx = tid; idx < s * nq; idx += SN_THREADS) {
      const int t = idx / nq, c = idx - t * nq;
      Pm[(int64_t)t * W + ca + c] = sm.T[t * LDX + c];
    }
    __syncthreads();
  }
  // panel: permute + U_panel = L_bb^-1 (P panel), rank-1 steps (t ascending per entry)
  for (int ca = L + s; ca < W; ca += TILE) {
    const int nq = min(TILE, W - ca);
    for (int idx = tid; idx < s * nq; idx += SN_THREADS) {
      const int t = idx / nq, c = idx - t * nq;
      sm.T[t * LDX + c] = Pm[(int64_t)sm.perm[t] * W + ca + c];
    }
    __syncthreads();
    for (int tt = 0; tt + 1 < s; ++tt) {
      const int rem = s - tt - 1;
      for (int idx = tid; idx < rem * nq; idx += SN_THREADS) {
        const int q = tt + 1 + idx / nq, c = idx % nq;
        sm.T[q * LDX + c] -= sm.X[q * LDX + tt] * sm.T[tt * LDX + c];
      }
      __syncthreads();
    }
    for (int idx = tid; idx < s * nq; idx += SN_THREADS) {
      const int t = idx / nq, c = idx - t * nq;
      Pm[(int64_t)t * W + ca + c] = sm.T[t * LDX + c];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < s * s; idx += SN_THREADS) {
    const int t = idx / s, tt = idx - t * s;
    Pm[(int64_t)t * W + L + tt] = sm.X[t * LDX + tt];
  }
  if (!P.refactor && tid < s) P.iperm[r + tid] = sm.perm[tid];
}

size_t sn_smem_bytes() { return sizeof(SnSmem); }

// ============================================================================ solve
// b_hat[i] = dr[a] * b[a], a = original row feeding factor row i (inner_perm applied)
__global__ void k_bhat(DevSym S, const int32_t *iperm, const double *b, double *y) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < S.n; i += gridDim.x * blockDim.x) {
    const int u = S.node_of[i];
    int src = i;
    if (S.kind[u] == 1) src = (int)S.first[u] + iperm[i];
    const int64_t a = S.mrow_src[src];
    y[i] = S.dr[a] * b[a];
  }
}

__global__ void k_xout(DevSym S, const double *z, double *x) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < S.n; k += gridDim.x * blockDim.x) {
    const int64_t c = S.perm[k];
    x[c] = S.dc[c] * z[k];
  }
}

// forward substitution, one warp per node (supernode rows: external dot products
// by all lanes, then the in-block unit-lower solve)
__global__ void k_fwd(DevSym S, const double *F, const int32_t *nodes, int count, double *y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x >> 5) + warp;
  if (idx >= count) return;
  const int u = nodes[idx];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *Fu = F + S.valoff[u];
  const int32_t *cc = S.cols + c0;
  double mine0 = 0.0, mine1 = 0.0;  // lane t / t+32 row partials
  for (int t = 0; t < s; ++t) {
    const double *row = Fu + (int64_t)t * W;
    double acc = 0.0;
    for (int p = lane; p < L; p += 32) acc += row[p] * y[cc[p]];
    acc = warp_sum(acc);
    if (lane == (t & 31)) {
      if (t < 32) mine0 = y[r + t] - acc; else mine1 = y[r + t] - acc;
    }
  }
  // in-block: y_t -= sum_{tt<t} L[t][tt] y_tt
  // in-block unit-lower solve; each lane's block-row entries are loaded 8 columns
  // at a time (all in flight together) instead of one dependent load per step
  const int t0 = lane, t1 = lane + 32;
  for (int b0 = 0; b0 < s; b0 += 8) {
    double e0[8], e1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tt = b0 + k;
      e0[k] = (tt < s && t0 > tt && t0 < s) ? Fu[(int64_t)t0 * W + L + tt] : 0.0;
      e1[k] = (tt < s && t1 > tt && t1 < s) ? Fu[(int64_t)t1 * W + L + tt] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tt = b0 + k;
      if (tt < s) {
        const double ytt = __shfl_sync(HY_FULL, tt < 32 ? mine0 : mine1, tt & 31);
        if (t0 > tt && t0 < s) mine0 -= e0[k] * ytt;
        if (t1 > tt && t1 < s) mine1 -= e1[k] * ytt;
      }
    }
  }
  if (lane < s) y[r + lane] = mine0;
  if (lane + 32 < s) y[r + lane + 32] = mine1;
}

__global__ void k_bwd(DevSym S, const double *F, const int32_t *nodes, int count, double *y) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x >> 5) + warp;
  if (idx >= count) return;
  const int u = nodes[idx];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *Fu = F + S.valoff[u];
  const int32_t *cc = S.cols + c0;
  double mine0 = 0.0, mine1 = 0.0;
  for (int t = 0; t < s; ++t) {
    const double *row = Fu + (int64_t)t * W;
    double acc = 0.0;
    for (int p = L + s + lane; p < W; p += 32) acc += row[p] * y[cc[p]];
    acc = warp_sum(acc);
    if (lane == (t & 31)) {
      if (t < 32) mine0 = y[r + t] - acc; else mine1 = y[r + t] - acc;
    }
  }
  for (int tt = s - 1; tt >= 0; --tt) {
    // finalize z_tt
    const double d = Fu[(int64_t)tt * W + L + tt];
    if (lane == (tt & 31)) {
      if (tt < 32) mine0 /= d; else mine1 /= d;
    }
    const double ztt = __shfl_sync(HY_FULL, tt < 32 ? mine0 : mine1, tt & 31);
    const int t0 = lane, t1 = lane + 32;
    if (t0 < tt) mine0 -= Fu[(int64_t)t0 * W + L + tt] * ztt;
    if (t1 < tt) mine1 -= Fu[(int64_t)t1 * W + L + tt] * ztt;
  }
  if (lane < s) y[r + lane] = mine0;
  if (lane + 32 < s) y[r + lane + 32] = mine1;
}

// ---------------------------------------------------------------------------
// Hub rows of the single-instance row path (ROWROW mode): one CTA per standalone
// row with thousands of L entries.  Pull programs (schedule.py): positions grouped
// by intra-row dependency level; a thread takes one <= 64-term work item (the
// position's contributions in ascending step order, the same operation order as
// the sequential row-row loop); longer positions are split into partial sums
// combined in slot order.  The row lives in its own factor storage (L2-resident).
constexpr int HUB1_THREADS = 1024;

__device__ __forceinline__ void hub1_final(const CallP &P, int64_t kd, double *w, int p, double acc,
                                           const double *F, double thr, int64_t row) {
  if (kd >= 0) {
    acc = acc / F[kd];
  } else if (kd == -2) {
    bool fired;
    const double piv = acc;
    acc = perturb(piv, thr, fired);
    log_pivot(P, row, piv, fired, thr);
  }
  w[p] = acc;
}

__global__ void __launch_bounds__(HUB1_THREADS) k_hub1(DevSym S, const CallP *__restrict__ Pd, DevProg R,
                                                       const int32_t *nodes, double *scratch,
                                                       int max_slots) {
  const CallP P = *Pd;
  const int u = nodes[blockIdx.x];
  const int tid = threadIdx.x;
  const int64_t i = S.first[u];
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  double *F = P.F;
  double *w = F + S.valoff[u];
  double *scr = scratch + (size_t)blockIdx.x * max_slots;
  const double thr = P.eps * P.anorm[0];
  for (int q = tid; q < W; q += HUB1_THREADS) w[q] = 0.0;
  __syncthreads();
  {
    const int64_t a = S.mrow_src[i];
    for (int64_t e = S.a_ptr[a] + tid; e < S.a_ptr[a + 1]; e += HUB1_THREADS)
      w[S.colpos[e]] = P.A[e] * S.scale[e];
  }
  __syncthreads();
  const int hr = R.hub_base[u];
  for (int64_t lev = R.hrow_lev[hr]; lev < R.hrow_lev[hr + 1]; ++lev) {
    for (int64_t it = R.lev_wi[lev] + tid; it < R.lev_wi[lev + 1]; it += HUB1_THREADS) {
      const int p = R.wi_p[it];
      const int slot = R.wi_slot[it];
      const int64_t y1 = R.wi_y1[it];
      double acc = slot < 0 ? w[p] : 0.0;
      for (int64_t y = R.wi_y0[it]; y < y1; ++y) acc -= w[R.pred_p[y]] * F[R.pred_u[y]];
      if (slot < 0)
        hub1_final(P, R.wi_kd[it], w, p, acc, F, thr, i);
      else
        scr[slot] = acc;
    }
    if (R.lev_sp[lev + 1] > R.lev_sp[lev]) {
      __syncthreads();
      for (int64_t k2 = R.lev_sp[lev] + tid; k2 < R.lev_sp[lev + 1]; k2 += HUB1_THREADS) {
        const int p = R.sp_p[k2];
        double acc = w[p];
        const int s0 = R.sp_s0[k2], ns = R.sp_n[k2];
        for (int c = 0; c < ns; ++c) acc += scr[s0 + c];
        hub1_final(P, R.sp_kd[k2], w, p, acc, F, thr, i);
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Chunked substitution: per level, (node, column chunk) partial dot products of
// every row of the node over its off-block part (L-union for forward, panel for
// backward), written to a scratch slot; then one warp per node combines the chunk
// partials in slot order and runs the in-block triangular solve.
struct SolveChunk {
  int32_t node;
  int32_t c0, c1;     // column positions [c0, c1) within the node's list
  int32_t slot;       // scratch slot (x 64 rows)
};

__global__ void k_solve_part(DevSym S, const double *const *Fp, const SolveChunk *ch, int count,
                             const double *y, double *scratch, int fwd) {
  pdl_wait();
  pdl_launch_dependents();
  const double *F = *Fp;   // factor values of this call (device-resident pointer: graph replay)
  const int j = blockIdx.x;
  if (j >= count) return;
  const SolveChunk c = ch[j];
  const int u = c.node;
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t cp = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - cp);
  const double *Fu = F + S.valoff[u];
  const int32_t *cc = S.cols + cp;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  // the chunk's (<= 512) gathered solution values, once per warp (lanes over
  // columns), reused by every row; two rows per reduction
  double yv[16];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    const int q = c.c0 + lane + 32 * k;
    yv[k] = q < c.c1 ? y[cc[q]] : 0.0;
  }
  for (int t = 2 * warp; t < s; t += 2 * nw) {
    const double *ra = Fu + (int64_t)t * W;
    const bool two = t + 1 < s;
    double a = 0.0, b = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int q = c.c0 + lane + 32 * k;
      if (q < c.c1) {
        a += ra[q] * yv[k];
        if (two) b += ra[W + q] * yv[k];
      }
    }
    a = warp_sum(a);
    b = warp_sum(b);
    if (lane == 0) {
      scratch[(int64_t)c.slot * 64 + t] = a;
      if (two) scratch[(int64_t)c.slot * 64 + t + 1] = b;
    }
  }
}

// forward finish: y_t = y_t - sum(chunk partials) - sum_{tt<t} L[t][tt] y_tt
// Off-block dot products of a small node's rows (columns [lo, hi) of each row)
// against the solution vector, done by one warp: per 128-column block the gathered
// solution values are loaded once (lanes over columns) and reused by every row;
// two rows per step, each reduced across the warp and subtracted from the lane
// that owns the row (row t lives on lane t&31, in mine0 for t < 32 else mine1).
__device__ __forceinline__ void offblock_dots(const double *Fu, int W, const int32_t *cc,
                                              const double *y, int lo, int hi, int s, int lane,
                                              double &mine0, double &mine1) {
  for (int q0 = lo; q0 < hi; q0 += 128) {
    double yv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int q = q0 + lane + 32 * k;
      yv[k] = q < hi ? y[cc[q]] : 0.0;
    }
    for (int t = 0; t < s; t += 2) {
      const double *ra = Fu + (int64_t)t * W;
      const bool two = t + 1 < s;
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int q = q0 + lane + 32 * k;
        if (q < hi) {
          a += ra[q] * yv[k];
          if (two) b += ra[W + q] * yv[k];
        }
      }
      a = warp_sum(a);
      b = warp_sum(b);
      if (lane == (t & 31)) {
        if (t < 32) mine0 -= a; else mine1 -= a;
      }
      if (two && lane == ((t + 1) & 31)) {
        if (t + 1 < 32) mine0 -= b; else mine1 -= b;
      }
    }
  }
}

__global__ void k_fwd_fin(DevSym S, const double *const *Fp, const SolveRec *recs, int count,
                          const double *scratch, double *y) {
  pdl_wait();
  pdl_launch_dependents();
  const double *F = *Fp;   // factor values of this call (device-resident pointer: graph replay)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x >> 5) + warp;
  if (idx >= count) return;
  const SolveRec sr = recs[idx];
  const int r = sr.r, s = sr.s, W = sr.W, L = sr.L;
  const double *Fu = F + sr.valoff;
  const int a0 = sr.slot0, an = sr.nslot;
  double mine0 = 0.0, mine1 = 0.0;
  if (lane < s) {
    double acc = y[r + lane];
    for (int k = 0; k < an; ++k) acc -= scratch[(int64_t)(a0 + k) * 64 + lane];
    mine0 = acc;
  }
  if (lane + 32 < s) {
    double acc = y[r + lane + 32];
    for (int k = 0; k < an; ++k) acc -= scratch[(int64_t)(a0 + k) * 64 + lane + 32];
    mine1 = acc;
  }
  if (an == 0 && L > 0)   // small node: the warp computes the off-block dot products itself
    offblock_dots(Fu, W, S.cols + sr.col0, y, 0, L, s, lane, mine0, mine1);
  // in-block unit-lower solve; each lane's block-row entries are loaded 8 columns
  // at a time (all in flight together) instead of one dependent load per step
  const int t0 = lane, t1 = lane + 32;
  for (int b0 = 0; b0 < s; b0 += 8) {
    double e0[8], e1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tt = b0 + k;
      e0[k] = (tt < s && t0 > tt && t0 < s) ? Fu[(int64_t)t0 * W + L + tt] : 0.0;
      e1[k] = (tt < s && t1 > tt && t1 < s) ? Fu[(int64_t)t1 * W + L + tt] : 0.0;
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tt = b0 + k;
      if (tt < s) {
        const double ytt = __shfl_sync(HY_FULL, tt < 32 ? mine0 : mine1, tt & 31);
        if (t0 > tt && t0 < s) mine0 -= e0[k] * ytt;
        if (t1 > tt && t1 < s) mine1 -= e1[k] * ytt;
      }
    }
  }
  if (lane < s) y[r + lane] = mine0;
  if (lane + 32 < s) y[r + lane + 32] = mine1;
}

__global__ void k_solve_rec(DevSym S, const int32_t *nodes, const int32_t *slot0, const int32_t *nslot, int64_t count,
                            SolveRec *out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x) {
    const int u = nodes[j];
    SolveRec r;
    r.valoff = S.valoff[u];
    r.col0 = S.colptr[u];
    r.r = (int32_t)S.first[u];
    r.s = (int32_t)(S.first[u + 1] - S.first[u]);
    r.W = (int32_t)(S.colptr[u + 1] - S.colptr[u]);
    r.L = S.nl[u];
    r.slot0 = slot0[j];
    r.nslot = nslot[j];
    r.pad[0] = r.pad[1] = 0;
    out[j] = r;
  }
}

// backward finish: z_t = (y_t - sum(partials) - sum_{tt>t} U[t][tt] z_tt) / U[t][t]
__global__ void k_bwd_fin(DevSym S, const double *const *Fp, const SolveRec *recs, int count,
                          const double *scratch, double *y) {
  pdl_wait();
  pdl_launch_dependents();
  const double *F = *Fp;   // factor values of this call (device-resident pointer: graph replay)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int idx = blockIdx.x * (blockDim.x >> 5) + warp;
  if (idx >= count) return;
  const SolveRec sr = recs[idx];
  const int r = sr.r, s = sr.s, W = sr.W, L = sr.L;
  const double *Fu = F + sr.valoff;
  const int a0 = sr.slot0, an = sr.nslot;
  double mine0 = 0.0, mine1 = 0.0;
  if (lane < s) {
    double acc = y[r + lane];
    for (int k = 0; k < an; ++k) acc -= scratch[(int64_t)(a0 + k) * 64 + lane];
    mine0 = acc;
  }
  if (lane + 32 < s) {
    double acc = y[r + lane + 32];
    for (int k = 0; k < an; ++k) acc -= scratch[(int64_t)(a0 + k) * 64 + lane + 32];
    mine1 = acc;
  }
  if (an == 0 && L + s < W)
    offblock_dots(Fu, W, S.cols + sr.col0, y, L + s, W, s, lane, mine0, mine1);
  // in-block upper solve (descending), entries loaded 8 columns at a time; the
  // diagonal entry of row tt is in its own lane's block (k = tt - b0)
  const int t0 = lane, t1 = lane + 32;
  for (int b0 = ((s - 1) / 8) * 8; b0 >= 0; b0 -= 8) {
    double e0[8], e1[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const int tt = b0 + k;
      e0[k] = (tt < s && t0 <= tt) ? Fu[(int64_t)t0 * W + L + tt] : 0.0;
      e1[k] = (tt < s && t1 <= tt) ? Fu[(int64_t)t1 * W + L + tt] : 0.0;
    }
#pragma unroll
    for (int k = 7; k >= 0; --k) {
      const int tt = b0 + k;
      if (tt < s) {
        if (lane == (tt & 31)) {
          if (tt < 32) mine0 /= e0[k]; else mine1 /= e1[k];
        }
        const double ztt = __shfl_sync(HY_FULL, tt < 32 ? mine0 : mine1, tt & 31);
        if (t0 < tt) mine0 -= e0[k] * ztt;
        if (t1 < tt) mine1 -= e1[k] * ztt;
      }
    }
  }
  if (lane < s) y[r + lane] = mine0;
  if (lane + 32 < s) y[r + lane + 32] = mine1;
}


// ---------------------------------------------------------------------------
// Residual and componentwise backward error in original coordinates
// (matrix.py:258-285; "r = b − A·x ... full precision"): thread
// per row, the row's entries in index order with separately rounded products and
// sums (no fused multiply-add), exactly as the reference's row loops — so both
// the residual and the backward error are bitwise the reference's for the same
// x.  max over rows through an integer atomicMax on the (non-negative) bits.
__global__ void k_resid_berr(int n, const int64_t *row_ptr, const int32_t *col_idx,
                             const double *vals, const double *x, const double *b, double *r,
                             unsigned long long *berr_bits) {
  double worst = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0, mag = 0.0;
    for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
      const double v = vals[t];
      const double xa = x[col_idx[t]];
      acc = __dadd_rn(acc, __dmul_rn(v, xa));
      mag = __dadd_rn(mag, __dmul_rn(fabs(v), fabs(xa)));
    }
    const double bi = b[i];
    if (r) r[i] = __dsub_rn(bi, acc);
    const double num = fabs(__dsub_rn(bi, acc));
    const double den = __dadd_rn(mag, fabs(bi));
    if (den != 0.0) {
      const double rel = __ddiv_rn(num, den);
      if (rel > worst) worst = rel;
    }
  }
  // warp max, then one atomic per warp (non-negative doubles order as their bits)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(HY_FULL, worst, o));
  if ((threadIdx.x & 31) == 0 && worst > 0.0)
    atomicMax(berr_bits, (unsigned long long)__double_as_longlong(worst));
}

// x += dx (the refinement update, elementwise as numpy)
__global__ void k_axpy1(int n, double *x, const double *dx) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    x[i] = __dadd_rn(x[i], dx[i]);
}

// Batched k_resid_berr: blockIdx.y = instance (skipped when mask[b] == 0); values,
// x, b, r row-major [B][nnz] / [B][n]; one backward error per instance.
__global__ void k_resid_berr_b(int n, int64_t nnz, const int64_t *row_ptr, const int32_t *col_idx,
                               const double *vals, const double *x, const double *b, double *r,
                               unsigned long long *berr_bits, const int32_t *mask) {
  const int64_t inst = blockIdx.y;
  if (mask && !mask[inst]) return;
  const double *v = vals + inst * nnz;
  const double *xi = x + inst * n;
  const double *bi_ = b + inst * n;
  double worst = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    double acc = 0.0, mag = 0.0;
    for (int64_t t = row_ptr[i]; t < row_ptr[i + 1]; ++t) {
      const double a = v[t];
      const double xa = xi[col_idx[t]];
      acc = __dadd_rn(acc, __dmul_rn(a, xa));
      mag = __dadd_rn(mag, __dmul_rn(fabs(a), fabs(xa)));
    }
    const double bi = bi_[i];
    if (r) r[inst * n + i] = __dsub_rn(bi, acc);
    const double num = fabs(__dsub_rn(bi, acc));
    const double den = __dadd_rn(mag, fabs(bi));
    if (den != 0.0) {
      const double rel = __ddiv_rn(num, den);
      if (rel > worst) worst = rel;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) worst = fmax(worst, __shfl_xor_sync(HY_FULL, worst, o));
  if ((threadIdx.x & 31) == 0 && worst > 0.0)
    atomicMax(berr_bits + inst, (unsigned long long)__double_as_longlong(worst));
}

// y[b] = x[b] (+ dx[b]) for the instances with mask[b] != 0 (all when mask == NULL)
__global__ void k_axpy_b(int n, double *y, const double *x, const double *dx, const int32_t *mask) {
  const int64_t inst = blockIdx.y;
  if (mask && !mask[inst]) return;
  const int64_t o = inst * n;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    y[o + i] = dx ? __dadd_rn(x[o + i], dx[o + i]) : x[o + i];
}
}  // namespace hy
