// hylu_slab.cu — supernode targets as column slabs (single-instance factorization).
//
// A supernode target T (s rows, W columns: L-union | diagonal block | panel) is cut
// by the host (schedule.build_slab_plan) into column slabs; one CTA owns one slab
// and keeps its s x sw accumulator in shared memory for its whole life.  Sources
// are applied in ascending order; for source v the slab owning
// v's block columns computes the multiplier block X_v = T[:, blk_v] · U_vv⁻¹
// (TRSM with the source's upper, non-unit diagonal block), stores it as T's final
// L values and publishes a flag; every slab whose columns meet v's beyond-block
// columns waits for that flag and applies T[:, cols] -= X_v · U_v[:, cols]
// (register-tiled FP64 GEMM into shared memory).  The block slab then runs the
// in-supernode LU with pivoting restricted to the diagonal block
// and perturbation and publishes L_bb / U_bb / inner_perm; panel
// slabs wait, apply the row permutation and the unit-lower TRSM.  A per-level pass
// (k_lperm) then applies the pivot row permutation to the L-union columns.
//
// CTAs take a ticket from an atomic counter and map it to slab ids in ascending
// order; a slab only ever waits for flags published by lower slab ids of the same
// target (owners of blocks left of its columns, the block slab), which were
// dispatched earlier, so the wait graph is acyclic and every waited-on CTA is
// resident or finished.
#include "hylu_common.cuh"

namespace hy {

struct SlabDev {
  const int32_t *sl_node;
  const int32_t *sl_c0;
  const int32_t *sl_c1;
  const int8_t *sl_kind;
  const int64_t *it_ptr;
  const int32_t *it_k;
  const int32_t *it_q0;
  const int32_t *it_q1;
  const int8_t *it_own;
  const int32_t *dep_pb;   // per dependency edge: block position of the source in the target
};

constexpr int SLAB_THREADS = 256;
constexpr int XLD = 65;

__device__ __forceinline__ int ld_acq(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(SLAB_THREADS, 1)
    k_slab(DevSym S, const CallP *__restrict__ Pd, SlabDev D, int slab_base, int *counter, int *dep_flags, int *lu_flags,
           int epoch, int Smax, int Mmax, int SWmax, int ACCmax) {
  const CallP P = *Pd;
  extern __shared__ __align__(16) double smd[];
  __shared__ int s_ticket;
  __shared__ int s_pinv[64];
  __shared__ int s_perm[64];
  __shared__ int s_pos[64];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) s_ticket = atomicAdd(counter, 1);
  __syncthreads();
  const int sid = slab_base + s_ticket;
  const int u = D.sl_node[sid];
  const int c_lo = D.sl_c0[sid], c_hi = D.sl_c1[sid];
  const int skind = D.sl_kind[sid];
  const int sw = c_hi - c_lo;
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  double *F = P.F;
  double *Pm = F + S.valoff[u];
  double *acc = smd;                                         // s x sw (stride sw)
  int32_t *tcol = reinterpret_cast<int32_t *>(acc + (size_t)ACCmax);
  double *Xs = reinterpret_cast<double *>(tcol + ((SWmax + 1) & ~1));  // Smax x XLD
  double *Ut = Xs + (size_t)Smax * XLD;                      // max(Mmax, Smax) x XLD
  const double thr = P.eps * P.anorm[0];

  for (int c = tid; c < sw; c += SLAB_THREADS) tcol[c] = S.cols[c0 + c_lo + c];
  for (int q = tid; q < s * sw; q += SLAB_THREADS) acc[q] = 0.0;
  if (tid < s) {
    if (P.refactor) {
      s_pinv[P.iperm_prior[r + tid]] = tid;
    } else {
      s_pinv[tid] = tid;
    }
  }
  __syncthreads();
  // scatter the target's M rows restricted to this slab's columns
  for (int t = warp; t < s; t += SLAB_THREADS / 32) {
    const int64_t a = S.mrow_src[r + t];
    double *row = acc + (size_t)s_pinv[t] * sw;
    for (int64_t e = S.a_ptr[a] + lane; e < S.a_ptr[a + 1]; e += 32) {
      const int cp = S.colpos[e] - c_lo;
      if (cp >= 0 && cp < sw) row[cp] = P.A[e] * S.scale[e];
    }
  }
  __syncthreads();

  // ---------------------------------------------------------------- source steps
  const int tr = tid >> 4, tcl = tid & 15;
  for (int64_t it = D.it_ptr[sid]; it < D.it_ptr[sid + 1]; ++it) {
    const int k = D.it_k[it];
    const int q0 = D.it_q0[it], q1 = D.it_q1[it];
    const bool own = D.it_own[it] != 0;
    const int64_t dk = S.dptr[u] + k;
    const int v = S.deps[dk];
    const int vf = (int)S.first[v];
    const int vs = (int)(S.first[v + 1] - vf);
    const int64_t vc0 = S.colptr[v];
    const int vW = (int)(S.colptr[v + 1] - vc0);
    const int vnl = S.nl[v];
    const double *vb = F + S.valoff[v];
    const int pb0 = D.dep_pb[dk];
    const int tb0 = S.cols[c0 + pb0] - vf;   // first present block row of v
    const int m = vs - tb0;                   // multipliers (block columns) present
    if (own) {
      // X = acc[:, pb0-c_lo .. +m) · U_bb^-1, U_bb = rows/cols tb0.. of v's diagonal block
      for (int idx = tid; idx < m * m; idx += SLAB_THREADS) {
        const int a = idx / m, b2 = idx - a * m;
        Ut[a * XLD + b2] = b2 >= a ? vb[(int64_t)(tb0 + a) * vW + vnl + tb0 + b2] : 0.0;
      }
      __syncthreads();
      // 4 threads per target row, columns interleaved mod 4; warp-synchronous
      {
        const int t = tid >> 2, qd = tid & 3;
        double *xr = acc + (size_t)t * sw + (pb0 - c_lo);
        const bool act = t < s;
        for (int a = 0; a < m; ++a) {
          double x = 0.0;
          if (act && (a & 3) == qd) {
            x = xr[a] / Ut[a * XLD + a];
            xr[a] = x;
          }
          x = __shfl_sync(HY_FULL, x, (lane & ~3) | (a & 3));
          if (act && x != 0.0)
            for (int b2 = a + 1 + ((qd - a - 1) & 3); b2 < m; b2 += 4) xr[b2] -= x * Ut[a * XLD + b2];
          __syncwarp();
        }
      }
      __syncthreads();
      for (int idx = tid; idx < s * m; idx += SLAB_THREADS) {
        const int t = idx / m, a = idx - t * m;
        const double x = acc[(size_t)t * sw + (pb0 - c_lo) + a];
        Xs[t * XLD + a] = x;
        Pm[(int64_t)t * W + pb0 + a] = x;
      }
      __threadfence();
      __syncthreads();
      if (tid == 0) st_rel(dep_flags + dk, epoch);
    } else {
      if (tid == 0)
        while (ld_acq(dep_flags + dk) != epoch) __nanosleep(128);
      __syncthreads();
      for (int idx = tid; idx < s * m; idx += SLAB_THREADS) {
        const int t = idx / m, a = idx - t * m;
        Xs[t * XLD + a] = __ldcg(Pm + (int64_t)t * W + pb0 + a);
      }
    }
    if (q1 <= q0) {
      __syncthreads();
      continue;
    }
    // GEMM: acc[:, pos(q)] -= X · U_v[tb0.., q] over beyond-block columns [q0, q1)
    const int qbase = vnl + vs;
    for (int qa = q0; qa < q1; qa += 64) {
      const int nq = min(64, q1 - qa);
      __syncthreads();
      for (int idx = tid; idx < m * 64; idx += SLAB_THREADS) {
        const int a = idx >> 6, c = idx & 63;
        Ut[a * XLD + c] = c < nq ? vb[(int64_t)(tb0 + a) * vW + qbase + qa + c] : 0.0;
      }
      if (tid < nq) {
        const int key = S.cols[vc0 + qbase + qa + tid];
        s_pos[tid] = lower_bound_i32(tcol, 0, sw, key);
      }
      __syncthreads();
      double c4[4][4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) c4[x][y] = 0.0;
      for (int a = 0; a < m; ++a) {
        double xv[4], uv[4];
#pragma unroll
        for (int x = 0; x < 4; ++x) xv[x] = (tr + 16 * x < s) ? Xs[(tr + 16 * x) * XLD + a] : 0.0;
#pragma unroll
        for (int y = 0; y < 4; ++y) uv[y] = Ut[a * XLD + tcl + 16 * y];
#pragma unroll
        for (int x = 0; x < 4; ++x)
#pragma unroll
          for (int y = 0; y < 4; ++y) c4[x][y] = fma(xv[x], uv[y], c4[x][y]);
      }
#pragma unroll
      for (int x = 0; x < 4; ++x) {
        const int t = tr + 16 * x;
        if (t < s) {
#pragma unroll
          for (int y = 0; y < 4; ++y) {
            const int c = tcl + 16 * y;
            if (c < nq) acc[(size_t)t * sw + s_pos[c]] -= c4[x][y];
          }
        }
      }
    }
    __syncthreads();
  }

  // ---------------------------------------------------------------- finalize
  if (skind == 0) {
    for (int idx = tid; idx < s * sw; idx += SLAB_THREADS) {
      const int t = idx / sw, c = idx - t * sw;
      Pm[(int64_t)t * W + c_lo + c] = acc[idx];
    }
    return;
  }
  if (skind == 1) {
    // block slab: columns [L, L+s) at acc offset L - c_lo (== 0); LU with block pivoting
    const int bo = L - c_lo;
    if (tid < s) s_perm[tid] = tid;
    __syncthreads();
    for (int t = 0; t < s; ++t) {
      if (!P.refactor && warp == 0) {
        double best = -1.0;
        int bi = s;
        for (int q = t + lane; q < s; q += 32) {
          const double av = fabs(acc[(size_t)q * sw + bo + t]);
          if (av > best) { best = av; bi = q; }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(HY_FULL, best, o);
          const int oi = __shfl_xor_sync(HY_FULL, bi, o);
          if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
        }
        if (bi != t && bi < s) {
          for (int c = lane; c < sw; c += 32) {
            const double tmp = acc[(size_t)t * sw + c];
            acc[(size_t)t * sw + c] = acc[(size_t)bi * sw + c];
            acc[(size_t)bi * sw + c] = tmp;
          }
          if (lane == 0) {
            const int tp = s_perm[t];
            s_perm[t] = s_perm[bi];
            s_perm[bi] = tp;
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        const double piv = acc[(size_t)t * sw + bo + t];
        bool fired;
        acc[(size_t)t * sw + bo + t] = perturb(piv, thr, fired);
        log_pivot(P, r + t, piv, fired, thr);
      }
      __syncthreads();
      const double pv = acc[(size_t)t * sw + bo + t];
      for (int q = t + 1 + tid; q < s; q += SLAB_THREADS) acc[(size_t)q * sw + bo + t] /= pv;
      __syncthreads();
      const int rem_r = s - t - 1, rem_c = sw - (bo + t + 1);
      if (rem_r > 0 && rem_c > 0) {
        for (int idx = tid; idx < rem_r * rem_c; idx += SLAB_THREADS) {
          const int q = t + 1 + idx / rem_c, c = bo + t + 1 + idx % rem_c;
          acc[(size_t)q * sw + c] -= acc[(size_t)q * sw + bo + t] * acc[(size_t)t * sw + c];
        }
      }
      __syncthreads();
    }
    for (int idx = tid; idx < s * sw; idx += SLAB_THREADS) {
      const int t = idx / sw, c = idx - t * sw;
      Pm[(int64_t)t * W + c_lo + c] = acc[idx];
    }
    if (tid < s) {
      if (P.refactor)
        P.iperm[r + tid] = P.iperm_prior[r + tid];
      else
        P.iperm[r + tid] = s_perm[tid];
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) st_rel(lu_flags + u, epoch);
    return;
  }
  // panel slab: wait for the block LU, permute rows, unit-lower TRSM
  if (tid == 0)
    while (ld_acq(lu_flags + u) != epoch) __nanosleep(128);
  __syncthreads();
  if (tid < s) s_perm[tid] = P.refactor ? tid : __ldcg(P.iperm + r + tid);
  for (int idx = tid; idx < s * s; idx += SLAB_THREADS) {
    const int t = idx / s, a = idx - t * s;
    Xs[t * XLD + a] = __ldcg(Pm + (int64_t)t * W + L + a);
  }
  __syncthreads();
  bool ident = true;
  for (int t = 0; t < s; ++t) ident &= (s_perm[t] == t);
  if (!ident) {
    for (int ca = 0; ca < sw; ca += 64) {
      const int nq = min(64, sw - ca);
      for (int idx = tid; idx < s * nq; idx += SLAB_THREADS) {
        const int t = idx / nq, c = idx - t * nq;
        Ut[t * XLD + c] = acc[(size_t)s_perm[t] * sw + ca + c];
      }
      __syncthreads();
      for (int idx = tid; idx < s * nq; idx += SLAB_THREADS) {
        const int t = idx / nq, c = idx - t * nq;
        acc[(size_t)t * sw + ca + c] = Ut[t * XLD + c];
      }
      __syncthreads();
    }
  }
  for (int t = 0; t + 1 < s; ++t) {
    const int rem = s - t - 1;
    for (int idx = tid; idx < rem * sw; idx += SLAB_THREADS) {
      const int q = t + 1 + idx / sw, c = idx % sw;
      acc[(size_t)q * sw + c] -= Xs[q * XLD + t] * acc[(size_t)t * sw + c];
    }
    __syncthreads();
  }
  for (int idx = tid; idx < s * sw; idx += SLAB_THREADS) {
    const int t = idx / sw, c = idx - t * sw;
    Pm[(int64_t)t * W + c_lo + c] = acc[idx];
  }
}

// Apply each supernode's pivot permutation to its L-union columns (after the level).
__global__ void k_lperm(DevSym S, const CallP *__restrict__ Pd, const int32_t *sns, int count) {
  const CallP P = *Pd;
  __shared__ double tile[64][65];
  __shared__ int perm[64];
  __shared__ int ident;
  const int j = blockIdx.x;
  if (j >= count) return;
  const int u = sns[j];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  const int L = S.nl[u];
  double *Pm = P.F + S.valoff[u];
  if (threadIdx.x == 0) ident = 1;
  __syncthreads();
  if (threadIdx.x < s) {
    perm[threadIdx.x] = P.iperm[r + threadIdx.x];
    if (perm[threadIdx.x] != (int)threadIdx.x) ident = 0;
  }
  __syncthreads();
  if (ident) return;
  for (int ca = blockIdx.y * 64; ca < L; ca += 64 * gridDim.y) {
    const int nq = min(64, L - ca);
    for (int idx = threadIdx.x; idx < s * nq; idx += blockDim.x) {
      const int t = idx / nq, c = idx - t * nq;
      tile[t][c] = Pm[(int64_t)perm[t] * W + ca + c];
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < s * nq; idx += blockDim.x) {
      const int t = idx / nq, c = idx - t * nq;
      Pm[(int64_t)t * W + ca + c] = tile[t][c];
    }
    __syncthreads();
  }
}

size_t slab_smem_bytes(int Smax, int Mmax, int SWmax, int ACCmax) {
  const int urows = Mmax > Smax ? Mmax : Smax;
  return (size_t)ACCmax * sizeof(double) + (size_t)((SWmax + 1) & ~1) * sizeof(int32_t) +
         (size_t)(Smax + urows) * XLD * sizeof(double);
}

}  // namespace hy
