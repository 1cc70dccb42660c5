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

constexpr int BW = 4;
// warps per block (bwd / fwd kernels); BWD_W / BWD_WL (hylu_common.cuh): backward-solve entries per batch
#ifndef HUB_THREADS_DEF
#define HUB_THREADS_DEF 768   // c4 ms/step, round-2 final kernels: 512: 14.37, 640: 14.29, 768: 14.14-14.17, 1024: 14.75
#endif
constexpr int HUB_THREADS = HUB_THREADS_DEF;
int hub_threads() { return HUB_THREADS; }
#ifndef HUB_I
#define HUB_I 1     // work items per warp per round (staged hub levels; 1-8 measured, 1 best)
#endif
#ifndef HUB_P
#define HUB_P 12    // predecessors per item per round (c4 ms/step with longest-first items: 8: 14.33, 10: 14.79, 12: 14.23, 14: 14.33, 16: 14.45)
#endif
constexpr int HUB_CAPI = 1024;   // staged work items per level (per buffer)
constexpr int HUB_CAPP = 4096;   // staged predecessor records per level (per buffer)
constexpr size_t HUB_BUF = (size_t)HUB_CAPP * (8 + 4) + (size_t)HUB_CAPI * (8 * 3 + 4 * 2);
size_t hub_smem_bytes() { return 2 * HUB_BUF; }

// ---------------------------------------------------------------------------
// Dependency flags: flag[node * G + g] == epoch once (node, group) is complete.
__device__ __forceinline__ int ld_acquire(const int *p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(int *p, int v) {
  asm volatile("st.relaxed.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// one-sided fences: the release side is a MEMBAR without the L1 invalidation (CCTL.IVALL)
// that fence.acq_rel appends; the acquire side is the invalidation alone
__device__ __forceinline__ void fence_release_gpu() { asm volatile("fence.release.gpu;" ::: "memory"); }
__device__ __forceinline__ void fence_acquire_gpu() { asm volatile("fence.acquire.gpu;" ::: "memory"); }
__device__ __forceinline__ void st_release(int *p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ void cp_async8(double *smem_dst, const double *gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async4(int32_t *smem_dst, const int32_t *gsrc) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(smem_dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(d), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

constexpr int PIPE_WARPS = 4;
#ifdef HYLU_TRACE
// phase cycle counters of a pipeline task (debug build, scripts/pipe_trace.py)
struct TraceAcc {
  long long init, mult, upd, fin;
};
#define TR_DECL , TraceAcc &tacc
#define TR_ARG , tacc
#define TR_T(x) const long long x = clock64();
#define TR_ADD(f, a, b) tacc.f += (b) - (a);
#else
#define TR_DECL
#define TR_ARG
#define TR_T(x)
#define TR_ADD(f, a, b)
#endif
// Persistent, dependency-driven row kernel for a segment of levels without hub
// nodes (the device form of SPEC's pipeline mode): warps claim
// (node, group) tasks in level-major order from an atomic counter, wait on the
// completion flags of the node's in-segment dependencies, run the task, then
// publish its flag.  Claim order is topological and every claimed task is held by
// a resident warp, so the earliest unfinished claimed task can always proceed.
// Task descriptor (built on the host in claim order): everything a task needs
// before its first data load, in one 48-byte record.


// ---------------------------------------------------------------------------
// Pair mode: one warp runs the same node for two adjacent groups (g, g+1), lane =
// instance g*32+lane and (g+1)*32+lane.  Every metadata load (task record, row
// record, step program, rel lists) and every dependency poll now serves 64
// instances, and each step has two independent FMA/load chains in flight.  The
// value layout is unchanged (the allocation is padded to an even group count, so
// the pair of the last odd group computes on padding: not live, no atomics).
#ifndef PIPE_RINV
#define PIPE_RINV 1      // multipliers = value x stored reciprocal of the source pivot (else a division)
#endif
#ifndef P2W_DEF
#define P2W_DEF 4
#endif
constexpr int P2W = P2W_DEF;   // update entries per batch in run_steps2 (all loads issued first)
template <typename WPtr>
__device__ __forceinline__ void run_steps2(const DevProg &R, int64_t s0, int64_t s1, WPtr wa,
                                           WPtr wc, const double *ga, const double *gc,
                                           const double *ya, const double *yc, double &acA,
                                           double &acC, const double *ria, const double *ric) {
  if (s0 >= s1) return;
  int p = __ldg(R.st_p + s0);
  int64_t src = __ldg(R.st_src + s0);
  int cnt = __ldg(R.st_cnt + s0);
  int64_t ro = __ldg(R.st_rel + s0);
  int64_t j = __ldg(R.st_j + s0);
  // pivot of the source row: its reciprocal (one multiply per step) when available
  double da = PIPE_RINV ? __ldcg(ria + j * 32) : __ldcg(ga + src * 32);
  double dc = PIPE_RINV ? __ldcg(ric + j * 32) : __ldcg(gc + src * 32);
  double yja = __ldcg(ya + j * 32), yjc = __ldcg(yc + j * 32);
  for (int64_t st = s0; st < s1; ++st) {
    int pn = 0, cn = 0;
    int64_t sn = 0, rn = 0;
    double dna = 1.0, dnc = 1.0, yna = 0.0, ync = 0.0;
    if (st + 1 < s1) {
      pn = __ldg(R.st_p + st + 1);
      sn = __ldg(R.st_src + st + 1);
      cn = __ldg(R.st_cnt + st + 1);
      rn = __ldg(R.st_rel + st + 1);
      const int64_t jn = __ldg(R.st_j + st + 1);
      dna = PIPE_RINV ? __ldcg(ria + jn * 32) : __ldcg(ga + sn * 32);
      dnc = PIPE_RINV ? __ldcg(ric + jn * 32) : __ldcg(gc + sn * 32);
      yna = __ldcg(ya + jn * 32);
      ync = __ldcg(yc + jn * 32);
    }
    const int32_t *rl = R.rel + ro;
    const double *ua = ga + (src + 1) * 32;
    const double *uc = gc + (src + 1) * 32;
    const double la = PIPE_RINV ? wa[p * 32] * da : wa[p * 32] / da;
    const double lc = PIPE_RINV ? wc[p * 32] * dc : wc[p * 32] / dc;
    wa[p * 32] = la;
    wc[p * 32] = lc;
    acA -= la * yja;
    acC -= lc * yjc;
    for (int q = 0; q < cnt; q += P2W) {
      int t[P2W];
      double xa[P2W], xc[P2W];
#pragma unroll
      for (int k = 0; k < P2W; ++k) {
        const bool ok = q + k < cnt;
        t[k] = ok ? __ldg(rl + q + k) : 0;
        xa[k] = ok ? __ldcg(ua + (q + k) * 32) : 0.0;
        xc[k] = ok ? __ldcg(uc + (q + k) * 32) : 0.0;
      }
      double va[P2W], vc[P2W];
#pragma unroll
      for (int k = 0; k < P2W; ++k) {
        va[k] = wa[t[k] * 32];
        vc[k] = wc[t[k] * 32];
      }
#pragma unroll
      for (int k = 0; k < P2W; ++k)
        if (q + k < cnt) {
          wa[t[k] * 32] = va[k] - la * xa[k];
          wc[t[k] * 32] = vc[k] - lc * xc[k];
        }
    }
    p = pn; src = sn; cnt = cn; ro = rn; da = dna; dc = dnc; yja = yna; yjc = ync;
  }
}

// run_steps2 over a program window staged in shared memory (packed step records and
// the window's target positions): the index loads of every step become shared loads.
template <typename WPtr>
__device__ __forceinline__ void run_steps2s(const StepRec *rec, const int32_t *relw, int s0, int s1, WPtr wa,
                                            WPtr wc, const double *ga, const double *gc,
                                            const double *ya, const double *yc, double &acA,
                                            double &acC, const double *ria, const double *ric TR_DECL) {
  if (s0 >= s1) return;
  StepRec cr = rec[s0];
  double da = PIPE_RINV ? __ldcg(ria + (int64_t)cr.j * 32) : __ldcg(ga + (int64_t)cr.src * 32);
  double dc = PIPE_RINV ? __ldcg(ric + (int64_t)cr.j * 32) : __ldcg(gc + (int64_t)cr.src * 32);
  double yja = __ldcg(ya + (int64_t)cr.j * 32), yjc = __ldcg(yc + (int64_t)cr.j * 32);
  for (int st = s0; st < s1; ++st) {
    StepRec nx = cr;
    double dna = 1.0, dnc = 1.0, yna = 0.0, ync = 0.0;
    if (st + 1 < s1) {
      nx = rec[st + 1];
      dna = PIPE_RINV ? __ldcg(ria + (int64_t)nx.j * 32) : __ldcg(ga + (int64_t)nx.src * 32);
      dnc = PIPE_RINV ? __ldcg(ric + (int64_t)nx.j * 32) : __ldcg(gc + (int64_t)nx.src * 32);
      yna = __ldcg(ya + (int64_t)nx.j * 32);
      ync = __ldcg(yc + (int64_t)nx.j * 32);
    }
    TR_T(c0)
    const int p = cr.p, cnt = cr.cnt;
    const int32_t *rl = relw + cr.rl;
    const double *ua = ga + ((int64_t)cr.src + 1) * 32;
    const double *uc = gc + ((int64_t)cr.src + 1) * 32;
    const double la = PIPE_RINV ? wa[p * 32] * da : wa[p * 32] / da;
    const double lc = PIPE_RINV ? wc[p * 32] * dc : wc[p * 32] / dc;
    wa[p * 32] = la;
    wc[p * 32] = lc;
    acA -= la * yja;
    acC -= lc * yjc;
    TR_T(c1)
    TR_ADD(mult, c0, c1)
    for (int q = 0; q < cnt; q += P2W) {
      int t[P2W];
      double xa[P2W], xc[P2W];
#pragma unroll
      for (int k = 0; k < P2W; ++k) {
        const bool ok = q + k < cnt;
        t[k] = ok ? rl[q + k] : 0;
        xa[k] = ok ? __ldcg(ua + (q + k) * 32) : 0.0;
        xc[k] = ok ? __ldcg(uc + (q + k) * 32) : 0.0;
      }
      double va[P2W], vc[P2W];
#pragma unroll
      for (int k = 0; k < P2W; ++k) {
        va[k] = wa[t[k] * 32];
        vc[k] = wc[t[k] * 32];
      }
#pragma unroll
      for (int k = 0; k < P2W; ++k)
        if (q + k < cnt) {
          wa[t[k] * 32] = va[k] - la * xa[k];
          wc[t[k] * 32] = vc[k] - lc * xc[k];
        }
    }
    TR_T(c2)
    TR_ADD(upd, c1, c2)
    cr = nx; da = dna; dc = dnc; yja = yna; yjc = ync;
  }
}

#ifndef RI_W
#define RI_W 8   // matrix entries per load batch of the row initialisation (c4 ms/step: 4: 14.79, 6: 14.79, 8: 14.75)
#endif
// Row initialisation of a pair task: zero the accumulators, scatter the row's
// matrix values (lanes over (instance, entry) pairs, 4 per lane per batch, loads
// before stores) and form b̂_i for both groups.  Needs no dependency: the pipeline
// runs it for the first row before polling the task's dependency flags.
__device__ __forceinline__ void row_init2(const DevSym &S, const BatchP &P, const longlong4 &rr, int W,
                                          double *wA, double *wC, const double *Ab, int nlive, int lane,
                                          int64_t ba, int64_t bc, bool liveA, bool liveC,
                                          const double *rhs, int xmask, double &yA, double &yC,
                                          const double *yiA, const double *yiC) {
  const int64_t e0 = rr.y, a = rr.w;
  const int k = (int)(rr.z >> 32);
  if (P.ypre) {   // b̂ prepared in Y by k_batch_bhat2 (one 256-byte line per row)
    yA = *yiA;
    yC = *yiC;
  } else {
    yA = (liveA && rhs) ? S.dr[a] * rhs[ba * S.n + a] : 0.0;
    yC = (liveC && rhs) ? S.dr[a] * rhs[bc * S.n + a] : 0.0;
  }
  for (int q = 0; q < W; ++q) {
    wA[q * 32 + lane] = 0.0;
    wC[q * 32 + lane] = 0.0;
  }
  __syncwarp();
  // lane = instance: each lane reads its own instance's k contiguous values (the
  // sectors are shared by consecutive entries, so DRAM efficiency matches a
  // transposing scatter) and writes its own column; 4 entries per batch, loads first
  if (!(xmask & 4)) {
    const double *rA = Ab + (int64_t)lane * S.nnz + e0;
    const double *rC = rA + (int64_t)32 * S.nnz;
    for (int e = 0; e < k; e += RI_W) {
      int cp[RI_W];
      double sc[RI_W], va[RI_W], vc[RI_W];
#pragma unroll
      for (int m = 0; m < RI_W; ++m) {
        const bool ok = e + m < k;
        cp[m] = ok ? __ldg(S.colpos + e0 + e + m) : 0;
        sc[m] = ok ? __ldg(S.scale + e0 + e + m) : 0.0;
        va[m] = (ok && liveA) ? __ldg(rA + e + m) : 0.0;
        vc[m] = (ok && liveC) ? __ldg(rC + e + m) : 0.0;
      }
#pragma unroll
      for (int m = 0; m < RI_W; ++m)
        if (e + m < k) {
          wA[cp[m] * 32 + lane] = va[m] * sc[m];
          wC[cp[m] * 32 + lane] = vc[m] * sc[m];
        }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  const unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(d), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned phase) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(a), "r"(phase) : "memory");
}

__device__ __forceinline__ void bt_node2(const DevSym &S, const BatchP &P, const DevProg &R,
                                         const longlong4 nr, int g, const double *rhs, double *Y,
                                         double *wsm0, int ws, int lane, int xmask, longlong4 rr,
                                         bool pre0, double y0A, double y0C,
                                         const StepRec *srec, const int32_t *srel, int64_t sk0,
                                         bool rowstage, uint64_t *mbar, unsigned *phase,
                                         StepRec *srecbuf, int32_t *srelbuf TR_DECL) {
  const int64_t ba = (int64_t)g * 32 + lane, bc = ba + 32;
  const bool liveA = ba < P.B, liveC = bc < P.B;
  const int64_t rem = P.B - (int64_t)g * 32;
  const int nlive = (int)(rem < 64 ? rem : 64);   // live instances of the pair
  const double thr = P.eps * P.anorm[0];
  const int64_t vbase = nr.x;
  const int r = (int)(nr.z & 0xffffffff);
  const int s = (int)(nr.z >> 32);
  const int W = (int)(nr.w & 0xffffffff);
  const int L = (int)(nr.w >> 32);
  double *ga0 = P.BF + (int64_t)g * P.stored * 32;
  double *gc0 = ga0 + P.stored * 32;
  double *ya = Y + (int64_t)g * S.n * 32 + lane;
  double *yc = ya + (int64_t)S.n * 32;
  double *ria = P.RI + (int64_t)g * S.n * 32 + lane;   // P.RI is set whenever PIPE_RINV
  double *ric = ria + (int64_t)S.n * 32;
  const double *Ab = P.A + (int64_t)g * 32 * S.nnz;
  for (int t = 0; t < s; ++t) {
    const int i = r + t;
    const int64_t s0 = rr.x;
    const int64_t s1 = s0 + (rr.z & 0xffffffff);
    const bool inSm = (s1 > s0) && W <= ws;
    double *growA = ga0 + (vbase + (int64_t)t * W) * 32;
    double *growC = gc0 + (vbase + (int64_t)t * W) * 32;
    double *wA = inSm ? wsm0 : growA;
    double *wC = inSm ? wsm0 + ws * 32 : growC;
    double yaccA = y0A, yaccC = y0C;
    // node too large for one program window: stage this row's window (its steps and
    // their target positions) instead, in flight while the row is initialised
    if (rowstage && s1 > s0) {
      const int64_t rl0 = R.row_rel[i], rl1 = R.row_rel[i + 1];
      if (lane == 0) {
        const int64_t a0 = (rl0 * 4) & ~(int64_t)15;
        const int64_t a1 = (rl1 * 4 + 15) & ~(int64_t)15;
        const unsigned brec = (unsigned)(s1 - s0) * 16u, brel = (unsigned)(a1 - a0);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(mbar, brec + brel);
        bulk_g2s(srecbuf, R.st_rec + s0, brec, mbar);
        bulk_g2s(srelbuf, reinterpret_cast<const char *>(R.rel) + a0, brel, mbar);
      }
      srec = srecbuf;
      srel = srelbuf + (int)(rl0 & 3);
      sk0 = s0;
    }
    TR_T(b0)
    if (!(t == 0 && pre0))
      row_init2(S, P, rr, W, wA, wC, Ab, nlive, lane, ba, bc, liveA, liveC, rhs, xmask, yaccA, yaccC,
                ya + (int64_t)i * 32, yc + (int64_t)i * 32);
    TR_T(b1)
    TR_ADD(init, b0, b1)
    if (t + 1 < s) rr = R.row_rec[i + 1];
    if (rowstage && s1 > s0) {
      mbar_wait(mbar, *phase);
      *phase ^= 1u;
    }
    if (!(xmask & 2)) {
      if (srec) {
        if (inSm)
          run_steps2s(srec, srel, (int)(s0 - sk0), (int)(s1 - sk0), wA + lane, wC + lane, ga0 + lane,
                      gc0 + lane, ya, yc, yaccA, yaccC, ria, ric TR_ARG);
        else
          run_steps2s(srec, srel, (int)(s0 - sk0), (int)(s1 - sk0), growA + lane, growC + lane, ga0 + lane,
                      gc0 + lane, ya, yc, yaccA, yaccC, ria, ric TR_ARG);
      } else if (inSm)
        run_steps2(R, s0, s1, wA + lane, wC + lane, ga0 + lane, gc0 + lane, ya, yc, yaccA, yaccC, ria, ric);
      else
        run_steps2(R, s0, s1, growA + lane, growC + lane, ga0 + lane, gc0 + lane, ya, yc, yaccA, yaccC, ria,
                   ric);
    }
    TR_T(b2)
    const int Lt = L + t;
    bool fa, fc;
    wA[Lt * 32 + lane] = perturb(wA[Lt * 32 + lane], thr, fa);
    wC[Lt * 32 + lane] = perturb(wC[Lt * 32 + lane], thr, fc);
    if (fa && liveA) atomicAdd(&P.npert[ba], 1);
    if (fc && liveC) atomicAdd(&P.npert[bc], 1);
    ya[(int64_t)i * 32] = yaccA;
    yc[(int64_t)i * 32] = yaccC;
    if (PIPE_RINV) {   // one division per row, off the consumers' step chains
      ria[(int64_t)i * 32] = 1.0 / wA[Lt * 32 + lane];
      ric[(int64_t)i * 32] = 1.0 / wC[Lt * 32 + lane];
    }
    if (inSm && !(xmask & 8))
      for (int q = 0; q < W; ++q) {
        growA[q * 32 + lane] = wA[q * 32 + lane];
        growC[q * 32 + lane] = wC[q * 32 + lane];
      }
    __syncwarp();
    TR_T(b3)
    TR_ADD(fin, b2, b3)
  }
}

// Pair-mode pipeline: task records carry the even group g of the pair; the warp
// waits for both groups' dependency flags and publishes both.
#ifndef PIPE_MINB_DEF
#define PIPE_MINB_DEF 4
#endif
#ifndef PIPE_REL
#define PIPE_REL 1   // producer fence: 1 fence.release (MEMBAR only), 0 fence.acq_rel (MEMBAR + L1 invalidation)
#endif
#ifndef PIPE_ACQ
#define PIPE_ACQ 2   // consumer acquire: 2 (default) one ld.acquire per observed flag after the relaxed spin, 1 one fence after the polls (+0.25 ms/step), 0 none (formally racy)
#endif
// Per-warp staging area after the 4 warps' accumulators: an mbarrier, the task's
// step records and its rel window (bulk copies issued at claim, before the polls).
constexpr int PIPE_STAGE = 16 + PIPE_REC_CAP * 16 + PIPE_REL_CAP * 4;
size_t pipe_smem(int ws) { return (size_t)PIPE_WARPS * (2 * ws * 32 * 8 + PIPE_STAGE); }

#ifdef HYLU_TRACE
// Debug build only (-DHYLU_TRACE, scripts/pipe_trace.py): per task {claim, ready, end}
// global timestamps and (node, group, SM id), written through hy_debug_pipe_trace's buffer.
__device__ unsigned long long *g_pipe_trace = nullptr;
__device__ unsigned long long *g_hub_trace = nullptr;   // [0] record counter, then 8 words per hub CTA
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned s;
  asm volatile("mov.u32 %0, %smid;" : "=r"(s));
  return s;
}
#endif

__global__ void __launch_bounds__(PIPE_WARPS * 32, PIPE_MINB_DEF)
    k_bt_pipe2(DevSym S, BatchP P, DevProg R, const TaskDesc *tasks, int64_t total, const double *rhs,
               double *Y, int *counter, int *flags, int epoch, int G, int ws) {
  extern __shared__ __align__(16) double pipe_smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double *wsm_w = pipe_smem + (size_t)warp * 2 * ws * 32;
  unsigned char *stg = reinterpret_cast<unsigned char *>(pipe_smem + (size_t)PIPE_WARPS * 2 * ws * 32) +
                       (size_t)warp * PIPE_STAGE;
  uint64_t *mbar = reinterpret_cast<uint64_t *>(stg);
  StepRec *srec = reinterpret_cast<StepRec *>(stg + 16);
  int32_t *srel = reinterpret_cast<int32_t *>(stg + 16 + PIPE_REC_CAP * 16);
  unsigned phase = 0;
  if (R.st_rec && lane == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  for (;;) {
    long long t = 0;
    if (lane == 0) t = (long long)atomicAdd(reinterpret_cast<unsigned long long *>(counter), 1ull);
    t = __shfl_sync(HY_FULL, t, 0);
    if (t >= total) return;
    const TaskDesc cur = tasks[t];
#ifdef HYLU_TRACE
    unsigned long long *tr = (g_pipe_trace && total > 1000) ? g_pipe_trace + 12 * t : nullptr;
    TraceAcc tacc{0, 0, 0, 0};
    const long long k0c = clock64();
    if (tr && lane == 0) {
      tr[0] = gtime();
      tr[3] = ((unsigned long long)cur.u << 32) | ((unsigned long long)cur.g << 16) | smid();
    }
#endif
    const int two = cur.g + 1 < G ? 2 : 1;
    const int64_t nd = cur.d1 - cur.d0;
    // the task's program window into shared memory, in flight while the polls wait
    const bool staged = R.st_rec != nullptr && cur.nk > 0;
    const bool rowstage = R.st_rec != nullptr && cur.nk == 0 && cur.nrel < 0;   // per-row windows
    int roff = 0;
    if (staged && lane == 0) {
      const int64_t a0 = (cur.rel0 * 4) & ~(int64_t)15;
      const int64_t a1 = ((cur.rel0 + cur.nrel) * 4 + 15) & ~(int64_t)15;
      const unsigned brec = (unsigned)cur.nk * 16u, brel = (unsigned)(a1 - a0);
      // the previous task's generic reads of the buffers precede the async writes
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_expect_tx(mbar, brec + brel);
      bulk_g2s(srec, R.st_rec + cur.k0, brec, mbar);
      bulk_g2s(srel, reinterpret_cast<const char *>(R.rel) + a0, brel, mbar);
    }
    if (staged) roff = (int)(cur.rel0 & 3);
    // relaxed polls (an acquire load would invalidate the SM's L1 on every poll);
    // every value a task reads from another task is loaded L2-coherent (ld.cg)
    // after the polls, and producers fence before publishing
    for (int64_t k = lane; k < nd * two; k += 32) {
      const int64_t kk = k < nd ? k : k - nd;
      const int dn = kk == 0 ? cur.dep[0] : kk == 1 ? cur.dep[1] : kk == 2 ? cur.dep[2] :
                     kk == 3 ? cur.dep[3] : __ldg(S.deps + cur.d0 + kk);
      const int *f = flags + (int64_t)dn * G + cur.g + (k < nd ? 0 : 1);
      while (ld_relaxed(f) != epoch) __nanosleep(64);
#if PIPE_ACQ == 2
      (void)ld_acquire(f);
#endif
    }
    // acquire side of the flag protocol: one fence after the observed flags (not one
    // per spin) pairs with the producer's fence + relaxed store (PTX fence-based
    // synchronization); __syncwarp then orders the other lanes after this lane
#if PIPE_ACQ == 1
    fence_acq_rel_gpu();
#elif PIPE_ACQ == 3
    if (nd > 0) fence_acquire_gpu();
#endif
    __syncwarp();
    if (staged) {
      mbar_wait(mbar, phase);
      phase ^= 1u;
    }
#ifdef HYLU_TRACE
    const long long k1c = clock64();
    if (tr && lane == 0) tr[1] = gtime();
#endif
    const longlong4 nr = make_longlong4(cur.valoff, cur.d0, (int64_t)cur.r | ((int64_t)cur.s << 32),
                                        (int64_t)cur.W | ((int64_t)cur.L << 32));
    bt_node2(S, P, R, nr, cur.g, rhs, Y, wsm_w, ws, lane, 0, cur.rr0, false, 0.0, 0.0,
             staged ? srec : nullptr, srel + roff, cur.k0, rowstage, mbar, &phase, srec, srel TR_ARG);
#ifdef HYLU_TRACE
    const long long k2c = clock64();
#endif
#if PIPE_REL == 1
    fence_release_gpu();
#else
    fence_acq_rel_gpu();
#endif
    __syncwarp();
#ifdef HYLU_TRACE
    if (tr && lane == 0) {
      tr[2] = gtime();
      tr[4] = tacc.init; tr[5] = tacc.mult; tr[6] = tacc.upd; tr[7] = tacc.fin;
      tr[8] = k1c - k0c; tr[9] = k2c - k1c; tr[10] = clock64() - k2c; tr[11] = 0;
    }
#endif
    if (lane < two) st_relaxed(flags + (int64_t)cur.u * G + cur.g + lane, epoch);
  }
}

#ifdef HYLU_TRACE
extern "C" int hy_debug_pipe_trace(unsigned long long *d_buf) {
  return (int)cudaMemcpyToSymbol(g_pipe_trace, &d_buf, sizeof(d_buf));
}
extern "C" int hy_debug_hub_trace(unsigned long long *d_buf) {
  return (int)cudaMemcpyToSymbol(g_hub_trace, &d_buf, sizeof(d_buf));
}
#endif

// ---------------------------------------------------------------------------
// Hub kernel: one CTA per (hub node, group).  Pull programs: the positions of a row
// are processed level by level (intra-row dependency levels); a position gathers
// its contributions (ascending step order) in work items of <= 64 terms; positions
// with more terms are split and their partial sums combined in slot order, so the
// result is deterministic.  Forward substitution is fused (fixed-order reduction).
__device__ __forceinline__ void hub_finalize(const BatchP &P, int64_t kd, int p, double acc,
                                             double *w, const double *gb, double thr, bool live,
                                             int64_t b) {
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

__global__ void __launch_bounds__(HUB_THREADS, 1) k_bt_hub(DevSym S, BatchP P, DevProg R,
                                                        const int32_t *nodes, int count, int G,
                                                        const double *rhs, double *Y,
                                                        double *scratch, int max_slots, int *flags,
                                                        int epoch) {
  __shared__ double red[HUB_THREADS / 32][32];
  constexpr int LVCAP = 512;
  __shared__ int64_t s_wi[LVCAP + 1], s_sp[LVCAP + 1], s_y[LVCAP + 1];
  __shared__ int s_bt[LVCAP + 1];
  __shared__ int s_next[2];   // next unclaimed work item of the current / the next level
  // per-level staging of work-item metadata and predecessor lists, double-buffered:
  // level l+1's records are copied (cp.async) while level l is processed
  extern __shared__ __align__(16) unsigned char hub_dyn[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = HUB_THREADS / 32;
  const int task = blockIdx.x;
  const int u = nodes[task / G];
  const int g = task % G;
  const int64_t b = (int64_t)g * 32 + lane;
  const bool live = b < P.B;
  const double thr = P.eps * P.anorm[0];
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int W = (int)(S.colptr[u + 1] - S.colptr[u]);
  double *gb0 = P.BF + (int64_t)g * P.stored * 32;
  const double *gb = gb0 + lane;
  double *yb = Y + (int64_t)g * S.n * 32 + lane;
  const double *Ab = P.A + (int64_t)g * 32 * S.nnz;
  double *scr = scratch + (size_t)blockIdx.x * max_slots * 32 + lane;
  const int hr0 = R.hub_base[u];
#ifdef HYLU_TRACE
  const long long h0 = clock64();
  long long hlev = 0, hfwd = 0;
#endif
  // initialise every row of the node first: a (joint) node program may span rows
  for (int t = 0; t < s; ++t) {
    const int i = r + t;
    double *w0 = gb0 + (S.valoff[u] + (int64_t)t * W) * 32;
    for (int q = threadIdx.x; q < W * 16; q += HUB_THREADS)   // 16-byte stores (rows are 256-byte aligned)
      reinterpret_cast<double2 *>(w0)[q] = make_double2(0.0, 0.0);
    __syncthreads();
    const int srow = S.kind[u] ? r + P.iperm[i] : r;
    const int64_t a = S.mrow_src[srow];
    const int64_t e0 = S.a_ptr[a];
    const int k = (int)(S.a_ptr[a + 1] - e0);
    // lane = instance, warps stride the entries: coalesced 256-byte stores
    // (4 consecutive entries per warp and iteration, loads before stores: one round trip
    // per 4 entries, and a lane's 4 values share one 32-byte sector)
    if (live)
      for (int e = warp * 4; e < k; e += nw * 4) {
        int cp[4];
        double v[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) {
          const bool ok = e + m < k;
          cp[m] = ok ? __ldg(S.colpos + e0 + e + m) : 0;
          v[m] = ok ? __ldg(Ab + (int64_t)lane * S.nnz + e0 + e + m) * __ldg(S.scale + e0 + e + m) : 0.0;
        }
#pragma unroll
        for (int m = 0; m < 4; ++m)
          if (e + m < k) w0[cp[m] * 32 + lane] = v[m];
      }
  }
  __syncthreads();
#ifdef HYLU_TRACE
  const long long h1 = clock64();
#endif
  for (int t = 0; t < s; ++t) {
    const int i = r + t;
#ifdef HYLU_TRACE
    const long long r0c = clock64();
#endif
    // positions are node-relative (t*W + p): every row's levels address the node base
    double *w = gb0 + S.valoff[u] * 32 + lane;
    double *w0 = gb0 + (S.valoff[u] + (int64_t)t * W) * 32;
    const int srow = S.kind[u] ? r + P.iperm[i] : r;
    const int64_t a = S.mrow_src[srow];
    const int hr = hr0 + t;
    const int64_t lv0 = R.hrow_lev[hr], lv1 = R.hrow_lev[hr + 1];
    // stage this row's level bounds and per-level predecessor offsets (the
    // predecessor records of consecutive levels are contiguous)
    const int nlv = (int)(lv1 - lv0);
    const bool lsm = nlv <= LVCAP;
    if (lsm) {
      for (int q = threadIdx.x; q <= nlv; q += HUB_THREADS) {
        s_wi[q] = R.lev_wi[lv0 + q];
        s_sp[q] = R.lev_sp[lv0 + q];
      }
      __syncthreads();
      const int64_t wlast = s_wi[nlv];
      for (int q = threadIdx.x; q <= nlv; q += HUB_THREADS)
        s_y[q] = s_wi[q] < wlast ? R.wi_y0[s_wi[q]] : (wlast > s_wi[0] ? R.wi_y1[wlast - 1] : 0);
    }
    __syncthreads();
    auto buf = [&](int k, int64_t *&pu, int64_t *&kd, int64_t *&y0, int64_t *&y1, int32_t *&pp,
                   int32_t *&pq, int32_t *&sl) {
      unsigned char *bb = hub_dyn + (size_t)k * HUB_BUF;
      pu = reinterpret_cast<int64_t *>(bb);
      kd = pu + HUB_CAPP;
      y0 = kd + HUB_CAPI;
      y1 = y0 + HUB_CAPI;
      pp = reinterpret_cast<int32_t *>(y1 + HUB_CAPI);
      pq = pp + HUB_CAPP;
      sl = pq + HUB_CAPI;
    };
    auto stageable = [&](int q) {
      return lsm && s_wi[q + 1] - s_wi[q] <= HUB_CAPI && s_y[q + 1] - s_y[q] <= HUB_CAPP;
    };
    auto issue = [&](int q) {   // cp.async level lv0+q's records into buffer q&1
      int64_t *pu, *kd, *y0, *y1;
      int32_t *pp, *pq, *sl;
      buf(q & 1, pu, kd, y0, y1, pp, pq, sl);
      const int64_t wi0 = s_wi[q], ni = s_wi[q + 1] - wi0;
      const int64_t yb0 = s_y[q], np_ = s_y[q + 1] - yb0;
      for (int64_t k2 = threadIdx.x; k2 < ni; k2 += HUB_THREADS) {
        cp_async4(pq + k2, R.wi_p + wi0 + k2);
        cp_async4(sl + k2, R.wi_slot + wi0 + k2);
        cp_async8(reinterpret_cast<double *>(y0 + k2), reinterpret_cast<const double *>(R.wi_y0 + wi0 + k2));
        cp_async8(reinterpret_cast<double *>(y1 + k2), reinterpret_cast<const double *>(R.wi_y1 + wi0 + k2));
        cp_async8(reinterpret_cast<double *>(kd + k2), reinterpret_cast<const double *>(R.wi_kd + wi0 + k2));
      }
      for (int64_t k2 = threadIdx.x; k2 < np_; k2 += HUB_THREADS) {
        cp_async4(pp + k2, R.pred_p + yb0 + k2);
        cp_async8(reinterpret_cast<double *>(pu + k2), reinterpret_cast<const double *>(R.pred_u + yb0 + k2));
      }
    };
    // One barrier per level: level q+1's records are issued at the top of level q and
    // awaited just before the barrier that ends level q, which so also publishes them
    // (the claim counters alternate, so the next level's is reset a level ahead).
    if (nlv > 0 && stageable(0)) issue(0);
    cp_async_wait_all();
    if (threadIdx.x == 0) s_next[0] = 0;
    __syncthreads();
    for (int64_t lev = lv0; lev < lv1; ++lev) {
      const int q = (int)(lev - lv0);
      if (lev + 1 < lv1 && stageable(q + 1)) issue(q + 1);
      cp_async_commit();
      if (threadIdx.x == 0) s_next[(q + 1) & 1] = 0;
      int *const nxt = &s_next[q & 1];
      const int64_t wi0 = lsm ? s_wi[q] : R.lev_wi[lev];
      const int64_t wi1 = lsm ? s_wi[q + 1] : R.lev_wi[lev + 1];
      const int64_t sp0 = lsm ? s_sp[q] : R.lev_sp[lev];
      const int64_t sp1 = lsm ? s_sp[q + 1] : R.lev_sp[lev + 1];
      const int64_t ni = wi1 - wi0;
      if (stageable(q)) {
        int64_t *st_pu, *st_kd, *st_y0, *st_y1;
        int32_t *st_pp, *st_p, *st_sl;
        buf(q & 1, st_pu, st_kd, st_y0, st_y1, st_pp, st_p, st_sl);
        const int64_t yb0 = s_y[q];
        // HUB_I items per warp at a time, HUB_P predecessors per item per round:
        // HUB_I x HUB_P x 2 independent gathers in flight per warp
        // warps claim the level's items one by one (the host lists them longest first)
        for (;;) {
          int64_t q0 = 0;
          if (lane == 0) q0 = atomicAdd(nxt, HUB_I);
          q0 = __shfl_sync(HY_FULL, q0, 0);
          if (q0 >= ni) break;
          int p[HUB_I], y[HUB_I], y1[HUB_I], slot[HUB_I];
          int64_t kd[HUB_I];
          double acc[HUB_I], dv[HUB_I];
#pragma unroll
          for (int jq = 0; jq < HUB_I; ++jq) {
            const int64_t qq = q0 + jq;
            const bool ok = qq < ni;
            p[jq] = ok ? st_p[qq] : 0;
            slot[jq] = ok ? st_sl[qq] : 0;
            y[jq] = ok ? (int)(st_y0[qq] - yb0) : 0;
            y1[jq] = ok ? (int)(st_y1[qq] - yb0) : 0;
            kd[jq] = ok ? st_kd[qq] : -1;
            dv[jq] = kd[jq] >= 0 ? gb[kd[jq] * 32] : 1.0;
            acc[jq] = (ok && slot[jq] < 0) ? w[p[jq] * 32] : 0.0;
          }
          int rem = 0;
#pragma unroll
          for (int jq = 0; jq < HUB_I; ++jq) rem = max(rem, y1[jq] - y[jq]);
          for (int step = 0; step < rem; step += HUB_P) {
            double lv[HUB_I][HUB_P], uv[HUB_I][HUB_P];
#pragma unroll
            for (int jq = 0; jq < HUB_I; ++jq)
#pragma unroll
              for (int e = 0; e < HUB_P; ++e) {
                const int yy = y[jq] + step + e;
                const bool act = yy < y1[jq];
                lv[jq][e] = act ? w[st_pp[yy] * 32] : 0.0;
                uv[jq][e] = act ? gb[st_pu[yy] * 32] : 0.0;
              }
#pragma unroll
            for (int jq = 0; jq < HUB_I; ++jq)
#pragma unroll
              for (int e = 0; e < HUB_P; ++e) acc[jq] -= lv[jq][e] * uv[jq][e];
          }
#pragma unroll
          for (int jq = 0; jq < HUB_I; ++jq) {
            const int64_t qq = q0 + jq;
            if (qq >= ni) continue;
            double a = acc[jq];
            if (slot[jq] < 0) {
              if (kd[jq] >= 0) {
                a = a / dv[jq];
              } else if (kd[jq] == -2) {
                bool fired;
                const double piv = a;
                a = perturb(piv, thr, fired);
                if (fired && live) atomicAdd(&P.npert[b], 1);
              }
              w[p[jq] * 32] = a;
            } else {
              scr[(size_t)slot[jq] * 32] = a;
            }
          }
        }
      } else
      for (int64_t it = wi0 + warp; it < wi1; it += nw) {
        const int p = R.wi_p[it];
        const int slot = R.wi_slot[it];
        const int64_t y1 = R.wi_y1[it];
        int64_t y = R.wi_y0[it];
        double acc = slot < 0 ? w[p * 32] : 0.0;
        for (; y + 8 <= y1; y += 8) {
          int pp[8];
          int64_t pu[8];
          double lv[8], uv[8];
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) {
            pp[k2] = R.pred_p[y + k2];
            pu[k2] = R.pred_u[y + k2];
          }
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) {
            lv[k2] = w[pp[k2] * 32];
            uv[k2] = gb[pu[k2] * 32];
          }
#pragma unroll
          for (int k2 = 0; k2 < 8; ++k2) acc -= lv[k2] * uv[k2];
        }
        for (; y < y1; ++y) acc -= w[R.pred_p[y] * 32] * gb[R.pred_u[y] * 32];
        if (slot < 0)
          hub_finalize(P, R.wi_kd[it], p, acc, w, gb, thr, live, b);
        else
          scr[(size_t)slot * 32] = acc;
      }
      if (sp1 > sp0) {
        __syncthreads();
        for (int64_t k2 = sp0 + warp; k2 < sp1; k2 += nw) {
          const int p = R.sp_p[k2];
          double acc = w[p * 32];
          const int s0 = R.sp_s0[k2], ns = R.sp_n[k2];
          for (int c = 0; c < ns; ++c) acc += scr[(size_t)(s0 + c) * 32];
          hub_finalize(P, R.sp_kd[k2], p, acc, w, gb, thr, live, b);
        }
      }
      cp_async_wait_all0();
      __syncthreads();
    }
#ifdef HYLU_TRACE
    const long long r1c = clock64();
    hlev += r1c - r0c;
#endif
    // forward substitution for row i: y_i = b̂_i − Σ_s l_s y_{j_s}
    double part = 0.0;
    for (int64_t st = R.row_ptr[i] + warp; st < R.row_ptr[i + 1]; st += nw)
      part += w0[R.st_p[st] * 32 + lane] * yb[(int64_t)R.st_j[st] * 32];
    red[warp][lane] = part;
    __syncthreads();
    if (warp == 0) {
      double yacc = P.ypre ? yb[(int64_t)i * 32] : (live && rhs) ? S.dr[a] * rhs[b * S.n + a] : 0.0;
      for (int k2 = 0; k2 < nw; ++k2) yacc -= red[k2][lane];
      yb[(int64_t)i * 32] = yacc;
      if (PIPE_RINV) P.RI[((int64_t)g * S.n + i) * 32 + lane] = 1.0 / w0[(int64_t)(S.nl[u] + t) * 32 + lane];
    }
    __syncthreads();
#ifdef HYLU_TRACE
    hfwd += clock64() - r1c;
#endif
  }
#ifdef HYLU_TRACE
  if (g_hub_trace && threadIdx.x == 0) {
    const unsigned long long k = atomicAdd(g_hub_trace, 1ull);
    unsigned long long *q = g_hub_trace + 1 + 8 * k;
    q[0] = u; q[1] = g; q[2] = clock64() - h0; q[3] = h1 - h0; q[4] = hlev; q[5] = hfwd; q[6] = gtime(); q[7] = smid();
  }
#endif
  if (flags && threadIdx.x == 0) {
    __threadfence();
    st_release(flags + (int64_t)u * G + g, epoch);
  }
}

// Factor row of every original row (the inverse of row i -> source row a, with the
// prior inner_perm applied inside supernodes).
__global__ void k_row_of(DevSym S, const int32_t *iperm, int32_t *rowof) {
  for (int row = blockIdx.x * blockDim.x + threadIdx.x; row < S.n; row += gridDim.x * blockDim.x) {
    const int u = S.node_of[row];
    int src = row;
    if (S.kind[u] == 1) src = (int)S.first[u] + iperm[row];
    rowof[S.mrow_src[src]] = row;
  }
}

// rhs [B][n] -> b̂ interleaved [G][n][32] in source-row order: a tile of 32
// consecutive original rows reads 256 contiguous bytes per instance and writes one
// full 256-byte line per row (b̂_i = dr[a] b[a], i = rowof[a]).
__global__ void k_batch_bhat2(DevSym S, const int32_t *rowof, const double *rhs, double *Y, int64_t B) {
  __shared__ double tile[32][33];
  const int g = blockIdx.y;
  const int a0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  for (int ii = wy; ii < 32; ii += 8) {
    const int64_t b = (int64_t)g * 32 + ii;
    const int a = a0 + lane;
    tile[ii][lane] = (a < S.n && b < B) ? S.dr[a] * rhs[b * S.n + a] : 0.0;
  }
  __syncthreads();
  for (int aa = wy; aa < 32; aa += 8) {
    const int a = a0 + aa;
    if (a < S.n) Y[((int64_t)g * S.n + rowof[a]) * 32 + lane] = tile[lane][aa];
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

// interleaved z [G][n][32] -> x [B][n] in output order: a tile of 32 consecutive
// output columns c reads the 32 lines z[pinv[c]] (one 256-byte line each, lane =
// instance) and writes 32 contiguous values per instance row.
__global__ void k_batch_xout2(DevSym S, const int32_t *pinv, const double *Y, double *X, int64_t B) {
  __shared__ double tile[32][33];
  const int g = blockIdx.y;
  const int c0 = blockIdx.x * 32;
  const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
  for (int cc = wy; cc < 32; cc += 8) {
    const int c = c0 + cc;
    tile[cc][lane] = c < S.n ? S.dc[c] * Y[((int64_t)g * S.n + pinv[c]) * 32 + lane] : 0.0;
  }
  __syncthreads();
  for (int ii = wy; ii < 32; ii += 8) {
    const int64_t b = (int64_t)g * 32 + ii;
    const int c = c0 + lane;
    if (c < S.n && b < B) X[b * S.n + c] = tile[lane][ii];
  }
}

__global__ void k_perm_inverse(int n, const int64_t *perm, int32_t *pinv) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
    pinv[perm[k]] = k;
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

// Pair mode backward substitution: one warp per (node, group pair); the padded
// allocation makes the odd tail group's partner valid memory (never copied out).
#ifndef BWD_MINB
#define BWD_MINB 10   // 48 registers for the 2-entry form: more resident warps on the wide (throughput-bound) levels (c4 14.45 -> 14.19 ms; 12: 14.30, 16: 14.41; re-swept at the end: 8: 14.68, 9: 14.16, 10: 14.14-14.17, 11: 14.26)
#endif
template <int BWDW>
__global__ void __launch_bounds__(BW * 32, BWDW <= 2 ? BWD_MINB : 1) k_batch_bwd2(DevSym S, const double *BF, int64_t stored,
                                                        const int32_t *nodes, int count, int GP,
                                                        double *Y) {
  pdl_wait();
  pdl_launch_dependents();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t task = (int64_t)blockIdx.x * BW + warp;
  if (task >= (int64_t)count * GP) return;
  const int u = nodes[task / GP];
  const int g = 2 * (int)(task % GP);
  const int r = (int)S.first[u];
  const int s = (int)(S.first[u + 1] - r);
  const int64_t c0 = S.colptr[u];
  const int W = (int)(S.colptr[u + 1] - c0);
  const int L = S.nl[u];
  const double *ga = BF + (int64_t)g * stored * 32 + lane;
  const double *gc = ga + stored * 32;
  double *ya = Y + (int64_t)g * S.n * 32 + lane;
  double *yc = ya + (int64_t)S.n * 32;
  const int32_t *cc = S.cols + c0;
  for (int t = s - 1; t >= 0; --t) {
    const int64_t ro = (S.valoff[u] + (int64_t)t * W) * 32;
    const int d = L + t;
    double accA = ya[(int64_t)(r + t) * 32], accC = yc[(int64_t)(r + t) * 32];
    const double dA = ga[ro + (int64_t)d * 32], dC = gc[ro + (int64_t)d * 32];
    for (int p0 = d + 1; p0 < W; p0 += BWDW) {
      int k[BWDW];
      double a[BWDW], c[BWDW], za[BWDW], zc[BWDW];
#pragma unroll
      for (int e = 0; e < BWDW; ++e) k[e] = p0 + e < W ? __ldg(cc + p0 + e) : -1;
#pragma unroll
      for (int e = 0; e < BWDW; ++e) {
        const bool ok = k[e] >= 0;
        a[e] = ok ? ga[ro + (int64_t)(p0 + e) * 32] : 0.0;
        c[e] = ok ? gc[ro + (int64_t)(p0 + e) * 32] : 0.0;
        za[e] = ok ? ya[(int64_t)k[e] * 32] : 0.0;
        zc[e] = ok ? yc[(int64_t)k[e] * 32] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < BWDW; ++e) {
        accA -= a[e] * za[e];
        accC -= c[e] * zc[e];
      }
    }
    ya[(int64_t)(r + t) * 32] = accA / dA;
    yc[(int64_t)(r + t) * 32] = accC / dC;
  }
}

// entries per batch: BWD_W (2) for the wide levels (throughput-bound, occupancy matters) and
// BWD_WL for the narrow top levels, where a row's batches are a dependent chain of round trips
template __global__ void k_batch_bwd2<BWD_W>(DevSym, const double *, int64_t, const int32_t *, int, int, double *);
template __global__ void k_batch_bwd2<BWD_WL>(DevSym, const double *, int64_t, const int32_t *, int, int, double *);

// de-interleave one instance's factor values into node layout
__global__ void k_batch_extract(const double *BF, int64_t stored, int64_t b, double *out) {
  const int64_t g = b / 32, lane = b % 32;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < stored;
       p += (int64_t)gridDim.x * blockDim.x)
    out[p] = BF[(g * stored + p) * 32 + lane];
}

}  // namespace hy
