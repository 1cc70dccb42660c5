// hylu_common.cuh — shared device structures and helpers for the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define HY_FULL 0xffffffffu

// Programmatic dependent launch (PDL): a kernel launched with programmatic stream
// serialization may start while its predecessor runs; it waits here until the
// predecessor grid has completed (and its writes are visible), then lets its own
// successor start launching.  Both are no-ops for a normally launched kernel.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

namespace hy {

// Symbolic structure resident on the device (uploaded once by hy_upload_symbolic).
struct DevSym {
  int32_t n, nn, mode;
  int64_t nnz;
  const int64_t *first;     // [nn+1]
  const int8_t *kind;       // [nn]
  const int64_t *colptr;    // [nn+1]
  const int32_t *cols;      // [colptr[nn]]
  const int32_t *nl;        // [nn]
  const int64_t *valoff;    // [nn+1]
  const int64_t *dptr;      // [nn+1]
  const int32_t *deps;
  const int32_t *node_of;   // [n]
  const int64_t *a_ptr;     // [n+1]
  const int64_t *mrow_src;  // [n]
  const int32_t *colpos;    // [nnz]
  const double *scale;      // [nnz]
  const double *dr, *dc;    // [n]
  const int64_t *perm;      // [n]
};

// Fan-in update item (target node, 64-column tile) in one 32-byte record, built on
// the device at plan upload (k_item_rec): the update kernels get everything their
// prologue needs from one load instead of two dependent rounds (item -> node).
// Multiplier-block (X) item of the level fan-in, packed once per plan upload (k_x_rec): what
// k_fi_x / k_fi_x_w otherwise chase through four dependent metadata rounds per item.
struct __align__(16) XRec {
  int64_t t_off;   // target block: valoff[T] + pb0 (first panel column of the source in T)
  int64_t u_off;   // source triangle: valoff[v] + tb0 * vW + nl[v] + tb0 (row/column tb0 of v's block)
  int32_t W, vW;   // row widths of target and source
  int16_t s, m;    // target rows, source block rows from the first present one
  int32_t pad;
};

// LU / panel item of the level fan-in, packed once per plan upload (k_node_rec): the node's
// layout (and the panel tile's columns) in one 32-byte load instead of a dependent round.
struct __align__(16) NodeItemRec {
  int64_t valoff;
  int32_t r, s, W, L;
  int32_t c0, c1;   // panel tile columns (LU items: unused)
};

// Node of a substitution level, packed once per symbolic upload (k_solve_rec): layout,
// column list and partial-sum slots in one record instead of a dependent metadata round.
struct __align__(16) SolveRec {
  int64_t valoff, col0;   // factor values / first entry of the node's column list
  int32_t r, s, W, L;
  int32_t slot0, nslot;   // partial sums of the level's chunk kernel
  int32_t pad[2];
};

struct __align__(16) ItemRec {
  int64_t valoff;   // target node's value offset
  int64_t zb;       // first source record
  int32_t nz;       // source records
  int32_t W;        // target width (row pitch)
  int32_t c0;       // tile columns [c0, c0 + tw) of the target's column list
  int16_t s;        // target rows (<= 64)
  int16_t tw;       // tile width (<= 64)
};

// Per-call parameters (single-instance path).
struct CallP {
  double *F;                 // factor values (node layout)
  const double *A;           // A values [nnz]
  int32_t *iperm;            // inner_perm [n] (written on factorize, read on refactorize)
  const int32_t *iperm_prior;
  const double *anorm;       // [1]
  const double *anorm_prior; // [1] (refactorize: copied into anorm by k_call_prep)
  double eps;
  int refactor;
  int32_t *status;           // [4]
  int64_t *pert_rows;
  double *pert_vals;
  int64_t pert_cap;
  int chain;                 // 1: row-row operation order (ROWROW tier): each source row's
                             // update subtracted from the running target value
};

// Per-call parameters (batched path).
struct BatchP {
  double *BF;            // interleaved factor workspace [G][stored][32]
  const double *A;       // [B][nnz]
  const int32_t *iperm;  // prior inner_perm [n]
  const double *anorm;   // prior anorm [1] (device)
  double eps;
  int32_t *npert;        // [B]
  int64_t B;
  int64_t stored;
  int ypre;              // 1: Y already holds b̂ (interleaved, factor-row order)
  double *RI;            // [G][n][32] reciprocal of each finished row's pivot (nullptr: divide)
};

// Row programs (schedule.py) resident on the device.
// One step of a batched row program in 16 bytes (the SoA arrays below, packed): the
// pipeline copies a task's steps into shared memory with one bulk copy.
struct __align__(16) StepRec {
  int32_t p;      // multiplier position in the target row
  int32_t src;    // offset of U(j,j) in node storage
  int32_t j;      // source row (forward-solve coupling)
  int16_t cnt;    // U(j,>j) entries
  int16_t rl;     // offset of the step's target positions in the task's rel window
};

// Batched backward solve (k_batch_bwd2): entries per load batch on wide levels (throughput-bound:
// 2-8 measured, 2 best) and on narrow levels, where a row's batches are a dependent chain
#ifndef BWD_W
#define BWD_W 2
#endif
#ifndef BWD_WL
#define BWD_WL 8
#endif
#ifndef BWD_NARROW
#define BWD_NARROW 4096   // (node, group pair) tasks per level up to which BWD_WL is used
#endif

#ifndef PIPE_REC_CAP
#define PIPE_REC_CAP 160   // steps of a task's program window staged in shared memory
#endif
#ifndef PIPE_REL_CAP
#define PIPE_REL_CAP 1024  // rel entries of the window (+ 16-byte alignment slack)
#endif

// Batched pipeline task (node, group pair), built on the host in claim order.
struct TaskDesc {
  int32_t u, g;
  int64_t valoff;
  int32_t r, s, W, L;
  int64_t d0, d1;
  longlong4 rr0;   // row record of the node's first row (no dependent load for it)
  int32_t dep[4];  // the first (up to) 4 dependencies, inline (no dependent index load)
  int64_t rel0;    // first rel entry of the node's program window
  int32_t k0, nk;  // the node's steps [k0, k0 + nk)
  int32_t nrel;    // rel entries of the window (0: not stageable; -1 with nk == 0: staged row by row)
  int32_t pad[3];
};

struct DevProg {
  const StepRec *st_rec;    // [nsteps (+1 pad)] packed steps (nullptr: not built)
  const int64_t *row_ptr;   // [n+1]
  const int32_t *st_p;
  const int32_t *st_j;
  const int64_t *st_src;
  const int32_t *st_cnt;
  const int64_t *st_rel;
  const int32_t *rel;
  const int64_t *row_rel;   // [n+1] first rel entry of each row's steps (per-row program windows)
  const int32_t *hub_base;  // [nn] first hub-row index of a hub node, -1 otherwise
  const int64_t *hrow_lev;
  const int64_t *lev_ptr;
  const int32_t *hpos;
  const int64_t *hdiv;
  const int64_t *hpp;
  const int32_t *pred_p;
  const int64_t *pred_u;
  const int64_t *lev_wi;    // work items per intra-row level
  const int32_t *wi_p;
  const int64_t *wi_kd;
  const int64_t *wi_y0;
  const int64_t *wi_y1;
  const int32_t *wi_slot;
  const int64_t *lev_sp;    // split positions per intra-row level
  const int32_t *sp_p;
  const int64_t *sp_kd;
  const longlong4 *node_rec;  // [nn]: valoff, dep0, first|rows<<32, W|L<<32
  const longlong4 *row_rec;   // [n]: step0, a_e0, nsteps|k<<32, a
  const int32_t *sp_s0;
  const int32_t *sp_n;
};

__device__ __forceinline__ int lower_bound_i32(const int32_t *c, int lo, int hi, int key) {
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (c[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// pivot_perturb: |p| < thr -> sign(p)*thr (sign(0) = +).
__device__ __forceinline__ double perturb(double p, double thr, bool &fired) {
  fired = fabs(p) < thr;
  if (fired) return p < 0.0 ? -thr : thr;
  return p;
}

__device__ __forceinline__ void log_pivot(const CallP &P, int64_t row, double orig, bool fired,
                                          double thr) {
  if (fired) {
    int k = atomicAdd(&P.status[0], 1);
    if (k < P.pert_cap) {
      P.pert_rows[k] = row;
      P.pert_vals[k] = orig;
    } else {
      P.status[2] = 1;
    }
  }
  if (thr == 0.0 && orig == 0.0) atomicCAS(&P.status[1], 0, (int)(row + 1));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(HY_FULL, v, o);
  return v;
}

// atomic max for non-negative doubles (bit patterns order like unsigned ints)
__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

}  // namespace hy
