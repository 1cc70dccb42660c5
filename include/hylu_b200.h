/* hylu_b200.h — C ABI of the B200-native HYLU numeric factorization / solve.
 *
 * The reference (arxiv/paper_2509_07690, Python package ``polylu``) exposes a pure
 * Python API and ships no numeric/solve code; each entry
 * point below replaces one SPEC operation and is bound by the ctypes layer in
 * paper_2509_07690_b200/device.py, which presents the SPEC Python signatures:
 *
 *   hy_upload_symbolic            <- SymbolicStructure/PivotScale/Ordering upload
 *                                    (outputs of SPEC.md:155,165,175-223)
 *   hy_factorize                  <- factorize(A, ps, ord, sym, opts)
 *   hy_refactorize                <- refactorize(A_new, prior, opts)
 *   hy_solve                      <- solve(A, factors, ps, ord, b) w/o refinement
 *                                    (forward/backward substitution)
 *   hy_upload_matrix, hy_residual, hy_axpy
 *                                 <- iterative_refinement's r = b - A x, backward_error
 *                                    and x += d (matrix.py:258-310)
 *   hy_refactorize_solve_batched  <- B x [refactorize -> solve] sharing one symbolic
 *                                    (BASELINE config 4; SURVEY §3 call stack 3)
 *
 * Conventions: plain pointers and sizes; device pointers are prefixed d_; every
 * call is asynchronous on the given CUDA stream (0 = legacy default stream).
 * Return codes map 1:1 to the reference exception classes (errors.py):
 *   HY_OK 0, HY_DIMENSION_MISMATCH 1 (DimensionMismatch, errors.py:32),
 *   HY_ZERO_DIAGONAL 2 (ZeroDiagonal, :52), HY_CYCLE_DETECTED 3 (CycleDetected, :56),
 *   HY_NUMERIC_BREAKDOWN 4 (NumericBreakdown, :60), HY_PATTERN_MISMATCH 5
 *   (PatternMismatch, :64), HY_CUDA_ERROR 10, HY_INVALID_ARGUMENT 11.
 * NumericBreakdown is detected on the device: it is reported through the
 * factors' status word (read it after synchronizing the stream).
 * No C++ exception crosses the ABI.  A handle is bound to one device and is
 * not re-entrant; use one handle per GPU.
 */
#ifndef HYLU_B200_H
#define HYLU_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  HY_OK = 0,
  HY_DIMENSION_MISMATCH = 1,
  HY_ZERO_DIAGONAL = 2,
  HY_CYCLE_DETECTED = 3,
  HY_NUMERIC_BREAKDOWN = 4,
  HY_PATTERN_MISMATCH = 5,
  HY_CUDA_ERROR = 10,
  HY_INVALID_ARGUMENT = 11
};

/* KernelMode (config.py:11-16) */
enum { HY_ROWROW = 0, HY_SUPROW = 1, HY_SUPSUP = 2 };

typedef struct hy_handle hy_handle;

/* Host arrays describing the symbolic structure in node layout:
 * node u spans factor rows [node_first[u], node_first[u+1]); its ascending column
 * list is cols[colptr[u] .. colptr[u+1]) with L width nl[u]; its values are a
 * dense row-major (rows x width) block at valoff[u].  Everything is copied to the
 * device once; the host arrays may be freed after the call returns. */
typedef struct {
  int64_t n;            /* dimension */
  int64_t nnodes;
  int64_t nnz;          /* nnz(A) */
  int32_t kernel_mode;  /* HY_ROWROW / HY_SUPROW / HY_SUPSUP (max tier) */
  const int64_t *node_first;   /* [nnodes+1] */
  const int8_t *node_kind;     /* [nnodes] 0 = standalone row, 1 = supernode */
  const int64_t *colptr;       /* [nnodes+1] */
  const int32_t *cols;         /* [colptr[nnodes]] */
  const int64_t *nl;           /* [nnodes] */
  const int64_t *valoff;       /* [nnodes+1] */
  const int64_t *dep_ptr;      /* [nnodes+1] */
  const int32_t *deps;         /* ascending source nodes per node */
  const int64_t *level_ptr;    /* [nlevels+1] factorization / forward-solve levels */
  const int32_t *level_nodes;
  int64_t nlevels;
  const int64_t *ulevel_ptr;   /* [nulevels+1] backward-solve levels */
  const int32_t *ulevel_nodes;
  int64_t nulevels;
  const int64_t *a_row_ptr;    /* [n+1] CSR row pointer of A (original rows) */
  const int64_t *a_col_idx;    /* [nnz]  (pattern check only) */
  const int64_t *mrow_src;     /* [n] original row feeding M row i */
  const int32_t *colpos;       /* [nnz] position of each A entry in its node's column list */
  const double *scale;         /* [nnz] dr[row]*dc[col] */
  const double *dr;            /* [n] */
  const double *dc;            /* [n] */
  const int64_t *perm;         /* [n] symmetric ordering, perm[k] = index at position k */
} hy_symbolic_desc;

/* NumericFactors on the device.  All buffers are caller-owned
 * device memory (torch tensors in the Python layer). */
typedef struct {
  double *d_values;        /* [stored values] node layout */
  int32_t *d_inner_perm;   /* [n] block-relative pivot order per supernode row */
  double *d_anorm;         /* [1] */
  int32_t *d_status;       /* [4]: [0] perturbation count, [1] breakdown row + 1 (0 = none),
                                   [2] log overflow flag, [3] reserved */
  int64_t *d_pert_rows;    /* [pert_cap] factor rows where perturbation fired */
  double *d_pert_vals;     /* [pert_cap] original pivot values */
  int64_t pert_cap;
  int32_t kernel_mode;     /* out: the kernel mode (maximum tier) the call ran with */
} hy_factors;

int hy_create(int device, hy_handle **out);
void hy_destroy(hy_handle *h);
const char *hy_last_error(void);

int hy_upload_symbolic(hy_handle *h, const hy_symbolic_desc *desc);
/* Number of doubles a hy_factors.d_values buffer needs. */
int64_t hy_stored_values(const hy_handle *h);

int hy_factorize(hy_handle *h, const double *d_avals, double eps, hy_factors *out,
                 uintptr_t stream);
int hy_refactorize(hy_handle *h, const double *d_avals, double eps, const hy_factors *prior,
                   hy_factors *out, uintptr_t stream);
int hy_solve(hy_handle *h, const hy_factors *f, const double *d_b, double *d_x,
             uintptr_t stream);
/* FactorOptions.kernel_override: the kernel mode of the following
 * hy_factorize / hy_refactorize calls on this handle (-1 = the uploaded analysis'
 * kernel_mode).  Device dispatch (DESIGN.md §3 "Kernel selection"):
 * kernel_mode is the maximum tier.  ROWROW: every update runs in row-row operation
 * order (the running target value minus each source row's product, source rows
 * ascending — update_row_by_row) in every update kernel;
 * SUPROW / SUPSUP: supernode sources act as blocks (multiplier block by TRSM, then
 * the block product summed and subtracted once — update_row_by_sup / sup_by_sup,
 * SPEC.md:300-318), the product on DMMA for multi-row targets (k_fi_upd_kc / kcp)
 * and as a warp GEMV for targets of <= 4 rows (k_fi_upd_w). */
int hy_set_kernel_mode(hy_handle *h, int mode);

/* Iterative refinement on the device.  hy_upload_matrix: A's
 * pattern in original coordinates (SparseMatrixCSR row_ptr / col_idx,
 * matrix.py:30-66), once per analysis.  hy_residual: d_r = b - A x (d_r may be
 * NULL) and *d_berr = max_i |b - Ax|_i / (|A||x| + |b|)_i with 0/0 = 0
 * (backward_error, matrix.py:267-285, 303-310), bitwise the reference's row loops
 * (index order, no fused multiply-add).  hy_axpy: x += dx elementwise. */
int hy_upload_matrix(hy_handle *h, const int64_t *row_ptr, const int32_t *col_idx);
int hy_residual(hy_handle *h, const double *d_avals, const double *d_x, const double *d_b,
                double *d_r, double *d_berr, uintptr_t stream);
int hy_axpy(hy_handle *h, double *d_x, const double *d_dx, uintptr_t stream);
/* Partition-based substitution for many right-hand sides (Fig. 3;
 * host side paper_2509_07690_b200/partition.py build_partition / device_launches).
 * Launch lists per direction: rows of 6 int64 (kind, seq, lo, hi, item offset, item
 * count); kind 0 = rectangular block (items: row-range pairs [r0, r1), one warp each;
 * forward entries with column < lo, backward column >= hi), kind 1 = triangular
 * level (items: nodes; entries with column in [lo, hi)); seq = 1: one warp walks the
 * items in order.  hy_solve_multi: d_B / d_X [nrhs][n] row-major (x_j = A^-1 b_j with
 * the factors' scaling and permutations, no refinement). */
typedef struct {
  int64_t nfwd, nbwd, nitems;
  const int64_t *fwd;      /* [nfwd][6] */
  const int64_t *bwd;      /* [nbwd][6] */
  const int32_t *items;    /* [nitems] */
} hy_partition_desc;
int hy_upload_partition(hy_handle *h, const hy_partition_desc *d);
int hy_solve_multi(hy_handle *h, const hy_factors *f, int64_t nrhs, const double *d_B, double *d_X,
                   uintptr_t stream);

/* Batched forms for the automatic refinement of perturbed batch instances
 * (SPEC.md:492, 499-507): d_vals [B][nnz], d_x / d_b / d_r [B][n] row-major,
 * d_berr [B] (one backward error per instance, same arithmetic as hy_residual);
 * instances with d_mask[b] == 0 are skipped (d_mask NULL = all).
 * hy_axpy_batched: d_y[b] = d_x[b] + d_dx[b] (d_dx NULL: a copy) where masked. */
int hy_residual_batched(hy_handle *h, int64_t B, const double *d_vals, const double *d_x,
                        const double *d_b, double *d_r, double *d_berr, const int32_t *d_mask,
                        uintptr_t stream);
int hy_axpy_batched(hy_handle *h, int64_t B, double *d_y, const double *d_x, const double *d_dx,
                    const int32_t *d_mask, uintptr_t stream);

/* Column-slab plan for supernode targets (schedule.build_slab_plan): one CTA per
 * slab, slabs grouped by factorization level.  Optional: without it supernodes
 * run the one-CTA-per-supernode kernel. */
typedef struct {
  int64_t nslabs, nitems, ndeps, nlevels;
  const int32_t *sl_node;       /* [nslabs] target supernode */
  const int32_t *sl_c0;         /* [nslabs] first column position */
  const int32_t *sl_c1;         /* [nslabs] end column position */
  const int8_t *sl_kind;        /* [nslabs] 0 L-region, 1 block, 2 panel */
  const int64_t *it_ptr;        /* [nslabs+1] */
  const int32_t *it_k;          /* [nitems] source index within the target's deps */
  const int32_t *it_q0;         /* [nitems] beyond-block column range of the source */
  const int32_t *it_q1;
  const int8_t *it_own;         /* [nitems] slab owns the source's block columns */
  const int32_t *dep_pb;        /* [ndeps] block position of each source in its target */
  const int64_t *level_slab_ptr;/* [nlevels+1] */
  const int32_t *level_smax;    /* [nlevels] max target rows */
  const int32_t *level_mmax;    /* [nlevels] max source rows */
  const int32_t *level_swmax;   /* [nlevels] max slab width */
  const int32_t *level_accmax;  /* [nlevels] max rows x width of a slab accumulator */
} hy_slab_plan;
int hy_upload_slab_plan(hy_handle *h, const hy_slab_plan *plan);

/* Level fan-in plan (schedule.build_fanin_plan), used in SUPROW / SUPSUP modes:
 * per level, the nodes to factor, their permutation / TRSM tiles, the dependency
 * edges leaving the level (multiplier blocks) and the (target, column tile)
 * update items with their source lists. */
typedef struct {
  int64_t nlevels, nsrc, ndeps;
  const int64_t *lu_ptr;  const int32_t *lu_nodes;                 /* [nlevels+1], [nnodes] */
  const int64_t *pt_ptr;  const int32_t *pt_node, *pt_c0, *pt_c1;  /* tiles */
  const int64_t *xp_ptr;  const int64_t *xp_edge; const int32_t *xp_tgt;
  const int64_t *lev_up;  const int32_t *up_t, *up_c0, *up_c1; const int64_t *up_ptr;
  const int32_t *src_k, *src_q0, *src_q1;                          /* [nsrc] */
  const int32_t *dep_pb;                                           /* [ndeps] */
  const int32_t *level_smax, *level_mmax;                          /* [nlevels] */
  const int32_t *src_v, *src_pb, *src_tb;   /* [nsrc] source node, block position, first block row */
  const int64_t *lev_up_big;                /* [nlevels] first item routed to the DMMA kernel */
  const int64_t *lev_up_reg;                /* [nlevels] first per-source item (before: packed) */
  const int64_t *lev_up_rs;                 /* [nlevels] first per-source item run CTA-per-item
                                               (before it, from lev_up_reg: warp-per-item) */
  const int64_t *lev_xp_big;                /* [nlevels] first multiplier item run CTA-per-item
                                               (before it: warp-per-item) */
  int64_t nhub;                             /* standalone rows computed by pull programs
                                               (hy_upload_hub_programs) instead of fan-in updates */
  const int64_t *lev_hub;                   /* [nlevels+1] offsets into hub_list */
  const int32_t *hub_list;                  /* [nhub] those rows' nodes, by level */
  int64_t nparts;                           /* split-K parts of heavy packed update items */
  const int32_t *up_part;                   /* [nitems] part id or -1 */
  const int32_t *part_first, *part_n;       /* [nparts] first part of the item, parts of the item */
  const int64_t *part_off;                  /* [nparts] partial-tile offset (doubles) in the scratch */
} hy_fanin_plan;
int hy_upload_fanin_plan(hy_handle *h, const hy_fanin_plan *plan);
/* Optional, after hy_upload_fanin_plan: per update-source record (nsrc records, plan
 * order) the tile position of each of its columns (pos[poff[z] .. poff[z+1]), int8) and
 * the source's value offset / width / first panel column / block height, so the
 * K-concatenated update kernel skips the per-item binary searches. */
int hy_upload_fanin_maps(hy_handle *h, int64_t nsrc, int64_t npos, const int64_t *poff,
                         const int8_t *pos, const int64_t *vb, const int32_t *vW, const int32_t *qb,
                         const int32_t *m);

/* Row programs for the batched path (built on the host by schedule.py for a given
 * prior inner_perm).  Must be uploaded before the
 * batched calls, and must match the inner_perm of the prior they are used with. */
typedef struct {
  int64_t nsteps, nrel, nhubrows, nlev, nhpos, npred, nwi, nsp, max_slots;
  const int64_t *row_ptr;   /* [n+1] */
  const int32_t *st_p;      /* [nsteps] */
  const int32_t *st_j;
  const int64_t *st_src;
  const int32_t *st_cnt;
  const int64_t *st_rel;
  const int32_t *rel;       /* [nrel] */
  const uint8_t *node_hub;  /* [nnodes] */
  const int64_t *hrow_lev;  /* [nhubrows+1] */
  const int64_t *lev_ptr;   /* [nlev+1] */
  const int32_t *hpos;      /* [nhpos] */
  const int64_t *hdiv;      /* [nhpos] */
  const int64_t *hpp;       /* [nhpos+1] */
  const int32_t *pred_p;    /* [npred] */
  const int64_t *pred_u;    /* [npred] */
  const int64_t *lev_wi;    /* [nlev+1] gather work items per intra-row level */
  const int32_t *wi_p;      /* [nwi] target position */
  const int64_t *wi_kd;     /* [nwi] finalize kind: diag offset / -1 U / -2 pivot */
  const int64_t *wi_y0;
  const int64_t *wi_y1;
  const int32_t *wi_slot;
  const int64_t *lev_sp;    /* [nlev+1] split positions per intra-row level */
  const int32_t *sp_p;      /* [nsp] */
  const int64_t *sp_kd;
  const int32_t *sp_s0;
  const int32_t *sp_n;
  const int32_t *level_ws;  /* [nlevels] widest non-hub node per factorization level */
  const int64_t *node_rec;  /* [nnodes][4] valoff, dep0, first|rows<<32, width|nl<<32 */
  const int64_t *row_rec;   /* [n][4] step0, A entry0, nsteps|nentries<<32, original row */
} hy_row_programs;
int hy_upload_row_programs(hy_handle *h, const hy_row_programs *progs);
/* Pull programs for standalone hub rows of the single-instance row path (ROWROW
 * mode); built with hub detection restricted to standalone rows. */
int hy_upload_hub_programs(hy_handle *h, const hy_row_programs *progs);

/* Batched refactorize + solve of B instances sharing the uploaded symbolic
 * structure and the prior's inner_perm / anorm.  d_vals [B][nnz], d_b / d_x [B][n]
 * (row-major), d_npert [B] receives each instance's perturbation count.  The
 * handle owns the interleaved factor workspace (grown on demand). */
int hy_refactorize_solve_batched(hy_handle *h, int64_t B, const double *d_vals,
                                 const double *d_b, double *d_x, double eps,
                                 const hy_factors *prior, int32_t *d_npert, uintptr_t stream);
/* The two phases of hy_refactorize_solve_batched (same semantics), exposed so a
 * caller can time them separately.  hy_solve_batched uses the factors of the last
 * hy_refactorize_batched call on this handle (same B). */
int hy_refactorize_batched(hy_handle *h, int64_t B, const double *d_vals, double eps,
                           const hy_factors *prior, int32_t *d_npert, const double *d_b_fuse,
                           uintptr_t stream);
/* d_b == NULL: use the forward substitution fused into the last
 * hy_refactorize_batched(..., d_b_fuse != NULL) call (only the backward pass runs). */
int hy_solve_batched(hy_handle *h, int64_t B, const double *d_b, double *d_x, uintptr_t stream);
/* Copy instance b's factor values from the last batched call into node layout. */
int hy_batched_factor_values(hy_handle *h, int64_t b, double *d_out, uintptr_t stream);

/* Tuning knobs (developer options; defaults are the measured best):
 *   "fanin_tc"      sup-sup / sup-row update kernels of the level fan-in: 0 FFMA per-source
 *                   (k_fi_upd), 2 per-source DMMA (k_fi_upd_tc, bitwise equal to 0),
 *                   4 K-concatenated DMMA (k_fi_upd_kc), 5 (default) = 4 plus the packed
 *                   small-source items on k_fi_upd_kcp; 1 / 3 route only targets >= 32 rows
 *   "fanin_overlap" 0/1 (default 1): independent kernels of a fan-in phase on two streams
 *   "fanin_warp_min" items below which a level keeps its small items on the CTA kernels
 *   "fanin_maps"    0/1 (default 1): host-precomputed source maps in the update kernels
 *   "pipe_ws", "pipe_blocks": batched-pipeline shared workspace / resident CTAs
 *   "refactor_panels" 0/1 (default 1): a refactorization launches only the panel tiles of the
 *                   panel kernel (the L-part tiles only apply row swaps the prior inner_perm holds)
 *   "lu1_kernel"    0/1 (default 1): single-row nodes of a fan-in level perturb their pivot in a
 *                   thread-per-node kernel (k_fi_lu1) instead of a CTA each
 *   "bwd_narrow"    batched backward solve: levels with at most this many (node, group pair) tasks
 *                   use 8-entry load batches (default 4096)
 *   "pipe_order"    claim order of the batched pipeline's (node, group pair) tasks: 1 (default)
 *                   level-major (every pair at level k, then level k+1), 0 diagonal (pair g at
 *                   level k with pair g+1 at level k-1), K >= 2 diagonal below level K-1 and
 *                   level-major from there; scheduling only, results bitwise equal
 *   (the measured-slower variants of round 1 were removed; DESIGN.md lists them). */
int hy_set_option(hy_handle *h, const char *name, int64_t value);

/* Number of kernel launches issued by this handle since creation (bench evidence). */
int64_t hy_launch_count(const hy_handle *h);

#ifdef __cplusplus
}
#endif
#endif
