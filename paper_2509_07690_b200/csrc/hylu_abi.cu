// hylu_abi.cu — the extern "C" boundary (include/hylu_b200.h): handle, one-time
// symbolic upload, level plans, and the launch sequences for factorize /
// refactorize / solve / batched refactorize+solve.
#include <cstdio>
#include <cstring>
#include <string>
#include <algorithm>
#include <map>
#include <vector>

#include "hylu_b200.h"
#include "hylu_common.cuh"

namespace hy {
// kernels (hylu_factor.cu / hylu_batch.cu)
__global__ void k_anorm(const double *, const double *, int64_t, double *);
__global__ void k_rows(DevSym, const CallP *, const int32_t *, int);
__global__ void k_sn(DevSym, const CallP *, const int32_t *);
size_t sn_smem_bytes();
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
  const int32_t *dep_pb;
};
__global__ void k_slab(DevSym, const CallP *, SlabDev, int, int *, int *, int *, int, int, int, int, int);
__global__ void k_lperm(DevSym, const CallP *, const int32_t *, int);
__global__ void k_hub1(DevSym, const CallP *, DevProg, const int32_t *, double *, int);
size_t slab_smem_bytes(int, int, int, int);
struct FaninDev {
  const int32_t *lu_nodes;
  const int32_t *pt_node;
  const int32_t *pt_c0;
  const int32_t *pt_c1;
  const int64_t *xp_edge;
  const int32_t *xp_tgt;
  const int32_t *up_t;
  const int32_t *up_c0;
  const int32_t *up_c1;
  const int64_t *up_ptr;
  const int32_t *src_k;
  const int32_t *src_q0;
  const int32_t *src_q1;
  const int32_t *dep_pb;
  const int32_t *src_v;
  const int32_t *src_pb;
  const int32_t *src_tb;
  const int32_t *up_part;    // layout shared with hylu_fanin.cu
  const int32_t *part_first;
  const int32_t *part_n;
  const int64_t *part_off;
  double *part_scr;
  int *part_cnt;
  const int64_t *src_poff;   // host-precomputed source maps (hy_upload_fanin_maps)
  const int8_t *src_pos;
  const int64_t *src_vb;
  const int32_t *src_vW;
  const int32_t *src_qb;
  const int32_t *src_m;
  const ItemRec *up_rec;     // [items] packed prologue records (k_item_rec)
  const uint64_t *up_mask;   // [items] tile columns any source touches (k_item_mask; needs the maps)
  const XRec *xp_rec;        // [X items] packed records (k_x_rec)
  const NodeItemRec *lu_rec; // [LU items] / [panel items] packed records (k_node_rec)
  const NodeItemRec *pt_rec;
};
__global__ void k_fi_scatter(DevSym, const CallP *);
__global__ void k_item_rec(DevSym, FaninDev, int64_t, ItemRec *);
__global__ void k_x_rec(DevSym, FaninDev, int64_t, XRec *);
__global__ void k_node_rec(DevSym, const int32_t *, const int32_t *, const int32_t *, int64_t, NodeItemRec *);
__global__ void k_item_mask(FaninDev, int64_t, uint64_t *);
size_t fi_lu_smem();
size_t fi_panel_smem();
size_t fi_upd_w_smem();
__global__ void k_call_set(CallP *, CallP);
__global__ void k_ptr_set(const double **, const double *);
__global__ void k_call_prep(const CallP *, int, int64_t, int);
__global__ void k_anorm_p(const CallP *, const double *, int64_t);
__global__ void k_resid_berr(int, const int64_t *, const int32_t *, const double *, const double *,
                             const double *, double *, unsigned long long *);
__global__ void k_axpy1(int, double *, const double *);
__global__ void k_resid_berr_b(int, int64_t, const int64_t *, const int32_t *, const double *,
                               const double *, const double *, double *, unsigned long long *,
                               const int32_t *);
__global__ void k_axpy_b(int, double *, const double *, const double *, const int32_t *);
__global__ void k_msolve(DevSym, const double *, int, int, int, int, const int32_t *, int, int, double *, int);
__global__ void k_mbhat(DevSym, const int32_t *, const double *, double *, int);
__global__ void k_msolve_long(DevSym, const double *, const int32_t *, int, double *, int);
__global__ void k_msolve_sn(DevSym, const double *, const int32_t *, int, double *, int);
__global__ void k_mxout(DevSym, const double *, double *, int);

__global__ void k_fi_lu(DevSym, const CallP *, FaninDev, int);
__global__ void k_fi_lu1(DevSym, const CallP *, FaninDev, int, int);
__global__ void k_fi_panel(DevSym, const CallP *, FaninDev, int);
__global__ void k_fi_x(DevSym, const CallP *, FaninDev, int);
__global__ void k_fi_upd(DevSym, const CallP *, FaninDev, int, int, int);
__global__ void k_fi_upd_pk(DevSym, const CallP *, FaninDev, int, int, int);
__global__ void k_fi_x_w(DevSym, const CallP *, FaninDev, int, int);
__global__ void k_fi_upd_w(DevSym, const CallP *, FaninDev, int, int);
size_t fi_upd_smem(int, int);
size_t fi_upd_tc_smem(int);
size_t fi_upd_kc_smem();
template <bool CHAIN> __global__ void k_fi_upd_kc(DevSym, const CallP *, FaninDev, int);
template <bool CHAIN> __global__ void k_fi_upd_kcp(DevSym, const CallP *, FaninDev, int);
__global__ void k_fi_upd_tc(DevSym, const CallP *, FaninDev, int, int);
size_t hub_smem_bytes();
int hub_threads();
__global__ void k_bhat(DevSym, const int32_t *, const double *, double *);
__global__ void k_xout(DevSym, const double *, double *);
__global__ void k_fwd(DevSym, const double *, const int32_t *, int, double *);
struct SolveChunk {
  int32_t node;
  int32_t c0, c1;
  int32_t slot;
};
__global__ void k_solve_part(DevSym, const double *const *, const SolveChunk *, int, const double *, double *, int);
__global__ void k_fwd_fin(DevSym, const double *const *, const SolveRec *, int, const double *, double *);
__global__ void k_bwd_fin(DevSym, const double *const *, const SolveRec *, int, const double *, double *);
__global__ void k_solve_rec(DevSym, const int32_t *, const int32_t *, const int32_t *, int64_t, SolveRec *);
__global__ void k_bwd(DevSym, const double *, const int32_t *, int, double *);

size_t pipe_smem(int ws);
__global__ void k_bt_pipe2(DevSym, BatchP, DevProg, const TaskDesc *, int64_t, const double *, double *, int *,
                           int *, int, int, int);
__global__ void k_bt_hub(DevSym, BatchP, DevProg, const int32_t *, int, int, const double *, double *,
                         double *, int, int *, int);
__global__ void k_batch_bhat(DevSym, const int32_t *, const double *, double *, int64_t);
__global__ void k_batch_fwd(DevSym, const double *, int64_t, const int32_t *, int, int, double *);
template <int BWDW>
__global__ void k_batch_bwd2(DevSym, const double *, int64_t, const int32_t *, int, int, double *);
__global__ void k_batch_xout2(DevSym, const int32_t *, const double *, double *, int64_t);
__global__ void k_perm_inverse(int, const int64_t *, int32_t *);
__global__ void k_row_of(DevSym, const int32_t *, int32_t *);
__global__ void k_batch_bhat2(DevSym, const int32_t *, const double *, double *, int64_t);
__global__ void k_batch_extract(const double *, int64_t, int64_t, double *);
}  // namespace hy

using namespace hy;

static thread_local std::string g_err;

static int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                              \
  do {                                                                                     \
    cudaError_t _e = (x);                                                                  \
    if (_e != cudaSuccess)                                                                 \
      return fail(HY_CUDA_ERROR, std::string(#x) + ": " + cudaGetErrorString(_e));         \
  } while (0)

// Per level: standalone-row nodes and supernode nodes, in level order.
struct Plan {
  std::vector<int64_t> rptr, sptr;  // [nlev+1] offsets into the concatenated lists
  int32_t *d_rows = nullptr, *d_sns = nullptr;
  int nlev = 0;
  // batched: all nodes per level
  std::vector<int64_t> aptr;
  int32_t *d_all = nullptr;
};

// Chunked-substitution plan for one direction: per level, chunk list and per-node
// slot ranges (nodes in the same order as the level plan's d_all list).
struct SolvePlan {
  std::vector<int64_t> cptr;         // [nlev+1] chunk offsets
  SolveChunk *d_chunks = nullptr;
  int32_t *d_slot0 = nullptr, *d_nslot = nullptr;  // per node in level order
  SolveRec *d_rec = nullptr;                       // packed per-node records (k_solve_rec)
  int64_t nslots = 0;
};

struct hy_handle {
  int device = 0;
  DevSym S{};
  std::vector<void *> allocs;
  Plan fplan, bplan;
  SolvePlan fsolve, bsolve;
  double *d_solve_scratch = nullptr;
  int64_t stored = 0;
  bool uploaded = false;
  // host copies of per-node data for descriptor building
  std::vector<int64_t> h_first, h_colptr, h_valoff, h_dptr, h_nl;
  std::vector<longlong4> h_row_rec;   // batched row programs' row records (task descriptors)
  struct Win { int64_t rel0, k0, nk, nrel; };
  std::vector<Win> h_win;              // per node: program window (nk == 0: not staged)
  std::vector<int32_t> h_deps;        // dependency lists (task descriptors inline the first 4)
  double *d_y = nullptr;          // single-solve workspace [n]
  double *d_bf = nullptr;         // batched factor workspace
  int64_t bf_cap = 0;             // doubles
  double *d_by = nullptr;         // batched solve workspace
  double *d_bri = nullptr;        // batched pivot reciprocals [G][n][32]
  int64_t by_cap = 0;
  int64_t last_B = 0;
  const int32_t *last_iperm = nullptr;
  bool last_fused = false;
  // batched row programs (schedule.py), built per prior inner_perm
  DevProg prog{};
  bool prog_ok = false;
  std::vector<void *> prog_allocs;
  std::vector<int64_t> bl_rptr, bl_hptr;   // per level: non-hub / hub node offsets
  std::vector<int32_t> level_ws;           // per level: widest non-hub node
  int max_slots = 0;
  int *d_flags = nullptr;                  // [nn * G] completion epochs
  int64_t flags_cap = 0;
  int *d_counters = nullptr;               // one claim counter (int64) per launch of a call
  int counters_cap = 0;
  int epoch = 0;
  int32_t *d_node_level = nullptr;
  int pipe_blocks = 0;
  int warp_min = 256;                      // fan-in: below this many small items per level, CTA kernels only
  int64_t bwd_narrow = BWD_NARROW;         // batched backward solve: levels with at most this many tasks use BWD_WL-entry batches
  int refactor_panels = 1;                 // refactorize launches only the panel tiles of k_fi_panel (the L-part tiles are no-ops there)
  int64_t lu1_min = 256;                   // ... for levels with at least this many single-row nodes
  int lu1_kernel = 1;                      // fan-in: single-row nodes' pivot perturbation as a thread-per-node kernel
  int pipe_order = 1;                      // claim order of the batched pipeline: 1 level-major (default), 0 diagonal, K >= 2 diagonal below level K-1 (build_segments)
  int pipe_ws = 6;                         // pair-mode shared workspace columns per group (c4 ms/step: 4: 15.50, 6: 15.48, 8: 15.64, 10: 15.64, 16: 16.65 before the reciprocals)
  // claim order per (segment, G)
  struct Seg {
    int l0, l1;
    TaskDesc *d_tasks = nullptr;   // task descriptors in claim order
    int64_t ntasks = 0;
  };
  std::vector<Seg> segs;
  int segs_G = -1;
  std::map<int, std::vector<Seg>> seg_cache;   // task lists per group count (chunked callers vary G)
  double *d_scratch = nullptr;             // hub partial sums
  int64_t scratch_cap = 0;
  int32_t *d_bl_rows = nullptr, *d_bl_hubs = nullptr;
  int64_t launches = 0;
  size_t sn_smem = 0;
  // slab plan for supernode targets (single-instance factorization)
  bool slab_ok = false;
  SlabDev slab{};
  std::vector<void *> slab_allocs;
  std::vector<int64_t> slab_lptr;          // slabs per level
  std::vector<int32_t> slab_smax, slab_mmax, slab_swmax, slab_accmax;
  int *d_slab_counters = nullptr;          // one per level
  int *d_dep_flags = nullptr;              // per dependency edge
  int *d_lu_flags = nullptr;               // per node
  int slab_epoch = 0;
  // level fan-in plan (SUPROW / SUPSUP modes)
  bool fanin_ok = false;
  FaninDev fi{};
  std::vector<void *> fi_allocs;
  std::vector<int64_t> fi_lu, fi_pt, fi_xp, fi_up;   // per-level offsets
  std::vector<int64_t> fi_lu1;                       // per level: single-row nodes at the head of its LU list
  std::vector<int64_t> fi_ptp;                       // per level: panel tiles at the head of its panel-item list
  std::vector<int64_t> fi_upbig;                     // per level: first DMMA-routed item
  std::vector<int64_t> fi_upreg;                     // per level: first per-source item
  std::vector<int64_t> fi_uprs;                      // per level: first CTA-per-item regular item
  std::vector<int64_t> fi_xpbig;                     // per level: first CTA-per-item multiplier item
  std::vector<int64_t> fi_hub;                       // per level: offsets of pull-program rows
  int32_t *d_fi_hubs = nullptr;
  int32_t *d_pinv = nullptr;   // inverse column permutation (batched output order)
  int32_t *d_rowof = nullptr;  // factor row of each original row (batched b̂ in source order)
  int64_t *d_arow = nullptr;   // A's pattern in original coordinates (refinement)
  int32_t *d_acol = nullptr;
  int fi_maps = 1;                                   // option "fanin_maps": use host-precomputed source maps in k_fi_upd_kc
  int fi_overlap = 1;                                // option "fanin_overlap": panel TRSM on a side stream, concurrent with the X blocks
  cudaStream_t fi_side = nullptr;
  cudaEvent_t fi_ev_lu = nullptr, fi_ev_pt = nullptr;
  int fi_tc = 5;                                     // option "fanin_tc": DMMA update kernels (1/2: per-source k_fi_upd_tc for targets >= 32 rows / all regular items; 3/4: K-concatenated k_fi_upd_kc, same split; 5 (default): k_fi_upd_kcp for the packed items too)
  std::vector<int32_t> fi_smax, fi_mmax;
  int64_t fi_nsrc = -1;                              // source records of the uploaded plan
  CallP *d_callp = nullptr;                          // per-call parameters (device), see k_call_set
  cudaStream_t cap_stream = nullptr;                 // graph capture stream
  cudaGraphExec_t fi_exec2[2] = {nullptr, nullptr};   // level fan-in graph per call kind (0 factorize, 1 refactorize; captured on first use)
  int cur_refactor = 0;                              // kind of the call being launched (run_fanin)
  cudaGraphExec_t sv_exec = nullptr;                 // substitution levels graph
  int64_t sv_graph_launches = 0;
  const double **d_fptr = nullptr;                   // factor values of the current solve (device slot)
  int64_t fi_graph_launches2[2] = {0, 0};            // kernels per graph replay
  int use_graphs = 1;                                // option "graphs"
  int use_pdl = 1;                                   // option "pdl": programmatic dependent launch in the fan-in
  // partition-based multi-RHS solve (hy_upload_partition / hy_solve_multi)
  std::vector<int64_t> ms_fwd, ms_bwd;               // [k][6] launch lists
  int32_t *d_ms_items = nullptr;
  double *d_my = nullptr;                            // Y [n][nrhs]
  int64_t my_cap = 0;
  int mode_an = 2;                                   // kernel_mode of the uploaded analysis
  int kmode = -1;                                    // hy_set_kernel_mode (-1: mode_an)
  int fi_chain = -1;                                 // row-row order instantiations in the captured fan-in graph
  int sm_count = 148;
  // single-instance hub rows (ROWROW path): programs + per-level hub node lists
  bool hub1_ok = false;
  DevProg prog1{};
  std::vector<void *> hub1_allocs;
  std::vector<int64_t> hub1_ptr;
  int32_t *d_hub1 = nullptr;
  int hub1_slots = 0;
  double *d_hub1_scratch = nullptr;
  int64_t hub1_scratch_cap = 0;

};

static void free_segments(hy_handle *h);
static void drop_graph(hy_handle *h) {
  for (int k = 0; k < 2; ++k) {
    if (h->fi_exec2[k]) cudaGraphExecDestroy(h->fi_exec2[k]);
    h->fi_exec2[k] = nullptr;
  }
  if (h->sv_exec) cudaGraphExecDestroy(h->sv_exec);
  h->sv_exec = nullptr;
}

template <class T>
static int upload(hy_handle *h, T **dst, const T *src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return HY_OK;
  CK(cudaMalloc((void **)dst, sizeof(T) * count));
  h->allocs.push_back(*dst);
  if (src) CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HY_OK;
}

#define UP(dst, src, cnt)                              \
  do {                                                 \
    int _r = upload(h, dst, src, (int64_t)(cnt));      \
    if (_r) return _r;                                 \
  } while (0)

static int build_plan(hy_handle *h, Plan &pl, const int64_t *lptr, const int32_t *lnodes,
                      int64_t nlev, const int8_t *kind) {
  pl.nlev = (int)nlev;
  pl.rptr.assign(nlev + 1, 0);
  pl.sptr.assign(nlev + 1, 0);
  pl.aptr.assign(nlev + 1, 0);
  std::vector<int32_t> rows, sns, all;
  for (int64_t l = 0; l < nlev; ++l) {
    for (int64_t k = lptr[l]; k < lptr[l + 1]; ++k) {
      const int32_t u = lnodes[k];
      (kind[u] ? sns : rows).push_back(u);
      all.push_back(u);
    }
    pl.rptr[l + 1] = (int64_t)rows.size();
    pl.sptr[l + 1] = (int64_t)sns.size();
    pl.aptr[l + 1] = (int64_t)all.size();
  }
  UP(&pl.d_rows, rows.data(), rows.size());
  UP(&pl.d_sns, sns.data(), sns.size());
  UP(&pl.d_all, all.data(), all.size());
  return HY_OK;
}

template <class T>
static int upload_prog(hy_handle *h, T **dst, const T *src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return HY_OK;
  CK(cudaMalloc((void **)dst, sizeof(T) * count));
  h->prog_allocs.push_back(*dst);
  CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HY_OK;
}

#define UPP(dst, src, cnt)                                 \
  do {                                                     \
    int _r = upload_prog(h, dst, src, (int64_t)(cnt));     \
    if (_r) return _r;                                     \
  } while (0)

static void free_segments(hy_handle *h) {
  for (auto &kv : h->seg_cache)
    for (auto &sg : kv.second) cudaFree(sg.d_tasks);
  h->seg_cache.clear();
  h->segs.clear();
  h->segs_G = -1;
}

// Per hub-free level segment, the flat (node, group pair) task list in claim order
// (pipe_order: level-major by default; the diagonal lists pair g at level l with pair g+1
// at level l-1).  Any order that lists a pair's levels ascending is deadlock-free.
static int build_segments(hy_handle *h, int G) {
  auto hit = h->seg_cache.find(G);
  if (hit != h->seg_cache.end()) {
    h->segs = hit->second;
    h->segs_G = G;
    return HY_OK;
  }
  if (h->seg_cache.size() >= 8) free_segments(h);
  h->segs.clear();
  const int nl = h->fplan.nlev;
  std::vector<int32_t> rows(h->bl_rptr[nl]);
  if (!rows.empty())
    CK(cudaMemcpy(rows.data(), h->d_bl_rows, sizeof(int32_t) * rows.size(), cudaMemcpyDeviceToHost));
  int l = 0;
  while (l < nl) {
    int l1 = l + 1;
    if (h->bl_hptr[l + 1] == h->bl_hptr[l])
      while (l1 < nl && h->bl_hptr[l1 + 1] == h->bl_hptr[l1]) ++l1;
    hy_handle::Seg sg;
    sg.l0 = l;
    sg.l1 = l1;
    const int lb = 0;
    const int L = l1 - l;
    std::vector<TaskDesc> tasks;
    tasks.reserve((size_t)(h->bl_rptr[l1] - h->bl_rptr[l]) * G);
    auto mk = [&](int32_t u, int32_t g) {
      TaskDesc t;
      t.u = u;
      t.g = g;
      t.valoff = h->h_valoff[u];
      t.r = (int32_t)h->h_first[u];
      t.s = (int32_t)(h->h_first[u + 1] - h->h_first[u]);
      t.W = (int32_t)(h->h_colptr[u + 1] - h->h_colptr[u]);
      t.L = (int32_t)h->h_nl[u];
      t.d0 = h->h_dptr[u];
      t.d1 = h->h_dptr[u + 1];
      t.rr0 = h->h_row_rec[t.r];
      const hy_handle::Win &w = h->h_win[u];
      t.rel0 = w.rel0;
      t.k0 = (int32_t)w.k0;
      t.nk = (int32_t)w.nk;
      t.nrel = (int32_t)w.nrel;
      t.pad[0] = t.pad[1] = t.pad[2] = 0;
      for (int k = 0; k < 4; ++k)
        t.dep[k] = t.d0 + k < t.d1 ? h->h_deps[t.d0 + k] : -1;
      return t;
    };
    const int sk = 1;   // diagonal slope (2-4 measured slower)
    const int gs = 2;                         // pair mode: tasks carry the even group of a pair
    const int GT = (G + gs - 1) / gs;
    // pipe_order = 0: diagonal over every level.  pipe_order = K >= 1: the levels
    // below K-1 stay diagonal, the levels from K-1 up are claimed level by level
    // across all pairs (K = 1: pure level-major), so every pair's narrow top levels
    // run concurrently instead of the last pairs' chains forming a tail.
    const int Ld = h->pipe_order == 0 ? L : std::min(L, h->pipe_order - 1);
    for (int d = 0; d < sk * (GT - 1) + Ld; ++d)
      for (int k = lb; k < Ld && k <= d; ++k) {
        if ((d - k) % sk) continue;
        const int g = (d - k) / sk;
        if (g >= GT) continue;
        for (int64_t q = h->bl_rptr[l + k]; q < h->bl_rptr[l + k + 1]; ++q) tasks.push_back(mk(rows[q], g * gs));
      }
    for (int k = Ld; k < L; ++k)
      for (int g = 0; g < GT; ++g)
        for (int64_t q = h->bl_rptr[l + k]; q < h->bl_rptr[l + k + 1]; ++q) tasks.push_back(mk(rows[q], g * gs));
    sg.ntasks = (int64_t)tasks.size();
    if (sg.ntasks) {
      CK(cudaMalloc((void **)&sg.d_tasks, sizeof(TaskDesc) * sg.ntasks));
      CK(cudaMemcpy(sg.d_tasks, tasks.data(), sizeof(TaskDesc) * sg.ntasks, cudaMemcpyHostToDevice));
    }
    h->segs.push_back(sg);
    l = l1;
  }
  h->seg_cache[G] = h->segs;
  h->segs_G = G;
  return HY_OK;
}

template <class T>
static int upload_slab(hy_handle *h, T **dst, const T *src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return HY_OK;
  CK(cudaMalloc((void **)dst, sizeof(T) * count));
  h->slab_allocs.push_back(*dst);
  if (src) CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HY_OK;
}

#define UPS(dst, src, cnt)                                 \
  do {                                                     \
    int _r = upload_slab(h, dst, src, (int64_t)(cnt));     \
    if (_r) return _r;                                     \
  } while (0)

template <class T>
static int upload_fi(hy_handle *h, T **dst, const T *src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return HY_OK;
  CK(cudaMalloc((void **)dst, sizeof(T) * count));
  h->fi_allocs.push_back(*dst);
  CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HY_OK;
}

#define UPF(dst, src, cnt)                                 \
  do {                                                     \
    int _r = upload_fi(h, dst, src, (int64_t)(cnt));       \
    if (_r) return _r;                                     \
  } while (0)

template <class T>
static int upload_h1(hy_handle *h, T **dst, const T *src, int64_t count) {
  *dst = nullptr;
  if (count <= 0) return HY_OK;
  CK(cudaMalloc((void **)dst, sizeof(T) * count));
  h->hub1_allocs.push_back(*dst);
  CK(cudaMemcpy(*dst, src, sizeof(T) * count, cudaMemcpyHostToDevice));
  return HY_OK;
}
#define UPH(dst, src, cnt)                                 \
  do {                                                     \
    int _r = upload_h1(h, dst, src, (int64_t)(cnt));       \
    if (_r) return _r;                                     \
  } while (0)

// Kernel launch with optional programmatic dependent launch (PDL, see pdl_wait): the
// fan-in kernels wait for their predecessor inside, so their launch latency and CTA
// scheduling overlap the predecessor's execution.
template <typename... KArgs, typename... Args>
static cudaError_t launchx(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                           bool pdl, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = pdl ? at : nullptr;
  cfg.numAttrs = pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, args...);
}


extern "C" {

const char *hy_last_error(void) { return g_err.c_str(); }

int hy_create(int device, hy_handle **out) {
  if (!out) return fail(HY_INVALID_ARGUMENT, "null output handle");
  CK(cudaSetDevice(device));
  hy_handle *h = new hy_handle();
  h->device = device;
  h->sn_smem = sn_smem_bytes();
  cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, device);
  cudaError_t e = cudaFuncSetAttribute(k_sn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)h->sn_smem);
  if (e != cudaSuccess) {
    delete h;
    return fail(HY_CUDA_ERROR, std::string("cudaFuncSetAttribute(k_sn): ") + cudaGetErrorString(e));
  }
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bt_hub, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hub_smem_bytes());
  if (e == cudaSuccess)
    e = cudaFuncSetAttribute(k_bt_pipe2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pipe_smem(64));
  if (e != cudaSuccess) {
    delete h;
    return fail(HY_CUDA_ERROR, std::string("cudaFuncSetAttribute(k_bt_pipe): ") + cudaGetErrorString(e));
  }
  *out = h;
  return HY_OK;
}

void hy_destroy(hy_handle *h) {
  if (!h) return;
  cudaSetDevice(h->device);
  for (void *p : h->allocs) cudaFree(p);
  for (void *p : h->prog_allocs) cudaFree(p);
  for (void *p : h->slab_allocs) cudaFree(p);
  for (void *p : h->fi_allocs) cudaFree(p);
  for (void *p : h->hub1_allocs) cudaFree(p);
  if (h->d_hub1_scratch) cudaFree(h->d_hub1_scratch);
  if (h->d_bf) cudaFree(h->d_bf);
  if (h->d_scratch) cudaFree(h->d_scratch);
  if (h->d_flags) cudaFree(h->d_flags);
  drop_graph(h);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  if (h->d_callp) cudaFree(h->d_callp);
  if (h->d_fptr) cudaFree(h->d_fptr);
  if (h->fi_side) cudaStreamDestroy(h->fi_side);
  if (h->fi_ev_lu) cudaEventDestroy(h->fi_ev_lu);
  if (h->fi_ev_pt) cudaEventDestroy(h->fi_ev_pt);
  free_segments(h);
  if (h->d_counters) cudaFree(h->d_counters);
  if (h->d_by) cudaFree(h->d_by);
  if (h->d_bri) cudaFree(h->d_bri);
  if (h->d_arow) cudaFree(h->d_arow);
  if (h->d_pinv) cudaFree(h->d_pinv);
  if (h->d_rowof) cudaFree(h->d_rowof);
  if (h->d_acol) cudaFree(h->d_acol);
  if (h->d_ms_items) cudaFree(h->d_ms_items);
  if (h->d_my) cudaFree(h->d_my);
  delete h;
}

int64_t hy_stored_values(const hy_handle *h) { return h ? h->stored : -1; }
int64_t hy_launch_count(const hy_handle *h) { return h ? h->launches : -1; }

int hy_set_option(hy_handle *h, const char *name, int64_t value) {
  if (!h || !name) return fail(HY_INVALID_ARGUMENT, "null handle/name");
  drop_graph(h);   // every option can change the fan-in launch sequence
  if (std::string(name) == "pdl") {
    h->use_pdl = value != 0;
    return HY_OK;
  }
  if (std::string(name) == "graphs") {
    h->use_graphs = value != 0;
    return HY_OK;
  }
  if (std::string(name) == "fanin_maps") {
    h->fi_maps = value != 0;
    return HY_OK;
  }
  if (std::string(name) == "fanin_overlap") {
    h->fi_overlap = value != 0;
    return HY_OK;
  }
  if (std::string(name) == "fanin_tc" && value >= 0 && value <= 5) {
    h->fi_tc = (int)value;
    return HY_OK;
  }
  if (std::string(name) == "fanin_warp_min" && value >= 1) {
    h->warp_min = (int)value;
    return HY_OK;
  }
  if (std::string(name) == "pipe_blocks" && value >= 0) {   // 0: occupancy-derived (default)
    h->pipe_blocks = (int)value;
    return HY_OK;
  }
  if (std::string(name) == "bwd_narrow" && value >= 0) {
    h->bwd_narrow = value;
    return HY_OK;
  }
  if (std::string(name) == "refactor_panels" && (value == 0 || value == 1)) {
    h->refactor_panels = (int)value;
    return HY_OK;
  }
  if (std::string(name) == "lu1_min" && value >= 1) {
    h->lu1_min = value;
    return HY_OK;
  }
  if (std::string(name) == "lu1_kernel" && (value == 0 || value == 1)) {
    h->lu1_kernel = (int)value;
    return HY_OK;
  }
  if (std::string(name) == "pipe_order" && value >= 0) {
    h->pipe_order = (int)value;
    free_segments(h);
    return HY_OK;
  }
  if (std::string(name) == "pipe_ws" && value >= 1 && value <= 64) {
    h->pipe_ws = (int)value;
    h->pipe_blocks = 0;
    return HY_OK;
  }
  return fail(HY_INVALID_ARGUMENT, std::string("unknown option ") + name);
}

int hy_upload_symbolic(hy_handle *h, const hy_symbolic_desc *d) {
  if (!h || !d) return fail(HY_INVALID_ARGUMENT, "null handle/descriptor");
  if (h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic already uploaded to this handle");
  if (d->n <= 0 || d->nnodes <= 0 || d->n > INT32_MAX)
    return fail(HY_DIMENSION_MISMATCH, "invalid dimension");
  if (d->kernel_mode < 0 || d->kernel_mode > 2) return fail(HY_INVALID_ARGUMENT, "bad kernel_mode");
  CK(cudaSetDevice(h->device));
  const int64_t n = d->n, nn = d->nnodes, nnz = d->nnz;
  // validate node structure (host side, cheap): rows partition [0,n), deps point backward
  if (d->node_first[0] != 0 || d->node_first[nn] != n)
    return fail(HY_DIMENSION_MISMATCH, "node rows do not partition [0, n)");
  for (int64_t u = 0; u < nn; ++u) {
    const int64_t s = d->node_first[u + 1] - d->node_first[u];
    if (s <= 0 || s > 64) return fail(HY_INVALID_ARGUMENT, "node row count outside [1, 64]");
    if (d->nl[u] < 0 || d->nl[u] > d->colptr[u + 1] - d->colptr[u])
      return fail(HY_INVALID_ARGUMENT, "bad L width");
    for (int64_t k = d->dep_ptr[u]; k < d->dep_ptr[u + 1]; ++k)
      if (d->deps[k] >= u || d->deps[k] < 0)
        return fail(HY_CYCLE_DETECTED, "dependency does not point to a lower node");
  }
  DevSym &S = h->S;
  S.n = (int32_t)n;
  S.nn = (int32_t)nn;
  S.mode = d->kernel_mode;
  h->mode_an = d->kernel_mode;
  h->kmode = -1;
  S.nnz = nnz;
  int64_t *p64;
  int32_t *p32;
  UP(&p64, d->node_first, nn + 1); S.first = p64;
  h->h_first.assign(d->node_first, d->node_first + nn + 1);
  h->h_colptr.assign(d->colptr, d->colptr + nn + 1);
  h->h_valoff.assign(d->valoff, d->valoff + nn + 1);
  h->h_dptr.assign(d->dep_ptr, d->dep_ptr + nn + 1);
  h->h_deps.assign(d->deps, d->deps + d->dep_ptr[nn]);
  h->h_nl.assign(d->nl, d->nl + nn);
  int8_t *p8;
  UP(&p8, d->node_kind, nn); S.kind = p8;
  UP(&p64, d->colptr, nn + 1); S.colptr = p64;
  UP(&p32, d->cols, d->colptr[nn]); S.cols = p32;
  std::vector<int32_t> nl32(nn), node_of(n);
  for (int64_t u = 0; u < nn; ++u) {
    nl32[u] = (int32_t)d->nl[u];
    for (int64_t r = d->node_first[u]; r < d->node_first[u + 1]; ++r) node_of[r] = (int32_t)u;
  }
  UP(&p32, nl32.data(), nn); S.nl = p32;
  UP(&p64, d->valoff, nn + 1); S.valoff = p64;
  UP(&p64, d->dep_ptr, nn + 1); S.dptr = p64;
  UP(&p32, d->deps, d->dep_ptr[nn]); S.deps = p32;
  UP(&p32, node_of.data(), n); S.node_of = p32;
  UP(&p64, d->a_row_ptr, n + 1); S.a_ptr = p64;
  UP(&p64, d->mrow_src, n); S.mrow_src = p64;
  UP(&p32, d->colpos, nnz); S.colpos = p32;
  double *pd;
  UP(&pd, d->scale, nnz); S.scale = pd;
  UP(&pd, d->dr, n); S.dr = pd;
  UP(&pd, d->dc, n); S.dc = pd;
  UP(&p64, d->perm, n); S.perm = p64;
  UP(&h->d_y, (const double *)nullptr, n);
  h->stored = d->valoff[nn];
  int rc = build_plan(h, h->fplan, d->level_ptr, d->level_nodes, d->nlevels, d->node_kind);
  if (rc) return rc;
  rc = build_plan(h, h->bplan, d->ulevel_ptr, d->ulevel_nodes, d->nulevels, d->node_kind);
  if (rc) return rc;
  {
    // chunked substitution plans (forward: L part [0, L); backward: panel [L+s, W))
    const int CH = 512;   // k_solve_part holds a chunk's gathered values in 16 registers per lane
    for (int dir = 0; dir < 2; ++dir) {
      const int64_t *lp = dir == 0 ? d->level_ptr : d->ulevel_ptr;
      const int32_t *ln = dir == 0 ? d->level_nodes : d->ulevel_nodes;
      const int64_t nlev = dir == 0 ? d->nlevels : d->nulevels;
      SolvePlan &sp = dir == 0 ? h->fsolve : h->bsolve;
      std::vector<SolveChunk> chunks;
      std::vector<int32_t> slot0, nslot;
      sp.cptr.assign(nlev + 1, 0);
      int64_t maxslots = 0;
      for (int64_t l = 0; l < nlev; ++l) {
        int32_t slot = 0;
        for (int64_t k = lp[l]; k < lp[l + 1]; ++k) {
          const int32_t u = ln[k];
          const int64_t s = d->node_first[u + 1] - d->node_first[u];
          const int64_t W = d->colptr[u + 1] - d->colptr[u];
          const int64_t lo = dir == 0 ? 0 : d->nl[u] + s, hi = dir == 0 ? d->nl[u] : W;
          slot0.push_back(slot);
          int32_t ns = 0;
          // small: the finish warp does it (one warp walks at most 512 off-block columns)
          const bool direct = (hi - lo) * s <= 8192 && hi - lo <= 512;
          for (int64_t c = lo; c < hi && !direct; c += CH) {
            chunks.push_back(SolveChunk{u, (int32_t)c, (int32_t)(c + CH < hi ? c + CH : hi), slot + ns});
            ++ns;
          }
          nslot.push_back(ns);
          slot += ns;
        }
        sp.cptr[l + 1] = (int64_t)chunks.size();
        if (slot > maxslots) maxslots = slot;
      }
      sp.nslots = maxslots;
      UP(&sp.d_chunks, chunks.data(), chunks.size());
      UP(&sp.d_slot0, slot0.data(), slot0.size());
      UP(&sp.d_nslot, nslot.data(), nslot.size());
      UP(&sp.d_rec, (const SolveRec *)nullptr, (int64_t)std::max<size_t>(slot0.size(), 1));
      if (!slot0.empty()) {
        k_solve_rec<<<(unsigned)std::min<int64_t>(((int64_t)slot0.size() + 255) / 256, 4096), 256>>>(
            h->S, (dir == 0 ? h->fplan : h->bplan).d_all, sp.d_slot0, sp.d_nslot, (int64_t)slot0.size(), sp.d_rec);
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
      }
    }
    const int64_t ns = (h->fsolve.nslots > h->bsolve.nslots ? h->fsolve.nslots : h->bsolve.nslots);
    UP(&h->d_solve_scratch, (const double *)nullptr, (ns > 0 ? ns : 1) * 64);
  }
  {
    std::vector<int32_t> lev(nn, 0);
    for (int64_t l = 0; l < d->nlevels; ++l)
      for (int64_t k = d->level_ptr[l]; k < d->level_ptr[l + 1]; ++k) lev[d->level_nodes[k]] = (int32_t)l;
    UP(&h->d_node_level, lev.data(), nn);
  }
  h->uploaded = true;
  return HY_OK;
}

int hy_upload_slab_plan(hy_handle *h, const hy_slab_plan *d) {
  if (!h || !h->uploaded || !d) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded / null");
  if (d->nlevels != h->fplan.nlev) return fail(HY_DIMENSION_MISMATCH, "slab plan level count mismatch");
  CK(cudaSetDevice(h->device));
  for (void *p : h->slab_allocs) cudaFree(p);
  h->slab_allocs.clear();
  SlabDev &D = h->slab;
  int32_t *p32;
  int8_t *p8;
  int64_t *p64;
  UPS(&p32, d->sl_node, d->nslabs); D.sl_node = p32;
  UPS(&p32, d->sl_c0, d->nslabs); D.sl_c0 = p32;
  UPS(&p32, d->sl_c1, d->nslabs); D.sl_c1 = p32;
  UPS(&p8, d->sl_kind, d->nslabs); D.sl_kind = p8;
  UPS(&p64, d->it_ptr, d->nslabs + 1); D.it_ptr = p64;
  UPS(&p32, d->it_k, d->nitems); D.it_k = p32;
  UPS(&p32, d->it_q0, d->nitems); D.it_q0 = p32;
  UPS(&p32, d->it_q1, d->nitems); D.it_q1 = p32;
  UPS(&p8, d->it_own, d->nitems); D.it_own = p8;
  UPS(&p32, d->dep_pb, d->ndeps); D.dep_pb = p32;
  h->slab_lptr.assign(d->level_slab_ptr, d->level_slab_ptr + d->nlevels + 1);
  h->slab_smax.assign(d->level_smax, d->level_smax + d->nlevels);
  h->slab_mmax.assign(d->level_mmax, d->level_mmax + d->nlevels);
  h->slab_swmax.assign(d->level_swmax, d->level_swmax + d->nlevels);
  h->slab_accmax.assign(d->level_accmax, d->level_accmax + d->nlevels);
  // re-split the factorization level plan: slab targets -> slab list, others -> rows
  {
    std::vector<uint8_t> isslab(h->S.nn, 0);
    for (int64_t k = 0; k < d->nslabs; ++k) isslab[d->sl_node[k]] = 1;
    Plan &pl = h->fplan;
    std::vector<int32_t> all(pl.aptr[pl.nlev]);
    if (!all.empty())
      CK(cudaMemcpy(all.data(), pl.d_all, sizeof(int32_t) * all.size(), cudaMemcpyDeviceToHost));
    std::vector<int32_t> rows, sns;
    for (int l = 0; l < pl.nlev; ++l) {
      for (int64_t k = pl.aptr[l]; k < pl.aptr[l + 1]; ++k) (isslab[all[k]] ? sns : rows).push_back(all[k]);
      pl.rptr[l + 1] = (int64_t)rows.size();
      pl.sptr[l + 1] = (int64_t)sns.size();
    }
    UPS(&pl.d_rows, rows.data(), rows.size());
    UPS(&pl.d_sns, sns.data(), sns.size());
  }
  UPS(&h->d_slab_counters, (const int *)nullptr, d->nlevels + 1);
  UPS(&h->d_dep_flags, (const int *)nullptr, d->ndeps + 1);
  UPS(&h->d_lu_flags, (const int *)nullptr, h->S.nn);
  CK(cudaMemset(h->d_dep_flags, 0, sizeof(int) * (d->ndeps + 1)));
  CK(cudaMemset(h->d_lu_flags, 0, sizeof(int) * h->S.nn));
  size_t mx = 0;
  for (int64_t l = 0; l < d->nlevels; ++l) {
    if (d->level_slab_ptr[l + 1] == d->level_slab_ptr[l]) continue;
    const size_t b = slab_smem_bytes(d->level_smax[l], d->level_mmax[l], d->level_swmax[l], d->level_accmax[l]);
    if (b > mx) mx = b;
  }
  if (mx > 227 * 1024) return fail(HY_INVALID_ARGUMENT, "slab shared memory exceeds 227 KB");
  if (mx) CK(cudaFuncSetAttribute(k_slab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
  h->slab_epoch = 0;
  h->slab_ok = true;
  return HY_OK;
}

int hy_upload_fanin_plan(hy_handle *h, const hy_fanin_plan *d) {
  if (!h || !h->uploaded || !d) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded / null");
  drop_graph(h);
  CK(cudaSetDevice(h->device));
  for (void *p : h->fi_allocs) cudaFree(p);
  h->fi_allocs.clear();
  const int64_t nl = d->nlevels;
  FaninDev &D = h->fi;
  D.src_poff = nullptr; D.src_pos = nullptr; D.src_vb = nullptr;
  D.src_vW = nullptr; D.src_qb = nullptr; D.src_m = nullptr;
  D.up_mask = nullptr;
  int32_t *p32;
  int64_t *p64;
  {   // per level: single-row nodes first (thread per node, k_fi_lu1), then the supernodes (CTA each)
    std::vector<int32_t> lun(d->lu_nodes, d->lu_nodes + d->lu_ptr[nl]);
    h->fi_lu1.assign(nl, 0);
    for (int64_t l = 0; l < nl; ++l) {
      auto b = lun.begin() + d->lu_ptr[l], e = lun.begin() + d->lu_ptr[l + 1];
      auto mid = std::stable_partition(b, e, [&](int32_t u) { return h->h_first[u + 1] - h->h_first[u] == 1; });
      h->fi_lu1[l] = (int64_t)(mid - b);
    }
    UPF(&p32, lun.data(), d->lu_ptr[nl]); D.lu_nodes = p32;
  }
  {   // per level: the panel tiles (right of the block) first, then the L-part tiles, which only
      // apply the block's row swaps: a refactorization (prior inner_perm pre-applied) skips them
    const int64_t npt = d->pt_ptr[nl];
    std::vector<int32_t> idx(npt), pn(npt), pc0(npt), pc1(npt);
    for (int64_t q = 0; q < npt; ++q) idx[q] = (int32_t)q;
    h->fi_ptp.assign(nl, 0);
    for (int64_t l = 0; l < nl; ++l) {
      auto b = idx.begin() + d->pt_ptr[l], e = idx.begin() + d->pt_ptr[l + 1];
      auto mid = std::stable_partition(b, e, [&](int32_t q) {
        const int32_t u = d->pt_node[q];
        return d->pt_c0[q] >= h->h_nl[u] + (h->h_first[u + 1] - h->h_first[u]);
      });
      h->fi_ptp[l] = (int64_t)(mid - b);
    }
    for (int64_t q = 0; q < npt; ++q) {
      pn[q] = d->pt_node[idx[q]];
      pc0[q] = d->pt_c0[idx[q]];
      pc1[q] = d->pt_c1[idx[q]];
    }
    UPF(&p32, pn.data(), npt); D.pt_node = p32;
    UPF(&p32, pc0.data(), npt); D.pt_c0 = p32;
    UPF(&p32, pc1.data(), npt); D.pt_c1 = p32;
  }
  UPF(&p64, d->xp_edge, d->xp_ptr[nl]); D.xp_edge = p64;
  UPF(&p32, d->xp_tgt, d->xp_ptr[nl]); D.xp_tgt = p32;
  UPF(&p32, d->up_t, d->lev_up[nl]); D.up_t = p32;
  UPF(&p32, d->up_c0, d->lev_up[nl]); D.up_c0 = p32;
  UPF(&p32, d->up_c1, d->lev_up[nl]); D.up_c1 = p32;
  UPF(&p64, d->up_ptr, d->lev_up[nl] + 1); D.up_ptr = p64;
  UPF(&p32, d->src_k, d->nsrc); D.src_k = p32;
  h->fi_nsrc = d->nsrc;
  UPF(&p32, d->src_q0, d->nsrc); D.src_q0 = p32;
  UPF(&p32, d->src_q1, d->nsrc); D.src_q1 = p32;
  UPF(&p32, d->dep_pb, d->ndeps); D.dep_pb = p32;
  UPF(&p32, d->src_v, d->nsrc); D.src_v = p32;
  UPF(&p32, d->src_pb, d->nsrc); D.src_pb = p32;
  UPF(&p32, d->src_tb, d->nsrc); D.src_tb = p32;
  {   // packed item records for the update kernels' prologue
    const int64_t ni = d->lev_up[nl];
    ItemRec *rec = nullptr;
    CK(cudaMalloc((void **)&rec, sizeof(ItemRec) * (ni > 0 ? ni : 1)));
    h->fi_allocs.push_back(rec);
    if (ni > 0) {
      k_item_rec<<<(unsigned)std::min<int64_t>((ni + 255) / 256, 4096), 256>>>(h->S, D, ni, rec);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
    }
    D.up_rec = rec;
  }
  {   // packed records of the multiplier-block (X) items
    const int64_t nx = d->xp_ptr[nl];
    XRec *xr = nullptr;
    CK(cudaMalloc((void **)&xr, sizeof(XRec) * (nx > 0 ? nx : 1)));
    h->fi_allocs.push_back(xr);
    if (nx > 0) {
      k_x_rec<<<(unsigned)std::min<int64_t>((nx + 255) / 256, 4096), 256>>>(h->S, D, nx, xr);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
    }
    D.xp_rec = xr;
  }
  {   // packed records of the LU and panel items
    const int64_t nlu = d->lu_ptr[nl], npt = d->pt_ptr[nl];
    NodeItemRec *lr = nullptr, *pr = nullptr;
    CK(cudaMalloc((void **)&lr, sizeof(NodeItemRec) * (nlu > 0 ? nlu : 1)));
    h->fi_allocs.push_back(lr);
    CK(cudaMalloc((void **)&pr, sizeof(NodeItemRec) * (npt > 0 ? npt : 1)));
    h->fi_allocs.push_back(pr);
    if (nlu > 0)
      k_node_rec<<<(unsigned)std::min<int64_t>((nlu + 255) / 256, 4096), 256>>>(h->S, D.lu_nodes, nullptr, nullptr, nlu, lr);
    if (npt > 0)
      k_node_rec<<<(unsigned)std::min<int64_t>((npt + 255) / 256, 4096), 256>>>(h->S, D.pt_node, D.pt_c0, D.pt_c1, npt, pr);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    D.lu_rec = lr;
    D.pt_rec = pr;
  }
  h->fi_lu.assign(d->lu_ptr, d->lu_ptr + nl + 1);
  h->fi_pt.assign(d->pt_ptr, d->pt_ptr + nl + 1);
  h->fi_xp.assign(d->xp_ptr, d->xp_ptr + nl + 1);
  h->fi_up.assign(d->lev_up, d->lev_up + nl + 1);
  h->fi_upbig.assign(d->lev_up_big, d->lev_up_big + nl);
  h->fi_upreg.assign(d->lev_up_reg, d->lev_up_reg + nl);
  h->fi_uprs.assign(d->lev_up_rs, d->lev_up_rs + nl);
  h->fi_xpbig.assign(d->lev_xp_big, d->lev_xp_big + nl);
  for (int64_t q = 0; q < d->pt_ptr[nl]; ++q)   // k_fi_panel: one thread per tile column
    if (d->pt_c1[q] - d->pt_c0[q] > 256) return fail(HY_INVALID_ARGUMENT, "panel tile wider than 256");
  D.up_part = nullptr; D.part_first = nullptr; D.part_n = nullptr; D.part_off = nullptr;
  D.part_scr = nullptr; D.part_cnt = nullptr;
  if (d->nparts > 0) {
    const int64_t nitems = d->lev_up[nl];
    UPF(&p32, d->up_part, nitems); D.up_part = p32;
    UPF(&p32, d->part_first, d->nparts); D.part_first = p32;
    UPF(&p32, d->part_n, d->nparts); D.part_n = p32;
    UPF(&p64, d->part_off, d->nparts); D.part_off = p64;
    // partial tiles (offsets restart per level): the largest offset plus one tile
    int64_t scr = 0;
    for (int64_t q = 0; q < d->nparts; ++q) scr = d->part_off[q] > scr ? d->part_off[q] : scr;
    scr += 64 * 64;
    CK(cudaMalloc((void **)&D.part_scr, sizeof(double) * scr));
    h->fi_allocs.push_back(D.part_scr);
    CK(cudaMalloc((void **)&D.part_cnt, sizeof(int) * d->nparts));
    h->fi_allocs.push_back(D.part_cnt);
    CK(cudaMemset(D.part_cnt, 0, sizeof(int) * d->nparts));
  }
  h->fi_hub.assign(nl + 1, 0);
  h->d_fi_hubs = nullptr;
  if (d->nhub > 0) {
    if (!d->lev_hub || !d->hub_list) return fail(HY_INVALID_ARGUMENT, "pull rows without their lists");
    h->fi_hub.assign(d->lev_hub, d->lev_hub + nl + 1);
    UPF(&p32, d->hub_list, d->nhub); h->d_fi_hubs = p32;
  }
  h->fi_smax.assign(d->level_smax, d->level_smax + nl);
  h->fi_mmax.assign(d->level_mmax, d->level_mmax + nl);
  size_t mx = 0;
  for (int64_t l = 0; l < nl; ++l) {
    const size_t b = fi_upd_smem(h->fi_smax[l], h->fi_mmax[l]);
    if (b > mx) mx = b;
  }
  CK(cudaFuncSetAttribute(k_fi_upd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
  CK(cudaFuncSetAttribute(k_fi_upd_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_tc_smem(64)));
  CK(cudaFuncSetAttribute(k_fi_upd_kc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_kc_smem()));
  CK(cudaFuncSetAttribute(k_fi_upd_kc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_kc_smem()));
  CK(cudaFuncSetAttribute(k_fi_upd_kcp<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_kc_smem()));
  CK(cudaFuncSetAttribute(k_fi_upd_kcp<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_kc_smem()));
  CK(cudaFuncSetAttribute(k_fi_upd_pk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)mx));
  CK(cudaDeviceGetAttribute(&h->sm_count, cudaDevAttrMultiProcessorCount, h->device));
  CK(cudaFuncSetAttribute(k_fi_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_panel_smem()));
  CK(cudaFuncSetAttribute(k_fi_lu, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_lu_smem()));
  CK(cudaFuncSetAttribute(k_fi_upd_w, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fi_upd_w_smem()));
  CK(cudaFuncSetAttribute(k_fi_x, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(2 * 64 * 65 * sizeof(double))));
  h->fanin_ok = true;
  return HY_OK;
}


static int run_fanin(hy_handle *h, const CallP *Pd, cudaStream_t st) {
  CK(launchx(k_fi_scatter, dim3((h->S.n * 32 + 255) / 256), dim3(256), 0, st, h->use_pdl, h->S, Pd));
  h->launches++;
  const int nfl = (int)h->fi_lu.size() - 1;
  for (int l = 0; l < nfl; ++l) {
    const int nlu = (int)(h->fi_lu[l + 1] - h->fi_lu[l]);
    const int npt = h->cur_refactor && h->refactor_panels ? (int)h->fi_ptp[l] : (int)(h->fi_pt[l + 1] - h->fi_pt[l]);
    const int nxp = (int)(h->fi_xp[l + 1] - h->fi_xp[l]);
    const int nup = (int)(h->fi_up[l + 1] - h->fi_up[l]);
    // PDL on latency-bound levels only: on a level with many CTAs the successor's
    // early-resident CTAs would take slots from the predecessor's last waves
    const int64_t lvmax = std::max<int64_t>(std::max<int64_t>(nlu, h->fi_pt[l + 1] - h->fi_pt[l]),
                                            std::max<int64_t>(h->fi_xp[l + 1] - h->fi_xp[l], nup));
    const bool pdl = h->use_pdl && lvmax <= 16 * (int64_t)h->sm_count;
    // pull-program rows of this level: every source is final, compute them whole
    const int nph = (int)(h->fi_hub[l + 1] - h->fi_hub[l]);
    if (nph) {
      if (!h->hub1_ok) return fail(HY_INVALID_ARGUMENT, "fan-in plan has pull rows but no hub programs");
      const int64_t need = (int64_t)nph * h->hub1_slots;
      if (need > h->hub1_scratch_cap) {
        if (h->d_hub1_scratch) CK(cudaFree(h->d_hub1_scratch));
        h->d_hub1_scratch = nullptr;
        CK(cudaMalloc((void **)&h->d_hub1_scratch, sizeof(double) * need));
        h->hub1_scratch_cap = need;
      }
      k_hub1<<<nph, 1024, 0, st>>>(h->S, Pd, h->prog1, h->d_fi_hubs + h->fi_hub[l], h->d_hub1_scratch,
                                   h->hub1_slots);
      h->launches++;
    }
    // single-row nodes: one thread each (their "LU" is the pivot perturbation); supernodes: a CTA each
    // (a level with few of them keeps them in k_fi_lu's grid: one launch less on the chain)
    const int nlu1 = h->lu1_kernel && h->fi_lu1[l] >= h->lu1_min ? (int)h->fi_lu1[l] : 0;
    if (nlu1) {
      CK(launchx(k_fi_lu1, dim3((nlu1 + 255) / 256), dim3(256), 0, st, pdl, h->S, Pd, h->fi, (int)h->fi_lu[l], nlu1));
      h->launches++;
    }
    if (nlu - nlu1) {
      CK(launchx(k_fi_lu, dim3(nlu - nlu1), dim3(256), fi_lu_smem(), st, pdl, h->S, Pd, h->fi,
                 (int)h->fi_lu[l] + nlu1));
      h->launches++;
    }
    // the panel TRSM of the level's nodes and the X blocks of their edges both need
    // only the nodes' LU: with fanin_overlap the panel runs on a side stream while the
    // X blocks run on `st`; the update kernels (which need both) wait for it
    // Independent kernels of a phase run on two streams (fanin_overlap): after the
    // LU, the panel TRSM (side) and the X blocks (st) need only the LU; after both,
    // the packed-item updates (side) and the other update groups (st) touch disjoint
    // target tiles.  Each phase joins back into `st`.
    auto fork = [&]() -> int {
      if (!h->fi_side) {
        CK(cudaStreamCreateWithFlags(&h->fi_side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&h->fi_ev_lu, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&h->fi_ev_pt, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(h->fi_ev_lu, st));
      CK(cudaStreamWaitEvent(h->fi_side, h->fi_ev_lu, 0));
      return HY_OK;
    };
    auto join = [&]() -> int {
      CK(cudaEventRecord(h->fi_ev_pt, h->fi_side));
      CK(cudaStreamWaitEvent(st, h->fi_ev_pt, 0));
      return HY_OK;
    };
    const int xb = nxp ? ((int)h->fi_xpbig[l] - (int)h->fi_xp[l] < h->warp_min ? (int)h->fi_xp[l]
                                                                                : (int)h->fi_xpbig[l])
                       : 0;
    const int nw = nxp ? xb - (int)h->fi_xp[l] : 0, nc = nxp ? (int)h->fi_xp[l + 1] - xb : 0;
    // phase A: panel on the side stream when anything else runs; else the warp X items
    const bool sideA = h->fi_overlap && ((npt && (nw || nc)) || (!npt && nw && nc));
    if (sideA) {
      int rc = fork();
      if (rc) return rc;
    }
    cudaStream_t sp = sideA && npt ? h->fi_side : st;
    cudaStream_t sw = sideA && !npt ? h->fi_side : st;
    if (npt) {
      CK(launchx(k_fi_panel, dim3(npt), dim3(256), fi_panel_smem(), sp, pdl && sp == st, h->S, Pd, h->fi,
                 (int)h->fi_pt[l]));
      h->launches++;
    }
    if (nw) {
      CK(launchx(k_fi_x_w, dim3((nw + 7) / 8), dim3(256), 0, sw, pdl && sw == st, h->S, Pd, h->fi,
                 (int)h->fi_xp[l], nw));
      h->launches++;
    }
    if (nc) {
      CK(launchx(k_fi_x, dim3(nc), dim3(256), 2 * 64 * 65 * sizeof(double), st, pdl, h->S, Pd, h->fi, xb));
      h->launches++;
    }
    if (sideA) {
      int rc = join();
      if (rc) return rc;
    }
    if (nup) {
      const size_t sm = fi_upd_smem(h->fi_smax[l], h->fi_mmax[l]);
      const int reg = (int)h->fi_upreg[l];
      const int split = (h->fi_tc == 1 || h->fi_tc == 3) ? (int)h->fi_upbig[l] : (int)h->fi_up[l + 1];
      const int npk = reg - (int)h->fi_up[l];
      const int nbig = (int)h->fi_up[l + 1] - split;
      const int rs = (int)h->fi_uprs[l] - reg < h->warp_min ? reg : (int)h->fi_uprs[l];
      // phase B: packed items on the side stream when other update groups exist
      const bool sideB = h->fi_overlap && npk && (rs > reg || split > rs || nbig);
      if (sideB) {
        int rc = fork();
        if (rc) return rc;
      }
      cudaStream_t sk = sideB ? h->fi_side : st;
      if (npk && h->fi_tc == 5) {
        FaninDev Dp = h->fi;
        if (!h->fi_maps) Dp.src_pos = nullptr;
        CK(launchx(h->fi_chain ? k_fi_upd_kcp<true> : k_fi_upd_kcp<false>, dim3(npk), dim3(256), fi_upd_kc_smem(),
                   sk, pdl && sk == st, h->S, Pd, Dp, (int)h->fi_up[l]));
        h->launches++;
      } else if (npk) {
        k_fi_upd_pk<<<npk, 256, sm, sk>>>(h->S, Pd, h->fi, (int)h->fi_up[l], h->fi_smax[l], h->fi_mmax[l]);
        h->launches++;
      }
      if (rs > reg) {
        FaninDev Dw = h->fi;
        if (!h->fi_maps) Dw.src_pos = nullptr;
        CK(launchx(k_fi_upd_w, dim3((rs - reg + 7) / 8), dim3(256), fi_upd_w_smem(), st, pdl, h->S, Pd, Dw,
                   reg, rs - reg));
        h->launches++;
      }
      if (split > rs && h->fi_tc >= 4) {
        FaninDev Dk = h->fi;
        if (!h->fi_maps) Dk.src_pos = nullptr;
        CK(launchx(h->fi_chain ? k_fi_upd_kc<true> : k_fi_upd_kc<false>, dim3(split - rs), dim3(256),
                   fi_upd_kc_smem(), st, pdl, h->S, Pd, Dk, rs));
        h->launches++;
      } else if (split > rs && h->fi_tc == 2) {
        k_fi_upd_tc<<<split - rs, 256, fi_upd_tc_smem(h->fi_smax[l]), st>>>(h->S, Pd, h->fi, rs, h->fi_smax[l]);
        h->launches++;
      } else if (split > rs) {
        const int nsm2 = split - rs;
        k_fi_upd<<<nsm2, 256, sm, st>>>(h->S, Pd, h->fi, rs, h->fi_smax[l], h->fi_mmax[l]);
        h->launches++;
      }
      if (nbig && h->fi_tc == 3) {
        if (h->fi_chain) k_fi_upd_kc<true><<<nbig, 256, fi_upd_kc_smem(), st>>>(h->S, Pd, h->fi, split);
        else k_fi_upd_kc<false><<<nbig, 256, fi_upd_kc_smem(), st>>>(h->S, Pd, h->fi, split);
        h->launches++;
      } else if (nbig && h->fi_tc == 1) {
        k_fi_upd_tc<<<nbig, 256, fi_upd_tc_smem(h->fi_smax[l]), st>>>(h->S, Pd, h->fi, split, h->fi_smax[l]);
        h->launches++;
      }
      if (sideB) {
        int rc = join();
        if (rc) return rc;
      }
    }
  }
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_upload_fanin_maps(hy_handle *h, int64_t nsrc, int64_t npos, const int64_t *poff,
                         const int8_t *pos, const int64_t *vb, const int32_t *vW, const int32_t *qb,
                         const int32_t *m) {
  if (!h || !h->uploaded || !h->fanin_ok) return fail(HY_INVALID_ARGUMENT, "fan-in plan not uploaded");
  drop_graph(h);
  if (nsrc < 0 || npos < 0 || (nsrc && (!poff || !vb || !vW || !qb || !m)) || (npos && !pos))
    return fail(HY_INVALID_ARGUMENT, "null source-map arrays");
  // the maps index the uploaded plan's source records one to one, and poff[nsrc]
  // bounds every position the update kernels read
  if (nsrc != h->fi_nsrc)
    return fail(HY_INVALID_ARGUMENT, "source-map count differs from the uploaded fan-in plan");
  if (nsrc && (poff[0] != 0 || poff[nsrc] != npos))
    return fail(HY_INVALID_ARGUMENT, "source-map offsets do not span the position array");
  CK(cudaSetDevice(h->device));
  FaninDev &D = h->fi;
  int64_t *p64;
  int32_t *p32;
  int8_t *p8;
  UPF(&p64, poff, nsrc + 1); D.src_poff = p64;
  UPF(&p8, pos, npos); D.src_pos = p8;
  UPF(&p64, vb, nsrc); D.src_vb = p64;
  UPF(&p32, vW, nsrc); D.src_vW = p32;
  UPF(&p32, qb, nsrc); D.src_qb = p32;
  UPF(&p32, m, nsrc); D.src_m = p32;
  {   // per item: the tile columns any of its sources touches (compact column space)
    const int64_t ni = h->fi_up.empty() ? 0 : h->fi_up.back();
    uint64_t *mk = nullptr;
    CK(cudaMalloc((void **)&mk, sizeof(uint64_t) * (ni > 0 ? ni : 1)));
    h->fi_allocs.push_back(mk);
    if (ni > 0) {
      k_item_mask<<<(unsigned)std::min<int64_t>((ni + 255) / 256, 4096), 256>>>(D, ni, mk);
      CK(cudaGetLastError());
      CK(cudaDeviceSynchronize());
    }
    D.up_mask = mk;
  }
  return HY_OK;
}

int hy_upload_hub_programs(hy_handle *h, const hy_row_programs *d) {
  if (!h || !h->uploaded || !d) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded / null");
  drop_graph(h);
  CK(cudaSetDevice(h->device));
  for (void *p : h->hub1_allocs) cudaFree(p);
  h->hub1_allocs.clear();
  h->hub1_ok = false;
  const int64_t nn = h->S.nn;
  DevProg &R = h->prog1;
  std::vector<int32_t> hub_base(nn, -1);
  std::vector<int64_t> first(nn + 1);
  CK(cudaMemcpy(first.data(), h->S.first, sizeof(int64_t) * (nn + 1), cudaMemcpyDeviceToHost));
  int32_t hr = 0;
  for (int64_t u = 0; u < nn; ++u)
    if (d->node_hub[u]) {
      if (first[u + 1] - first[u] != 1) return fail(HY_INVALID_ARGUMENT, "single-path hub must be a row");
      hub_base[u] = hr++;
    }
  if (hr != d->nhubrows) return fail(HY_INVALID_ARGUMENT, "hub row count mismatch");
  if (hr == 0) return HY_OK;
  int32_t *p32;
  int64_t *p64;
  UPH(&p32, hub_base.data(), nn); R.hub_base = p32;
  UPH(&p64, d->hrow_lev, d->nhubrows + 1); R.hrow_lev = p64;
  UPH(&p64, d->lev_wi, d->nlev + 1); R.lev_wi = p64;
  UPH(&p32, d->wi_p, d->nwi); R.wi_p = p32;
  UPH(&p64, d->wi_kd, d->nwi); R.wi_kd = p64;
  UPH(&p64, d->wi_y0, d->nwi); R.wi_y0 = p64;
  UPH(&p64, d->wi_y1, d->nwi); R.wi_y1 = p64;
  UPH(&p32, d->wi_slot, d->nwi); R.wi_slot = p32;
  UPH(&p64, d->lev_sp, d->nlev + 1); R.lev_sp = p64;
  UPH(&p32, d->sp_p, d->nsp); R.sp_p = p32;
  UPH(&p64, d->sp_kd, d->nsp); R.sp_kd = p64;
  UPH(&p32, d->sp_s0, d->nsp); R.sp_s0 = p32;
  UPH(&p32, d->sp_n, d->nsp); R.sp_n = p32;
  UPH(&p32, d->pred_p, d->npred); R.pred_p = p32;
  UPH(&p64, d->pred_u, d->npred); R.pred_u = p64;
  h->hub1_slots = (int)(d->max_slots > 0 ? d->max_slots : 1);
  // per factorization level: hub rows out of the row list
  Plan &pl = h->fplan;
  std::vector<int32_t> rows(pl.rptr[pl.nlev]);
  if (!rows.empty())
    CK(cudaMemcpy(rows.data(), pl.d_rows, sizeof(int32_t) * rows.size(), cudaMemcpyDeviceToHost));
  std::vector<int32_t> keep, hubs;
  std::vector<int64_t> rptr(pl.nlev + 1, 0);
  h->hub1_ptr.assign(pl.nlev + 1, 0);
  for (int l = 0; l < pl.nlev; ++l) {
    for (int64_t k = pl.rptr[l]; k < pl.rptr[l + 1]; ++k) (d->node_hub[rows[k]] ? hubs : keep).push_back(rows[k]);
    rptr[l + 1] = (int64_t)keep.size();
    h->hub1_ptr[l + 1] = (int64_t)hubs.size();
  }
  pl.rptr = rptr;
  UPH(&pl.d_rows, keep.data(), keep.size());
  UPH(&h->d_hub1, hubs.data(), hubs.size());
  h->hub1_ok = true;
  return HY_OK;
}


// Level fan-in as one CUDA graph per handle: the launch sequence depends only on the
// uploaded plan and the options (all per-call pointers are read from the handle's
// device-resident CallP), so it is captured once and replayed; an option change or
// a new plan drops it.  Pull-row scratch is sized before capture (no allocation
// inside a capture).

static int fanin_scratch(hy_handle *h) {
  int64_t need = 0;
  for (size_t l = 0; l + 1 < h->fi_hub.size(); ++l)
    need = std::max<int64_t>(need, (h->fi_hub[l + 1] - h->fi_hub[l]) * (int64_t)h->hub1_slots);
  if (need > h->hub1_scratch_cap) {
    if (h->d_hub1_scratch) CK(cudaFree(h->d_hub1_scratch));
    h->d_hub1_scratch = nullptr;
    CK(cudaMalloc((void **)&h->d_hub1_scratch, sizeof(double) * need));
    h->hub1_scratch_cap = need;
  }
  return HY_OK;
}

static int run_fanin_graph(hy_handle *h, cudaStream_t st) {
  cudaGraphExec_t &fi_exec = h->fi_exec2[h->cur_refactor];
  int64_t &fi_graph_launches = h->fi_graph_launches2[h->cur_refactor];
  if (!fi_exec) {
    int rc = fanin_scratch(h);
    if (rc) return rc;
    if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
    if (!h->fi_side) {   // the fork/join stream and events exist before the capture starts
      CK(cudaStreamCreateWithFlags(&h->fi_side, cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&h->fi_ev_lu, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&h->fi_ev_pt, cudaEventDisableTiming));
    }
    const int64_t l0 = h->launches;
    CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
    rc = run_fanin(h, h->d_callp, h->cap_stream);
    cudaGraph_t g = nullptr;
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    fi_graph_launches = h->launches - l0;
    h->launches = l0;
    if (rc) {
      if (g) cudaGraphDestroy(g);
      return rc;
    }
    if (e != cudaSuccess) return fail(HY_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(e));
    e = cudaGraphInstantiate(&fi_exec, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) {
      fi_exec = nullptr;
      return fail(HY_CUDA_ERROR, std::string("graph instantiate: ") + cudaGetErrorString(e));
    }
  }
  CK(cudaGraphLaunch(fi_exec, st));
  h->launches += fi_graph_launches;
  return HY_OK;
}

static int run_factor(hy_handle *h, const double *d_avals, double eps, const hy_factors *prior,
                      hy_factors *out, cudaStream_t st) {
  if (!h || !h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded");
  if (!d_avals || !out || !out->d_values || !out->d_inner_perm || !out->d_anorm || !out->d_status)
    return fail(HY_INVALID_ARGUMENT, "null buffer");
  if (prior && (!prior->d_inner_perm || !prior->d_anorm)) return fail(HY_INVALID_ARGUMENT, "null prior buffer");
  if (eps < 0.0 || eps >= 1.0) return fail(HY_INVALID_ARGUMENT, "perturbation_epsilon outside [0,1)");
  CK(cudaSetDevice(h->device));
  CallP P{};
  P.F = out->d_values;
  P.A = d_avals;
  P.iperm = out->d_inner_perm;
  P.anorm = out->d_anorm;
  P.eps = eps;
  P.status = out->d_status;
  P.pert_rows = out->d_pert_rows;
  P.pert_vals = out->d_pert_vals;
  P.pert_cap = out->d_pert_rows && out->d_pert_vals ? out->pert_cap : 0;
  P.refactor = prior ? 1 : 0;
  P.iperm_prior = prior ? prior->d_inner_perm : nullptr;
  P.anorm_prior = prior ? prior->d_anorm : nullptr;
  // SPEC dispatch: kernel_mode is the maximum tier; on the
  // device the ROWROW tier is the row-row operation order in every update kernel
  const int mode = h->kmode >= 0 ? h->kmode : h->mode_an;
  P.chain = mode == HY_ROWROW;
  if (h->fi_chain != P.chain) {     // the DMMA update kernels are instantiated per order
    drop_graph(h);
    h->fi_chain = P.chain;
  }
  h->S.mode = mode;                 // row path: per-(target, source) dispatch by mode
  out->kernel_mode = mode;
  if (!h->d_callp) CK(cudaMalloc((void **)&h->d_callp, sizeof(CallP)));
  const CallP *Pd = h->d_callp;
  // stream-ordered: the previous call's kernels have read their CallP before this
  // write runs (one stream per handle, include/hylu_b200.h)
  k_call_set<<<1, 1, 0, st>>>(h->d_callp, P);
  const int pb = (int)std::min<int64_t>(h->sm_count * 8, (h->stored / 2 + 255) / 256 + 1);
  k_call_prep<<<h->fanin_ok ? pb : (h->S.n + 255) / 256 + 1, 256, 0, st>>>(Pd, (int)h->S.n, h->stored,
                                                                         h->fanin_ok ? 1 : 0);
  k_anorm_p<<<296, 256, 0, st>>>(Pd, h->S.scale, h->S.nnz);
  h->launches += 3;
  h->cur_refactor = prior ? 1 : 0;
  if (h->fanin_ok) return h->use_graphs ? run_fanin_graph(h, st) : run_fanin(h, Pd, st);
  const Plan &pl = h->fplan;
  if (h->slab_ok) {
    h->slab_epoch++;
    CK(cudaMemsetAsync(h->d_slab_counters, 0, sizeof(int) * (pl.nlev + 1), st));
  }
  for (int l = 0; l < pl.nlev; ++l) {
    const int nr = (int)(pl.rptr[l + 1] - pl.rptr[l]);
    const int ns = (int)(pl.sptr[l + 1] - pl.sptr[l]);
    if (nr) {
      k_rows<<<(nr + 3) / 4, 128, 0, st>>>(h->S, Pd, pl.d_rows + pl.rptr[l], nr);
      h->launches++;
    }
    const int nh1 = h->hub1_ok ? (int)(h->hub1_ptr[l + 1] - h->hub1_ptr[l]) : 0;
    if (nh1) {
      const int64_t need = (int64_t)nh1 * h->hub1_slots;
      if (need > h->hub1_scratch_cap) {
        if (h->d_hub1_scratch) CK(cudaFree(h->d_hub1_scratch));
        h->d_hub1_scratch = nullptr;
        CK(cudaMalloc((void **)&h->d_hub1_scratch, sizeof(double) * need));
        h->hub1_scratch_cap = need;
      }
      k_hub1<<<nh1, 1024, 0, st>>>(h->S, Pd, h->prog1, h->d_hub1 + h->hub1_ptr[l], h->d_hub1_scratch,
                                   h->hub1_slots);
      h->launches++;
    }
    if (ns && h->slab_ok) {
      const int nsl = (int)(h->slab_lptr[l + 1] - h->slab_lptr[l]);
      const size_t smem = slab_smem_bytes(h->slab_smax[l], h->slab_mmax[l], h->slab_swmax[l], h->slab_accmax[l]);
      k_slab<<<nsl, 256, smem, st>>>(h->S, Pd, h->slab, (int)h->slab_lptr[l], h->d_slab_counters + l,
                                     h->d_dep_flags, h->d_lu_flags, h->slab_epoch, h->slab_smax[l],
                                     h->slab_mmax[l], h->slab_swmax[l], h->slab_accmax[l]);
      h->launches++;
      if (!prior) {
        dim3 g(ns, 4);
        k_lperm<<<g, 256, 0, st>>>(h->S, Pd, pl.d_sns + pl.sptr[l], ns);
        h->launches++;
      }
    } else if (ns) {
      k_sn<<<ns, 256, h->sn_smem, st>>>(h->S, Pd, pl.d_sns + pl.sptr[l]);
      h->launches++;
    }
  }
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_factorize(hy_handle *h, const double *d_avals, double eps, hy_factors *out,
                 uintptr_t stream) {
  return run_factor(h, d_avals, eps, nullptr, out, (cudaStream_t)stream);
}

int hy_refactorize(hy_handle *h, const double *d_avals, double eps, const hy_factors *prior,
                   hy_factors *out, uintptr_t stream) {
  if (!prior || !prior->d_inner_perm || !prior->d_anorm)
    return fail(HY_INVALID_ARGUMENT, "refactorize needs prior factors");
  return run_factor(h, d_avals, eps, prior, out, (cudaStream_t)stream);
}


int hy_upload_matrix(hy_handle *h, const int64_t *row_ptr, const int32_t *col_idx) {
  if (!h || !h->uploaded || !row_ptr || !col_idx) return fail(HY_INVALID_ARGUMENT, "null handle/arrays");
  const int64_t n = h->S.n;
  if (row_ptr[0] != 0 || row_ptr[n] != h->S.nnz) return fail(HY_DIMENSION_MISMATCH, "row_ptr does not match nnz");
  CK(cudaSetDevice(h->device));
  if (h->d_arow) CK(cudaFree(h->d_arow));
  if (h->d_acol) CK(cudaFree(h->d_acol));
  h->d_arow = nullptr;
  h->d_acol = nullptr;
  CK(cudaMalloc((void **)&h->d_arow, sizeof(int64_t) * (n + 1)));
  CK(cudaMalloc((void **)&h->d_acol, sizeof(int32_t) * (h->S.nnz > 0 ? h->S.nnz : 1)));
  CK(cudaMemcpy(h->d_arow, row_ptr, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice));
  if (h->S.nnz > 0)
    CK(cudaMemcpy(h->d_acol, col_idx, sizeof(int32_t) * h->S.nnz, cudaMemcpyHostToDevice));
  return HY_OK;
}

int hy_residual(hy_handle *h, const double *d_avals, const double *d_x, const double *d_b, double *d_r,
                double *d_berr, uintptr_t stream) {
  if (!h || !h->d_arow) return fail(HY_INVALID_ARGUMENT, "matrix pattern not uploaded");
  if (!d_avals || !d_x || !d_b || !d_berr) return fail(HY_INVALID_ARGUMENT, "null buffer");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(d_berr, 0, sizeof(double), st));
  const int n = h->S.n;
  const int grid = (n + 255) / 256 < h->sm_count * 8 ? (n + 255) / 256 : h->sm_count * 8;
  k_resid_berr<<<grid > 0 ? grid : 1, 256, 0, st>>>(n, h->d_arow, h->d_acol, d_avals, d_x, d_b, d_r,
                                                    reinterpret_cast<unsigned long long *>(d_berr));
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_axpy(hy_handle *h, double *d_x, const double *d_dx, uintptr_t stream) {
  if (!h || !d_x || !d_dx) return fail(HY_INVALID_ARGUMENT, "null buffer");
  CK(cudaSetDevice(h->device));
  const int n = h->S.n;
  k_axpy1<<<(n + 255) / 256, 256, 0, (cudaStream_t)stream>>>(n, d_x, d_dx);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_upload_partition(hy_handle *h, const hy_partition_desc *d) {
  if (!h || !h->uploaded || !d) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded / null");
  if (d->nfwd < 0 || d->nbwd < 0 || d->nitems < 0 || (d->nfwd && !d->fwd) || (d->nbwd && !d->bwd) ||
      (d->nitems && !d->items))
    return fail(HY_INVALID_ARGUMENT, "bad partition arrays");
  for (int dir = 0; dir < 2; ++dir) {
    const int64_t k = dir ? d->nbwd : d->nfwd;
    const int64_t *L = dir ? d->bwd : d->fwd;
    for (int64_t q = 0; q < k; ++q) {
      const int64_t kind = L[6 * q], lo = L[6 * q + 2], hi = L[6 * q + 3], off = L[6 * q + 4],
                    cnt = L[6 * q + 5];
      const int64_t span = kind == 0 ? 2 * cnt : cnt;
      if (kind < 0 || kind > 4 || kind == 2 || lo < 0 || hi > h->S.n || lo > hi || off < 0 || cnt < 0 ||
          off + span > d->nitems)
        return fail(HY_INVALID_ARGUMENT, "partition launch out of range");
    }
  }
  CK(cudaSetDevice(h->device));
  if (h->d_ms_items) CK(cudaFree(h->d_ms_items));
  h->d_ms_items = nullptr;
  if (d->nitems) {
    CK(cudaMalloc((void **)&h->d_ms_items, sizeof(int32_t) * d->nitems));
    CK(cudaMemcpy(h->d_ms_items, d->items, sizeof(int32_t) * d->nitems, cudaMemcpyHostToDevice));
  }
  h->ms_fwd.assign(d->fwd, d->fwd + 6 * d->nfwd);
  h->ms_bwd.assign(d->bwd, d->bwd + 6 * d->nbwd);
  return HY_OK;
}

int hy_solve_multi(hy_handle *h, const hy_factors *f, int64_t nrhs, const double *d_B, double *d_X,
                   uintptr_t stream) {
  if (!h || !h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded");
  if (!f || !f->d_values || !f->d_inner_perm || !d_B || !d_X) return fail(HY_INVALID_ARGUMENT, "null buffer");
  if (nrhs <= 0 || nrhs > (1 << 20)) return fail(HY_INVALID_ARGUMENT, "nrhs outside [1, 2^20]");
  if (h->ms_fwd.empty() && h->ms_bwd.empty() && h->S.n > 0)
    return fail(HY_INVALID_ARGUMENT, "solve partition not uploaded");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t need = (int64_t)h->S.n * nrhs;
  if (need > h->my_cap) {
    if (h->d_my) CK(cudaFree(h->d_my));
    h->d_my = nullptr;
    CK(cudaMalloc((void **)&h->d_my, sizeof(double) * (need > 0 ? need : 1)));
    h->my_cap = need;
  }
  const int gb = (int)std::min<int64_t>((need + 255) / 256 + 1, (int64_t)h->sm_count * 16);
  k_mbhat<<<gb, 256, 0, st>>>(h->S, f->d_inner_perm, d_B, h->d_my, (int)nrhs);
  h->launches++;
  for (int dir = 0; dir < 2; ++dir) {
    const std::vector<int64_t> &L = dir ? h->ms_bwd : h->ms_fwd;
    for (size_t q = 0; q + 5 < L.size(); q += 6) {
      const int kind = (int)L[q], seq = (int)L[q + 1], lo = (int)L[q + 2], hi = (int)L[q + 3];
      const int cnt = (int)L[q + 5];
      if (!cnt) continue;
      if (kind == 3 || kind == 4) {   // level form: CTA per wide row / per supernode
        const dim3 g((unsigned)cnt, (unsigned)((nrhs + 31) / 32));
        if (kind == 3)
          k_msolve_long<<<g, 256, 0, st>>>(h->S, f->d_values, h->d_ms_items + L[q + 4], dir == 0, h->d_my,
                                           (int)nrhs);
        else
          k_msolve_sn<<<g, 512, 0, st>>>(h->S, f->d_values, h->d_ms_items + L[q + 4], dir == 0, h->d_my,
                                         (int)nrhs);
        h->launches++;
        continue;
      }
      const int blocks = seq ? 1 : (cnt + 3) / 4;
      k_msolve<<<blocks, 128, 0, st>>>(h->S, f->d_values, kind, seq, lo, hi, h->d_ms_items + L[q + 4], cnt,
                                       dir == 0, h->d_my, (int)nrhs);
      h->launches++;
    }
  }
  k_mxout<<<gb, 256, 0, st>>>(h->S, h->d_my, d_X, (int)nrhs);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_set_kernel_mode(hy_handle *h, int mode) {
  if (!h || !h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded");
  if (mode < -1 || mode > 2) return fail(HY_INVALID_ARGUMENT, "kernel mode outside {-1, 0, 1, 2}");
  h->kmode = mode;
  return HY_OK;
}

int hy_residual_batched(hy_handle *h, int64_t B, const double *d_vals, const double *d_x,
                        const double *d_b, double *d_r, double *d_berr, const int32_t *d_mask,
                        uintptr_t stream) {
  if (!h || !h->d_arow) return fail(HY_INVALID_ARGUMENT, "matrix pattern not uploaded");
  if (B <= 0 || B > 65535 || !d_vals || !d_x || !d_b || !d_berr)
    return fail(HY_INVALID_ARGUMENT, "null buffer or batch size outside [1, 65535]");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  CK(cudaMemsetAsync(d_berr, 0, sizeof(double) * B, st));
  const int n = h->S.n;
  const int gx = (n + 255) / 256 < 64 ? (n + 255) / 256 : 64;
  k_resid_berr_b<<<dim3(gx > 0 ? gx : 1, (unsigned)B), 256, 0, st>>>(
      n, h->S.nnz, h->d_arow, h->d_acol, d_vals, d_x, d_b, d_r,
      reinterpret_cast<unsigned long long *>(d_berr), d_mask);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_axpy_batched(hy_handle *h, int64_t B, double *d_y, const double *d_x, const double *d_dx,
                    const int32_t *d_mask, uintptr_t stream) {
  if (!h || !d_y || !d_x) return fail(HY_INVALID_ARGUMENT, "null buffer");
  if (B <= 0 || B > 65535) return fail(HY_INVALID_ARGUMENT, "batch size outside [1, 65535]");
  CK(cudaSetDevice(h->device));
  const int n = h->S.n;
  const int gx = (n + 255) / 256 < 64 ? (n + 255) / 256 : 64;
  k_axpy_b<<<dim3(gx > 0 ? gx : 1, (unsigned)B), 256, 0, (cudaStream_t)stream>>>(n, d_y, d_x, d_dx,
                                                                                   d_mask);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

// Substitution levels as one CUDA graph per handle (captured on first use): the
// level kernels read the factor-value pointer from the handle's device slot, which
// k_ptr_set fills per call; b̂ and the output permutation run outside the graph.
static int solve_levels(hy_handle *h, cudaStream_t st) {
  for (int dir = 0; dir < 2; ++dir) {
    const Plan &pl = dir == 0 ? h->fplan : h->bplan;
    const SolvePlan &sp = dir == 0 ? h->fsolve : h->bsolve;
    for (int l = 0; l < pl.nlev; ++l) {
      const int c = (int)(pl.aptr[l + 1] - pl.aptr[l]);
      const int nch = (int)(sp.cptr[l + 1] - sp.cptr[l]);
      if (nch) {
        CK(launchx(k_solve_part, dim3(nch), dim3(256), 0, st, h->use_pdl, h->S, (const double *const *)h->d_fptr,
                   (const SolveChunk *)(sp.d_chunks + sp.cptr[l]), nch, (const double *)h->d_y,
                   h->d_solve_scratch, (int)(dir == 0)));
        h->launches++;
      }
      CK(launchx(dir == 0 ? k_fwd_fin : k_bwd_fin, dim3((c + 3) / 4), dim3(128), 0, st, h->use_pdl, h->S,
                 (const double *const *)h->d_fptr, (const SolveRec *)(sp.d_rec + pl.aptr[l]), c,
                 (const double *)h->d_solve_scratch, h->d_y));
      h->launches++;
    }
  }
  return HY_OK;
}

int hy_solve(hy_handle *h, const hy_factors *f, const double *d_b, double *d_x, uintptr_t stream) {
  if (!h || !h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded");
  if (!f || !f->d_values || !f->d_inner_perm || !d_b || !d_x) return fail(HY_INVALID_ARGUMENT, "null buffer");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int n = h->S.n;
  if (!h->d_fptr) CK(cudaMalloc((void **)&h->d_fptr, sizeof(double *)));
  k_ptr_set<<<1, 1, 0, st>>>(h->d_fptr, f->d_values);
  k_bhat<<<(n + 255) / 256, 256, 0, st>>>(h->S, f->d_inner_perm, d_b, h->d_y);
  h->launches += 2;
  if (h->use_graphs) {
    if (!h->sv_exec) {
      if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
      const int64_t l0 = h->launches;
      CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
      solve_levels(h, h->cap_stream);
      cudaGraph_t g = nullptr;
      cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
      h->sv_graph_launches = h->launches - l0;
      h->launches = l0;
      if (e != cudaSuccess) return fail(HY_CUDA_ERROR, std::string("graph capture: ") + cudaGetErrorString(e));
      e = cudaGraphInstantiate(&h->sv_exec, g, 0);
      cudaGraphDestroy(g);
      if (e != cudaSuccess) {
        h->sv_exec = nullptr;
        return fail(HY_CUDA_ERROR, std::string("graph instantiate: ") + cudaGetErrorString(e));
      }
    }
    CK(cudaGraphLaunch(h->sv_exec, st));
    h->launches += h->sv_graph_launches;
  } else {
    solve_levels(h, st);
  }
  k_xout<<<(n + 255) / 256, 256, 0, st>>>(h->S, h->d_y, d_x);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_upload_row_programs(hy_handle *h, const hy_row_programs *d) {
  if (!h || !h->uploaded || !d) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded / null");
  CK(cudaSetDevice(h->device));
  CK(cudaDeviceSynchronize());
  for (void *p : h->prog_allocs) cudaFree(p);
  h->prog_allocs.clear();
  h->prog_ok = false;
  const int64_t n = h->S.n, nn = h->S.nn;
  DevProg &R = h->prog;
  int64_t *p64;
  int32_t *p32;
  UPP(&p64, d->row_ptr, n + 1); R.row_ptr = p64;
  UPP(&p32, d->st_p, d->nsteps); R.st_p = p32;
  UPP(&p32, d->st_j, d->nsteps); R.st_j = p32;
  UPP(&p64, d->st_src, d->nsteps); R.st_src = p64;
  UPP(&p32, d->st_cnt, d->nsteps); R.st_cnt = p32;
  UPP(&p64, d->st_rel, d->nsteps); R.st_rel = p64;
  {   // rel padded by 4 entries: the pipeline's aligned bulk copy of a window may read past the end
    std::vector<int32_t> relp(d->rel, d->rel + d->nrel);
    relp.resize(d->nrel + 4, 0);
    UPP(&p32, relp.data(), d->nrel + 4); R.rel = p32;
  }
  {   // packed step records + per-node program windows (k_bt_pipe2 stages them in shared memory)
    const int64_t ns = d->nsteps;
    bool ok = h->stored < ((int64_t)1 << 31);
    std::vector<StepRec> rec(ns + 1);
    for (int64_t k = 0; k < ns && ok; ++k) {
      rec[k].p = d->st_p[k];
      rec[k].src = (int32_t)d->st_src[k];
      rec[k].j = d->st_j[k];
      if (d->st_cnt[k] > 32767) ok = false;
      rec[k].cnt = (int16_t)d->st_cnt[k];
      rec[k].rl = 0;
    }
    h->h_win.assign(nn, {0, 0, 0, 0});
    for (int64_t u = 0; u < nn && ok; ++u) {
      const int64_t k0 = d->row_ptr[h->h_first[u]], k1 = d->row_ptr[h->h_first[u + 1]];
      if (k1 <= k0) continue;
      const int64_t rel0 = d->st_rel[k0];
      const int64_t nrel = d->st_rel[k1 - 1] + d->st_cnt[k1 - 1] - rel0;
      if (k1 - k0 > PIPE_REC_CAP || nrel + 6 > PIPE_REL_CAP) {
        // too large for one window: stage row by row when every row fits
        bool rows_ok = true;
        for (int64_t i = h->h_first[u]; i < h->h_first[u + 1] && rows_ok; ++i) {
          const int64_t a = d->row_ptr[i], b = d->row_ptr[i + 1];
          if (b > a && (b - a > PIPE_REC_CAP || d->st_rel[b - 1] + d->st_cnt[b - 1] - d->st_rel[a] + 6 > PIPE_REL_CAP))
            rows_ok = false;
        }
        if (!rows_ok) continue;   // global step arrays
        for (int64_t i = h->h_first[u]; i < h->h_first[u + 1]; ++i)
          for (int64_t k = d->row_ptr[i]; k < d->row_ptr[i + 1]; ++k)
            rec[k].rl = (int16_t)(d->st_rel[k] - d->st_rel[d->row_ptr[i]]);
        h->h_win[u] = {0, 0, 0, -1};
        continue;
      }
      for (int64_t k = k0; k < k1; ++k) rec[k].rl = (int16_t)(d->st_rel[k] - rel0);
      h->h_win[u] = {rel0, k0, k1 - k0, nrel};
    }
    R.st_rec = nullptr;
    if (ok) {
      StepRec *q;
      UPP(&q, rec.data(), ns + 1);
      R.st_rec = q;
    }
    std::vector<int64_t> row_rel(n + 1);
    for (int64_t i = 0; i <= n; ++i) row_rel[i] = d->row_ptr[i] < ns ? d->st_rel[d->row_ptr[i]] : d->nrel;
    UPP(&p64, row_rel.data(), n + 1); R.row_rel = p64;
  }
  std::vector<int32_t> hub_base(nn, -1);
  std::vector<int64_t> first(nn + 1);
  CK(cudaMemcpy(first.data(), h->S.first, sizeof(int64_t) * (nn + 1), cudaMemcpyDeviceToHost));
  int32_t hr = 0;
  for (int64_t u = 0; u < nn; ++u)
    if (d->node_hub[u]) {
      hub_base[u] = hr;
      hr += (int32_t)(first[u + 1] - first[u]);
    }
  if (hr != d->nhubrows) return fail(HY_INVALID_ARGUMENT, "hub row count mismatch");
  UPP(&p32, hub_base.data(), nn); R.hub_base = p32;
  UPP(&p64, d->hrow_lev, d->nhubrows + 1); R.hrow_lev = p64;
  UPP(&p64, d->lev_ptr, d->nlev + 1); R.lev_ptr = p64;
  UPP(&p32, d->hpos, d->nhpos); R.hpos = p32;
  UPP(&p64, d->hdiv, d->nhpos); R.hdiv = p64;
  UPP(&p64, d->hpp, d->nhpos + 1); R.hpp = p64;
  UPP(&p32, d->pred_p, d->npred); R.pred_p = p32;
  UPP(&p64, d->pred_u, d->npred); R.pred_u = p64;
  UPP(&p64, d->lev_wi, d->nlev + 1); R.lev_wi = p64;
  UPP(&p32, d->wi_p, d->nwi); R.wi_p = p32;
  UPP(&p64, d->wi_kd, d->nwi); R.wi_kd = p64;
  UPP(&p64, d->wi_y0, d->nwi); R.wi_y0 = p64;
  UPP(&p64, d->wi_y1, d->nwi); R.wi_y1 = p64;
  UPP(&p32, d->wi_slot, d->nwi); R.wi_slot = p32;
  UPP(&p64, d->lev_sp, d->nlev + 1); R.lev_sp = p64;
  UPP(&p32, d->sp_p, d->nsp); R.sp_p = p32;
  UPP(&p64, d->sp_kd, d->nsp); R.sp_kd = p64;
  UPP(&p32, d->sp_s0, d->nsp); R.sp_s0 = p32;
  UPP(&p32, d->sp_n, d->nsp); R.sp_n = p32;
  {
    longlong4 *q;
    UPP(&q, (const longlong4 *)d->node_rec, nn); R.node_rec = q;
    UPP(&q, (const longlong4 *)d->row_rec, n); R.row_rec = q;
    h->h_row_rec.assign((const longlong4 *)d->row_rec, (const longlong4 *)d->row_rec + n);
  }
  free_segments(h);
  h->max_slots = (int)d->max_slots;
  h->level_ws.assign(d->level_ws, d->level_ws + h->fplan.nlev);
  // per level split: non-hub nodes / hub nodes
  const Plan &pl = h->fplan;
  std::vector<int32_t> all(pl.aptr[pl.nlev]);
  if (!all.empty())
    CK(cudaMemcpy(all.data(), pl.d_all, sizeof(int32_t) * all.size(), cudaMemcpyDeviceToHost));
  std::vector<int32_t> rows, hubs;
  h->bl_rptr.assign(pl.nlev + 1, 0);
  h->bl_hptr.assign(pl.nlev + 1, 0);
  for (int l = 0; l < pl.nlev; ++l) {
    for (int64_t k = pl.aptr[l]; k < pl.aptr[l + 1]; ++k)
      (d->node_hub[all[k]] ? hubs : rows).push_back(all[k]);
    h->bl_rptr[l + 1] = (int64_t)rows.size();
    h->bl_hptr[l + 1] = (int64_t)hubs.size();
  }
  UPP(&h->d_bl_rows, rows.data(), rows.size());
  UPP(&h->d_bl_hubs, hubs.data(), hubs.size());
  h->prog_ok = true;
  return HY_OK;
}

static int batch_prepare(hy_handle *h, int64_t B) {
  const int G = (int)((B + 63) / 64) * 2;   // even group count: pair mode's padding group
  const int64_t need = (int64_t)G * 32 * h->stored;
  if (need > h->bf_cap) {
    if (h->d_bf) CK(cudaFree(h->d_bf));
    h->d_bf = nullptr;
    CK(cudaMalloc((void **)&h->d_bf, sizeof(double) * need));
    h->bf_cap = need;
  }
  const int64_t needy = (int64_t)G * 32 * h->S.n;
  if (needy > h->by_cap) {
    if (h->d_by) CK(cudaFree(h->d_by));
    if (h->d_bri) CK(cudaFree(h->d_bri));
    h->d_by = nullptr;
    h->d_bri = nullptr;
    CK(cudaMalloc((void **)&h->d_by, sizeof(double) * needy));
    CK(cudaMalloc((void **)&h->d_bri, sizeof(double) * needy));
    h->by_cap = needy;
  }
  return HY_OK;
}

int hy_refactorize_batched(hy_handle *h, int64_t B, const double *d_vals, double eps,
                           const hy_factors *prior, int32_t *d_npert, const double *d_b_fuse,
                           uintptr_t stream) {
  if (!h || !h->uploaded) return fail(HY_INVALID_ARGUMENT, "symbolic not uploaded");
  if (B <= 0 || !d_vals || !prior || !d_npert)
    return fail(HY_INVALID_ARGUMENT, "null buffer or empty batch");
  if (!h->prog_ok) return fail(HY_INVALID_ARGUMENT, "row programs not uploaded");
  if (eps < 0.0 || eps >= 1.0) return fail(HY_INVALID_ARGUMENT, "perturbation_epsilon outside [0,1)");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  int rc = batch_prepare(h, B);
  if (rc) return rc;
  h->last_B = B;
  h->last_iperm = prior->d_inner_perm;
  CK(cudaMemsetAsync(d_npert, 0, sizeof(int32_t) * B, st));
  const int G = (int)((B + 31) / 32);
  BatchP P{h->d_bf, d_vals, prior->d_inner_perm, prior->d_anorm, eps, d_npert, B, h->stored, 0,
           h->d_bri};
  h->last_fused = d_b_fuse != nullptr;
  if (d_b_fuse) {
    // b̂ into Y first (coalesced transpose in source-row order); the row kernels then
    // read one line per row instead of gathering one value per instance
    if (!h->d_rowof) CK(cudaMalloc((void **)&h->d_rowof, sizeof(int32_t) * h->S.n));
    k_row_of<<<(h->S.n + 255) / 256, 256, 0, st>>>(h->S, prior->d_inner_perm, h->d_rowof);
    dim3 tg((h->S.n + 31) / 32, G);
    k_batch_bhat2<<<tg, 256, 0, st>>>(h->S, h->d_rowof, d_b_fuse, h->d_by, B);
    h->launches += 2;
    P.ypre = 1;
  }
  const int64_t nflags = (int64_t)h->S.nn * G;
  if (nflags > h->flags_cap) {
    if (h->d_flags) CK(cudaFree(h->d_flags));
    h->d_flags = nullptr;
    CK(cudaMalloc((void **)&h->d_flags, sizeof(int) * nflags));
    CK(cudaMemset(h->d_flags, 0, sizeof(int) * nflags));
    h->flags_cap = nflags;
    h->epoch = 0;
  }
  const int nl = h->fplan.nlev;
  if (h->counters_cap < nl + 2) {
    if (h->d_counters) CK(cudaFree(h->d_counters));
    CK(cudaMalloc((void **)&h->d_counters, sizeof(long long) * (nl + 2)));
    h->counters_cap = nl + 2;
  }
  CK(cudaMemsetAsync(h->d_counters, 0, sizeof(long long) * (nl + 2), st));
  h->epoch++;
  if (h->pipe_blocks == 0) {
    int per_sm = 0, sms = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_bt_pipe2, 128,
                                                     pipe_smem(h->pipe_ws)));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device));
    h->pipe_blocks = per_sm * sms;
  }
  // segments: maximal level runs without hub nodes -> one persistent launch each
  // (claim order: build_segments); hub levels -> one CTA per (hub node, group), then the
  // level's non-hub nodes
  if (h->segs_G != G) {
    int rc2 = build_segments(h, G);
    if (rc2) return rc2;
  }
  for (size_t si = 0; si < h->segs.size(); ++si) {
    const hy_handle::Seg &sg = h->segs[si];
    const int l = sg.l0;
    if (h->bl_hptr[l + 1] > h->bl_hptr[l]) {
      const int nh = (int)(h->bl_hptr[l + 1] - h->bl_hptr[l]);
      const int64_t need = (int64_t)nh * G * (h->max_slots > 0 ? h->max_slots : 1) * 32;
      if (need > h->scratch_cap) {
        if (h->d_scratch) CK(cudaFree(h->d_scratch));
        h->d_scratch = nullptr;
        CK(cudaMalloc((void **)&h->d_scratch, sizeof(double) * need));
        h->scratch_cap = need;
      }
      k_bt_hub<<<(unsigned)(nh * G), hub_threads(), hub_smem_bytes(), st>>>(h->S, P, h->prog, h->d_bl_hubs + h->bl_hptr[l], nh, G,
                                                   d_b_fuse, h->d_by, h->d_scratch, h->max_slots,
                                                   h->d_flags, h->epoch);
      h->launches++;
    }
    if (sg.ntasks) {
      int *ctr = (int *)((long long *)h->d_counters + si);
      k_bt_pipe2<<<h->pipe_blocks, 128, pipe_smem(h->pipe_ws), st>>>(
          h->S, P, h->prog, sg.d_tasks, sg.ntasks, d_b_fuse, h->d_by, ctr, h->d_flags, h->epoch, G,
          h->pipe_ws);
      h->launches++;
    }
  }
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_solve_batched(hy_handle *h, int64_t B, const double *d_b, double *d_x, uintptr_t stream) {
  if (!h || !h->uploaded || B != h->last_B || !h->d_bf)
    return fail(HY_INVALID_ARGUMENT, "no batched factors of this batch size");
  if (!d_x) return fail(HY_INVALID_ARGUMENT, "null buffer");
  if (!d_b && !h->last_fused)
    return fail(HY_INVALID_ARGUMENT, "d_b == NULL needs a refactorization with a fused rhs");
  CK(cudaSetDevice(h->device));
  cudaStream_t st = (cudaStream_t)stream;
  const int G = (int)((B + 31) / 32);
  const Plan &pl = h->fplan;
  dim3 tg((h->S.n + 31) / 32, G);
  if (d_b) {
  k_batch_bhat<<<tg, 256, 0, st>>>(h->S, h->last_iperm, d_b, h->d_by, B);
  h->launches++;
  for (int l = 0; l < pl.nlev; ++l) {
    const int c = (int)(pl.aptr[l + 1] - pl.aptr[l]);
    const int64_t tasks = (int64_t)c * G;
    k_batch_fwd<<<(unsigned)((tasks + 3) / 4), 128, 0, st>>>(h->S, h->d_bf, h->stored,
                                                           pl.d_all + pl.aptr[l], c, G, h->d_by);
    h->launches++;
  }
  }
  const Plan &bp = h->bplan;
  for (int l = 0; l < bp.nlev; ++l) {
    const int c = (int)(bp.aptr[l + 1] - bp.aptr[l]);
    const int GP = (G + 1) / 2;
    const int64_t tasks = (int64_t)c * GP;
    // narrow levels are latency chains (wider load batches), wide levels throughput-bound
    CK(launchx(tasks <= h->bwd_narrow ? k_batch_bwd2<BWD_WL> : k_batch_bwd2<BWD_W>,
               dim3((unsigned)((tasks + 3) / 4)), dim3(128), 0, st, h->use_pdl, h->S,
               (const double *)h->d_bf, h->stored, (const int32_t *)(bp.d_all + bp.aptr[l]), c, GP, h->d_by));
    h->launches++;
  }
  if (!h->d_pinv) {
    CK(cudaMalloc((void **)&h->d_pinv, sizeof(int32_t) * h->S.n));
    k_perm_inverse<<<(h->S.n + 255) / 256, 256, 0, st>>>(h->S.n, h->S.perm, h->d_pinv);
    h->launches++;
  }
  k_batch_xout2<<<tg, 256, 0, st>>>(h->S, h->d_pinv, h->d_by, d_x, B);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

int hy_refactorize_solve_batched(hy_handle *h, int64_t B, const double *d_vals, const double *d_b,
                                 double *d_x, double eps, const hy_factors *prior, int32_t *d_npert,
                                 uintptr_t stream) {
  int rc = hy_refactorize_batched(h, B, d_vals, eps, prior, d_npert, d_b, stream);
  if (rc) return rc;
  return hy_solve_batched(h, B, nullptr, d_x, stream);
}

int hy_batched_factor_values(hy_handle *h, int64_t b, double *d_out, uintptr_t stream) {
  if (!h || !h->d_bf || b < 0 || b >= h->last_B || !d_out)
    return fail(HY_INVALID_ARGUMENT, "no batched factors for this index");
  CK(cudaSetDevice(h->device));
  k_batch_extract<<<296, 256, 0, (cudaStream_t)stream>>>(h->d_bf, h->stored, b, d_out);
  h->launches++;
  CK(cudaGetLastError());
  return HY_OK;
}

}  // extern "C"
