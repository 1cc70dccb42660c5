"""ctypes binding of ``lib/libhylu_b200.so`` (C ABI: ``include/hylu_b200.h``).

PyTorch is used only for device memory and streams: every buffer handed to the
library is a CUDA tensor's ``data_ptr()``.  There is no CPU fallback: if the
library or a CUDA device is missing, constructing a ``DeviceContext`` raises.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from ._ref import errors

_LIB_PATH = os.environ.get("HYLU_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "lib", "libhylu_b200.so")
_lib = None

HY_CODES = {
    1: errors.DimensionMismatch,
    2: errors.ZeroDiagonal,
    3: errors.CycleDetected,
    4: errors.NumericBreakdown,
    5: errors.PatternMismatch,
}


class DeviceError(RuntimeError):
    """CUDA / ABI failure (HY_CUDA_ERROR, HY_INVALID_ARGUMENT)."""


class SymbolicDesc(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64), ("nnodes", ctypes.c_int64), ("nnz", ctypes.c_int64),
        ("kernel_mode", ctypes.c_int32),
        ("node_first", ctypes.c_void_p), ("node_kind", ctypes.c_void_p),
        ("colptr", ctypes.c_void_p), ("cols", ctypes.c_void_p), ("nl", ctypes.c_void_p),
        ("valoff", ctypes.c_void_p), ("dep_ptr", ctypes.c_void_p), ("deps", ctypes.c_void_p),
        ("level_ptr", ctypes.c_void_p), ("level_nodes", ctypes.c_void_p), ("nlevels", ctypes.c_int64),
        ("ulevel_ptr", ctypes.c_void_p), ("ulevel_nodes", ctypes.c_void_p), ("nulevels", ctypes.c_int64),
        ("a_row_ptr", ctypes.c_void_p), ("a_col_idx", ctypes.c_void_p), ("mrow_src", ctypes.c_void_p),
        ("colpos", ctypes.c_void_p), ("scale", ctypes.c_void_p), ("dr", ctypes.c_void_p),
        ("dc", ctypes.c_void_p), ("perm", ctypes.c_void_p),
    ]


class FactorsDesc(ctypes.Structure):
    _fields_ = [
        ("d_values", ctypes.c_void_p), ("d_inner_perm", ctypes.c_void_p), ("d_anorm", ctypes.c_void_p),
        ("d_status", ctypes.c_void_p), ("d_pert_rows", ctypes.c_void_p), ("d_pert_vals", ctypes.c_void_p),
        ("pert_cap", ctypes.c_int64), ("kernel_mode", ctypes.c_int32),
    ]


class PartitionDesc(ctypes.Structure):
    _fields_ = [("nfwd", ctypes.c_int64), ("nbwd", ctypes.c_int64), ("nitems", ctypes.c_int64),
                ("fwd", ctypes.c_void_p), ("bwd", ctypes.c_void_p), ("items", ctypes.c_void_p)]


class ProgramsDesc(ctypes.Structure):
    _fields_ = [
        ("nsteps", ctypes.c_int64), ("nrel", ctypes.c_int64), ("nhubrows", ctypes.c_int64),
        ("nlev", ctypes.c_int64), ("nhpos", ctypes.c_int64), ("npred", ctypes.c_int64),
        ("nwi", ctypes.c_int64), ("nsp", ctypes.c_int64), ("max_slots", ctypes.c_int64),
        ("row_ptr", ctypes.c_void_p), ("st_p", ctypes.c_void_p), ("st_j", ctypes.c_void_p),
        ("st_src", ctypes.c_void_p), ("st_cnt", ctypes.c_void_p), ("st_rel", ctypes.c_void_p),
        ("rel", ctypes.c_void_p), ("node_hub", ctypes.c_void_p), ("hrow_lev", ctypes.c_void_p),
        ("lev_ptr", ctypes.c_void_p), ("hpos", ctypes.c_void_p), ("hdiv", ctypes.c_void_p),
        ("hpp", ctypes.c_void_p), ("pred_p", ctypes.c_void_p), ("pred_u", ctypes.c_void_p),
        ("lev_wi", ctypes.c_void_p), ("wi_p", ctypes.c_void_p), ("wi_kd", ctypes.c_void_p),
        ("wi_y0", ctypes.c_void_p), ("wi_y1", ctypes.c_void_p), ("wi_slot", ctypes.c_void_p),
        ("lev_sp", ctypes.c_void_p), ("sp_p", ctypes.c_void_p), ("sp_kd", ctypes.c_void_p),
        ("sp_s0", ctypes.c_void_p), ("sp_n", ctypes.c_void_p),
        ("level_ws", ctypes.c_void_p), ("node_rec", ctypes.c_void_p), ("row_rec", ctypes.c_void_p),
    ]


class SlabPlanDesc(ctypes.Structure):
    _fields_ = [
        ("nslabs", ctypes.c_int64), ("nitems", ctypes.c_int64), ("ndeps", ctypes.c_int64),
        ("nlevels", ctypes.c_int64),
        ("sl_node", ctypes.c_void_p), ("sl_c0", ctypes.c_void_p), ("sl_c1", ctypes.c_void_p),
        ("sl_kind", ctypes.c_void_p), ("it_ptr", ctypes.c_void_p), ("it_k", ctypes.c_void_p),
        ("it_q0", ctypes.c_void_p), ("it_q1", ctypes.c_void_p), ("it_own", ctypes.c_void_p),
        ("dep_pb", ctypes.c_void_p), ("level_slab_ptr", ctypes.c_void_p),
        ("level_smax", ctypes.c_void_p), ("level_mmax", ctypes.c_void_p),
        ("level_swmax", ctypes.c_void_p), ("level_accmax", ctypes.c_void_p),
    ]


class FaninPlanDesc(ctypes.Structure):
    _fields_ = [
        ("nlevels", ctypes.c_int64), ("nsrc", ctypes.c_int64), ("ndeps", ctypes.c_int64),
        ("lu_ptr", ctypes.c_void_p), ("lu_nodes", ctypes.c_void_p),
        ("pt_ptr", ctypes.c_void_p), ("pt_node", ctypes.c_void_p), ("pt_c0", ctypes.c_void_p),
        ("pt_c1", ctypes.c_void_p),
        ("xp_ptr", ctypes.c_void_p), ("xp_edge", ctypes.c_void_p), ("xp_tgt", ctypes.c_void_p),
        ("lev_up", ctypes.c_void_p), ("up_t", ctypes.c_void_p), ("up_c0", ctypes.c_void_p),
        ("up_c1", ctypes.c_void_p), ("up_ptr", ctypes.c_void_p),
        ("src_k", ctypes.c_void_p), ("src_q0", ctypes.c_void_p), ("src_q1", ctypes.c_void_p),
        ("dep_pb", ctypes.c_void_p), ("level_smax", ctypes.c_void_p), ("level_mmax", ctypes.c_void_p),
        ("src_v", ctypes.c_void_p), ("src_pb", ctypes.c_void_p), ("src_tb", ctypes.c_void_p),
        ("lev_up_big", ctypes.c_void_p), ("lev_up_reg", ctypes.c_void_p),
        ("lev_up_rs", ctypes.c_void_p), ("lev_xp_big", ctypes.c_void_p),
        ("nhub", ctypes.c_int64), ("lev_hub", ctypes.c_void_p), ("hub_list", ctypes.c_void_p),
        ("nparts", ctypes.c_int64), ("up_part", ctypes.c_void_p), ("part_first", ctypes.c_void_p),
        ("part_n", ctypes.c_void_p), ("part_off", ctypes.c_void_p),
    ]


def library():
    """Load the CUDA library (building it in-tree first if it is absent)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        from . import build
        build.build_cuda()
    lib = ctypes.CDLL(_LIB_PATH)
    vp, i64, u = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64
    lib.hy_create.argtypes = [ctypes.c_int, ctypes.POINTER(vp)]
    lib.hy_destroy.argtypes = [vp]
    lib.hy_destroy.restype = None
    lib.hy_last_error.restype = ctypes.c_char_p
    lib.hy_upload_symbolic.argtypes = [vp, ctypes.POINTER(SymbolicDesc)]
    lib.hy_stored_values.argtypes = [vp]
    lib.hy_stored_values.restype = i64
    lib.hy_launch_count.argtypes = [vp]
    lib.hy_launch_count.restype = i64
    lib.hy_factorize.argtypes = [vp, vp, ctypes.c_double, ctypes.POINTER(FactorsDesc), u]
    lib.hy_refactorize.argtypes = [vp, vp, ctypes.c_double, ctypes.POINTER(FactorsDesc),
                                   ctypes.POINTER(FactorsDesc), u]
    lib.hy_solve.argtypes = [vp, ctypes.POINTER(FactorsDesc), vp, vp, u]
    lib.hy_upload_matrix.argtypes = [vp, vp, vp]
    lib.hy_residual.argtypes = [vp, vp, vp, vp, vp, vp, u]
    lib.hy_axpy.argtypes = [vp, vp, vp, u]
    lib.hy_set_kernel_mode.argtypes = [vp, ctypes.c_int]
    lib.hy_upload_partition.argtypes = [vp, ctypes.POINTER(PartitionDesc)]
    lib.hy_solve_multi.argtypes = [vp, ctypes.POINTER(FactorsDesc), i64, vp, vp, u]
    lib.hy_residual_batched.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, u]
    lib.hy_axpy_batched.argtypes = [vp, i64, vp, vp, vp, vp, u]
    lib.hy_refactorize_solve_batched.argtypes = [vp, i64, vp, vp, vp, ctypes.c_double,
                                                 ctypes.POINTER(FactorsDesc), vp, u]
    lib.hy_refactorize_batched.argtypes = [vp, i64, vp, ctypes.c_double,
                                           ctypes.POINTER(FactorsDesc), vp, vp, u]
    lib.hy_upload_row_programs.argtypes = [vp, ctypes.POINTER(ProgramsDesc)]
    lib.hy_solve_batched.argtypes = [vp, i64, vp, vp, u]
    lib.hy_batched_factor_values.argtypes = [vp, i64, vp, u]
    lib.hy_set_option.argtypes = [vp, ctypes.c_char_p, i64]
    lib.hy_upload_slab_plan.argtypes = [vp, ctypes.POINTER(SlabPlanDesc)]
    lib.hy_upload_fanin_plan.argtypes = [vp, ctypes.POINTER(FaninPlanDesc)]
    lib.hy_upload_fanin_maps.argtypes = [vp, i64, i64, vp, vp, vp, vp, vp, vp]
    lib.hy_upload_hub_programs.argtypes = [vp, ctypes.POINTER(ProgramsDesc)]
    _lib = lib
    return lib


def check(rc):
    if rc == 0:
        return
    msg = library().hy_last_error().decode(errors="replace")
    if rc in HY_CODES:
        raise HY_CODES[rc](msg)
    raise DeviceError("hylu_b200 error %d: %s" % (rc, msg))


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


class DeviceContext:
    """One handle = one device + one uploaded symbolic structure."""

    def __init__(self, analysis, device=0):
        import torch
        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device: the hylu_b200 path has no CPU fallback")
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.lib = library()
        self.analysis = analysis
        h = ctypes.c_void_p()
        check(self.lib.hy_create(device, ctypes.byref(h)))
        self.h = h
        # developer knobs: HYLU_OPTIONS="name=value,name=value" (hy_set_option)
        for kv in filter(None, os.environ.get("HYLU_OPTIONS", "").split(",")):
            k, v = kv.split("=")
            self.set_option(k.strip(), int(v))
        s = analysis.symbolic
        A = analysis.A
        vm = analysis.vmap
        ps = analysis.pivot_scale
        keep = dict(
            node_first=np.ascontiguousarray(s.node_first, np.int64),
            node_kind=np.ascontiguousarray(s.node_kind, np.int8),
            colptr=np.ascontiguousarray(s.colptr, np.int64),
            cols=np.ascontiguousarray(s.cols, np.int32),
            nl=np.ascontiguousarray(s.nl, np.int64),
            valoff=np.ascontiguousarray(s.valoff, np.int64),
            dep_ptr=np.ascontiguousarray(s.dep_ptr, np.int64),
            deps=np.ascontiguousarray(s.deps, np.int32),
            level_ptr=np.ascontiguousarray(s.level_ptr, np.int64),
            level_nodes=np.ascontiguousarray(s.level_nodes, np.int32),
            ulevel_ptr=np.ascontiguousarray(s.ulevel_ptr, np.int64),
            ulevel_nodes=np.ascontiguousarray(s.ulevel_nodes, np.int32),
            a_row_ptr=np.ascontiguousarray(A.row_ptr, np.int64),
            a_col_idx=np.ascontiguousarray(A.col_idx, np.int64),
            mrow_src=np.ascontiguousarray(vm.mrow_src, np.int64),
            colpos=np.ascontiguousarray(vm.colpos, np.int32),
            scale=np.ascontiguousarray(vm.scale, np.float64),
            dr=np.ascontiguousarray(ps.dr, np.float64),
            dc=np.ascontiguousarray(ps.dc, np.float64),
            perm=np.ascontiguousarray(analysis.ordering.perm, np.int64),
        )
        d = SymbolicDesc()
        d.n, d.nnodes, d.nnz = s.n, s.nnodes, A.nnz
        d.kernel_mode = int(s.kernel_mode)
        for k, v in keep.items():
            setattr(d, k, v.ctypes.data)
        d.nlevels = len(s.level_ptr) - 1
        d.nulevels = len(s.ulevel_ptr) - 1
        with torch.cuda.device(self.device):
            check(self.lib.hy_upload_symbolic(self.h, ctypes.byref(d)))
        self.stored = int(self.lib.hy_stored_values(self.h))
        self.n = s.n
        self.nnz = A.nnz
        from . import schedule as _sc
        self.wide_row = int(os.environ.get("HYLU_WIDE_ROW", _sc.WIDE_ROW))
        want = os.environ.get("HYLU_PATH", "auto")
        # level fan-in for every mode (supernode sources applied as blocks; in ROWROW
        # mode this equals row-row up to summation order); the row
        # path (row-row loop, hub pull rows, column slabs) stays selectable
        self.path = "fanin" if want == "auto" else want
        if self.path == "fanin":
            self.upload_fanin_plan()
        else:
            if _sc.slab_nodes(s, self.wide_row).any():
                self.upload_slab_plan()
            self.upload_hub_programs()

    def upload_hub_programs(self):
        """Pull programs for standalone hub rows of the row path (ROWROW mode)."""
        from . import schedule
        hub = int(os.environ.get("HYLU_HUB_STEPS", schedule.HUB_STEPS))
        progs = schedule.build_programs(self.analysis, np.zeros(self.n, np.int64), hub,
                                        standalone_only=True)
        if not len(progs.hub_nodes):
            return
        self._desc_programs(progs, self.lib.hy_upload_hub_programs)

    def upload_fanin_plan(self):
        from . import schedule
        s = self.analysis.symbolic
        plan = getattr(s, "_fanin_plan", None)
        if plan is None:
            # standalone hub rows (thousands of row sources) run as pull programs
            pull = None
            if os.environ.get("HYLU_FANIN_PULL", "0") != "0":
                hub = int(os.environ.get("HYLU_HUB_STEPS", schedule.HUB_STEPS))
                progs = schedule.build_programs(self.analysis, np.zeros(self.n, np.int64), hub,
                                                standalone_only=True)
                if len(progs.hub_nodes):
                    pull = np.zeros(s.nnodes, bool)
                    pull[progs.hub_nodes] = True
                    s._pull_programs = progs
            plan = schedule.build_fanin_plan(s, pull=pull)
            s._fanin_plan = plan
        progs = getattr(s, "_pull_programs", None)
        if progs is not None and len(plan.hub_list):
            self._desc_programs(progs, self.lib.hy_upload_hub_programs)
        arrs = {k: np.ascontiguousarray(getattr(plan, k)) for k in (
            "lu_ptr", "lu_nodes", "pt_ptr", "pt_node", "pt_c0", "pt_c1", "xp_ptr", "xp_edge", "xp_tgt",
            "lev_up", "up_t", "up_c0", "up_c1", "up_ptr", "src_k", "src_q0", "src_q1", "dep_pb",
            "level_smax", "level_mmax", "lev_up_big", "lev_up_reg", "lev_up_rs", "lev_xp_big",
            "lev_hub", "hub_list", "up_part", "part_first", "part_n", "part_off")}
        arrs["lu_nodes"] = arrs["lu_nodes"].astype(np.int32)
        sv, spb, stb = schedule.fanin_source_records(s, plan)
        arrs["src_v"], arrs["src_pb"], arrs["src_tb"] = sv, spb, stb
        arrs["xp_edge"] = arrs["xp_edge"].astype(np.int64)
        d = FaninPlanDesc()
        d.nlevels, d.nsrc, d.ndeps = plan.nlevels, len(plan.src_k), len(plan.dep_pb)
        d.nhub = len(plan.hub_list)
        d.nparts = len(plan.part_n)
        for k, v in arrs.items():
            setattr(d, k, v.ctypes.data if v.size else None)
        with self.torch.cuda.device(self.device):
            check(self.lib.hy_upload_fanin_plan(self.h, ctypes.byref(d)))
        self._fanin_arrays = arrs
        if os.environ.get("HYLU_FANIN_MAPS", "1") != "0":
            # per source record: tile positions of its columns + source metadata
            # (k_fi_upd_kc skips its per-item binary searches); cached with the plan
            # (built per upload, not cached on the analysis: the device copy is the one used)
            off, pos, vb, vW, qb, mm = schedule.kc_source_maps(s, plan)
            ptr = lambda a: a.ctypes.data if a.size else None  # noqa: E731
            with self.torch.cuda.device(self.device):
                check(self.lib.hy_upload_fanin_maps(self.h, len(vb), len(pos), ptr(off), ptr(pos), ptr(vb),
                                                    ptr(vW), ptr(qb), ptr(mm)))

    def upload_slab_plan(self):
        from . import schedule
        s = self.analysis.symbolic
        plan = getattr(s, "_slab_plan", None)
        if plan is None or getattr(s, "_slab_wide", None) != self.wide_row:
            plan = schedule.build_slab_plan(s, wide_row=self.wide_row)
            s._slab_plan = plan
            s._slab_wide = self.wide_row
        need = schedule.slab_level_smem(s, plan)
        dep_pb = schedule._dep_block_pos(s.node_first, s.node_kind, s.colptr, s.cols, s.nl,
                                         s.dep_ptr, s.deps)
        arrs = dict(
            sl_node=np.ascontiguousarray(plan.sl_node, np.int32),
            sl_c0=np.ascontiguousarray(plan.sl_c0, np.int32),
            sl_c1=np.ascontiguousarray(plan.sl_c1, np.int32),
            sl_kind=np.ascontiguousarray(plan.sl_kind, np.int8),
            it_ptr=np.ascontiguousarray(plan.it_ptr, np.int64),
            it_k=np.ascontiguousarray(plan.it_k, np.int32),
            it_q0=np.ascontiguousarray(plan.it_q0, np.int32),
            it_q1=np.ascontiguousarray(plan.it_q1, np.int32),
            it_own=np.ascontiguousarray(plan.it_own, np.int8),
            dep_pb=np.ascontiguousarray(dep_pb, np.int32),
            level_slab_ptr=np.ascontiguousarray(plan.level_slab_ptr, np.int64),
            level_smax=np.ascontiguousarray(need[:, 0], np.int32),
            level_mmax=np.ascontiguousarray(need[:, 1], np.int32),
            level_swmax=np.ascontiguousarray(need[:, 2], np.int32),
            level_accmax=np.ascontiguousarray(need[:, 3], np.int32),
        )
        d = SlabPlanDesc()
        d.nslabs, d.nitems, d.ndeps = plan.nslabs, len(plan.it_k), len(dep_pb)
        d.nlevels = len(plan.level_slab_ptr) - 1
        for k, v in arrs.items():
            setattr(d, k, v.ctypes.data if v.size else None)
        with self.torch.cuda.device(self.device):
            check(self.lib.hy_upload_slab_plan(self.h, ctypes.byref(d)))
        self._slab_arrays = arrs

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.hy_destroy(self.h)
                self.h = None
        except Exception:
            pass

    def stream_handle(self, stream=None):
        t = self.torch
        st = stream if stream is not None else t.cuda.current_stream(self.device)
        return ctypes.c_uint64(st.cuda_stream)

    def alloc_factors(self, pert_cap=1024):
        t = self.torch
        dev = self.device
        bufs = dict(
            values=t.empty(self.stored, dtype=t.float64, device=dev),
            inner_perm=t.zeros(self.n, dtype=t.int32, device=dev),
            anorm=t.zeros(1, dtype=t.float64, device=dev),
            status=t.zeros(4, dtype=t.int32, device=dev),
            pert_rows=t.zeros(pert_cap, dtype=t.int64, device=dev),
            pert_vals=t.zeros(pert_cap, dtype=t.float64, device=dev),
        )
        desc = FactorsDesc(bufs["values"].data_ptr(), bufs["inner_perm"].data_ptr(),
                           bufs["anorm"].data_ptr(), bufs["status"].data_ptr(),
                           bufs["pert_rows"].data_ptr(), bufs["pert_vals"].data_ptr(), pert_cap, -1)
        return bufs, desc

    def upload_programs(self, progs):
        """Upload schedule.RowPrograms (built for a prior inner_perm)."""
        self._desc_programs(progs, self.lib.hy_upload_row_programs)

    def _desc_programs(self, progs, fn):
        arrs = {k: np.ascontiguousarray(getattr(progs, k)) for k in (
            "row_ptr", "st_p", "st_j", "st_src", "st_cnt", "st_rel", "rel", "node_hub", "hrow_lev",
            "lev_ptr", "hpos", "hdiv", "hpp", "pred_p", "pred_u", "lev_wi", "wi_p", "wi_kd", "wi_y0",
            "wi_y1", "wi_slot", "lev_sp", "sp_p", "sp_kd", "sp_s0", "sp_n", "level_ws", "node_rec",
            "row_rec")}
        d = ProgramsDesc()
        d.nsteps, d.nrel = len(progs.st_p), len(progs.rel)
        d.nhubrows = len(progs.hrow_lev) - 1
        d.nlev = len(progs.lev_ptr) - 1
        d.nhpos, d.npred = len(progs.hpos), len(progs.pred_p)
        d.nwi, d.nsp, d.max_slots = len(progs.wi_p), len(progs.sp_p), progs.max_slots
        for k, v in arrs.items():
            setattr(d, k, v.ctypes.data if v.size else None)
        with self.torch.cuda.device(self.device):
            check(fn(self.h, ctypes.byref(d)))
        self._programs = getattr(self, "_programs", [])
        self._programs.append(arrs)

    def ensure_matrix(self, A):
        """Upload A's pattern (original coordinates) for device refinement, once.
        The pattern must be the analysed one (SPEC.md:343 same-pattern contract)."""
        if getattr(self, "_matrix_uploaded", False):
            return
        A0 = self.analysis.A
        if A.n != A0.n or A.nnz != A0.nnz or not np.array_equal(A.row_ptr, A0.row_ptr) or \
                not np.array_equal(A.col_idx, A0.col_idx):
            raise errors.PatternMismatch("refinement matrix pattern differs from the analysed one")
        rp = np.ascontiguousarray(A.row_ptr, np.int64)
        ci = np.ascontiguousarray(A.col_idx, np.int32)
        with self.torch.cuda.device(self.device):
            check(self.lib.hy_upload_matrix(self.h, rp.ctypes.data, ci.ctypes.data))
        self._matrix_uploaded = True

    def ensure_partition(self, threads=None, config=None, method="partition"):
        """Build and upload the launch lists of the multi-RHS solve, cached per method
        and parameters.  ``method="partition"``: ``partition.build_partition`` (SPEC.md:
        461-469) + ``device_launches``; ``threads`` defaults to the device's resident
        warps (SM count x 8) for the balanced row ranges; unless the config sets
        ``seg_nnz_threshold``, segments hold >= 1/32 of the stored entries (each segment
        costs launches, not a thread barrier).  ``method="levels"``:
        ``partition.device_launches_levels`` (supernode panels on DMMA)."""
        from . import partition as pt
        s = self.analysis.symbolic
        if method == "levels":
            key = ("levels",)
            if getattr(self, "_partition_key", None) == key:
                return self._partition
            fwd, bwd, items = pt.device_launches_levels(s)
            part = None
        else:
            if threads is None:
                threads = self.torch.cuda.get_device_properties(self.device).multi_processor_count * 8
            cfg = config or self.analysis.config
            if cfg.seg_nnz_threshold is None:
                cfg = cfg.with_overrides(seg_nnz_threshold=max(4096, int(s.stored_values) // 32))
            key = (int(threads), int(cfg.seg_nnz_threshold), int(cfg.small_tri_threshold),
                   int(cfg.bulk_width_factor))
            if getattr(self, "_partition_key", None) == key:
                return self._partition
            part = pt.build_partition(s, threads, cfg)
            fwd, bwd, items = pt.device_launches(s, part)
        fwd, bwd = np.ascontiguousarray(fwd), np.ascontiguousarray(bwd)
        items = np.ascontiguousarray(items)
        d = PartitionDesc(len(fwd), len(bwd), len(items), fwd.ctypes.data if fwd.size else None,
                          bwd.ctypes.data if bwd.size else None, items.ctypes.data if items.size else None)
        with self.torch.cuda.device(self.device):
            check(self.lib.hy_upload_partition(self.h, ctypes.byref(d)))
        self._partition, self._partition_key = part, key
        return part

    def set_option(self, name, value):
        check(self.lib.hy_set_option(self.h, name.encode(), int(value)))

    def launches(self):
        return int(self.lib.hy_launch_count(self.h))
