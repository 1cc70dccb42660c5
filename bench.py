#!/usr/bin/env python
"""bench.py — headline benchmark (driver contract).

Workload (BASELINE.json configs[4], the config BASELINE's "refactors/sec" metric
is quoted on and the only one that shards): 4096 same-pattern circuit-like
matrices (n = 20000, ~102k nnz each), ONE host analysis on instance 0, then per
instance refactorize + solve on the device.  A step = one refactorize+solve pass
over every instance of the job (4096 in total, split contiguously across the N
ranks: strong scaling, no collective on the data path).

value  = instances (refactorize+solve) per second, whole job, inputs resident in HBM.
e2e    = the same through the public API with host (pinned) buffers: values and
         rhs H2D, refactorize+solve, x D2H, every step inside the timed region.
roofline (dominant kernel = batched refactorization): algorithmic bytes per
         instance 8·(nnz + fill_nnz) x instances / factor-phase time,
         against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the CPU oracle (numba restatement of SPEC, oracle/numeric.py) on
         a bounded sample of the same workload, all host threads.
``--impl reference`` times that CPU path alone as the reference arm.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_INST = 4096
N = 20000


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Poll SM clock + throttle reasons (NVML) during the timed region."""

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.index = index
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False

    def _run(self):
        nv = self.nv
        names = {
            getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4): "sw_power_cap",
            getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8): "hw_slowdown",
            getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20): "sw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40): "hw_thermal_slowdown",
            getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80): "hw_power_brake_slowdown",
        }
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in names.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": len(self.samples)}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_problem(lo, hi, threads):
    from paper_2509_07690_b200 import generators as gen
    base = gen.circuit(N, 3, 2000, gen.SEEDS["c4"])
    bv = gen.BatchValues(base.A, gen.SEEDS["c4"])
    vals = np.empty((hi - lo, base.A.nnz))
    rhs = np.empty((hi - lo, N))
    bv.fill(range(lo, hi), vals, rhs, threads)
    A0 = base.A.with_values(bv.instance(0)[0])
    return A0, bv, vals, rhs


def analysis_for(A0):
    from paper_2509_07690_b200 import analysis
    from paper_2509_07690_b200._ref import SolverConfig
    return analysis.analyze(A0, SolverConfig(ordering="amd"))


def cpu_sample(an, bv, count, threads):
    """Oracle refactorize+solve over ``count`` instances (all host threads)."""
    import numba
    from oracle import numeric as on
    numba.set_num_threads(threads)
    prior = on.factorize(an)
    vals = np.empty((count, bv.nnz))
    rhs = np.empty((count, bv.n))
    bv.fill(range(count), vals, rhs, threads)
    on.refactor_solve_batch(an, prior, vals[:2], rhs[:2])          # JIT warm-up
    reps = 0
    t0 = time.perf_counter()
    while True:                      # about 10 s of CPU work (whole passes over the sample)
        on.refactor_solve_batch(an, prior, vals, rhs)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= 10.0 or reps >= 64:
            break
    return count * reps / dt, dt, reps


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import numba
    threads = numba.config.NUMBA_NUM_THREADS
    A0, bv, _, _ = make_problem(0, 1, threads)
    an = analysis_for(A0)
    from oracle import numeric as on
    numba.set_num_threads(threads)
    prior = on.factorize(an)
    sample = args.ref_sample
    vals = np.empty((sample, bv.nnz))
    rhs = np.empty((sample, bv.n))
    bv.fill(range(sample), vals, rhs, threads)
    for _ in range(max(1, args.warmup)):
        on.refactor_solve_batch(an, prior, vals, rhs)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        on.refactor_solve_batch(an, prior, vals, rhs)
    dt = time.perf_counter() - t0
    value = sample * args.steps / dt
    s = an.symbolic
    line = {
        "impl": "reference",
        "metric": "refactors/sec (c4: batched FP64 refactorize+solve, n=20000)",
        "value": value, "unit": "instances/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded)",
        "config": {"workload": "c4 batched refactorize+solve", "batch": N_INST, "n": N,
                   "nnz": int(A0.nnz), "fill_nnz": int(s.fill_nnz), "kernel_mode": s.kernel_mode.name},
        "cpu_baseline": {"value": value, "unit": "instances/s", "cores": threads, "kind": "port",
                         "sample": "%d of the 4096 instances per step (oracle/numeric.py, numba, "
                                   "instances in parallel)" % sample},
        "e2e": {"value": value, "unit": "instances/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
    from paper_2509_07690_b200 import api
    threads = max(1, (os.cpu_count() or 8) // max(1, world))
    from paper_2509_07690_b200.sharding import shard_range
    lo, hi = shard_range(N_INST, rank, world)
    B = hi - lo
    A0, bv, vals, rhs = make_problem(lo, hi, threads)
    an = analysis_for(A0)
    s = an.symbolic
    prior = api.factorize_analysis(an, opts=api.FactorOptions(device=local))
    br = api.BatchedRefactorizer(prior)
    ctx = br.ctx
    lib = ctx.lib
    d_vals = torch.from_numpy(vals).to(dev)
    d_rhs = torch.from_numpy(rhs).to(dev)
    d_x = torch.empty((B, N), dtype=torch.float64, device=dev)
    d_np = torch.empty(B, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream(dev)
    sh = ctx.stream_handle(stream)
    from paper_2509_07690_b200.device import check

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        check(lib.hy_refactorize_batched(ctx.h, B, d_vals.data_ptr(), 1e-8, prior._desc,
                                         d_np.data_ptr(), d_rhs.data_ptr(), sh))
        if ev is not None:
            ev[1].record(stream)
        check(lib.hy_solve_batched(ctx.h, B, None, d_x.data_ptr(), sh))

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    fac_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)]
    t_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    l0 = ctx.launches()
    barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_ev[0].record(stream)
        for k in range(args.steps):
            step(fac_ev[k])
        t_ev[1].record(stream)
        torch.cuda.synchronize()
    barrier()
    launches = ctx.launches() - l0
    elapsed = max_over_ranks(t_ev[0].elapsed_time(t_ev[1]) / 1e3)
    fac_ms = float(np.mean([a.elapsed_time(b) for a, b in fac_ev]))
    value = N_INST * args.steps / elapsed

    # correctness spot check (outside the timed region)
    from paper_2509_07690_b200._ref import matrix as refmatrix
    xh = d_x[:2].cpu().numpy()
    resid = max(np.linalg.norm(refmatrix.spmv(A0.with_values(vals[b]), xh[b]) - rhs[b])
                / np.linalg.norm(rhs[b]) for b in range(2))

    # ---- e2e through the public API with pinned host buffers
    h_vals = torch.from_numpy(vals).pin_memory()
    h_rhs = torch.from_numpy(rhs).pin_memory()
    h_x = torch.empty((B, N), dtype=torch.float64).pin_memory()
    h_np = torch.empty(B, dtype=torch.int32).pin_memory()

    def e2e_step():
        # public API, host buffers: chunked, H2D / compute / D2H on three streams;
        # streaming use (pipelined): the next step's H2D starts while this step's
        # last chunks compute, per-chunk events guard buffer reuse
        br.run_host(h_vals, h_rhs, h_x, h_np, chunks=args.e2e_chunks, pipelined=True)

    for _ in range(max(1, args.warmup)):
        e2e_step()
    br.host_wait(stream)
    torch.cuda.synchronize()
    barrier()
    e_ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    e_ev[0].record(stream)
    for _ in range(args.steps):
        e2e_step()
    br.host_wait(stream)   # every step's D2H inside the timed region
    e_ev[1].record(stream)
    torch.cuda.synchronize()
    e_elapsed = max_over_ranks(e_ev[0].elapsed_time(e_ev[1]) / 1e3)
    e2e_value = N_INST * args.steps / e_elapsed

    # ---- CPU baseline (rank 0 at N=1 only)
    cpu = None
    if world == 1 and not args.no_cpu:
        import numba
        cthreads = numba.config.NUMBA_NUM_THREADS
        sample = args.cpu_sample
        cv, cdt, reps = cpu_sample(an, bv, sample, cthreads)
        cpu = {"value": cv, "unit": "instances/s", "cores": cthreads, "kind": "port",
               "sample": "%d passes over %d of the 4096 instances (refactorize+solve, "
                         "oracle/numeric.py, numba parallel over instances), %.1f s"
                         % (reps, sample, cdt)}

    peak, peak_kind = _peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_traffic.json")) as fh:
            tj = json.load(fh)
        traffic = float(sum(v for k, v in tj.items() if k.startswith("k_"))) * B / N_INST
    except Exception:
        traffic = None
    bytes_per_inst = 8 * (A0.nnz + s.fill_nnz)
    achieved = B * bytes_per_inst / (fac_ms / 1e3) / 1e9
    if rank == 0:
        line = {
            "metric": "refactors/sec (c4: batched FP64 refactorize+solve, n=20000)",
            "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed / args.steps * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded generators, paper_2509_07690_b200/generators.py)",
            "config": {"workload": "c4 batched refactorize+solve (BASELINE configs[4])",
                       "batch": N_INST, "per_rank": B, "n": N, "nnz": int(A0.nnz),
                       "fill_nnz": int(s.fill_nnz), "stored_values": int(s.stored_values),
                       "kernel_mode": s.kernel_mode.name, "levels": int(len(s.level_ptr) - 1),
                       "l2": "inputs larger than L2 (values %.2f GB/step)" % (vals.nbytes * world / 1e9),
                       "parallelism": "shard%d" % world},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "traffic_unit": "bytes per factor phase (ncu)",
                         "kernel": "k_bt_pipe + k_bt_hub (one batched refactorization pass, forward substitution fused)",
                         "algorithmic_bytes_per_instance": bytes_per_inst,
                         "factor_ms_per_step": fac_ms, "peak_source": peak_kind},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "instances/s",
                    "h2d_bytes_per_step": int(h_vals.numel() * 8 + h_rhs.numel() * 8) * world,
                    "d2h_bytes_per_step": int(h_x.numel() * 8 + h_np.numel() * 4) * world},
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "residual_max": resid,
        }
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=4096)
    ap.add_argument("--ref-sample", type=int, default=512)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-chunks", type=int, default=6)
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
