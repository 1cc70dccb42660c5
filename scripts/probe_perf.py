"""Per-config device timings (factor / refactor / solve / batched) with CUDA events.

Usage: python scripts/probe_perf.py c0 c1 c2 c4 [--c3k 24]
Prints one JSON line per config.  Development probe; bench.py is the contract.
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2509_07690_b200 import api, generators as gen, analysis as an_mod  # noqa: E402
from paper_2509_07690_b200._ref import SolverConfig, matrix as refmatrix  # noqa: E402


def timed(fn, reps=5):
    ts = []
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        out = fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    return min(ts), out


def single(name, p):
    t0 = time.perf_counter()
    cap = int(os.environ.get("PROBE_SUPCAP", 64))   # SolverConfig.max_supernode_rows (SPEC default 64)
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering, max_supernode_rows=cap))
    ta = time.perf_counter() - t0
    s = an.symbolic
    dv = torch.from_numpy(np.array(p.A.values)).cuda()
    db = torch.from_numpy(np.array(p.b)).cuda()
    f = api.factorize_analysis(an, dv)
    tf, f = timed(lambda: api.factorize_analysis(an, dv), 3)
    tr, f2 = timed(lambda: api.refactorize(dv, f), 3)
    ts, x = timed(lambda: api.substitute(f, db), 5)
    xh = x.cpu().numpy()
    res = np.linalg.norm(refmatrix.spmv(p.A, xh) - p.b) / np.linalg.norm(p.b)
    out = dict(config=name, n=s.n, nnz=p.A.nnz, fill=s.fill_nnz, flops=s.flops, mode=s.kernel_mode.name,
               nodes=s.nnodes, levels=len(s.level_ptr) - 1, stored=s.stored_values,
               analyze_s=round(ta, 2), factor_ms=tf, refactor_ms=tr, solve_ms=ts,
               gflops=s.flops / tf / 1e6, residual=res, npert=len(f.perturbed))
    plan = getattr(s, "_fanin_plan", None)
    if plan is not None:   # executed (union-padded) update flops, SURVEY §8(d)
        from paper_2509_07690_b200 import schedule
        ex = schedule.executed_update_flops(s, plan)
        out.update(exec_update_flops=ex, exec_update_gflops=ex / tf / 1e6)
    print(json.dumps(out), flush=True)


def batch(B):
    t0 = time.perf_counter()
    bp = gen.circuit_batch(B)
    tg = time.perf_counter() - t0
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    s = an.symbolic
    prior = api.factorize_analysis(an)
    br = api.BatchedRefactorizer(prior)
    dv = torch.from_numpy(bp.values).cuda()
    dr = torch.from_numpy(bp.rhs).cuda()
    t, (x, npert) = timed(lambda: br.run(dv, dr), 3)
    xh = x[:4].cpu().numpy()
    res = max(np.linalg.norm(refmatrix.spmv(bp.A0.with_values(bp.values[b]), xh[b]) - bp.rhs[b])
              / np.linalg.norm(bp.rhs[b]) for b in range(4))
    byt = B * 8 * (bp.A0.nnz + s.fill_nnz)
    out = dict(config="c4", B=B, gen_s=round(tg, 1), ms=t, per_s=B / t * 1e3, stored=s.stored_values,
               fill=s.fill_nnz, levels=len(s.level_ptr) - 1, ulevels=len(s.ulevel_ptr) - 1,
               refactor_bytes_GBs=byt / t / 1e6, residual=res, npert=int(npert.sum().item()))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--c3k", type=int, default=24)
    ap.add_argument("--B", type=int, default=4096)
    a = ap.parse_args()
    for c in a.configs:
        if c == "c4":
            batch(a.B)
        elif c == "c3":
            single("c3_k%d" % a.c3k, gen.fem27(a.c3k))
        else:
            single(c, gen.config(c))
