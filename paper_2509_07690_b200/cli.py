"""Benchmark harness / CLI (module ``cli``).

    python -m paper_2509_07690_b200.cli --matrix A.mtx [--rhs ones|random:SEED|PATH]
        [--threads N] [--repeat K] [--kernel auto|rowrow|suprow|supsup]
        [--ordering amd|natural|nd] [--perturb-eps X] [--perturb-values EPS]
        [--report PATH] [--set name=value ...]

Loads a Matrix Market file with the reference reader (``polylu.matrix.
read_matrix_market``, matrix.py:155), runs preprocess (reference matching + ordering +
symbolic) → device factorize → solve (with refinement when perturbation fired), then
``--repeat K`` device refactorize+solve cycles, and writes a ``SolveReport`` JSON with
SPEC's fields.  Exit codes: 0 success, 1 solver error (the error class and
matrix name are printed), 2 usage error (the flag reference is printed).  Phase times
are monotonic wall clocks around each phase, device work synchronised.
``--threads`` is recorded (SPEC's thread count; the device path ignores it).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from dataclasses import dataclass, field, asdict, fields

import numpy as np

from ._ref import SolverConfig, errors, matrix as refmatrix


@dataclass
class SolveReport:
    """SPEC.md:543-546."""
    matrix_name: str
    n: int
    nnz: int
    kernel_mode: str
    fill_nnz: int
    flops: float
    supernode_count: int
    standalone_row_count: int
    phase_times_seconds: dict
    repeat_times_seconds: list = field(default_factory=list)
    backward_error_final: float = 0.0
    refinement_iterations: int = 0
    perturbation_count: int = 0
    threads: int = 1
    device_routing: dict = field(default_factory=dict)   # B200 extension: schedule.device_routing


def generate_rhs(mode, n):
    """ones | random:SEED | path of whitespace-separated reals."""
    if mode == "ones":
        return np.ones(n)
    if mode.startswith("random"):
        _, _, seed = mode.partition(":")
        return np.random.default_rng(int(seed or 0)).uniform(-1.0, 1.0, n)
    with open(mode) as fh:
        vals = np.array([float(t) for t in fh.read().split()])
    if len(vals) != n:
        raise errors.LengthMismatch("rhs file has %d values, matrix has n = %d" % (len(vals), n))
    return vals


def _parse_set(items, cfg):
    over = {}
    names = {f.name: f for f in fields(SolverConfig)}
    for it in items:
        name, _, val = it.partition("=")
        if name not in names:
            raise ValueError("unknown configuration field %r" % name)
        cur = getattr(cfg, name)
        if isinstance(cur, bool):
            over[name] = val.lower() in ("1", "true", "yes")
        elif isinstance(cur, int):
            over[name] = int(val)
        elif isinstance(cur, float):
            over[name] = float(val)
        elif val.lower() == "none":
            over[name] = None
        else:
            try:
                over[name] = int(val)
            except ValueError:
                over[name] = val
    return cfg.with_overrides(**over) if over else cfg


def _parser():
    ap = argparse.ArgumentParser(prog="paper_2509_07690_b200.cli", add_help=True,
                                 description="HYLU B200 solve driver (SPEC.md cli module)")
    ap.add_argument("--matrix", required=True)
    ap.add_argument("--rhs", default="ones")
    ap.add_argument("--threads", type=int, default=1)
    ap.add_argument("--repeat", type=int, default=0)
    ap.add_argument("--kernel", default="auto", choices=["auto", "rowrow", "suprow", "supsup"])
    ap.add_argument("--ordering", default="amd", choices=["amd", "natural", "nd"])
    ap.add_argument("--perturb-eps", type=float, default=1e-8)
    ap.add_argument("--perturb-values", type=float, default=0.0)
    ap.add_argument("--report", default=None)
    ap.add_argument("--set", action="append", default=[])
    return ap


class _UsageError(Exception):
    pass


def main(argv=None):
    ap = _parser()
    try:
        try:
            args = ap.parse_args(argv)
        except SystemExit as e:   # argparse prints the flag reference itself
            return 0 if e.code == 0 else 2
        if args.threads < 1 or args.repeat < 0 or not (0.0 <= args.perturb_eps < 1.0):
            raise _UsageError("threads >= 1, repeat >= 0, 0 <= perturb-eps < 1")
        try:
            cfg = _parse_set(args.set, SolverConfig(ordering=args.ordering))
        except ValueError as e:
            raise _UsageError(str(e))
    except _UsageError as e:
        print("usage error: %s" % e, file=sys.stderr)
        ap.print_help(sys.stderr)
        return 2
    name = os.path.basename(args.matrix)
    try:
        return _run(args, cfg, name)
    except errors.PolyLUError as e:
        print("%s: %s (%s)" % (type(e).__name__, e, name), file=sys.stderr)
        return 1


def _run(args, cfg, name):
    import torch
    from . import analysis as an_mod
    from . import api
    A = refmatrix.read_matrix_market(args.matrix)
    b = generate_rhs(args.rhs, A.n)
    kov = None if args.kernel == "auto" else args.kernel.upper()
    from ._ref import KernelMode
    kov = None if kov is None else KernelMode[kov]
    t0 = time.perf_counter()
    an = an_mod.analyze(A, cfg, kernel_override=kov, threads=args.threads)
    t_pre = time.perf_counter() - t0
    opts = api.FactorOptions(perturbation_epsilon=args.perturb_eps, threads=args.threads)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    f = api.factorize_analysis(an, opts=opts)
    torch.cuda.synchronize()
    t_fac = time.perf_counter() - t0
    t0 = time.perf_counter()
    x, rep = api.solve(A, f, b=b, config=cfg)
    t_sol = time.perf_counter() - t0
    repeats = []
    rng = np.random.default_rng(12345)
    vals = np.asarray(A.values)
    for _ in range(args.repeat):
        Ak = A if args.perturb_values == 0.0 else A.with_values(
            vals * (1.0 + args.perturb_values * rng.uniform(-1.0, 1.0, len(vals))))
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fk = api.refactorize(Ak, f, opts)
        torch.cuda.synchronize()
        t_r = time.perf_counter() - t0
        t0 = time.perf_counter()
        x, rep = api.solve(Ak, fk, b=b, config=cfg)
        t_s = time.perf_counter() - t0
        repeats.append({"refactorize": t_r, "solve": t_s})
        A_last, f_last = Ak, fk
    if not args.repeat:
        A_last, f_last = A, f
    s = an.symbolic
    report = SolveReport(
        matrix_name=name, n=int(A.n), nnz=int(A.nnz), kernel_mode=s.kernel_mode.name,
        fill_nnz=int(s.fill_nnz), flops=float(s.flops), supernode_count=int(s.supernode_count),
        standalone_row_count=int(s.standalone_row_count),
        phase_times_seconds={"preprocess": t_pre, "factorize": t_fac, "solve": t_sol},
        repeat_times_seconds=repeats,
        backward_error_final=float(refmatrix.backward_error(A_last, x, b)),
        refinement_iterations=int(rep.iterations), perturbation_count=len(f_last.perturbed),
        threads=int(args.threads), device_routing=f_last.routing())
    text = json.dumps(asdict(report), indent=1)
    if args.report:
        with open(args.report, "w") as fh:
            fh.write(text + "\n")
    else:
        print(text)
    return 0


if __name__ == "__main__":
    sys.exit(main())
