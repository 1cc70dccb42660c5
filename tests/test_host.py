"""Host-side logic on CPU: generators, orderings, row programs (executed by a CPU
interpreter and compared with the oracle), sharding (gloo, world size 2), and the
C-ABI library exports."""
import ctypes
import os
import re

import numpy as np
import pytest

from paper_2509_07690_b200 import analysis as an_mod
from paper_2509_07690_b200 import generators as gen
from paper_2509_07690_b200 import preprocess as pp
from paper_2509_07690_b200 import schedule, sharding
from paper_2509_07690_b200._ref import KernelMode, SolverConfig
from oracle import numeric as on

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_generators_shapes_and_modes():
    p = gen.lap2d(64)
    assert p.A.n == 4096 and p.A.nnz == 20224
    an = an_mod.analyze(p.A, SolverConfig(ordering="amd"))
    assert an.symbolic.kernel_mode == KernelMode.SUPROW
    assert an.symbolic.fill_nnz == 127414 and an.symbolic.flops == 4751353
    p2 = gen.convdiff3d(8)
    assert p2.A.nnz == 7 * 512 - 6 * 64
    p3 = gen.fem27(4)
    assert p3.A.nnz == 9 * (3 * 4 - 2) ** 3
    bp = gen.circuit_batch(4, 3000, 2, 300)
    assert bp.values.shape == (4, bp.A0.nnz) and bp.rhs.shape == (4, 3000)
    an4 = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    assert an4.symbolic.kernel_mode == KernelMode.ROWROW          # c4 acceptance


def test_batch_values_deterministic_and_dominant():
    bp = gen.circuit_batch(3, 2000, 1, 100)
    bv = bp.meta["gen"]
    v, r = bv.instance(1)
    assert np.array_equal(v, bp.values[1]) and np.array_equal(r, bp.rhs[1])
    A = bp.A0.with_values(v)
    D = A.to_dense()
    off = np.abs(D).sum(1) - np.abs(np.diag(D))
    assert np.all(np.abs(np.diag(D)) > off)


def test_nd_ordering_is_permutation_and_deterministic():
    p = gen.convdiff3d(10)
    ps = pp.static_pivot(p.A)
    ap, ai = pp.pivoted_sym_pattern(p.A, ps)
    o1 = pp.nd_order(ap, ai)
    o2 = pp.nd_order(ap, ai)
    assert np.array_equal(np.sort(o1.perm), np.arange(p.A.n))
    assert np.array_equal(o1.perm, o2.perm)
    assert np.array_equal(o1.perm[o1.inverse_perm], np.arange(p.A.n))


def _run_programs_cpu(an, prog, values):
    """Interpret the batched row programs on the CPU (one instance) — the exact
    arithmetic the device executes (push loop for every row)."""
    s = an.symbolic
    vm = an.vmap
    F = np.zeros(s.stored_values)
    thr = 1e-8 * on.anorm_kernel(an.A.values, vm.scale)
    for u in range(s.nnodes):
        r = int(s.node_first[u])
        W = int(s.colptr[u + 1] - s.colptr[u])
        for t in range(int(s.node_first[u + 1]) - r):
            i = r + t
            rec = prog.row_rec[i]
            w = np.zeros(W)
            e0, k = int(rec[1]), int(rec[2] >> 32)
            w[vm.colpos[e0:e0 + k]] = values[e0:e0 + k] * vm.scale[e0:e0 + k]
            for st in range(prog.row_ptr[i], prog.row_ptr[i + 1]):
                p = prog.st_p[st]
                src = prog.st_src[st]
                l = w[p] / F[src]
                w[p] = l
                cnt = prog.st_cnt[st]
                rel = prog.rel[prog.st_rel[st]:prog.st_rel[st] + cnt]
                w[rel] -= l * F[src + 1:src + 1 + cnt]
            d = int(s.nl[u]) + t
            if abs(w[d]) < thr:
                w[d] = thr if w[d] >= 0 else -thr
            F[s.valoff[u] + t * W: s.valoff[u] + (t + 1) * W] = w
    return F


@pytest.mark.parametrize("name", ["c1", "c4"])
def test_row_programs_reproduce_oracle(name):
    if name == "c4":
        bp = gen.circuit_batch(2, 1500, 2, 150)
        A = bp.A0
    else:
        A = gen.circuit(1500, 2, 150).A
    an = an_mod.analyze(A, SolverConfig(ordering="amd"))
    f = on.factorize(an)
    prog = schedule.build_programs(an, f.inner_perm, hub_steps=50)
    F = _run_programs_cpu(an, prog, A.values)
    ref = on.factorize(an, prior=f)
    assert np.abs(F - ref.values).max() <= 1e-12 * np.abs(ref.values).max()
    # hub pull programs cover every structurally nonzero position exactly once
    assert len(prog.hub_nodes) > 0
    assert len(prog.hpos) == len(prog.hdiv) == len(prog.hpp) - 1


def test_shard_ranges_cover_exactly():
    for world in (1, 2, 3, 4, 8):
        got = [sharding.shard_range(4096, r, world) for r in range(world)]
        assert got[0][0] == 0 and got[-1][1] == 4096
        assert all(a[1] == b[0] for a, b in zip(got, got[1:]))


def _gloo_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = sharding.shard_range(4096, rank, world)
    m = sharding.max_over_ranks(float(rank + 1), dist)
    q.put((rank, lo, hi, m))
    dist.destroy_process_group()


def test_sharding_gloo_world2():
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_gloo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(120)
    res = sorted(q.get(timeout=5) for _ in range(2))
    assert res[0][1:3] == (0, 2048) and res[1][1:3] == (2048, 4096)
    assert res[0][3] == res[1][3] == 2.0


def test_c_abi_library_exports_every_header_symbol():
    from paper_2509_07690_b200 import build
    path = build.build_cuda()
    lib = ctypes.CDLL(path)
    hdr = open(os.path.join(ROOT, "include", "hylu_b200.h")).read()
    names = set(re.findall(r"\b(hy_[a-z_]+)\s*\(", hdr))
    assert len(names) >= 12
    for nm in sorted(names):
        assert hasattr(lib, nm), nm
