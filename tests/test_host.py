"""Host-side logic on CPU: generators, orderings, row programs (executed by a CPU
interpreter and compared with the oracle), sharding (gloo, world size 2), and the
C-ABI library exports."""
import ctypes
import os
import re

import numba
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


def test_integration_doc_names_every_header_symbol():
    """INTEGRATION.md (the reference-side binding) covers the whole C ABI."""
    hdr = open(os.path.join(ROOT, "include", "hylu_b200.h")).read()
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    names = set(re.findall(r"\b(hy_[a-z_]+)\s*\(", hdr))
    missing = sorted(nm for nm in names if nm not in doc)
    assert not missing, missing


def _run_fanin_cpu(an, plan):
    """CPU interpreter of the level fan-in plan (the device kernels' arithmetic)."""
    s = an.symbolic
    vm = an.vmap
    A = an.A
    F = np.zeros(s.stored_values)
    thr = 1e-8 * on.anorm_kernel(A.values, vm.scale)
    rows = np.diff(s.node_first)
    W = np.diff(s.colptr)

    def blk(u):
        return F[s.valoff[u]:s.valoff[u] + rows[u] * W[u]].reshape(rows[u], W[u])

    for i in range(s.n):
        u = s.node_of[i]
        a = vm.mrow_src[i]
        e0, e1 = A.row_ptr[a], A.row_ptr[a + 1]
        blk(u)[i - s.node_first[u], vm.colpos[e0:e1]] = A.values[e0:e1] * vm.scale[e0:e1]
    iperm = np.zeros(s.n, np.int64)
    for lv in range(plan.nlevels):
        for u in plan.lu_nodes[plan.lu_ptr[lv]:plan.lu_ptr[lv + 1]]:
            B = blk(u)
            r, L, sr = s.node_first[u], s.nl[u], rows[u]
            perm = np.arange(sr)
            for t in range(sr):
                p = t + int(np.argmax(np.abs(B[t:, L + t])))
                if p != t:
                    B[[t, p]] = B[[p, t]]
                    perm[[t, p]] = perm[[p, t]]
                if abs(B[t, L + t]) < thr:
                    B[t, L + t] = thr if B[t, L + t] >= 0 else -thr
                for q in range(t + 1, sr):
                    B[q, L + t] /= B[t, L + t]
                    B[q, L + t + 1:] -= B[q, L + t] * B[t, L + t + 1:]
            iperm[r:r + sr] = perm
        for x in range(plan.xp_ptr[lv], plan.xp_ptr[lv + 1]):
            k = plan.xp_edge[x]
            T = plan.xp_tgt[x]
            v = s.deps[k]
            Tb = blk(T)
            pb0 = plan.dep_pb[k]
            tb0 = s.node_cols(T)[pb0] - s.node_first[v]
            m = rows[v] - tb0
            Ub = blk(v)[tb0:, s.nl[v] + tb0:s.nl[v] + rows[v]]
            X = Tb[:, pb0:pb0 + m].copy()
            for a_ in range(m):
                X[:, a_] /= Ub[a_, a_]
                X[:, a_ + 1:] -= np.outer(X[:, a_], Ub[a_, a_ + 1:])
            Tb[:, pb0:pb0 + m] = X
        for it in range(plan.lev_up[lv], plan.lev_up[lv + 1]):
            T = plan.up_t[it]
            Tb = blk(T)
            tcols = s.node_cols(T)
            for z in range(plan.up_ptr[it], plan.up_ptr[it + 1]):
                k = s.dep_ptr[T] + plan.src_k[z]
                v = s.deps[k]
                pb0 = plan.dep_pb[k]
                tb0 = tcols[pb0] - s.node_first[v]
                m = rows[v] - tb0
                qb = s.nl[v] + rows[v]
                q0, q1 = plan.src_q0[z], plan.src_q1[z]
                vc = s.node_cols(v)[qb + q0:qb + q1]
                pos = np.searchsorted(tcols, vc)
                X = Tb[:, pb0:pb0 + m]
                Tb[:, pos] -= X @ blk(v)[tb0:, qb + q0:qb + q1]
    return F, iperm


@pytest.mark.parametrize("name,mode", [("c0", None), ("c1", 1), ("c3", 2), ("c2", 1)])
def test_fanin_plan_reproduces_oracle(name, mode):
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering), kernel_override=mode)
    plan = schedule.build_fanin_plan(an.symbolic)
    F, ip = _run_fanin_cpu(an, plan)
    ref = on.factorize(an)
    # the interpreter applies permutations to whole rows, like the device
    assert np.array_equal(ip, ref.inner_perm)
    assert np.abs(F - ref.values).max() <= 1e-11 * max(1.0, np.abs(ref.values).max())


def test_joint_hub_programs_reproduce_oracle():
    """Hub supernodes (several hub rows) through the joint pull programs: rows'
    levels below their first cross-row level run together, the rest row by row."""
    bp = gen.circuit_batch(2, 3000, 3, 400)
    A = bp.A0
    an = an_mod.analyze(A, SolverConfig(ordering="amd"))
    f = on.factorize(an)
    ref = on.factorize(an, prior=f)
    prog = schedule.build_programs(an, f.inner_perm, hub_steps=40)
    s = an.symbolic
    multi = [u for u in prog.hub_nodes if s.node_first[u + 1] - s.node_first[u] > 1]
    assert multi, "want a hub supernode with several rows"
    # hub nodes read their sources' values: take every non-hub node from the oracle,
    # run the hub programs, compare the hub ranges
    F_all = ref.values.copy()
    for u in prog.hub_nodes:
        F_all[int(s.valoff[u]):int(s.valoff[u + 1])] = 0.0
    F2 = _run_pull_with(an, prog, A.values, F_all)
    for u in prog.hub_nodes:
        a, b = int(s.valoff[u]), int(s.valoff[u + 1])
        assert np.abs(F2[a:b] - ref.values[a:b]).max() <= 1e-12 * np.abs(ref.values).max()
    # the joint form merged the rows' levels: fewer levels than row by row
    schedule.JOINT_HUB_ROWS = False
    try:
        per_row = schedule.build_programs(an, f.inner_perm, hub_steps=40)
    finally:
        schedule.JOINT_HUB_ROWS = True
    assert len(prog.lev_ptr) < len(per_row.lev_ptr)
    F3 = _run_pull_with(an, per_row, A.values, F_all)
    for u in prog.hub_nodes:
        a, b = int(s.valoff[u]), int(s.valoff[u + 1])
        assert np.array_equal(F2[a:b], F3[a:b])   # same arithmetic, bit for bit


def _run_pull_with(an, prog, values, F):
    s = an.symbolic
    vm = an.vmap
    F = F.copy()
    thr = 1e-8 * on.anorm_kernel(an.A.values, vm.scale)
    hr = 0
    for u in prog.hub_nodes:
        r = int(s.node_first[u])
        nr = int(s.node_first[u + 1]) - r
        W = int(s.colptr[u + 1] - s.colptr[u])
        base = int(s.valoff[u])
        for t in range(nr):
            rec = prog.row_rec[r + t]
            e0, k = int(rec[1]), int(rec[2] >> 32)
            F[base + t * W: base + (t + 1) * W] = 0.0
            F[base + t * W + vm.colpos[e0:e0 + k]] = values[e0:e0 + k] * vm.scale[e0:e0 + k]
        for t in range(nr):
            h = hr + t
            for lev in range(prog.hrow_lev[h], prog.hrow_lev[h + 1]):
                for x in range(prog.lev_ptr[lev], prog.lev_ptr[lev + 1]):
                    p = base + int(prog.hpos[x])
                    acc = F[p]
                    for y in range(prog.hpp[x], prog.hpp[x + 1]):
                        acc -= F[base + int(prog.pred_p[y])] * F[prog.pred_u[y]]
                    kd = int(prog.hdiv[x])
                    if kd >= 0:
                        acc /= F[kd]
                    elif kd == -2 and abs(acc) < thr:
                        acc = thr if acc >= 0 else -thr
                    F[p] = acc
        hr += nr
    return F


def test_chain_accelerated_symbolic_is_exact():
    """The U-nesting-chain reach (symbolic._general_symbolic_chains, used for
    unsymmetric patterns) returns exactly the plain Gilbert-Peierls row reach's L/U
    patterns on unsymmetric, symmetric and random patterns."""
    import numpy as np
    import scipy.sparse as sp
    from paper_2509_07690_b200 import generators as gen, analysis as an_mod, symbolic as sy
    from paper_2509_07690_b200._ref import SolverConfig
    pats = []
    for p, order in [(gen.fem27(6, recipe="literal"), "nd"), (gen.config("c1", "small"), "amd"),
                     (gen.config("c0", "small"), "amd")]:
        s = an_mod.analyze(p.A, SolverConfig(ordering=order)).symbolic
        pats.append((s.n, np.asarray(s.mp), np.asarray(s.mc)))
    for t in range(4):
        M = (sp.random(200, 200, density=0.01 + 0.015 * t, random_state=t, format="csr") + sp.eye(200)).tocsr()
        M.sort_indices()
        pats.append((200, M.indptr.astype(np.int64), M.indices.astype(np.int64)))
    for n, mp, mc in pats:
        a = sy._general_symbolic(n, mp, mc)
        b = sy._general_symbolic_chains(n, mp, mc)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


def test_cli_usage_and_input_errors(tmp_path, capsys):
    """SPEC.md cli: exit 2 on usage errors, exit 1 on solver/input errors (error class
    and matrix name printed), generate_rhs modes."""
    import numpy as np
    import pytest
    from paper_2509_07690_b200 import cli
    from paper_2509_07690_b200._ref import errors
    assert cli.main([]) == 2                                        # --matrix missing
    bad = tmp_path / "bad.mtx"
    bad.write_text("not a matrix market file\n")
    assert cli.main(["--matrix", str(bad), "--set", "no_such_field=1"]) == 2
    assert cli.main(["--matrix", str(bad), "--repeat", "-1"]) == 2
    assert cli.main(["--matrix", str(bad)]) == 1
    assert "ParseError" in capsys.readouterr().err
    assert np.array_equal(cli.generate_rhs("ones", 3), np.ones(3))
    assert np.array_equal(cli.generate_rhs("random:7", 4), cli.generate_rhs("random:7", 4))
    f = tmp_path / "b.txt"
    f.write_text("1 2\n")
    with pytest.raises(errors.LengthMismatch):
        cli.generate_rhs(str(f), 3)


def test_kc_source_maps_match_direct_search():
    """schedule.kc_source_maps: every source column's tile position equals a direct
    search of the target tile's columns, and the metadata matches the node arrays."""
    import numpy as np
    from paper_2509_07690_b200 import generators as gen, analysis as an_mod, schedule
    from paper_2509_07690_b200._ref import SolverConfig
    for name in ("c2", "c3", "c1"):
        p = gen.config(name, "small")
        s = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering)).symbolic
        plan = schedule.build_fanin_plan(s)
        off, pos, vb, vW, qb, mm = schedule.kc_source_maps(s, plan)
        sv, _, stb = schedule.fanin_source_records(s, plan)
        cols, colptr = np.asarray(s.cols), np.asarray(s.colptr)
        first, nl, valoff = np.asarray(s.node_first), np.asarray(s.nl), np.asarray(s.valoff)
        for it in range(len(plan.up_t)):
            T = plan.up_t[it]
            tc = cols[colptr[T] + plan.up_c0[it]:colptr[T] + plan.up_c1[it]]
            for z in range(plan.up_ptr[it], plan.up_ptr[it + 1]):
                v = sv[z]
                vs = first[v + 1] - first[v]
                q = nl[v] + vs + plan.src_q0[z]
                sc = cols[colptr[v] + q:colptr[v] + q + plan.src_q1[z] - plan.src_q0[z]]
                assert np.array_equal(pos[off[z]:off[z + 1]], np.searchsorted(tc, sc))
                assert (vb[z], vW[z], qb[z], mm[z]) == (valoff[v], colptr[v + 1] - colptr[v], q, vs - stb[z])


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_parallel_oracle_is_bitwise_sequential(name):
    """The oracle's level-parallel executor (SPEC.md:397-405 run_bulk) gives the
    sequential restatement's factors bit for bit, in every kernel mode, for
    factorize and refactorize (the CPU baseline's 'all threads' leg uses it)."""
    p = gen.config(name, "small")
    for mode in (None, 0, 1, 2):
        an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering), kernel_override=mode)
        f1 = on.factorize(an)
        f2 = on.factorize(an, threads=4)
        assert np.array_equal(f1.values, f2.values)
        assert np.array_equal(f1.inner_perm, f2.inner_perm)
        assert f1.perturbed == f2.perturbed and f1.breakdown == f2.breakdown
        v2 = np.asarray(p.A.values) * 1.01
        r1 = on.factorize(an, v2, prior=f1)
        r2 = on.factorize(an, v2, prior=f1, threads=3)
        assert np.array_equal(r1.values, r2.values)


def test_parallel_oracle_perturbation_and_breakdown_logs():
    """Zero pivots: the parallel executor's per-row flags reproduce the sequential
    perturbation log (factor-row order)."""
    p = gen.lap2d(8)
    an = an_mod.analyze(p.A, SolverConfig(ordering="amd"))
    v = np.array(p.A.values)
    rows = np.repeat(np.arange(p.A.n), np.diff(p.A.row_ptr))
    v[rows == p.A.col_idx] = 0.0                       # every diagonal zero
    f1 = on.factorize(an, v)
    f2 = on.factorize(an, v, threads=4)
    assert len(f1.perturbed) > 0
    assert f1.perturbed == f2.perturbed and f1.breakdown == f2.breakdown


def _gloo_shard_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    bp = gen.circuit_batch(24, 2000, 2, 200)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    prior = on.factorize(an)
    lo, hi = sharding.shard_range(24, rank, world)
    X, npert = on.refactor_solve_batch(an, prior, bp.values[lo:hi], bp.rhs[lo:hi])
    Xall = sharding.gather_shards(X, 24, dist)
    nall = sharding.gather_shards(npert, 24, dist)
    t = sharding.all_values(float(rank) + 0.5, dist)
    if rank == 0:
        X1, n1 = on.refactor_solve_batch(an, prior, bp.values, bp.rhs)
        q.put((bool(np.array_equal(Xall, X1)), bool(np.array_equal(nall, n1)), t))
    dist.destroy_process_group()


def test_sharded_batch_gloo_world2_matches_single_rank():
    """the c4 workload sharded contiguously over 2 ranks (gloo, CPU)
    with no data-path collective; the gathered solutions equal a single-rank run
    bit for bit."""
    import multiprocessing as mp
    import random
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = random.randint(20000, 40000)
    ps = [ctx.Process(target=_gloo_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(300)
    same_x, same_n, t = q.get(timeout=5)
    assert same_x and same_n
    assert t == [0.5, 1.5]


def test_oracle_batch_refines_perturbed_instances():
    """a batch instance whose refactorization perturbs a pivot is refined
    automatically (oracle side of the batched refinement parity)."""
    bp = gen.circuit_batch(6, 1500, 2, 150)
    an = an_mod.analyze(bp.A0, SolverConfig(ordering="amd"))
    prior = on.factorize(an)
    vals = bp.values.copy()
    gen.zero_first_pivot(an, vals[3])
    reps = {}
    X, npert = on.refactor_solve_batch(an, prior, vals, bp.rhs, reports=reps)
    assert npert[3] >= 1 and sorted(reps) == [b for b in range(6) if npert[b] > 0]
    rep = reps[3]
    assert rep["iterations"] >= 1 and rep["converged"]
    assert rep["backward_errors"][-1] <= 1e-13
    assert all(b <= a for a, b in zip(rep["backward_errors"], rep["backward_errors"][1:]))
    from paper_2509_07690_b200._ref import matrix as refmatrix
    A3 = bp.A0.with_values(vals[3])
    assert refmatrix.backward_error(A3, X[3], bp.rhs[3]) <= 1e-13
    X0, _ = on.refactor_solve_batch(an, prior, vals, bp.rhs, refine_perturbed=False)
    assert refmatrix.backward_error(A3, X0[3], bp.rhs[3]) > 1e-13   # refinement did the work


@pytest.mark.parametrize("name", ["c0", "c2"])
def test_device_routing_table(name):
    """The device dispatch written down: every dependency
    edge gets tier min(kernel_mode, natural tier); ROWROW runs the row-row operation
    order; the kernel counts cover every item of the fan-in plan."""
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    s = an.symbolic
    plan = schedule.build_fanin_plan(s)
    s._fanin_plan = plan
    nd = int(s.dep_ptr[-1])
    for m in (0, 1, 2):
        r = schedule.device_routing(s, m)
        assert sum(r["edges"].values()) == nd == sum(r["edge_tiers"].values())
        assert r["kernel_mode"] == KernelMode(m).name
        assert r["update_order"].startswith("row-row") == (m == 0)
        t = r["edge_tiers"]
        if m == 0:
            assert t["sup-row"] == t["sup-sup"] == 0
        if m == 1:
            assert t["sup-sup"] == 0 and t["sup-row"] == r["edges"]["row<-sup"] + r["edges"]["sup<-sup"]
        if m == 2:
            assert t["row-row"] == r["edges"]["row<-row"] + r["edges"]["sup<-row"]
            assert t["sup-sup"] == r["edges"]["sup<-sup"]
        k = r["kernels"]
        assert k["k_fi_upd_kcp"] + k["k_fi_upd_w"] + k["k_fi_upd_kc"] == len(plan.up_t)
        assert k["k_fi_x_w"] + k["k_fi_x"] == len(plan.xp_edge)
    assert r["edges"]["sup<-sup"] > 0 and r["tensor_core_items"] > 0


@pytest.mark.parametrize("name", ["c0", "c1", "c2", "c3"])
def test_parallel_fanin_updates_equal_serial(name):
    """The update items built in parallel over (level, target) groups are the serial
    plan loop's arrays, element for element."""
    p = gen.config(name, "small")
    an = an_mod.analyze(p.A, SolverConfig(ordering=p.ordering))
    s = an.symbolic
    flev = schedule._fanin_levels(s.node_first, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps, s.node_of)
    nlev = int(flev.max()) + 1
    ser = schedule._fanin_plan(s.node_first, s.node_kind, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps,
                               flev, nlev, schedule.FANIN_TILE, schedule.PANEL_TILE)
    par = schedule._fanin_updates_par(s.node_first, s.colptr, s.cols, s.nl, s.dep_ptr, s.deps,
                                      ser[6], ser[7], ser[8], nlev, schedule.FANIN_TILE,
                                      numba.config.NUMBA_NUM_THREADS)
    for a, b in zip(ser[9:], par):
        assert np.array_equal(np.asarray(a), np.asarray(b))
