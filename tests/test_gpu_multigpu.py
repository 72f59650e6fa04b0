"""Row-sharded (multi-GPU) path on one B200: the partial-sum local step,
explicit shard ranges and x = S/Q, for world 1 through the production driver
and for 2 and 4 emulated ranks in one process (each rank's local step is an
independent kernel; the all-reduce is the host sum of the ranks' S, which is
what NCCL's sum returns), against the sequential oracle with q_total workers
and the distributed scheme."""

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err

pytestmark = pytest.mark.gpu


def _system():
    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    return generate_mother(GeneratorConfig(m_max=4000, n_max=64, seed=5))


def test_world1_driver(gpu, oracle):
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards, solve_sharded

    s = _system()
    for variant, q, bs in (("rka", 8, 1), ("rkab", 4, 6)):
        plan = plan_shards(s.m, 1, 0, q)
        shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
        cfg = SolverConfig(variant=variant, q=q, block_size=bs, base_seed=2, sampling_scheme="distributed")
        r = solve_sharded(shard, cfg)
        shard.close()
        o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=2, scheme="distributed")
        assert r.converged and r.iterations == o["iterations"] and r.error_evals == o["error_evals"]
        assert rel_err(r.x, o["x"]) <= PARITY_TOL


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("variant,bs", [("rka", 1), ("rkab", 5)])
def test_emulated_ranks_one_gpu(gpu, oracle, world, variant, bs):
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards

    s = _system()
    q_local, budget = 4, 60
    cfg = SolverConfig(variant=variant, q=q_local, block_size=bs, base_seed=7, sampling_scheme="distributed")
    shards = []
    for g in range(world):
        p = plan_shards(s.m, world, g, q_local)
        shards.append(CudaShard(s.A[p.lo:p.hi + 1], s.b[p.lo:p.hi + 1], s.x_star, p, device=0))
    for sh in shards:
        sh.reset()
    for k in range(budget):
        S = [sh.step(cfg, k) for sh in shards]
        tot = S[0].clone()
        for extra in S[1:]:
            tot += extra
        errs = [sh.finish(tot, world * q_local) for sh in shards]
        assert len(set(errs)) == 1
    xs = [sh.x() for sh in shards]
    for sh in shards:
        sh.close()
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=world * q_local, block_size=bs, base_seed=7,
                     scheme="distributed", budget=budget)
    assert rel_err(xs[0], o["x"]) <= PARITY_TOL


def test_counter_shard_is_exact_row_slice(gpu):
    """kz_generate_counter_rows: a shard generated in place equals those rows of the
    full counter-keyed matrix (so row-sharded config-3 runs need no host copy)."""
    from paper_2401_17474_b200 import DeviceSystem

    with DeviceSystem(m=3000, n=700) as full:
        full.generate_counter(7)
        A, b, xr = full.download()
    with DeviceSystem(m=1000, n=700) as part:
        part.generate_counter(7, row0=1500)
        A2, b2, xr2 = part.download()
    assert np.array_equal(A2, A[1500:2500]) and np.array_equal(b2, b[1500:2500]) and np.array_equal(xr2, xr)


def _native_vs_host(s, variant, q, bs, seed, budget=None, comm=None, kernel="auto"):
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards, solve_sharded, solve_sharded_native

    plan = plan_shards(s.m, 1, 0, q)
    shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
    cfg = SolverConfig(variant=variant, q=q, block_size=bs, base_seed=seed, sampling_scheme="distributed",
                       kernel=kernel)
    rn = solve_sharded_native(shard, cfg, budget=budget, comm=comm, loop=True)
    rh = solve_sharded(shard, cfg, budget=budget)
    rn2 = solve_sharded_native(shard, cfg, budget=budget, comm=comm, loop=True)  # a second solve, same shard
    shard.close()
    return rn, rh, rn2


@pytest.mark.parametrize("variant,q,bs", [("rka", 8, 1), ("rkab", 4, 6)])
def test_native_sharded_loop_world1(gpu, oracle, variant, q, bs):
    """kz_solve_sharded (device stop flag, one host sync per chunk) against the host-driven
    loop (bitwise: same kernels, same collective, same average) and the oracle."""
    s = _system()
    rn, rh, rn2 = _native_vs_host(s, variant, q, bs, seed=2)
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=2, scheme="distributed")
    for r in (rn, rn2):
        assert r.converged and r.iterations == rh.iterations == o["iterations"]
        assert r.error_evals == rh.error_evals == o["error_evals"]
        # the rka step kernel checks x_k with its own (cluster-tree) error sum: same value to rounding
        assert abs(r.final_error_sq - rh.final_error_sq) <= 1e-12 * rh.final_error_sq
        assert np.array_equal(r.x, rh.x)
    assert rel_err(rn.x, o["x"]) <= PARITY_TOL


def test_native_sharded_budget_multi_cluster(gpu, oracle):
    """Budget mode on rows wide enough for several rka clusters (tagged-word exchange with
    per-launch tag ranges, one launch per outer iteration)."""
    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    s = generate_mother(GeneratorConfig(m_max=5000, n_max=4500, seed=3))
    rn, rh, rn2 = _native_vs_host(s, "rka", 16, 1, seed=4, budget=37)
    assert rn.iterations == rh.iterations == 37 and rn.error_evals == 0
    assert np.array_equal(rn.x, rh.x) and np.array_equal(rn2.x, rh.x)
    o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=16, base_seed=4, scheme="distributed", budget=37)
    assert rel_err(rn.x, o["x"]) <= PARITY_TOL


def test_native_sharded_max_iterations(gpu, oracle):
    """Stop mode that runs out of iterations: not converged, evals = max + 1."""
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards, solve_sharded, solve_sharded_native

    s = _system()
    plan = plan_shards(s.m, 1, 0, 8)
    shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
    cfg = SolverConfig(variant="rka", q=8, base_seed=1, sampling_scheme="distributed", max_iterations=150)
    rn = solve_sharded_native(shard, cfg, loop=True)
    rh = solve_sharded(shard, cfg)
    shard.close()
    assert not rn.converged and rn.iterations == rh.iterations == 150
    assert rn.error_evals == rh.error_evals == 151
    assert np.array_equal(rn.x, rh.x)


@pytest.mark.parametrize("variant,q,bs", [("rka", 8, 1), ("rkab", 4, 6)])
def test_one_rank_without_comm_runs_kz_solve(gpu, oracle, variant, q, bs):
    """With one rank and no communicator kz_solve_sharded delegates to kz_solve's chunked kernels
    (the bench's N = 1 headline path): same iteration counts and iterates as the per-iteration
    sharded loop and the oracle."""
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards, solve_sharded_native

    s = _system()
    plan = plan_shards(s.m, 1, 0, q)
    shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
    cfg = SolverConfig(variant=variant, q=q, block_size=bs, base_seed=3, sampling_scheme="distributed")
    rd = solve_sharded_native(shard, cfg)
    rl = solve_sharded_native(shard, cfg, loop=True)
    rb = solve_sharded_native(shard, cfg, budget=17)
    shard.close()
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=3, scheme="distributed")
    ob = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=3, scheme="distributed",
                      budget=17)
    assert rd.converged and rd.iterations == rl.iterations == o["iterations"]
    assert rd.error_evals == o["error_evals"]
    assert rel_err(rd.x, rl.x) <= PARITY_TOL and rel_err(rd.x, o["x"]) <= PARITY_TOL
    assert rb.iterations == 17 and rel_err(rb.x, ob["x"]) <= PARITY_TOL


def test_native_sharded_nccl_world1(gpu):
    """The NCCL communicator path (kz_comm_*, in-place all-reduce on the solve stream) with one
    rank: bitwise the same as the collective-free loop."""
    from paper_2401_17474_b200.multigpu import ShardComm

    s = _system()
    comm = ShardComm(0, 1, 0)
    try:
        rn, rh, _ = _native_vs_host(s, "rka", 8, 1, seed=5, comm=comm)
    finally:
        comm.close()
    assert rn.converged and rn.iterations == rh.iterations
    assert np.array_equal(rn.x, rh.x)


@pytest.mark.parametrize("n,budget", [(64, None), (4500, 40)])
def test_fused_cross_rank_exchange_world1(gpu, oracle, n, budget):
    """kz_solve_sharded's fused path (one launch per chunk, column sums through the communicator's
    NVLink exchange buffers, stop rule in the kernel) at one rank: bit-identical to the
    per-iteration loop, same iteration counts as the oracle; one and several local clusters."""
    from paper_2401_17474_b200 import GeneratorConfig, SolverConfig, generate_mother
    from paper_2401_17474_b200.multigpu import CudaShard, ShardComm, plan_shards, solve_sharded_native

    s = _system() if n == 64 else generate_mother(GeneratorConfig(m_max=5000, n_max=n, seed=3))
    q = 8
    plan = plan_shards(s.m, 1, 0, q)
    shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
    comm = ShardComm(0, 1, 0)
    try:
        cfg = SolverConfig(variant="rka", q=q, base_seed=6, sampling_scheme="distributed")
        rf = solve_sharded_native(shard, cfg, budget=budget, comm=comm)
        rf2 = solve_sharded_native(shard, cfg.replace(base_seed=7), budget=budget, comm=comm)
        rl = solve_sharded_native(shard, cfg, budget=budget, comm=comm, fused=False)
    finally:
        shard.close()
        comm.close()
    assert rf.gpu["fused"] and not rl.gpu["fused"]
    assert rf.iterations == rl.iterations and rf.error_evals == rl.error_evals
    assert np.array_equal(rf.x, rl.x)
    o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=q, base_seed=6, scheme="distributed", budget=budget)
    assert rf.iterations == o["iterations"] and rel_err(rf.x, o["x"]) <= PARITY_TOL
    o2 = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=q, base_seed=7, scheme="distributed", budget=budget)
    assert rf2.iterations == o2["iterations"] and rel_err(rf2.x, o2["x"]) <= PARITY_TOL


@pytest.mark.parametrize("world", [2, 4, 8])
def test_c3_width_world_emulation(gpu, oracle, world):
    """The c3 configuration at N = 2 / 4 / 8 GPUs (64 workers per GPU, bs = 1000, distributed scheme)
    as its one-GPU equivalent -- the sequential solver with q = 64 N, whose workers run in waves --
    on a 64000 x 20000 leading crop of the counter-keyed system, against the oracle at every outer
    iteration; and N emulated ranks (row shards, local steps summed in rank order) bit-identical
    to it for the first two outer iterations (SURVEY 8(c) T5 / T6 at the c3 row width)."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq
    from paper_2401_17474_b200.multigpu import CudaShard, plan_shards

    Q, budget = 64 * world, 2
    with DeviceSystem(m=64000, n=20000) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        cfg = SolverConfig(variant="rkab", q=Q, block_size=1000, base_seed=2, sampling_scheme="distributed")
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=budget, capture=cap)
    assert r.gpu["plan"]["waves"] >= 1 and len(cap) == budget
    o = oracle.solve(A, b, xr, variant="rkab", q=Q, block_size=1000, base_seed=2, scheme="distributed",
                     budget=budget, ckpt_every=1, nthreads=oracle.max_threads())
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, (world, j)
    # the row-sharded protocol: rank g's shard and its 64 workers, the worker sums added in rank order
    shards = [CudaShard(A[p.lo:p.hi + 1], b[p.lo:p.hi + 1], xr, p, device=0)
              for p in (plan_shards(A.shape[0], world, g, 64) for g in range(world))]
    try:
        lcfg = cfg.replace(q=64)
        for sh in shards:
            sh.reset()
        for k in range(budget):
            S = [sh.step(lcfg, k) for sh in shards]
            tot = S[0].clone()
            for extra in S[1:]:
                tot += extra
            for sh in shards:
                sh.finish(tot, Q)
        xs = [sh.x() for sh in shards]
    finally:
        for sh in shards:
            sh.close()
    for x in xs[1:]:
        assert np.array_equal(x, xs[0])
    assert rel_err(xs[0], cap[-1]) <= PARITY_TOL
