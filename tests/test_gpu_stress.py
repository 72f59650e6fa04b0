"""Protocol stress: the kernels' asynchronous protocols (mbarrier rings, st.async pushes into
peer CTAs' shared memory, tagged words polled across clusters and over the cross-rank exchange
buffers, grid barriers) repeated many times on small systems.  A missing acquire, a reused slot
or a lost arrival shows up as a hang (the spin bounds turn it into an error), as results that
differ between repeats, or as a drift from the oracle -- every repeat must be bit-identical
and match the oracle.  (compute-sanitizer is closed on the GPU pool; see profiles/README.md.)"""

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err

pytestmark = pytest.mark.gpu

REPEATS = 20


def _sys(m, n, seed=3):
    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    return generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=seed))


CASES = [  # (id, (m, n), SolverConfig kwargs, expected kernel)
    ("rka_one_cluster", (2000, 500), dict(variant="rka", q=64), "rka"),
    ("rka_two_clusters", (2000, 500), dict(variant="rka", q=64, kernel="sync_cluster", ctas=32), "rka"),
    ("rka_seven_clusters", (4000, 2000), dict(variant="rka", q=64, kernel="sync_cluster", ctas=112,
                                                     max_iterations=300), "rka"),
    ("rka_worker_groups", (4000, 500), dict(variant="rka", q=300, max_iterations=400), "rka"),
    ("sync_grid", (2000, 500), dict(variant="rka", q=64, kernel="sync_grid"), "sync_grid"),
    ("chain_rkab", (2000, 50), dict(variant="rkab", q=16, block_size=10), "chain"),
    ("chain_pairs", (6000, 3000), dict(variant="rkab", q=8, block_size=20, max_iterations=10), "chain"),
    ("chain_cluster4", (3000, 2000), dict(variant="rk", max_iterations=500), "chain"),
    ("chain_threads", (2000, 50), dict(variant="rka", q=8, engine="threads"), "chain"),
    ("warp", (2000, 50), dict(variant="rk"), "warp"),
]


@pytest.mark.parametrize("case", CASES, ids=[c[0] for c in CASES])
def test_repeated_solves_are_bit_identical(gpu, oracle, case):
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver

    name, (m, n), kw, kernel = case
    s = _sys(m, n)
    cfgs = [SolverConfig(base_seed=k % 3, **kw) for k in range(REPEATS)]
    with DeviceSystem(s) as ds:
        runs = [run_solver(ds, c) for c in cfgs]
    assert runs[0].gpu["kernel"] == kernel, runs[0].gpu
    for k, r in enumerate(runs[3:], start=3):
        ref = runs[k % 3]
        assert r.iterations == ref.iterations and r.error_evals == ref.error_evals, (name, k)
        assert np.array_equal(r.x, ref.x), (name, k)
    engine = "threads" if kw.get("engine") == "threads" else "seq"
    for seed in range(3):
        o = oracle.solve(s.A, s.b, s.x_star, variant=kw["variant"], q=kw.get("q", 1),
                         block_size=kw.get("block_size", 1), base_seed=seed, engine=engine,
                         max_iterations=kw.get("max_iterations", 1_000_000))
        assert runs[seed].iterations == o["iterations"], (name, seed)
        assert rel_err(runs[seed].x, o["x"]) <= PARITY_TOL, (name, seed)


def test_fused_exchange_repeated(gpu):
    """rka kernel mode 2 (cross-rank exchange buffers, slot parity by global iteration, tags
    advancing across launches and solves) at one rank: many solves on one communicator."""
    from paper_2401_17474_b200 import SolverConfig
    from paper_2401_17474_b200.multigpu import CudaShard, ShardComm, plan_shards, solve_sharded_native

    s = _sys(5000, 2000)
    plan = plan_shards(s.m, 1, 0, 8)
    shard = CudaShard(s.A, s.b, s.x_star, plan, device=0)
    comm = ShardComm(0, 1, 0)
    try:
        cfg = SolverConfig(variant="rka", q=8, sampling_scheme="distributed")
        runs = [solve_sharded_native(shard, cfg.replace(base_seed=k % 2), budget=40 + (k % 2), comm=comm)
                for k in range(REPEATS)]
    finally:
        shard.close()
        comm.close()
    assert runs[0].gpu["fused"]
    for k, r in enumerate(runs[2:], start=2):
        assert r.iterations == runs[k % 2].iterations and np.array_equal(r.x, runs[k % 2].x), k
