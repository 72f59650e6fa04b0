"""Multi-rank host logic on CPU (gloo, world_size 2): shard planning, worker
ids / ranges, the all-reduce-sum + average protocol and rank agreement of the
row-sharded RKA / RKAB driver (paper_2401_17474_b200.multigpu), checked
against the sequential oracle with q_total workers and the distributed
scheme (reference distributed.py:189-336)."""

import os
import socket

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_plan_shards_nest_and_tile():
    from paper_2401_17474_b200.multigpu import plan_shards
    from paper_2401_17474_b200 import partition_bounds

    for m in (160000, 20000, 1001, 97):
        for G in (1, 2, 3, 4, 8):
            for q in (1, 3, 64):
                if m < G * q:
                    continue
                covered = []
                for g in range(G):
                    p = plan_shards(m, G, g, q)
                    for w, (lo, ln) in enumerate(zip(p.worker_lo, p.worker_len)):
                        t = g * q + w
                        a, b = partition_bounds(m, G * q, t)
                        assert (p.lo + lo, p.lo + lo + ln - 1) == (a, b)
                        covered.extend(range(a, b + 1))
                assert covered == list(range(m))


def _rank_main(rank, world, port, variant, bs, q_local, budget, out_dir):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle.local_step import CpuShard
    from paper_2401_17474_b200 import GeneratorConfig, SolverConfig, generate_mother
    from paper_2401_17474_b200.multigpu import plan_shards, solve_sharded

    s = generate_mother(GeneratorConfig(m_max=600, n_max=20, seed=3))
    plan = plan_shards(s.m, world, rank, q_local)
    shard = CpuShard(s.A[plan.lo:plan.hi + 1], s.b[plan.lo:plan.hi + 1], s.x_star, plan)
    cfg = SolverConfig(variant=variant, q=q_local, block_size=bs, base_seed=4, sampling_scheme="distributed")
    r = solve_sharded(shard, cfg, budget=budget)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=r.x, it=r.iterations, ev=r.error_evals,
             conv=r.converged)
    dist.destroy_process_group()


@pytest.mark.parametrize("variant,bs,budget", [("rka", 1, None), ("rkab", 4, None), ("rka", 1, 37)])
def test_two_rank_driver_matches_sequential_oracle(tmp_path, oracle, variant, bs, budget):
    import torch.multiprocessing as mp

    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    world, q_local = 2, 3
    mp.spawn(_rank_main, args=(world, _free_port(), variant, bs, q_local, budget, str(tmp_path)), nprocs=world)
    r0, r1 = (np.load(tmp_path / f"r{i}.npz") for i in range(world))
    assert np.array_equal(r0["x"], r1["x"])  # rank agreement, bitwise
    assert int(r0["it"]) == int(r1["it"])
    s = generate_mother(GeneratorConfig(m_max=600, n_max=20, seed=3))
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=world * q_local, block_size=bs, base_seed=4,
                     scheme="distributed", budget=budget)
    assert int(r0["it"]) == o["iterations"]
    if budget is None:
        assert bool(r0["conv"]) and int(r0["ev"]) == o["error_evals"]
    assert rel_err(r0["x"], o["x"]) <= PARITY_TOL
