"""engine="threads" on the B200 (solve_rka_parallel / solve_rkab_parallel, parallel.py:175-304):
the threaded engine's combine in worker order on the chain kernel, against the oracle's
restatement (1e-10 per checkpoint) and the reference's own threaded runs (tests/golden/threads.npz,
within the reference's threads-vs-seq tolerance 1e-9, test_parallel.py:38-44)."""

import numpy as np
import pytest

from conftest import PARITY_TOL, golden, rel_err

pytestmark = pytest.mark.gpu


def _cases():
    from golden.common import THREAD_CASES

    return THREAD_CASES


@pytest.mark.parametrize("case", _cases(), ids=[c[0] for c in _cases()])
def test_threaded_engine_matches_reference_and_oracle(gpu, oracle, case):
    from golden.common import THREADS_TOL

    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, run_solver

    name, (m, n, seed), variant, q, bs, base = case
    g = golden("threads.npz")
    s = generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=seed))
    cfg = SolverConfig(variant=variant, q=q, block_size=bs, base_seed=base, engine="threads")
    with DeviceSystem(s) as ds:
        cap = []
        r = run_solver(ds, cfg, capture=cap)
    assert r.gpu["kernel"] == "chain"
    assert r.iterations == int(g[f"{name}_it"]) and r.converged
    assert r.barrier_events == 2 * (r.iterations + 1)  # test_parallel.py:62-65
    assert rel_err(r.x, g[f"{name}_x"]) <= THREADS_TOL
    for j, ck in enumerate(g[f"{name}_ckpt"]):
        assert rel_err(cap[10 * (j + 1) - 1], ck) <= THREADS_TOL, (name, j)
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=base, engine="threads",
                     ckpt_every=1)
    assert r.iterations == o["iterations"]
    for k, (a, b) in enumerate(zip(cap, o["checkpoints"])):
        assert rel_err(a, b) <= PARITY_TOL, (name, k)


def test_threaded_rka_q1_is_rk(gpu, systems):
    """test_parallel.py:32-36: one worker is sequential RK (same iterations; x to rounding)."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    s = systems["s500"]
    rk = run_solver(s, SolverConfig(variant="rk", base_seed=5))
    par = run_solver(s, SolverConfig(variant="rka", q=1, base_seed=5, engine="threads"))
    assert par.iterations == rk.iterations
    assert rel_err(par.x, rk.x) <= PARITY_TOL


def test_threaded_engine_budget_and_errors(gpu, systems):
    """Fixed-budget replay runs the same combine; tracing is rejected as in harness.py:106-108."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    s = systems["s2000"]
    cfg = SolverConfig(variant="rka", q=8, base_seed=3, engine="threads")
    full = run_solver(s, cfg)
    rep = run_solver(s, cfg, budget=full.iterations)
    assert rep.error_evals == 0 and np.array_equal(rep.x, full.x)
    with pytest.raises(ValueError):
        run_solver(s, cfg, trace_step=10)
