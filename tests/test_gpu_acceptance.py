"""The reference's acceptance criteria (test_acceptance.py:94-250) re-run through the B200 engine:
sampler statistics, the averaging and block-size trends, the convergence horizons of an
inconsistent system, the optimal weight's effect, CGLS.  (Criteria 01-03 are
test_gpu_solves.py::test_reduction_identities_bitwise / test_projection_property_1000_steps and
test_gpu_threads.py; 10 is test_gpu_solves.py::test_run_distributed_solve_matches_reference; 12 is
the CLI, out of scope.)"""

import math

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_sampler_statistics(gpu):
    """100k seeded device draws from a 6-row sampler: within 3 standard errors of the
    squared-norm distribution, and identical when drawn again."""
    from paper_2401_17474_b200 import DeviceSystem

    sq = np.array([1.0, 2.5, 4.0, 6.0, 9.0, 12.5])
    A = np.zeros((6, 2))
    A[:, 0] = np.sqrt(sq)
    with DeviceSystem(m=6, n=2) as ds:
        ds.upload(A, np.zeros(6))
        d1 = ds.dump_rows(777, 0, 100_000)
        d2 = ds.dump_rows(777, 0, 100_000)
    assert np.array_equal(d1, d2)
    exact = sq / sq.sum()
    for i in range(6):
        f = float(np.mean(d1 == i))
        assert abs(f - exact[i]) <= 3 * math.sqrt(exact[i] * (1 - exact[i]) / 100_000), i


def _mean_iterations(ds, seeds=10, **kw):
    from paper_2401_17474_b200 import SolverConfig, solve_concurrent

    return float(np.mean([r.iterations for r in solve_concurrent(ds, [SolverConfig(base_seed=k, **kw)
                                                                       for k in range(seeds)])]))


def test_averaging_and_block_size_trends(gpu, systems):
    """Unit-weight RKA needs strictly fewer iterations as q grows (1 > 4 > 16); RKAB's outer
    iterations drop strictly with the block size (5 > 10 > 50) while its total rows stay within 2x."""
    from paper_2401_17474_b200 import DeviceSystem

    with DeviceSystem(systems["s2000"]) as ds:
        rka = [_mean_iterations(ds, variant="rka" if q > 1 else "rk", q=q) for q in (1, 4, 16)]
        assert rka[0] > rka[1] > rka[2], rka
        rkab = [_mean_iterations(ds, variant="rkab", q=4, block_size=bs) for bs in (5, 10, 50)]
        assert rkab[0] > rkab[1] > rkab[2], rkab
        rows = [m * 4 * bs for m, bs in zip(rkab, (5, 10, 50))]
        assert max(rows) / min(rows) <= 2.0, rows


def test_convergence_horizons(gpu, inc2000):
    """The error plateau against x_LS shrinks by >= 20 % per worker jump (RKA q 1 -> 5 -> 20), and the
    block variant at block = n agrees (q 1 -> 20)."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, plateau_error, trace_run

    s = inc2000
    with DeviceSystem(s) as ds:
        p = {q: plateau_error(trace_run(ds, SolverConfig(variant="rka" if q > 1 else "rk", q=q, base_seed=1), 30_000,
                                        100, s.x_ls)) for q in (1, 5, 20)}
        assert p[5] <= 0.8 * p[1] and p[20] <= 0.8 * p[5], p
        b = {q: plateau_error(trace_run(ds, SolverConfig(variant="rkab", q=q, block_size=s.n, base_seed=1), 600, 2,
                                        s.x_ls)) for q in (1, 20)}
        assert b[20] < b[1], b


def test_optimal_weight_cuts_iterations(gpu, systems):
    """The optimal uniform weight (device spectral estimate) cuts 8-worker iterations to <= 0.5x."""
    from paper_2401_17474_b200 import DeviceSystem
    from paper_2401_17474_b200.spectral import optimal_alpha, spectral_stats

    with DeviceSystem(systems["s2000"]) as ds:
        alpha = optimal_alpha(spectral_stats(ds), 8)
        unit = _mean_iterations(ds, variant="rka", q=8)
        best = _mean_iterations(ds, variant="rka", q=8, alpha_policy="fixed", alpha=alpha)
    assert best <= 0.5 * unit, (best, unit)


def test_cgls_criterion(gpu, inc2000, systems):
    """CGLS reaches the least-squares normal-equations tolerance on the inconsistent system and
    recovers x* on a consistent one (run_solver variant "cgls", harness.py:72-95)."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    r = run_solver(inc2000, SolverConfig(variant="cgls"))
    A, b = inc2000.A, inc2000.b
    assert np.linalg.norm(A.T @ (A @ r.x - b)) <= 1e-9 * np.linalg.norm(A.T @ b)
    s = systems["s500"]
    r2 = run_solver(s, SolverConfig(variant="cgls"))
    assert np.max(np.abs(r2.x - s.x_star)) <= 1e-6 * np.max(np.abs(s.x_star))
