"""Concurrent solves of one resident system (kz_system_view + solve_concurrent): every
report is bit-identical to the same solve run alone, for the chain kernel (RK, RKAB) and
the rka kernel (one cluster, several clusters, worker groups), and the harness protocol
(measure_iterations) gives the same counts either way."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _alone_and_together(system, cfgs, lanes, budget=None):
    from paper_2401_17474_b200 import DeviceSystem, run_solver, solve_concurrent

    with DeviceSystem(system) as ds:
        alone = [run_solver(ds, c, budget=budget) for c in cfgs]
        together = solve_concurrent(ds, cfgs, lanes=lanes, budget=budget)
    return alone, together


@pytest.mark.parametrize("variant,q,bs,lanes", [("rk", 1, 1, 5), ("rka", 64, 1, 7), ("rkab", 8, 20, 4),
                                                ("rka", 64, 1, 10)])
def test_concurrent_equals_sequential(gpu, systems, variant, q, bs, lanes):
    from paper_2401_17474_b200 import SolverConfig

    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    s = systems["c0"] if variant == "rk" else generate_mother(GeneratorConfig(m_max=4000, n_max=200, seed=11))
    cfgs = [SolverConfig(variant=variant, q=q, block_size=bs, base_seed=k) for k in range(10)]
    alone, together = _alone_and_together(s, cfgs, lanes)
    for a, t in zip(alone, together):
        assert t.converged == a.converged and t.iterations == a.iterations and t.error_evals == a.error_evals
        assert t.final_error_sq == a.final_error_sq
        assert np.array_equal(t.x, a.x)


@pytest.mark.parametrize("n,q", [(5000, 32), (1000, 300)])
def test_concurrent_multi_cluster_budget(gpu, n, q):
    """Several clusters per solve (tagged-word exchange; worker groups for q = 300) in concurrent lanes."""
    from paper_2401_17474_b200 import GeneratorConfig, SolverConfig, generate_mother

    s = generate_mother(GeneratorConfig(m_max=6000, n_max=n, seed=4))
    cfgs = [SolverConfig(variant="rka", q=q, base_seed=k) for k in range(4)]
    alone, together = _alone_and_together(s, cfgs, 2, budget=40)
    for a, t in zip(alone, together):
        assert t.iterations == a.iterations == 40 and np.array_equal(t.x, a.x)


def test_measure_iterations_lanes(gpu, systems):
    from paper_2401_17474_b200 import Protocol, SolverConfig, measure_iterations

    s = systems["c0"]
    cfg = SolverConfig(variant="rka", q=4)
    seq = measure_iterations(s, cfg, Protocol(n_seeds=6), lanes=1)
    par = measure_iterations(s, cfg, Protocol(n_seeds=6))
    assert [r.iterations for r in seq.reports] == [r.iterations for r in par.reports]
    assert seq.budget == par.budget


def test_view_refuses_writes(gpu, systems):
    from paper_2401_17474_b200 import DeviceSystem

    s = systems["c0"]
    with DeviceSystem(s) as ds:
        v = ds.view()
        try:
            with pytest.raises(ValueError):
                v.upload(s.A, s.b, s.x_star)
        finally:
            v.close()


def test_views_follow_reupload(gpu, systems):
    """Cached lane views stay attached across a re-upload of the base (kz_system_view_refresh):
    solves after the upload see the new system."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver, solve_concurrent

    a, b = systems["c0"], systems["s2000"]
    cfgs = [SolverConfig(variant="rka", q=4, base_seed=k) for k in range(4)]
    with DeviceSystem(a) as ds:
        solve_concurrent(ds, cfgs, lanes=4)
        ds.upload(b.A, b.b, b.x_star)
        together = solve_concurrent(ds, cfgs, lanes=4)
        alone = [run_solver(ds, c) for c in cfgs]
    for t, s_ in zip(together, alone):
        assert t.iterations == s_.iterations and np.array_equal(t.x, s_.x)


def test_concurrent_traces_with_shared_reference(gpu, inc2000):
    """Trace mode side by side with one x_ref for all solves (the c4 horizon protocol): the
    trace records equal those of the solves run alone."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver, solve_concurrent

    s = inc2000
    x_ls = s.x_ls if s.x_ls is not None else None
    cfgs = [SolverConfig(variant="rka", q=8, base_seed=k, max_iterations=3000) for k in range(4)]
    with DeviceSystem(s) as ds:
        xr = x_ls if x_ls is not None else ds.cgls(tol=1e-12)
        alone = [run_solver(ds, c, x_ref=xr, trace_step=500) for c in cfgs]
        together = solve_concurrent(ds, cfgs, lanes=4, x_ref=xr, trace_step=500)
    for a, t in zip(alone, together):
        assert [(r.iteration, r.error_norm, r.residual_norm) for r in a.trace] == \
               [(r.iteration, r.error_norm, r.residual_norm) for r in t.trace]
        assert np.array_equal(a.x, t.x)


@pytest.mark.parametrize("budget", [None, 2500])
def test_seed_batch_equals_solves_alone(gpu, systems, budget):
    """kz_solve_seeds (one warp per seed, one launch per chunk for all seeds) vs each seed solved
    alone on the warp kernel: bit-identical iterates, same counts, errors and residuals; and
    against the reference's own c0 runs (tests/golden/solves.npz)."""
    from conftest import PARITY_TOL, golden, rel_err

    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver, solve_concurrent, solve_seeds

    s = systems["c0"]
    cfg = SolverConfig(variant="rk")
    with DeviceSystem(s) as ds:
        batch = solve_seeds(ds, cfg, list(range(10)), budget=budget)
        alone = [run_solver(ds, cfg.replace(base_seed=k), budget=budget) for k in range(10)]
        via = solve_concurrent(ds, [cfg.replace(base_seed=k) for k in range(10)], budget=budget)
    for b, a, v in zip(batch, alone, via):
        assert b.gpu["seed_batch"] == 10 and v.gpu.get("seed_batch") == 10
        assert b.iterations == a.iterations and b.converged == a.converged and b.error_evals == a.error_evals
        assert np.array_equal(b.x, a.x) and np.array_equal(v.x, b.x)
        if budget is None:
            assert b.final_error_sq == a.final_error_sq
            assert abs(b.final_residual - a.final_residual) <= 1e-12 * (1 + a.final_residual)
    if budget is None:
        g = golden("solves.npz")
        for k, b in enumerate(batch):
            assert b.iterations == int(g[f"c0_rk_s{k}_iterations"])
            assert rel_err(b.x, g[f"c0_rk_s{k}_x"]) <= PARITY_TOL
