"""Tiny and structured systems through the B200 kernels: the reference's unit-level behaviours
(test_solvers_seq.py: one-by-one, orthogonal rows, identity systems, a coherent bundle where
cyclic sweeps crawl, non-convergence flagged not raised, zero weights, the seed-mean error
decreasing) on n = 1, 2, 3 -- edge shapes for the warp, chain and rka kernels -- each checked
against the oracle as well."""

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err

pytestmark = pytest.mark.gpu


def _tiny(a, b, x):
    from paper_2401_17474_b200 import LinearSystem

    a = np.asarray(a, dtype=np.float64)
    return LinearSystem(A=a, b=np.asarray(b, dtype=np.float64), x_star=np.asarray(x, dtype=np.float64), seed=0)


def _coherent():
    """100 nearly parallel unit rows, then 10 spread rows of norm 20 (two unknowns)."""
    th = np.concatenate([np.linspace(0.0, 0.005, 100), np.linspace(0.005, 0.7, 10)])
    a = np.column_stack([np.cos(th), np.sin(th)])
    a[100:] *= 20.0
    return _tiny(a, a @ np.array([1.5, -2.0]), [1.5, -2.0])


def test_one_by_one(gpu):
    from paper_2401_17474_b200 import SolverConfig, solve_ck, solve_rk

    s = _tiny([[2.0]], [6.0], [3.0])
    for fn, variant in ((solve_ck, "ck"), (solve_rk, "rk")):
        r = fn(s, SolverConfig(variant=variant))
        assert r.converged and r.iterations == 1 and np.array_equal(r.x, [3.0]), variant


def test_orthogonal_rows_one_cyclic_sweep(gpu):
    from paper_2401_17474_b200 import SolverConfig, solve_ck

    r = solve_ck(_tiny([[1.0, 0.0], [0.0, 2.0]], [1.0, 4.0], [1.0, 2.0]), SolverConfig(variant="ck"))
    assert r.converged and r.iterations == 2
    assert np.allclose(r.x, [1.0, 2.0], atol=1e-12)


def test_identity_systems(gpu, oracle):
    from paper_2401_17474_b200 import SolverConfig, run_solver

    s = _tiny(np.eye(3), [1.0, 2.0, 3.0], [1.0, 2.0, 3.0])
    for cfg in (SolverConfig(variant="rk", base_seed=4), SolverConfig(variant="rka", q=2, base_seed=4),
                SolverConfig(variant="rkab", q=2, block_size=3, base_seed=4)):
        r = run_solver(s, cfg)
        assert r.converged and np.allclose(r.x, [1.0, 2.0, 3.0], atol=np.sqrt(1e-8)), cfg.variant
        o = oracle.solve(s.A, s.b, s.x_star, variant=cfg.variant, q=cfg.q, block_size=cfg.block_size, base_seed=4)
        assert r.iterations == o["iterations"] and rel_err(r.x, o["x"]) <= PARITY_TOL, cfg.variant


def test_coherent_bundle(gpu, oracle):
    """Cyclic sweeps crawl through the bundle; norm-weighted sampling does not (>= 10x fewer)."""
    from paper_2401_17474_b200 import SolverConfig, solve_ck, solve_rk

    s = _coherent()
    short = solve_ck(s, SolverConfig(variant="ck", max_iterations=10))
    assert not short.converged and short.iterations == 10  # flagged, not raised
    ck = solve_ck(s, SolverConfig(variant="ck", max_iterations=5_000_000))
    rk = [solve_rk(s, SolverConfig(variant="rk", base_seed=k)).iterations for k in range(10)]
    assert ck.converged and ck.iterations >= 10 * np.median(rk)
    o = oracle.solve(s.A, s.b, s.x_star, variant="ck", max_iterations=5_000_000)
    assert ck.iterations == o["iterations"] and rel_err(ck.x, o["x"]) <= PARITY_TOL


def test_zero_weight_is_a_no_op(gpu, systems):
    """alpha = 0 (fixed): every projection scale is 0, x stays at x0 = 0 (RK, RKA, RKAB)."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    s = systems["s500"]
    for kw in (dict(variant="rk"), dict(variant="rka", q=4), dict(variant="rkab", q=3, block_size=5)):
        r = run_solver(s, SolverConfig(alpha_policy="fixed", alpha=0.0, **kw), budget=20)
        assert np.array_equal(r.x, np.zeros(s.n)), kw


def test_seed_mean_error_decreases(gpu, systems):
    """The seed-mean squared error at fixed checkpoints never increases (test_solvers_seq.py:92-104)."""
    from paper_2401_17474_b200 import SolverConfig, trace_run

    s = systems["s500"]
    curves = [[t.error_norm ** 2 for t in trace_run(s, SolverConfig(variant="rk", base_seed=k), 800, 100, s.x_star)]
              for k in range(10)]
    assert np.all(np.diff(np.mean(np.array(curves), axis=0)) <= 0)


@pytest.mark.parametrize("n", [1, 2, 3, 5])
def test_narrow_rows_every_variant(gpu, oracle, n):
    """n = 1..5 columns through RK, RKA (q = 2, 7) and RKAB against the oracle."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, run_solver

    s = generate_mother(GeneratorConfig(m_max=200, n_max=n, seed=9))
    with DeviceSystem(s) as ds:
        for kw in (dict(variant="rk"), dict(variant="rka", q=2), dict(variant="rka", q=7),
                   dict(variant="rkab", q=3, block_size=4)):
            r = run_solver(ds, SolverConfig(base_seed=2, max_iterations=200000, **kw))
            o = oracle.solve(s.A, s.b, s.x_star, q=kw.get("q", 1), block_size=kw.get("block_size", 1), base_seed=2,
                             variant=kw["variant"], max_iterations=200000)
            assert r.iterations == o["iterations"] and r.converged == o["converged"], (n, kw)
            assert rel_err(r.x, o["x"]) <= PARITY_TOL, (n, kw)


def test_row_norm_cache_and_block_sequential(gpu, systems, oracle):
    """row_norm_cache (linalg.py:80-88) on the device: numpy's einsum bit for bit, the total, the
    zero-row error; solve_rk_block_sequential (parallel.py:307-368) is RK's iterate sequence and
    rejects more workers than columns (test_parallel.py:7-30)."""
    from paper_2401_17474_b200 import DegenerateRowError, SolverConfig, row_norm_cache, solve_rk
    from paper_2401_17474_b200 import solve_rk_block_sequential

    s = systems["s500"]
    c = row_norm_cache(s.A)
    assert np.array_equal(c.sq_norms, np.einsum("ij,ij->i", s.A, s.A)) and c.m == s.A.shape[0]
    assert c.frobenius_sq == float(np.einsum("ij,ij->i", s.A, s.A).sum())
    A0 = s.A.copy()
    A0[7] = 0.0
    with pytest.raises(DegenerateRowError) as exc:
        row_norm_cache(A0)
    assert exc.value.row == 7
    rk = solve_rk(s, SolverConfig(variant="rk", base_seed=3))
    for q in (1, 4):
        par = solve_rk_block_sequential(s, SolverConfig(variant="rk", q=q, base_seed=3))
        assert par.iterations == rk.iterations and np.array_equal(par.x, rk.x)
    with pytest.raises(ValueError):
        solve_rk_block_sequential(s, SolverConfig(variant="rk", q=s.n + 1, base_seed=0))
