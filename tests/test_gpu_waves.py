"""Workers beyond the co-resident CTAs (RKAB, solvers.py:337-371, with q larger than the chain
kernel can hold at once): each outer iteration runs its workers in waves, every wave adding its
ordered worker sum to the previous waves' (bit-identical to one launch over all q), then
x = S / q and the stop rule (kz_solve_sharded's per-iteration driver).  Against the oracle at
every outer iteration; the reference accepts any q (SolverConfig.validate, solvers.py:85-101)."""

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err

pytestmark = pytest.mark.gpu


def test_rkab_waves_one_cta_per_worker(gpu, oracle):
    """q = 200 on rows of 1000 columns: one CTA per worker, 148 co-resident -> two waves."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rkab_seq

    s = generate_mother(GeneratorConfig(m_max=20000, n_max=1000, seed=2))
    cfg = SolverConfig(variant="rkab", q=200, block_size=20, base_seed=4)
    with DeviceSystem(s) as ds:
        cap = []
        r = solve_rkab_seq(ds, cfg, capture=cap)
        rb = solve_rkab_seq(ds, cfg, budget=r.iterations)
    assert r.gpu["plan"]["waves"] >= 2, r.gpu
    o = oracle.solve(s.A, s.b, s.x_star, variant="rkab", q=200, block_size=20, base_seed=4, ckpt_every=1,
                     nthreads=oracle.max_threads())
    assert r.converged and r.iterations == o["iterations"] and r.error_evals == o["error_evals"]
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, j
    assert rel_err(r.x, o["x"]) <= PARITY_TOL
    assert rb.error_evals == 0 and np.array_equal(rb.x, r.x)  # budget replay: same iterate


def test_rkab_waves_on_cta_pairs_long_rows(gpu, oracle):
    """q = 160 on the c3 row width (n = 20000): pairs of CTAs per worker, 74 co-resident ->
    three waves; a leading crop of the counter-keyed c3 system, distributed scheme."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq

    with DeviceSystem(m=32000, n=20000) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        cfg = SolverConfig(variant="rkab", q=160, block_size=40, base_seed=1, sampling_scheme="distributed")
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=3, capture=cap)
    assert r.gpu["plan"]["cluster"] == 2 and r.gpu["plan"]["waves"] >= 3, r.gpu
    o = oracle.solve(A, b, xr, variant="rkab", q=160, block_size=40, base_seed=1, scheme="distributed", budget=3,
                     ckpt_every=1, nthreads=oracle.max_threads())
    assert len(cap) == 3
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, j


def test_rka_on_chain_in_waves(gpu, oracle):
    """RKA forced onto the chain kernel with q = 300 on rows of 1000 columns (block_size 1, one
    CTA per worker, two waves) against the oracle, every 100 iterations."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rka_seq

    s = generate_mother(GeneratorConfig(m_max=6000, n_max=1000, seed=5))
    cfg = SolverConfig(variant="rka", q=300, base_seed=7, kernel="chain", max_iterations=1500)
    with DeviceSystem(s) as ds:
        cap = []
        r = solve_rka_seq(ds, cfg, checkpoint_every=100, capture=cap)
    assert r.gpu["plan"]["waves"] >= 2, r.gpu
    o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=300, base_seed=7, max_iterations=1500, ckpt_every=100,
                     nthreads=oracle.max_threads())
    assert r.iterations == o["iterations"] and r.converged == o["converged"]
    assert rel_err(r.x, o["x"]) <= PARITY_TOL
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, j


def test_rka_beyond_512_workers(gpu, oracle):
    """RKA with q = 600: past the column-sliced kernels' 512 workers, the chain kernel in waves."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rka_seq

    s = generate_mother(GeneratorConfig(m_max=8000, n_max=600, seed=6))
    cfg = SolverConfig(variant="rka", q=600, base_seed=2, max_iterations=800)
    with DeviceSystem(s) as ds:
        r = solve_rka_seq(ds, cfg)
    assert r.gpu["kernel"] == "chain", r.gpu
    o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=600, base_seed=2, max_iterations=800,
                     nthreads=oracle.max_threads())
    assert r.iterations == o["iterations"] and rel_err(r.x, o["x"]) <= PARITY_TOL


def test_rkab_rows_beyond_a_pair(gpu, oracle):
    """RKAB on n = 24000 (> 2 x 10240 columns): workers of 4 CTAs (chain_kernel<16, 1, 4, WIDE>),
    16 workers -> 64 CTAs; q = 48 -> 192 CTAs in waves; a counter-keyed crop, every outer iteration."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq

    with DeviceSystem(m=24000, n=24000) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        for q in (16, 48):
            cfg = SolverConfig(variant="rkab", q=q, block_size=30, base_seed=3, sampling_scheme="distributed")
            cap = []
            r = solve_rkab_seq(ds, cfg, budget=2, capture=cap)
            assert r.gpu["plan"]["cluster"] == 4, r.gpu
            assert (r.gpu["plan"]["waves"] > 1) == (q == 48), r.gpu
            o = oracle.solve(A, b, xr, variant="rkab", q=q, block_size=30, base_seed=3, scheme="distributed",
                             budget=2, ckpt_every=1, nthreads=oracle.max_threads())
            for j, ck in enumerate(o["checkpoints"]):
                assert rel_err(cap[j], ck) <= PARITY_TOL, (q, j)
