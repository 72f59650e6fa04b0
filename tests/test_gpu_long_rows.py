"""Long rows (n >= 2000): every chain-kernel instantiation the planner picks above n = 2048
against the oracle, on leading crops of BASELINE config 3's counter-keyed system (entries
depend only on (seed, i, j), so these are exact crops of the 160000 x 20000 matrix).

* RKAB q = 8 on CTA pairs: n = 3000 plans EP 8 (R 2), n = 8192 and n = 20000 plan EP 16
  (R 1) -- the c3 headline kernel ``chain_kernel<16, 1, 2>``.  Every outer iteration is
  checkpointed (solvers.py:361-367 averaging) and compared at 1e-10.
* RK and CK (q = 1) on a cluster of 4 CTAs at n = 4100, 8192, 20000: EP 8 / 16 with
  R 2 / 1 (solvers.py:294-310, 271-291), checkpoints every 100 iterations (T2).
* BASELINE c4 at full shape (80000 x 2000 inconsistent): the horizon runs' iterates (RK, RKA
  q = 64, q = 512) every 1000 iterations.
"""

import numpy as np
import pytest

from conftest import PARITY_TOL, rel_err

pytestmark = pytest.mark.gpu


def _crop(m, n):
    from paper_2401_17474_b200 import DeviceSystem

    ds = DeviceSystem(m=m, n=n)
    ds.generate_counter(0)
    A, b, xr = ds.download()
    return ds, A, b, xr


@pytest.mark.parametrize("n,ep,rows", [(3000, 8, 2), (8192, 16, 1), (20000, 16, 1)])
def test_rkab_long_rows_every_outer_iteration(gpu, oracle, n, ep, rows):
    from paper_2401_17474_b200 import SolverConfig, solve_rkab_seq

    ds, A, b, xr = _crop(24000, n)
    with ds:
        cfg = SolverConfig(variant="rkab", q=8, block_size=50, base_seed=3, sampling_scheme="distributed")
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=4, capture=cap)
    assert r.gpu["kernel"] == "chain" and r.gpu["plan"]["cluster"] == 2, r.gpu
    assert (r.gpu["plan"]["ep"], r.gpu["plan"]["rows"]) == (ep, rows), r.gpu
    o = oracle.solve(A, b, xr, variant="rkab", q=8, block_size=50, base_seed=3, scheme="distributed", budget=4,
                     ckpt_every=1, nthreads=oracle.max_threads())
    assert r.iterations == 4 and len(cap) == 4
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, j
    assert rel_err(r.x, o["x"]) <= PARITY_TOL


def test_rkab_c3_width_q64_bs1000(gpu, oracle):
    """The c3 headline configuration itself (q = 64, bs = 1000, distributed scheme, n = 20000)
    on a 64000-row leading crop (1000 rows per worker block), two outer iterations."""
    from paper_2401_17474_b200 import SolverConfig, solve_rkab_seq

    ds, A, b, xr = _crop(64000, 20000)
    with ds:
        cfg = SolverConfig(variant="rkab", q=64, block_size=1000, base_seed=0, sampling_scheme="distributed")
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=2, capture=cap)
    assert (r.gpu["plan"]["ep"], r.gpu["plan"]["rows"], r.gpu["plan"]["cluster"]) == (16, 1, 2), r.gpu
    assert r.gpu["ctas"] == 128
    o = oracle.solve(A, b, xr, variant="rkab", q=64, block_size=1000, scheme="distributed", budget=2, ckpt_every=1,
                     nthreads=oracle.max_threads())
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[j], ck) <= PARITY_TOL, j
    assert rel_err(r.x, o["x"]) <= PARITY_TOL


@pytest.mark.parametrize("variant", ["rk", "ck"])
@pytest.mark.parametrize("n,ep", [(4100, 8), (8192, 8), (20000, 16)])
def test_long_chain_rk_ck_matches_oracle(gpu, oracle, variant, n, ep):
    from paper_2401_17474_b200 import SolverConfig, run_solver

    ds, A, b, xr = _crop(6000, n)
    budget = 600
    with ds:
        cap = []
        r = run_solver(ds, SolverConfig(variant=variant, base_seed=4), budget=budget, capture=cap)
    assert r.gpu["kernel"] == "chain" and r.gpu["plan"]["cluster"] == 4 and r.gpu["plan"]["ep"] == ep, r.gpu
    o = oracle.solve(A, b, xr, variant=variant, base_seed=4, budget=budget, ckpt_every=100)
    assert r.iterations == budget
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[100 * (j + 1) - 1], ck) <= PARITY_TOL, j
    assert rel_err(r.x, o["x"]) <= PARITY_TOL


def test_rk_long_chain_stop_rule(gpu, oracle):
    """RK to ||x - x*||^2 < eps on a short wide crop: stop decisions, iteration counts and
    error_evals equal to the oracle's (the stop rule rides along the Gram-block reduction)."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    ds, A, b, xr = _crop(6000, 4100)
    eps = 0.3 * float(xr @ xr)  # ||x0 - x*||^2 = ||x*||^2: a threshold the chain crosses mid-run
    with ds:
        r = run_solver(ds, SolverConfig(variant="rk", base_seed=1, epsilon=eps, max_iterations=20000))
    o = oracle.solve(A, b, xr, variant="rk", base_seed=1, epsilon=eps, max_iterations=20000)
    assert o["converged"]
    assert r.iterations == o["iterations"] and r.converged == o["converged"] and r.error_evals == o["error_evals"]
    assert rel_err(r.x, o["x"]) <= PARITY_TOL


def test_chain_limits_are_errors_not_crashes(gpu):
    """Rows wider than the chain kernel's register-resident iterate raise ValueError
    (KZ_EINVAL) instead of failing inside a launch."""
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver

    with DeviceSystem(m=64, n=82000) as ds:  # past one chain of 8 CTAs (81920 columns)
        ds.generate_counter(0)
        with pytest.raises(ValueError):
            run_solver(ds, SolverConfig(variant="rk"), budget=1)
        with pytest.raises(ValueError):
            run_solver(ds, SolverConfig(variant="rkab", q=4, block_size=2), budget=1)


@pytest.fixture(scope="module")
def c4_inconsistent():
    """BASELINE c4: generate_mother(80000, 2000, seed 0), b_LS = b + xi (sysgen.py:175-176, noise seed 0),
    x_LS by the device CGLS (pinned to the reference's CGLS in test_gpu_solves / test_host)."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, LinearSystem, generate_mother
    from paper_2401_17474_b200.sysgen import inconsistent_rhs

    s = generate_mother(GeneratorConfig(m_max=80000, n_max=2000, seed=0))
    b_ls = inconsistent_rhs(s, 0)
    inc = LinearSystem(A=s.A, b=b_ls, x_star=None, x_ls=None, consistent=False, seed=0)
    ds = DeviceSystem(inc)
    x_ls = ds.cgls(tol=1e-12)
    yield ds, inc, x_ls
    ds.close()


@pytest.mark.parametrize("variant,q,budget", [("rk", 1, 120000), ("rka", 64, 60000), ("rka", 512, 48000)])
def test_c4_horizon_iterates_match_oracle(gpu, oracle, c4_inconsistent, variant, q, budget):
    """The full c4 horizon runs (80000 x 2000 inconsistent, the SURVEY 8(d) budgets, seed 0): the iterate every 1000
    iterations against the oracle at 1e-10 (the bench's trace records are ||x - x_LS|| of these
    iterates), and the distance to x_LS at the last checkpoint equal to the oracle's."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    ds, inc, x_ls = c4_inconsistent
    cfg = SolverConfig(variant=variant, q=q, base_seed=0)
    cap = []
    r = run_solver(ds, cfg, budget=budget, checkpoint_every=1000, capture=cap)
    o = oracle.solve(inc.A, inc.b, x_ls, variant=variant, q=q, base_seed=0, budget=budget, ckpt_every=1000,
                     nthreads=oracle.max_threads())
    assert r.iterations == budget and len(o["checkpoints"]) == budget // 1000 == len(cap)
    for j, ck in enumerate(o["checkpoints"]):  # cap[j]: the iterate after 1000 (j + 1) iterations
        assert rel_err(cap[j], ck) <= PARITY_TOL, (variant, q, j)
    h_gpu = float(np.linalg.norm(cap[-1] - x_ls))
    h_ora = float(np.linalg.norm(o["checkpoints"][-1] - x_ls))
    assert abs(h_gpu - h_ora) <= 1e-8 * h_ora


def test_rows_beyond_40960_columns(gpu, oracle):
    """n = 50000: RK on one chain of 8 CTAs (chain_kernel<16, 1, 8>) and RKAB on workers of 8 CTAs
    (WIDE) against the oracle (a 4000-row crop of the counter-keyed generator: the loop does not
    need m >= n)."""
    from paper_2401_17474_b200 import SolverConfig, run_solver

    ds, A, b, xr = _crop(4000, 50000)
    with ds:
        cap = []
        r = run_solver(ds, SolverConfig(variant="rk", base_seed=4), budget=300, capture=cap)
        assert r.gpu["plan"]["cluster"] == 8, r.gpu
        o = oracle.solve(A, b, xr, variant="rk", base_seed=4, budget=300, ckpt_every=50)
        for j, ck in enumerate(o["checkpoints"]):
            assert rel_err(cap[50 * (j + 1) - 1], ck) <= PARITY_TOL, j
        cap = []
        cfg = SolverConfig(variant="rkab", q=6, block_size=20, base_seed=1, sampling_scheme="distributed")
        r = run_solver(ds, cfg, budget=2, capture=cap)
        assert r.gpu["plan"]["cluster"] == 8, r.gpu
        o = oracle.solve(A, b, xr, variant="rkab", q=6, block_size=20, base_seed=1, scheme="distributed", budget=2,
                         ckpt_every=1)
        for j, ck in enumerate(o["checkpoints"]):
            assert rel_err(cap[j], ck) <= PARITY_TOL, j
