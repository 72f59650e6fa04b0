"""T2-T4, T7: full B200 solves against the reference's own solves (golden
fixtures) and the oracle: iteration counts equal, error_evals equal, every
checkpoint within 1e-10 relative; the reference's KATs and reduction
identities re-run through the B200 engine."""

import numpy as np
import pytest

from conftest import PARITY_TOL, golden, rel_err

pytestmark = pytest.mark.gpu


def _cfg(**kw):
    from paper_2401_17474_b200 import SolverConfig

    return SolverConfig(**kw)


def _check(report, g, tag, cap=None):
    assert report.iterations == int(g[f"{tag}_iterations"]), tag
    assert report.error_evals == int(g[f"{tag}_error_evals"]), tag
    assert report.converged == bool(g[f"{tag}_converged"]), tag
    assert rel_err(report.x, g[f"{tag}_x"]) <= PARITY_TOL, tag
    if cap is not None:
        ck = g[f"{tag}_ckpt"]
        assert len(cap) == len(ck), tag
        for j, (a, b) in enumerate(zip(cap, ck)):
            assert rel_err(a, b) <= PARITY_TOL, (tag, j)


def test_c0_rk_ten_seeds(gpu, systems):
    from paper_2401_17474_b200 import DeviceSystem, solve_rk

    g = golden("solves.npz")
    with DeviceSystem(systems["c0"]) as ds:
        for seed in range(10):
            tag = f"c0_rk_s{seed}"
            r = solve_rk(ds, _cfg(variant="rk", base_seed=seed), checkpoint_every=100)
            cap = []
            solve_rk(ds, _cfg(variant="rk", base_seed=seed), capture=cap)
            _check(r, g, tag, cap[99::100])
            assert abs(r.final_error_sq - float(g[f"{tag}_final_error_sq"])) <= 1e-12
            assert abs(r.final_residual - float(g[f"{tag}_final_residual"])) <= 1e-8 * (1 + abs(r.final_residual))


@pytest.mark.parametrize("kernel", ["auto", "chain", "sync_cluster", "sync_grid"])
def test_c1_rka_q64(gpu, c1_system, kernel):
    from paper_2401_17474_b200 import DeviceSystem, solve_rka_seq

    g = golden("solves.npz")
    with DeviceSystem(c1_system) as ds:
        seeds = range(3) if kernel == "auto" else range(1)
        for seed in seeds:
            r = solve_rka_seq(ds, _cfg(variant="rka", q=64, base_seed=seed, kernel=kernel), checkpoint_every=1000)
            tag = f"c1_rka64_s{seed}"
            cap = []
            _check(r, g, tag)
            ck = g[f"{tag}_ckpt"]
            r2 = solve_rka_seq(ds, _cfg(variant="rka", q=64, base_seed=seed, kernel=kernel), capture=cap)
            assert r2.iterations == r.iterations and np.array_equal(r2.x, r.x)  # deterministic
            for j, b in enumerate(ck):
                assert rel_err(cap[1000 * (j + 1) - 1], b) <= PARITY_TOL, (kernel, seed, j)
            # the reference's iterate every 100 iterations (golden/c1_ckpt100.npz)
            g100 = golden("c1_ckpt100.npz")
            assert r.iterations == int(g100[f"s{seed}_iterations"])
            ck100 = g100[f"s{seed}_ckpt"]
            assert len(ck100) == r.iterations // 100
            for j, b in enumerate(ck100):
                assert rel_err(cap[100 * (j + 1) - 1], b) <= PARITY_TOL, (kernel, seed, 100 * (j + 1))


def test_c2_rkab_q64_bs500(gpu, c2_system):
    from paper_2401_17474_b200 import DeviceSystem, solve_rkab_seq

    g = golden("solves.npz")
    tag = "c2_rkab64_bs500_s0"
    with DeviceSystem(c2_system) as ds:
        cap = []
        r = solve_rkab_seq(ds, _cfg(variant="rkab", q=64, block_size=500, base_seed=0), capture=cap)
    _check(r, g, tag, cap)


DESK = [
    ("s500_rk_s5", "s500", dict(variant="rk", base_seed=5), {}),
    ("s500_rka3_s2", "s500", dict(variant="rka", q=3, base_seed=2), {}),
    ("s500_rkab3_bs1_s2", "s500", dict(variant="rkab", q=3, block_size=1, base_seed=2), {}),
    ("s500_rkab4_bs8_s3", "s500", dict(variant="rkab", q=4, block_size=8, base_seed=3), {}),
    ("s2000_rka8_dist_s1", "s2000", dict(variant="rka", q=8, base_seed=1, sampling_scheme="distributed"), {}),
    ("s2000_rkab8_bs50_dist_s4", "s2000", dict(variant="rkab", q=8, block_size=50, base_seed=4,
                                                sampling_scheme="distributed"), {}),
    ("s2000_rka16_fixed_s0", "s2000", dict(variant="rka", q=16, alpha_policy="fixed", alpha=1.7, base_seed=0), {}),
    ("s500_rka4_budget50_s9", "s500", dict(variant="rka", q=4, base_seed=9), dict(budget=50)),
    ("s500_rkab5_bs7_budget20_s6", "s500", dict(variant="rkab", q=5, block_size=7, base_seed=6), dict(budget=20)),
]


@pytest.mark.parametrize("tag,sysname,cfgkw,kw", DESK, ids=[d[0] for d in DESK])
def test_desk_scale_solves(gpu, systems, tag, sysname, cfgkw, kw):
    from paper_2401_17474_b200 import run_solver

    g = golden("solves.npz")
    cap = []
    r = run_solver(systems[sysname], _cfg(**cfgkw), capture=cap, **kw)
    every = int(g[f"{tag}_every"])
    _check(r, g, tag, cap[every - 1::every])
    if "budget" in kw:
        assert r.error_evals == 0 and np.isnan(r.final_error_sq)


def test_reduction_identities_bitwise(gpu, systems):
    """RKA(q=1) == RK, RKAB(bs=1) == RKA, RKAB(q=1,bs=1) == RK (test_acceptance.py:28-55)."""
    from paper_2401_17474_b200 import DeviceSystem, solve_rk, solve_rka_seq, solve_rkab_seq

    with DeviceSystem(systems["s500"]) as ds:
        c1, c2 = [], []
        rk = solve_rk(ds, _cfg(variant="rk", base_seed=3), capture=c1)
        rka1 = solve_rka_seq(ds, _cfg(variant="rka", q=1, base_seed=3), capture=c2)
        assert rk.iterations == rka1.iterations and all(np.array_equal(u, v) for u, v in zip(c1, c2))
        c3, c4 = [], []
        rka3 = solve_rka_seq(ds, _cfg(variant="rka", q=3, base_seed=3), capture=c3)
        rkab3 = solve_rkab_seq(ds, _cfg(variant="rkab", q=3, block_size=1, base_seed=3), capture=c4)
        assert rka3.iterations == rkab3.iterations and all(np.array_equal(u, v) for u, v in zip(c3, c4))
        rkab11 = solve_rkab_seq(ds, _cfg(variant="rkab", q=1, block_size=1, base_seed=3))
        assert rkab11.iterations == rk.iterations and np.array_equal(rkab11.x, rk.x)


def test_projection_kats(gpu):
    """test_solvers_seq.py:14-25, 127-132, 188-201 through the B200 engine."""
    from paper_2401_17474_b200 import LinearSystem, run_solver, solve_rka_seq, solve_rk

    axis = LinearSystem(A=np.array([[1.0, 0.0]]), b=np.array([2.0]), x_star=np.array([2.0, 0.0]))
    r = solve_rk(axis, _cfg(variant="rk"), budget=1)
    assert np.array_equal(r.x, [2.0, 0.0])
    obl = LinearSystem(A=np.array([[3.0, 4.0]]), b=np.array([10.0]), x_star=np.array([1.2, 1.6]))
    r = solve_rk(obl, _cfg(variant="rk"), budget=1)
    assert np.allclose(r.x, [1.2, 1.6], rtol=0, atol=1e-15)
    r = solve_rk(obl, _cfg(variant="rk", alpha_policy="fixed", alpha=0.0), budget=3)
    assert np.array_equal(r.x, [0.0, 0.0])
    one = LinearSystem(A=np.array([[2.0]]), b=np.array([6.0]), x_star=np.array([3.0]))
    r = run_solver(one, _cfg(variant="rk"))
    assert r.converged and r.iterations == 1 and np.array_equal(r.x, [3.0])
    ident = LinearSystem(A=np.eye(3), b=np.array([1.0, 2.0, 3.0]), x_star=np.array([1.0, 2.0, 3.0]))
    r = run_solver(ident, _cfg(variant="rk", base_seed=4))
    assert r.converged and np.allclose(r.x, [1, 2, 3], atol=1e-4)
    # identity averaging (test_solvers_seq.py:165-170): two draws from x = 0 average to
    # (2, 0), (0, 4) or, for distinct rows, (1, 2)
    eye2 = LinearSystem(A=np.eye(2), b=np.array([2.0, 4.0]), x_star=np.array([2.0, 4.0]))
    seen = set()
    for seed in range(50):
        r = solve_rka_seq(eye2, _cfg(variant="rka", q=2, base_seed=seed), budget=1)
        seen.add(tuple(r.x.tolist()))
    assert seen <= {(2.0, 0.0), (0.0, 4.0), (1.0, 2.0)} and (1.0, 2.0) in seen


def test_projection_property_1000_steps(gpu):
    """test_acceptance.py:58-71: after one unit step the sampled equation holds to 1e-10 (1+|b_i|)."""
    from paper_2401_17474_b200 import LinearSystem, Prng, solve_rk

    rng = Prng(2024, 1)
    for _ in range(200):
        n = 2 + int(rng.random() * 10)
        a = rng.standard_normal((1, n)) * (1 + 9 * rng.random())
        b = rng.standard_normal(1) * 10
        r = solve_rk(LinearSystem(A=a, b=b, x_star=np.zeros(n)), _cfg(variant="rk"), budget=1)
        assert abs(float(a[0] @ r.x) - b[0]) <= 1e-10 * (1 + abs(b[0]))


def test_trace_mode_matches_reference(gpu, inc2000):
    from paper_2401_17474_b200 import DeviceSystem, plateau_error, trace_run

    g = golden("traces.npz")
    with DeviceSystem(inc2000) as ds:
        for q in (1, 4, 16):
            recs = trace_run(ds, _cfg(variant="rka", q=q, base_seed=0), 3000, 100, inc2000.x_ls)
            ref = g[f"inc2000_rka{q}"]
            assert len(recs) == len(ref)
            for rec, row in zip(recs, ref):
                assert rec.iteration == int(row[0])
                assert abs(rec.error_norm - row[1]) <= 1e-9 * (1 + row[1])
                assert abs(rec.residual_norm - row[2]) <= 1e-9 * (1 + row[2])
            assert abs(plateau_error(recs) - float(g[f"inc2000_rka{q}_plateau"])) <= 1e-9


def test_max_iterations_exhausted_is_flagged(gpu, systems):
    from paper_2401_17474_b200 import run_solver

    r = run_solver(systems["c0"], _cfg(variant="rk", max_iterations=37))
    assert not r.converged and r.iterations == 37 and r.error_evals == 38
    r = run_solver(systems["c0"], _cfg(variant="rka", q=8, max_iterations=5))
    assert not r.converged and r.iterations == 5 and r.error_evals == 6


def test_oracle_agreement_random_configs(gpu, oracle, systems):
    """Cross-check against the oracle on configurations with no reference fixture."""
    from paper_2401_17474_b200 import DeviceSystem, solve_rka_seq, solve_rkab_seq

    s = systems["s2000"]
    with DeviceSystem(s) as ds:
        for q, scheme in ((2, "full_access"), (5, "distributed"), (33, "full_access"), (128, "distributed")):
            for kernel in ("chain", "sync_cluster", "sync_grid"):
                r = solve_rka_seq(ds, _cfg(variant="rka", q=q, base_seed=q, sampling_scheme=scheme, kernel=kernel),
                                  checkpoint_every=50)
                o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=q, base_seed=q, scheme=scheme, ckpt_every=50)
                assert r.iterations == o["iterations"], (q, kernel)
                assert rel_err(r.x, o["x"]) <= PARITY_TOL
        for q, bs in ((2, 3), (7, 64), (64, 10)):
            r = solve_rkab_seq(ds, _cfg(variant="rkab", q=q, block_size=bs, base_seed=1))
            o = oracle.solve(s.A, s.b, s.x_star, variant="rkab", q=q, block_size=bs, base_seed=1)
            assert r.iterations == o["iterations"], (q, bs)
            assert rel_err(r.x, o["x"]) <= PARITY_TOL


@pytest.mark.parametrize("ctas", [32, 80, 112])
def test_multi_cluster_matches_reference(gpu, c1_system, ctas):
    """Several 16-CTA clusters exchanging cluster totals through tagged words
    (rka_kernel, kz_rka.cu): same iterates and stop decisions as the reference's c1 solve."""
    from paper_2401_17474_b200 import DeviceSystem, solve_rka_seq

    g = golden("solves.npz")
    tag = "c1_rka64_s0"
    with DeviceSystem(c1_system) as ds:
        r = solve_rka_seq(ds, _cfg(variant="rka", q=64, base_seed=0, kernel="sync_cluster", ctas=ctas),
                          checkpoint_every=1000)
        assert r.gpu["kernel"] == "rka" and r.gpu["ctas"] == ctas
        _check(r, g, tag)
        cap = []
        solve_rka_seq(ds, _cfg(variant="rka", q=64, base_seed=0, kernel="sync_cluster", ctas=ctas), capture=cap)
        for j, b in enumerate(g[f"{tag}_ckpt"]):
            assert rel_err(cap[1000 * (j + 1) - 1], b) <= PARITY_TOL, (ctas, j)


@pytest.mark.parametrize("q,ctas", [(64, 112), (300, 96), (512, 0)])
def test_multi_cluster_oracle_c2(gpu, oracle, c2_system, q, ctas):
    """Long rows (80000 x 1000), q up to 512 (two scale blocks per warp), vs the oracle."""
    from paper_2401_17474_b200 import DeviceSystem, solve_rka_seq

    s = c2_system
    o = oracle.solve(s.A, s.b, s.x_star, variant="rka", q=q, base_seed=2, ckpt_every=250,
                     nthreads=oracle.max_threads())
    with DeviceSystem(s) as ds:
        kernel = "sync_cluster" if ctas else "auto"
        r = solve_rka_seq(ds, _cfg(variant="rka", q=q, base_seed=2, kernel=kernel, ctas=ctas))
        assert ctas == 0 or r.gpu["ctas"] == ctas
        assert r.iterations == o["iterations"] and r.error_evals == o["error_evals"]
        assert rel_err(r.x, o["x"]) <= PARITY_TOL
        cap = []
        solve_rka_seq(ds, _cfg(variant="rka", q=q, base_seed=2, kernel=kernel, ctas=ctas), capture=cap)
        for j, ck in enumerate(o["checkpoints"]):
            assert rel_err(cap[250 * (j + 1) - 1], ck) <= PARITY_TOL, (q, j)


CK_CASES = [("c0_ck", "c0", {}, {}), ("s500_ck", "s500", {}, {}),
            ("s2000_ck_fixed", "s2000", dict(alpha_policy="fixed", alpha=1.5), {}),
            ("crop300x40_ck", "crop300x40", {}, {}), ("s500_ck_budget777", "s500", {}, dict(budget=777)),
            ("c0_ck_max300", "c0", dict(max_iterations=300), {})]


@pytest.mark.parametrize("tag,sysname,cfgkw,kw", CK_CASES, ids=[c[0] for c in CK_CASES])
def test_cyclic_kaczmarz_matches_reference(gpu, systems, tag, sysname, cfgkw, kw):
    """solve_ck (solvers.py:271-291) through the B200 engine vs the reference's own run."""
    from paper_2401_17474_b200 import run_solver

    g = golden("ck.npz")
    cap = []
    r = run_solver(systems[sysname], _cfg(variant="ck", **cfgkw), capture=cap, **kw)
    assert r.iterations == int(g[f"{tag}_iterations"])
    assert r.error_evals == int(g[f"{tag}_error_evals"])
    assert r.converged == bool(g[f"{tag}_converged"])
    assert rel_err(r.x, g[f"{tag}_x"]) <= PARITY_TOL
    every = int(g[f"{tag}_every"])
    for j, ck in enumerate(g[f"{tag}_ckpt"]):
        assert rel_err(cap[every * (j + 1) - 1], ck) <= PARITY_TOL, (tag, j)


def test_device_cgls_matches_reference_xls(gpu, inc2000):
    """kz_cgls (cgls.py:42-75 on the device) reproduces the reference's x_LS of the
    inconsistent fixture system to rounding; the budget error mirrors ConvergenceError."""
    from paper_2401_17474_b200 import DeviceSystem, errors, run_solver

    g = golden("systems.npz")
    with DeviceSystem(inc2000) as ds:
        x = ds.cgls(tol=1e-12)
        assert rel_err(x, g["inc2000_xls"]) <= 1e-9
        # the reference's stop rule holds on a fresh residual
        A, b = inc2000.A, inc2000.b
        assert np.linalg.norm(A.T @ (A @ x - b)) <= 1e-12 * np.linalg.norm(A.T @ b) * 10
        with pytest.raises(errors.ConvergenceError) as ei:
            ds.cgls(tol=1e-14, max_it=2)
        assert ei.value.best_x is not None and ei.value.best_x.shape == (A.shape[1],)
    r = run_solver(inc2000, _cfg(variant="cgls"))
    assert rel_err(r.x, g["inc2000_xls"]) <= 1e-7


def test_device_cgls_c4_shape(gpu):
    """c4-like shape (20000 x 800, b_LS = b + xi): device CGLS vs the host checker
    (oracle/cgls_host.py, pinned to the reference's x_LS in test_host.py)."""
    from oracle.cgls_host import cgls

    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, generate_mother
    from paper_2401_17474_b200.sysgen import Prng

    s = generate_mother(GeneratorConfig(m_max=20000, n_max=800, seed=3))
    b_ls = s.b + Prng(5, 3).standard_normal(s.A.shape[0])
    x_host = cgls(s.A, b_ls, tol=1e-12)
    with DeviceSystem(s) as ds:
        x_dev = ds.cgls(b=b_ls, tol=1e-12)
    assert rel_err(x_dev, x_host) <= 1e-9


def test_kzsys_file_straight_to_device(gpu, systems, tmp_path):
    """kz_system_load_file: the reference's own KZSYS file and a row shard of a larger one
    land in HBM equal to the uploaded arrays; solves from them match the golden run."""
    import os

    from paper_2401_17474_b200 import DeviceSystem, run_solver, sysgen as G
    from paper_2401_17474_b200.errors import SystemFormatError

    gdir = os.path.join(os.path.dirname(__file__), "golden")
    with DeviceSystem.from_file(os.path.join(gdir, "kzsys_s500.bin")) as ds:
        assert (ds.m, ds.n) == (500, 20) and ds.file_flags & 2
        A, b, xr = ds.download()
        s = systems["s500"]
        assert np.array_equal(A, s.A) and np.array_equal(b, s.b) and np.array_equal(xr, s.x_star)
        g = golden("solves.npz")
        r = run_solver(ds, _cfg(variant="rk", base_seed=5))
        assert r.iterations == int(g["s500_rk_s5_iterations"])
        assert rel_err(r.x, g["s500_rk_s5_x"]) <= PARITY_TOL
    big = G.generate_mother(G.GeneratorConfig(m_max=5000, n_max=300, seed=2))
    p = tmp_path / "big.kzsys"
    G.save_system(big, p)
    with DeviceSystem.from_file(p, rows=(1200, 3999)) as ds:
        A, b, xr = ds.download()
        assert np.array_equal(A, big.A[1200:4000]) and np.array_equal(b, big.b[1200:4000])
        assert ds.file_m == 5000
    p.write_bytes(open(p, "rb").read()[:-100])
    with pytest.raises(SystemFormatError):
        DeviceSystem.from_file(p)


def test_chain_cta_pairs_match_oracle(gpu, oracle):
    """Rows of n >= 1024 run on CTA pairs (thread-block clusters of 2, DSMEM join per row
    block): RK and RKAB against the oracle, checkpoints every 500 rows / 2 outer iterations."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, generate_mother, solve_rk, solve_rkab_seq

    s = generate_mother(GeneratorConfig(m_max=12000, n_max=1500, seed=6))
    with DeviceSystem(s) as ds:
        cap = []
        r = solve_rk(ds, _cfg(variant="rk", base_seed=2), budget=3000, capture=cap)
        assert r.gpu["ctas"] == 2, r.gpu
        o = oracle.solve(s.A, s.b, s.x_star, variant="rk", base_seed=2, budget=3000, ckpt_every=500)
        for j, ck in enumerate(o["checkpoints"]):
            assert rel_err(cap[500 * (j + 1) - 1], ck) <= PARITY_TOL, ("rk", j)
        cap = []
        r = solve_rkab_seq(ds, _cfg(variant="rkab", q=8, block_size=60, base_seed=4), budget=12, capture=cap)
        assert r.gpu["ctas"] == 16, r.gpu
        o = oracle.solve(s.A, s.b, s.x_star, variant="rkab", q=8, block_size=60, base_seed=4, budget=12,
                         ckpt_every=2)
        for j, ck in enumerate(o["checkpoints"]):
            assert rel_err(cap[2 * (j + 1) - 1], ck) <= PARITY_TOL, ("rkab", j)


def test_c3_crop_rkab_matches_oracle(gpu, oracle):
    """BASELINE config 3's counter-keyed system (entries depend only on (seed, i, j), so a
    16000 x 2000 system is the exact leading crop of the 160000 x 20000 one), RKAB q=64
    bs=1000 with the distributed scheme -- the c3 solve-to-eps configuration -- for 25 outer
    iterations: every iterate within 1e-10 of the oracle's."""
    from paper_2401_17474_b200 import DeviceSystem, solve_rkab_seq

    with DeviceSystem(m=16000, n=2000) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        cfg = _cfg(variant="rkab", q=64, block_size=1000, sampling_scheme="distributed")
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=25, capture=cap)
    o = oracle.solve(A, b, xr, variant="rkab", q=64, block_size=1000, scheme="distributed", budget=25,
                     ckpt_every=5, nthreads=oracle.max_threads())
    assert r.iterations == 25
    assert rel_err(r.x, o["x"]) <= PARITY_TOL
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[5 * (j + 1) - 1], ck) <= PARITY_TOL, j


@pytest.mark.parametrize("tag", ["c0_rka_np4", "c0_rka_np8_s3", "s2000_rkab_np4_bs20", "s2000_rkab_np2_bs7_budget",
                                 "c0_rka_np4_fixed"])
def test_run_distributed_solve_matches_reference(gpu, systems, tag):
    """run_distributed_solve (the reference's simulated-MPI engine, Algorithms 2 and 4) on the
    B200 against the reference's own runs (tests/golden/dist.npz)."""
    from test_oracle_golden import DIST_CASES

    from paper_2401_17474_b200 import run_distributed_solve

    g = golden("dist.npz")
    sysname, variant, bs, seed, alpha, budget = DIST_CASES[tag]
    s = systems[sysname]
    size = int(g[f"{tag}_size"])
    kw = dict(alpha_policy="fixed", alpha=alpha) if alpha is not None else {}
    caps = [[] for _ in range(size)]
    reps = run_distributed_solve(s, _cfg(variant=variant, block_size=bs, base_seed=seed, **kw), size,
                                 budget=budget, captures=caps)
    assert len(reps) == size and all(np.array_equal(r.x, reps[0].x) for r in reps)
    r = reps[0]
    assert r.iterations == int(g[f"{tag}_iterations"]) and r.converged == bool(g[f"{tag}_converged"])
    if budget is None:
        assert r.error_evals == int(g[f"{tag}_error_evals"])
    assert rel_err(r.x, g[f"{tag}_x"]) <= PARITY_TOL
    every = int(g[f"{tag}_every"])
    for j, ck in enumerate(g[f"{tag}_ckpt"]):
        assert rel_err(caps[0][every * (j + 1) - 1], ck) <= PARITY_TOL, j


@pytest.mark.parametrize("variant", ["rk", "ck"])
def test_chain_cluster_of_4_matches_oracle(gpu, oracle, variant):
    """One long chain (RK / CK, n >= 1536) runs on a cluster of 4 CTAs, each a column slice, the
    Gram-block reductions joined all-to-all over DSMEM in CTA order: iterates vs the oracle."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, generate_mother, run_solver

    s = generate_mother(GeneratorConfig(m_max=6000, n_max=2000, seed=9))
    budget = 3000
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, base_seed=4, budget=budget, ckpt_every=500)
    with DeviceSystem(s) as ds:
        cap = []
        r = run_solver(ds, _cfg(variant=variant, base_seed=4), budget=budget, capture=cap)
        assert r.gpu["ctas"] == 4, r.gpu
        r2 = run_solver(ds, _cfg(variant=variant, base_seed=4, max_iterations=200000))
    assert rel_err(r.x, o["x"]) <= PARITY_TOL
    for j, ck in enumerate(o["checkpoints"]):
        assert rel_err(cap[500 * (j + 1) - 1], ck) <= PARITY_TOL, j
    o2 = oracle.solve(s.A, s.b, s.x_star, variant=variant, base_seed=4, max_iterations=200000)
    assert r2.iterations == o2["iterations"] and r2.converged == o2["converged"]
    assert r2.error_evals == o2["error_evals"]
    assert rel_err(r2.x, o2["x"]) <= PARITY_TOL


@pytest.mark.parametrize("n", [50, 120, 250])
def test_warp_kernel_matches_oracle(gpu, oracle, n):
    """The one-warp RK kernel (short rows; register ring, per-row butterflies) vs the oracle:
    stop mode with checkpoints, and budget mode, at each EPL width."""
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, generate_mother, run_solver

    s = generate_mother(GeneratorConfig(m_max=3000, n_max=n, seed=n))
    o = oracle.solve(s.A, s.b, s.x_star, variant="rk", base_seed=5, ckpt_every=50, max_iterations=400000)
    ob = oracle.solve(s.A, s.b, s.x_star, variant="rk", base_seed=6, budget=777)
    with DeviceSystem(s) as ds:
        cap = []
        r = run_solver(ds, _cfg(variant="rk", base_seed=5, kernel="warp", max_iterations=400000), capture=cap)
        rb = run_solver(ds, _cfg(variant="rk", base_seed=6, kernel="warp"), budget=777)
    assert r.gpu["kernel"] == "warp"
    assert r.iterations == o["iterations"] and r.converged == o["converged"] and r.error_evals == o["error_evals"]
    assert rel_err(r.x, o["x"]) <= PARITY_TOL
    for j, ck in enumerate(o["checkpoints"][:200]):
        assert rel_err(cap[50 * (j + 1) - 1], ck) <= PARITY_TOL, j
    assert rb.iterations == 777 and rel_err(rb.x, ob["x"]) <= PARITY_TOL


def test_trace_records_past_one_residual_batch(gpu, inc2000):
    """Trace records are evaluated 32 to a pass over A (kz_api.cu flush_trace); 71 records cross
    two batch boundaries.  Each record must equal ||A x_k - b|| and ||x_k - x_ref|| of the
    iterate checkpointed at the same k (harness.py:188, solvers.py:210-224)."""
    from paper_2401_17474_b200 import DeviceSystem, run_solver

    a, b, xr = inc2000.A, inc2000.b, inc2000.x_ls
    with DeviceSystem(inc2000) as ds:
        cap = []
        r = run_solver(ds, _cfg(variant="rka", q=4, base_seed=1, max_iterations=7000), x_ref=xr, trace_step=100,
                       capture=cap, checkpoint_every=100)
    assert len(r.trace) == 71 and len(cap) == 70
    for j, rec in enumerate(r.trace):
        x = np.zeros(a.shape[1]) if j == 0 else cap[j - 1]
        assert rec.iteration == 100 * j
        res, err = float(np.linalg.norm(a @ x - b)), float(np.linalg.norm(x - xr))
        assert abs(rec.residual_norm - res) <= 1e-9 * (1 + res), j
        assert abs(rec.error_norm - err) <= 1e-9 * (1 + err), j
