"""Pin the CPU oracle (oracle/) against fixtures produced by executing the
reference (tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from conftest import PARITY_TOL, golden, rel_err


def test_prng_streams_and_seedsequence(oracle):
    g = golden("prng.npz")
    k = 0
    while f"draws_{k}" in g:
        ent = [int(e) for e in g[f"entropy_{k}"]]
        assert np.array_equal(oracle.seedseq_state(ent), g[f"ssw_{k}"])
        if len(ent) == 2:
            assert np.array_equal(oracle.random_doubles(ent[0], ent[1], 1000), g[f"draws_{k}"])
        k += 1
    assert k >= 6


def test_row_norms_einsum_order(oracle):
    from golden.common import NORM_WIDTHS, norm_matrix, sha

    g = golden("norms.npz")
    for n in NORM_WIDTHS:
        a = norm_matrix(n)
        assert sha(a) == str(g[f"sha_{n}"])
        assert np.array_equal(oracle.row_sqnorms(a), g[f"sq_{n}"]), n


def test_cdf_terminates_at_one_and_is_monotone(oracle):
    sq = np.array([3.0, 2.0, 7.0])
    c = oracle.cdf(sq)
    assert c[-1] == 1.0 and np.all(np.diff(c) >= 0)
    assert oracle.cdf(np.array([1.0, 4.0]), 1, 1).tolist() == [1.0]
    with pytest.raises(ValueError):
        oracle.cdf(np.array([1.0, 1.0]), 1, 0)


def test_sampler_streams(oracle, systems):
    g = golden("rows.npz")
    sq = oracle.row_sqnorms(systems["c0"].A)
    for seed in range(10):
        assert np.array_equal(oracle.dump_rows(sq, "full_access", 1, seed, 0, 2000), g[f"c0_rk_s{seed}"][0])
    sq = oracle.row_sqnorms(systems["s2000"].A)
    for scheme in ("full_access", "distributed"):
        ref = g[f"s2000_q8_{scheme}_s5"]
        for t in range(8):
            assert np.array_equal(oracle.dump_rows(sq, scheme, 8, 5, t, 1000), ref[t]), (scheme, t)


@pytest.mark.parametrize("seed", range(10))
def test_c0_rk_solves(oracle, systems, seed):
    g = golden("solves.npz")
    s = systems["c0"]
    tag = f"c0_rk_s{seed}"
    r = oracle.solve(s.A, s.b, s.x_star, variant="rk", base_seed=seed, ckpt_every=100)
    assert r["iterations"] == int(g[f"{tag}_iterations"])
    assert r["error_evals"] == int(g[f"{tag}_error_evals"])
    assert rel_err(r["x"], g[f"{tag}_x"]) <= PARITY_TOL
    ck = g[f"{tag}_ckpt"]
    assert len(r["checkpoints"]) == len(ck)
    for a, b in zip(r["checkpoints"], ck):
        assert rel_err(a, b) <= PARITY_TOL


DESK = [
    ("s500_rk_s5", "s500", dict(variant="rk", base_seed=5)),
    ("s500_rka3_s2", "s500", dict(variant="rka", q=3, base_seed=2)),
    ("s500_rkab3_bs1_s2", "s500", dict(variant="rkab", q=3, block_size=1, base_seed=2)),
    ("s500_rkab4_bs8_s3", "s500", dict(variant="rkab", q=4, block_size=8, base_seed=3)),
    ("s2000_rka8_dist_s1", "s2000", dict(variant="rka", q=8, base_seed=1, scheme="distributed")),
    ("s2000_rkab8_bs50_dist_s4", "s2000", dict(variant="rkab", q=8, block_size=50, base_seed=4,
                                                scheme="distributed")),
    ("s2000_rka16_fixed_s0", "s2000", dict(variant="rka", q=16, alphas=1.7, base_seed=0)),
    ("s500_rka4_budget50_s9", "s500", dict(variant="rka", q=4, base_seed=9, budget=50)),
    ("s500_rkab5_bs7_budget20_s6", "s500", dict(variant="rkab", q=5, block_size=7, base_seed=6, budget=20)),
]


@pytest.mark.parametrize("tag,sysname,kw", DESK, ids=[d[0] for d in DESK])
@pytest.mark.parametrize("nthreads", [1, 4])
def test_desk_solves(oracle, systems, tag, sysname, kw, nthreads):
    g = golden("solves.npz")
    s = systems[sysname]
    every = int(g[f"{tag}_every"])
    r = oracle.solve(s.A, s.b, s.x_star, ckpt_every=every, nthreads=nthreads, **kw)
    assert r["iterations"] == int(g[f"{tag}_iterations"])
    assert r["error_evals"] == int(g[f"{tag}_error_evals"])
    for a, b in zip(r["checkpoints"], g[f"{tag}_ckpt"]):
        assert rel_err(a, b) <= PARITY_TOL
    assert rel_err(r["x"], g[f"{tag}_x"]) <= PARITY_TOL


def test_multithreaded_oracle_is_bitwise_serial(oracle, systems):
    s = systems["s2000"]
    for kw in (dict(variant="rka", q=16), dict(variant="rkab", q=8, block_size=20)):
        a = oracle.solve(s.A, s.b, s.x_star, nthreads=1, **kw)
        b = oracle.solve(s.A, s.b, s.x_star, nthreads=5, **kw)
        assert a["iterations"] == b["iterations"] and np.array_equal(a["x"], b["x"])


def test_zero_row_is_degenerate(oracle):
    A = np.array([[1.0, 0.0], [0.0, 0.0], [0.0, 1.0]])
    with pytest.raises(ValueError, match="row 1"):
        oracle.solve(A, np.ones(3), np.zeros(2))


def test_oracle_cyclic_kaczmarz_matches_reference(oracle, systems):
    """The oracle's CK restatement against the reference's solve_ck fixtures (golden/ck.npz)."""
    g = golden("ck.npz")
    cases = [("c0_ck", "c0", {}, None), ("s500_ck", "s500", {}, None),
             ("s2000_ck_fixed", "s2000", {"alphas": 1.5}, None), ("crop300x40_ck", "crop300x40", {}, None),
             ("s500_ck_budget777", "s500", {}, 777), ("c0_ck_max300", "c0", {"max_iterations": 300}, None)]
    for tag, name, kw, budget in cases:
        s = systems[name]
        every = int(g[f"{tag}_every"])
        o = oracle.solve(s.A, s.b, s.x_star, variant="ck", budget=budget, ckpt_every=every, **kw)
        assert o["iterations"] == int(g[f"{tag}_iterations"]), tag
        assert o["error_evals"] == int(g[f"{tag}_error_evals"]), tag
        assert o["converged"] == bool(g[f"{tag}_converged"]), tag
        assert rel_err(o["x"], g[f"{tag}_x"]) <= PARITY_TOL, tag
        for j, ck in enumerate(g[f"{tag}_ckpt"]):
            assert rel_err(o["checkpoints"][j], ck) <= PARITY_TOL, (tag, j)


DIST_CASES = {  # tag: (system, variant, block_size, seed, alpha, budget)
    "c0_rka_np4": ("c0", "rka", 1, 0, None, None),
    "c0_rka_np8_s3": ("c0", "rka", 1, 3, None, None),
    "s2000_rkab_np4_bs20": ("s2000", "rkab", 20, 1, None, None),
    "s2000_rkab_np2_bs7_budget": ("s2000", "rkab", 7, 2, None, 60),
    "c0_rka_np4_fixed": ("c0", "rka", 1, 0, 1.3, None),
}


@pytest.mark.parametrize("tag", sorted(DIST_CASES))
def test_distributed_engine_is_distributed_scheme(oracle, systems, tag):
    """The reference's simulated-MPI engine (run_distributed_solve, distributed.py:339-363) equals
    the sequential solve with q = ranks, the distributed scheme and block_size + 1 rows for RKAB
    (Algorithm 4) -- the mapping paper_2401_17474_b200.run_distributed_solve uses."""
    g = golden("dist.npz")
    sysname, variant, bs, seed, alpha, budget = DIST_CASES[tag]
    s = systems[sysname]
    size = int(g[f"{tag}_size"])
    o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=size, block_size=bs + (1 if variant == "rkab" else 0),
                     base_seed=seed, scheme="distributed", budget=budget,
                     alphas=None if alpha is None else [alpha] * size, ckpt_every=int(g[f"{tag}_every"]))
    assert o["iterations"] == int(g[f"{tag}_iterations"]) and o["converged"] == bool(g[f"{tag}_converged"])
    if budget is None:
        assert o["error_evals"] == int(g[f"{tag}_error_evals"])
    assert rel_err(o["x"], g[f"{tag}_x"]) <= PARITY_TOL
    for j, ck in enumerate(g[f"{tag}_ckpt"]):
        assert rel_err(o["checkpoints"][j], ck) <= PARITY_TOL, j


def test_oracle_threaded_engine_matches_reference(oracle):
    """The oracle's threaded-engine combine (parallel.py:214-226, 286-298 in worker order)
    against the reference's threaded runs: iterations equal, x and every 10th iterate within
    the reference's own threads-vs-seq tolerance; serial and pthreads oracles bitwise equal."""
    from golden.common import THREAD_CASES, THREADS_TOL

    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    g = golden("threads.npz")
    for name, (m, n, seed), variant, q, bs, base in THREAD_CASES:
        s = generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=seed))
        o = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=base, engine="threads",
                         ckpt_every=10)
        assert o["iterations"] == int(g[f"{name}_it"]) and o["converged"]
        assert rel_err(o["x"], g[f"{name}_x"]) <= THREADS_TOL, name
        assert len(o["checkpoints"]) == len(g[f"{name}_ckpt"])
        for a, b in zip(o["checkpoints"], g[f"{name}_ckpt"]):
            assert rel_err(a, b) <= THREADS_TOL, name
        o4 = oracle.solve(s.A, s.b, s.x_star, variant=variant, q=q, block_size=bs, base_seed=base, engine="threads",
                          nthreads=4)
        assert np.array_equal(o4["x"], o["x"])
