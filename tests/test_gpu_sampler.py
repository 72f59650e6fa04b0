"""T1: the B200 sampler subsystem is bit-exact -- row norms (linalg.py:80-88),
CDFs (sampling.py:101-111) and row-index streams (sampling.py:89-94,
solvers.py:162-171) -- against the reference fixtures and the oracle."""

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def test_row_norms_bitwise_all_widths(gpu, oracle):
    from golden.common import NORM_WIDTHS, norm_matrix
    from paper_2401_17474_b200 import DeviceSystem, LinearSystem

    g = golden("norms.npz")
    for n in NORM_WIDTHS:
        a = norm_matrix(n)
        with DeviceSystem(LinearSystem(A=a, b=np.zeros(a.shape[0]))) as ds:
            sq = ds.row_norms()
        assert np.array_equal(sq, g[f"sq_{n}"]), n
        assert np.array_equal(sq, oracle.row_sqnorms(a)), n


def test_row_norms_large_random_widths(gpu, oracle):
    from paper_2401_17474_b200 import DeviceSystem, LinearSystem

    rng = np.random.default_rng(3)
    for n in (4, 6, 10, 13, 31, 33, 63, 65, 127, 999, 4097):
        a = rng.normal(2.0, 7.0, size=(300, n))
        with DeviceSystem(LinearSystem(A=a, b=np.zeros(300))) as ds:
            assert np.array_equal(ds.row_norms(), oracle.row_sqnorms(a)), n


@pytest.mark.parametrize("scheme,q", [("full_access", 1), ("full_access", 64), ("distributed", 8),
                                      ("distributed", 64)])
def test_cdf_bitwise(gpu, oracle, systems, scheme, q):
    from paper_2401_17474_b200 import DeviceSystem, partition_bounds

    s = systems["s2000"]
    sq = oracle.row_sqnorms(s.A)
    with DeviceSystem(s) as ds:
        c = ds.cdf(scheme, q)
    if scheme == "full_access":
        assert np.array_equal(c, oracle.cdf(sq))
    else:
        for t in range(q):
            lo, hi = partition_bounds(s.m, q, t)
            assert np.array_equal(c[lo:hi + 1], oracle.cdf(sq, lo, hi)), t


def test_row_streams_match_reference_fixtures(gpu, systems, c1_system):
    from paper_2401_17474_b200 import DeviceSystem

    g = golden("rows.npz")
    with DeviceSystem(systems["c0"]) as ds:
        for seed in range(10):
            assert np.array_equal(ds.dump_rows(seed, 0, 2000), g[f"c0_rk_s{seed}"][0]), seed
    with DeviceSystem(systems["s2000"]) as ds:
        for scheme in ("full_access", "distributed"):
            ref = g[f"s2000_q8_{scheme}_s5"]
            for t in range(8):
                assert np.array_equal(ds.dump_rows(5, t, 1000, scheme=scheme, q=8), ref[t])
    with DeviceSystem(c1_system) as ds:
        for scheme in ("full_access", "distributed"):
            for seed in (0, 1):
                ref = g[f"c1_q64_{scheme}_s{seed}"]
                for t in range(64):
                    assert np.array_equal(ds.dump_rows(seed, t, 256, scheme=scheme, q=64), ref[t]), (scheme, t)


def test_long_streams_and_offsets_match_oracle(gpu, oracle, c1_system):
    """1e5 draws per worker, and arbitrary start offsets (PCG64 jump-ahead)."""
    from paper_2401_17474_b200 import DeviceSystem

    sq = oracle.row_sqnorms(c1_system.A)
    with DeviceSystem(c1_system) as ds:
        for scheme, q, workers in (("full_access", 64, (0, 17, 63)), ("distributed", 64, (0, 31, 63))):
            for t in workers:
                ref = oracle.dump_rows(sq, scheme, q, 9, t, 100_000)
                got = ds.dump_rows(9, t, 100_000, scheme=scheme, q=q)
                assert np.array_equal(got, ref), (scheme, t)
                for start in (1, 7, 8, 4095, 77_777):
                    part = ds.dump_rows(9, t, 1000, scheme=scheme, q=q, start=start)
                    assert np.array_equal(part, ref[start:start + 1000]), (scheme, t, start)


def test_degenerate_and_empty_ranges(gpu):
    from paper_2401_17474_b200 import DegenerateRowError, DeviceSystem, EmptyRangeError, LinearSystem

    a = np.array([[1.0, 2.0], [0.0, 0.0], [3.0, 1.0], [0.0, 0.0]])
    with DeviceSystem(LinearSystem(A=a, b=np.ones(4), x_star=np.zeros(2))) as ds:
        with pytest.raises(DegenerateRowError) as ei:
            ds.row_norms()
        assert ei.value.row == 1
    a = np.eye(3)
    with DeviceSystem(LinearSystem(A=a, b=np.ones(3), x_star=np.ones(3))) as ds:
        with pytest.raises(EmptyRangeError):
            ds.cdf("distributed", 4)


def test_uploaded_row_norms(gpu, systems):
    """kz_row_norms_upload: host norms (the Appendix-A fallback for another numpy build) drive the
    sampler exactly like the device norms when they agree; a zero norm is DegenerateRowError."""
    import numpy as np

    from paper_2401_17474_b200 import DegenerateRowError, DeviceSystem, SolverConfig, run_solver

    s = systems["c0"]
    cfg = SolverConfig(variant="rka", q=4, base_seed=3)
    with DeviceSystem(s) as ds:
        a = run_solver(ds, cfg)
        ds.set_row_norms(np.einsum("ij,ij->i", s.A, s.A))
        b = run_solver(ds, cfg)
        assert a.iterations == b.iterations and np.array_equal(a.x, b.x)
        sq = np.einsum("ij,ij->i", s.A, s.A)
        sq[17] = 0.0
        ds.set_row_norms(sq)
        with pytest.raises(DegenerateRowError):
            run_solver(ds, cfg)
