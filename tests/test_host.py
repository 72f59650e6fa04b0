"""Host-side logic on CPU: configuration validation, partitions, report CSV
schema, and the package's restatement of the reference generator (bitwise
against tests/golden/systems.npz)."""

import io
import math

import numpy as np
import pytest

from conftest import golden


def test_solver_config_validation():
    from paper_2401_17474_b200 import SolverConfig

    SolverConfig().validate()
    for bad in (dict(variant="nope"), dict(alpha_policy="x"), dict(sampling_scheme="x"), dict(engine="x"),
                dict(kernel="x"), dict(q=0), dict(block_size=0), dict(epsilon=0.0), dict(max_iterations=0)):
        with pytest.raises(ValueError):
            SolverConfig(**bad).validate()
    c = SolverConfig(variant="rka", q=4)
    assert c.replace(q=8).q == 8 and c.q == 4


def test_partition_bounds():
    from paper_2401_17474_b200 import EmptyRangeError, partition_bounds

    for m, q in ((10, 3), (2000, 64), (7, 7)):
        rows = []
        for t in range(q):
            lo, hi = partition_bounds(m, q, t)
            rows.extend(range(lo, hi + 1))
        assert rows == list(range(m))
    with pytest.raises(EmptyRangeError):
        partition_bounds(3, 4, 0)
    with pytest.raises(EmptyRangeError):
        partition_bounds(10, 2, 2)


def test_report_csv_roundtrip():
    from paper_2401_17474_b200.reports import (REPORT_HEADER, RunReport, TraceRecord, format_report_csv,
                                              read_report_csv, read_trace_csv, trace_row, write_csv)

    r = RunReport("rka", 64, 1, "unit", 1.0, 3, 9431, True, 0.0123456789, 9.87e-9, 1.5e-5)
    text = format_report_csv([("run", r), ("summary", r)])
    assert text.splitlines()[0].split(",") == REPORT_HEADER
    back = read_report_csv(io.StringIO(text))
    assert back[0][0] == "run" and back[0][1].iterations == 9431 and back[0][1].wall_time_s == 0.0123456789
    buf = io.StringIO()
    write_csv(buf, ["iteration", "error_norm", "residual_norm"], [trace_row(TraceRecord(5, 0.5, 1.25))])
    buf.seek(0)
    assert read_trace_csv(buf)[0] == TraceRecord(5, 0.5, 1.25)


def test_generator_restatement_is_bitwise(systems):
    from golden.common import sha

    from oracle.cgls_host import cgls

    from paper_2401_17474_b200 import crop
    from paper_2401_17474_b200.sysgen import inconsistent_rhs

    g = golden("systems.npz")
    for name in ("c0", "s500", "s2000"):
        s = systems[name]
        assert sha(s.A) == str(g[f"{name}_A"]) and sha(s.b) == str(g[f"{name}_b"])
        assert sha(s.x_star) == str(g[f"{name}_xref"])
    c = crop(systems["s2000"], 300, 40)
    assert sha(c.A) == str(g["crop300x40_A"]) and sha(c.b) == str(g["crop300x40_b"])
    assert sha(c.x_star) == str(g["crop300x40_xref"])
    b_ls = inconsistent_rhs(systems["s2000"], noise_seed=11)
    assert sha(b_ls) == str(g["inc2000_b"])
    # the host CGLS checker (oracle/cgls_host.py) against the reference's x_LS
    ref = g["inc2000_xls"]
    x_ls = cgls(systems["s2000"].A, b_ls, tol=1e-10)
    assert np.max(np.abs(x_ls - ref)) <= 1e-8 * np.max(np.abs(ref))


def test_generator_c1_shape_is_bitwise(c1_system):
    from golden.common import sha

    g = golden("systems.npz")
    assert sha(c1_system.A) == str(g["c1_A"]) and sha(c1_system.x_star) == str(g["c1_xref"])


def test_generator_validation():
    from paper_2401_17474_b200 import DimensionMismatchError, GeneratorConfig, generate_mother

    with pytest.raises(DimensionMismatchError):
        generate_mother(GeneratorConfig(m_max=5, n_max=10))
    with pytest.raises(ValueError):
        generate_mother(GeneratorConfig(sigma_range=(0.0, 1.0)))


def test_harness_helpers():
    from paper_2401_17474_b200 import Protocol, TraceRecord, plateau_error

    recs = [TraceRecord(i, float(i), 0.0) for i in range(12)]
    assert plateau_error(recs) == pytest.approx(np.mean(range(2, 12)))
    with pytest.raises(ValueError):
        plateau_error(recs[:5])
    with pytest.raises(ValueError):
        Protocol(n_seeds=0).validate()


def test_spectral_alpha_formula():
    """optimal_alpha (spectral.py:124-134) reproduces the reference's weights from the
    reference's own estimates, bit for bit (golden/spectral.npz), and its edge cases."""
    from paper_2401_17474_b200.spectral import SpectralStats, optimal_alpha

    g = golden("spectral.npz")
    qs = [int(q) for q in g["q_list"]]
    names = [k[:-len("_stats")] for k in g if k.endswith("_stats")]
    assert len(names) >= 4
    for name in names:
        smax, smin, lo, hi = g[f"{name}_stats"]
        st = SpectralStats(sigma_max=smax, sigma_min=smin, s_min=lo, s_max=hi)
        assert [optimal_alpha(st, q) for q in qs] == list(g[f"{name}_alpha"])
    assert optimal_alpha(SpectralStats(1, 1, s_min=0.3, s_max=0.9), 1) == 1.0
    assert abs(optimal_alpha(SpectralStats(1, 1, s_min=0.5, s_max=0.5), 2) - 4 / 3) <= 1e-12
    assert abs(optimal_alpha(SpectralStats(1, 1, s_min=0.1, s_max=0.9), 3) - 2.0) <= 1e-12
    with pytest.raises(ValueError):
        optimal_alpha(SpectralStats(1, 1, s_min=0.1, s_max=0.9), 0)


def test_kzsys_round_trip_and_reference_files(tmp_path):
    """save_system / load_system restate sysgen.py:190-271; files written by the
    reference (golden/kzsys_*.bin) load bit-identically, and damage raises the
    reference's errors with offsets."""
    import os

    from paper_2401_17474_b200 import sysgen as G
    from paper_2401_17474_b200.errors import SystemFormatError, UnsupportedVersionError

    s = G.generate_mother(G.GeneratorConfig(m_max=300, n_max=20, seed=4))
    p = tmp_path / "s.kzsys"
    G.save_system(s, p)
    r = G.load_system(p)
    assert np.array_equal(r.A, s.A) and np.array_equal(r.b, s.b) and np.array_equal(r.x_star, s.x_star)
    assert r.seed == s.seed and r.consistent == s.consistent
    gdir = os.path.join(os.path.dirname(__file__), "golden")
    ref = G.load_system(os.path.join(gdir, "kzsys_s500.bin"))
    mine = G.generate_mother(G.GeneratorConfig(m_max=500, n_max=20, seed=1))
    assert np.array_equal(ref.A, mine.A) and np.array_equal(ref.x_star, mine.x_star)
    assert open(os.path.join(gdir, "kzsys_s500.bin"), "rb").read() == (G.save_system(mine, tmp_path / "m"), open(tmp_path / "m", "rb").read())[1]
    data = bytearray(open(p, "rb").read())
    bad = tmp_path / "bad"
    bad.write_bytes(b"XXSYS" + bytes(data[5:]))
    with pytest.raises(SystemFormatError) as e:
        G.load_system(bad)
    assert e.value.offset == 0
    data[5] = 2
    bad.write_bytes(bytes(data))
    with pytest.raises(UnsupportedVersionError):
        G.load_system(bad)
    bad.write_bytes(open(p, "rb").read()[:-8])
    with pytest.raises(SystemFormatError):
        G.load_system(bad)


def test_einsum_order_restatement_matches_reference_norms():
    """sysgen.einsum_row_norms (the order row_sqnorm_kernel restates) equals the reference's
    row_norm_cache bitwise on the golden matrices, and this numpy's einsum agrees with it."""
    from conftest import golden
    from golden.common import NORM_WIDTHS, norm_matrix

    from paper_2401_17474_b200.sysgen import einsum_order_matches, einsum_row_norms

    g = golden("norms.npz")
    for n in NORM_WIDTHS:
        assert np.array_equal(einsum_row_norms(norm_matrix(n)), g[f"sq_{n}"]), n
    assert einsum_order_matches()
