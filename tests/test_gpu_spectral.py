"""kz_spectral (spectral.py:66-121 on the device) and the optimal weights built on it
(spectral.py:124-156, solvers.py:148-159) against the reference's own outputs
(tests/golden/spectral.npz, produced by make_golden.py executing kaczbench).

The estimators stop at a relative change <= tol = 1e-6 in the Rayleigh quotient; the
device's GEMVs round differently from OpenBLAS, so the iterate at which each loop stops
can differ by one and the estimates agree to the estimator's own tolerance, not bitwise.
"""

import numpy as np
import pytest

from conftest import PARITY_TOL, golden, rel_err

pytestmark = pytest.mark.gpu

SPECTRAL_TOL = 1e-5  # 10x the estimators' stopping tolerance (spectral.py:66, tol=1e-6)

SYSTEMS = {"s500": (500, 20, 1), "s2000": (2000, 50, 7), "c0": (2000, 50, 0), "s3000x120": (3000, 120, 4)}


def _system(name):
    from paper_2401_17474_b200 import GeneratorConfig, generate_mother

    m, n, seed = SYSTEMS[name]
    return generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=seed))


@pytest.mark.parametrize("name", sorted(SYSTEMS))
def test_spectral_stats_match_reference(gpu, name):
    from paper_2401_17474_b200 import DeviceSystem
    from paper_2401_17474_b200.spectral import optimal_alpha, partial_alphas, spectral_stats

    g = golden("spectral.npz")
    s = _system(name)
    smax, smin, lo, hi = g[f"{name}_stats"]
    with DeviceSystem(s) as ds:
        st = spectral_stats(ds)
        assert abs(st.sigma_max - smax) <= SPECTRAL_TOL * smax
        assert abs(st.sigma_min - smin) <= SPECTRAL_TOL * smin
        assert abs(st.s_max - hi) <= SPECTRAL_TOL * hi
        assert abs(st.s_min - lo) <= SPECTRAL_TOL * lo
        for q, ref in zip(g["q_list"], g[f"{name}_alpha"]):
            assert abs(optimal_alpha(st, int(q)) - ref) <= SPECTRAL_TOL * ref
        for q in (4, 8):
            key = f"{name}_partial_q{q}"
            if key in g:
                pa = partial_alphas(ds, q)
                assert np.max(np.abs(pa - g[key]) / g[key]) <= SPECTRAL_TOL
    # a host matrix goes through a temporary upload: same estimates
    st_h = spectral_stats(s.A)
    assert abs(st_h.sigma_min - st.sigma_min) <= 1e-12 * st.sigma_min


def test_partial_alphas_short_block_error(gpu):
    from paper_2401_17474_b200 import DimensionMismatchError
    from paper_2401_17474_b200.spectral import partial_alphas

    g = golden("spectral.npz")
    with pytest.raises(DimensionMismatchError) as exc:
        partial_alphas(_system("s500").A, 32)
    assert str(exc.value) == str(g["short_block_error"])


def test_optimal_weight_solve_matches_oracle(gpu):
    """A solve with the device-estimated weights (alpha_policy optimal_full / optimal_partial)
    agrees with the oracle run on the same weights, and the weights with the reference's."""
    import oracle as O

    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rka_seq
    from paper_2401_17474_b200.solvers import resolve_alphas

    g = golden("spectral.npz")
    s = _system("s2000")
    with DeviceSystem(s) as ds:
        for policy in ("optimal_full", "optimal_partial"):
            cfg = SolverConfig(variant="rka", q=8, alpha_policy=policy, base_seed=3, max_iterations=20000)
            alphas = resolve_alphas(ds, cfg, 8)
            ref = np.full(8, g["s2000_alpha"][list(g["q_list"]).index(8)]) if policy == "optimal_full" \
                else g["s2000_partial_q8"]
            assert np.max(np.abs(alphas - ref) / ref) <= SPECTRAL_TOL
            r = solve_rka_seq(ds, cfg)
            o = O.solve(s.A, s.b, s.x_star, variant="rka", q=8, base_seed=3, alphas=alphas, max_iterations=20000)
            assert r.iterations == o["iterations"]
            assert rel_err(r.x, o["x"]) <= PARITY_TOL
