"""Shared fixtures.  GPU tests are marked ``gpu`` and run on the B200 box;
everything else runs on CPU.  Nothing here reads /root/reference: the
reference's outputs are committed under tests/golden/ (make_golden.py)."""

from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


def golden(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name), allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def rel_err(a, b) -> float:
    """max-norm error of a against b, relative to max|b| (checkpoint parity metric)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


PARITY_TOL = 1e-10  # north_star: iterates within 1e-10 relative per checkpoint


@pytest.fixture(scope="session")
def systems():
    """The golden systems regenerated with the package's numpy generator."""
    from paper_2401_17474_b200 import sysgen as G

    out = {}
    out["c0"] = G.generate_mother(G.GeneratorConfig(m_max=2000, n_max=50, seed=0))
    out["s500"] = G.generate_mother(G.GeneratorConfig(m_max=500, n_max=20, seed=1))
    out["s2000"] = G.generate_mother(G.GeneratorConfig(m_max=2000, n_max=50, seed=7))
    out["crop300x40"] = G.crop(out["s2000"], 300, 40)
    return out


@pytest.fixture(scope="session")
def c1_system():
    from paper_2401_17474_b200 import sysgen as G

    return G.generate_mother(G.GeneratorConfig(m_max=20000, n_max=500, seed=0))


@pytest.fixture(scope="session")
def c2_system():
    from paper_2401_17474_b200 import sysgen as G

    return G.generate_mother(G.GeneratorConfig(m_max=80000, n_max=1000, seed=0))


@pytest.fixture(scope="session")
def inc2000(systems):
    from paper_2401_17474_b200 import sysgen as G

    return G.make_inconsistent(systems["s2000"], noise_seed=11)


@pytest.fixture(scope="session")
def oracle():
    import oracle as O

    O.lib()
    return O


@pytest.fixture(scope="session")
def gpu():
    from paper_2401_17474_b200 import _native as N

    if N.device_count() < 1:
        pytest.fail("gpu test selected but no CUDA device is visible")
    return N
