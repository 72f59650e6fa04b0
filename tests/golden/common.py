"""Helpers shared by make_golden.py (fixture producer) and the tests (consumers).
Depends on numpy only -- never on the reference."""

import hashlib

import numpy as np

NORM_WIDTHS = [1, 2, 3, 5, 7, 8, 9, 15, 16, 17, 50, 101, 500, 1000, 2000, 8191, 8193, 20000]


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def norm_matrix(n: int) -> np.ndarray:
    """Seeded test matrix for the row-norm fixtures (regenerable from numpy alone)."""
    g = np.random.default_rng(1000 + n)
    rows = 16
    return g.normal(0.0, 1.0, size=(rows, n)) * g.uniform(1, 20, size=(rows, 1)) + g.uniform(-5, 5, size=(rows, 1))
