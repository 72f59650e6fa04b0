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


# threaded-engine fixtures (make_golden.gen_threads): name, (m, n, seed), variant, q, block_size, base_seed
THREAD_CASES = [
    ("s500_rka_q2", (500, 20, 1), "rka", 2, 1, 1),
    ("s500_rka_q4", (500, 20, 1), "rka", 4, 1, 1),
    ("s2000_rka_q8", (2000, 50, 7), "rka", 8, 1, 3),
    ("c0_rka_q16", (2000, 50, 0), "rka", 16, 1, 0),
    ("s500_rkab_q4_bs10", (500, 20, 1), "rkab", 4, 10, 2),
    ("s2000_rkab_q8_bs25", (2000, 50, 7), "rkab", 8, 25, 5),
]
# the reference's own tolerance between its threaded and sequential engines (test_parallel.py:38-44)
THREADS_TOL = 1e-9
