"""Diagnose a counter-keyed crop solve against the oracle: norms, cdfs, row draws, b, first iterate."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq  # noqa: E402

for (m, n, q, bs, seed) in [(16000, 2000, 64, 1000, 0), (24000, 2000, 8, 50, 3), (16000, 2000, 8, 50, 3),
                            (24000, 2000, 64, 50, 3), (24000, 2000, 8, 50, 0)]:
    with DeviceSystem(m=m, n=n) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        sq_d = ds.row_norms()
        sq_o = O.row_sqnorms(A)
        print("norms equal", np.array_equal(sq_d, sq_o), "b=Ax*", float(np.max(np.abs(A @ xr - b)) / np.max(np.abs(b))))
        cdf_d = ds.cdf("distributed", q)
        lo, hi = 0, m // q - 1
        print("cdf block0 equal", np.array_equal(cdf_d[lo:hi + 1], O.cdf(sq_o, lo, hi)))
        for w in (0, q - 1):
            rd = ds.dump_rows(seed, w, 200, scheme="distributed", q=q)
            ro = O.dump_rows(sq_o, "distributed", q, seed, w, 200)
            print("worker", w, "rows equal", np.array_equal(rd, ro), rd[:5], ro[:5])
        cap = []
        r = solve_rkab_seq(ds, SolverConfig(variant="rkab", q=q, block_size=bs, base_seed=seed,
                                            sampling_scheme="distributed"), budget=2, capture=cap)
    o = O.solve(A, b, xr, variant="rkab", q=q, block_size=bs, scheme="distributed", budget=2, ckpt_every=1,
                base_seed=seed, nthreads=O.max_threads())
    o1 = O.solve(A, b, xr, variant="rkab", q=q, block_size=bs, scheme="distributed", budget=2, ckpt_every=1,
                 base_seed=seed, nthreads=1)
    e = [float(np.max(np.abs(c - k)) / np.max(np.abs(k))) for c, k in zip(cap, o["checkpoints"])]
    print(m, n, q, bs, seed, "gpu vs oracle", e, "oracle mt vs serial", np.array_equal(o["x"], o1["x"]), flush=True)
