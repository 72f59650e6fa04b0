"""Time the reference's own seq engine (kaczbench.solve_rkab_seq, pure Python + numpy) against the
oracle port on the same c3-width workload, in THIS container (the reference is not on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tools/time_reference_python.py

A 24000 x 20000 matrix with c3's row distribution (generate_mother: per-row N(mu_i, sigma_i)),
RKAB q = 64, block size 1000, distributed scheme, a budget of 1 outer iteration (64000 row
projections at n = 20000): rows/s of the reference and of oracle/kz_oracle.c (1 thread and all
threads).  Output: one JSON line.
"""
import json
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import kaczbench as kb

    import oracle as O

    s = kb.generate_mother(kb.GeneratorConfig(m_max=24000, n_max=20000, seed=0))
    cfg = kb.SolverConfig(variant="rkab", q=64, block_size=1000, sampling_scheme="distributed", base_seed=0)
    t0 = time.perf_counter()
    r = kb.solve_rkab_seq(s, cfg, budget=1)
    ref_wall = time.perf_counter() - t0
    rows = 64 * 1000
    out = {"workload": "24000x20000 generate_mother(seed 0), RKAB q=64 bs=1000 distributed, budget 1 outer iteration",
           "rows": rows, "reference_loop_s": r.wall_time_s, "reference_wall_s": ref_wall,
           "reference_rows_per_s": rows / r.wall_time_s}
    for nt in (1, O.max_threads()):
        o = O.solve(s.A, s.b, s.x_star, variant="rkab", q=64, block_size=1000, scheme="distributed", base_seed=0,
                    budget=1, nthreads=nt)
        out[f"oracle_{nt}thr_rows_per_s"] = rows / o["loop_seconds"]
        out[f"oracle_{nt}thr_vs_reference_x"] = float(np.max(np.abs(o["x"] - r.x)) / np.max(np.abs(r.x)))
    out["host"] = {"cpu": platform.processor() or platform.machine(), "nproc": os.cpu_count(),
                   "numpy": np.__version__}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
