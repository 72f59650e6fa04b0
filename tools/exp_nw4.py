"""c1: four-compute-warp rka CTAs (threads=160, two CTAs per SM) alone and in side-by-side batches."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2401_17474_b200 import (DeviceSystem, GeneratorConfig, SolverConfig, generate_mother,  # noqa: E402
                                   run_solver, solve_concurrent)

s = generate_mother(GeneratorConfig(m_max=20000, n_max=500, seed=0))
with DeviceSystem(s) as ds:
    ref = run_solver(ds, SolverConfig(variant="rka", q=64, base_seed=1))
    for thr in (0, 160):
        r = run_solver(ds, SolverConfig(variant="rka", q=64, threads=thr, base_seed=1))
        print(f"threads={thr}: alone {r.gpu['loop_ms']:.2f} ms it={r.iterations} (ref {ref.iterations}) "
              f"maxdiff={np.max(np.abs(r.x - ref.x)):.2e} {r.gpu['threads']} thr", flush=True)
        cfgs = [SolverConfig(variant="rka", q=64, threads=thr, base_seed=k) for k in range(10)]
        for lanes in (10,):
            best = 1e9
            for rep in range(3):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rc = solve_concurrent(ds, cfgs, lanes=lanes)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            rows = sum(x.gpu["rows_projected"] for x in rc)
            print(f"  lanes={lanes}: batch {best * 1e3:.2f} ms {rows / best:.3e} rows/s; per-solve "
                  f"{np.mean([x.gpu['loop_ms'] for x in rc]):.2f} ms", flush=True)
