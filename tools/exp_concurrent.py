"""c1: 10 seed-solves one after another vs side by side (solve_concurrent lanes), device-timed."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_17474_b200 import (DeviceSystem, GeneratorConfig, SolverConfig, generate_mother,  # noqa: E402
                                   run_solver, solve_concurrent)

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
m, n, kw = {"c1": (20000, 500, dict(variant="rka", q=64)), "c0": (2000, 50, dict(variant="rk", q=1)),
            "c2": (80000, 1000, dict(variant="rkab", q=64, block_size=500))}[name]
s = generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=0))
cfgs = [SolverConfig(base_seed=k, **kw) for k in range(10)]
with DeviceSystem(s) as ds:
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = [run_solver(ds, c) for c in cfgs]
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        rows = sum(r.gpu["rows_projected"] for r in rs)
        print(f"{name} sequential: {dt * 1e3:.2f} ms  {rows / dt:.3e} rows/s", flush=True)
        for lanes in (4, 7, 10):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = solve_concurrent(ds, cfgs, lanes=lanes)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            assert [r.iterations for r in rc] == [r.iterations for r in rs]
            print(f"{name} lanes={lanes}: {dt * 1e3:.2f} ms  {rows / dt:.3e} rows/s  "
                  f"per-solve loop ms {min(r.gpu['loop_ms'] for r in rc):.2f}..{max(r.gpu['loop_ms'] for r in rc):.2f}",
                  flush=True)
