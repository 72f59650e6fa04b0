"""c1: cluster size per solve (ctas = 16 / 8 / 4) alone and in a side-by-side batch of 10 seeds."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_17474_b200 import (DeviceSystem, GeneratorConfig, SolverConfig, generate_mother,  # noqa: E402
                                   run_solver, solve_concurrent)

s = generate_mother(GeneratorConfig(m_max=20000, n_max=500, seed=0))
with DeviceSystem(s) as ds:
    for ctas in (16, 8, 4):
        cfgs = [SolverConfig(variant="rka", q=64, ctas=ctas, base_seed=k) for k in range(10)]
        r = run_solver(ds, cfgs[0])
        print(f"ctas={ctas} alone: {r.gpu['loop_ms']:.2f} ms ({r.gpu['ctas']} CTAs)", flush=True)
        for lanes in (7, 10):
            for rep in range(2):
                solve_concurrent(ds, cfgs, lanes=lanes)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rc = solve_concurrent(ds, cfgs, lanes=lanes)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
            rows = sum(x.gpu["rows_projected"] for x in rc)
            print(f"  lanes={lanes}: batch {dt * 1e3:.2f} ms {rows / dt:.3e} rows/s", flush=True)
