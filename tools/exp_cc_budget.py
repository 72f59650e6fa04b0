"""c1 side by side: stop mode (chunked launches) vs budget mode (one launch per solve) -- host vs device contention."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_17474_b200 import (DeviceSystem, GeneratorConfig, SolverConfig, generate_mother,  # noqa: E402
                                   run_solver, solve_concurrent)

s = generate_mother(GeneratorConfig(m_max=20000, n_max=500, seed=0))
with DeviceSystem(s) as ds:
    for ctas in (16, 8):
        cfgs = [SolverConfig(variant="rka", q=64, ctas=ctas, base_seed=k) for k in range(10)]
        for budget in (None, 9400):
            r = run_solver(ds, cfgs[0], budget=budget)
            alone = r.gpu["loop_ms"]
            for lanes in (2, 5, 10):
                solve_concurrent(ds, cfgs, lanes=lanes, budget=budget)
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                rc = solve_concurrent(ds, cfgs, lanes=lanes, budget=budget)
                torch.cuda.synchronize()
                dt = time.perf_counter() - t0
                per = sum(x.gpu["loop_ms"] for x in rc) / len(rc)
                print(f"ctas={ctas} budget={budget} alone={alone:.2f}ms lanes={lanes}: batch {dt * 1e3:.2f} ms, "
                      f"per-solve loop {per:.2f} ms", flush=True)
