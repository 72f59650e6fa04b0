"""c1 batch of 10 seeds side by side with a mix of cluster sizes per lane (16-CTA and 8-CTA solves)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_concurrent  # noqa

s = generate_mother(GeneratorConfig(m_max=20000, n_max=500, seed=0))
with DeviceSystem(s) as ds:
    for n16 in (10, 8, 7, 6, 5, 0):
        cfgs = [SolverConfig(variant="rka", q=64, ctas=16 if k < n16 else 8, base_seed=k) for k in range(10)]
        best = 1e9
        for rep in range(3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rc = solve_concurrent(ds, cfgs, lanes=10)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        rows = sum(x.gpu["rows_projected"] for x in rc)
        print(f"16-CTA lanes={n16} 8-CTA lanes={10 - n16}: batch {best * 1e3:.2f} ms {rows / best:.3e} rows/s",
              flush=True)
