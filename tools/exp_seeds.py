"""c0: the 10 seeds one after another vs one kz_solve_seeds batch (device time)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, run_solver, solve_seeds  # noqa

s = generate_mother(GeneratorConfig(m_max=2000, n_max=50, seed=0))
cfg = SolverConfig(variant="rk")
with DeviceSystem(s) as ds:
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rs = [run_solver(ds, cfg.replace(base_seed=k)) for k in range(10)]
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rb = solve_seeds(ds, cfg, list(range(10)))
        torch.cuda.synchronize()
        t2 = time.perf_counter()
        rows = sum(r.iterations for r in rs)
        print(f"sequential {1e3 * (t1 - t0):.2f} ms ({rows / (t1 - t0):.3e} rows/s); batch {1e3 * (t2 - t1):.2f} ms "
              f"({rows / (t2 - t1):.3e} rows/s), device loop {rb[0].gpu['loop_ms']:.2f} ms", flush=True)
