"""First diverging row of RK on CTA pairs vs the oracle (checkpoint every row)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle as O
from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rk

s = generate_mother(GeneratorConfig(m_max=12000, n_max=1500, seed=6))
B = 1200
o = O.solve(s.A, s.b, s.x_star, variant="rk", base_seed=2, budget=B, ckpt_every=1)
rows = None
for rep in range(3):
    with DeviceSystem(s) as ds:
        cap = []
        r = solve_rk(ds, SolverConfig(variant="rk", base_seed=2), budget=B, capture=cap)
        bad = [k for k in range(B) if np.max(np.abs(cap[k] - o["checkpoints"][k])) > 1e-9 * np.max(np.abs(o["checkpoints"][k]))]
        if bad:
            k = bad[0]
            d = cap[k] - o["checkpoints"][k]
            half = s.A.shape[1] // 2
            print(f"rep {rep}: first bad row {k}; bad columns in lower half {np.sum(np.abs(d[:half]) > 1e-9)} upper half {np.sum(np.abs(d[half:]) > 1e-9)}; nbad {len(bad)}")
        else:
            print(f"rep {rep}: all good")
