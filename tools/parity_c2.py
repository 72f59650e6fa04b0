"""c2 parity vs the committed reference fixture for different chain settings."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
from conftest import golden, rel_err
from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rkab_seq
g = golden("solves.npz")
tag = "c2_rkab64_bs500_s0"
s = generate_mother(GeneratorConfig(m_max=80000, n_max=1000, seed=0))
with DeviceSystem(s) as ds:
    cap = []
    r = solve_rkab_seq(ds, SolverConfig(variant="rkab", q=64, block_size=500, base_seed=0), capture=cap)
    errs = [rel_err(a, b) for a, b in zip(cap, g[f"{tag}_ckpt"])]
    print(f"R={os.environ.get('KZ_CHAIN_ROWS','auto')} it={r.iterations} final rel={rel_err(r.x, g[tag + '_x']):.2e} "
          f"ckpt max rel={max(errs):.2e} first={errs[0]:.2e}")
print(" ".join(f"{e:.0e}" for e in errs))
