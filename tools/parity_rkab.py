"""RKAB parity vs the oracle on a c2-shaped crop for chain-kernel settings (debug aid)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import oracle as O
from conftest import rel_err
from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, solve_rkab_seq
m, n, q, bs, budget = [int(v) for v in sys.argv[1:6]]
s = generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=0))
o = O.solve(s.A, s.b, s.x_star, variant="rkab", q=q, block_size=bs, base_seed=0, budget=budget, ckpt_every=1)
with DeviceSystem(s) as ds:
    cap = []
    r = solve_rkab_seq(ds, SolverConfig(variant="rkab", q=q, block_size=bs, base_seed=0), budget=budget, capture=cap)
errs = [rel_err(a, b) for a, b in zip(cap, o["checkpoints"])]
print(f"m={m} n={n} q={q} bs={bs} R={os.environ.get('KZ_CHAIN_ROWS','auto')} D={os.environ.get('KZ_CHAIN_STAGES','auto')} "
      f"max={max(errs):.1e} :: " + " ".join(f"{e:.0e}" for e in errs[:12]))
