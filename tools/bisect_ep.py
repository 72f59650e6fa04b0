"""Chain-kernel instantiations vs the oracle on counter-keyed crops (RKAB, distributed scheme):
prints the plan and the relative error of each outer iteration."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import oracle as O  # noqa: E402
from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq, run_solver  # noqa: E402


def rel(a, b):
    return float(np.max(np.abs(a - b)) / np.max(np.abs(b)))


cases = [(24000, 3008, 8, 50, 0), (24000, 2992, 8, 50, 0), (24000, 3000, 8, 50, 0), (24000, 3000, 8, 50, 192), (24000, 3000, 8, 1, 0), (24000, 3000, 2, 50, 0),
         (24000, 2000, 8, 50, 0), (24000, 8192, 8, 50, 0), (24000, 20000, 8, 50, 0), (24000, 4096, 8, 50, 0)]
for m, n, q, bs, thr in cases:
  try:
    with DeviceSystem(m=m, n=n) as ds:
        ds.generate_counter(0)
        A, b, xr = ds.download()
        cfg = SolverConfig(variant="rkab", q=q, block_size=bs, base_seed=3, sampling_scheme="distributed",
                           threads=thr)
        cap = []
        r = solve_rkab_seq(ds, cfg, budget=3, capture=cap)
    o = O.solve(A, b, xr, variant="rkab", q=q, block_size=bs, scheme="distributed", budget=3, ckpt_every=1, base_seed=3,
                nthreads=O.max_threads())
    errs = [rel(c, k) for c, k in zip(cap, o["checkpoints"])]
    print(f"m={m} n={n} q={q} bs={bs} thr={thr}: plan={r.gpu['plan']} ctas={r.gpu['ctas']} "
          f"threads={r.gpu['threads']} errs={['%.1e' % e for e in errs]}", flush=True)
  except Exception as exc:
    print(f"m={m} n={n} q={q} bs={bs} thr={thr}: {exc!r}", flush=True)
