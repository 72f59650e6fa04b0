"""One native row-sharded c3 solve at N = 1 (ncu target): RKA q=64, `--budget` outer iterations."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

ap = argparse.ArgumentParser()
ap.add_argument("--budget", type=int, default=20)
ap.add_argument("--variant", default="rka")
ap.add_argument("--bs", type=int, default=1)
args = ap.parse_args()
from paper_2401_17474_b200 import SolverConfig  # noqa: E402
from paper_2401_17474_b200.multigpu import CudaShard, plan_shards, solve_sharded_native  # noqa: E402

plan = plan_shards(160000, 1, 0, 64)
shard = CudaShard.counter(160000, 20000, plan, 0, 0)
cfg = SolverConfig(variant=args.variant, q=64, block_size=args.bs, sampling_scheme="distributed")
for s in range(3):
    r = solve_sharded_native(shard, cfg.replace(base_seed=s), budget=args.budget)
    print(r.iterations, r.gpu["loop_ms"], r.gpu["launches"], flush=True)
