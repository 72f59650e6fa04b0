"""Row-sharded c3 RKA at one rank: fused cross-rank kernel vs the per-iteration loop (us / outer iteration)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2401_17474_b200 import SolverConfig  # noqa: E402
from paper_2401_17474_b200.multigpu import CudaShard, ShardComm, plan_shards, solve_sharded_native  # noqa: E402

m, n = (160000, 20000) if len(sys.argv) < 3 else (int(sys.argv[1]), int(sys.argv[2]))
plan = plan_shards(m, 1, 0, 64)
shard = CudaShard.counter(m, n, plan, 0, 0)
comm = ShardComm(0, 1, 0)
cfg = SolverConfig(variant="rka", q=64, sampling_scheme="distributed")
for fused in (True, False, True):
    solve_sharded_native(shard, cfg, budget=200, comm=comm, fused=fused)
    r = solve_sharded_native(shard, cfg.replace(base_seed=1), budget=200, comm=comm, fused=fused)
    print(f"{m}x{n} fused={fused}: {1e3 * r.gpu['loop_ms'] / 200:.2f} us/iteration, launches {r.gpu['launches']}",
          flush=True)
shard.close()
comm.close()
