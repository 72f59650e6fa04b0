"""The row-sharded c3 solve at G GPUs emulated on one GPU: solve_rkab_seq with q = 64 G workers and
the distributed scheme on the whole 160000 x 20000 system is the same arithmetic as G ranks with 64
workers each (the nesting identity), run here in waves of co-resident workers.
Reports the outer iterations to ||x - x*||^2 < 1e-8 per G (what bench.py --gpus G would solve).

    python tools/emulate_scale.py [--gpus 1 2 4 8] [--seeds 1]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--seeds", type=int, default=1)
    ap.add_argument("--max-iterations", type=int, default=20000)
    ap.add_argument("--scheme", default="distributed", choices=["distributed", "shard_full_access"],
                    help="distributed: worker t samples partition_bounds(m, 64 G, t); shard_full_access: every "
                         "worker of GPU g samples the whole shard partition_bounds(m, G, g)")
    args = ap.parse_args()
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, solve_rkab_seq

    out = []
    with DeviceSystem(m=160000, n=20000) as ds:
        ds.generate_counter(0)
        for G in args.gpus:
            for seed in range(args.seeds):
                cfg = SolverConfig(variant="rkab", q=64 * G, block_size=1000, sampling_scheme="distributed",
                                   base_seed=seed, max_iterations=args.max_iterations)
                t0 = time.perf_counter()
                if args.scheme == "shard_full_access":
                    from paper_2401_17474_b200.sysgen import partition_bounds

                    lo, ln = [], []
                    for t in range(64 * G):
                        a, b = partition_bounds(160000, G, t // 64)
                        lo.append(a)
                        ln.append(b - a + 1)
                    ds.set_ranges(lo, ln)
                    d = ds.solve_sharded(cfg, worker_offset=0)
                    rec = {"scheme": args.scheme, "G": G, "q_total": 64 * G, "seed": seed, "iterations": d["iterations"],
                           "converged": d["converged"], "final_error_sq": d["final_error_sq"], "loop_ms": d["loop_ms"],
                           "waves": d["plan"]["waves"], "wall_s": time.perf_counter() - t0,
                           "per_gpu_ms_per_iteration_estimate": d["loop_ms"] / max(d["iterations"], 1) / G}
                    print(json.dumps(rec), flush=True)
                    out.append(rec)
                    continue
                r = solve_rkab_seq(ds, cfg)
                rec = {"scheme": args.scheme, "G": G, "q_total": 64 * G, "seed": seed, "iterations": r.iterations,
                       "converged": r.converged,
                       "final_error_sq": r.final_error_sq, "loop_ms": r.gpu["loop_ms"], "waves": r.gpu["plan"]["waves"],
                       "wall_s": time.perf_counter() - t0,
                       "per_gpu_ms_per_iteration_estimate": r.gpu["loop_ms"] / max(r.iterations, 1) / G}
                print(json.dumps(rec), flush=True)
                out.append(rec)
    return out


if __name__ == "__main__":
    main()
