"""Run one workload's solve a few times (for ncu / quick timing on the GPU box).

    python tools/prof_case.py --workload c1 --solves 3 [--kernel auto] [--budget N]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import WORKLOADS, build_system  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c1", choices=sorted(WORKLOADS))
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    args = ap.parse_args()
    from paper_2401_17474_b200 import DeviceSystem, SolverConfig, run_solver

    system, kw = build_system(args.workload)
    cfg = SolverConfig(kernel=args.kernel, threads=args.threads, ctas=args.ctas, **kw)
    with DeviceSystem(system) as ds:
        run_solver(ds, cfg, budget=args.budget)
        for s in range(args.solves):
            t0 = time.perf_counter()
            r = run_solver(ds, cfg.replace(base_seed=s), budget=args.budget)
            dt = time.perf_counter() - t0
            g = r.gpu
            print(f"{args.workload} seed={s} it={r.iterations} conv={r.converged} loop={g['loop_ms']:.3f}ms "
                  f"kernel={g['kernel_ms']:.3f}ms ({g['kernel']} ctas={g['ctas']} thr={g['threads']}) "
                  f"rows/s={g['rows_projected'] / (g['loop_ms'] / 1e3):.3e} us/it={1e3 * g['kernel_ms'] / max(r.iterations, 1):.3f} "
                  f"host={dt * 1e3:.1f}ms", flush=True)


if __name__ == "__main__":
    main()
