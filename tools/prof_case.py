"""Run one solve configuration a few times (quick timing / ncu target on the GPU box).

    python tools/prof_case.py --workload c1 --solves 3 [--kernel auto] [--budget N]
    python tools/prof_case.py --m 160000 --n 20000 --gen counter --variant rkab --q 64 --bs 1000 \
        --scheme distributed --budget 1
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = {  # BASELINE.json configs[0..2]: (m, n, solver kwargs, description)
    "c0": (2000, 50, dict(variant="rk", q=1), "c0: RK 2000x50"),
    "c1": (20000, 500, dict(variant="rka", q=64), "c1: RKA q=64 20000x500"),
    "c2": (80000, 1000, dict(variant="rkab", q=64, block_size=500), "c2: RKAB q=64 bs=500 80000x1000"),
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--n", type=int, default=0)
    ap.add_argument("--gen", default="mother", choices=["mother", "counter"])
    ap.add_argument("--variant", default="rka")
    ap.add_argument("--q", type=int, default=64)
    ap.add_argument("--bs", type=int, default=1)
    ap.add_argument("--scheme", default="full_access")
    ap.add_argument("--solves", type=int, default=3)
    ap.add_argument("--kernel", default="auto")
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--threads", type=int, default=0)
    ap.add_argument("--ctas", type=int, default=0)
    ap.add_argument("--profile-range", action="store_true",
                    help="bracket the timed solves with cudaProfilerStart/Stop (ncu --replay-mode app-range)")
    args = ap.parse_args()
    from paper_2401_17474_b200 import DeviceSystem, GeneratorConfig, SolverConfig, generate_mother, run_solver

    if args.workload:
        m, n, kw, _ = WORKLOADS[args.workload]
    else:
        m, n = args.m, args.n
        kw = dict(variant=args.variant, q=args.q, block_size=args.bs)
    kw = dict(kw)
    kw.setdefault("sampling_scheme", args.scheme)
    cfg = SolverConfig(kernel=args.kernel, threads=args.threads, ctas=args.ctas, **kw)
    t0 = time.perf_counter()
    if args.gen == "counter":
        ds = DeviceSystem(m=m, n=n)
        ds.generate_counter(0)
    else:
        ds = DeviceSystem(generate_mother(GeneratorConfig(m_max=m, n_max=n, seed=0)))
    print(f"system {m}x{n} ({args.gen}) ready in {time.perf_counter() - t0:.1f}s", flush=True)
    with ds:
        run_solver(ds, cfg, budget=args.budget)
        if args.profile_range:
            import torch

            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        for s in range(args.solves):
            t0 = time.perf_counter()
            r = run_solver(ds, cfg.replace(base_seed=s), budget=args.budget)
            dt = time.perf_counter() - t0
            g = r.gpu
            gbs = g["rows_projected"] * 8 * n / (g["kernel_ms"] / 1e3) / 1e9
            print(f"{cfg.variant} q={cfg.q} bs={cfg.block_size} seed={s} it={r.iterations} conv={r.converged} "
                  f"loop={g['loop_ms']:.3f}ms kernel={g['kernel_ms']:.3f}ms ({g['kernel']} ctas={g['ctas']} "
                  f"thr={g['threads']}) rows/s={g['rows_projected'] / (g['loop_ms'] / 1e3):.3e} "
                  f"kernelGB/s={gbs:.0f} us/it={1e3 * g['kernel_ms'] / max(r.iterations, 1):.3f} host={dt * 1e3:.1f}ms",
                  flush=True)
        if args.profile_range:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()


if __name__ == "__main__":
    main()
