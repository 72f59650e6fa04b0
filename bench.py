"""Benchmark: row projections/s and time-to-||x - x*||^2 < 1e-8 (fp64) of the
B200 RK / RKA / RKAB engine on BASELINE.json config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--dry-run]

Workload (BASELINE.json configs[3], the largest single-GPU configuration):
the 160000 x 20000 (25.6 GB) counter-keyed system, rows sharded over the N
GPUs (partition_bounds(m, N, g), sampling.py:119-131), 64 RKAB workers per
GPU (Q = 64 N), block size 1000, the reference's `distributed` sampling
scheme (worker t samples partition_bounds(m, Q, t) with stream Prng(seed, t);
its oracle is solve_rkab_seq(q=Q, sampling_scheme="distributed"),
solvers.py:337-371), alpha = 1, x0 = 0.

The timing protocol is the reference's (harness.bench, harness.py:127-175):
the solves to ||x - x*||^2 < 1e-8 give the iteration count, and the timed
steps are fixed-budget replays of that many outer iterations (stop rule off).
A *step* is one replay of C3_BUDGET = 1094 outer iterations (ceil of the mean
iterations-to-eps of solver seeds 0-4 at N = 1; the warm-up solves measure it
again at N <= 2) for one solver seed (seeds cycle 0..9), the shard resident in
HBM before timing starts; per-GPU work is the same at every N (weak scaling).
At N = 1 a step is one kz_solve; at N > 1 every rank runs kz_solve_sharded
(per outer iteration the local step, an in-place NCCL all-reduce of the worker
sum over NVLink, x = S / Q) and the ranks' final x must agree bitwise.
`time_to_eps_ms` reports the warm-up solves to eps.  The distributed scheme's
per-worker blocks shrink to m / 64 N rows (under n = 20000 columns), so the
solve needs more outer iterations as N grows -- 1094 / 1344 / 1870 / 2952 at
N = 1 / 2 / 4 / 8 (seed 0, tools/emulate_scale.py on one GPU, the same
arithmetic as N ranks) -- which is why the timed steps replay a fixed budget.
`value` = rows projected by all ranks / max-over-ranks device time of the K
steps.  The inputs (25.6 GB / N per GPU) are larger than L2, so no flush.
`e2e` runs the same replays through the public API from pinned host arrays
(the H2D of the shard and the D2H of x inside the timed region).

`--impl reference` times the reference algorithm's CPU implementation -- the
oracle port in oracle/ (the reference itself is pure Python + numpy; it
cannot be compiled into oracle/_ref and does not travel to the GPU box) --
on the box's host cores: same matrix (generated on the GPU, copied back),
same configuration, fixed budgets of outer iterations per step, rows/s over
the iteration loop's wall time (the reference times the loop only,
solvers.py:203-208).
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import socket
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "row projections/s (fp64, solve to ||x-x*||^2<1e-8)"
UNIT = "rows/s"

# BASELINE.json configs[3]
C3_M, C3_N, C3_Q, C3_BS, C3_SEED = 160000, 20000, 64, 1000, 0
C3_BUDGET = 1094  # outer iterations per timed step: ceil(mean iterations to eps), seeds 0-4 at N = 1
EPS_MAX_GPUS = 8  # time-to-eps warm-up solves up to here (N = 8: 2952 outer iterations, tools/emulate_scale.py)
SEEDS = 10  # solver seeds of every BASELINE configuration
REF_BUDGET = 4  # outer iterations per reference-arm step (256000 projections at N = 1, ~0.5 s on 16 cores)
CPU_BASELINE_BUDGET = 24  # outer iterations of the cpu_baseline sample at N = 1 (~3-5 s of loop)


def read_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def c3_config(world: int) -> dict:
    """The workload description shared by both arms (identical dicts at the same N)."""
    return {"workload": "BASELINE c3: 160000x20000 counter-keyed (seed 0) fp64 system, RKAB 64 workers per GPU, "
                        "block size 1000, distributed sampling scheme; time-to-eps ||x-x*||^2<1e-8 and fixed-budget "
                        "replays",
            "m": C3_M, "n": C3_N, "variant": "rkab", "q_per_gpu": C3_Q, "q_total": C3_Q * world,
            "block_size": C3_BS, "sampling_scheme": "distributed", "alpha": 1.0, "epsilon": 1e-8,
            "step": f"fixed-budget replay of {C3_BUDGET} outer iterations (harness.bench protocol: budget = "
                    f"ceil(mean iterations to eps) at N = 1)",
            "solver_seeds": f"0..{SEEDS - 1} cycling, one replay per step",
            "parallelism": f"rows sharded over {world} GPU(s) (partition_bounds), x averaged across GPUs "
                           f"every outer iteration" if world > 1 else "1 GPU, whole system resident",
            "l2": "inputs larger than L2 (25.6 GB / N per GPU vs 126 MB), no flush"}


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def host_info() -> dict:
    """The CPU side of the comparison: model, cores, the oracle's toolchain and numpy's BLAS."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name')} {b.get('version')}"
    except Exception:
        pass
    cc = None
    try:
        cc = subprocess.run(["gcc", "--version"], capture_output=True, text=True).stdout.splitlines()[0]
    except (OSError, IndexError):
        pass
    return {"cpu_model": model, "nproc": os.cpu_count(), "numpy": np.__version__, "blas": blas,
            "oracle_cc": cc, "oracle_flags": "-O2 -ffp-contract=off (oracle/Makefile)"}


def c3_host_system(device: int):
    """The full c3 matrix on the host: generated on the GPU (the counter-keyed generator is
    defined by its device code, kz_gen.cu), copied back once, outside any timing."""
    from paper_2401_17474_b200 import DeviceSystem

    with DeviceSystem(m=C3_M, n=C3_N, device=device) as ds:
        ds.generate_counter(C3_SEED)
        return ds.download()


def oracle_sample(A, b, xr, q_total: int, budget: int, seed: int, cores: int) -> dict:
    import oracle as O

    r = O.solve(A, b, xr, variant="rkab", q=q_total, block_size=C3_BS, scheme="distributed", base_seed=seed,
                budget=budget, nthreads=cores)
    return {"rows": budget * q_total * C3_BS, "loop_s": r["loop_seconds"]}


def run_reference(args, rank, world, local_rank):
    """CPU arm: the oracle port of the reference algorithm on all host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle as O

    cores = O.max_threads()
    A, b, xr = c3_host_system(local_rank)
    Q = C3_Q * world
    for w in range(args.warmup):
        oracle_sample(A, b, xr, Q, REF_BUDGET, w % SEEDS, cores)
    rows, loop_s = 0, 0.0
    for k in range(args.steps):
        s = oracle_sample(A, b, xr, Q, REF_BUDGET, k % SEEDS, cores)
        rows += s["rows"]
        loop_s += s["loop_s"]
    value = rows / loop_s
    sample = (f"{args.steps} steps, each {REF_BUDGET} outer iterations ({REF_BUDGET * Q * C3_BS} row projections) "
              f"of the c3 RKAB solve (q={Q}, bs={C3_BS}, distributed scheme) on the same 160000x20000 matrix, "
              f"oracle/kz_oracle.c with {cores} pthreads over the workers; loop wall time only")
    emit({"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
          "warmup": args.warmup, "ms_per_step": 1e3 * loop_s / args.steps, "higher_is_better": True,
          "scaling": "weak", "vs_baseline": None, "dtype": "f64",
          "data": "synthetic (counter-keyed c3 generator, seed 0, generated on the GPU and copied back)",
          "config": c3_config(world),
          "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                           "host": host_info()},
          "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}})


def x_digest(x) -> str:
    return hashlib.sha256(np.ascontiguousarray(x, dtype=np.float64).tobytes()).hexdigest()[:16]


# top-level keys of the b200 arm's line at any N (the dry run emits the same set)
HEADLINE_KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                 "scaling", "vs_baseline", "dtype", "data", "config", "time_to_eps_ms", "iterations", "seeds",
                 "roofline", "clocks", "e2e", "gpu_launches", "setup_s")


def run_dry(args, rank, world):
    """The launcher path without GPU work (--dry-run; CPU, gloo): every rank plans its c3 shard,
    the plans are all-gathered and must tile [0, m) in rank order, rank 0 prints a line with
    the b200 arm's keys (values null)."""
    import torch.distributed as dist

    from paper_2401_17474_b200.multigpu import plan_shards

    plan = plan_shards(C3_M, world, rank, C3_Q)
    mine = (rank, plan.lo, plan.hi, len(plan.worker_lo))
    every = [mine] * world
    if world > 1:
        dist.all_gather_object(every, mine)
    assert [e[0] for e in every] == list(range(world))
    assert every[0][1] == 0 and every[-1][2] == C3_M - 1
    assert all(every[g][2] + 1 == every[g + 1][1] for g in range(world - 1))
    assert all(e[3] == C3_Q for e in every)
    if rank != 0:
        return
    line = {k: None for k in HEADLINE_KEYS}
    line.update(metric=METRIC, unit=UNIT, n_gpus=world, steps=args.steps, warmup=args.warmup,
                higher_is_better=True, scaling="weak", dtype="f64", config=c3_config(world),
                dry_run={"shards": [list(e[1:3]) for e in every], "launcher": "torch.distributed.run"
                         if os.environ.get("TORCHELASTIC_RUN_ID") else "direct"})
    emit(line)


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_2401_17474_b200 import LinearSystem, SolverConfig, solve_rkab_seq
    from paper_2401_17474_b200 import _native as N
    from paper_2401_17474_b200.multigpu import CudaShard, ShardComm, plan_shards, solve_sharded_native

    torch.cuda.set_device(local_rank)
    dev = f"cuda:{local_rank}"
    t_setup = time.perf_counter()
    plan = plan_shards(C3_M, world, rank, C3_Q)
    shard = CudaShard.counter(C3_M, C3_N, plan, C3_SEED, local_rank)
    comm = ShardComm(local_rank, world, rank) if world > 1 else None
    cfg = SolverConfig(variant="rkab", q=C3_Q, block_size=C3_BS, sampling_scheme="distributed", device=local_rank)
    setup_s = time.perf_counter() - t_setup

    def step(k):  # one fixed-budget replay (stop rule off)
        return solve_sharded_native(shard, cfg.replace(base_seed=k % SEEDS), comm=comm, budget=C3_BUDGET)

    # warm-up: the solves to eps (iterations, time-to-eps) where the scheme converges, then replays
    eps_runs = []
    if world <= EPS_MAX_GPUS:
        for w in range(args.warmup):
            r = solve_sharded_native(shard, cfg.replace(base_seed=w % SEEDS), comm=comm)
            assert r.converged, f"warm-up seed {w % SEEDS} did not converge"
            eps_runs.append(r)
    for w in range(args.warmup):
        step(w)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = N.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = []
    with ClockSampler(local_rank) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for k in range(args.steps):
            reps.append(step(k))
        ev1.record()
        torch.cuda.synchronize()
    launches = N.launch_count() - launches0
    t_ms = ev0.elapsed_time(ev1)
    rows = sum(r.iterations * C3_Q * C3_BS for r in reps)
    kernel_ms = sum(r.gpu["kernel_ms"] for r in reps)
    for r in reps:
        assert r.iterations == C3_BUDGET, f"seed {r.seed}: {r.iterations} of {C3_BUDGET} outer iterations"
    digests = [x_digest(r.x) for r in reps]
    agree = None
    tt = torch.tensor([t_ms], device=dev)
    rr = torch.tensor([float(rows)], device=dev)
    if world > 1:
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dist.all_reduce(rr, op=dist.ReduceOp.SUM)
        every = [None] * world
        dist.all_gather_object(every, digests)
        agree = all(d == digests for d in every)
        assert agree, "ranks disagree on x (the all-reduced iterate must be bit-identical on every rank)"
    t_all_ms, rows_all = float(tt.item()), float(rr.item())

    # e2e through the public API from pinned host arrays: per step the H2D of this rank's rows,
    # the solve and the D2H of x (N = 1: the reference entry point solve_rkab_seq on a host
    # LinearSystem; N > 1: a CudaShard uploaded from host rows + the sharded solve)
    pinned = lambda *shape: torch.empty(shape, dtype=torch.float64, pin_memory=True).numpy()  # noqa: E731
    A_h, b_h, xr_h = pinned(plan.m_local, C3_N), pinned(plan.m_local), pinned(C3_N)
    shard.ds.download(out=(A_h, b_h, xr_h))
    e2e_steps = min(args.steps, 3)

    def e2e_step(k):
        c = cfg.replace(base_seed=k % SEEDS)
        if world == 1:
            return solve_rkab_seq(LinearSystem(A=A_h, b=b_h, x_star=xr_h, seed=C3_SEED), c, budget=C3_BUDGET)
        sh = CudaShard(A_h, b_h, xr_h, plan, device=local_rank)
        try:
            return solve_sharded_native(sh, c, comm=comm, budget=C3_BUDGET)
        finally:
            sh.close()

    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_rows = 0
    for k in range(e2e_steps):
        r = e2e_step(k)
        e2e_rows += r.iterations * C3_Q * C3_BS
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    ee = torch.tensor([e2e_s], device=dev)
    er = torch.tensor([float(e2e_rows)], device=dev)
    if world > 1:
        dist.all_reduce(ee, op=dist.ReduceOp.MAX)
        dist.all_reduce(er, op=dist.ReduceOp.SUM)
    e2e_val = float(er.item()) / float(ee.item())
    h2d = A_h.nbytes + b_h.nbytes + xr_h.nbytes
    d2h = C3_N * 8

    extras = []
    if world == 1 and not args.no_extra:
        extras = extra_workloads(local_rank, read_peak()[0])
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:  # cpu_baseline: rank 0 at N = 1 only
        import oracle as O

        cores = O.max_threads()
        s = oracle_sample(A_h, b_h, xr_h, C3_Q, CPU_BASELINE_BUDGET, 0, cores)
        cpu = {"value": s["rows"] / s["loop_s"], "unit": UNIT, "cores": cores, "kind": "port",
               "sample": f"{CPU_BASELINE_BUDGET} outer iterations ({s['rows']} row projections) of the c3 RKAB solve, "
                         f"seed 0, same matrix and configuration, oracle/kz_oracle.c with {cores} pthreads over the "
                         f"workers (the GPU's decomposition: all workers of one solve in parallel); loop wall time",
               "host": host_info()}
    del A_h, b_h, xr_h
    shard.close()
    if comm is not None:
        comm.close()
    if rank != 0:
        return

    peak, peak_src = read_peak()
    bytes_per_row = 8 * C3_N
    achieved = rows * bytes_per_row / (kernel_ms / 1e3) / 1e9
    traffic, traffic_note = None, None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):  # measured once with ncu --set full (never under this timing run)
        tr = json.load(open(tpath)).get("c3")
        if tr:
            traffic = tr["dram_bytes_per_launch"]
            traffic_note = {k: tr[k] for k in ("launch", "algorithmic_bytes_per_launch", "source", "note") if k in tr}
    value = rows_all / (t_all_ms / 1e3)
    if eps_runs:
        eps_ms = [r.gpu["loop_ms"] for r in eps_runs]
        time_to_eps = {"mean": float(np.mean(eps_ms)), "min": float(np.min(eps_ms)), "max": float(np.max(eps_ms)),
                       "iterations": [r.iterations for r in eps_runs], "seeds": [r.seed for r in eps_runs],
                       "rows_per_s": float(np.sum([r.iterations * C3_Q * C3_BS * world for r in eps_runs])
                                           / (np.sum(eps_ms) / 1e3)),
                       "note": "warm-up solves to ||x-x*||^2<1e-8 (stop rule on every outer iteration)"}
    else:
        time_to_eps = {"mean": None, "note": f"not measured above N = {EPS_MAX_GPUS}"}
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t_all_ms / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (counter-keyed generator keyed on (seed, i, j), seed 0, generated in place on each GPU)",
        "config": c3_config(world),
        "time_to_eps_ms": time_to_eps,
        "iterations": [r.iterations for r in reps],
        "seeds": [r.seed for r in reps],
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": traffic, "traffic_detail": traffic_note, "peak_source": peak_src,
                     "kernel": reps[-1].gpu.get("kernel"),
                     "algorithmic_bytes": "8*n = 160000 bytes per row projection; one outer iteration = "
                                          f"{C3_Q} workers x {C3_BS} rows = 10.24 GB per GPU",
                     "note": "achieved = rows x 8n / summed device time of the solve-kernel launches (CUDA events "
                             "on the launching stream, rank 0); the peak is a COPY bandwidth (read + write), the "
                             "kernel a read-only stream (6.98 TB/s of DRAM reads in the ncu capture), so frac can "
                             "pass 1"},
        "clocks": clk.summary(),
        "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "steps": e2e_steps, "api": "solve_rkab_seq(LinearSystem(host arrays), cfg)" if world == 1
                else "CudaShard(host rows) + solve_sharded_native"},
        "gpu_launches": launches,
        "setup_s": setup_s,
    }
    if world > 1:
        line["rank_agreement"] = {"bitwise_x_all_steps": agree, "digests": digests}
    if extras:
        line["extra_workloads"] = extras
    if cpu is not None:
        line["cpu_baseline"] = cpu
    assert set(HEADLINE_KEYS) <= set(line), set(HEADLINE_KEYS) - set(line)
    emit(line)


def extra_workloads(device, peak, steps=3):
    """The other BASELINE configurations on this GPU (same metric; fixed budgets for the RKA
    shapes, time-to-eps where the configuration asks for it).  Kernel-time roofline each."""
    import torch

    from paper_2401_17474_b200 import (DeviceSystem, GeneratorConfig, LinearSystem, SolverConfig, generate_mother,
                                       run_solver, solve_concurrent, solve_seeds)

    out = []

    def measure(tag, ds, n, cfg, budget, desc, n_steps=steps):
        run_solver(ds, cfg, budget=budget)  # warm-up
        torch.cuda.synchronize()
        rows, kms, lms, its, conv = 0, 0.0, 0.0, [], []
        for k in range(n_steps):
            r = run_solver(ds, cfg.replace(base_seed=k), budget=budget)
            rows += r.gpu["rows_projected"]
            kms += r.gpu["kernel_ms"]
            lms += r.gpu["loop_ms"]
            its.append(r.iterations)
            conv.append(r.converged)
        gbs = rows * 8 * n / (kms / 1e3) / 1e9
        out.append({"workload": tag, "desc": desc, "rows_per_s": rows / (lms / 1e3),
                    "ms_per_step": lms / n_steps, "iterations": its, "kernel": r.gpu["kernel"],
                    "ctas": r.gpu["ctas"], "threads": r.gpu["threads"], "plan": r.gpu.get("plan"),
                    **({"converged": conv} if budget is None else {}),
                    "roofline": {"achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak}})

    def guarded(fn):
        try:
            fn()
        except Exception as exc:  # extras must never sink the headline line
            out.append({"error": f"{fn.__name__}: {exc!r}"})

    def c3_rka():
        with DeviceSystem(m=C3_M, n=C3_N, device=device) as ds:
            ds.generate_counter(C3_SEED)
            measure("c3_rka", ds, C3_N, SolverConfig(variant="rka", q=64, sampling_scheme="distributed",
                                                       device=device), 400,
                    "c3: 160000x20000 counter-keyed, RKA q=64 (bs=1) distributed, 400 iterations per step")

    def c3_sharded_protocol():
        # the multi-GPU protocol at one rank: per outer iteration the local chain-kernel step, an
        # in-place NCCL all-reduce (a one-rank communicator) and x = S / Q, against kz_solve's
        # in-kernel average -- the per-iteration cost the N-GPU bench adds to the same local work
        from paper_2401_17474_b200.multigpu import CudaShard, ShardComm, plan_shards, solve_sharded_native

        plan = plan_shards(C3_M, 1, 0, C3_Q)
        shard = CudaShard.counter(C3_M, C3_N, plan, C3_SEED, device)
        comm = ShardComm(device, 1, 0)
        try:
            cfg = SolverConfig(variant="rkab", q=C3_Q, block_size=C3_BS, sampling_scheme="distributed",
                               device=device)
            budget = 100
            solve_sharded_native(shard, cfg, budget=budget, comm=comm)  # warm-up
            loop = [solve_sharded_native(shard, cfg.replace(base_seed=k), budget=budget, comm=comm) for k in range(2)]
            solo = [solve_sharded_native(shard, cfg.replace(base_seed=k), budget=budget) for k in range(2)]
            same = all(np.array_equal(a.x, b.x) for a, b in zip(loop, solo))
            lms = float(np.mean([r.gpu["loop_ms"] for r in loop])) / budget
            sms = float(np.mean([r.gpu["loop_ms"] for r in solo])) / budget
            out.append({"workload": "c3_sharded_protocol_world1",
                        "desc": "c3 RKAB q=64 bs=1000, 100-iteration replays: the row-sharded protocol at one rank "
                                "(per iteration: chain step, NCCL all-reduce, average kernel) vs kz_solve's in-kernel "
                                "average",
                        "ms_per_iteration_protocol": lms, "ms_per_iteration_in_kernel": sms,
                        "protocol_overhead": lms / sms - 1.0, "x_bitwise_equal": same})
        finally:
            shard.close()
            comm.close()

    def c4():
        s4 = generate_mother(GeneratorConfig(m_max=80000, n_max=2000, seed=0))
        with DeviceSystem(s4, device=device) as ds:
            measure("c4_rka_q64", ds, 2000, SolverConfig(variant="rka", q=64, device=device), 2000,
                    "c4 shape 80000x2000: RKA q=64, 2000 iterations per step")
            measure("c4_rka_q512", ds, 2000, SolverConfig(variant="rka", q=512, device=device), 500,
                    "c4 shape 80000x2000: RKA q=512, 500 iterations per step")
            measure("c4_rk_q1", ds, 2000, SolverConfig(variant="rk", device=device), 20000,
                    "c4 shape 80000x2000: RK (q=1), 20000 iterations per step")
            measure("c4shape_rkab_bs2000_to_eps", ds, 2000, SolverConfig(variant="rkab", q=64, block_size=2000,
                    device=device), None, "c4 shape 80000x2000 consistent: RKAB q=64 bs=2000, solved to 1e-8")
        # c4 proper: inconsistent b_LS = b + xi (sysgen.py:175-176), x_LS by CGLS on the device,
        # RKA horizons = mean of the last 10 trace records (harness.py:192-196), SURVEY 8(d) budgets
        from paper_2401_17474_b200.sysgen import TAG_NOISE, Prng

        b_ls = s4.b + Prng(0, TAG_NOISE).standard_normal(size=s4.m)
        inc = LinearSystem(A=s4.A, b=b_ls, x_star=None, x_ls=None, consistent=False, seed=0)
        with DeviceSystem(inc, device=device) as ds:
            t0 = time.perf_counter()
            x_ls = ds.cgls(tol=1e-12)
            cg_ms = (time.perf_counter() - t0) * 1e3
            for q, budget in ((1, 120000), (64, 60000), (512, 48000)):
                cfg = SolverConfig(variant="rka" if q > 1 else "rk", q=q, device=device, max_iterations=budget)
                cfgs = [cfg.replace(base_seed=k) for k in range(SEEDS)]
                lanes = 1 if q > 64 else SEEDS
                # warm-up (untimed): the lanes' system views, streams and samplers are built on first use
                solve_concurrent(ds, [c.replace(max_iterations=2000) for c in cfgs], lanes=lanes, x_ref=x_ls,
                                 trace_step=1000)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rs = solve_concurrent(ds, cfgs, lanes=lanes, x_ref=x_ls, trace_step=1000)
                e1.record()
                torch.cuda.synchronize()
                wall_ms = e0.elapsed_time(e1)
                hs = [float(np.mean([t.error_norm for t in r.trace[-10:]])) for r in rs]
                h = float(np.mean(hs))
                rows = sum(r.gpu["rows_projected"] for r in rs)
                # every trace record carries ||Ax - b||: records are evaluated 32 to a pass over A
                gemv_bytes = sum(-(-len(r.trace) // 32) for r in rs) * 8 * (inc.m * 2000 + inc.m)
                kms = sum(r.gpu["kernel_ms"] for r in rs)
                gbs = rows * 8 * 2000 / (kms / 1e3) / 1e9
                g = rs[0].gpu
                tot = (rows * 8 * 2000 + gemv_bytes) / (wall_ms / 1e3) / 1e9
                out.append({"workload": f"c4_horizon_q{q}", "desc": f"c4: 80000x2000 inconsistent (noise seed 0), "
                            f"{'RK' if q == 1 else 'RKA'} q={q}, {budget} iterations, trace every 1000 vs CGLS "
                            f"x_LS, solver seeds 0..9", "rows_per_s": rows / (wall_ms / 1e3), "ms_per_step": wall_ms,
                            "iterations": [r.iterations for r in rs], "kernel": g["kernel"], "ctas": g["ctas"],
                            "horizon_norm": h, "horizon_sq": h * h, "horizon_norm_per_seed": hs,
                            "trace_records": len(rs[0].trace), "cgls_ms": cg_ms,
                            "cgls_iterations": ds.cgls_iterations,
                            "roofline": {"achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
                                         "note": "per-solve kernel time"},
                            "step_traffic": {"row_bytes": rows * 8 * 2000, "residual_bytes": gemv_bytes,
                                             "gbs": tot, "frac": tot / peak}})

    def c2():
        s2 = generate_mother(GeneratorConfig(m_max=80000, n_max=1000, seed=0))
        with DeviceSystem(s2, device=device) as ds:
            cfg = SolverConfig(variant="rkab", q=64, block_size=500, device=device)
            measure("c2", ds, 1000, cfg, None, "c2: RKAB q=64 bs=500 80000x1000, solve to eps")
            # BASELINE c2's 10 seeds, two solves side by side: one solve occupies 64 of the 148 SMs
            # (64 workers, one CTA each), so a second lane runs on the others
            cfgs = [cfg.replace(base_seed=k) for k in range(SEEDS)]
            solve_concurrent(ds, cfgs, lanes=2)
            best = None
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rs = solve_concurrent(ds, cfgs, lanes=2)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                best = (ms, rs) if best is None or ms < best[0] else best
            ms, rs = best
            rows = sum(r.gpu["rows_projected"] for r in rs)
            gbs = rows * 8 * 1000 / (ms / 1e3) / 1e9
            out.append({"workload": "c2_ten_seeds", "desc": "c2: RKAB q=64 bs=500 80000x1000, the 10 seed-solves to "
                        "eps two at a time (solve_concurrent, lanes=2)", "rows_per_s": rows / (ms / 1e3),
                        "ms_per_step": ms, "iterations": [r.iterations for r in rs],
                        "converged": [r.converged for r in rs], "kernel": rs[0].gpu["kernel"],
                        "roofline": {"achieved_gbs": gbs, "peak_gbs": peak, "frac": gbs / peak,
                                     "note": "aggregate over the two lanes"}})

    def c1():
        # c1's 10 seed-solves side by side (solve_concurrent: 10 lanes, one 16-CTA cluster each)
        s1 = generate_mother(GeneratorConfig(m_max=20000, n_max=500, seed=0))
        cfg = SolverConfig(variant="rka", q=64, device=device)
        with DeviceSystem(s1, device=device) as ds:
            cfgs = [cfg.replace(base_seed=k) for k in range(SEEDS)]
            solve_concurrent(ds, cfgs, lanes=SEEDS)
            best = None
            for _ in range(3):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                rs = solve_concurrent(ds, cfgs, lanes=SEEDS)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                best = (ms, rs) if best is None or ms < best[0] else best
            ms, rs = best
            rows = sum(r.gpu["rows_projected"] for r in rs)
            alone = run_solver(ds, cfg)
            out.append({"workload": "c1_ten_seeds", "desc": "c1: RKA q=64 20000x500, the 10 seed-solves to eps side "
                        "by side (solve_concurrent)", "rows_per_s": rows / (ms / 1e3), "ms_per_step": ms,
                        "iterations": [r.iterations for r in rs], "converged": [r.converged for r in rs],
                        "kernel": rs[0].gpu["kernel"], "one_solve_alone_ms": alone.gpu["loop_ms"]})

    def c0():
        s0 = generate_mother(GeneratorConfig(m_max=2000, n_max=50, seed=0))
        with DeviceSystem(s0, device=device) as ds:
            c0cfg = SolverConfig(variant="rk", device=device)
            solve_seeds(ds, c0cfg, list(range(SEEDS)))
            best = None
            for _ in range(3):
                rb = solve_seeds(ds, c0cfg, list(range(SEEDS)))
                if best is None or rb[0].gpu["loop_ms"] < best[0].gpu["loop_ms"]:
                    best = rb
            rows = sum(r.iterations for r in best)
            out.append({"workload": "c0_ten_seeds", "desc": "c0: RK 2000x50, the 10 solver seeds to eps side by side "
                        "(one warp each, one launch per chunk)", "rows_per_s": rows / (best[0].gpu["loop_ms"] / 1e3),
                        "ms_per_step": best[0].gpu["loop_ms"], "iterations": [r.iterations for r in best],
                        "converged": [r.converged for r in best], "kernel": "warp"})

    for fn in (c3_rka, c3_sharded_protocol, c4, c2, c1, c0):
        guarded(fn)
    return out


_JSON_OUT = None  # the process's original stdout: the one JSON line goes there, everything else to stderr


def emit(line) -> None:
    out = _JSON_OUT if _JSON_OUT is not None else sys.stdout
    out.write(json.dumps(line) + "\n")
    out.flush()


def _free_port() -> int:
    with socket.socket(socket.AF_INET, socket.SOCK_STREAM) as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def spawn_ranks(n: int) -> int:
    """`--gpus N` without a launcher: one process per GPU through torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.run(cmd).returncode


def parse_args(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["b200", "reference"], default="b200")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extra", action="store_true", help="skip the other BASELINE workloads")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher path only (CPU, gloo): shard plans, rank agreement, the line's keys")
    return ap.parse_args(argv)


def main():
    global _JSON_OUT
    args = parse_args()
    if args.warmup < 3:
        sys.exit("bench.py: at least 3 warm-up steps (--warmup >= 3)")
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))
    world = int(env_world or "1")
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} disagrees with WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # libraries print to stdout at the C level (e.g. NCCL's version banner): keep stdout for the
    # JSON line only by pointing fd 1 at stderr for the rest of the run
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    if args.impl == "reference":
        run_reference(args, rank, world, local_rank)  # rank 0 alone; no process group needed
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        if args.dry_run:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # the init log names every communicator's nranks
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    try:
        if args.dry_run:
            run_dry(args, rank, world)
        else:
            run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


if __name__ == "__main__":
    main()
