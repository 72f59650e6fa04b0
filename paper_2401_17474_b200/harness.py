"""The reference's measurement protocol (kaczbench/harness.py:45-225) over the
B200 engine: per-seed iteration counts to the squared-error threshold, the
ceiling of their mean as the replay budget, timed fixed-budget replays with
the stop rule off, traces and plateaus.  The system is made resident once and
reused by every seed and replay; wall times are the device-timed loop."""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .errors import ConvergenceError
from .reports import RunReport, TraceRecord
from .solvers import DeviceSystem, SolverConfig, run_solver, solve_concurrent


@dataclass
class Protocol:
    n_seeds: int = 10
    epsilon: float = 1e-8
    trace_step: int = 1
    n_replay_runs: int = 10
    strict: bool = False

    def validate(self) -> None:
        if self.n_seeds < 1:
            raise ValueError(f"n_seeds must be >= 1, got {self.n_seeds}")
        if self.trace_step < 1:
            raise ValueError(f"trace_step must be >= 1, got {self.trace_step}")
        if self.n_replay_runs < 1:
            raise ValueError(f"n_replay_runs must be >= 1, got {self.n_replay_runs}")


@dataclass
class MeasureResult:
    reports: list[RunReport]
    mean_iterations: float
    budget: int
    all_converged: bool


@dataclass
class ReplayResult:
    total_s: float
    per_run_s: list[float]


def _resident(system, cfg):
    if isinstance(system, DeviceSystem):
        return system, False
    return DeviceSystem(system, device=cfg.device), True


def measure_iterations(system, cfg: SolverConfig, protocol: Protocol, *, lanes: int | None = None) -> MeasureResult:
    """Per-seed solves to epsilon (harness.py:127-149).  The seeds are independent solves of one
    resident system, so they run side by side (solve_concurrent, `lanes` at a time; lanes=1:
    one after another) -- bit-identical reports either way."""
    protocol.validate()
    ds, own = _resident(system, cfg)
    try:
        cfgs = [cfg.replace(base_seed=cfg.base_seed + j, epsilon=protocol.epsilon) for j in range(protocol.n_seeds)]
        if lanes == 1:
            reports = [run_solver(ds, c) for c in cfgs]
        else:
            reports = solve_concurrent(ds, cfgs, lanes=lanes)
    finally:
        if own:
            ds.close()
    counts = [r.iterations for r in reports if r.converged]
    if not counts:
        raise ConvergenceError(f"no seed converged within max_iterations={cfg.max_iterations}")
    mean = sum(counts) / len(counts)
    return MeasureResult(reports, mean, math.ceil(mean), len(counts) == len(reports))


def timed_replay(system, cfg: SolverConfig, fixed_iterations: int, n_runs: int = 10) -> ReplayResult:
    if fixed_iterations < 1:
        raise ValueError(f"fixed_iterations must be >= 1, got {fixed_iterations}")
    ds, own = _resident(system, cfg)
    per = []
    try:
        for _ in range(n_runs):
            r = run_solver(ds, cfg, budget=fixed_iterations)
            if r.error_evals != 0:
                raise RuntimeError("timed replay evaluated the stopping criterion; timing protocol violated")
            per.append(r.wall_time_s)
    finally:
        if own:
            ds.close()
    return ReplayResult(sum(per), per)


def trace_run(system, cfg: SolverConfig, max_iterations: int, trace_step: int, x_ref) -> list[TraceRecord]:
    return run_solver(system, cfg.replace(max_iterations=max_iterations), x_ref=x_ref, trace_step=trace_step).trace


def plateau_error(records: list[TraceRecord], tail: int = 10) -> float:
    if len(records) < tail:
        raise ValueError(f"need at least {tail} trace records, got {len(records)}")
    return float(np.mean([r.error_norm for r in records[-tail:]]))


def bench(system, cfg: SolverConfig, protocol: Protocol):
    ds, own = _resident(system, cfg)
    try:
        measure = measure_iterations(ds, cfg, protocol)
        replay = timed_replay(ds, cfg, measure.budget, n_runs=protocol.n_replay_runs)
    finally:
        if own:
            ds.close()
    first = measure.reports[0]
    summary = RunReport(variant=first.variant, q=first.q, block_size=first.block_size,
                        alpha_policy=first.alpha_policy, alpha=first.alpha, seed=-1, iterations=measure.budget,
                        converged=measure.all_converged, wall_time_s=replay.total_s,
                        final_error_sq=float("nan"), final_residual=float("nan"))
    rows = [("run", r) for r in measure.reports] + [("summary", summary)]
    return rows, measure, replay
