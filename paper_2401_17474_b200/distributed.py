"""The reference's simulated-MPI engine (kaczbench/distributed.py:282-363, the
paper's Algorithms 2 and 4) on the B200.

``run_distributed_solve(system, cfg, size)`` runs ``size`` ranks of one worker
each: rank r owns rows ``partition_bounds(m, size, r)`` (make_partition,
distributed.py:204-213), samples them norm-weighted with stream
``Prng(seed, r)`` and, per outer iteration, projects once (RKA) or
``block_size + 1`` times in a chain (RKAB, Algorithm 4 literal: bs chained
projections and one more folded into the division), then x = the rank average
(``x /= np`` and the all-reduce sum, distributed.py:296-301 / 321-331).

That is exactly the sequential engine with q = size workers, the
``distributed`` sampling scheme (worker t = rank t's block and stream) and, for
RKAB, ``lead_row`` (block_size + 1 rows per worker): one GPU solve replaces the
``size`` simulated ranks and their transport.  Iterates agree with the
reference to rounding (its x / np before the hypercube sum vs the ordered sum
then / q here; tests/test_gpu_solves.py::test_run_distributed_solve_matches_reference
pins them against the reference's own runs, tests/golden/dist.npz).  Every rank's
report carries the same iterate, as the reference's byte-identical ranks do.
For the row-sharded multi-GPU path with q workers per GPU see multigpu.py.
"""

from __future__ import annotations

import dataclasses

from .reports import RunReport
from .solvers import SolverConfig, solve_rka_seq, solve_rkab_seq


def run_distributed_solve(system, cfg: SolverConfig, size: int, *, x_ref=None, budget=None, latency=None,
                          captures: list | None = None) -> list[RunReport]:
    """distributed.py:339-363 -- returns the ``size`` per-rank reports (identical iterates).
    ``latency`` (the SimTransport's simulated network delay) has no counterpart here."""
    cfg.validate()
    if cfg.variant not in ("rka", "rkab"):
        raise ValueError(f"distributed solve supports rka/rkab, got {cfg.variant!r}")
    if size < 1:
        raise ValueError(f"size must be >= 1, got {size}")
    if budget is None and x_ref is None:
        x_ref = system.x_ref() if hasattr(system, "x_ref") and callable(system.x_ref) else None
    c = cfg.replace(q=size, sampling_scheme="distributed")
    cap = [] if captures is not None else None
    if cfg.variant == "rka":
        r = solve_rka_seq(system, c, x_ref=x_ref, budget=budget, capture=cap)
    else:
        r = solve_rkab_seq(system, c, x_ref=x_ref, budget=budget, capture=cap, lead_row=True)
    if captures is not None:
        for lst in captures[:size]:
            lst.extend(x.copy() for x in cap)
    # the rank sees only its block: no global residual (distributed.py:276)
    r = dataclasses.replace(r, final_residual=float("nan"))
    return [dataclasses.replace(r, x=r.x.copy()) for _ in range(size)]
