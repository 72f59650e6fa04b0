"""Row-sharded RKA / RKAB across GPUs of one node (one process per GPU).

Reference: kaczbench/distributed.py:189-336 (row shards per rank, one
all-reduce of x per outer iteration) generalised to q workers per rank, and
the sequential oracle it must match, solvers.py:313-371 with
``sampling_scheme="distributed"`` and q_total = q_per_rank * world:

* rank g owns rows ``partition_bounds(m, G, g)`` (make_partition,
  distributed.py:204-213) and, of the global matrix, nothing else;
* its workers are global workers ``t = g*q + w``; worker t samples block
  ``partition_bounds(m, Q, t)`` with stream ``Prng(seed, t)``
  (solvers.py:162-171).  These blocks nest exactly inside the rank's shard
  (floor(g*q*m / (G*q)) == floor(g*m/G)), so every draw is local;
* per outer iteration each rank forms the ordered local sum
  ``S_g = sum_w v_w`` on its GPU, the ranks all-reduce S (NCCL over NVLink;
  every rank ends bit-identical, as the reference's hypercube sum does,
  distributed.py:11-14), and x = S / Q;
* the stop rule is evaluated on the replicated x by every rank with the
  same deterministic reduction, so all ranks agree without communication
  (distributed.py:233-235).

The local step is pluggable: ``CudaShard`` (libkz_b200 kernels) in
production; tests drive the identical host logic with a CPU backend over
gloo (tests/test_multirank_gloo.py).
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from .reports import RunReport
from .sysgen import partition_bounds


@dataclass(frozen=True)
class ShardPlan:
    rank: int
    world: int
    m: int
    q_local: int
    lo: int  # first global row of this rank's shard
    hi: int  # last global row (inclusive)
    worker_offset: int  # global id of local worker 0
    worker_lo: tuple  # per local worker: first row, shard-local
    worker_len: tuple

    @property
    def q_total(self) -> int:
        return self.q_local * self.world

    @property
    def m_local(self) -> int:
        return self.hi - self.lo + 1


def plan_shards(m: int, world: int, rank: int, q_local: int) -> ShardPlan:
    """Shard and worker ranges of one rank; raises if the blocks do not nest."""
    lo, hi = partition_bounds(m, world, rank)
    Q = q_local * world
    wlo, wlen = [], []
    for w in range(q_local):
        t = rank * q_local + w
        a, b = partition_bounds(m, Q, t)
        if a < lo or b > hi:
            raise AssertionError(f"worker block {t} [{a}, {b}] escapes shard [{lo}, {hi}]")
        wlo.append(a - lo)
        wlen.append(b - a + 1)
    return ShardPlan(rank, world, m, q_local, lo, hi, rank * q_local, tuple(wlo), tuple(wlen))


class CudaShard:
    """The rank's shard resident on its GPU; local steps run in libkz_b200."""

    def __init__(self, A_shard, b_shard, x_ref, plan: ShardPlan, device: int):
        import torch

        from .solvers import DeviceSystem

        self.plan = plan
        self.ds = DeviceSystem(m=A_shard.shape[0], n=A_shard.shape[1], device=device)
        self.ds.upload(A_shard, b_shard, x_ref)
        self.ds.set_ranges(plan.worker_lo, plan.worker_len)
        self.S = torch.zeros(self.ds.pitch, dtype=torch.float64, device=f"cuda:{device}")
        self.kernel_ms = 0.0
        self.rows = 0
        self.kernel = None

    @classmethod
    def counter(cls, m_total: int, n: int, plan: ShardPlan, seed: int, device: int) -> "CudaShard":
        """The rank's rows of the counter-keyed config-3 system, generated in place on its GPU
        (bit-identical to rows [lo, hi] of the full matrix; no host copy)."""
        import torch

        from .solvers import DeviceSystem

        self = cls.__new__(cls)
        self.plan = plan
        self.ds = DeviceSystem(m=plan.m_local, n=n, device=device)
        self.ds.generate_counter(seed, row0=plan.lo)
        self.ds.set_ranges(plan.worker_lo, plan.worker_len)
        self.S = torch.zeros(self.ds.pitch, dtype=torch.float64, device=f"cuda:{device}")
        self.kernel_ms = 0.0
        self.rows = 0
        self.kernel = None
        return self

    def reset(self) -> float:
        self.ds.set_x(None)
        return self.ds.error_sq()

    def step(self, cfg, k: int):
        info = self.ds.local_step(cfg, k=k, worker_offset=self.plan.worker_offset, partial_ptr=self.S.data_ptr())
        self.kernel_ms += info["kernel_ms"]
        self.rows += info["rows"]
        self.kernel = info["kernel"]
        return self.S

    def finish(self, S, Q: int) -> float:
        return self.ds.average_from(S.data_ptr(), Q)

    def x(self) -> np.ndarray:
        return self.ds.x_host()

    def close(self):
        self.ds.close()


class ShardComm:
    """The ranks' NCCL communicator for the native sharded loop (kz_comm_*): rank 0 draws
    the unique id, torch.distributed broadcasts its bytes, every rank joins."""

    def __init__(self, device: int, world: int, rank: int, group=None):
        import ctypes as C

        from . import _native as N

        self._lib = N.load_library()
        obj = [None]
        if rank == 0:
            buf = C.create_string_buffer(N.COMM_ID_BYTES)
            N.check(self._lib.kz_comm_unique_id(buf))
            obj = [bytes(buf.raw)]
        if world > 1:
            import torch.distributed as dist

            dist.broadcast_object_list(obj, src=0, group=group)
        h = C.c_void_p()
        N.check(self._lib.kz_comm_create(int(device), obj[0], int(world), int(rank), C.byref(h)))
        self.handle, self.world, self.rank, self.group = h, world, rank, group
        self.exchange_ld = None

    def connect_exchange(self, ld: int) -> None:
        """The fused cross-rank exchange (kz_comm_exchange_*): every rank exports the IPC handle of
        its column-sum buffer, the handles are all-gathered in rank order, every rank maps the
        others' buffers.  Collective: all ranks call it with the same shard pitch."""
        import ctypes as C

        from . import _native as N

        if self.exchange_ld == ld:
            return
        buf = C.create_string_buffer(N.COMM_HANDLE_BYTES)
        N.check(self._lib.kz_comm_exchange_handle(self.handle, int(ld), buf))
        handles = [bytes(buf.raw)]
        if self.world > 1:
            import torch.distributed as dist

            handles = [None] * self.world
            dist.all_gather_object(handles, bytes(buf.raw), group=self.group)
        N.check(self._lib.kz_comm_exchange_connect(self.handle, b"".join(handles)))
        self.exchange_ld = ld

    def close(self):
        if getattr(self, "handle", None):
            self._lib.kz_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_sharded_native(shard: "CudaShard", cfg, *, budget: int | None = None, comm: ShardComm | None = None,
                         fused: bool = True, loop: bool = False) -> RunReport:
    """The same protocol as :func:`solve_sharded`, run by the library (kz_solve_sharded).
    RKA with ``fused`` (default): one step-kernel launch per chunk of outer iterations, the
    ranks' column sums exchanged inside the kernel over NVLink peer memory (the communicator's
    exchange buffers) and the stop rule applied in-kernel.  Otherwise (RKAB, or fused=False):
    per outer iteration a local step, an in-place NCCL all-reduce and x = S / Q, enqueued on one
    stream without a host round trip; a device stop flag freezes x at the stopping iteration.
    Same iteration counts as the host-driven loop; the same x bit for bit at one rank.
    Without a communicator (one rank) the library runs kz_solve's chunked kernels on the shard
    unless ``loop`` asks for the per-iteration loop."""
    plan = shard.plan
    if comm is None and plan.world > 1:
        raise ValueError("a multi-rank sharded solve needs a ShardComm")
    if comm is not None and fused and cfg.variant == "rka":
        comm.connect_exchange(shard.ds.pitch)
    t0 = time.perf_counter()
    r = shard.ds.solve_sharded(cfg, worker_offset=plan.worker_offset, comm=comm, budget=budget, fused=fused,
                               loop=loop)
    wall = time.perf_counter() - t0
    shard.rows += r["rows"]
    shard.kernel_ms += r["loop_ms"]
    shard.kernel = r["kernel"]
    return RunReport(variant=cfg.variant, q=plan.q_total, block_size=cfg.block_size if cfg.variant == "rkab" else 1,
                     alpha_policy=cfg.alpha_policy, alpha=1.0, seed=cfg.base_seed, iterations=r["iterations"],
                     converged=r["converged"], wall_time_s=wall, final_error_sq=r["final_error_sq"],
                     final_residual=float("nan"), error_evals=r["error_evals"], x=r["x"],
                     gpu={"world": plan.world, "q_local": plan.q_local, "shard": (plan.lo, plan.hi),
                          "native": True, "fused": bool(fused and comm is not None and cfg.variant == "rka"),
                          "loop_ms": r["loop_ms"], "kernel_ms": r["kernel_ms"], "launches": r["launches"],
                          "kernel": r["kernel"], "ctas": r["ctas"], "threads": r["threads"], "plan": r["plan"]})


def solve_sharded(shard, cfg, *, budget: int | None = None, group=None) -> RunReport:
    """The _drive protocol (solvers.py:182-263) over row shards with one
    all-reduce-sum per outer iteration.  ``shard`` provides reset/step/finish/x
    (CudaShard, or the CPU backend in the tests)."""
    import torch.distributed as dist

    plan = shard.plan
    Q = plan.q_total
    t0 = time.perf_counter()
    err = shard.reset()
    k, evals, converged = 0, 0, False
    while True:
        if budget is None:
            evals += 1
            if err < cfg.epsilon:
                converged = True
                break
            if k >= cfg.max_iterations:
                break
        elif k >= budget:
            break
        S = shard.step(cfg, k)
        if plan.world > 1:
            dist.all_reduce(S, op=dist.ReduceOp.SUM, group=group)
        err = shard.finish(S, Q)
        k += 1
    wall = time.perf_counter() - t0
    return RunReport(variant=cfg.variant, q=Q, block_size=cfg.block_size if cfg.variant == "rkab" else 1,
                     alpha_policy=cfg.alpha_policy, alpha=1.0, seed=cfg.base_seed, iterations=k,
                     converged=converged, wall_time_s=wall,
                     final_error_sq=float(err) if budget is None else float("nan"),
                     final_residual=float("nan"), error_evals=evals, x=shard.x(),
                     gpu={"world": plan.world, "q_local": plan.q_local, "shard": (plan.lo, plan.hi)})
