"""CPU backend of one rank's local step for the row-sharded driver.

TEST INFRASTRUCTURE ONLY: lets tests/test_multirank_gloo.py run the
production host logic (paper_2401_17474_b200.multigpu.solve_sharded) over
gloo without a GPU.  It restates the reference's per-worker arithmetic
(solvers.py:107-117, 140-145; sampling.py:89-111) in numpy on the shard:
worker t draws from Prng(seed, t) over its shard-local block and the local
step returns the ordered sum S = sum_w v_w as a torch tensor.
"""

from __future__ import annotations

import numpy as np

import oracle as O


class CpuShard:
    def __init__(self, A_shard, b_shard, x_ref, plan):
        import torch

        self.torch = torch
        self.plan = plan
        self.A = np.ascontiguousarray(A_shard, dtype=np.float64)
        self.b = np.ascontiguousarray(b_shard, dtype=np.float64)
        self.xr = np.ascontiguousarray(x_ref, dtype=np.float64)
        self.sq = O.row_sqnorms(self.A)
        self.cdfs = [O.cdf(self.sq, lo, lo + ln - 1) for lo, ln in zip(plan.worker_lo, plan.worker_len)]
        self.xv = np.zeros(self.A.shape[1])
        self.gens = None

    def _gen(self, seed, t):
        return np.random.Generator(np.random.PCG64(np.random.SeedSequence(entropy=(seed, t))))

    def reset(self) -> float:
        self.xv[:] = 0.0
        self.gens = None
        return float(np.dot(self.xv - self.xr, self.xv - self.xr))

    def _draw(self, w):
        u = float(self.gens[w].random())
        c = self.cdfs[w]
        j = int(np.searchsorted(c, u, side="right"))
        return self.plan.worker_lo[w] + min(j, len(c) - 1)

    def step(self, cfg, k: int):
        if self.gens is None:
            self.gens = [self._gen(cfg.base_seed, self.plan.worker_offset + w) for w in range(self.plan.q_local)]
        steps = cfg.block_size if cfg.variant == "rkab" else 1
        S = None
        for w in range(self.plan.q_local):
            v = self.xv.copy()
            for _ in range(steps):
                i = self._draw(w)
                row = self.A[i]
                s = 1.0 * (self.b[i] - float(np.dot(row, v))) / self.sq[i]
                v += s * row
            S = v if S is None else S + v
        return self.torch.from_numpy(S.copy())

    def finish(self, S, Q: int) -> float:
        self.xv = S.numpy() / Q
        d = self.xv - self.xr
        return float(np.dot(d, d))

    def x(self):
        return self.xv.copy()
