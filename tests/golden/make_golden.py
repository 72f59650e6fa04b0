"""Generate the golden fixtures under tests/golden/ by EXECUTING the reference.

Run in the build container only (the reference is not on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture records numpy's version; the reference's arithmetic lives in
numpy 2.3.5 / OpenBLAS 0.3.30 (third-party, pkg/pyproject.toml:10).  The
fixtures pin:

* prng.npz     -- Prng(seed, stream).random() streams and SeedSequence words
                  (sampling.py:34-74)
* norms.npz    -- row_norm_cache(A).sq_norms for seeded matrices of many widths
                  (linalg.py:80-88)
* systems.npz  -- sha256 of generate_mother / crop / make_inconsistent outputs
                  (sysgen.py:118-187), so the package's generator restatement
                  can be checked bitwise without the reference
* rows.npz     -- RowSampler.sample streams per worker (solvers.py:162-171,
                  sampling.py:89-111) for RK / RKA / RKAB configurations
* solves.npz   -- full reference solves: iteration counts, error_evals,
                  final_error_sq, final x and x checkpoints (capture lists)
                  for the BASELINE configs c0, c1, c2 and desk-scale cases
* traces.npz   -- trace_run records on an inconsistent system (harness.py:180-196)
* spectral.npz -- spectral_stats / optimal_alpha / partial_alphas (spectral.py:66-156) of
                  seeded systems, incl. a row block too short for its estimate
* threads.npz  -- the threaded engine's runs (parallel.py:175-304): delta-form RKA under a
                  lock and lead-row RKAB, final x, iterations and x checkpoints
* c1_ckpt100.npz -- c1 RKA q=64 seeds 0-2, the iterate every 100 iterations
* dist.npz     -- run_distributed_solve (distributed.py:339-363): the simulated-MPI
                  engine's RKA / RKAB (Algorithm 4: block_size + 1 rows, x / np
                  before the all-reduce) per-rank iterates
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

import kaczbench as kb  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from common import NORM_WIDTHS, THREAD_CASES, norm_matrix, sha  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
META = {"numpy_version": np.__version__, "generator": "tests/golden/make_golden.py"}


def save(name, **arrays):
    arrays.update({f"meta_{k}": np.array(v) for k, v in META.items()})
    np.savez_compressed(os.path.join(OUT, name), **arrays)
    print("wrote", name, flush=True)


PRNG_TUPLES = [(0, 0), (0, 1), (7, 3), (12345, 63), (2**33 + 1, 2), (2**40 + 5, 511), (3, 0, 5, 6)]
def gen_prng():
    out = {}
    for k, ent in enumerate(PRNG_TUPLES):
        p = kb.Prng(*ent)
        out[f"draws_{k}"] = np.array([p.random() for _ in range(1000)])
        out[f"entropy_{k}"] = np.array(ent, dtype=np.uint64)
        out[f"ssw_{k}"] = np.random.SeedSequence(entropy=ent).generate_state(8, np.uint32)
    save("prng.npz", **out)


def gen_norms():
    out = {}
    for n in NORM_WIDTHS:
        a = norm_matrix(n)
        out[f"sq_{n}"] = kb.row_norm_cache(a).sq_norms.copy()
        out[f"sha_{n}"] = np.array(sha(a))
    save("norms.npz", **out)


def system(m, n, seed):
    return kb.generate_mother(kb.GeneratorConfig(m_max=m, n_max=n, seed=seed))


def streams(sys_, cfg, count):
    cache = kb.row_norm_cache(sys_.A)
    samplers, rngs = kb.solvers.worker_streams(cache, cfg)
    return np.array([[samplers[t].sample(rngs[t]) for _ in range(count)] for t in range(cfg.q)],
                    dtype=np.int32)


def main():
    t0 = time.time()
    gen_prng()
    gen_norms()

    systems = {}
    c0 = system(2000, 50, 0)
    s500 = system(500, 20, 1)
    s2000 = system(2000, 50, 7)
    inc = kb.make_inconsistent(s2000, noise_seed=11)
    crop = kb.crop(s2000, 300, 40)
    c1 = system(20000, 500, 0)
    for name, s in [("c0", c0), ("s500", s500), ("s2000", s2000), ("inc2000", inc), ("crop300x40", crop),
                    ("c1", c1)]:
        systems[f"{name}_A"] = np.array(sha(s.A))
        systems[f"{name}_b"] = np.array(sha(s.b))
        ref = s.x_star if s.x_star is not None else s.x_ls
        systems[f"{name}_xref"] = np.array(sha(ref))
        systems[f"{name}_shape"] = np.array(s.A.shape)
    # x_ls itself (CGLS restatement is tolerance-checked, not hashed)
    systems["inc2000_xls"] = inc.x_ls.copy()
    print("systems done", time.time() - t0, flush=True)

    rows = {}
    for seed in range(10):
        rows[f"c0_rk_s{seed}"] = streams(c0, kb.SolverConfig(variant="rk", base_seed=seed), 2000)
    for scheme in ("full_access", "distributed"):
        for seed in (0, 1):
            cfg = kb.SolverConfig(variant="rka", q=64, base_seed=seed, sampling_scheme=scheme)
            rows[f"c1_q64_{scheme}_s{seed}"] = streams(c1, cfg, 256)
        cfg = kb.SolverConfig(variant="rka", q=8, base_seed=5, sampling_scheme=scheme)
        rows[f"s2000_q8_{scheme}_s5"] = streams(s2000, cfg, 1000)
    systems_c2 = system(80000, 1000, 0)
    systems["c2_A"] = np.array(sha(systems_c2.A))
    systems["c2_b"] = np.array(sha(systems_c2.b))
    systems["c2_xref"] = np.array(sha(systems_c2.x_star))
    systems["c2_shape"] = np.array(systems_c2.A.shape)
    rows["c2_q64_full_access_s0"] = streams(systems_c2, kb.SolverConfig(variant="rkab", q=64, block_size=500,
                                                                        base_seed=0), 256)
    save("systems.npz", **systems)
    save("rows.npz", **rows)
    print("rows done", time.time() - t0, flush=True)

    solves = {}

    def record(tag, sys_, cfg, every, **kw):
        cap = []
        r = kb.run_solver(sys_, cfg, capture=cap, **kw)
        solves[f"{tag}_iterations"] = np.array(r.iterations)
        solves[f"{tag}_error_evals"] = np.array(r.error_evals)
        solves[f"{tag}_converged"] = np.array(r.converged)
        solves[f"{tag}_final_error_sq"] = np.array(r.final_error_sq)
        solves[f"{tag}_final_residual"] = np.array(r.final_residual)
        solves[f"{tag}_x"] = r.x.copy()
        solves[f"{tag}_every"] = np.array(every)
        solves[f"{tag}_ckpt"] = np.array(cap[every - 1::every]) if len(cap) >= every else np.zeros((0, sys_.n))
        print(tag, r.iterations, r.converged, f"{time.time() - t0:.1f}s", flush=True)

    for seed in range(10):
        record(f"c0_rk_s{seed}", c0, kb.SolverConfig(variant="rk", base_seed=seed), 100)
    for seed in range(3):
        record(f"c1_rka64_s{seed}", c1, kb.SolverConfig(variant="rka", q=64, base_seed=seed), 1000)
    record("c2_rkab64_bs500_s0", systems_c2, kb.SolverConfig(variant="rkab", q=64, block_size=500,
                                                             base_seed=0), 1)
    # desk-scale cases: reduction identities, schemes, weights, budget replay
    record("s500_rk_s5", s500, kb.SolverConfig(variant="rk", base_seed=5), 1)
    record("s500_rka3_s2", s500, kb.SolverConfig(variant="rka", q=3, base_seed=2), 1)
    record("s500_rkab3_bs1_s2", s500, kb.SolverConfig(variant="rkab", q=3, block_size=1, base_seed=2), 1)
    record("s500_rkab4_bs8_s3", s500, kb.SolverConfig(variant="rkab", q=4, block_size=8, base_seed=3), 1)
    record("s2000_rka8_dist_s1", s2000, kb.SolverConfig(variant="rka", q=8, base_seed=1,
                                                        sampling_scheme="distributed"), 10)
    record("s2000_rkab8_bs50_dist_s4", s2000, kb.SolverConfig(variant="rkab", q=8, block_size=50, base_seed=4,
                                                              sampling_scheme="distributed"), 1)
    record("s2000_rka16_fixed_s0", s2000, kb.SolverConfig(variant="rka", q=16, alpha_policy="fixed",
                                                          alpha=1.7, base_seed=0), 10)
    record("s500_rka4_budget50_s9", s500, kb.SolverConfig(variant="rka", q=4, base_seed=9), 1, budget=50)
    record("s500_rkab5_bs7_budget20_s6", s500, kb.SolverConfig(variant="rkab", q=5, block_size=7, base_seed=6),
           1, budget=20)
    save("solves.npz", **solves)

    traces = {}
    for q in (1, 4, 16):
        recs = kb.trace_run(inc, kb.SolverConfig(variant="rka", q=q, base_seed=0), 3000, 100, inc.x_ls)
        traces[f"inc2000_rka{q}"] = np.array([[r.iteration, r.error_norm, r.residual_norm] for r in recs])
        traces[f"inc2000_rka{q}_plateau"] = np.array(kb.plateau_error(recs))
    save("traces.npz", **traces)
    print("all done", time.time() - t0)


def gen_ck():
    """Cyclic Kaczmarz (solvers.py:271-291): rows i = k mod m, no stream."""
    t0 = time.time()
    c0 = system(2000, 50, 0)
    s500 = system(500, 20, 1)
    s2000 = system(2000, 50, 7)
    crop = kb.crop(s2000, 300, 40)
    out = {}

    def record(tag, sys_, cfg, every, **kw):
        cap = []
        r = kb.run_solver(sys_, cfg, capture=cap, **kw)
        out[f"{tag}_iterations"] = np.array(r.iterations)
        out[f"{tag}_error_evals"] = np.array(r.error_evals)
        out[f"{tag}_converged"] = np.array(r.converged)
        out[f"{tag}_final_error_sq"] = np.array(r.final_error_sq)
        out[f"{tag}_x"] = r.x.copy()
        out[f"{tag}_every"] = np.array(every)
        out[f"{tag}_ckpt"] = np.array(cap[every - 1::every]) if len(cap) >= every else np.zeros((0, sys_.n))
        print(tag, r.iterations, r.converged, f"{time.time() - t0:.1f}s", flush=True)

    record("c0_ck", c0, kb.SolverConfig(variant="ck"), 100)
    record("s500_ck", s500, kb.SolverConfig(variant="ck"), 1)
    record("s2000_ck_fixed", s2000, kb.SolverConfig(variant="ck", alpha_policy="fixed", alpha=1.5), 10)
    record("crop300x40_ck", crop, kb.SolverConfig(variant="ck"), 10)
    record("s500_ck_budget777", s500, kb.SolverConfig(variant="ck"), 1, budget=777)
    record("c0_ck_max300", c0, kb.SolverConfig(variant="ck", max_iterations=300), 10)
    save("ck.npz", **out)


def gen_dist():
    """The reference's simulated-MPI engine (distributed.py:282-363, the paper's Algorithms 2 and 4):
    run_distributed_solve over `size` ranks, one worker per rank, x/np before the all-reduce."""
    t0 = time.time()
    c0 = system(2000, 50, 0)
    s2000 = system(2000, 50, 7)
    out = {}

    def record(tag, sys_, cfg, size, every, **kw):
        caps = [[] for _ in range(size)]
        reps = kb.run_distributed_solve(sys_, cfg, size, captures=caps, **kw)
        r = reps[0]
        assert all(np.array_equal(q.x, r.x) for q in reps)
        out[f"{tag}_size"] = np.array(size)
        out[f"{tag}_iterations"] = np.array(r.iterations)
        out[f"{tag}_error_evals"] = np.array(r.error_evals)
        out[f"{tag}_converged"] = np.array(r.converged)
        out[f"{tag}_final_error_sq"] = np.array(r.final_error_sq)
        out[f"{tag}_x"] = r.x.copy()
        out[f"{tag}_every"] = np.array(every)
        cap = caps[0]
        out[f"{tag}_ckpt"] = np.array(cap[every - 1::every]) if len(cap) >= every else np.zeros((0, sys_.n))
        print(tag, r.iterations, r.converged, f"{time.time() - t0:.1f}s", flush=True)

    record("c0_rka_np4", c0, kb.SolverConfig(variant="rka", base_seed=0), 4, 50)
    record("c0_rka_np8_s3", c0, kb.SolverConfig(variant="rka", base_seed=3), 8, 50)
    record("s2000_rkab_np4_bs20", s2000, kb.SolverConfig(variant="rkab", block_size=20, base_seed=1), 4, 5)
    record("s2000_rkab_np2_bs7_budget", s2000, kb.SolverConfig(variant="rkab", block_size=7, base_seed=2), 2, 10,
           budget=60)
    record("c0_rka_np4_fixed", c0, kb.SolverConfig(variant="rka", alpha_policy="fixed", alpha=1.3), 4, 50)
    save("dist.npz", **out)


SPECTRAL_SYSTEMS = [("s500", 500, 20, 1), ("s2000", 2000, 50, 7), ("c0", 2000, 50, 0), ("s3000x120", 3000, 120, 4)]
SPECTRAL_Q = [1, 2, 8, 64]


def gen_spectral():
    """spectral.py:66-156 executed: the extreme eigenvalue estimates, the optimal weights for
    several q, per-block partial weights (q = 4 and 8), and the rank-deficient-block error."""
    out = {}
    for name, m, n, seed in SPECTRAL_SYSTEMS:
        a = system(m, n, seed).A
        st = kb.spectral_stats(a)
        out[f"{name}_stats"] = np.array([st.sigma_max, st.sigma_min, st.s_min, st.s_max])
        out[f"{name}_alpha"] = np.array([kb.optimal_alpha(st, q) for q in SPECTRAL_Q])
        for q in (4, 8):
            if m // q >= n:
                out[f"{name}_partial_q{q}"] = kb.partial_alphas(a, q)
    try:
        kb.partial_alphas(system(500, 20, 1).A, 32)
        out["short_block_error"] = np.array("")
    except kb.DimensionMismatchError as exc:
        out["short_block_error"] = np.array(str(exc))
    out["q_list"] = np.array(SPECTRAL_Q)
    save("spectral.npz", **out)


def gen_threads():
    """parallel.py:175-304 executed: solve_rka_parallel (x += alpha (b - <a, x_prev>) / (q sq) a
    under a lock, arrival order) and solve_rkab_parallel (lead row + block, x += (v - x) / q);
    every iterate captured, every 10th stored."""
    out = {}
    for name, (m, n, seed), variant, q, bs, base in THREAD_CASES:
        s = system(m, n, seed)
        cfg = kb.SolverConfig(variant=variant, q=q, block_size=bs, base_seed=base)
        cap = []
        fn = kb.solve_rka_parallel if variant == "rka" else kb.solve_rkab_parallel
        r = fn(s, cfg, capture=cap)
        out[f"{name}_x"] = r.x.copy()
        out[f"{name}_it"] = np.array(r.iterations)
        out[f"{name}_conv"] = np.array(r.converged)
        out[f"{name}_err"] = np.array(r.final_error_sq)
        out[f"{name}_ckpt"] = np.array(cap[9::10]) if len(cap) >= 10 else np.zeros((0, n))
        print(name, r.iterations, flush=True)
    save("threads.npz", **out)


def gen_c1_ckpt100():
    """c1 (RKA q=64, 20000 x 500) seeds 0-2: the reference's iterate every 100 iterations
    (SURVEY 8(c) T3 cadence; solves.npz keeps every 1000th)."""
    c1 = system(20000, 500, 0)
    out = {}
    for seed in range(3):
        cap = []
        r = kb.run_solver(c1, kb.SolverConfig(variant="rka", q=64, base_seed=seed), capture=cap)
        out[f"s{seed}_iterations"] = np.array(r.iterations)
        out[f"s{seed}_ckpt"] = np.array(cap[99::100])
        print("c1 ckpt100", seed, r.iterations, flush=True)
    save("c1_ckpt100.npz", **out)


def gen_kzsys():
    """A KZSYS v1 file written by the reference's own save_system (sysgen.py:190-214)."""
    kb.save_system(system(500, 20, 1), os.path.join(OUT, "kzsys_s500.bin"))
    print("wrote kzsys_s500.bin")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "ck":
        gen_ck()
    elif len(sys.argv) > 1 and sys.argv[1] == "kzsys":
        gen_kzsys()
    elif len(sys.argv) > 1 and sys.argv[1] == "dist":
        gen_dist()
    elif len(sys.argv) > 1 and sys.argv[1] == "spectral":
        gen_spectral()
    elif len(sys.argv) > 1 and sys.argv[1] == "threads":
        gen_threads()
    elif len(sys.argv) > 1 and sys.argv[1] == "c1ckpt":
        gen_c1_ckpt100()
    else:
        main()
        gen_ck()
        gen_kzsys()
        gen_dist()
        gen_spectral()
        gen_threads()
        gen_c1_ckpt100()
