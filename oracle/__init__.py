"""ctypes binding of the CPU oracle (``oracle/libkz_oracle.so``).

TEST INFRASTRUCTURE ONLY.  Imported by ``tests/``, ``__graft_entry__.smoke()``
and the CPU legs of ``bench.py`` (``cpu_baseline`` and ``--impl reference``)
as the checker / CPU baseline.  The product package
``paper_2401_17474_b200`` never imports this module.

Each function restates one reference function (paths relative to
``/root/reference/pkg/src/kaczbench``); see ``kz_oracle.c`` for the
arithmetic and ``tests/golden/make_golden.py`` for the pinning fixtures.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libkz_oracle.so")
_lib = None

VARIANTS = {"rk": 0, "rka": 1, "rkab": 2, "ck": 3}
SCHEMES = {"full_access": 0, "distributed": 1}

OK, EINVAL, EDEGENERATE, EEMPTYRANGE, ENOMEM = range(5)


class _Params(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("scheme", C.c_int32),
        ("q", C.c_int64),
        ("block_size", C.c_int64),
        ("alphas", C.POINTER(C.c_double)),
        ("base_seed", C.c_uint64),
        ("epsilon", C.c_double),
        ("max_iterations", C.c_int64),
        ("budget", C.c_int64),
        ("ckpt_every", C.c_int64),
        ("ckpt_capacity", C.c_int64),
        ("nthreads", C.c_int32),
        ("combine", C.c_int32),
    ]


class _Result(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("converged", C.c_int32),
        ("pad", C.c_int32),
        ("final_error_sq", C.c_double),
        ("error_evals", C.c_int64),
        ("n_ckpt", C.c_int64),
        ("bad_row", C.c_int64),
        ("loop_seconds", C.c_double),
    ]


def build() -> str:
    """Compile the oracle from its sources with the committed Makefile."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        dp = C.POINTER(C.c_double)
        L.kzo_random_doubles.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, dp]
        L.kzo_row_sqnorms.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, dp]
        L.kzo_cdf_build.argtypes = [dp, C.c_int64, C.c_int64, C.c_int64, dp]
        L.kzo_cdf_build.restype = C.c_int32
        L.kzo_upper_bound.argtypes = [dp, C.c_int64, C.c_double]
        L.kzo_upper_bound.restype = C.c_int64
        L.kzo_dump_rows.argtypes = [dp, C.c_int64, C.c_int32, C.c_int64, C.c_uint64, C.c_int64,
                                    C.c_int64, C.POINTER(C.c_int64)]
        L.kzo_dump_rows.restype = C.c_int32
        L.kzo_seedseq_generate.argtypes = [C.POINTER(C.c_uint64), C.c_int32,
                                           C.POINTER(C.c_uint32), C.c_int32]
        L.kzo_solve.argtypes = [dp, dp, dp, C.c_int64, C.c_int64, C.POINTER(_Params),
                                C.POINTER(_Result), dp, dp]
        L.kzo_solve.restype = C.c_int32
        L.kzo_max_threads.restype = C.c_int32
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a, ndim):
    a = np.ascontiguousarray(a, dtype=np.float64)
    assert a.ndim == ndim
    return a


def max_threads() -> int:
    return int(lib().kzo_max_threads())


def seedseq_state(entropy, n_words=8) -> np.ndarray:
    """SeedSequence(entropy).generate_state(n_words, uint32) (sampling.py:47)."""
    ent = (C.c_uint64 * len(entropy))(*[int(e) for e in entropy])
    out = np.empty(n_words, dtype=np.uint32)
    lib().kzo_seedseq_generate(ent, len(entropy), out.ctypes.data_as(C.POINTER(C.c_uint32)), n_words)
    return out


def random_doubles(seed: int, stream: int, count: int) -> np.ndarray:
    """Prng(seed, stream).random() repeated (sampling.py:44-52)."""
    out = np.empty(count)
    lib().kzo_random_doubles(seed, stream, count, _dp(out))
    return out


def row_sqnorms(a) -> np.ndarray:
    """np.einsum('ij,ij->i', a, a) (linalg.py:83)."""
    a = _f64(a, 2)
    out = np.empty(a.shape[0])
    lib().kzo_row_sqnorms(_dp(a), a.shape[0], a.shape[1], a.shape[1], _dp(out))
    return out


def cdf(sq, lo=0, hi=None) -> np.ndarray:
    """make_sampler's cdf (sampling.py:101-111)."""
    sq = _f64(sq, 1)
    hi = sq.shape[0] - 1 if hi is None else hi
    out = np.empty(max(hi - lo + 1, 1))
    rc = lib().kzo_cdf_build(_dp(sq), sq.shape[0], lo, hi, _dp(out))
    if rc:
        raise ValueError(f"empty range [{lo}, {hi}]")
    return out


def dump_rows(sq, scheme: str, q: int, seed: int, worker: int, count: int) -> np.ndarray:
    """First `count` draws of worker `worker` (solvers.py:162-171, sampling.py:89-94)."""
    sq = _f64(sq, 1)
    out = np.empty(count, dtype=np.int64)
    rc = lib().kzo_dump_rows(_dp(sq), sq.shape[0], SCHEMES[scheme], q, seed, worker, count,
                             out.ctypes.data_as(C.POINTER(C.c_int64)))
    if rc:
        raise ValueError(f"dump_rows failed with status {rc}")
    return out


def solve(A, b, x_ref, *, variant="rk", q=1, block_size=1, alphas=None, base_seed=0,
          scheme="full_access", epsilon=1e-8, max_iterations=1_000_000, budget=None,
          ckpt_every=0, ckpt_capacity=None, nthreads=1, engine="seq") -> dict:
    """The reference solve protocol (solvers.py:182-263, 294-371).  engine="threads": the
    threaded engine's combine in worker order (parallel.py:175-304); RKAB then draws
    block_size + 1 rows per worker (the lead row), as solve_rkab_parallel does."""
    if engine not in ("seq", "threads"):
        raise ValueError(f"unknown engine {engine!r}")
    threads = engine == "threads" and variant in ("rka", "rkab") and q > 1
    if engine == "threads" and variant == "rkab":
        block_size += 1
    A = _f64(A, 2)
    b = _f64(b, 1)
    m, n = A.shape
    xr = _f64(x_ref if x_ref is not None else np.zeros(n), 1)
    al = None if alphas is None else _f64(np.broadcast_to(np.asarray(alphas, float), (q,)), 1)
    if ckpt_every and ckpt_capacity is None:
        ckpt_capacity = (budget if budget else max_iterations) // ckpt_every
    ckpt_capacity = int(ckpt_capacity or 0)
    ck = np.empty((max(ckpt_capacity, 1), n))
    p = _Params(VARIANTS[variant], SCHEMES[scheme], q, block_size,
                _dp(al) if al is not None else None, int(base_seed), float(epsilon),
                int(max_iterations), int(budget or 0), int(ckpt_every), ckpt_capacity,
                int(nthreads), int(threads))
    r = _Result()
    x = np.empty(n)
    rc = lib().kzo_solve(_dp(A), _dp(b), _dp(xr), m, n, C.byref(p), C.byref(r), _dp(x), _dp(ck))
    if rc == EDEGENERATE:
        raise ValueError(f"row {r.bad_row} has zero norm")
    if rc:
        raise ValueError(f"oracle solve failed with status {rc}")
    return {
        "iterations": int(r.iterations),
        "converged": bool(r.converged),
        "final_error_sq": float(r.final_error_sq) if not budget else float("nan"),
        "error_evals": int(r.error_evals),
        "x": x,
        "checkpoints": ck[: r.n_ckpt].copy(),
        "loop_seconds": float(r.loop_seconds),
    }
