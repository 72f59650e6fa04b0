"""RK / RKA / RKAB on the B200 behind the reference's entry points.

Same names, signatures, argument meaning and error behaviour as
kaczbench/solvers.py:55-371 and kaczbench/harness.py:98-114:

    fn(system, cfg, *, x_ref=None, budget=None, trace_step=None, capture=None) -> RunReport

``system`` is a :class:`~.sysgen.LinearSystem` (host arrays, uploaded per
call, like the reference recomputes its row norms per call) or a
:class:`DeviceSystem` (resident in HBM; norms and samplers cached).  The whole
iteration loop -- sampling, projections, averaging, the stop rule -- runs in
``libkz_b200.so``; there is no host fallback.
"""

from __future__ import annotations

import ctypes as C
import dataclasses
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionMismatchError
from .reports import RunReport, TraceRecord
from .sysgen import LinearSystem, einsum_order_matches, partition_bounds

VARIANTS = ("ck", "rk", "rka", "rkab", "cgls")
ALPHA_POLICIES = ("unit", "fixed", "optimal_full", "optimal_partial")
SAMPLING_SCHEMES = ("full_access", "distributed")
# "seq" and "threads" name the reference engines whose semantics are honoured
# (threads: the delta-form combine in worker order and RKAB's leading row,
# parallel.py:175-304; solve_rka_parallel / solve_rkab_parallel); all run on the B200.
ENGINES = ("b200", "seq", "threads")
KERNELS = tuple(N.KERNELS)

# capture=list keeps every iterate (reference semantics); refuse absurd sizes
_CAPTURE_LIMIT_BYTES = 4 << 30
_CAPTURE_FIRST_BYTES = 256 << 20


@dataclass
class SolverConfig:
    """Mirror of kaczbench.SolverConfig (solvers.py:61-104) plus device knobs."""

    variant: str = "rk"
    q: int = 1
    alpha_policy: str = "unit"
    alpha: float = 1.0
    block_size: int = 1
    epsilon: float = 1e-8
    max_iterations: int = 1_000_000
    base_seed: int = 0
    sampling_scheme: str = "full_access"
    engine: str = "b200"
    kernel: str = "auto"
    device: int = 0
    threads: int = 0  # CTA size override (0 = auto)
    ctas: int = 0     # CTA count override for the sync kernels (0 = auto)
    short_launches: bool = False  # stop mode: 2048-iteration launches (set by solve_concurrent)

    def validate(self) -> None:
        if self.variant not in VARIANTS:
            raise ValueError(f"unknown variant {self.variant!r}")
        if self.alpha_policy not in ALPHA_POLICIES:
            raise ValueError(f"unknown alpha policy {self.alpha_policy!r}")
        if self.sampling_scheme not in SAMPLING_SCHEMES:
            raise ValueError(f"unknown sampling scheme {self.sampling_scheme!r}")
        if self.engine not in ENGINES:
            raise ValueError(f"unknown engine {self.engine!r}")
        if self.kernel not in KERNELS:
            raise ValueError(f"unknown kernel {self.kernel!r}")
        if self.q < 1:
            raise ValueError(f"q must be >= 1, got {self.q}")
        if self.block_size < 1:
            raise ValueError(f"block_size must be >= 1, got {self.block_size}")
        if not self.epsilon > 0:
            raise ValueError(f"epsilon must be > 0, got {self.epsilon}")
        if self.max_iterations < 1:
            raise ValueError(f"max_iterations must be >= 1, got {self.max_iterations}")

    def replace(self, **kw) -> "SolverConfig":
        return dataclasses.replace(self, **kw)


class DeviceSystem:
    """A linear system resident in one GPU's HBM (C-ABI kz_system).

    A is stored row-major with a 128-byte row pitch.  Row norms and samplers
    are computed on first use and cached; inputs are never modified.
    """

    def __init__(self, system: LinearSystem | None = None, *, m: int | None = None, n: int | None = None,
                 device: int = 0):
        self._lib = N.load_library()
        if system is not None:
            m, n = system.A.shape if system.A.ndim == 2 else (None, None)
        if m is None or n is None:
            raise DimensionMismatchError("DeviceSystem needs a 2-D system or (m, n)")
        self.m, self.n, self.device = int(m), int(n), int(device)
        self.host = system
        h = C.c_void_p()
        N.check(self._lib.kz_system_create(self.device, self.m, self.n, C.byref(h)))
        self.handle = h
        self._xref_set = False
        if system is not None:
            xr = system.x_star if system.x_star is not None else system.x_ls
            self.upload(system.A, system.b, xr)

    @classmethod
    def from_file(cls, path, *, device: int = 0, rows: tuple[int, int] | None = None) -> "DeviceSystem":
        """A KZSYS v1 file (sysgen.py:190-271) loaded straight into HBM (kz_system_load_file);
        `rows` = (lo, hi) inclusive loads one row shard.  The host copy stays on disk."""
        lib = N.load_library()
        h = C.c_void_p()
        m_tot, n, flags = C.c_int64(), C.c_int64(), C.c_uint32()
        meta = np.empty(5)
        lo, hi = rows if rows is not None else (0, -1)
        N.check(lib.kz_system_load_file(int(device), str(path).encode(), C.c_int64(lo), C.c_int64(hi), C.byref(h),
                                        C.byref(m_tot), C.byref(n), C.byref(flags), N.ptr(meta)))
        self = cls.__new__(cls)
        self._lib = lib
        self.m = (int(hi) if hi >= 0 else int(m_tot.value) - 1) - int(lo) + 1
        self.n, self.device = int(n.value), int(device)
        self.host = None
        self.handle = h
        self._xref_set = bool(flags.value & 6)
        self.file_m, self.file_flags = int(m_tot.value), int(flags.value)
        self.file_meta = meta
        return self

    # -- residency -------------------------------------------------------------
    def upload(self, A, b, x_ref=None, stream=None) -> None:
        A = N.f64(A)
        b = N.f64(b)
        if A.ndim != 2:
            raise DimensionMismatchError(f"expected a 2-D matrix, got ndim={A.ndim}")
        if A.shape != (self.m, self.n):
            raise DimensionMismatchError(f"matrix {A.shape} does not match ({self.m}, {self.n})")
        if b.shape != (self.m,):
            raise DimensionMismatchError(f"expected length {self.m}, got {b.shape}")
        xr = None
        if x_ref is not None:
            xr = N.f64(x_ref)
            if xr.shape != (self.n,):
                raise DimensionMismatchError(f"expected length {self.n}, got {xr.shape}")
        N.check(self._lib.kz_system_upload(self.handle, N.ptr(A), self.n, N.ptr(b),
                                           N.ptr(xr) if xr is not None else None, stream))
        self._xref_set = xr is not None
        if not einsum_order_matches():  # another numpy build: the reference's own norms (Appendix A)
            self.set_row_norms(np.einsum("ij,ij->i", A, A))
        self._refresh_views()

    def set_row_norms(self, sq) -> None:
        """Host-computed squared row norms replace the device's (kz_row_norms_upload); a zero norm
        surfaces as DegenerateRowError at solve time, as in the reference."""
        sq = N.f64(sq)
        if sq.shape != (self.m,):
            raise DimensionMismatchError(f"expected length {self.m}, got {sq.shape}")
        rc = self._lib.kz_row_norms_upload(self.handle, N.ptr(sq), None)
        if rc != N.KZ_EDEGENERATE:
            N.check(rc)
        self._refresh_views()

    def upload_device(self, A_ptr: int, lda: int, b_ptr: int, xref_ptr: int | None = None, stream=None) -> None:
        """Copy from caller-owned device arrays (e.g. torch tensors' data_ptr())."""
        N.check(self._lib.kz_system_upload_device(self.handle, C.c_void_p(A_ptr), lda, C.c_void_p(b_ptr),
                                                  C.c_void_p(xref_ptr) if xref_ptr else None, stream))
        self._xref_set = bool(xref_ptr)
        self._refresh_views()

    def device_ptrs(self) -> tuple[int, int, int, int]:
        """(A, b, x_ref, pitch) device pointers, for in-place generation."""
        a, b, x = C.c_void_p(), C.c_void_p(), C.c_void_p()
        N.check(self._lib.kz_system_device_ptrs(self.handle, C.byref(a), C.byref(b), C.byref(x)))
        self._xref_set = True
        return a.value, b.value, x.value, self.pitch

    def generate_counter(self, seed: int = 0, mu_range=(-5.0, 5.0), sigma_range=(1.0, 20.0), row0: int = 0) -> None:
        """Fill the system with the counter-keyed BASELINE config-3 generator (device only);
        `row0` makes it rows [row0, row0 + m) of the full system (a row shard)."""
        N.check(self._lib.kz_generate_counter_rows(self.handle, C.c_uint64(int(seed)), C.c_int64(int(row0)),
                                                   C.c_double(mu_range[0]), C.c_double(mu_range[1]),
                                                   C.c_double(sigma_range[0]), C.c_double(sigma_range[1]), None))
        self._xref_set = True
        self._refresh_views()

    def download(self, m2: int | None = None, n2: int | None = None, out=None):
        """(A[:m2, :n2], b[:m2], x_ref[:n2]) copied to the host (into ``out`` = (A, b, x_ref)
        C-contiguous float64 arrays of those shapes when given, e.g. pinned buffers)."""
        m2 = self.m if m2 is None else m2
        n2 = self.n if n2 is None else n2
        if out is not None:
            A, b, xr = out
            for a, shp in ((A, (m2, n2)), (b, (m2,)), (xr, (n2,))):
                if a.shape != shp or a.dtype != np.float64 or not a.flags.c_contiguous:
                    raise DimensionMismatchError(f"download buffer {a.shape} {a.dtype} does not match {shp} f64")
        else:
            A = np.empty((m2, n2))
            b = np.empty(m2)
            xr = np.empty(n2)
        N.check(self._lib.kz_system_download(self.handle, m2, n2, N.ptr(A), N.ptr(b), N.ptr(xr), None))
        return A, b, xr

    def touch(self) -> None:
        N.check(self._lib.kz_system_touch(self.handle))
        self._refresh_views()

    def set_x_ref(self, x_ref) -> None:
        xr = N.f64(x_ref)
        if xr.shape != (self.n,):
            raise DimensionMismatchError(f"expected length {self.n}, got {xr.shape}")
        N.check(self._lib.kz_system_set_xref(self.handle, N.ptr(xr), None))
        self._xref_set = True
        self._refresh_views()

    @property
    def pitch(self) -> int:
        return int(self._lib.kz_system_pitch(self.handle))

    # -- sampler subsystem -----------------------------------------------------
    def row_norms(self) -> np.ndarray:
        """Squared row norms, bit-exact with np.einsum (linalg.py:80-88)."""
        out = np.empty(self.m)
        bad = C.c_int64(-1)
        rc = self._lib.kz_row_norms(self.handle, N.ptr(out), C.byref(bad), None)
        N.check(rc, bad_row=bad.value)
        return out

    def cdf(self, scheme: str = "full_access", q: int = 1) -> np.ndarray:
        """make_sampler cdf(s) (sampling.py:101-111), concatenated per block."""
        out = np.empty(self.m)
        N.check(self._lib.kz_sampler_build(self.handle, N.SCHEME_IDS[scheme], int(q), N.ptr(out), None))
        return out

    def dump_rows(self, base_seed: int, worker: int, count: int, *, scheme: str = "full_access", q: int = 1,
                  start: int = 0) -> np.ndarray:
        """Draws start..start+count-1 of worker `worker` (RowSampler.sample)."""
        out = np.empty(count, dtype=np.int32)
        N.check(self._lib.kz_dump_rows(self.handle, N.SCHEME_IDS[scheme], int(q), int(base_seed), int(worker),
                                       int(start), int(count), out.ctypes.data_as(C.POINTER(C.c_int32)), None))
        return out

    # -- row-sharded (multi-GPU) primitives -------------------------------------
    def set_ranges(self, lo, length) -> None:
        """Explicit per-worker support ranges (sampling scheme "ranges")."""
        lo = np.ascontiguousarray(lo, dtype=np.int64)
        ln = np.ascontiguousarray(length, dtype=np.int64)
        N.check(self._lib.kz_sampler_set_ranges(self.handle, len(lo), lo.ctypes.data_as(C.POINTER(C.c_int64)),
                                                ln.ctypes.data_as(C.POINTER(C.c_int64)), None))

    def error_sq(self) -> float:
        """||x - x_ref||^2 of the resident iterate."""
        out = C.c_double()
        N.check(self._lib.kz_error_sq(self.handle, C.byref(out), None))
        return out.value

    def average_from(self, S_ptr: int, Q: int) -> float:
        """x = S / Q from a reduced worker sum (device pointer); returns ||x - x_ref||^2."""
        out = C.c_double()
        N.check(self._lib.kz_average_from(self.handle, C.c_void_p(S_ptr), int(Q), C.byref(out), None))
        return out.value

    def local_step(self, cfg: "SolverConfig", *, k: int, worker_offset: int, partial_ptr: int,
                   alphas=None) -> dict:
        """One iteration of this shard's workers from the resident x; writes the
        un-normalised worker sum S = sum_t v_t to `partial_ptr` (device)."""
        variant = cfg.variant
        q = 1 if variant in ("rk", "ck") else cfg.q
        key = (cfg, int(worker_offset), int(partial_ptr), None if alphas is None else tuple(np.asarray(alphas).ravel()))
        cached = getattr(self, "_step_cache", None)
        if cached is not None and cached[0] == key:  # same step shape: only the iteration index moves
            _, p, al, r = cached
            p.k_start = int(k)
            N.check(self._lib.kz_solve(self.handle, C.byref(p), C.byref(r), None, None))
            return {"kernel_ms": 0.0, "loop_ms": 0.0, "rows": int(r.rows_projected),
                    "kernel": N.KERNEL_NAMES.get(int(r.kernel_used), "?"), "launches": int(r.kernel_launches)}
        al = N.f64(np.ones(q) if alphas is None else alphas)
        p = N.Params()
        p.variant = N.VARIANT_IDS[variant]
        p.scheme = N.SCHEME_IDS["ranges"]
        p.q = q
        p.block_size = cfg.block_size if variant == "rkab" else 1
        p.alphas_host = N.ptr(al)
        p.base_seed = int(cfg.base_seed)
        p.epsilon = float(cfg.epsilon)
        p.max_iterations = int(cfg.max_iterations)
        p.budget = 1
        p.kernel = N.KERNELS[cfg.kernel]
        p.threads, p.ctas = int(cfg.threads), int(cfg.ctas)
        p.worker_offset, p.k_start, p.keep_x = int(worker_offset), int(k), 1
        p.partial_dev = C.c_void_p(partial_ptr)
        r = N.Result()
        N.check(self._lib.kz_solve(self.handle, C.byref(p), C.byref(r), None, None))
        self._step_cache = (key, p, al, r)
        return {"kernel_ms": float(r.kernel_ms), "loop_ms": float(r.loop_ms), "rows": int(r.rows_projected),
                "kernel": N.KERNEL_NAMES.get(int(r.kernel_used), "?"), "launches": int(r.kernel_launches)}

    def solve_sharded(self, cfg: "SolverConfig", *, worker_offset: int, comm=None, budget: int | None = None,
                      alphas=None, fused: bool = True, loop: bool = False) -> dict:
        """The whole row-sharded _drive loop of this shard natively (kz_solve_sharded): per outer
        iteration the local step, an in-place all-reduce of the worker sum over ``comm`` (a
        :class:`ShardComm`; None = one rank) and x = S / (q * world) with the stop rule on the
        device.  Worker ranges come from :meth:`set_ranges`."""
        variant = cfg.variant
        if variant not in ("rka", "rkab"):
            raise ValueError(f"row-sharded solves run rka or rkab, not {variant!r}")
        al = N.f64(np.ones(cfg.q) if alphas is None else alphas)
        p = N.Params()
        p.variant = N.VARIANT_IDS[variant]
        p.scheme = N.SCHEME_IDS["ranges"]
        p.q = cfg.q
        p.block_size = cfg.block_size if variant == "rkab" else 1
        p.alphas_host = N.ptr(al)
        p.base_seed = int(cfg.base_seed)
        p.epsilon = float(cfg.epsilon)
        p.max_iterations = int(cfg.max_iterations)
        p.budget = 0 if budget is None else int(budget)
        p.kernel = N.KERNELS[cfg.kernel]
        p.threads, p.ctas = int(cfg.threads), int(cfg.ctas)
        p.worker_offset = int(worker_offset)
        p.flags = (0 if fused else 1) | (4 if loop else 0)  # KZ_FLAG_NO_FUSED_EXCHANGE, KZ_FLAG_SHARDED_LOOP
        r = N.Result()
        x = np.empty(self.n, dtype=np.float64)
        N.check(self._lib.kz_solve_sharded(self.handle, None if comm is None else comm.handle, C.byref(p),
                                           C.byref(r), N.ptr(x), None))
        return {"iterations": int(r.iterations), "converged": bool(r.converged),
                "final_error_sq": float(r.final_error_sq), "error_evals": int(r.error_evals), "x": x,
                "rows": int(r.rows_projected), "loop_ms": float(r.loop_ms), "kernel_ms": float(r.kernel_ms),
                "kernel": N.KERNEL_NAMES.get(int(r.kernel_used), "?"), "launches": int(r.kernel_launches),
                "ctas": int(r.ctas), "threads": int(r.threads),
                "plan": {"ep": int(r.plan_ep), "rows": int(r.plan_rows), "cluster": int(r.plan_cluster),
                         "stages": int(r.plan_stages), "waves": int(r.plan_waves)}}

    def set_x(self, x=None) -> None:
        """Overwrite the resident iterate (None = zeros)."""
        xv = None if x is None else N.f64(x)
        N.check(self._lib.kz_set_x(self.handle, N.ptr(xv) if xv is not None else None, None))

    def x_host(self) -> np.ndarray:
        out = np.empty(self.n)
        N.check(self._lib.kz_solution_host(self.handle, N.ptr(out), None))
        return out

    def norms(self, x) -> tuple[float, float]:
        """(||A x - b||, ||x - x_ref||) on the device."""
        xv = N.f64(x)
        res, err = C.c_double(), C.c_double()
        N.check(self._lib.kz_norms(self.handle, N.ptr(xv), C.byref(res), C.byref(err), None))
        return res.value, err.value

    def cgls(self, b=None, tol: float = 1e-10, max_it: int | None = None) -> np.ndarray:
        """x_LS = argmin ||A x - b|| on the device (cgls.py:42-75 `cgls_solve`); b defaults to the
        system's right-hand side.  Raises ConvergenceError (best_x attached) like the reference."""
        bv = None if b is None else N.f64(b)
        if bv is not None and bv.shape != (self.m,):
            raise DimensionMismatchError(f"b has shape {bv.shape}, expected ({self.m},)")
        x = np.empty(self.n)
        its = C.c_int64()
        rc = self._lib.kz_cgls(self.handle, N.ptr(bv) if bv is not None else None, C.c_double(float(tol)),
                               C.c_int64(int(max_it) if max_it is not None else 0), N.ptr(x), C.byref(its), None)
        if rc == N.KZ_ENOCONV:
            from .errors import ConvergenceError

            raise ConvergenceError(self._lib.kz_last_error().decode(errors="replace"), best_x=x)
        N.check(rc)
        self.cgls_iterations = int(its.value)
        return x

    def spectral(self, row_lo: int = 0, row_hi: int | None = None, tol: float = 1e-6, max_it: int = 5000):
        """(lambda_max, lambda_min) of A_blk^T A_blk for rows [row_lo, row_hi] on the device
        (spectral.py:66-121; start vectors Prng(0x5EED, 0/1) normalised on the host)."""
        from .errors import SpectralConvergenceError
        from .spectral import START_SEED
        from .sysgen import Prng

        row_hi = self.m - 1 if row_hi is None else row_hi
        v0 = Prng(START_SEED, 0).standard_normal(self.n)
        v0 /= np.linalg.norm(v0)
        v1 = Prng(START_SEED, 1).standard_normal(self.n)
        v1 /= np.linalg.norm(v1)
        out = np.empty(2)
        rc = self._lib.kz_spectral(self.handle, C.c_int64(row_lo), C.c_int64(row_hi), N.ptr(v0), N.ptr(v1),
                                   C.c_double(tol), C.c_int64(max_it), N.ptr(out), None)
        if rc == N.KZ_ESPECTRAL:
            msg = self._lib.kz_last_error().decode(errors="replace")
            raise SpectralConvergenceError(msg.split(":")[0], msg)
        N.check(rc)
        return float(out[0]), float(out[1])

    def _drop_views(self) -> None:
        for v in self.__dict__.pop("_lane_views", []):
            v.close()

    def _refresh_views(self) -> None:
        """Re-attach the cached lane views after this system's contents changed (no allocation)."""
        for v in self.__dict__.get("_lane_views", []):
            rc = self._lib.kz_system_view_refresh(v.handle)
            if rc not in (N.KZ_OK, N.KZ_EDEGENERATE):  # a zero row surfaces at solve time, as in the reference
                N.check(rc)
            v._xref_set = self._xref_set  # views alias the base's x_ref: its state, not the one at creation

    def view(self) -> "DeviceSystem":
        """A view for concurrent solves (kz_system_view): it shares this system's matrix, b,
        x_ref, row norms and packed records, and owns its iterate, samplers and CUDA stream.
        Close views before this system; do not re-upload this system while views exist."""
        h = C.c_void_p()
        N.check(self._lib.kz_system_view(self.handle, C.byref(h)))
        v = DeviceSystem.__new__(DeviceSystem)
        v._lib, v.m, v.n, v.device = self._lib, self.m, self.n, self.device
        v.host, v.handle, v._xref_set, v._base = self.host, h, self._xref_set, self
        return v

    def close(self) -> None:
        self._drop_views()  # views first: they alias this system's buffers
        if getattr(self, "handle", None):
            self._lib.kz_system_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# Device allocations for host-array calls are recycled by shape (a caching
# allocator): every call still uploads A, b, x_ref and recomputes the row norms
# and sampler, like the reference's per-call row_norm_cache (solvers.py:299).
_POOL: dict[tuple[int, int, int], list[DeviceSystem]] = {}
# the pool keeps at most one system per shape and this many bytes of matrices in total (the B200's
# 180 GB hold a c3-size 25.6 GB system with room to spare); release_pool() frees them
_POOL_MAX_BYTES = 64 << 30


def _pool_bytes() -> int:
    return sum(d.m * d.n * 8 for lst in _POOL.values() for d in lst)


def _pool_acquire(system: LinearSystem, device: int) -> DeviceSystem:
    A = system.A
    if getattr(A, "ndim", 0) != 2:
        raise DimensionMismatchError(f"expected a 2-D matrix, got ndim={getattr(A, 'ndim', None)}")
    key = (A.shape[0], A.shape[1], device)
    free = _POOL.get(key)
    if free:
        ds = free.pop()
        ds.host = system
        xr = system.x_star if system.x_star is not None else system.x_ls
        ds.upload(system.A, system.b, xr)
        return ds
    return DeviceSystem(system, device=device)


def _pool_release(ds: DeviceSystem) -> None:
    ds.host = None
    if not _POOL.get((ds.m, ds.n, ds.device)) and _pool_bytes() + ds.m * ds.n * 8 <= _POOL_MAX_BYTES:
        _POOL.setdefault((ds.m, ds.n, ds.device), []).append(ds)
    else:
        ds.close()


def release_pool() -> None:
    """Free the cached device allocations of host-array calls."""
    for lst in _POOL.values():
        for ds in lst:
            ds.close()
    _POOL.clear()


def resolve_alphas(system, cfg: SolverConfig, q: int | None = None) -> np.ndarray:
    """Per-worker weights (solvers.py:148-159).  The optimal_* policies run their spectral
    estimates (spectral.py:66-156) on the device (kz_spectral): on the resident system, or
    on a temporary upload of a host LinearSystem."""
    q = cfg.q if q is None else q
    if cfg.alpha_policy == "unit":
        return np.ones(q)
    if cfg.alpha_policy == "fixed":
        return np.full(q, float(cfg.alpha))
    from .spectral import optimal_alpha, partial_alphas, spectral_stats  # setup, off the hot path

    target = system if isinstance(system, DeviceSystem) else system.A
    if cfg.alpha_policy == "optimal_full":
        return np.full(q, optimal_alpha(spectral_stats(target), q))
    return partial_alphas(target, q)


def _uniform_alpha(alphas: np.ndarray) -> float:
    return float(alphas[0]) if np.all(alphas == alphas[0]) else float("nan")


def _solve(system, cfg: SolverConfig, variant: str, *, x_ref=None, budget=None, trace_step=None, capture=None,
           lead_row: bool = False, checkpoint_every: int | None = None, threads_combine: bool = False) -> RunReport:
    cfg.validate()
    q = 1 if variant in ("rk", "ck") else cfg.q
    steps = cfg.block_size + (1 if lead_row else 0) if variant == "rkab" else 1
    if budget is not None and budget < 1:
        raise ValueError(f"fixed iteration budget must be >= 1, got {budget}")
    if budget is None and trace_step is not None and trace_step < 1:
        raise ValueError(f"trace_step must be >= 1, got {trace_step}")

    own = not isinstance(system, DeviceSystem)
    ds = _pool_acquire(system, cfg.device) if own else system
    try:
        alphas = N.f64(resolve_alphas(ds, cfg, q))  # optimal_* policies: spectral estimates on the device
        if x_ref is not None:
            ds.set_x_ref(x_ref)
        elif budget is None and not ds._xref_set:
            host = ds.host if not own else system
            if host is None:
                raise ValueError("system carries no reference solution")
            ds.set_x_ref(host.x_ref())
        p = N.Params()
        p.variant = N.VARIANT_IDS[variant]
        p.scheme = N.SCHEME_IDS[cfg.sampling_scheme]
        p.q = q
        p.block_size = steps
        p.alphas_host = N.ptr(alphas)
        p.base_seed = int(cfg.base_seed)
        p.epsilon = float(cfg.epsilon)
        p.max_iterations = int(cfg.max_iterations)
        p.budget = int(budget) if budget is not None else 0
        limit = budget if budget is not None else cfg.max_iterations
        trace_buf = None
        if budget is None and trace_step is not None:
            p.trace_step = int(trace_step)
            trace_buf = np.empty((cfg.max_iterations // trace_step + 2, 3))
            p.trace_host = N.ptr(trace_buf)
        every = checkpoint_every if checkpoint_every else (1 if capture is not None else 0)
        ck_buf = None
        if every:
            # start with a modest buffer; a stop-mode run that outgrows it is
            # replayed below with an exact one (runs are deterministic)
            cap = min(limit // every, max(1, _CAPTURE_FIRST_BYTES // (8 * ds.n)))
            ck_buf = np.empty((max(cap, 1), ds.n))
            p.ckpt_every, p.ckpt_capacity, p.ckpt_host = every, cap, N.ptr(ck_buf)
        p.kernel = N.KERNELS[cfg.kernel]
        p.threads = int(cfg.threads)
        p.ctas = int(cfg.ctas)
        p.flags = (2 if cfg.short_launches else 0) | (8 if threads_combine else 0)  # KZ_FLAG_SHORT_LAUNCHES, _THREADS_COMBINE
        p.want_residual = 1
        r = N.Result()
        x = np.empty(ds.n)
        N.check(N.load_library().kz_solve(ds.handle, C.byref(p), C.byref(r), N.ptr(x), None))
        if every and r.n_ckpt < r.iterations // every:
            need = r.iterations // every
            if need * ds.n * 8 > _CAPTURE_LIMIT_BYTES:
                raise ValueError(f"capture of {need} iterates of length {ds.n} exceeds "
                                 f"{_CAPTURE_LIMIT_BYTES >> 30} GiB; pass checkpoint_every")
            ck_buf = np.empty((need, ds.n))
            p2 = N.Params.from_buffer_copy(p)
            p2.budget, p2.trace_step = int(r.iterations), 0
            p2.ckpt_capacity, p2.ckpt_host = need, N.ptr(ck_buf)
            r2 = N.Result()
            N.check(N.load_library().kz_solve(ds.handle, C.byref(p2), C.byref(r2), None, None))
            r.n_ckpt = r2.n_ckpt
    finally:
        if own:
            _pool_release(ds)

    if capture is not None and ck_buf is not None:
        capture.extend(ck_buf[i].copy() for i in range(r.n_ckpt))
    trace = None
    if trace_buf is not None:
        trace = [TraceRecord(int(t[0]), float(t[1]), float(t[2])) for t in trace_buf[: r.n_trace]]
    stop_mode = budget is None and trace_step is None
    return RunReport(
        variant=variant,
        q=q,
        block_size=cfg.block_size if variant == "rkab" else 1,
        alpha_policy=cfg.alpha_policy,
        alpha=_uniform_alpha(alphas),
        seed=cfg.base_seed,
        iterations=int(r.iterations),
        converged=bool(r.converged),
        wall_time_s=float(r.loop_ms) / 1e3,
        final_error_sq=float(r.final_error_sq) if stop_mode else float("nan"),
        final_residual=float(r.final_residual) if stop_mode else float("nan"),
        error_evals=int(r.error_evals),
        x=x,
        trace=trace,
        gpu={
            "kernel": N.KERNEL_NAMES.get(int(r.kernel_used), "?"),
            "loop_ms": float(r.loop_ms),
            "kernel_ms": float(r.kernel_ms),
            "rows_projected": int(r.rows_projected),
            "launches": int(r.kernel_launches),
            "ctas": int(r.ctas),
            "threads": int(r.threads),
            "plan": {"ep": int(r.plan_ep), "rows": int(r.plan_rows), "cluster": int(r.plan_cluster),
                     "stages": int(r.plan_stages), "waves": int(r.plan_waves)},
            "checkpoint_every": every,
        },
    )


def solve_ck(system, cfg: SolverConfig, *, x_ref=None, budget=None, trace_step=None, capture=None,
             checkpoint_every=None) -> RunReport:
    """Cyclic Kaczmarz: rows in order i = k mod m (solvers.py:271-291)."""
    return _solve(system, cfg, "ck", x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture,
                  checkpoint_every=checkpoint_every)


def solve_rk(system, cfg: SolverConfig, *, x_ref=None, budget=None, trace_step=None, capture=None,
             checkpoint_every=None) -> RunReport:
    """Randomized Kaczmarz, worker stream 0 (solvers.py:294-310)."""
    return _solve(system, cfg, "rk", x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture,
                  checkpoint_every=checkpoint_every)


def solve_rka_seq(system, cfg: SolverConfig, *, x_ref=None, budget=None, trace_step=None, capture=None,
                  checkpoint_every=None) -> RunReport:
    """Averaged RK: q rows from one snapshot, ordered mean (solvers.py:313-334)."""
    return _solve(system, cfg, "rka", x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture,
                  checkpoint_every=checkpoint_every)


def solve_rkab_seq(system, cfg: SolverConfig, *, x_ref=None, budget=None, trace_step=None, capture=None,
                   lead_row: bool = False, checkpoint_every=None) -> RunReport:
    """Block-averaged RK: q private chains of block_size rows (solvers.py:337-371)."""
    return _solve(system, cfg, "rkab", x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture,
                  lead_row=lead_row, checkpoint_every=checkpoint_every)


def solve_rka_parallel(system, cfg: SolverConfig, *, x_ref=None, budget=None, capture=None,
                       checkpoint_every=None) -> RunReport:
    """The threaded engine's RKA (parallel.py:175-235): every worker projects against the
    iteration's snapshot and adds alpha (b_i - <a_i, x_prev>) / (q sq_i) a_i to the shared x;
    the increments are added in worker order (one of the reference's arrival orders)."""
    r = _solve(system, cfg, "rka", x_ref=x_ref, budget=budget, capture=capture, checkpoint_every=checkpoint_every,
               threads_combine=True)
    return dataclasses.replace(r, barrier_events=2 * (r.iterations + 1)) if budget is None else r


def solve_rkab_parallel(system, cfg: SolverConfig, *, x_ref=None, budget=None, capture=None,
                        checkpoint_every=None) -> RunReport:
    """The threaded engine's RKAB (parallel.py:238-304): block_size + 1 rows per worker (a lead
    row from the shared x, then the chain) and x += (v - x) / q in worker order."""
    r = _solve(system, cfg, "rkab", x_ref=x_ref, budget=budget, capture=capture, lead_row=True,
               checkpoint_every=checkpoint_every, threads_combine=True)
    return dataclasses.replace(r, barrier_events=2 * (r.iterations + 1)) if budget is None else r


def solve_rk_block_sequential(system, cfg: SolverConfig, *, x_ref=None, budget=None, capture=None,
                              checkpoint_every=None) -> RunReport:
    """RK with the work of each iteration split over q workers (parallel.py:307-368): one sampling
    stream, one row per iteration, partial inner products over column slices combined in a fixed
    order -- the iterate sequence of solve_rk (bitwise at q = 1 in the reference, <= 1e-12
    otherwise, test_parallel.py:7-24).  On the B200 every RK solve already splits each row over the
    CTA's threads (or 4 / 8 CTAs) with a fixed reduction order, so this is solve_rk after the
    reference's validation (q <= n)."""
    cfg.validate()
    n = system.n if isinstance(system, DeviceSystem) else system.A.shape[1]
    if cfg.q > n:
        raise ValueError(f"q={cfg.q} workers exceed n={n} columns")
    return solve_rk(system, cfg.replace(q=1), x_ref=x_ref, budget=budget, capture=capture,
                    checkpoint_every=checkpoint_every)


@dataclass(frozen=True)
class RowNormCache:
    """Squared row norms and their total (linalg.py:64-78), computed on the device."""

    sq_norms: np.ndarray
    frobenius_sq: float

    @property
    def m(self) -> int:
        return self.sq_norms.shape[0]


def row_norm_cache(a) -> RowNormCache:
    """linalg.py:80-88 on the device: np.einsum("ij,ij->i") order bit for bit (kz_row_norms),
    DegenerateRowError on a zero row; ``a`` is a host matrix or a DeviceSystem."""
    if isinstance(a, DeviceSystem):
        sq = a.row_norms()
    else:
        A = np.ascontiguousarray(a, dtype=np.float64)
        if A.ndim != 2:
            raise DimensionMismatchError(f"expected a 2-D matrix, got ndim={A.ndim}")
        with DeviceSystem(m=A.shape[0], n=A.shape[1]) as ds:
            ds.upload(A, np.zeros(A.shape[0]))
            sq = ds.row_norms()
    sq.flags.writeable = False
    return RowNormCache(sq_norms=sq, frobenius_sq=float(sq.sum()))


def _run_cgls(system, cfg, x_ref):
    """harness._run_cgls (harness.py:72-95): CGLS on the device (kz_cgls)."""
    import time

    own = not isinstance(system, DeviceSystem)
    ds = _pool_acquire(system, cfg.device) if own else system
    try:
        t0 = time.perf_counter()
        x = ds.cgls(tol=1e-10)
        wall = time.perf_counter() - t0
        host = system if own else system.host
        if x_ref is None and host is not None and (host.x_star is not None or host.x_ls is not None):
            x_ref = host.x_ref()
        if x_ref is not None:
            ds.set_x_ref(x_ref)
        res, err = ds.norms(x)
    finally:
        if own:
            _pool_release(ds)
    return RunReport(variant="cgls", q=1, block_size=1, alpha_policy=cfg.alpha_policy, alpha=float("nan"),
                     seed=cfg.base_seed, iterations=-1, converged=True, wall_time_s=wall,
                     final_error_sq=err * err if x_ref is not None else float("nan"), final_residual=res, x=x)


def _seed_batchable(system, cfgs, budget, trace_step) -> bool:
    """RK solves that differ only in the seed, on rows short enough for the warp kernel."""
    c0 = cfgs[0]
    n = system.n if isinstance(system, DeviceSystem) else getattr(system.A, "shape", (0, 0))[1]
    return (trace_step is None and len(cfgs) > 1 and c0.variant == "rk" and c0.kernel in ("auto", "warp")
            and n <= 128 and all(c.replace(base_seed=c0.base_seed) == c0 for c in cfgs))


def solve_seeds(system, cfg: SolverConfig, seeds, *, budget=None) -> list[RunReport]:
    """The seeds of one RK configuration side by side in one launch per chunk (kz_solve_seeds):
    one warp per seed on short rows.  Reports in seed order, bit-identical to solving each
    seed alone on the warp kernel."""
    cfg.validate()
    seeds = [int(x) for x in seeds]
    own = not isinstance(system, DeviceSystem)
    ds = _pool_acquire(system, cfg.device) if own else system
    try:
        alphas = N.f64(resolve_alphas(ds, cfg, 1))
        if budget is None and not ds._xref_set:
            host = ds.host if not own else system
            if host is None:
                raise ValueError("system carries no reference solution")
            ds.set_x_ref(host.x_ref())
        p = N.Params()
        p.variant = N.VARIANT_IDS["rk"]
        p.scheme = N.SCHEME_IDS["full_access"]
        p.q = 1
        p.block_size = 1
        p.alphas_host = N.ptr(alphas)
        p.epsilon = float(cfg.epsilon)
        p.max_iterations = int(cfg.max_iterations)
        p.budget = 0 if budget is None else int(budget)
        S = len(seeds)
        res = (N.Result * S)()
        sv = (C.c_uint64 * S)(*seeds)
        X = np.empty((S, ds.n))
        N.check(ds._lib.kz_solve_seeds(ds.handle, C.byref(p), sv, S, res, N.ptr(X), None))
        out = []
        for i, sd in enumerate(seeds):
            r = res[i]
            resid = ds.norms(X[i])[0] if budget is None else float("nan")  # ||A x - b||, solvers.py:246
            out.append(RunReport(variant="rk", q=1, block_size=1, alpha_policy=cfg.alpha_policy,
                                 alpha=float(alphas[0]), seed=sd, iterations=int(r.iterations),
                                 converged=bool(r.converged), wall_time_s=float(r.loop_ms) / 1e3,
                                 final_error_sq=float(r.final_error_sq), final_residual=float(resid),
                                 error_evals=int(r.error_evals), x=X[i].copy(),
                                 gpu={"kernel": "warp", "ctas": int(r.ctas), "threads": int(r.threads),
                                      "loop_ms": float(r.loop_ms), "kernel_ms": float(r.kernel_ms),
                                      "rows_projected": int(r.rows_projected),
                                      "launches": int(r.kernel_launches), "seed_batch": S}))
        return out
    finally:
        if own:
            _pool_release(ds)


DEFAULT_LANES = 10  # measured best for c1 (7 co-resident 16-CTA clusters; chunk boundaries interleave the rest)


def solve_concurrent(system, cfgs, *, budget=None, lanes: int | None = None, x_ref=None,
                     trace_step=None) -> list[RunReport]:
    """Independent solves of one resident system side by side (e.g. the per-seed solves of
    harness.measure_iterations, harness.py:127-149): each of `lanes` host threads drives its
    own system view (kz_system_view: shared matrix, own iterate / samplers / stream), so the
    latency-bound solves of a small system share the GPU's SMs instead of queueing.  Reports
    come back in the order of `cfgs` and are bit-identical to solving them one by one."""
    from concurrent.futures import ThreadPoolExecutor

    cfgs = list(cfgs)
    if not cfgs:
        return []
    if _seed_batchable(system, cfgs, budget, trace_step):  # short-row RK: all seeds in one launch
        return solve_seeds(system, cfgs[0], [c.base_seed for c in cfgs], budget=budget)
    device = cfgs[0].device
    if isinstance(system, DeviceSystem):
        ds, own = system, False
    else:  # host arrays: uploaded once for all the solves (recycled allocation)
        ds, own = _pool_acquire(system, device), True
    n_lanes = max(1, min(lanes or DEFAULT_LANES, len(cfgs)))
    try:
        # views persist on the system (allocations and streams are made once, not per call:
        # a cudaFree inside a batch would synchronise the device under the other lanes)
        if x_ref is not None:  # one reference for all the solves, set on the system the views alias
            ds.set_x_ref(x_ref)
        cache = ds.__dict__.setdefault("_lane_views", [])
        while len(cache) < n_lanes:
            cache.append(ds.view())
        views = cache[:n_lanes]
        out: list[RunReport | None] = [None] * len(cfgs)

        def lane(i):
            for j in range(i, len(cfgs), n_lanes):
                c = cfgs[j].replace(short_launches=True) if n_lanes > 1 else cfgs[j]
                out[j] = run_solver(views[i], c, budget=budget, trace_step=trace_step)

        with ThreadPoolExecutor(n_lanes) as pool:
            for f in [pool.submit(lane, i) for i in range(n_lanes)]:
                f.result()
        return out  # type: ignore[return-value]
    finally:
        if own:
            _pool_release(ds)


def run_solver(system, cfg: SolverConfig, *, x_ref=None, budget=None, trace_step=None, capture=None,
               checkpoint_every=None) -> RunReport:
    """Dispatch on cfg.variant / cfg.engine (harness.py:98-114)."""
    cfg.validate()
    if cfg.variant == "cgls":
        if budget is not None or trace_step is not None:
            raise ValueError("cgls supports neither fixed-budget replay nor tracing")
        return _run_cgls(system, cfg, x_ref)
    if cfg.variant == "ck":
        return solve_ck(system, cfg, x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture,
                        checkpoint_every=checkpoint_every)
    if cfg.engine == "threads" and trace_step is not None:
        raise ValueError("tracing is supported by the sequential engine only")
    kw = dict(x_ref=x_ref, budget=budget, trace_step=trace_step, capture=capture, checkpoint_every=checkpoint_every)
    if cfg.variant == "rk":
        return solve_rk(system, cfg, **kw)
    if cfg.engine == "threads":
        del kw["trace_step"]
        return (solve_rka_parallel if cfg.variant == "rka" else solve_rkab_parallel)(system, cfg, **kw)
    if cfg.variant == "rka":
        return solve_rka_seq(system, cfg, **kw)
    return solve_rkab_seq(system, cfg, **kw)
