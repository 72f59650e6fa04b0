"""ctypes binding of ``libkz_b200.so`` (the C-ABI declared in include/kz_b200.h).

The product path goes through this module only.  There is no CPU fallback:
if the library is missing or no CUDA device is visible, every entry point
raises :class:`NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DegenerateRowError, DimensionMismatchError, EmptyRangeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkz_b200.so")

KZ_OK, KZ_EINVAL, KZ_EDEGENERATE, KZ_EEMPTYRANGE, KZ_ENOMEM, KZ_ECUDA, KZ_ENODEV, KZ_ENOCONV, KZ_ESPECTRAL, \
    KZ_EFORMAT, KZ_EVERSION = range(11)
KERNELS = {"auto": 0, "chain": 1, "sync_cluster": 2, "sync_grid": 3, "warp": 4, "rka": 5}
KERNEL_NAMES = {v: k for k, v in KERNELS.items()}
VARIANT_IDS = {"rk": 0, "rka": 1, "rkab": 2, "ck": 3}
SCHEME_IDS = {"full_access": 0, "distributed": 1, "ranges": 2}

# Every symbol include/kz_b200.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "kz_last_error", "kz_version", "kz_launch_count", "kz_device_count",
    "kz_system_create", "kz_system_destroy", "kz_system_pitch", "kz_system_upload",
    "kz_system_upload_device", "kz_system_device_ptrs", "kz_system_set_xref", "kz_system_touch",
    "kz_generate_counter", "kz_system_download",
    "kz_row_norms", "kz_sampler_build", "kz_sampler_set_ranges", "kz_dump_rows", "kz_solve",
    "kz_average_from", "kz_error_sq", "kz_solution_host", "kz_set_x", "kz_solution_device", "kz_norms",
    "kz_cgls", "kz_spectral", "kz_system_load_file", "kz_generate_counter_rows",
    "kz_comm_unique_id", "kz_comm_create", "kz_comm_destroy", "kz_solve_sharded", "kz_system_view",
    "kz_system_view_refresh", "kz_comm_exchange_handle", "kz_comm_exchange_connect", "kz_row_norms_upload",
    "kz_solve_seeds",
)
COMM_HANDLE_BYTES = 64
COMM_ID_BYTES = 128


class NativeUnavailable(RuntimeError):
    """The CUDA library could not be loaded or no device is visible."""


class NativeError(RuntimeError):
    """A CUDA-side failure reported by the library."""


class Params(C.Structure):
    _fields_ = [
        ("variant", C.c_int32),
        ("scheme", C.c_int32),
        ("q", C.c_int64),
        ("block_size", C.c_int64),
        ("alphas_host", C.POINTER(C.c_double)),
        ("base_seed", C.c_uint64),
        ("epsilon", C.c_double),
        ("max_iterations", C.c_int64),
        ("budget", C.c_int64),
        ("trace_step", C.c_int64),
        ("trace_host", C.POINTER(C.c_double)),
        ("ckpt_every", C.c_int64),
        ("ckpt_capacity", C.c_int64),
        ("ckpt_host", C.POINTER(C.c_double)),
        ("kernel", C.c_int32),
        ("threads", C.c_int32),
        ("ctas", C.c_int32),
        ("want_residual", C.c_int32),
        ("worker_offset", C.c_int64),
        ("k_start", C.c_int64),
        ("keep_x", C.c_int32),
        ("flags", C.c_int32),
        ("partial_dev", C.c_void_p),
    ]


class Result(C.Structure):
    _fields_ = [
        ("iterations", C.c_int64),
        ("converged", C.c_int32),
        ("kernel_used", C.c_int32),
        ("final_error_sq", C.c_double),
        ("final_residual", C.c_double),
        ("error_evals", C.c_int64),
        ("n_ckpt", C.c_int64),
        ("n_trace", C.c_int64),
        ("rows_projected", C.c_int64),
        ("loop_ms", C.c_double),
        ("kernel_ms", C.c_double),
        ("kernel_launches", C.c_int64),
        ("ctas", C.c_int32),
        ("threads", C.c_int32),
        ("plan_ep", C.c_int32),
        ("plan_rows", C.c_int32),
        ("plan_cluster", C.c_int32),
        ("plan_stages", C.c_int32),
        ("plan_waves", C.c_int32),
        ("pad", C.c_int32),
    ]


_lib = None
_lock = threading.Lock()
_dp = C.POINTER(C.c_double)


def load_library():
    """Load (never build) the shared library and declare its signatures."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeUnavailable(
                f"{LIB_PATH} is missing; build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.kz_last_error.restype = C.c_char_p
        L.kz_version.restype = C.c_int32
        L.kz_launch_count.restype = C.c_int64
        L.kz_device_count.argtypes = [C.POINTER(C.c_int32)]
        L.kz_system_create.argtypes = [C.c_int32, C.c_int64, C.c_int64, C.POINTER(vp)]
        L.kz_system_destroy.argtypes = [vp]
        L.kz_system_pitch.argtypes = [vp]
        L.kz_system_pitch.restype = C.c_int64
        L.kz_system_upload.argtypes = [vp, _dp, C.c_int64, _dp, _dp, vp]
        L.kz_system_upload_device.argtypes = [vp, vp, C.c_int64, vp, vp, vp]
        L.kz_system_device_ptrs.argtypes = [vp, C.POINTER(vp), C.POINTER(vp), C.POINTER(vp)]
        L.kz_system_set_xref.argtypes = [vp, _dp, vp]
        L.kz_system_touch.argtypes = [vp]
        L.kz_generate_counter.argtypes = [vp, C.c_uint64, C.c_double, C.c_double, C.c_double, C.c_double, vp]
        L.kz_system_download.argtypes = [vp, C.c_int64, C.c_int64, _dp, _dp, _dp, vp]
        L.kz_row_norms.argtypes = [vp, _dp, C.POINTER(C.c_int64), vp]
        L.kz_sampler_build.argtypes = [vp, C.c_int32, C.c_int64, _dp, vp]
        L.kz_dump_rows.argtypes = [vp, C.c_int32, C.c_int64, C.c_uint64, C.c_int64, C.c_int64, C.c_int64,
                                   C.POINTER(C.c_int32), vp]
        L.kz_solve.argtypes = [vp, C.POINTER(Params), C.POINTER(Result), _dp, vp]
        L.kz_solution_device.argtypes = [vp, C.POINTER(vp)]
        L.kz_sampler_set_ranges.argtypes = [vp, C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_int64), vp]
        L.kz_average_from.argtypes = [vp, vp, C.c_int64, _dp, vp]
        L.kz_error_sq.argtypes = [vp, _dp, vp]
        L.kz_solution_host.argtypes = [vp, _dp, vp]
        L.kz_set_x.argtypes = [vp, _dp, vp]
        L.kz_norms.argtypes = [vp, _dp, _dp, _dp, vp]
        L.kz_system_view.argtypes = [vp, C.POINTER(vp)]
        L.kz_row_norms_upload.argtypes = [vp, _dp, vp]
        L.kz_solve_seeds.argtypes = [vp, C.POINTER(Params), C.POINTER(C.c_uint64), C.c_int64,
                                     C.POINTER(Result), _dp, vp]
        L.kz_system_view_refresh.argtypes = [vp]
        L.kz_comm_unique_id.argtypes = [C.c_char_p]
        L.kz_comm_create.argtypes = [C.c_int32, C.c_char_p, C.c_int32, C.c_int32, C.POINTER(vp)]
        L.kz_comm_destroy.argtypes = [vp]
        L.kz_comm_exchange_handle.argtypes = [vp, C.c_int64, C.c_char_p]
        L.kz_comm_exchange_connect.argtypes = [vp, C.c_char_p]
        L.kz_solve_sharded.argtypes = [vp, vp, C.POINTER(Params), C.POINTER(Result), _dp, vp]
        for name in EXPORTS:
            fn = getattr(L, name)
            if name not in ("kz_last_error", "kz_launch_count", "kz_system_pitch"):
                fn.restype = C.c_int32
        _lib = L
        return _lib


def launch_count() -> int:
    return int(load_library().kz_launch_count())


def device_count() -> int:
    L = load_library()
    c = C.c_int32(0)
    L.kz_device_count(C.byref(c))
    return int(c.value)


def check(rc: int, bad_row: int | None = None) -> None:
    """Map a kz_status onto the reference's exception taxonomy (errors.py)."""
    if rc == KZ_OK:
        return
    msg = load_library().kz_last_error().decode(errors="replace")
    if rc == KZ_EDEGENERATE:
        raise DegenerateRowError(int(bad_row) if bad_row is not None else _parse_row(msg))
    if rc == KZ_EEMPTYRANGE:
        raise EmptyRangeError(msg)
    if rc == KZ_EINVAL:
        if "dimension" in msg or "lda" in msg:
            raise DimensionMismatchError(msg)
        raise ValueError(msg)
    if rc == KZ_ENODEV:
        raise NativeUnavailable(msg)
    if rc in (KZ_EFORMAT, KZ_EVERSION):
        from .errors import SystemFormatError, UnsupportedVersionError

        off = _parse_offset(msg)
        raise (UnsupportedVersionError if rc == KZ_EVERSION else SystemFormatError)(msg.split(" (offset")[0], off)
    if rc == KZ_ENOMEM:
        raise MemoryError(msg)
    raise NativeError(msg)


def _parse_offset(msg: str) -> int:
    try:
        return int(msg.split("(offset ")[1].split(")")[0])
    except (IndexError, ValueError):
        return -1


def _parse_row(msg: str) -> int:
    try:
        return int(msg.split("row ")[1].split()[0])
    except (IndexError, ValueError):
        return -1


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def ptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)
