"""B200-native RK / RKA / RKAB iteration loop (arXiv 2401.17474) behind the
reference kaczbench entry points.  See DESIGN.md for the architecture and
include/kz_b200.h for the C-ABI boundary."""

from .errors import (ConvergenceError, DegenerateRowError, DimensionMismatchError, EmptyRangeError,
                     SpectralConvergenceError, SystemFormatError, TransportProtocolError, UnsupportedVersionError)
from .distributed import run_distributed_solve
from .harness import (MeasureResult, Protocol, ReplayResult, bench, measure_iterations, plateau_error,
                      timed_replay, trace_run)
from .reports import REPORT_HEADER, TRACE_HEADER, RunReport, TraceRecord
from .solvers import (ALPHA_POLICIES, ENGINES, SAMPLING_SCHEMES, VARIANTS, DeviceSystem, RowNormCache, SolverConfig,
                      resolve_alphas, row_norm_cache, run_solver, solve_ck, solve_concurrent, solve_rk,
                      solve_rk_block_sequential, solve_rka_parallel, solve_rka_seq, solve_rkab_parallel, solve_rkab_seq,
                      solve_seeds)
from .spectral import SpectralStats, optimal_alpha, partial_alphas, spectral_stats
from .sysgen import (GeneratorConfig, LinearSystem, Prng, cgls_solve, crop, generate_mother, load_system,
                     make_inconsistent, partition_bounds, save_system, worker_rng)

__version__ = "0.1.0"
