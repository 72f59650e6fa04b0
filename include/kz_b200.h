/*
 * kz_b200.h -- C-ABI of the B200-native RK / RKA / RKAB iteration loop.
 *
 * This is the drop-in boundary between the reference's Python entry points
 * (kaczbench, /root/reference/pkg/src/kaczbench) and the sm_100a kernels.
 * A ctypes binding (paper_2401_17474_b200/_native.py, or the stub in
 * INTEGRATION.md) calls these functions; no torch or C++ types cross it.
 *
 * Conventions
 *   - Every function returns an int status (KZ_OK = 0).  On failure a
 *     thread-local message is available from kz_last_error().  Status codes
 *     map onto the reference's exception taxonomy (errors.py:4-58).
 *   - Pointers suffixed _host are host memory (pageable or pinned); the
 *     library copies them.  Pointers suffixed _dev are device memory owned
 *     by the caller.  `stream` is a cudaStream_t (NULL = legacy default).
 *   - All calls are synchronous with respect to the host on return unless
 *     stated otherwise ("at most one solve in flight per process",
 *     SPEC.md:593; the reference solvers are blocking calls).
 *   - Inputs are never modified (solvers.py:194: the solver owns x).
 */
#ifndef KZ_B200_H
#define KZ_B200_H

#include <stdint.h>

#if defined(__GNUC__)
#define KZ_API __attribute__((visibility("default")))
#else
#define KZ_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

enum kz_status {
    KZ_OK = 0,
    KZ_EINVAL = 1,      /* ValueError / DimensionMismatchError (solvers.py:85-101, linalg.py:30-47) */
    KZ_EDEGENERATE = 2, /* DegenerateRowError (linalg.py:84-86)                                      */
    KZ_EEMPTYRANGE = 3, /* EmptyRangeError (sampling.py:106-107, 213-218)                            */
    KZ_ENOMEM = 4,      /* device allocation failed                                                  */
    KZ_ECUDA = 5,       /* CUDA runtime / launch error                                               */
    KZ_ENODEV = 6,      /* no CUDA device                                                            */
    KZ_ENOCONV = 7,     /* ConvergenceError (cgls.py:71-75): iterate returned, tolerance not met     */
    KZ_ESPECTRAL = 8,   /* SpectralConvergenceError (spectral.py:84-112)                             */
    KZ_EFORMAT = 9,     /* SystemFormatError (sysgen.py:226-246): bad magic, dimensions, truncation  */
    KZ_EVERSION = 10    /* UnsupportedVersionError (sysgen.py:240-244)                               */
};

enum kz_variant { KZ_RK = 0, KZ_RKA = 1, KZ_RKAB = 2, KZ_CK = 3 };          /* solvers.py:55 VARIANTS        */
enum kz_scheme { KZ_FULL_ACCESS = 0, KZ_DISTRIBUTED = 1 };        /* solvers.py:57 SAMPLING_SCHEMES */
enum kz_kernel {                                                  /* engine selection (auto = 0)    */
    KZ_KERNEL_AUTO = 0,
    KZ_KERNEL_CHAIN = 1,        /* worker-per-CTA persistent kernel (RK, RKAB)                   */
    KZ_KERNEL_SYNC_CLUSTER = 2, /* column-sliced kernel, one thread-block cluster, DSMEM reduce  */
    KZ_KERNEL_SYNC_GRID = 3,    /* column-sliced kernel, whole grid, global-memory reduce        */
    KZ_KERNEL_WARP = 4,         /* one warp, register-resident x: RK / CK on rows of <= 256 columns */
    KZ_KERNEL_RKA = 5           /* column-sliced TMA kernel (rka_kernel): the plan SYNC_CLUSTER tries
                                   first; as a selector it has no fallback, and kz_result.kernel_used
                                   reports it whenever it ran                                     */
};

typedef struct kz_system kz_system;

/* ---- library ---------------------------------------------------------- */
KZ_API const char* kz_last_error(void);
KZ_API int32_t kz_version(void);
/* Kernels this library has launched in this process (all devices). */
KZ_API int64_t kz_launch_count(void);
KZ_API int32_t kz_device_count(int32_t* count);

/* ---- system residency ----------------------------------------------------
 * Replaces the numpy views of LinearSystem (sysgen.py:84-115) that every
 * solver reads (solvers.py:193).  A is stored row-major with a padded pitch
 * (kz_system_pitch) so every row starts on a 128-byte boundary.
 * x_ref is the stopping reference (LinearSystem.x_ref, sysgen.py:110-115). */
KZ_API int32_t kz_system_create(int32_t device, int64_t m, int64_t n, kz_system** out);
KZ_API int32_t kz_system_destroy(kz_system* sys);
KZ_API int64_t kz_system_pitch(const kz_system* sys);
/* Host -> device copies.  lda >= n.  b_host: m values; xref_host: n values or NULL. */
KZ_API int32_t kz_system_upload(kz_system* sys, const double* A_host, int64_t lda, const double* b_host,
                         const double* xref_host, void* stream);
/* Device -> device copies from caller-owned device arrays (lda >= n). */
KZ_API int32_t kz_system_upload_device(kz_system* sys, const double* A_dev, int64_t lda, const double* b_dev,
                                const double* xref_dev, void* stream);
/* Raw device pointers of the resident arrays (pitched A, b, x_ref), for
 * in-place generation of large systems. */
KZ_API int32_t kz_system_device_ptrs(kz_system* sys, double** A_dev, double** b_dev, double** xref_dev);
/* Replace the stopping reference x_ref (n values, host). */
KZ_API int32_t kz_system_set_xref(kz_system* sys, const double* xref_host, void* stream);
/* BASELINE config 3 generator: fills A (leading m x n of the counter-keyed
 * mother system), x_ref = x* and b = A x* on the device.  Entries depend only
 * on (seed, i, j), so any m' x n' system is an exact leading crop. */
KZ_API int32_t kz_generate_counter(kz_system* sys, uint64_t seed, double mu_lo, double mu_hi, double sigma_lo,
                                   double sigma_hi, void* stream);
/* Rows [row0, row0 + m) of the same counter-keyed system into this system (a
 * GPU's row shard is bit-identical to those rows of the full matrix). */
KZ_API int32_t kz_generate_counter_rows(kz_system* sys, uint64_t seed, int64_t row0, double mu_lo, double mu_hi,
                                        double sg_lo, double sg_hi, void* stream);
/* Copy the leading m2 x n2 block of A (row-major, ld n2), b[:m2] and x_ref[:n2] to the host (any may be NULL). */
KZ_API int32_t kz_system_download(kz_system* sys, int64_t m2, int64_t n2, double* A_host, double* b_host,
                                  double* xref_host, void* stream);
/* Invalidate cached row norms / samplers after A was written in place. */
KZ_API int32_t kz_system_touch(kz_system* sys);
/* A view of a resident system for concurrent solves (e.g. the seeds of harness.bench's
 * measure_iterations, harness.py:127-149, run side by side instead of one after another):
 * it aliases the base system's A, b, x_ref, row norms and packed records and owns its
 * iterate, samplers, scratch and a CUDA stream (used when a call passes stream = NULL).
 * Destroy views with kz_system_destroy before the base; upload / generate / touch are
 * refused on a view. */
KZ_API int32_t kz_system_view(kz_system* base, kz_system** out);
/* Re-attach a view after its base system was re-uploaded / regenerated (no allocation):
 * the base's norms and packed records are rebuilt, the view's samplers dropped. */
KZ_API int32_t kz_system_view_refresh(kz_system* view);

/* ---- row norms: row_norm_cache (linalg.py:80-88) ------------------------
 * Bit-exact with np.einsum("ij,ij->i") (SSE2 two-lane order).  Cached on
 * the system.  Returns KZ_EDEGENERATE with *bad_row = first zero row.
 * sq_host (m values) may be NULL. */
KZ_API int32_t kz_row_norms(kz_system* sys, double* sq_host, int64_t* bad_row, void* stream);
/* Host-computed squared row norms (m values) replace the device computation -- the fallback of
 * SURVEY Appendix A when the host numpy's einsum summation order differs from the one the device
 * kernel restates (sysgen.einsum_order_matches); sampler and packed records are rebuilt from them. */
KZ_API int32_t kz_row_norms_upload(kz_system* sys, const double* sq_host, void* stream);

/* ---- sampler: make_sampler / worker_streams (sampling.py:101-111,
 * solvers.py:162-171) ------------------------------------------------------
 * Builds the inclusive CDF(s) for (scheme, q): one CDF over all rows
 * (full_access) or one per block partition_bounds(m, q, t) (distributed).
 * cdf_host (m values, concatenated per block) may be NULL. */
KZ_API int32_t kz_sampler_build(kz_system* sys, int32_t scheme, int64_t q, double* cdf_host, void* stream);
/* Row draws `start .. start+count-1` of worker `worker` for Prng(base_seed,
 * worker) (RowSampler.sample, sampling.py:89-94): bit-exact indices. */
KZ_API int32_t kz_dump_rows(kz_system* sys, int32_t scheme, int64_t q, uint64_t base_seed, int64_t worker,
                     int64_t start, int64_t count, int32_t* out_host, void* stream);

/* Explicit per-worker support ranges [lo_t, lo_t + len_t) (row shards: the
 * reference's distributed scheme restricted to this device's rows,
 * partition_bounds(m, Q, t) shifted by the shard offset).  Selected with
 * scheme = KZ_SCHEME_RANGES. */
#define KZ_SCHEME_RANGES 2
KZ_API int32_t kz_sampler_set_ranges(kz_system* sys, int64_t q, const int64_t* lo_host, const int64_t* len_host,
                                     void* stream);

/* ---- solve: solve_rk / solve_rka_seq / solve_rkab_seq via _drive
 * (solvers.py:182-263, 294-371) ---------------------------------------- */
typedef struct {
    int32_t variant;        /* kz_variant                                                     */
    int32_t scheme;         /* kz_scheme                                                      */
    int64_t q;              /* workers (SolverConfig.q)                                       */
    int64_t block_size;     /* RKAB chain length (SolverConfig.block_size)                    */
    const double* alphas_host; /* q row weights (resolve_alphas); NULL = unit                  */
    uint64_t base_seed;     /* SolverConfig.base_seed                                         */
    double epsilon;         /* stop when ||x - x_ref||^2 < epsilon                            */
    int64_t max_iterations; /* SolverConfig.max_iterations                                    */
    int64_t budget;         /* > 0: fixed-budget replay, stop rule disabled (_drive budget)   */
    int64_t trace_step;     /* > 0: trace mode, records at 0, s, 2s ... (_drive trace)         */
    double* trace_host;     /* (max_iterations/trace_step + 1) x 3: iteration, ||x-xref||, ||Ax-b|| */
    int64_t ckpt_every;     /* > 0: store x after every ckpt_every iterations (capture)        */
    int64_t ckpt_capacity;  /* rows of ckpt_host                                               */
    double* ckpt_host;      /* ckpt_capacity x n                                               */
    int32_t kernel;         /* kz_kernel (0 = auto)                                            */
    int32_t threads;        /* CTA size override (0 = auto)                                    */
    int32_t ctas;           /* CTA count override for sync kernels (0 = auto)                  */
    int32_t want_residual;  /* compute ||Ax - b|| at the end of a stop-mode run                */
    /* row-sharded (multi-GPU) operation, see kz_average_from / kz_sampler_set_ranges: */
    int64_t worker_offset;  /* stream id of local worker 0: worker t draws from Prng(seed, offset+t) */
    int64_t k_start;        /* index of the first iteration (row-draw offset k_start * block_size)   */
    int32_t keep_x;         /* start from the resident iterate instead of x0 = 0                     */
    int32_t flags;          /* KZ_FLAG_* bits (0 = none)                                             */
    double* partial_dev;    /* non-NULL: run ONE iteration and write the un-normalised worker sum   */
                            /* S = sum_t v_t (n values, device) instead of updating x                */
} kz_params;
/* kz_params.flags: kz_solve_sharded keeps the per-iteration NCCL all-reduce even when the
 * communicator's fused cross-rank exchange is connected. */
#define KZ_FLAG_NO_FUSED_EXCHANGE 1
/* kz_params.flags: stop-mode launches of at most 2048 outer iterations (instead of growing to
 * the index buffer's capacity) -- for solves running side by side on one GPU. */
#define KZ_FLAG_SHORT_LAUNCHES 2
/* kz_params.flags: kz_solve_sharded without a communicator (one rank) runs its per-iteration
 * sharded loop instead of delegating to kz_solve's chunked kernels (tests of the loop itself). */
#define KZ_FLAG_SHARDED_LOOP 4
/* kz_params.flags: the threaded engine's combine (engine="threads", parallel.py:175-304):
 * RKA adds alpha (b - <a_t, x>) / (q sq_t) a_t to x, RKAB adds (v_t - x) / q, in worker
 * order, instead of the sequential engine's average.  RKA / RKAB with q > 1 only; runs
 * on the chain kernel. */
#define KZ_FLAG_THREADS_COMBINE 8

typedef struct {
    int64_t iterations;     /* RunReport.iterations                                           */
    int32_t converged;      /* RunReport.converged                                            */
    int32_t kernel_used;    /* kz_kernel actually run                                         */
    double final_error_sq;  /* RunReport.final_error_sq (NaN outside stop mode)               */
    double final_residual;  /* RunReport.final_residual (NaN unless computed)                 */
    int64_t error_evals;    /* RunReport.error_evals                                          */
    int64_t n_ckpt;         /* checkpoints written                                            */
    int64_t n_trace;        /* trace records written                                          */
    int64_t rows_projected; /* row projections performed (iterations x q x block_size)        */
    double loop_ms;         /* device time of the iteration loop (CUDA events)                */
    double kernel_ms;       /* device time inside the solve kernels only                      */
    int64_t kernel_launches;/* kernels launched by this call                                  */
    int32_t ctas;           /* CTAs of the solve kernel                                       */
    int32_t threads;        /* threads per CTA of the solve kernel                            */
    int32_t plan_ep;        /* chain kernel: 16-byte column pairs per thread (EP); rka: pairs per lane */
    int32_t plan_rows;      /* chain kernel: rows per CTA reduction (R)                        */
    int32_t plan_cluster;   /* CTAs per thread-block cluster (chain: CTAs per worker)           */
    int32_t plan_stages;    /* shared-memory ring stages                                        */
    int32_t plan_waves;     /* chain kernel: launches per outer iteration (workers beyond the
                               co-resident CTAs run in waves; 1 = all workers at once)          */
    int32_t pad;
} kz_result;

/* Full solve with host output x_host (n values, may be NULL): the _drive protocol
 * (solvers.py:182-263) of solve_rk / solve_rka_seq / solve_rkab_seq / solve_ck
 * (solvers.py:271-371).  Any q: workers beyond the CTAs the GPU holds at once run
 * in waves per outer iteration (kz_result.plan_waves), bit-identical to one launch;
 * rows up to 81920 columns on the chain kernel (RK, CK, RKAB), any width for RKA.
 * Trace mode needs the workers co-resident (KZ_EINVAL otherwise). */
KZ_API int32_t kz_solve(kz_system* sys, const kz_params* params, kz_result* result, double* x_host, void* stream);
/* The seeds of one RK configuration (seeds[S]) solved side by side in one launch per chunk:
 * one warp per seed on short rows (n <= 256), each with its own iterate, row draws
 * (Prng(seed, worker_offset)), status and stop flag.  results[S]; x_host: S x n (may be NULL).
 * Stop or budget mode (no trace / checkpoints).  The BASELINE config-0 protocol's 10 seeds
 * (harness.py:127-149) in one go instead of ten latency-bound solves. */
KZ_API int32_t kz_solve_seeds(kz_system* sys, const kz_params* params, const uint64_t* seeds, int64_t S,
                              kz_result* results, double* x_host, void* stream);
/* Resident iterate: copy out (n values) / overwrite (NULL = zeros). */
KZ_API int32_t kz_solution_host(kz_system* sys, double* x_host, void* stream);
KZ_API int32_t kz_set_x(kz_system* sys, const double* x_host, void* stream);
/* Device pointer of the final iterate of the last kz_solve on this system (n values). */
KZ_API int32_t kz_solution_device(kz_system* sys, double** x_dev);

/* x = S / Q from a (reduced) worker sum S (device), then ||x - x_ref||^2 -> *err_host.
 * The closing half of one row-sharded iteration (distributed.py:296-301). */
KZ_API int32_t kz_average_from(kz_system* sys, const double* S_dev, int64_t Q, double* err_host, void* stream);
/* ||x - x_ref||^2 of the resident iterate (deterministic, identical on every rank). */
KZ_API int32_t kz_error_sq(kz_system* sys, double* err_host, void* stream);

/* ---- norms used by traces and reports (solvers.py:174-179, 246) ---------- */
/* ||A x - b||_2 and ||x - x_ref||_2 for a host x (n values). */
KZ_API int32_t kz_norms(kz_system* sys, const double* x_host, double* residual, double* error, void* stream);

/* CGLS on the resident matrix (replaces cgls.py:42-75 `cgls_solve`): x_out[n]
 * = argmin ||A x - b|| with the reference's stop rule ||A^T(Ax-b)|| <= tol ||A^T b||
 * and one restart.  b_host = NULL uses the system's b.  max_it <= 0 means
 * 10 n + 100.  KZ_ENOCONV when the budget runs out (x_out holds the best
 * iterate, like ConvergenceError.best_x). */
KZ_API int32_t kz_cgls(kz_system* sys, const double* b_host, double tol, int64_t max_it, double* x_out,
                       int64_t* iterations, void* stream);

/* Extreme eigenvalues of A_blk^T A_blk for the row block [row_lo, row_hi]
 * (replaces spectral.py:66-121 `spectral_stats`): out[0] = sigma_max^2 by power
 * iteration, out[1] = sigma_min^2 by inverse iteration with a matrix-free CG
 * inner solve; v0/v1 are the normalised start vectors (n each).  KZ_ESPECTRAL
 * maps to SpectralConvergenceError. */
/* Load a KZSYS v1 system file (sysgen.py:190-271) straight into device memory:
 * rows [row_lo, row_hi] (row_hi < 0: all; a GPU's shard), b of those rows and
 * x_ref (x_star if present, else x_ls).  Reports the file's full m, n, flags and
 * generator metadata (seed, mu_lo, mu_hi, sigma_lo, sigma_hi; seed -1 if none). */
KZ_API int32_t kz_system_load_file(int32_t device, const char* path, int64_t row_lo, int64_t row_hi,
                                   kz_system** out, int64_t* m_total, int64_t* n_out, uint32_t* flags_out,
                                   double* meta5);

KZ_API int32_t kz_spectral(kz_system* sys, int64_t row_lo, int64_t row_hi, const double* v0_host,
                           const double* v1_host, double tol, int64_t max_it, double* out, void* stream);

/* ---- row-sharded multi-GPU solve (replaces distributed.py:282-363
 * solve_rka_dist / solve_rkab_dist / run_distributed_solve and the
 * SimTransport.allreduce_sum of distributed.py:119-148) ----------------------
 * One process per GPU.  Rank 0 draws an id with kz_comm_unique_id, the caller
 * broadcasts its KZ_COMM_ID_BYTES bytes (e.g. torch.distributed), and every
 * rank creates its communicator (NCCL over NVLink / NVSwitch; libnccl.so.2 is
 * loaded at first use -- the process's own copy when one is loaded). */
typedef struct kz_comm kz_comm;
#define KZ_COMM_ID_BYTES 128
KZ_API int32_t kz_comm_unique_id(uint8_t* id_out);
KZ_API int32_t kz_comm_create(int32_t device, const uint8_t* id, int32_t world, int32_t rank, kz_comm** out);
KZ_API int32_t kz_comm_destroy(kz_comm* comm);
/* The fused cross-rank exchange (optional; kz_solve_sharded uses it for RKA when connected):
 * every rank sizes its exchange buffer for the shard pitch (kz_system_pitch) and exports its
 * CUDA IPC handle (KZ_COMM_HANDLE_BYTES bytes); the caller all-gathers the handles in rank
 * order and every rank connects.  The step kernel then writes its column sums straight into
 * every rank's buffer over NVLink and reads the world's sums from its own (no NCCL call, one
 * launch per chunk of iterations). */
#define KZ_COMM_HANDLE_BYTES 64
KZ_API int32_t kz_comm_exchange_handle(kz_comm* comm, int64_t ld, uint8_t* handle_out);
KZ_API int32_t kz_comm_exchange_connect(kz_comm* comm, const uint8_t* handles);
/* The whole _drive loop (solvers.py:182-263) of one rank's row shard, natively:
 * per outer iteration the local step writes the rank's worker sum S_g, S is
 * all-reduced in place over `comm` (NULL: a single rank), and x = S / (q *
 * world) with ||x - x_ref||^2 and the stop rule evaluated on the device.  No
 * host synchronisation per iteration: a device stop flag turns every launch
 * after convergence into a no-op and the host reads the per-iteration errors
 * once per chunk.  Every rank computes bit-identical x and errors, so all stop
 * together (distributed.py:233-235).  params: variant RKA or RKAB, scheme
 * KZ_SCHEME_RANGES (kz_sampler_set_ranges with the rank's worker blocks),
 * worker_offset = rank * q, stop or budget mode (no trace / checkpoints);
 * partial_dev is ignored.  result->rows_projected counts this rank's rows.
 * With comm = NULL (one rank, nothing to exchange) the solve is kz_solve on the shard's
 * worker ranges -- whole chunks of outer iterations per launch -- unless
 * KZ_FLAG_SHARDED_LOOP asks for the per-iteration loop. */
KZ_API int32_t kz_solve_sharded(kz_system* shard, kz_comm* comm, const kz_params* params, kz_result* result,
                                double* x_host, void* stream);

#ifdef __cplusplus
}
#endif
#endif
