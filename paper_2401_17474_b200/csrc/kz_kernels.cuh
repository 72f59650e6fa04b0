// kz_kernels.cuh -- kernel argument blocks and launch declarations.
#pragma once

#include <cuda.h>

#include "kz_common.cuh"

namespace kz {

// Per-launch status written by the solve kernels (device memory).
struct SolveStatus {
    long long iters_done;  // advances applied in this launch
    int converged;         // stop rule met (||x - x_ref||^2 < eps)
    int checks;            // stop-rule evaluations in this launch
    double err;            // last evaluated ||x - x_ref||^2
    int aborted;           // cross-cluster exchange timed out (co-residency violated)
    int pad;
};

// Shared by both solve kernels.
struct SolveArgs {
    const double* A;       // m x ld, row-major, pitched
    const double* b;       // m
    const double* sq;      // m squared row norms (einsum order)
    const double* bs2;     // m x 4 packed (b_i, sq_i, RN(1/sq_i), 0)
    const double* xref;    // ld (zero padded)
    double* x;             // ld, the iterate (in/out)
    double* partial;       // non-null: one iteration, write sum_t v_t here instead of x
    double* V;             // q x ld worker estimates (chain kernel, q > 1)
    const int32_t* idx;    // row indices of this chunk (layout per kernel)
    const double* alphas;  // q row weights
    double* part;          // cross-CTA partial sums (sync kernel, grid mode)
    unsigned* barrier;     // grid barrier counter (zeroed per launch)
    SolveStatus* status;
    double* ckpt;          // checkpoints (ckpt_cap x n, row stride n)
    int64_t n, ld, q, bs;
    int64_t k0, count;     // iterations [k0, k0 + count) in this launch
    int64_t idx_stride;    // chain: draws per worker in the chunk; sync: q
    int64_t ckpt_every, ckpt_cap;
    double eps;
    int use_stop;          // evaluate the stop rule before each iteration
    int final_check;       // also evaluate it at k0 + count (max_iterations reached)
    int stages;            // cp.async ring depth
    long long* dbg;        // optional phase timestamps (KZ_PHASE_TIMING=1)
    int ablate;            // debug: bit mask of phases to skip (KZ_ABLATE), timing experiments only
    int box;               // rka kernel: TMA box width (columns of the row slice)
    int* halt;             // optional: nonzero = the solve already stopped, the launch is a no-op
                           // (device-side stop flag of the row-sharded driver, kz_solve_sharded);
                           // the rka kernel raises it (stop iteration + 1) when its stop rule fires
    const double* x_sum;   // rka kernel, optional: x_k = x_sum / x_div (the all-reduced worker sum of the
    double x_div;          // previous row-sharded step) instead of x
    int wg;                // rka kernel: worker-group mode (cluster g runs workers [g q/G, (g+1) q/G))
    // rka kernel, cross-rank mode (row-sharded multi-GPU in one launch): every rank's column sums
    // go as tagged words into every rank's exchange buffer over NVLink peer memory
    unsigned long long* const* xr_peers;  // device array: each rank's exchange buffer (own rank's is local)
    int xr_ranks, xr_rank;
    unsigned xr_tag0;      // tag of iteration k0 (unique across launches and solves of the communicator)
    // chain kernel, q > 1: how the worker estimates meet (KZ_COMBINE_*): the sequential engine's
    // ordered average, or the threaded engine's increments added to x in worker order
    int combine;
    // chain kernel, row-sharded / wave steps (partial != nullptr): 1 = add this launch's worker sum to
    // the sum already in partial, in worker order (the workers of one outer iteration in several
    // launches when they are more than the co-resident CTAs)
    int accumulate;
};

// rka kernel, column-sliced plans with several clusters: u64 words per slot of the cluster-total
// tagged-word exchange.  One 128-byte line per (cluster, worker): slots written by different owner
// CTAs and polled by all of them no longer share L2 lines (c3 RKA 5.10 -> 4.87 us per iteration
// against 16-byte slots, measured with a runtime stride)
constexpr int RKA_LL_PAD = 16;

enum {
    KZ_COMBINE_AVERAGE = 0,    // x = (sum_t v_t) / q                         (solvers.py:131-137, 366-367)
    KZ_COMBINE_RKA_DELTA = 1,  // x += alpha (b_t - <a_t, x>) / (q sq_t) a_t   (parallel.py:214-226)
    KZ_COMBINE_RKAB_DELTA = 2  // x += (v_t - x) / q                           (parallel.py:286-298)
};

// chain kernel: worker-per-CTA (RK, RKAB).  EP = 16-byte pairs per thread,
// R = rows resolved per CTA reduction (Gram-corrected block), C = CTAs per worker.
template <int EP, int R, int C, bool DELTA = false, bool WIDE = false>
__global__ void chain_kernel(SolveArgs a);

// one-warp RK / CK kernel for short rows (n <= 64 EPL); P rows prefetched in registers
template <int EPL, int P>
__global__ void rkw_kernel(SolveArgs a);

// sync kernel: column-sliced (RKA, RKAB bs=1).  CLUSTER: reduce via DSMEM.
template <bool CLUSTER, int LPR>
__global__ void sync_kernel(SolveArgs a);

// rka kernel: column-sliced RKA with TMA-gather row staging by a producer warp,
// 8 compute warps, DSMEM exchange inside each cluster and tagged global words
// between clusters.  LG = lanes per row group, EPL = column pairs per lane.
constexpr int RKA_NW = 8;                  // compute warps
constexpr int RKA_NT = (RKA_NW + 1) * 32;  // + the producer warp
constexpr int RKA_MAXG = 10;               // clusters exchanging through tagged words
constexpr int RKA_MAXR = 8;                // ranks (GPUs of one node) exchanging column sums
// MODE 0: column-sliced; 1: worker groups; 2: column-sliced + cross-rank column sums (kz_solve_sharded)
template <int LG, int EPL, bool TIMING, bool SR, int MODE>
__global__ void rka_kernel(const __grid_constant__ SolveArgs a, const __grid_constant__ CUtensorMap tmA,
                           const __grid_constant__ CUtensorMap tmB);

__global__ void row_sqnorm_kernel(const double* __restrict__ A, int64_t m, int64_t n, int64_t ld,
                                  double* __restrict__ sq, unsigned long long* __restrict__ first_zero);
__global__ void cyclic_rows_kernel(int32_t* __restrict__ idx, int64_t k0, int64_t count, int64_t m);
// CGLS (kz_cgls.cu)
__global__ void cg_gemv_n_kernel(const double* __restrict__ A, const double* __restrict__ x,
                                 const double* __restrict__ b, int64_t m, int64_t n, int64_t ld, int mode,
                                 double* __restrict__ y);
__global__ void cg_gemv_t_partial_kernel(const double* __restrict__ A, const double* __restrict__ r, int64_t m,
                                         int64_t n, int64_t ld, int64_t rows_per_chunk, double* __restrict__ partial);
__global__ void cg_gemv_t_reduce_kernel(const double* __restrict__ partial, int64_t nchunks, int64_t n, int64_t ld,
                                        double* __restrict__ s);
__global__ void cg_dot_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                              double* __restrict__ out);
__global__ void cg_update_xr_kernel(double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
                                    const double* __restrict__ t, const double* __restrict__ scal, int64_t n,
                                    int64_t m);
__global__ void cg_update_p_kernel(double* __restrict__ p, const double* __restrict__ s,
                                   const double* __restrict__ scal, int64_t n);
__global__ void cg_scale_div_kernel(const double* __restrict__ w, const double* __restrict__ nw, int64_t n,
                                    double* __restrict__ v);
__global__ void repack_rows_kernel(const double* __restrict__ src, int64_t m, int64_t n, int64_t ld,
                                   double* __restrict__ dst);
constexpr int CDF_SCAN_THREADS = 256;
__global__ void cdf_scan_kernel(const double* __restrict__ sq, const int64_t* __restrict__ lo,
                                const int64_t* __restrict__ len, int64_t nranges, double* __restrict__ cdf);
__global__ void cdf_div_kernel(double* __restrict__ cdf, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ len);
__global__ void cdf_div_last_kernel(double* __restrict__ cdf, const int64_t* __restrict__ lo,
                                    const int64_t* __restrict__ len, int64_t nranges);
__global__ void sample_rows_kernel(const double* __restrict__ cdf, const int64_t* __restrict__ lo,
                                   const int64_t* __restrict__ len, const PcgPod* __restrict__ base_states,
                                   int64_t q, int64_t d0, int64_t count, int32_t* __restrict__ out,
                                   int64_t stride_w, int64_t stride_d);
__global__ void residual_rows_kernel(const double* __restrict__ A, const double* __restrict__ b,
                                     const double* __restrict__ x, int64_t m, int64_t n, int64_t ld,
                                     double* __restrict__ out);
__global__ void residual_batch_kernel(const double* __restrict__ A, const double* __restrict__ b,
                                      const double* __restrict__ X, int64_t m, int64_t n, int64_t ld, int K,
                                      double* __restrict__ out);
__global__ void diff_sq_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                               double* __restrict__ out);
__global__ void pack_bs2_kernel(const double* __restrict__ b, const double* __restrict__ sq, int64_t m,
                                double* __restrict__ out);
__global__ void scale_copy_kernel(const double* __restrict__ S, double inv_div, int64_t n, double* __restrict__ x);
__global__ void sum_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out);
__global__ void shard_average_kernel(const double* __restrict__ S, double Q, int64_t n, int64_t ld,
                                     const double* __restrict__ xref, double* __restrict__ x, double eps,
                                     int use_stop, int64_t k_next, double* __restrict__ err_out,
                                     int* __restrict__ halt);

__global__ void gen_counter_kernel(double* __restrict__ A, int64_t m, int64_t n, int64_t ld, uint64_t seed,
                                   double mu_lo, double mu_hi, double sg_lo, double sg_hi, int64_t row0);
__global__ void gen_xstar_kernel(double* __restrict__ x, int64_t n, int64_t ld, uint64_t seed, double mu_lo,
                                 double mu_hi, double sg_lo, double sg_hi);
__global__ void gemv_rows_kernel(const double* __restrict__ A, const double* __restrict__ x, int64_t m, int64_t n,
                                 int64_t ld, double* __restrict__ b);

constexpr int NORM_ROWS_PER_CTA = 128;
constexpr int SAMPLE_RUN = 8;
constexpr int IDX_WINDOW = 1024;  // chain kernel: smem ring of row indices

}  // namespace kz
