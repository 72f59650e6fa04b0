/*
 * kz_oracle.h -- CPU restatement of the reference's RK / RKA / RKAB hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker and the
 * CPU baseline ("port") for bench.py.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path (paper_2401_17474_b200) never links or calls it.
 *
 * Parity is pinned against golden vectors produced by executing the
 * reference (kaczbench, numpy 2.3.5 / OpenBLAS 0.3.30) in the build
 * container: tests/golden/make_golden.py writes tests/golden/ fixtures and
 * tests/test_oracle_golden.py checks this library against them.
 *
 * Third-party arithmetic restated here (numpy 2.3.5, not vendored in the
 * reference; call sites in /root/reference/pkg/src/kaczbench):
 *   - SeedSequence(entropy=(seed, stream)) -> PCG64 -> Generator.random()
 *     (sampling.py:44-52)
 *   - np.einsum("ij,ij->i") row norms, SSE2 2-lane x4 order (linalg.py:83)
 *   - np.cumsum then "/= cdf[-1]" (sampling.py:108-109)
 *   - np.searchsorted(side="right") + clamp (sampling.py:89-94)
 *   - np.sum(v_all, axis=0) sequential over workers, then "/= q"
 *     (solvers.py:136-137, 366-367)
 * np.dot (OpenBLAS ddot, runtime-dispatched kernel) is restated as a
 * plain left-to-right sum; iterates therefore match the reference to
 * rounding (tolerance parity, 1e-10 relative), row indices bit-exactly.
 */
#ifndef KZ_ORACLE_H
#define KZ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* PCG64 (XSL-RR 128/64) generator state, 128-bit words split hi/lo. */
typedef struct {
    uint64_t state_hi, state_lo;
    uint64_t inc_hi, inc_lo;
} kzo_pcg64;

enum { KZO_RK = 0, KZO_RKA = 1, KZO_RKAB = 2, KZO_CK = 3 };
enum { KZO_FULL_ACCESS = 0, KZO_DISTRIBUTED = 1 };

enum {
    KZO_OK = 0,
    KZO_EINVAL = 1,       /* ValueError (solvers.py:85-101)           */
    KZO_EDEGENERATE = 2,  /* DegenerateRowError (linalg.py:84-86)     */
    KZO_EEMPTYRANGE = 3,  /* EmptyRangeError (sampling.py:106-107,213-218) */
    KZO_ENOMEM = 4
};

typedef struct {
    int32_t variant;          /* KZO_RK / KZO_RKA / KZO_RKAB / KZO_CK        */
    int32_t scheme;           /* KZO_FULL_ACCESS / KZO_DISTRIBUTED           */
    int64_t q;                /* workers                                     */
    int64_t block_size;       /* RKAB chain length                           */
    const double* alphas;     /* q weights, NULL = all 1.0                   */
    uint64_t base_seed;
    double epsilon;
    int64_t max_iterations;
    int64_t budget;           /* > 0: fixed-budget replay, no stop checks    */
    int64_t ckpt_every;       /* > 0: store x after every ckpt_every iters  */
    int64_t ckpt_capacity;    /* rows available in ckpt_out                  */
    int32_t nthreads;         /* <= 1 serial; > 1 pthreads (bitwise identical) */
    int32_t combine;          /* 0: sequential engine's average; 1: threaded engine's
                                 increments in worker order (parallel.py:214-226, 286-298) */
} kzo_params;

typedef struct {
    int64_t iterations;
    int32_t converged;
    int32_t pad;
    double final_error_sq;
    int64_t error_evals;
    int64_t n_ckpt;
    int64_t bad_row;          /* KZO_EDEGENERATE: first zero row            */
    double loop_seconds;      /* wall time of the iteration loop alone      */
} kzo_result;

/* SeedSequence(entropy).generate_state(n_words, uint32) */
void kzo_seedseq_generate(const uint64_t* entropy, int32_t n_entropy,
                          uint32_t* out_words, int32_t n_words);
/* PCG64(SeedSequence(entropy)) */
void kzo_pcg64_seed(const uint64_t* entropy, int32_t n_entropy, kzo_pcg64* g);
uint64_t kzo_pcg64_next(kzo_pcg64* g);
double kzo_pcg64_random(kzo_pcg64* g);
void kzo_pcg64_advance(kzo_pcg64* g, uint64_t delta_hi, uint64_t delta_lo);
/* Prng(seed, stream).random() x count */
void kzo_random_doubles(uint64_t seed, uint64_t stream, int64_t count, double* out);

/* np.einsum("ij,ij->i", A, A) for row-major A (m x n, leading dim lda) */
void kzo_row_sqnorms(const double* A, int64_t m, int64_t n, int64_t lda, double* out);
/* cdf = cumsum(sq[lo..hi]) / last  (len = hi-lo+1) */
int32_t kzo_cdf_build(const double* sq, int64_t m, int64_t lo, int64_t hi, double* cdf);
int64_t kzo_upper_bound(const double* cdf, int64_t len, double u);
/* first `count` row draws of worker `worker` (stream (seed, worker)) */
int32_t kzo_dump_rows(const double* sq, int64_t m, int32_t scheme, int64_t q,
                      uint64_t seed, int64_t worker, int64_t count, int64_t* out);

/* Full solve: reference _drive protocol (solvers.py:182-263). */
int32_t kzo_solve(const double* A, const double* b, const double* x_ref,
                  int64_t m, int64_t n, const kzo_params* p,
                  kzo_result* r, double* x_out, double* ckpt_out);

int32_t kzo_max_threads(void);

#ifdef __cplusplus
}
#endif
#endif
