/*
 * kz_oracle.c -- CPU restatement (oracle) of the reference RK/RKA/RKAB loop.
 *
 * TEST INFRASTRUCTURE ONLY (see kz_oracle.h).  Compiled with
 * -ffp-contract=off so every "a*b + c" is two roundings, as numpy does.
 *
 * Reference anchors (paths relative to /root/reference/pkg/src/kaczbench):
 *   Prng / worker_rng ............ sampling.py:34-74
 *   RowSampler.sample ............ sampling.py:89-94
 *   make_sampler ................. sampling.py:101-111
 *   partition_bounds ............. sampling.py:119-131
 *   row_norm_cache ............... linalg.py:80-88
 *   kaczmarz_step ................ solvers.py:107-117
 *   rka_combined_step ............ solvers.py:120-137
 *   rkab_worker_block ............ solvers.py:140-145
 *   worker_streams ............... solvers.py:162-171
 *   _drive (stop/budget/capture) . solvers.py:182-263
 *   solve_rk/rka_seq/rkab_seq .... solvers.py:294-371
 */
#include "kz_oracle.h"

#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <time.h>
#include <unistd.h>

typedef unsigned __int128 u128;

/* ---------------------------------------------------------------------
 * numpy SeedSequence (bit_generator.pyx), restated.  All arithmetic is
 * mod 2^32.  Entropy ints are split into little-endian 32-bit words;
 * the int 0 contributes one zero word.
 * ------------------------------------------------------------------- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u
#define SS_POOL 4

static uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
    v ^= *hc;
    *hc *= SS_MULT_A;
    v *= *hc;
    v ^= v >> 16;
    return v;
}

static uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
    r ^= r >> 16;
    return r;
}

void kzo_seedseq_generate(const uint64_t* entropy, int32_t n_entropy,
                          uint32_t* out_words, int32_t n_words) {
    uint32_t words[64];
    int nw = 0;
    for (int e = 0; e < n_entropy && nw < 60; ++e) {
        uint64_t v = entropy[e];
        if (v == 0) {
            words[nw++] = 0;
        } else {
            while (v) {
                words[nw++] = (uint32_t)(v & 0xffffffffu);
                v >>= 32;
            }
        }
    }
    uint32_t pool[SS_POOL];
    uint32_t hc = SS_INIT_A;
    for (int i = 0; i < SS_POOL; ++i) pool[i] = ss_hashmix(i < nw ? words[i] : 0u, &hc);
    for (int s = 0; s < SS_POOL; ++s)
        for (int d = 0; d < SS_POOL; ++d)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
    for (int s = SS_POOL; s < nw; ++s)
        for (int d = 0; d < SS_POOL; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], &hc));
    uint32_t hb = SS_INIT_B;
    for (int i = 0; i < n_words; ++i) {
        uint32_t v = pool[i % SS_POOL];
        v ^= hb;
        hb *= SS_MULT_B;
        v *= hb;
        v ^= v >> 16;
        out_words[i] = v;
    }
}

/* ---------------------------------------------------------------------
 * PCG64 (numpy pcg64.h): 128-bit LCG, XSL-RR output of the stepped state.
 * ------------------------------------------------------------------- */
static const u128 PCG_MULT = (((u128)2549297995355413924ULL) << 64) | 4865540595714422341ULL;

static inline u128 g_state(const kzo_pcg64* g) { return ((u128)g->state_hi << 64) | g->state_lo; }
static inline u128 g_inc(const kzo_pcg64* g) { return ((u128)g->inc_hi << 64) | g->inc_lo; }
static inline void g_set_state(kzo_pcg64* g, u128 s) {
    g->state_hi = (uint64_t)(s >> 64);
    g->state_lo = (uint64_t)s;
}

void kzo_pcg64_seed(const uint64_t* entropy, int32_t n_entropy, kzo_pcg64* g) {
    uint32_t w[8];
    kzo_seedseq_generate(entropy, n_entropy, w, 8);
    uint64_t u[4];
    for (int i = 0; i < 4; ++i) u[i] = (uint64_t)w[2 * i] | ((uint64_t)w[2 * i + 1] << 32);
    u128 initstate = ((u128)u[0] << 64) | u[1];
    u128 initseq = ((u128)u[2] << 64) | u[3];
    u128 inc = (initseq << 1) | 1u;
    u128 s = 0;
    s = s * PCG_MULT + inc;
    s += initstate;
    s = s * PCG_MULT + inc;
    g->inc_hi = (uint64_t)(inc >> 64);
    g->inc_lo = (uint64_t)inc;
    g_set_state(g, s);
}

uint64_t kzo_pcg64_next(kzo_pcg64* g) {
    u128 s = g_state(g) * PCG_MULT + g_inc(g);
    g_set_state(g, s);
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    uint64_t x = hi ^ lo;
    unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

double kzo_pcg64_random(kzo_pcg64* g) {
    return (double)(kzo_pcg64_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

/* state <- state advanced by delta steps (Brown's LCG jump-ahead). */
void kzo_pcg64_advance(kzo_pcg64* g, uint64_t delta_hi, uint64_t delta_lo) {
    u128 delta = ((u128)delta_hi << 64) | delta_lo;
    u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = g_inc(g);
    while (delta) {
        if (delta & 1u) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    g_set_state(g, acc_mult * g_state(g) + acc_plus);
}

static void worker_stream(uint64_t seed, uint64_t worker, kzo_pcg64* g) {
    uint64_t ent[2] = {seed, worker};
    kzo_pcg64_seed(ent, 2, g);
}

void kzo_random_doubles(uint64_t seed, uint64_t stream, int64_t count, double* out) {
    kzo_pcg64 g;
    worker_stream(seed, stream, &g);
    for (int64_t i = 0; i < count; ++i) out[i] = kzo_pcg64_random(&g);
}

/* ---------------------------------------------------------------------
 * Row norms: np.einsum("ij,ij->i") (linalg.py:83).  Two lanes; each full
 * chunk of 8 updates lane l as e_l^2 + (e_{2+l}^2 + (e_{4+l}^2 +
 * (e_{6+l}^2 + acc_l))); the tail is consumed in zero-filled pairs, low
 * to high; result lane0 + lane1.
 * ------------------------------------------------------------------- */
static double einsum_sqnorm(const double* r, int64_t n) {
    double l0 = 0.0, l1 = 0.0;
    int64_t j = 0;
    for (; j + 8 <= n; j += 8) {
        l0 = r[j] * r[j] + (r[j + 2] * r[j + 2] + (r[j + 4] * r[j + 4] + (r[j + 6] * r[j + 6] + l0)));
        l1 = r[j + 1] * r[j + 1] + (r[j + 3] * r[j + 3] + (r[j + 5] * r[j + 5] + (r[j + 7] * r[j + 7] + l1)));
    }
    for (; j < n; j += 2) {
        double e0 = r[j];
        double e1 = (j + 1 < n) ? r[j + 1] : 0.0;
        l0 = e0 * e0 + l0;
        l1 = e1 * e1 + l1;
    }
    return l0 + l1;
}

void kzo_row_sqnorms(const double* A, int64_t m, int64_t n, int64_t lda, double* out) {
    for (int64_t i = 0; i < m; ++i) out[i] = einsum_sqnorm(A + i * lda, n);
}

/* Row norms over row bands on `nt` threads: each row is still one einsum_sqnorm, so the
 * result is bitwise the serial one (the CPU baseline's setup on 25.6 GB systems). */
typedef struct {
    const double* A;
    int64_t m, n, lda;
    double* out;
    int tid, nt;
} norms_arg_t;

static void* norms_body(void* argp) {
    norms_arg_t* a = (norms_arg_t*)argp;
    const int64_t r0 = (a->m * a->tid) / a->nt, r1 = (a->m * (a->tid + 1)) / a->nt;
    for (int64_t i = r0; i < r1; ++i) a->out[i] = einsum_sqnorm(a->A + i * a->lda, a->n);
    return NULL;
}

static void row_sqnorms_mt(const double* A, int64_t m, int64_t n, int64_t lda, double* out, int nt) {
    if (nt <= 1 || m < 4096) {
        kzo_row_sqnorms(A, m, n, lda, out);
        return;
    }
    if (nt > 256) nt = 256;
    pthread_t th[256];
    norms_arg_t args[256];
    for (int i = 0; i < nt; ++i) {
        args[i] = (norms_arg_t){A, m, n, lda, out, i, nt};
        if (i > 0) pthread_create(&th[i], NULL, norms_body, &args[i]);
    }
    norms_body(&args[0]);
    for (int i = 1; i < nt; ++i) pthread_join(th[i], NULL);
}

static double now_seconds(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

static int64_t first_zero(const double* sq, int64_t m) {
    for (int64_t i = 0; i < m; ++i)
        if (sq[i] == 0.0) return i;
    return -1;
}

/* make_sampler (sampling.py:101-111): sequential cumsum, divide by last. */
int32_t kzo_cdf_build(const double* sq, int64_t m, int64_t lo, int64_t hi, double* cdf) {
    if (!(0 <= lo && lo <= hi && hi < m)) return KZO_EEMPTYRANGE;
    int64_t len = hi - lo + 1;
    double acc = 0.0;
    for (int64_t j = 0; j < len; ++j) {
        acc = acc + sq[lo + j];
        cdf[j] = acc;
    }
    double last = cdf[len - 1];
    for (int64_t j = 0; j < len; ++j) cdf[j] = cdf[j] / last;
    return KZO_OK;
}

/* searchsorted(cdf, u, side="right") (sampling.py:91) */
int64_t kzo_upper_bound(const double* cdf, int64_t len, double u) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        int64_t mid = lo + ((hi - lo) >> 1);
        if (cdf[mid] <= u)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

/* partition_bounds (sampling.py:119-131) */
static int bounds(int64_t m, int64_t parts, int64_t idx, int64_t* lo, int64_t* hi) {
    if (!(0 <= idx && idx < parts)) return KZO_EEMPTYRANGE;
    *lo = (idx * m) / parts;
    *hi = ((idx + 1) * m) / parts - 1;
    if (*hi < *lo) return KZO_EEMPTYRANGE;
    return KZO_OK;
}

typedef struct {
    const double* cdf; /* cdf of this worker's support */
    int64_t lo, len;
} sampler_t;

/* RowSampler.sample (sampling.py:89-94) */
static inline int64_t sampler_draw(const sampler_t* s, kzo_pcg64* g) {
    double u = kzo_pcg64_random(g);
    int64_t j = kzo_upper_bound(s->cdf, s->len, u);
    if (j >= s->len) j = s->len - 1;
    return s->lo + j;
}

/* worker_streams (solvers.py:162-171).  cdf_store has m entries: the
 * full-access cdf, or the concatenated per-block cdfs (blocks tile [0,m)). */
static int build_samplers(const double* sq, int64_t m, int32_t scheme, int64_t q,
                          double* cdf_store, sampler_t* samplers) {
    if (scheme == KZO_FULL_ACCESS) {
        int rc = kzo_cdf_build(sq, m, 0, m - 1, cdf_store);
        if (rc) return rc;
        for (int64_t t = 0; t < q; ++t) {
            samplers[t].cdf = cdf_store;
            samplers[t].lo = 0;
            samplers[t].len = m;
        }
        return KZO_OK;
    }
    for (int64_t t = 0; t < q; ++t) {
        int64_t lo, hi;
        int rc = bounds(m, q, t, &lo, &hi);
        if (rc) return rc;
        rc = kzo_cdf_build(sq, m, lo, hi, cdf_store + lo);
        if (rc) return rc;
        samplers[t].cdf = cdf_store + lo;
        samplers[t].lo = lo;
        samplers[t].len = hi - lo + 1;
    }
    return KZO_OK;
}

int32_t kzo_dump_rows(const double* sq, int64_t m, int32_t scheme, int64_t q,
                      uint64_t seed, int64_t worker, int64_t count, int64_t* out) {
    if (q < 1 || worker < 0 || worker >= q) return KZO_EINVAL;
    double* cdf = (double*)malloc(sizeof(double) * (size_t)m);
    sampler_t* s = (sampler_t*)malloc(sizeof(sampler_t) * (size_t)q);
    if (!cdf || !s) {
        free(cdf);
        free(s);
        return KZO_ENOMEM;
    }
    int rc = build_samplers(sq, m, scheme, q, cdf, s);
    if (rc == KZO_OK) {
        kzo_pcg64 g;
        worker_stream(seed, (uint64_t)worker, &g);
        for (int64_t k = 0; k < count; ++k) out[k] = sampler_draw(&s[worker], &g);
    }
    free(cdf);
    free(s);
    return rc;
}

/* ---------------------------------------------------------------------
 * Projection primitive (solvers.py:107-117):
 *   scale = alpha * (b_i - <a_i, x>) / sq_i ;  x += scale * a_i
 * The dot is a plain left-to-right sum (OpenBLAS order is unspecified).
 * ------------------------------------------------------------------- */
static inline double row_dot(const double* a, const double* x, int64_t n) {
    double d = 0.0;
    for (int64_t j = 0; j < n; ++j) d = d + a[j] * x[j];
    return d;
}

static inline double proj_scale(const double* A, const double* b, const double* sq, int64_t n,
                                int64_t i, const double* x, double alpha) {
    return alpha * (b[i] - row_dot(A + i * n, x, n)) / sq[i];
}

static inline void kaczmarz_step(double* x, const double* A, const double* b, const double* sq,
                                 int64_t n, int64_t i, double alpha) {
    double s = proj_scale(A, b, sq, n, i, x, alpha);
    const double* a = A + i * n;
    for (int64_t j = 0; j < n; ++j) x[j] = x[j] + s * a[j];
}

static double err_sq(const double* x, const double* xr, int64_t n) {
    double e = 0.0;
    for (int64_t j = 0; j < n; ++j) {
        double d = x[j] - xr[j];
        e = e + d * d;
    }
    return e;
}

typedef struct {
    const double *A, *b, *sq;
    int64_t m, n, q, bs;
    int32_t variant, nthreads, combine;
    const double* alphas;
    sampler_t* samplers;
    kzo_pcg64* rngs;
    int64_t* rows;   /* q   (RKA row of each worker this iteration) */
    double* scales;  /* q                                            */
    double* vbuf;    /* q*n (RKAB private estimates)                 */
    int64_t k;       /* iterations applied (CK row = k mod m)        */
} run_t;

/* Column range [c0,c1) of the averaging for thread `tid` of `nt`. */
static void col_range(int64_t n, int nt, int tid, int64_t* c0, int64_t* c1) {
    *c0 = (n * tid) / nt;
    *c1 = (n * (tid + 1)) / nt;
}

/* RKA averaging (solvers.py:131-137), columns [c0,c1):
 * x_j <- (sum_t fl(x_j + fl(s_t a_tj))) / q, summed t = 0..q-1. */
static void rka_average(run_t* R, double* x, int64_t c0, int64_t c1) {
    const int64_t n = R->n, q = R->q;
    for (int64_t j = c0; j < c1; ++j) {
        double xj = x[j];
        double acc = xj + R->scales[0] * R->A[R->rows[0] * n + j];
        for (int64_t t = 1; t < q; ++t) acc = acc + (xj + R->scales[t] * R->A[R->rows[t] * n + j]);
        x[j] = acc / (double)q;
    }
}

/* Threaded engine, RKA (parallel.py:214-226): the workers' increments
 * fl(s_t a_tj), s_t = alpha (b - <a, x_prev>) / (q sq), added to x in worker order. */
static void rka_delta(run_t* R, double* x, int64_t c0, int64_t c1) {
    const int64_t n = R->n, q = R->q;
    for (int64_t j = c0; j < c1; ++j)
        for (int64_t t = 0; t < q; ++t) x[j] = x[j] + R->scales[t] * R->A[R->rows[t] * n + j];
}

/* Threaded engine, RKAB (parallel.py:286-298): v -= x_prev; x += v / q, worker order. */
static void rkab_delta(run_t* R, double* x, int64_t c0, int64_t c1) {
    const int64_t n = R->n, q = R->q;
    for (int64_t j = c0; j < c1; ++j) {
        const double xp = x[j];
        double acc = xp;
        for (int64_t t = 0; t < q; ++t) acc = acc + (R->vbuf[t * n + j] - xp) / (double)q;
        x[j] = acc;
    }
}

/* RKAB averaging (solvers.py:366-367) */
static void rkab_average(run_t* R, double* x, int64_t c0, int64_t c1) {
    const int64_t n = R->n, q = R->q;
    for (int64_t j = c0; j < c1; ++j) {
        double acc = R->vbuf[j];
        for (int64_t t = 1; t < q; ++t) acc = acc + R->vbuf[t * n + j];
        x[j] = acc / (double)q;
    }
}

static void combine(run_t* R, double* x, int64_t c0, int64_t c1) {
    if (R->variant == KZO_RKA)
        (R->combine ? rka_delta : rka_average)(R, x, c0, c1);
    else
        (R->combine ? rkab_delta : rkab_average)(R, x, c0, c1);
}

/* Worker part of one outer iteration (parallel over t). */
static void worker_part(run_t* R, const double* x, int64_t t) {
    const int64_t n = R->n;
    double alpha = R->alphas ? R->alphas[t] : 1.0;
    if (R->variant == KZO_RKA) {
        int64_t i = sampler_draw(&R->samplers[t], &R->rngs[t]);
        R->rows[t] = i;
        if (R->combine) /* parallel.py:221: the weight carries 1/q */
            R->scales[t] = alpha * (R->b[i] - row_dot(R->A + i * n, x, n)) / ((double)R->q * R->sq[i]);
        else
            R->scales[t] = proj_scale(R->A, R->b, R->sq, n, i, x, alpha);
    } else { /* RKAB: v = x; bs chained projections (solvers.py:140-145) */
        double* v = R->vbuf + t * n;
        memcpy(v, x, sizeof(double) * (size_t)n);
        for (int64_t s = 0; s < R->bs; ++s) {
            int64_t i = sampler_draw(&R->samplers[t], &R->rngs[t]);
            kaczmarz_step(v, R->A, R->b, R->sq, n, i, alpha);
        }
    }
}

/* One iteration (advance) of the variant, serial. */
static void advance_serial(run_t* R, double* x) {
    if (R->variant == KZO_CK) { /* solvers.py:286-287: row k mod m */
        kaczmarz_step(x, R->A, R->b, R->sq, R->n, R->k % R->m, R->alphas ? R->alphas[0] : 1.0);
        ++R->k;
        return;
    }
    if (R->variant == KZO_RK) {
        int64_t i = sampler_draw(&R->samplers[0], &R->rngs[0]);
        kaczmarz_step(x, R->A, R->b, R->sq, R->n, i, R->alphas ? R->alphas[0] : 1.0);
        return;
    }
    for (int64_t t = 0; t < R->q; ++t) worker_part(R, x, t);
    combine(R, x, 0, R->n);
}

/* ---------------------------------------------------------------------
 * Multi-threaded driver (CPU baseline).  Same arithmetic as the serial
 * loop, hence bitwise-identical results: each worker's chain and stream
 * are private to one thread, the averaging is split by columns with the
 * per-column worker order unchanged, and thread 0 evaluates the stop
 * rule serially.  Two barriers per iteration.
 * ------------------------------------------------------------------- */
typedef struct {
    run_t* R;
    const kzo_params* p;
    double* x;
    const double* x_ref;
    double* ckpt_out;
    int64_t limit, k, evals, n_ck;
    double e;
    int use_stop, converged, stop, nt;
    pthread_barrier_t bar;
} mt_shared_t;

typedef struct {
    mt_shared_t* S;
    int tid;
} mt_arg_t;

static void* mt_body(void* argp) {
    mt_arg_t* a = (mt_arg_t*)argp;
    mt_shared_t* S = a->S;
    run_t* R = S->R;
    const kzo_params* p = S->p;
    const int tid = a->tid, nt = S->nt;
    const int64_t n = R->n;
    int64_t c0, c1;
    col_range(n, nt, tid, &c0, &c1);
    for (;;) {
        if (tid == 0) {
            if (S->use_stop) {
                S->e = err_sq(S->x, S->x_ref, n);
                ++S->evals;
                if (S->e < p->epsilon) {
                    S->converged = 1;
                    S->stop = 1;
                }
            }
            if (!S->stop && S->k >= S->limit) S->stop = 1;
        }
        pthread_barrier_wait(&S->bar);
        if (S->stop) break;
        for (int64_t t = tid; t < R->q; t += nt) worker_part(R, S->x, t);
        pthread_barrier_wait(&S->bar);
        combine(R, S->x, c0, c1);
        pthread_barrier_wait(&S->bar);
        if (tid == 0) {
            ++S->k;
            if (p->ckpt_every > 0 && S->k % p->ckpt_every == 0 && S->n_ck < p->ckpt_capacity)
                memcpy(S->ckpt_out + (S->n_ck++) * n, S->x, sizeof(double) * (size_t)n);
        }
    }
    return NULL;
}

int32_t kzo_max_threads(void) {
    long c = sysconf(_SC_NPROCESSORS_ONLN);
    return c > 0 ? (int32_t)c : 1;
}

int32_t kzo_solve(const double* A, const double* b, const double* x_ref, int64_t m, int64_t n,
                  const kzo_params* p, kzo_result* r, double* x_out, double* ckpt_out) {
    memset(r, 0, sizeof(*r));
    r->bad_row = -1;
    if (m < 1 || n < 1 || p->q < 1 || p->block_size < 1 || !(p->epsilon > 0) ||
        p->max_iterations < 1 || p->variant < KZO_RK || p->variant > KZO_CK)
        return KZO_EINVAL;
    if ((p->variant == KZO_RK || p->variant == KZO_CK) && p->q != 1) return KZO_EINVAL;
    if (p->budget <= 0 && !x_ref) return KZO_EINVAL;

    run_t R;
    memset(&R, 0, sizeof(R));
    R.A = A;
    R.b = b;
    R.m = m;
    R.n = n;
    R.q = p->q;
    R.bs = p->block_size;
    R.variant = p->variant;
    R.alphas = p->alphas;
    R.nthreads = p->nthreads;
    R.combine = p->combine;

    double* sq = (double*)malloc(sizeof(double) * (size_t)m);
    double* cdf = (double*)malloc(sizeof(double) * (size_t)m);
    R.samplers = (sampler_t*)malloc(sizeof(sampler_t) * (size_t)R.q);
    R.rngs = (kzo_pcg64*)malloc(sizeof(kzo_pcg64) * (size_t)R.q);
    R.rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)R.q);
    R.scales = (double*)malloc(sizeof(double) * (size_t)R.q);
    R.vbuf = (p->variant == KZO_RKAB) ? (double*)malloc(sizeof(double) * (size_t)(R.q * n)) : NULL;
    int rc = KZO_OK;
    if (!sq || !cdf || !R.samplers || !R.rngs || !R.rows || !R.scales ||
        (p->variant == KZO_RKAB && !R.vbuf)) {
        rc = KZO_ENOMEM;
        goto done;
    }
    row_sqnorms_mt(A, m, n, n, sq, p->nthreads);
    R.sq = sq;
    r->bad_row = first_zero(sq, m);
    if (r->bad_row >= 0) {
        rc = KZO_EDEGENERATE;
        goto done;
    }
    if (p->variant != KZO_CK) {
        rc = build_samplers(sq, m, p->scheme, R.q, cdf, R.samplers);
        if (rc) goto done;
    }
    for (int64_t t = 0; t < R.q; ++t) worker_stream(p->base_seed, (uint64_t)t, &R.rngs[t]);

    double* x = x_out;
    memset(x, 0, sizeof(double) * (size_t)n);
    int64_t n_ck = 0;
    const int64_t limit = p->budget > 0 ? p->budget : p->max_iterations;
    const int use_stop = p->budget <= 0;
    int64_t k = 0;
    double e = 0.0;
    int converged = 0;
    int64_t evals = 0;

    const int nt = (p->nthreads > 1 && p->variant != KZO_RK && p->variant != KZO_CK) ? p->nthreads : 1;
    const double t_loop0 = now_seconds(); /* the reference times the loop only (solvers.py:203-208) */
    if (nt <= 1) {
        for (;;) {
            if (use_stop) {
                e = err_sq(x, x_ref, n);
                ++evals;
                if (e < p->epsilon) {
                    converged = 1;
                    break;
                }
            }
            if (k >= limit) break;
            advance_serial(&R, x);
            ++k;
            if (p->ckpt_every > 0 && k % p->ckpt_every == 0 && n_ck < p->ckpt_capacity)
                memcpy(ckpt_out + (n_ck++) * n, x, sizeof(double) * (size_t)n);
        }
    } else {
        mt_shared_t S;
        memset(&S, 0, sizeof(S));
        S.R = &R;
        S.p = p;
        S.x = x;
        S.x_ref = x_ref;
        S.ckpt_out = ckpt_out;
        S.limit = limit;
        S.use_stop = use_stop;
        pthread_t th[256];
        mt_arg_t args[256];
        const int nth = nt > 256 ? 256 : nt;
        S.nt = nth;
        pthread_barrier_init(&S.bar, NULL, (unsigned)nth);
        for (int i = 1; i < nth; ++i) {
            args[i].S = &S;
            args[i].tid = i;
            pthread_create(&th[i], NULL, mt_body, &args[i]);
        }
        args[0].S = &S;
        args[0].tid = 0;
        mt_body(&args[0]);
        for (int i = 1; i < nth; ++i) pthread_join(th[i], NULL);
        pthread_barrier_destroy(&S.bar);
        k = S.k;
        e = S.e;
        converged = S.converged;
        evals = S.evals;
        n_ck = S.n_ck;
    }
    r->loop_seconds = now_seconds() - t_loop0;
    r->iterations = k;
    r->converged = converged;
    r->final_error_sq = use_stop ? e : 0.0;
    r->error_evals = evals;
    r->n_ckpt = n_ck;

done:
    free(sq);
    free(cdf);
    free(R.samplers);
    free(R.rngs);
    free(R.rows);
    free(R.scales);
    free(R.vbuf);
    return rc;
}
