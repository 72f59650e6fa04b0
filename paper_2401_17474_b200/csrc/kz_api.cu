// kz_api.cu -- the C-ABI (include/kz_b200.h): system residency, row norms,
// samplers, and the solve driver that replaces the reference's _drive loop
// (solvers.py:182-263) for RK / RKA / RKAB (solvers.py:294-371).
//
// The driver is native: it samples row indices for a chunk of iterations on
// the device (x-independent, bit-exact with RowSampler.sample), launches one
// persistent solve kernel per chunk, and reads back a 24-byte status word to
// learn whether the stop rule fired.  Python never runs per iteration.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <dlfcn.h>
#include <fcntl.h>
#include <unistd.h>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing unless a tool attaches
#include <nccl.h>  // types only: the library is dlopen'ed (the process's already-loaded libnccl.so.2 if any)

#include "../../include/kz_b200.h"
#include "kz_kernels.cuh"

// NVTX ranges around every entry point and every chunk launch (nsys / ncu --nvtx show the
// solve's setup, chunks and host round trips on the timeline)
struct NvtxScope {
    explicit NvtxScope(const char* name) { nvtxRangePushA(name); }
    ~NvtxScope() { nvtxRangePop(); }
    NvtxScope(const NvtxScope&) = delete;
    NvtxScope& operator=(const NvtxScope&) = delete;
};

using namespace kz;

// ---------------------------------------------------------------------------
// errors
// ---------------------------------------------------------------------------
static thread_local std::string g_err;
static std::atomic<long long> g_launches{0};

static int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define KZ_CUDA(call)                                                                                    \
    do {                                                                                                 \
        cudaError_t e_ = (call);                                                                         \
        if (e_ != cudaSuccess) return fail(KZ_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_));     \
    } while (0)

#define KZ_TRY(call)              \
    do {                          \
        int rc_ = (call);         \
        if (rc_ != KZ_OK) return rc_; \
    } while (0)

// Experiment switches (plan overrides, phase timing, ablations) are read only when
// KZ_EXPERIMENTS=1 is set in the environment: a production solve never consults them.
static const char* dbg_env(const char* name) {
    static const bool on = [] {
        const char* e = getenv("KZ_EXPERIMENTS");
        return e != nullptr && atoi(e) != 0;
    }();
    return on ? getenv(name) : nullptr;
}

static int check_launch(const char* what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(KZ_ECUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// SeedSequence -> PCG64 seeding on the host (numpy bit_generator.pyx / pcg64.c,
// as used by Prng(seed, worker), sampling.py:44-48).  Integer-exact.
// ---------------------------------------------------------------------------
namespace {

uint32_t ss_hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    v ^= v >> 16;
    return v;
}
uint32_t ss_mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    r ^= r >> 16;
    return r;
}

PcgPod seed_stream(uint64_t seed, uint64_t stream) {
    std::vector<uint32_t> words;
    for (uint64_t v : {seed, stream}) {
        if (v == 0) {
            words.push_back(0);
        } else {
            while (v) {
                words.push_back((uint32_t)(v & 0xffffffffu));
                v >>= 32;
            }
        }
    }
    uint32_t pool[4];
    uint32_t hc = 0x43b0d7e5u;
    for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < (int)words.size() ? words[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
        for (int d = 0; d < 4; ++d)
            if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], hc));
    for (size_t s = 4; s < words.size(); ++s)
        for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(words[s], hc));
    uint32_t out[8];
    uint32_t hb = 0x8b51f9ddu;
    for (int i = 0; i < 8; ++i) {
        uint32_t v = pool[i % 4];
        v ^= hb;
        hb *= 0x58f38dedu;
        v *= hb;
        v ^= v >> 16;
        out[i] = v;
    }
    uint64_t u[4];
    for (int i = 0; i < 4; ++i) u[i] = (uint64_t)out[2 * i] | ((uint64_t)out[2 * i + 1] << 32);
    const u128 initstate = ((u128)u[0] << 64) | u[1];
    const u128 initseq = ((u128)u[2] << 64) | u[3];
    Pcg g;
    g.inc = (initseq << 1) | 1u;
    g.s = 0;
    g.s = g.s * pcg_mult() + g.inc;
    g.s += initstate;
    g.s = g.s * pcg_mult() + g.inc;
    PcgPod p;
    p.s_hi = (unsigned long long)(g.s >> 64);
    p.s_lo = (unsigned long long)g.s;
    p.inc_hi = (unsigned long long)(g.inc >> 64);
    p.inc_lo = (unsigned long long)g.inc;
    return p;
}

template <typename T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;         // elements
    bool borrowed = false;  // a system view's alias of its base system's buffer: never freed or grown here
    int ensure(size_t n) {
        if (n <= cap) return KZ_OK;
        if (borrowed) return fail(KZ_EINVAL, "a system view cannot grow its base system's buffers");
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) {
            cudaGetLastError();
            return fail(KZ_ENOMEM, "cudaMalloc of %zu bytes failed", n * sizeof(T));
        }
        cap = n;
        return KZ_OK;
    }
    void release() {
        if (p && !borrowed) cudaFree(p);
        p = nullptr;
        cap = 0;
        borrowed = false;
    }
    void borrow(const DevBuf& o) {
        p = o.p;
        cap = o.cap;
        borrowed = true;
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// system
// ---------------------------------------------------------------------------
struct kz_system {
    int device = 0;
    int64_t m = 0, n = 0, ld = 0;
    int sms = 0;
    DevBuf<double> A, b, xref, x, sq, cdf, tmp, V, part, ckpt, alphas, bs2;
    DevBuf<int64_t> lo, len;
    DevBuf<int32_t> idx, rows_out;
    DevBuf<PcgPod> states;
    DevBuf<unsigned> barrier;
    DevBuf<SolveStatus> status;
    DevBuf<unsigned long long> zero_row;
    DevBuf<long long> dbg;
    DevBuf<double> cg;     // CGLS work vectors (kz_cgls)
    DevBuf<double> stage;  // dense host-upload staging (one 1-D copy, then a device repack)
    DevBuf<unsigned long long> ll;  // rka kernel: tagged words of the cross-cluster exchange
    size_t ll_words = 0;            // words the current plan uses
    DevBuf<double> S;               // kz_solve_sharded: the rank's worker sum (all-reduced in place)
    DevBuf<double> xs;              // kz_solve_seeds: one iterate per seed
    DevBuf<double> errs;            // kz_solve_sharded: ||x_k - x_ref||^2 per iteration of a chunk
    DevBuf<int> halt;               // kz_solve_sharded: device stop flag (k + 1 of the stop, 0 = running)
    DevBuf<double> tsnap, tr2, tsum;  // trace mode: pending iterate snapshots, their squared residuals, sums
    // per-call host work reused across kz_solve calls (row-sharded loops call it every iteration):
    // worker streams, weights and the kernel plan
    uint64_t pods_seed = 0;
    int64_t pods_off = -1, pods_q = -1;
    std::vector<double> alphas_cache;
    int64_t plan_key[6] = {-1, -1, -1, -1, -1, -1};
    unsigned char plan_blob[128];  // the cached Plan (trivially copyable)
    bool no_pairs = false;         // CTA-pair clusters not launchable cooperatively on this device
    SolveStatus* h_status = nullptr;  // pinned
    bool norms_valid = false;
    bool bs2_valid = false;
    int64_t bad_row = -1;
    int sampler_scheme = -1;
    int64_t sampler_q = 0;
    std::vector<int64_t> custom_lo, custom_len;  // KZ_SCHEME_RANGES
    bool has_xref = false;
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    // TMA descriptors of A (box = one CTA's column slice) and of the packed (b, sq) pairs
    CUtensorMap tmA{}, tmB{};
    int tm_box = 0;
    const void* tm_a = nullptr;
    const void* tm_b = nullptr;
    // system views (kz_system_view): A, b, x_ref, row norms and packed records alias the base
    // system's; the iterate, sampler, scratch, status and a stream of its own let several
    // solves of one resident system run concurrently
    bool is_view = false;
    kz_system* base = nullptr;          // views: the system whose buffers they alias
    cudaStream_t own_stream = nullptr;  // used when a call passes stream = NULL (views only)
};

// the stream of a call: the caller's, else the system's own (views), else the legacy default stream
static inline cudaStream_t pick_stream(const kz_system* s, void* stream) {
    return stream ? (cudaStream_t)stream : s->own_stream;
}
#define KZ_NOT_VIEW(s) \
    if ((s)->is_view) return fail(KZ_EINVAL, "not allowed on a system view (it shares its base system's matrix)")

extern "C" const char* kz_last_error(void) { return g_err.c_str(); }
extern "C" int32_t kz_version(void) { return 1; }
extern "C" int64_t kz_launch_count(void) { return g_launches.load(); }

extern "C" int32_t kz_device_count(int32_t* count) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *count = 0;
        return fail(KZ_ENODEV, "no CUDA device: %s", cudaGetErrorString(e));
    }
    *count = c;
    return KZ_OK;
}

extern "C" int32_t kz_system_create(int32_t device, int64_t m, int64_t n, kz_system** out) {
    *out = nullptr;
    if (m < 1 || n < 1) return fail(KZ_EINVAL, "matrix dimensions must be >= 1, got (%lld, %lld)", (long long)m, (long long)n);
    if (m > INT32_MAX) return fail(KZ_EINVAL, "m=%lld exceeds the 32-bit row index range", (long long)m);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
        cudaGetLastError();
        return fail(KZ_ENODEV, "no CUDA device available");
    }
    if (device < 0 || device >= ndev) return fail(KZ_EINVAL, "device %d out of range (%d devices)", device, ndev);
    KZ_CUDA(cudaSetDevice(device));
    kz_system* s = new kz_system();
    s->device = device;
    s->m = m;
    s->n = n;
    s->ld = (n + 15) / 16 * 16;  // 128-byte row pitch
    cudaDeviceGetAttribute(&s->sms, cudaDevAttrMultiProcessorCount, device);
    int rc = KZ_OK;
    if ((rc = s->A.ensure((size_t)m * s->ld)) || (rc = s->b.ensure(m)) || (rc = s->xref.ensure(s->ld)) ||
        (rc = s->x.ensure(s->ld)) || (rc = s->sq.ensure(m)) || (rc = s->cdf.ensure(m)) ||
        (rc = s->tmp.ensure(std::max<int64_t>(m, s->ld))) || (rc = s->status.ensure(1)) ||
        (rc = s->barrier.ensure(1)) || (rc = s->zero_row.ensure(1))) {
        kz_system_destroy(s);
        return rc;
    }
    if (cudaMallocHost(&s->h_status, sizeof(SolveStatus)) != cudaSuccess) {
        cudaGetLastError();
        kz_system_destroy(s);
        return fail(KZ_ENOMEM, "pinned status allocation failed");
    }
    for (auto& e : s->ev) cudaEventCreate(&e);
    cudaMemset(s->xref.p, 0, s->ld * sizeof(double));
    cudaMemset(s->x.p, 0, s->ld * sizeof(double));
    *out = s;
    return KZ_OK;
}

extern "C" int32_t kz_system_destroy(kz_system* s) {
    if (!s) return KZ_OK;
    cudaSetDevice(s->device);
    for (auto* b : {&s->A, &s->b, &s->xref, &s->x, &s->sq, &s->cdf, &s->tmp, &s->V, &s->part, &s->ckpt, &s->alphas, &s->bs2,
                    &s->cg, &s->stage, &s->S, &s->errs, &s->xs, &s->tsnap, &s->tr2, &s->tsum})
        b->release();
    s->ll.release();
    s->halt.release();
    s->dbg.release();
    s->lo.release();
    s->len.release();
    s->idx.release();
    s->rows_out.release();
    s->states.release();
    s->barrier.release();
    s->status.release();
    s->zero_row.release();
    if (s->h_status) cudaFreeHost(s->h_status);
    for (auto& e : s->ev)
        if (e) cudaEventDestroy(e);
    if (s->own_stream) cudaStreamDestroy(s->own_stream);
    delete s;
    return KZ_OK;
}

extern "C" int64_t kz_system_pitch(const kz_system* s) { return s ? s->ld : 0; }

static int upload_common(kz_system* s, const double* A, int64_t lda, const double* b, const double* xref,
                         cudaStream_t st, cudaMemcpyKind kind) {
    KZ_NOT_VIEW(s);
    if (lda < s->n) return fail(KZ_EINVAL, "lda=%lld < n=%lld", (long long)lda, (long long)s->n);
    KZ_CUDA(cudaSetDevice(s->device));
    if (kind == cudaMemcpyHostToDevice && lda == s->n && s->ld > s->n) {
        // dense host rows: one 1-D copy at full link speed into staging, then a device
        // repack into the 128-byte row pitch (a pitched 2-D copy of ~4 KB rows runs far
        // below the link rate)
        KZ_TRY(s->stage.ensure((size_t)s->m * s->n));
        KZ_CUDA(cudaMemcpyAsync(s->stage.p, A, (size_t)s->m * s->n * sizeof(double), kind, st));
        const int64_t total = s->m * s->ld;
        repack_rows_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)s->sms * 32), 256, 0, st>>>(
            s->stage.p, s->m, s->n, s->ld, s->A.p);
        KZ_TRY(check_launch("repack_rows_kernel"));
    } else {
        KZ_CUDA(cudaMemcpy2DAsync(s->A.p, s->ld * sizeof(double), A, lda * sizeof(double), s->n * sizeof(double),
                                  s->m, kind, st));
        if (s->ld > s->n)
            KZ_CUDA(cudaMemset2DAsync(s->A.p + s->n, s->ld * sizeof(double), 0, (s->ld - s->n) * sizeof(double), s->m,
                                      st));
    }
    KZ_CUDA(cudaMemcpyAsync(s->b.p, b, s->m * sizeof(double), kind, st));
    if (xref) {
        KZ_CUDA(cudaMemcpyAsync(s->xref.p, xref, s->n * sizeof(double), kind, st));
        s->has_xref = true;
    } else {
        s->has_xref = false;
    }
    s->norms_valid = false;
    s->bs2_valid = false;
    s->sampler_scheme = -1;
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_system_upload(kz_system* s, const double* A, int64_t lda, const double* b, const double* xref,
                                    void* stream) {
    NvtxScope nvtx_("kz_system_upload");
    if (!s || !A || !b) return fail(KZ_EINVAL, "null argument");
    return upload_common(s, A, lda, b, xref, (cudaStream_t)stream, cudaMemcpyHostToDevice);
}

extern "C" int32_t kz_system_upload_device(kz_system* s, const double* A, int64_t lda, const double* b,
                                           const double* xref, void* stream) {
    NvtxScope nvtx_("kz_system_upload_device");
    if (!s || !A || !b) return fail(KZ_EINVAL, "null argument");
    return upload_common(s, A, lda, b, xref, (cudaStream_t)stream, cudaMemcpyDeviceToDevice);
}

extern "C" int32_t kz_system_device_ptrs(kz_system* s, double** A, double** b, double** xref) {
    if (!s) return fail(KZ_EINVAL, "null system");
    if (A) *A = s->A.p;
    if (b) *b = s->b.p;
    if (xref) *xref = s->xref.p;
    s->has_xref = true;
    return KZ_OK;
}

extern "C" int32_t kz_system_set_xref(kz_system* s, const double* xref, void* stream) {
    if (!s || !xref) return fail(KZ_EINVAL, "null argument");
    KZ_NOT_VIEW(s);
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_CUDA(cudaMemcpyAsync(s->xref.p, xref, s->n * sizeof(double), cudaMemcpyHostToDevice, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    s->has_xref = true;
    return KZ_OK;
}

extern "C" int32_t kz_generate_counter(kz_system* s, uint64_t seed, double mu_lo, double mu_hi, double sg_lo,
                                       double sg_hi, void* stream) {
    NvtxScope nvtx_("kz_generate_counter");
    return kz_generate_counter_rows(s, seed, 0, mu_lo, mu_hi, sg_lo, sg_hi, stream);
}

extern "C" int32_t kz_generate_counter_rows(kz_system* s, uint64_t seed, int64_t row0, double mu_lo, double mu_hi,
                                            double sg_lo, double sg_hi, void* stream) {
    NvtxScope nvtx_("kz_generate_counter_rows");
    if (row0 < 0) return fail(KZ_EINVAL, "row0 must be >= 0");
    if (!s) return fail(KZ_EINVAL, "null system");
    KZ_NOT_VIEW(s);
    if (!(sg_lo > 0) || sg_hi < sg_lo || mu_hi < mu_lo) return fail(KZ_EINVAL, "bad generator ranges");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    const int64_t pairs = s->m * (s->ld / 2);
    const unsigned blocks = (unsigned)std::min<int64_t>((pairs + 255) / 256, (int64_t)s->sms * 64);
    gen_counter_kernel<<<blocks, 256, 0, st>>>(s->A.p, s->m, s->n, s->ld, seed, mu_lo, mu_hi, sg_lo, sg_hi, row0);
    KZ_TRY(check_launch("gen_counter_kernel"));
    gen_xstar_kernel<<<(unsigned)((s->ld / 2 + 255) / 256), 256, 0, st>>>(s->xref.p, s->n, s->ld, seed, mu_lo, mu_hi,
                                                                          sg_lo, sg_hi);
    KZ_TRY(check_launch("gen_xstar_kernel"));
    gemv_rows_kernel<<<(unsigned)((s->m + 7) / 8), 256, 0, st>>>(s->A.p, s->xref.p, s->m, s->n, s->ld, s->b.p);
    KZ_TRY(check_launch("gemv_rows_kernel"));
    KZ_CUDA(cudaStreamSynchronize(st));
    s->has_xref = true;
    s->norms_valid = false;
    s->bs2_valid = false;
    s->sampler_scheme = -1;
    return KZ_OK;
}

extern "C" int32_t kz_system_download(kz_system* s, int64_t m2, int64_t n2, double* A_host, double* b_host,
                                      double* xref_host, void* stream) {
    NvtxScope nvtx_("kz_system_download");
    if (!s || m2 < 0 || n2 < 0 || m2 > s->m || n2 > s->n) return fail(KZ_EINVAL, "bad crop");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    if (A_host && m2 > 0 && n2 > 0)
        KZ_CUDA(cudaMemcpy2DAsync(A_host, n2 * sizeof(double), s->A.p, s->ld * sizeof(double), n2 * sizeof(double), m2,
                                  cudaMemcpyDeviceToHost, st));
    if (b_host && m2 > 0) KZ_CUDA(cudaMemcpyAsync(b_host, s->b.p, m2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (xref_host && n2 > 0)
        KZ_CUDA(cudaMemcpyAsync(xref_host, s->xref.p, n2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_system_touch(kz_system* s) {
    if (!s) return fail(KZ_EINVAL, "null system");
    KZ_NOT_VIEW(s);
    s->norms_valid = false;
    s->bs2_valid = false;
    s->sampler_scheme = -1;
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// row norms (linalg.py:80-88)
// ---------------------------------------------------------------------------
static int ensure_norms(kz_system* s, cudaStream_t st) {
    if (s->norms_valid) return s->bad_row >= 0 ? fail(KZ_EDEGENERATE, "row %lld has zero norm; sampling probabilities "
                                                                       "and projection denominators are undefined for "
                                                                       "zero rows", (long long)s->bad_row)
                                               : KZ_OK;
    KZ_CUDA(cudaMemsetAsync(s->zero_row.p, 0xff, sizeof(unsigned long long), st));
    const int64_t blocks = (s->m + NORM_ROWS_PER_CTA - 1) / NORM_ROWS_PER_CTA;
    row_sqnorm_kernel<<<(unsigned)blocks, NORM_ROWS_PER_CTA, 0, st>>>(s->A.p, s->m, s->n, s->ld, s->sq.p, s->zero_row.p);
    KZ_TRY(check_launch("row_sqnorm_kernel"));
    unsigned long long first = 0;
    KZ_CUDA(cudaMemcpyAsync(&first, s->zero_row.p, sizeof(first), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    s->norms_valid = true;
    s->bs2_valid = false;
    s->bad_row = (first == ~0ULL) ? -1 : (int64_t)first;
    s->sampler_scheme = -1;
    if (s->bad_row >= 0)
        return fail(KZ_EDEGENERATE, "row %lld has zero norm; sampling probabilities and projection denominators "
                    "are undefined for zero rows", (long long)s->bad_row);
    return KZ_OK;
}

extern "C" int32_t kz_row_norms_upload(kz_system* s, const double* sq_host, void* stream) {
    if (!s || !sq_host) return fail(KZ_EINVAL, "null argument");
    KZ_NOT_VIEW(s);
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_CUDA(cudaMemcpyAsync(s->sq.p, sq_host, s->m * sizeof(double), cudaMemcpyHostToDevice, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    s->bad_row = -1;
    for (int64_t i = 0; i < s->m; ++i)
        if (sq_host[i] == 0.0) {
            s->bad_row = i;
            break;
        }
    s->norms_valid = true;
    s->bs2_valid = false;
    s->sampler_scheme = -1;
    if (s->bad_row >= 0)
        return fail(KZ_EDEGENERATE, "row %lld has zero norm; sampling probabilities and projection denominators "
                    "are undefined for zero rows", (long long)s->bad_row);
    return KZ_OK;
}

extern "C" int32_t kz_row_norms(kz_system* s, double* sq_host, int64_t* bad_row, void* stream) {
    NvtxScope nvtx_("kz_row_norms");
    if (!s) return fail(KZ_EINVAL, "null system");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    int rc = ensure_norms(s, st);
    if (bad_row) *bad_row = s->bad_row;
    if (sq_host && s->norms_valid) {
        KZ_CUDA(cudaMemcpyAsync(sq_host, s->sq.p, s->m * sizeof(double), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
    }
    return rc;
}

// packed (b_i, ||a_i||^2, RN(1/||a_i||^2), 0) records of every row (after the norms)
static int ensure_bs2(kz_system* s, cudaStream_t st) {
    if (s->bs2_valid) return KZ_OK;
    KZ_TRY(s->bs2.ensure(4 * (size_t)s->m));
    pack_bs2_kernel<<<(unsigned)((s->m + 255) / 256), 256, 0, st>>>(s->b.p, s->sq.p, s->m, s->bs2.p);
    KZ_TRY(check_launch("pack_bs2_kernel"));
    s->bs2_valid = true;
    return KZ_OK;
}

// A view of a resident system for concurrent solves: it aliases the base's matrix, right-hand
// side, reference solution, row norms and packed records (built here first if needed), and owns
// its iterate, samplers, scratch, status words and a CUDA stream.  The base must outlive its
// views and must not be re-uploaded or regenerated while they exist.
extern "C" int32_t kz_system_view(kz_system* base, kz_system** out) {
    if (!base || !out) return fail(KZ_EINVAL, "null argument");
    *out = nullptr;
    if (base->is_view) return fail(KZ_EINVAL, "a view of a view: make views of the base system");
    KZ_CUDA(cudaSetDevice(base->device));
    KZ_TRY(ensure_norms(base, nullptr));
    KZ_TRY(ensure_bs2(base, nullptr));
    KZ_CUDA(cudaStreamSynchronize(nullptr));
    kz_system* v = new kz_system();
    v->device = base->device;
    v->m = base->m;
    v->n = base->n;
    v->ld = base->ld;
    v->sms = base->sms;
    v->A.borrow(base->A);
    v->b.borrow(base->b);
    v->xref.borrow(base->xref);
    v->sq.borrow(base->sq);
    v->bs2.borrow(base->bs2);
    v->norms_valid = true;
    v->bad_row = base->bad_row;
    v->bs2_valid = true;
    v->has_xref = base->has_xref;
    v->no_pairs = base->no_pairs;
    v->is_view = true;
    v->base = base;
    int rc = KZ_OK;
    if ((rc = v->x.ensure(v->ld)) || (rc = v->cdf.ensure(v->m)) || (rc = v->tmp.ensure(std::max<int64_t>(v->m, v->ld))) ||
        (rc = v->status.ensure(1)) || (rc = v->barrier.ensure(1)) || (rc = v->zero_row.ensure(1))) {
        kz_system_destroy(v);
        return rc;
    }
    if (cudaMallocHost(&v->h_status, sizeof(SolveStatus)) != cudaSuccess ||
        cudaStreamCreate(&v->own_stream) != cudaSuccess) {
        cudaGetLastError();
        kz_system_destroy(v);
        return fail(KZ_ENOMEM, "view allocation failed");
    }
    for (auto& e : v->ev) cudaEventCreate(&e);
    cudaMemset(v->x.p, 0, v->ld * sizeof(double));
    *out = v;
    return KZ_OK;
}

// After the base was re-uploaded or regenerated: rebuild its norms and packed records, and
// drop the view's samplers built from the old norms (no allocation: the buffers stay aliased).
extern "C" int32_t kz_system_view_refresh(kz_system* v) {
    if (!v || !v->is_view || !v->base) return fail(KZ_EINVAL, "not a system view");
    kz_system* base = v->base;
    KZ_CUDA(cudaSetDevice(base->device));
    const int rc = ensure_norms(base, nullptr);
    if (rc != KZ_OK && rc != KZ_EDEGENERATE) return rc;
    if (rc == KZ_OK) KZ_TRY(ensure_bs2(base, nullptr));
    KZ_CUDA(cudaStreamSynchronize(nullptr));
    v->norms_valid = true;
    v->bad_row = base->bad_row;
    v->bs2_valid = base->bs2_valid;
    v->has_xref = base->has_xref;
    v->sampler_scheme = -1;
    v->sampler_q = 0;
    return rc;
}

// ---------------------------------------------------------------------------
// samplers (sampling.py:101-131, solvers.py:162-171)
// ---------------------------------------------------------------------------
static int ensure_sampler(kz_system* s, int scheme, int64_t q, cudaStream_t st) {
    KZ_TRY(ensure_norms(s, st));
    if (scheme != KZ_FULL_ACCESS && scheme != KZ_DISTRIBUTED && scheme != KZ_SCHEME_RANGES)
        return fail(KZ_EINVAL, "unknown sampling scheme %d", scheme);
    if (scheme == KZ_SCHEME_RANGES && (int64_t)s->custom_lo.size() != q)
        return fail(KZ_EINVAL, "explicit ranges were set for %zu workers, not q=%lld", s->custom_lo.size(), (long long)q);
    if (q < 1) return fail(KZ_EINVAL, "q must be >= 1, got %lld", (long long)q);
    if (s->sampler_scheme == scheme && (scheme == KZ_FULL_ACCESS || s->sampler_q == q)) {
        if (scheme == KZ_FULL_ACCESS && s->sampler_q != q) {
            // full access: one range replicated per worker
            std::vector<int64_t> lo(q, 0), len(q, s->m);
            KZ_TRY(s->lo.ensure(q));
            KZ_TRY(s->len.ensure(q));
            KZ_CUDA(cudaMemcpyAsync(s->lo.p, lo.data(), q * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            KZ_CUDA(cudaMemcpyAsync(s->len.p, len.data(), q * sizeof(int64_t), cudaMemcpyHostToDevice, st));
            KZ_CUDA(cudaStreamSynchronize(st));
            s->sampler_q = q;
        }
        return KZ_OK;
    }
    std::vector<int64_t> lo(q), len(q);
    int64_t nranges;
    if (scheme == KZ_FULL_ACCESS) {
        std::fill(lo.begin(), lo.end(), 0);
        std::fill(len.begin(), len.end(), s->m);
        nranges = 1;
    } else if (scheme == KZ_SCHEME_RANGES) {
        lo = s->custom_lo;
        len = s->custom_len;
        nranges = q;
    } else {
        for (int64_t t = 0; t < q; ++t) {
            const int64_t a = (t * s->m) / q, b = ((t + 1) * s->m) / q - 1;
            if (b < a) return fail(KZ_EEMPTYRANGE, "block %lld of %lld is empty for m=%lld", (long long)t, (long long)q,
                                   (long long)s->m);
            lo[t] = a;
            len[t] = b - a + 1;
        }
        nranges = q;
    }
    KZ_TRY(s->lo.ensure(q));
    KZ_TRY(s->len.ensure(q));
    KZ_CUDA(cudaMemcpyAsync(s->lo.p, lo.data(), q * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    KZ_CUDA(cudaMemcpyAsync(s->len.p, len.data(), q * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    cdf_scan_kernel<<<(unsigned)nranges, CDF_SCAN_THREADS, 0, st>>>(s->sq.p, s->lo.p, s->len.p, nranges, s->cdf.p);
    KZ_TRY(check_launch("cdf_scan_kernel"));
    const int64_t maxlen = *std::max_element(len.begin(), len.end());
    dim3 grid((unsigned)std::min<int64_t>((maxlen + 255) / 256, 1024), (unsigned)nranges);
    cdf_div_kernel<<<grid, 256, 0, st>>>(s->cdf.p, s->lo.p, s->len.p);
    KZ_TRY(check_launch("cdf_div_kernel"));
    cdf_div_last_kernel<<<(unsigned)((nranges + 127) / 128), 128, 0, st>>>(s->cdf.p, s->lo.p, s->len.p, nranges);
    KZ_TRY(check_launch("cdf_div_last_kernel"));
    KZ_CUDA(cudaStreamSynchronize(st));
    s->sampler_scheme = scheme;
    s->sampler_q = q;
    return KZ_OK;
}

extern "C" int32_t kz_sampler_set_ranges(kz_system* s, int64_t q, const int64_t* lo, const int64_t* len, void* stream) {
    if (!s || !lo || !len || q < 1) return fail(KZ_EINVAL, "bad ranges");
    std::vector<int64_t> l(lo, lo + q), n(len, len + q);
    for (int64_t t = 0; t < q; ++t)
        if (n[t] < 1 || l[t] < 0 || l[t] + n[t] > s->m)
            return fail(KZ_EEMPTYRANGE, "row range [%lld, %lld) invalid for m=%lld", (long long)l[t],
                        (long long)(l[t] + n[t]), (long long)s->m);
    s->custom_lo = l;
    s->custom_len = n;
    if (s->sampler_scheme == KZ_SCHEME_RANGES) s->sampler_scheme = -1;
    (void)stream;
    return KZ_OK;
}

extern "C" int32_t kz_sampler_build(kz_system* s, int32_t scheme, int64_t q, double* cdf_host, void* stream) {
    NvtxScope nvtx_("kz_sampler_build");
    if (!s) return fail(KZ_EINVAL, "null system");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_TRY(ensure_sampler(s, scheme, q, st));
    if (cdf_host) {
        KZ_CUDA(cudaMemcpyAsync(cdf_host, s->cdf.p, s->m * sizeof(double), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
    }
    return KZ_OK;
}

static int launch_sampler(kz_system* s, const PcgPod* states_dev, const int64_t* lo, const int64_t* len, int64_t q,
                          int64_t d0, int64_t count, int32_t* out, int64_t stride_w, int64_t stride_d, cudaStream_t st) {
    const int64_t runs = (count + SAMPLE_RUN - 1) / SAMPLE_RUN;
    const int64_t threads = runs * q;
    const int64_t blocks = std::max<int64_t>(1, std::min<int64_t>((threads + 255) / 256, (int64_t)s->sms * 16));
    sample_rows_kernel<<<(unsigned)blocks, 256, 0, st>>>(s->cdf.p, lo, len, states_dev, q, d0, count, out, stride_w,
                                                         stride_d);
    return check_launch("sample_rows_kernel");
}

extern "C" int32_t kz_dump_rows(kz_system* s, int32_t scheme, int64_t q, uint64_t seed, int64_t worker, int64_t start,
                                int64_t count, int32_t* out_host, void* stream) {
    NvtxScope nvtx_("kz_dump_rows");
    if (!s || !out_host) return fail(KZ_EINVAL, "null argument");
    if (worker < 0 || worker >= q) return fail(KZ_EINVAL, "worker %lld out of range for q=%lld", (long long)worker, (long long)q);
    if (start < 0 || count < 0) return fail(KZ_EINVAL, "negative range");
    if (count == 0) return KZ_OK;
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_TRY(ensure_sampler(s, scheme, q, st));
    KZ_TRY(s->states.ensure(std::max<int64_t>(q, 1)));
    s->pods_q = -1;  // kz_solve's cached worker streams are overwritten below
    PcgPod pod = seed_stream(seed, (uint64_t)worker);
    KZ_CUDA(cudaMemcpyAsync(s->states.p, &pod, sizeof(pod), cudaMemcpyHostToDevice, st));
    KZ_TRY(s->rows_out.ensure(count));
    KZ_TRY(launch_sampler(s, s->states.p, s->lo.p + worker, s->len.p + worker, 1, start, count, s->rows_out.p, 0, 1, st));
    KZ_CUDA(cudaMemcpyAsync(out_host, s->rows_out.p, count * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// norms for traces / reports
// ---------------------------------------------------------------------------
static int device_norms(kz_system* s, const double* xdev, double* residual, double* error, cudaStream_t st) {
    // both sums land in part[0..1] and come back with one copy and one host sync (a trace
    // record costs one round trip, not two)
    double h[2] = {NAN, NAN};
    if (residual) {
        const int rows_per_cta = 8;
        residual_rows_kernel<<<(unsigned)((s->m + rows_per_cta - 1) / rows_per_cta), rows_per_cta * 32, 0, st>>>(
            s->A.p, s->b.p, xdev, s->m, s->n, s->ld, s->tmp.p);
        KZ_TRY(check_launch("residual_rows_kernel"));
        sum_kernel<<<1, 1024, 0, st>>>(s->tmp.p, s->m, s->part.p);
        KZ_TRY(check_launch("sum_kernel"));
    }
    if (error) {
        // tmp is reused: stream order puts this after the residual sum has consumed it
        diff_sq_kernel<<<(unsigned)((s->n + 255) / 256), 256, 0, st>>>(xdev, s->xref.p, s->n, s->tmp.p);
        KZ_TRY(check_launch("diff_sq_kernel"));
        sum_kernel<<<1, 1024, 0, st>>>(s->tmp.p, s->n, s->part.p + 1);
        KZ_TRY(check_launch("sum_kernel"));
    }
    if (residual || error) {
        KZ_CUDA(cudaMemcpyAsync(h, s->part.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
    }
    if (residual) *residual = std::sqrt(h[0]);
    if (error) *error = std::sqrt(h[1]);
    return KZ_OK;
}

extern "C" int32_t kz_norms(kz_system* s, const double* x_host, double* residual, double* error, void* stream) {
    NvtxScope nvtx_("kz_norms");
    if (!s || !x_host) return fail(KZ_EINVAL, "null argument");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_TRY(s->part.ensure(16));
    KZ_TRY(s->V.ensure(s->ld));
    KZ_CUDA(cudaMemsetAsync(s->V.p, 0, s->ld * sizeof(double), st));
    KZ_CUDA(cudaMemcpyAsync(s->V.p, x_host, s->n * sizeof(double), cudaMemcpyHostToDevice, st));
    return device_norms(s, s->V.p, residual, error, st);
}

static int error_sq_dev(kz_system* s, double* out, cudaStream_t st) {
    KZ_TRY(s->part.ensure(16));
    diff_sq_kernel<<<(unsigned)((s->n + 255) / 256), 256, 0, st>>>(s->x.p, s->xref.p, s->n, s->tmp.p);
    KZ_TRY(check_launch("diff_sq_kernel"));
    sum_kernel<<<1, 1024, 0, st>>>(s->tmp.p, s->n, s->part.p);
    KZ_TRY(check_launch("sum_kernel"));
    KZ_CUDA(cudaMemcpyAsync(out, s->part.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_error_sq(kz_system* s, double* err_host, void* stream) {
    if (!s || !err_host) return fail(KZ_EINVAL, "null argument");
    KZ_CUDA(cudaSetDevice(s->device));
    return error_sq_dev(s, err_host, pick_stream(s, stream));
}

extern "C" int32_t kz_average_from(kz_system* s, const double* S_dev, int64_t Q, double* err_host, void* stream) {
    if (!s || !S_dev || Q < 1) return fail(KZ_EINVAL, "bad arguments");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    scale_copy_kernel<<<(unsigned)((s->ld + 255) / 256), 256, 0, st>>>(S_dev, (double)Q, s->ld, s->x.p);
    KZ_TRY(check_launch("scale_copy_kernel"));
    if (err_host) return error_sq_dev(s, err_host, st);
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_solution_host(kz_system* s, double* x_host, void* stream) {
    if (!s || !x_host) return fail(KZ_EINVAL, "null argument");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_CUDA(cudaMemcpyAsync(x_host, s->x.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_set_x(kz_system* s, const double* x_host, void* stream) {
    if (!s) return fail(KZ_EINVAL, "null system");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_CUDA(cudaMemsetAsync(s->x.p, 0, s->ld * sizeof(double), st));
    if (x_host) KZ_CUDA(cudaMemcpyAsync(s->x.p, x_host, s->n * sizeof(double), cudaMemcpyHostToDevice, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}

extern "C" int32_t kz_solution_device(kz_system* s, double** x_dev) {
    if (!s || !x_dev) return fail(KZ_EINVAL, "null argument");
    *x_dev = s->x.p;
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// solve driver
// ---------------------------------------------------------------------------
namespace {

struct Plan {
    int kernel = KZ_KERNEL_CHAIN;
    int rows = 1;       // chain: rows per CTA reduction (R)
    int pair = 1;       // chain: CTAs per worker (cluster of 1 or 2)
    int threads = 256;
    int ctas = 1;
    int stages = 2;
    int ep = 1;         // chain: pairs per thread
    int lpr = 8;        // sync: lanes per row
    int cluster = 1;    // sync (cluster mode): CTAs per thread-block cluster
    bool tma = false;   // sync: the TMA-gather rka kernel
    int lg = 32, epl = 1, box = 0;  // rka kernel: lanes per row group, pairs per lane, TMA box width
    bool sr = false;    // rka kernel: single round of 8 rows per warp (<= 64 workers per cluster)
    bool wg = false;    // rka kernel: worker groups (cluster g runs q/G workers over all columns)
    bool xr = false;    // rka kernel: cross-rank column sums (set per launch by kz_solve_sharded, not planned)
    bool delta = false; // chain: the threaded engine's RKA increments (chain_kernel<..., DELTA = true>)
    int waves = 1;      // chain: launches per outer iteration when the workers exceed the co-resident CTAs
    bool wide = false;  // chain: averaged workers of 4 CTAs (chain_kernel<..., WIDE = true>)
    size_t smem = 0;
};

const int kChainEP[] = {1, 2, 4, 8, 16};
int chain_max_threads(int ep) { return ep <= 8 ? 128 : 320; }  // compute threads (kz_chain.cu ChainMaxThreads)

int chain_nv(int R) { return R + R * (R - 1) / 2 + R + 1; }

// ldr: the ring row pitch, 2 EP T columns (kz_chain.cu)
int chain_smem(int64_t ldr, int stages, int R, int T, int C = 2) {
    return (int)(288 + (2 * std::max(C, 1) * chain_nv(R) + 2) * sizeof(double) + stages * ldr * sizeof(double) +
                 stages * 2 * sizeof(double) + IDX_WINDOW * sizeof(int32_t) +
                 ((size_t)chain_nv(R) * T + chain_nv(R) + 1) * sizeof(double));
}

size_t sync_smem(int64_t q, int64_t cw, int stages, int P, bool cluster) {
    const int nwarp = 256 / 32, seg_max = 64;
    const int64_t rs = cw + 2, q1p = (q + 2) & ~(int64_t)1;
    return 16 + (size_t)stages * q * rs * sizeof(double) + (size_t)stages * q * 2 * sizeof(double) +
           2 * cw * sizeof(double) + (cluster ? 2 * (size_t)P * q1p * sizeof(double) : 0) +
           (size_t)nwarp * cw * sizeof(double) + (size_t)nwarp * seg_max * sizeof(double) +
           nwarp * sizeof(double) + q * sizeof(double) + 8 * q * sizeof(int32_t);
}

void* rkw_fn(int epl) {
    return epl == 1 ? (void*)rkw_kernel<1, 8> : epl == 2 ? (void*)rkw_kernel<2, 8> : (void*)rkw_kernel<4, 8>;
}

void* chain_fn(int ep, int R, int C, bool delta = false, bool wide = false) {
    if (wide) {  // averaged workers on clusters of 4 (RKAB rows beyond a pair's reach)
        switch (C * 10000 + ep * 100 + R) {
            case 40801: return (void*)chain_kernel<8, 1, 4, false, true>;
            case 40802: return (void*)chain_kernel<8, 2, 4, false, true>;
            case 41601: return (void*)chain_kernel<16, 1, 4, false, true>;
            case 80801: return (void*)chain_kernel<8, 1, 8, false, true>;
            case 80802: return (void*)chain_kernel<8, 2, 8, false, true>;
            case 81601: return (void*)chain_kernel<16, 1, 8, false, true>;
            default: return nullptr;
        }
    }
    if (delta) {  // the threaded engine's RKA (one CTA per worker)
        switch (C * 10000 + ep * 100 + R) {
            case 10101: return (void*)chain_kernel<1, 1, 1, true>;
            case 10104: return (void*)chain_kernel<1, 4, 1, true>;
            case 10201: return (void*)chain_kernel<2, 1, 1, true>;
            case 10204: return (void*)chain_kernel<2, 4, 1, true>;
            case 10401: return (void*)chain_kernel<4, 1, 1, true>;
            case 10402: return (void*)chain_kernel<4, 2, 1, true>;
            case 10404: return (void*)chain_kernel<4, 4, 1, true>;
            case 10801: return (void*)chain_kernel<8, 1, 1, true>;
            case 10802: return (void*)chain_kernel<8, 2, 1, true>;
            case 11601: return (void*)chain_kernel<16, 1, 1, true>;
            default: return nullptr;
        }
    }
    switch (C * 10000 + ep * 100 + R) {
        case 10101: return (void*)chain_kernel<1, 1, 1>;
        case 10104: return (void*)chain_kernel<1, 4, 1>;
        case 10201: return (void*)chain_kernel<2, 1, 1>;
        case 10204: return (void*)chain_kernel<2, 4, 1>;
        case 10401: return (void*)chain_kernel<4, 1, 1>;
        case 10402: return (void*)chain_kernel<4, 2, 1>;
        case 10404: return (void*)chain_kernel<4, 4, 1>;
        case 10801: return (void*)chain_kernel<8, 1, 1>;
        case 10802: return (void*)chain_kernel<8, 2, 1>;
        case 11601: return (void*)chain_kernel<16, 1, 1>;
        case 20104: return (void*)chain_kernel<1, 4, 2>;
        case 20204: return (void*)chain_kernel<2, 4, 2>;
        case 20402: return (void*)chain_kernel<4, 2, 2>;
        case 20404: return (void*)chain_kernel<4, 4, 2>;
        case 20801: return (void*)chain_kernel<8, 1, 2>;
        case 20802: return (void*)chain_kernel<8, 2, 2>;
        case 21601: return (void*)chain_kernel<16, 1, 2>;
        case 40104: return (void*)chain_kernel<1, 4, 4>;
        case 40204: return (void*)chain_kernel<2, 4, 4>;
        case 40404: return (void*)chain_kernel<4, 4, 4>;
        case 40801: return (void*)chain_kernel<8, 1, 4>;
        case 40802: return (void*)chain_kernel<8, 2, 4>;
        case 41601: return (void*)chain_kernel<16, 1, 4>;
        case 80104: return (void*)chain_kernel<1, 4, 8>;
        case 80204: return (void*)chain_kernel<2, 4, 8>;
        case 80801: return (void*)chain_kernel<8, 1, 8>;
        case 80802: return (void*)chain_kernel<8, 2, 8>;
        case 81601: return (void*)chain_kernel<16, 1, 8>;
        default: return nullptr;
    }
}

void* sync_fn(bool cluster, int lpr) {
    if (cluster) return lpr == 4 ? (void*)sync_kernel<true, 4> : lpr == 8 ? (void*)sync_kernel<true, 8>
                                                                          : (void*)sync_kernel<true, 32>;
    return lpr == 4 ? (void*)sync_kernel<false, 4> : lpr == 8 ? (void*)sync_kernel<false, 8>
                                                              : (void*)sync_kernel<false, 32>;
}

constexpr size_t kSmemLimit = 227 * 1024;
constexpr int MAXG_CLUSTERS = 10;  // = MAXG in kz_sync.cu

}  // namespace

// Chain-kernel plan for a worker of C CTAs (a thread-block cluster of C column slices).
static int plan_chain_c(kz_system* s, const kz_params* p, int64_t q, int C, Plan& pl) {
    pl.wide = q > 1 && C >= 4;
    const int64_t pairs = s->ld / 2 / C;
    auto round32 = [](int64_t t) { return (int)std::max<int64_t>(32, (t + 31) / 32 * 32); };
    int ep = 0, T = 0;
    if (p->threads > 0) {
        T = round32(p->threads);
        for (int e : kChainEP)
            if ((int64_t)e * T >= pairs) {
                ep = e;
                break;
            }
    } else {
        for (int e : kChainEP) {
            ep = e;
            T = round32((pairs + e - 1) / e);
            if (T <= 128) break;  // fewer warps per CTA reduction (c2: 207 -> 200 us per outer iteration)
        }
    }
    if (ep == 0 || T > chain_max_threads(ep) || (int64_t)ep * T < pairs)
        return fail(KZ_EINVAL, "n=%lld too large for the chain kernel", (long long)s->n);
    // rows per reduction: as many as registers allow (EP small) and the ring holds (> R rows)
    int R = ep <= 4 ? 4 : (ep == 8 ? 2 : 1);  // R = 8 measured slower since the reduction got cheap (not built)
    if (C == 2) R = std::min(R, 4);
    if (C > 2) R = std::min(R, 4);
    if (const char* e = dbg_env("KZ_CHAIN_ROWS")) R = std::max(1, atoi(e));
    const int64_t ldr = ep < 16 ? 2 * (int64_t)ep * T : s->ld / C;  // ring row pitch (kz_chain.cu PADDED)
    const int64_t stage_bytes = ldr * (int64_t)sizeof(double);
    int stages = 0;
    for (;;) {
        while (R > 1 && !chain_fn(ep, R, C, pl.delta, pl.wide)) R /= 2;
        const int64_t fixed = chain_smem(ldr, 0, R, T, C);
        stages = (int)std::min<int64_t>(16, ((int64_t)200 * 1024 - fixed) / stage_bytes);
        if (const char* e = dbg_env("KZ_CHAIN_STAGES")) stages = std::min(16, atoi(e));
        if (stages >= R + 1 || R == 1) break;
        R = R > 4 ? 4 : (R > 2 ? 2 : 1);
    }
    if (stages < 1 || (size_t)chain_smem(ldr, stages, R, T, C) > kSmemLimit)
        return fail(KZ_EINVAL, "row of n=%lld does not fit the shared-memory ring", (long long)s->n);
    void* fn = chain_fn(ep, R, C, pl.delta, pl.wide);
    // the instantiations carry one driver each for these shapes (kz_chain.cu ONE_CHAIN / AVERAGED)
    if (q == 1 && C == 2 && ep >= 8)
        return fail(KZ_EINVAL, "no chain kernel drives q=%lld on %d-CTA workers with EP=%d", (long long)q, C, ep);
    if (!fn) return fail(KZ_EINVAL, "no chain kernel for EP=%d R=%d C=%d", ep, R, C);
    pl.kernel = KZ_KERNEL_CHAIN;
    pl.threads = T + 32;  // + the producer warp
    pl.ep = ep;
    pl.rows = R;
    pl.pair = C;
    pl.stages = stages;
    pl.smem = chain_smem(ldr, stages, R, T, C);
    pl.ctas = (int)(q * C);
    KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    pl.waves = 1;
    if (pl.ctas > 1) {
        int per_sm = 0;
        KZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, T + 32, pl.smem));
        const int64_t cap = (int64_t)per_sm * s->sms / C;  // co-resident workers
        if (cap * C < pl.ctas) {
            // more workers than co-resident CTAs: each outer iteration runs its workers in waves of
            // at most `cap`, every wave adding its ordered worker sum to the previous waves'
            // (the per-iteration driver, kz_solve_sharded's loop); waves of one worker would take
            // the single-chain path, so every wave keeps at least two
            const int64_t W = (q + cap - 1) / std::max<int64_t>(cap, 1);
            if (cap < 2 || q / W < 2 || pl.delta || p->variant == KZ_CK)
                return fail(KZ_EINVAL, "q=%lld workers exceed the %lld co-resident workers of the chain kernel",
                            (long long)q, (long long)cap);
            pl.waves = (int)W;
            pl.ctas = (int)((q + W - 1) / W * C);
        }
    }
    return KZ_OK;
}

// A worker is one CTA, or a cluster of C CTAs each owning ld / C columns: a pair when the rows
// are long and the pairs fit the SMs, 4 for one long chain (RK, CK).  When the preferred width
// has no kernel for the row length (the EP x R x C instantiations in kz_chain.cu) or does not
// fit, narrower clusters are tried, so every n up to the chain kernel's limit is accepted:
// 16 pairs x 320 threads x 2 columns per CTA, i.e. n <= 10240 C (C = 1, 2, or 4 for q = 1).
static int plan_chain(kz_system* s, const kz_params* p, int64_t q, Plan& pl) {
    int C = (s->ld >= 1024 && 2 * q <= s->sms && !s->no_pairs) ? 2 : 1;  // measured: pairs win from n ~ 1000
    if (pl.delta) C = 1;  // the threaded engine's RKA runs on one CTA per worker (its own instantiations)
    // one chain (RK, CK) over long rows: a cluster of 4 (measured on 80000 x 2000 with the
    // producer warp: 0.40 us per row against 0.42 for 8 CTAs and 0.45 for a pair; at n = 512
    // the pair is best)
    if (q == 1 && s->ld >= 1536 && !s->no_pairs) C = 4;
    if (const char* e = dbg_env("KZ_CHAIN_PAIR")) {  // experiment: 1, 2, or (one chain, q = 1) 4 / 8
        const int want = atoi(e);
        C = want == 2 && 2 * q <= s->sms ? 2 : ((want == 4 || want == 8) && q == 1 ? want : 1);
    }
    int rc = KZ_EINVAL;
    std::string first_err;
    // the preferred width, narrower ones, then (workers averaged over long rows) pairs in waves
    int cand[6], nc = 0;
    for (int c = C; c >= 1; c /= 2) cand[nc++] = c;
    if (q > 1 && C < 2 && !pl.delta) cand[nc++] = 2;
    if (q > 1 && !pl.delta) cand[nc++] = 4;  // rows beyond a pair's reach: workers of 4 CTAs (in waves)
    if (!pl.delta) cand[nc++] = 8;           // and of 8 CTAs (one chain, or averaged workers in waves)
    for (int i = 0; i < nc; ++i) {
        const int c = cand[i];
        if (c > 1 && (s->ld % (2 * c) != 0 || s->no_pairs)) continue;  // whole 16-byte pairs
        if (c > 1 && i == 0 && c * q > s->sms) continue;  // preferred pairs: only without waves
        rc = plan_chain_c(s, p, q, c, pl);
        if (rc == KZ_OK) return KZ_OK;
        if (first_err.empty()) first_err = g_err;
    }
    return fail(rc, "%s", first_err.empty() ? "no chain-kernel plan" : first_err.c_str());
}

static int plan_sync(kz_system* s, const kz_params* p, int64_t q, bool cluster, Plan& pl) {
    pl.threads = 256;
    if (q > 512) return fail(KZ_EINVAL, "q=%lld exceeds the sync kernel's 512 workers", (long long)q);
    // cluster mode: G clusters of Pc CTAs (column slices over all G*Pc CTAs);
    // grid mode: P CTAs behind a grid barrier
    int Pc = 16, G = 1, P = 0;
    if (cluster) {
        if (p->ctas > 16) {
            G = p->ctas / 16;
        } else if (p->ctas > 0) {
            Pc = p->ctas;
        } else {
            // several clusters once every CTA of one cluster would carry > 128 columns
            G = (int)std::max<int64_t>(1, std::min<int64_t>(MAXG_CLUSTERS, s->ld / (16 * 128)));
        }
        if (const char* e = dbg_env("KZ_SYNC_CLUSTERS")) G = std::max(1, std::min(MAXG_CLUSTERS, atoi(e)));
    } else {
        P = p->ctas > 0 ? p->ctas : s->sms;
    }
    // grow G / P until the slice ring fits; shrink until the launch is schedulable
    for (;;) {
        if (cluster) P = Pc * G;
        if (P < 1 || Pc < 1) return fail(KZ_EINVAL, "no feasible sync-kernel configuration for q=%lld n=%lld",
                                         (long long)q, (long long)s->n);
        const int64_t cw = (((s->ld + P - 1) / P) + 1) & ~(int64_t)1;
        int stages = 4;
        while (stages > 2 && sync_smem(q, cw, stages, cluster ? Pc : P, cluster) > 200 * 1024) --stages;
        if (sync_smem(q, cw, stages, cluster ? Pc : P, cluster) > kSmemLimit) {
            if (cluster) {
                if (G >= MAXG_CLUSTERS || Pc < 16)
                    return fail(KZ_EINVAL, "q=%lld row slices do not fit the cluster CTAs", (long long)q);
                ++G;
                continue;
            }
            if (P >= 4 * s->sms) return fail(KZ_EINVAL, "q=%lld too large for the sync kernel", (long long)q);
            P *= 2;  // thinner slices, several CTAs per SM
            continue;
        }
        pl.stages = stages;
        pl.smem = sync_smem(q, cw, stages, cluster ? Pc : P, cluster);
        pl.lpr = cw > 64 ? 32 : (q > 32 ? 4 : 8);
        void* fn = sync_fn(cluster, pl.lpr);
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        if (cluster) {
            KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(P);
            cfg.blockDim = dim3(pl.threads);
            cfg.dynamicSmemBytes = pl.smem;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = Pc;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            int nclusters = 0;
            cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
            if (e != cudaSuccess || nclusters < 1) {
                cudaGetLastError();
                if (Pc == 1) return fail(KZ_EINVAL, "cluster kernel not schedulable");
                Pc /= 2;
                continue;
            }
            if (nclusters < G) {  // every cluster must be co-resident (they poll each other)
                G = nclusters;
                continue;
            }
        } else {
            int per_sm = 0;
            KZ_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, pl.threads, pl.smem));
            if ((int64_t)per_sm * s->sms < P) {
                if (p->ctas > 0)
                    return fail(KZ_EINVAL, "%d CTAs exceed co-residency (%d per SM)", P, per_sm);
                P = per_sm * s->sms;
                continue;
            }
        }
        pl.kernel = cluster ? KZ_KERNEL_SYNC_CLUSTER : KZ_KERNEL_SYNC_GRID;
        pl.ctas = P;
        pl.cluster = cluster ? Pc : 1;
        return KZ_OK;
    }
}

namespace {

template <bool TM, bool SR, int MODE>
void* rka_fn_t(int lg, int epl) {
    if (lg == 8) return epl == 2 ? (void*)rka_kernel<8, 2, TM, SR, MODE> : (void*)rka_kernel<8, 1, TM, SR, MODE>;
    if (lg == 16) return (void*)rka_kernel<16, 1, TM, SR, MODE>;
    switch (epl) {
        case 1: return (void*)rka_kernel<32, 1, TM, SR, MODE>;
        case 2: return (void*)rka_kernel<32, 2, TM, SR, MODE>;
        case 3: return (void*)rka_kernel<32, 3, TM, SR, MODE>;
        case 4: return (void*)rka_kernel<32, 4, TM, SR, MODE>;
        default: return nullptr;
    }
}

// the timing variant (per-phase clock stamps) only under KZ_PHASE_TIMING (column-sliced plans);
// SR = one round of 8 rows per warp (<= 64 workers per cluster); mode 1 = worker groups,
// mode 2 = cross-rank column sums (kz_solve_sharded)
void* rka_fn(int lg, int epl, bool sr, int mode = 0) {
    if (mode == 1) return sr ? rka_fn_t<false, true, 1>(lg, epl) : rka_fn_t<false, false, 1>(lg, epl);
    if (mode == 2) return sr ? rka_fn_t<false, true, 2>(lg, epl) : rka_fn_t<false, false, 2>(lg, epl);
    const bool tm = dbg_env("KZ_PHASE_TIMING") != nullptr;
    if (tm) return sr ? rka_fn_t<true, true, 0>(lg, epl) : rka_fn_t<true, false, 0>(lg, epl);
    return sr ? rka_fn_t<false, true, 0>(lg, epl) : rka_fn_t<false, false, 0>(lg, epl);
}

size_t rka_smem(int64_t q, int box, int stages, int Pc) {
    const int64_t q4 = (q + 3) & ~(int64_t)3;
    const int64_t rpo = (((q + Pc - 1) / Pc) + 1) & ~(int64_t)1;
    const int64_t rpo4 = (rpo + 3) & ~(int64_t)3;
    const size_t stage = (size_t)q4 * box * sizeof(double) + (size_t)rpo4 * 32;
    return 256 + (size_t)stages * stage +
           (size_t)(2 * Pc * rpo + 2 * q4 + 2 * Pc + 2 + rpo + RKA_NW * box + 2 * box + q) * sizeof(double) +
           (size_t)q * sizeof(int32_t);
}

typedef CUresult (*TmapEncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

TmapEncodeFn tmap_encode() {
    static TmapEncodeFn fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &qr) == cudaSuccess &&
            qr == cudaDriverEntryPointSuccess)
            fn = (TmapEncodeFn)ptr;
        else
            cudaGetLastError();
    }
    return fn;
}

}  // namespace

// Tensor maps for the rka kernel: A as (columns = ld, rows = m) with a box of
// `box` columns x 1 row (gather4 fetches 4 rows per instruction); the packed
// (b_i, ||a_i||^2, 1/||a_i||^2, 0) records as (4, m) with a 4 x 1 box.
static int ensure_tmaps(kz_system* s, int box) {
    if (s->tm_box == box && s->tm_a == s->A.p && s->tm_b == s->bs2.p) return KZ_OK;
    TmapEncodeFn enc = tmap_encode();
    if (!enc) return fail(KZ_ECUDA, "cuTensorMapEncodeTiled unavailable");
    const cuuint32_t es[2] = {1, 1};
    {
        const cuuint64_t dims[2] = {(cuuint64_t)s->ld, (cuuint64_t)s->m};
        const cuuint64_t strides[1] = {(cuuint64_t)s->ld * sizeof(double)};
        const cuuint32_t bx[2] = {(cuuint32_t)box, 1};
        CUresult r = enc(&s->tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)s->A.p, dims, strides, bx, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(KZ_ECUDA, "tensor map of A failed (%d)", (int)r);
    }
    {
        const cuuint64_t dims[2] = {4, (cuuint64_t)s->m};
        const cuuint64_t strides[1] = {4 * sizeof(double)};
        const cuuint32_t bx[2] = {4, 1};
        CUresult r = enc(&s->tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, (void*)s->bs2.p, dims, strides, bx, es,
                         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(KZ_ECUDA, "tensor map of (b, sq) failed (%d)", (int)r);
    }
    s->tm_box = box;
    s->tm_a = s->A.p;
    s->tm_b = s->bs2.p;
    return KZ_OK;
}

// rka kernel plan: G clusters of Pc CTAs; every CTA's slice <= 256 columns (one
// TMA box) and at least two ring stages.
// Worker-group plan (q > 64, rows narrow enough for one cluster's 16 TMA boxes):
// G clusters of 16 CTAs, cluster g runs workers [g q/G, (g+1) q/G) over all
// columns, so each CTA gathers ~q/G row slices per iteration instead of q
// (the column-sliced plan needs G x 16 slices of ~n/(16 G) columns and is
// bound by the TMA unit's per-gather cost); the clusters add their column sums
// through tagged words once per iteration.
static int plan_rka_wg(kz_system* s, const kz_params* p, int64_t q, Plan& pl) {
    const int64_t ld = s->ld;
    const int Pc = 16;
    const int64_t cw = (((ld + Pc - 1) / Pc) + 1) & ~(int64_t)1;
    const int box = (int)((cw + 3) & ~(int64_t)3);
    if (box > 256) return fail(KZ_EINVAL, "rows too wide for worker groups");
    const int npairs = box / 2;
    const int lg = npairs <= 8 ? 8 : (npairs <= 16 ? 16 : 32);
    const int epl = lg == 32 ? (npairs + 31) / 32 : 1;
    int G = (int)std::min<int64_t>(RKA_MAXG, (q + 8 * RKA_NW - 1) / (8 * RKA_NW));
    if (const char* e = dbg_env("KZ_RKA_WG_G")) G = std::max(2, std::min(RKA_MAXG, atoi(e)));
    for (int guard = 0; guard < 16 && G >= 2; ++guard) {
        const int64_t qmax = (q + G - 1) / G;
        const size_t stage = rka_smem(qmax, box, 1, Pc) - rka_smem(qmax, box, 0, Pc);
        const size_t fixed = rka_smem(qmax, box, 0, Pc);
        int stages = (int)std::min<int64_t>(8, ((int64_t)kSmemLimit - (int64_t)fixed) / (int64_t)stage);
        if (const char* e = dbg_env("KZ_SYNC_STAGES")) stages = std::max(2, std::min(8, atoi(e)));
        if (stages < 2 || rka_smem(qmax, box, stages, Pc) > kSmemLimit) {
            ++G;  // fewer workers per cluster
            if (G > RKA_MAXG) break;
            continue;
        }
        const bool sr = qmax <= 8 * RKA_NW;
        void* fn = rka_fn(lg, epl, sr, 1);
        if (!fn) return fail(KZ_EINVAL, "no rka kernel for LG=%d EPL=%d", lg, epl);
        const size_t smem = rka_smem(qmax, box, stages, Pc);
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(Pc * G);
        cfg.blockDim = dim3(RKA_NT);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = Pc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
        if (e != cudaSuccess || nclusters < 2) {
            cudaGetLastError();
            return fail(KZ_EINVAL, "worker groups not schedulable");
        }
        if (nclusters < G) {  // every cluster must be co-resident (they poll each other)
            G = nclusters;
            continue;
        }
        pl.kernel = KZ_KERNEL_SYNC_CLUSTER;
        pl.tma = true;
        pl.sr = sr;
        pl.wg = true;
        pl.threads = RKA_NT;
        pl.ctas = Pc * G;
        pl.cluster = Pc;
        pl.stages = stages;
        pl.smem = smem;
        pl.lg = lg;
        pl.epl = epl;
        pl.box = box;
        return KZ_OK;
    }
    return fail(KZ_EINVAL, "no feasible worker-group plan for q=%lld n=%lld", (long long)q, (long long)s->n);
}

static int plan_rka(kz_system* s, const kz_params* p, int64_t q, Plan& pl) {
    if (dbg_env("KZ_SYNC_V5")) return fail(KZ_EINVAL, "rka kernel disabled (KZ_SYNC_V5)");
    if (q > 512) return fail(KZ_EINVAL, "q=%lld exceeds the rka kernel's 512 workers", (long long)q);
    const int64_t ld = s->ld;
    {
        const char* e = dbg_env("KZ_RKA_WG");
        const bool want = e ? atoi(e) != 0 : true;
        if (want && q > 8 * RKA_NW && p->ctas == 0 && p->partial_dev == nullptr && plan_rka_wg(s, p, q, pl) == KZ_OK)
            return KZ_OK;
    }
    int Pc = 16, G = 1;
    if (p->ctas > 16) {
        G = p->ctas / 16;
    } else if (p->ctas > 0) {
        Pc = 1;
        while (2 * Pc <= p->ctas) Pc *= 2;
    } else {
        // as few clusters as the 256-column TMA box and the shared-memory ring allow: every
        // extra cluster adds a tagged-word round trip through L2 per iteration (measured:
        // 80000 x 2000, q = 64: 1 cluster 2.54 us / iteration, 3 clusters 2.89 us)
        G = 1;
    }
    if (const char* e = dbg_env("KZ_SYNC_CLUSTERS")) G = atoi(e);
    G = std::max<int>(G, (int)((ld + Pc * 256 - 1) / (Pc * 256)));
    G = std::max(1, std::min(RKA_MAXG, G));
    int gcap = RKA_MAXG;
    for (int guard = 0; guard < 64; ++guard) {
        if (G > gcap) return fail(KZ_EINVAL, "rka kernel: %d clusters needed, %d co-resident", G, gcap);
        const int P = Pc * G;
        const int64_t cw = (((ld + P - 1) / P) + 1) & ~(int64_t)1;
        const int box = (int)((cw + 3) & ~(int64_t)3);
        if (box > 256) {
            ++G;
            continue;
        }
        const int npairs = box / 2;
        int lg = npairs <= 8 ? 8 : (npairs <= 16 ? 16 : 32);
        int epl = lg == 32 ? (npairs + 31) / 32 : 1;
        if (const char* e = dbg_env("KZ_RKA_LG8"))  // experiment: 8 lanes per row, 2 pairs per lane
            if (atoi(e) && npairs <= 16) lg = 8, epl = 2;
        const size_t stage = rka_smem(q, box, 1, Pc) - rka_smem(q, box, 0, Pc);
        const size_t fixed = rka_smem(q, box, 0, Pc);
        int stages = (int)std::min<int64_t>(8, ((int64_t)kSmemLimit - (int64_t)fixed) / (int64_t)stage);
        if (const char* e = dbg_env("KZ_SYNC_STAGES")) stages = std::max(2, std::min(8, atoi(e)));
        if (stages < 2 || rka_smem(q, box, stages, Pc) > kSmemLimit) {
            ++G;  // thinner slices
            continue;
        }
        void* fn = rka_fn(lg, epl, q <= 8 * RKA_NW);
        pl.sr = q <= 8 * RKA_NW;
        pl.wg = false;
        if (!fn) return fail(KZ_EINVAL, "no rka kernel for LG=%d EPL=%d", lg, epl);
        const size_t smem = rka_smem(q, box, stages, Pc);
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(P);
        cfg.blockDim = dim3(RKA_NT);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = Pc;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        int nclusters = 0;
        cudaError_t e = cudaOccupancyMaxActiveClusters(&nclusters, fn, &cfg);
        if (e != cudaSuccess || nclusters < 1) {
            cudaGetLastError();
            if (Pc == 1) return fail(KZ_EINVAL, "rka kernel not schedulable");
            Pc /= 2;
            G *= 2;
            continue;
        }
        if (nclusters < G) {  // every cluster must be co-resident (they poll each other)
            gcap = std::min(gcap, nclusters);
            G = gcap;
            continue;
        }
        pl.kernel = KZ_KERNEL_SYNC_CLUSTER;
        pl.tma = true;
        pl.threads = RKA_NT;
        pl.ctas = P;
        pl.cluster = Pc;
        pl.stages = stages;
        pl.smem = smem;
        pl.lg = lg;
        pl.epl = epl;
        pl.box = box;
        return KZ_OK;
    }
    return fail(KZ_EINVAL, "no feasible rka kernel configuration for q=%lld n=%lld", (long long)q, (long long)s->n);
}

static int launch_solve(kz_system* s, const Plan& pl, SolveArgs& args, cudaStream_t st) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(pl.ctas);
    cfg.blockDim = dim3(pl.threads);
    cfg.dynamicSmemBytes = pl.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    cfg.attrs = attr;
    void* fn;
    cudaLaunchAttribute attr2[2];
    if (pl.kernel == KZ_KERNEL_CHAIN) {
        fn = chain_fn(pl.ep, pl.rows, pl.pair, pl.delta, pl.wide);
        int na = 0;
        // KZ_NO_COOP (experiments): drop the cooperative attribute so a profiler can replay the
        // launch; safe only when every CTA fits at once (one per SM, ctas <= SMs)
        static const bool no_coop = dbg_env("KZ_NO_COOP") != nullptr;
        if (pl.ctas > 1 && !(no_coop && pl.ctas <= s->sms)) {
            attr2[na].id = cudaLaunchAttributeCooperative;
            attr2[na].val.cooperative = 1;
            ++na;
        }
        if (pl.pair >= 2) {
            attr2[na].id = cudaLaunchAttributeClusterDimension;
            attr2[na].val.clusterDim.x = pl.pair;
            attr2[na].val.clusterDim.y = 1;
            attr2[na].val.clusterDim.z = 1;
            ++na;
        }
        cfg.attrs = attr2;
        cfg.numAttrs = na;
    } else if (pl.kernel == KZ_KERNEL_SYNC_CLUSTER) {
        fn = pl.tma ? rka_fn(pl.lg, pl.epl, pl.sr, pl.wg ? 1 : (pl.xr ? 2 : 0)) : sync_fn(true, pl.lpr);
        int na = 0;
        attr2[na].id = cudaLaunchAttributeClusterDimension;
        attr2[na].val.clusterDim.x = pl.cluster;
        attr2[na].val.clusterDim.y = 1;
        attr2[na].val.clusterDim.z = 1;
        ++na;
        static const bool no_coop_rka = dbg_env("KZ_NO_COOP") != nullptr;  // experiments: ncu replay
        if (pl.ctas > pl.cluster && !(no_coop_rka && pl.ctas <= s->sms)) {  // clusters poll each other: co-resident
            attr2[na].id = cudaLaunchAttributeCooperative;
            attr2[na].val.cooperative = 1;
            ++na;
        }
        cfg.attrs = attr2;
        cfg.numAttrs = na;
    } else {
        fn = sync_fn(false, pl.lpr);
        attr[0].id = cudaLaunchAttributeCooperative;
        attr[0].val.cooperative = 1;
        cfg.numAttrs = 1;
    }
    if (pl.kernel == KZ_KERNEL_WARP) {
        fn = rkw_fn(pl.ep);
        cfg.numAttrs = 0;
    }
    void* kargs[] = {&args, &s->tmA, &s->tmB};
    cudaError_t e = cudaLaunchKernelExC(&cfg, fn, kargs);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return fail(KZ_ECUDA, "solve kernel launch failed: %s", cudaGetErrorString(e));
    }
    return KZ_OK;
}

namespace {
// Everything a solve needs between setup and its iteration loop (kz_solve, kz_solve_sharded).
struct SolveCtx {
    bool sharded = false;  // kz_solve_sharded: partial steps driven per iteration by the native loop
    int64_t q = 1, bs = 1;
    bool budget_mode = false, trace_mode = false, stop_mode = false, cyclic = false, partial_mode = false;
    Plan pl;
    SolveArgs args = {};
    int64_t n_ck_cap = 0, chunk_cap = 1;
    bool phase_timing = false;
};
}  // namespace

// Validation, cached setup (norms, sampler, packed records, worker streams,
// weights), kernel plan, scratch and the kernel arguments.
static int solve_setup(kz_system* s, const kz_params* p, kz_result* r, cudaStream_t st, SolveCtx& cx) {
    // --- validation (SolverConfig.validate, solvers.py:85-101; _drive 200-214) ---
    if (p->variant < KZ_RK || p->variant > KZ_CK) return fail(KZ_EINVAL, "unknown variant %d", p->variant);
    if (p->q < 1) return fail(KZ_EINVAL, "q must be >= 1, got %lld", (long long)p->q);
    if (p->block_size < 1) return fail(KZ_EINVAL, "block_size must be >= 1, got %lld", (long long)p->block_size);
    if (p->block_size > (1 << 28)) return fail(KZ_EINVAL, "block_size %lld exceeds 2^28", (long long)p->block_size);
    if (!(p->epsilon > 0)) return fail(KZ_EINVAL, "epsilon must be > 0, got %g", p->epsilon);
    if (p->max_iterations < 1) return fail(KZ_EINVAL, "max_iterations must be >= 1, got %lld", (long long)p->max_iterations);
    if (p->budget < 0) return fail(KZ_EINVAL, "fixed iteration budget must be >= 1, got %lld", (long long)p->budget);
    if (p->trace_step < 0) return fail(KZ_EINVAL, "trace_step must be >= 1, got %lld", (long long)p->trace_step);
    const bool budget_mode = p->budget > 0;
    const bool trace_mode = !budget_mode && p->trace_step > 0;
    const bool stop_mode = !budget_mode && !trace_mode;
    if ((stop_mode || trace_mode) && !s->has_xref) return fail(KZ_EINVAL, "system carries no reference solution");
    if (trace_mode && !p->trace_host) return fail(KZ_EINVAL, "trace mode needs a trace buffer");
    const bool cyclic = p->variant == KZ_CK;  // solve_ck (solvers.py:271-291): row k mod m, no stream
    const int64_t q = (p->variant == KZ_RK || cyclic) ? 1 : p->q;
    const int64_t bs = p->variant == KZ_RKAB ? p->block_size : 1;
    KZ_CUDA(cudaSetDevice(s->device));

    // --- setup: row norms, sampler, packed (b, sq), streams, weights ---
    if (cyclic)
        KZ_TRY(ensure_norms(s, st));
    else
        KZ_TRY(ensure_sampler(s, p->scheme, q, st));
    KZ_TRY(ensure_bs2(s, st));
    if (!(s->pods_q == q && s->pods_seed == p->base_seed && s->pods_off == p->worker_offset)) {
        std::vector<PcgPod> pods(q);
        for (int64_t t = 0; t < q; ++t) pods[t] = seed_stream(p->base_seed, (uint64_t)(p->worker_offset + t));
        KZ_TRY(s->states.ensure(q));
        KZ_CUDA(cudaMemcpyAsync(s->states.p, pods.data(), q * sizeof(PcgPod), cudaMemcpyHostToDevice, st));
        s->pods_q = q;
        s->pods_seed = p->base_seed;
        s->pods_off = p->worker_offset;
    }
    std::vector<double> al(q, 1.0);
    if (p->alphas_host) std::copy(p->alphas_host, p->alphas_host + q, al.begin());
    if (al != s->alphas_cache) {
        KZ_TRY(s->alphas.ensure(q));
        KZ_CUDA(cudaMemcpyAsync(s->alphas.p, al.data(), q * sizeof(double), cudaMemcpyHostToDevice, st));
        s->alphas_cache = al;
    }
    if (!p->keep_x) KZ_CUDA(cudaMemsetAsync(s->x.p, 0, s->ld * sizeof(double), st));
    const bool partial_mode = p->partial_dev != nullptr;
    if (partial_mode && !cx.sharded && !(budget_mode && p->budget == 1))
        return fail(KZ_EINVAL, "partial (row-sharded) steps run exactly one iteration: set budget = 1");

    // --- kernel plan ---
    Plan pl;
    int kern = p->kernel;
    const bool threads_combine = (p->flags & KZ_FLAG_THREADS_COMBINE) != 0 && q > 1;
    if (threads_combine) {
        if (p->variant != KZ_RKA && p->variant != KZ_RKAB)
            return fail(KZ_EINVAL, "the threaded engine's combine applies to RKA / RKAB");
        if (partial_mode || cx.sharded) return fail(KZ_EINVAL, "the threaded engine's combine is single-system only");
        if (kern != KZ_KERNEL_AUTO && kern != KZ_KERNEL_CHAIN)
            return fail(KZ_EINVAL, "the threaded engine's combine runs on the chain kernel");
        kern = KZ_KERNEL_CHAIN;
    }
    if (kern == KZ_KERNEL_AUTO) {
        if (q == 1 && bs == 1 && s->ld <= 128 && p->partial_dev == nullptr && p->threads == 0) {
            // short rows: one warp beats the chain kernel's block machinery (measured, budget mode:
            // n = 50 0.32 vs 0.38 us per row, n = 120 0.35 vs 0.36; the chain wins from n ~ 250)
            kern = KZ_KERNEL_WARP;
        } else if (q == 1 || bs > 1) {
            kern = KZ_KERNEL_CHAIN;
        } else {
            kern = KZ_KERNEL_SYNC_CLUSTER;  // one or several clusters; grid barrier as the fallback
        }
    }
    pl.delta = threads_combine && p->variant == KZ_RKA;
    const int64_t key[6] = {kern + (pl.delta ? 100 : 0), q, bs, p->ctas, p->threads, p->kernel};
    static_assert(sizeof(Plan) <= sizeof(s->plan_blob), "plan cache");
    if (std::equal(key, key + 6, s->plan_key)) {
        memcpy(&pl, s->plan_blob, sizeof(Plan));  // same shape as the previous call: reuse its plan
        // the dynamic shared-memory limit is a property of the kernel function, which another
        // system may have lowered since: restore it for this plan
        void* fn = pl.kernel == KZ_KERNEL_WARP    ? rkw_fn(pl.ep)
                   : pl.kernel == KZ_KERNEL_CHAIN ? chain_fn(pl.ep, pl.rows, pl.pair, pl.delta, pl.wide)
                   : pl.tma                     ? rka_fn(pl.lg, pl.epl, pl.sr, pl.wg ? 1 : (pl.xr ? 2 : 0))
                                                : sync_fn(pl.kernel == KZ_KERNEL_SYNC_CLUSTER, pl.lpr);
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
    } else if (kern == KZ_KERNEL_WARP) {
        if (q != 1 || bs != 1 || s->ld > 256)
            return fail(KZ_EINVAL, "the warp kernel runs RK / CK on rows of at most 256 columns");
        pl.kernel = KZ_KERNEL_WARP;
        pl.ep = s->ld <= 64 ? 1 : (s->ld <= 128 ? 2 : 4);
        pl.ctas = 1;
        pl.threads = 32;
        pl.smem = 0;
    } else if (kern == KZ_KERNEL_CHAIN) {
        KZ_TRY(plan_chain(s, p, q, pl));
    } else if (kern == KZ_KERNEL_RKA) {
        if (bs != 1 || q < 2) return fail(KZ_EINVAL, "the rka kernel runs RKA / RKAB with q > 1, block_size 1");
        KZ_TRY(plan_rka(s, p, q, pl));
    } else if (kern == KZ_KERNEL_SYNC_CLUSTER || kern == KZ_KERNEL_SYNC_GRID) {
        if (bs != 1) return fail(KZ_EINVAL, "the sync kernels run RKA / RKAB with block_size 1 only");
        int rc = kern == KZ_KERNEL_SYNC_CLUSTER ? plan_rka(s, p, q, pl) : KZ_EINVAL;
        if (rc != KZ_OK && kern == KZ_KERNEL_SYNC_CLUSTER && dbg_env("KZ_DEBUG_PLAN"))
            fprintf(stderr, "[kz plan] rka kernel not used: %s\n", g_err.c_str());
        if (rc != KZ_OK) rc = plan_sync(s, p, q, kern == KZ_KERNEL_SYNC_CLUSTER, pl);
        if (rc != KZ_OK && kern == KZ_KERNEL_SYNC_CLUSTER && p->kernel == KZ_KERNEL_AUTO)
            rc = plan_sync(s, p, q, false, pl);
        // more workers than the column-sliced kernels take (q > 512): one CTA (or pair) per worker
        // on the chain kernel, in waves
        if (rc != KZ_OK && p->kernel == KZ_KERNEL_AUTO) rc = plan_chain(s, p, q, pl);
        KZ_TRY(rc);
    } else {
        return fail(KZ_EINVAL, "unknown kernel selector %d", kern);
    }
    memcpy(s->plan_blob, &pl, sizeof(Plan));
    std::copy(key, key + 6, s->plan_key);
    r->kernel_used = pl.tma ? KZ_KERNEL_RKA : pl.kernel;
    r->ctas = pl.ctas;
    r->threads = pl.threads;
    r->plan_ep = pl.kernel == KZ_KERNEL_CHAIN || pl.kernel == KZ_KERNEL_WARP ? pl.ep : pl.epl;
    r->plan_rows = pl.kernel == KZ_KERNEL_CHAIN ? pl.rows : 1;
    r->plan_cluster = pl.kernel == KZ_KERNEL_CHAIN ? pl.pair : pl.cluster;
    r->plan_stages = pl.stages;
    r->plan_waves = pl.waves;

    // --- scratch ---
    const int64_t draws_per_iter = q * bs;
    const int64_t idx_cap = std::max<int64_t>(draws_per_iter, (int64_t)8 << 20);
    const int64_t chunk_cap = std::max<int64_t>(1, idx_cap / draws_per_iter);
    KZ_TRY(s->idx.ensure(std::min<int64_t>(idx_cap, chunk_cap * draws_per_iter)));
    if (pl.kernel == KZ_KERNEL_CHAIN && q > 1) KZ_TRY(s->V.ensure((size_t)((q + pl.waves - 1) / pl.waves) * s->ld));
    KZ_TRY(s->part.ensure(std::max<size_t>(16, 2 * (size_t)pl.ctas * (q + 1))));
    if (pl.tma && pl.ctas > pl.cluster) {
        // tagged words of the rka kernel's cluster exchange (a buffer of their own; tags restart
        // at 1 every launch, so launch_step zeroes the words before each launch)
        s->ll_words = (size_t)2 * (pl.ctas / pl.cluster) * (pl.wg ? 2 * (size_t)s->ld : (size_t)RKA_LL_PAD * (q + 1));
        KZ_TRY(s->ll.ensure(s->ll_words));
        KZ_CUDA(cudaMemsetAsync(&s->status.p->aborted, 0, sizeof(int), st));
    }
    const int64_t n_ck_cap = p->ckpt_every > 0 ? std::max<int64_t>(0, p->ckpt_capacity) : 0;
    if (n_ck_cap > 0) KZ_TRY(s->ckpt.ensure((size_t)n_ck_cap * s->n));

    SolveArgs args = {};
    args.A = s->A.p;
    args.b = s->b.p;
    args.sq = s->sq.p;
    args.bs2 = s->bs2.p;
    args.xref = s->xref.p;
    args.x = s->x.p;
    args.partial = p->partial_dev;
    args.V = s->V.p;
    args.idx = s->idx.p;
    args.alphas = s->alphas.p;
    args.part = (pl.tma && pl.ctas > pl.cluster) ? reinterpret_cast<double*>(s->ll.p) : s->part.p;
    args.barrier = s->barrier.p;
    args.status = s->status.p;
    args.ckpt = s->ckpt.p;
    args.n = s->n;
    args.ld = s->ld;
    args.q = q;
    args.bs = bs;
    args.ckpt_every = n_ck_cap > 0 ? p->ckpt_every : 0;
    args.ckpt_cap = n_ck_cap;
    args.eps = p->epsilon;
    args.use_stop = stop_mode ? 1 : 0;
    args.stages = pl.stages;
    args.box = pl.box;
    args.wg = pl.wg ? 1 : 0;
    args.combine = !threads_combine ? KZ_COMBINE_AVERAGE
                   : (p->variant == KZ_RKA ? KZ_COMBINE_RKA_DELTA : KZ_COMBINE_RKAB_DELTA);
    if (pl.tma) KZ_TRY(ensure_tmaps(s, pl.box));
    const bool phase_timing = dbg_env("KZ_PHASE_TIMING") != nullptr;
    args.ablate = dbg_env("KZ_ABLATE") ? atoi(dbg_env("KZ_ABLATE")) : 0;
    if (phase_timing) {
        KZ_TRY(s->dbg.ensure(32 * 128 * 16 + 32768));
        KZ_CUDA(cudaMemsetAsync(s->dbg.p, 0, (32 * 128 * 16 + 32768) * sizeof(long long), st));
        args.dbg = s->dbg.p;
    }

    cx.q = q;
    cx.bs = bs;
    cx.budget_mode = budget_mode;
    cx.trace_mode = trace_mode;
    cx.stop_mode = stop_mode;
    cx.cyclic = cyclic;
    cx.partial_mode = partial_mode;
    cx.pl = pl;
    cx.args = args;
    cx.n_ck_cap = n_ck_cap;
    cx.chunk_cap = chunk_cap;
    cx.phase_timing = phase_timing;
    return KZ_OK;
}

// One launch of the planned solve kernel over args.count iterations, with the
// plan fallbacks a first launch may need (CTA pairs / several clusters not
// launchable cooperatively on this device).
static int launch_step(kz_system* s, const kz_params* p, kz_result* r, SolveCtx& cx, bool first, cudaStream_t st) {
    Plan& pl = cx.pl;
    SolveArgs& args = cx.args;
    const int64_t q = cx.q;
    if (!pl.tma) KZ_CUDA(cudaMemsetAsync(s->barrier.p, 0, sizeof(unsigned), st));
    if (pl.kernel == KZ_KERNEL_SYNC_CLUSTER && !pl.tma && pl.ctas > pl.cluster) {  // sync kernel: tags restart at 1
        KZ_CUDA(cudaMemsetAsync(s->part.p, 0, 4 * (size_t)(pl.ctas / pl.cluster) * (q + 1) * sizeof(double), st));
        KZ_CUDA(cudaMemsetAsync(&s->status.p->aborted, 0, sizeof(int), st));
    }
    if (pl.tma && pl.ctas > pl.cluster)
        KZ_CUDA(cudaMemsetAsync(s->ll.p, 0, s->ll_words * sizeof(unsigned long long), st));
    int lrc = launch_solve(s, pl, args, st);
    if (lrc != KZ_OK && pl.kernel == KZ_KERNEL_CHAIN && pl.pair >= 2 && first) {
        // CTA-pair clusters not launchable cooperatively here: one CTA per worker
        s->no_pairs = true;  // remembered for this system (no process-wide side effects)
        const int waves_before = pl.waves;
        KZ_TRY(plan_chain(s, p, q, pl));
        if (pl.waves != waves_before)
            return fail(KZ_ECUDA, "CTA pairs not launchable here and one CTA per worker changes the wave count");
        memcpy(s->plan_blob, &pl, sizeof(Plan));
        args.stages = pl.stages;
        r->ctas = pl.ctas;
        r->threads = pl.threads;
        r->plan_ep = pl.ep;
        r->plan_rows = pl.rows;
        r->plan_cluster = pl.pair;
        r->plan_stages = pl.stages;
        if (pl.ctas > 1) KZ_CUDA(cudaMemsetAsync(s->barrier.p, 0, sizeof(unsigned), st));
        lrc = launch_solve(s, pl, args, st);
    }
    if (lrc != KZ_OK && pl.kernel == KZ_KERNEL_SYNC_CLUSTER && pl.ctas > pl.cluster && first &&
        p->kernel == KZ_KERNEL_AUTO) {
        // several clusters not launchable cooperatively here: grid-barrier kernel
        KZ_TRY(plan_sync(s, p, q, false, pl));
        memcpy(s->plan_blob, &pl, sizeof(Plan));
        KZ_TRY(s->part.ensure(std::max<size_t>(16, 2 * (size_t)pl.ctas * (q + 1))));
        args.part = s->part.p;
        args.stages = pl.stages;
        r->kernel_used = pl.tma ? KZ_KERNEL_RKA : pl.kernel;
        r->ctas = pl.ctas;
        KZ_CUDA(cudaMemsetAsync(s->barrier.p, 0, sizeof(unsigned), st));
        lrc = launch_solve(s, pl, args, st);
    }
    return lrc;
}

// One outer iteration's local step in waves of co-resident workers (chain kernel, partial mode):
// wave j runs workers [q j / W, q (j + 1) / W) and adds their ordered sum to the previous waves'
// (SolveArgs::accumulate), so S is bit-identical to one launch over all q workers.
static int launch_waves(kz_system* s, const kz_params* p, kz_result* r, SolveCtx& cx, bool first, cudaStream_t st) {
    Plan& pl = cx.pl;
    SolveArgs& a = cx.args;
    const int W = pl.waves;
    if (W <= 1) {
        a.accumulate = 0;
        return launch_step(s, p, r, cx, first, st);
    }
    const SolveArgs saved = a;
    const int ctas = pl.ctas;
    const int64_t q = cx.q;
    int rc = KZ_OK;
    for (int j = 0; j < W && rc == KZ_OK; ++j) {
        const int64_t w0 = q * j / W, w1 = q * (j + 1) / W;
        a.q = w1 - w0;
        a.alphas = saved.alphas + w0;
        a.idx = saved.idx + w0 * saved.idx_stride;
        a.accumulate = j > 0 ? 1 : 0;
        pl.ctas = (int)((w1 - w0) * pl.pair);
        rc = launch_step(s, p, r, cx, first && j == 0, st);
        pl.ctas = ctas;
    }
    a = saved;
    return rc;
}

extern "C" int32_t kz_solve(kz_system* s, const kz_params* p, kz_result* r, double* x_host, void* stream) {
    NvtxScope nvtx_("kz_solve");
    if (!s || !p || !r) return fail(KZ_EINVAL, "null argument");
    memset(r, 0, sizeof(*r));
    r->final_error_sq = NAN;
    r->final_residual = NAN;
    cudaStream_t st = pick_stream(s, stream);
    SolveCtx cx;
    KZ_TRY(solve_setup(s, p, r, st, cx));
    if (cx.pl.waves > 1) {
        // more workers than co-resident CTAs: the per-outer-iteration driver runs them in waves
        if (cx.trace_mode) return fail(KZ_EINVAL, "trace mode with more workers than co-resident CTAs");
        if (cx.partial_mode) return fail(KZ_EINVAL, "partial steps with more workers than co-resident CTAs");
        kz_params pp = *p;
        pp.flags |= KZ_FLAG_SHARDED_LOOP;
        return kz_solve_sharded(s, nullptr, &pp, r, x_host, stream);
    }
    const int64_t q = cx.q, bs = cx.bs;
    const bool budget_mode = cx.budget_mode, trace_mode = cx.trace_mode, stop_mode = cx.stop_mode,
               cyclic = cx.cyclic, partial_mode = cx.partial_mode, phase_timing = cx.phase_timing;
    const int64_t n_ck_cap = cx.n_ck_cap, chunk_cap = cx.chunk_cap;
    Plan& pl = cx.pl;
    SolveArgs& args = cx.args;

    const int64_t limit = budget_mode ? p->budget : p->max_iterations;
    int64_t k = 0, evals = 0;
    bool converged = false;
    double err = NAN;
    int64_t n_trace = 0;
    const long long launches0 = g_launches.load();
    float kernel_ms = 0.f;

    // trace records are taken as device snapshots of x and evaluated in batches of up to 32:
    // one pass over A gives all their residuals (residual_batch_kernel), one host round trip
    // returns residuals and errors; the loop itself never waits for a record
    constexpr int TRACE_BATCH = 32;
    int64_t pending = 0;
    if (trace_mode) {
        KZ_TRY(s->tsnap.ensure((size_t)TRACE_BATCH * s->ld));
        KZ_TRY(s->tr2.ensure((size_t)TRACE_BATCH * s->m));
        KZ_TRY(s->tsum.ensure(2 * TRACE_BATCH));
        KZ_TRY(s->tmp.ensure((size_t)std::max(s->m, s->n)));
    }
    auto flush_trace = [&]() -> int {
        if (pending == 0) return KZ_OK;
        const int K = (int)pending;
        residual_batch_kernel<<<(unsigned)((s->m + 31) / 32), 256, 0, st>>>(s->A.p, s->b.p, s->tsnap.p, s->m, s->n,
                                                                              s->ld, K, s->tr2.p);
        KZ_TRY(check_launch("residual_batch_kernel"));
        for (int j = 0; j < K; ++j) {
            sum_kernel<<<1, 1024, 0, st>>>(s->tr2.p + (int64_t)j * s->m, s->m, s->tsum.p + 2 * j);
            KZ_TRY(check_launch("sum_kernel"));
            diff_sq_kernel<<<(unsigned)((s->n + 255) / 256), 256, 0, st>>>(s->tsnap.p + (int64_t)j * s->ld,
                                                                            s->xref.p, s->n, s->tmp.p);
            KZ_TRY(check_launch("diff_sq_kernel"));
            sum_kernel<<<1, 1024, 0, st>>>(s->tmp.p, s->n, s->tsum.p + 2 * j + 1);
            KZ_TRY(check_launch("sum_kernel"));
        }
        double h[2 * TRACE_BATCH];
        KZ_CUDA(cudaMemcpyAsync(h, s->tsum.p, 2 * (size_t)K * sizeof(double), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        for (int j = 0; j < K; ++j) {
            const int64_t t = n_trace - K + j;
            p->trace_host[3 * t + 1] = std::sqrt(h[2 * j + 1]);
            p->trace_host[3 * t + 2] = std::sqrt(h[2 * j]);
        }
        pending = 0;
        return KZ_OK;
    };
    auto record_trace = [&]() -> int {
        KZ_CUDA(cudaMemcpyAsync(s->tsnap.p + pending * s->ld, s->x.p, s->ld * sizeof(double),
                                cudaMemcpyDeviceToDevice, st));
        p->trace_host[3 * n_trace + 0] = (double)k;
        ++n_trace;
        if (++pending == TRACE_BATCH) KZ_TRY(flush_trace());
        return KZ_OK;
    };

    KZ_CUDA(cudaEventRecord(s->ev[0], st));
    if (trace_mode) KZ_TRY(record_trace());
    int64_t chunk = stop_mode ? std::min<int64_t>(chunk_cap, std::max<int64_t>(64, 4096 / bs)) : chunk_cap;
    int64_t chunk_max = chunk_cap;  // stop mode: launches grow to this many iterations
    if (stop_mode && (p->flags & KZ_FLAG_SHORT_LAUNCHES)) {
        // solves side by side on one GPU: short launches let the lanes interleave over the
        // co-resident clusters (c1 batch of 10: 26.2 -> 24.4 ms; a solve alone loses ~1 %)
        chunk = chunk_max = std::min<int64_t>(chunk_cap, std::max<int64_t>(64, 2048 / bs));
    }
    for (;;) {
        const int64_t remaining = limit - k;
        if (remaining <= 0 && !stop_mode) break;
        int64_t c = std::min<int64_t>(chunk, remaining);
        if (trace_mode) c = std::min<int64_t>(c, p->trace_step - (k % p->trace_step));
        if (c > 0 && cyclic) {
            cyclic_rows_kernel<<<(unsigned)std::min<int64_t>((c + 255) / 256, 4096), 256, 0, st>>>(
                s->idx.p, p->k_start + k, c, s->m);
            KZ_TRY(check_launch("cyclic_rows_kernel"));
        } else if (c > 0) {
            const int64_t count = c * bs;
            if (pl.kernel == KZ_KERNEL_CHAIN)
                KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, q, (p->k_start + k) * bs, count, s->idx.p,
                                      count, 1, st));
            else
                KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, q, (p->k_start + k) * bs, count, s->idx.p, 1,
                                      q, st));
        }
        args.k0 = p->k_start + k;
        args.count = c;
        args.idx_stride = c * bs;
        args.final_check = (stop_mode && k + c == p->max_iterations) ? 1 : 0;
        KZ_CUDA(cudaEventRecord(s->ev[2], st));
        NvtxScope nvtx_chunk("kz_solve chunk");
        KZ_TRY(launch_step(s, p, r, cx, k == 0, st));
        if (partial_mode) {
            // row-sharded local step: exactly one iteration, left in flight on the stream (the
            // collective and kz_average_from that follow are stream-ordered); no host sync
            r->iterations = 1;
            r->rows_projected = q * bs;
            r->kernel_launches = g_launches.load() - launches0;
            return KZ_OK;
        }
        KZ_CUDA(cudaEventRecord(s->ev[3], st));
        KZ_CUDA(cudaMemcpyAsync(s->h_status, s->status.p, sizeof(SolveStatus), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        float ms = 0.f;
        cudaEventElapsedTime(&ms, s->ev[2], s->ev[3]);
        kernel_ms += ms;
        const SolveStatus hs = *s->h_status;
        if (pl.kernel == KZ_KERNEL_SYNC_CLUSTER && pl.ctas > pl.cluster && hs.aborted)
            return fail(KZ_ECUDA, "cross-cluster exchange timed out (clusters not co-resident)");
        k += hs.iters_done;
        evals += hs.checks;
        if (hs.checks > 0) err = hs.err;
        if (hs.converged) {
            converged = true;
            break;
        }
        if (hs.iters_done != c) return fail(KZ_ECUDA, "solve kernel stopped early (%lld of %lld iterations)",
                                            (long long)hs.iters_done, (long long)c);
        if (trace_mode && k % p->trace_step == 0) KZ_TRY(record_trace());
        if (stop_mode && k >= p->max_iterations) break;
        if (stop_mode) chunk = std::min<int64_t>(chunk_max, chunk * 2);
    }
    KZ_TRY(flush_trace());
    KZ_CUDA(cudaEventRecord(s->ev[1], st));
    KZ_CUDA(cudaEventSynchronize(s->ev[1]));
    float loop_ms = 0.f;
    cudaEventElapsedTime(&loop_ms, s->ev[0], s->ev[1]);

    r->iterations = k;
    r->converged = converged ? 1 : 0;
    r->error_evals = evals;
    r->final_error_sq = stop_mode ? err : NAN;
    r->rows_projected = k * q * bs;
    r->loop_ms = loop_ms;
    r->kernel_ms = kernel_ms;
    r->n_trace = n_trace;
    if (n_ck_cap > 0) {
        r->n_ckpt = std::min<int64_t>(n_ck_cap, k / p->ckpt_every);
        if (r->n_ckpt > 0 && p->ckpt_host)
            KZ_CUDA(cudaMemcpyAsync(p->ckpt_host, s->ckpt.p, (size_t)r->n_ckpt * s->n * sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
    }
    if (stop_mode && p->want_residual) {
        double res = NAN;
        KZ_TRY(device_norms(s, s->x.p, &res, nullptr, st));
        r->final_residual = res;
    }
    if (x_host) KZ_CUDA(cudaMemcpyAsync(x_host, s->x.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    r->kernel_launches = g_launches.load() - launches0;
    if (phase_timing && pl.kernel == KZ_KERNEL_CHAIN) {  // chain: block phases of CTA 0 thread 0
        std::vector<long long> h(32 * 64);
        KZ_CUDA(cudaMemcpy(h.data(), s->dbg.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        double acc[8] = {0};
        int nrec = 0;
        for (int b = 4; b < 63; ++b) {
            const long long* r = &h[b * 8];
            if (r[6] == 0 || h[(b + 1) * 8] == 0) continue;
            for (int ph = 0; ph < 6; ++ph) acc[ph] += (double)(r[ph + 1] - r[ph]);
            acc[6] += (double)(h[(b + 1) * 8] - r[6]);
            ++nrec;
        }
        if (nrec)
            fprintf(stderr, "[kz chain block cycles] issue %.0f wait %.0f partials %.0f reduce %.0f solve %.0f apply %.0f "
                            "gap %.0f (n=%d, R=%d)\n", acc[0] / nrec, acc[1] / nrec, acc[2] / nrec, acc[3] / nrec,
                    acc[4] / nrec, acc[5] / nrec, acc[6] / nrec, nrec, pl.rows);
    } else if (phase_timing) {  // per-phase completion (max over warps) relative to the earliest warp start, CTA 0
        std::vector<long long> h(32 * 128);
        KZ_CUDA(cudaMemcpy(h.data(), s->dbg.p, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        const int SL = pl.tma ? 16 : 8;  // stamp slots per (iteration, warp)
        double acc[8] = {0}, span = 0;
        int nrec = 0;
        for (int k = 4; k < 31; ++k) {
            long long t0 = -1, nxt = -1;
            long long mx[8];
            for (int ph = 0; ph < 8; ++ph) mx[ph] = -1;
            bool ok = true;
            for (int w = 0; w < 8; ++w) {
                const long long* r = &h[(k * 8 + w) * SL];
                const long long* rn = &h[((k + 1) * 8 + w) * SL];
                if (r[0] == 0 || rn[0] == 0) { ok = false; break; }
                t0 = (t0 < 0 || r[0] < t0) ? r[0] : t0;
                nxt = (nxt < 0 || rn[0] < nxt) ? rn[0] : nxt;
                for (int ph = 0; ph < 7; ++ph) if (r[ph] && r[ph] > mx[ph]) mx[ph] = r[ph];
            }
            if (!ok) continue;
            for (int ph = 0; ph < 7; ++ph) acc[ph] += (double)(mx[ph] - t0);
            span += (double)(nxt - t0);
            ++nrec;
        }
        if (nrec)
            fprintf(stderr, "[kz phase end, max over warps, cycles from start] top %.0f issued %.0f dots %.0f waited %.0f "
                            "err %.0f scales %.0f update %.0f | iteration %.0f (n=%d)\n", acc[0] / nrec, acc[1] / nrec,
                    acc[2] / nrec, acc[3] / nrec, acc[4] / nrec, acc[5] / nrec, acc[6] / nrec, span / nrec, nrec);
        if (atoi(dbg_env("KZ_PHASE_TIMING")) >= 3 && pl.tma) {
            // every cluster's rank-0 CTA: owner-warp and warp-0 stamps relative to its own iteration
            // start, and the spread of the iteration starts across clusters (globaltimer, ns)
            const int G = pl.ctas / pl.cluster;
            std::vector<long long> hh((size_t)32 * 128 * 16);
            KZ_CUDA(cudaMemcpy(hh.data(), s->dbg.p, hh.size() * sizeof(long long), cudaMemcpyDeviceToHost));
            auto at = [&](int g, int k, int w, int sl) { return hh[(((size_t)g * 32 + k) * 8 + w) * 16 + sl]; };
            double spread = 0;
            int ns = 0;
            for (int k = 4; k < 31; ++k) {
                long long lo = -1, hi = -1;
                for (int g = 0; g < G; ++g) {
                    const long long t = at(g, k, 0, 14);
                    if (!t) continue;
                    lo = lo < 0 || t < lo ? t : lo;
                    hi = hi < 0 || t > hi ? t : hi;
                }
                if (lo >= 0) spread += (double)(hi - lo), ++ns;
            }
            fprintf(stderr, "[kz clusters] %d clusters; iteration-start spread across clusters %.0f ns (mean)\n", G,
                    ns ? spread / ns : 0.0);
            {  // every CTA's events (globaltimer): spread across CTAs and the latest CTA relative to the earliest
                std::vector<long long> gg((size_t)32768);
                KZ_CUDA(cudaMemcpy(gg.data(), s->dbg.p + 65536, gg.size() * sizeof(long long), cudaMemcpyDeviceToHost));
                const char* names[4] = {"dots done", "owner total", "cross-cluster sum", "scales arrived"};
                double sp[4] = {0}, lat[4] = {0};
                int nk2 = 0;
                for (int k = 4; k < 31; ++k) {
                    long long lo[4], hi[4];
                    bool ok = true;
                    for (int ev = 0; ev < 4; ++ev) {
                        lo[ev] = -1, hi[ev] = -1;
                        for (int c = 0; c < pl.ctas; ++c) {
                            const long long t = gg[((size_t)c * 32 + k) * 4 + ev];
                            if (!t) continue;
                            lo[ev] = lo[ev] < 0 || t < lo[ev] ? t : lo[ev];
                            hi[ev] = hi[ev] < 0 || t > hi[ev] ? t : hi[ev];
                        }
                        ok = ok && lo[ev] > 0;
                    }
                    if (!ok) continue;
                    for (int ev = 0; ev < 4; ++ev) {
                        sp[ev] += (double)(hi[ev] - lo[ev]);
                        lat[ev] += (double)(hi[ev] - lo[0]);
                    }
                    ++nk2;
                }
                for (int ev = 0; ev < 4 && nk2; ++ev)
                    fprintf(stderr, "[kz all CTAs] %-18s spread %6.0f ns, latest %6.0f ns after the earliest dots done\n",
                            names[ev], sp[ev] / nk2, lat[ev] / nk2);
            }
            const int ow = 6;
            for (int g = 0; g < G; ++g) {
                double m[8] = {0};
                int nk = 0;
                for (int k = 4; k < 31; ++k) {
                    const long long t0 = at(g, k, 0, 0), t0o = at(g, k, ow, 0), tn = at(g, k + 1, 0, 0);
                    if (!t0 || !tn || !t0o) continue;
                    m[0] += (double)(at(g, k, 0, 13) - t0);    // dots + pushes done (warp 0)
                    m[1] += (double)(at(g, k, ow, 7) - t0o);   // partials at the owner
                    m[2] += (double)(at(g, k, ow, 10) - t0o);  // owner total
                    m[3] += (double)(at(g, k, ow, 11) - t0o);  // scale formed (after the cross-cluster sum)
                    m[4] += (double)(at(g, k, ow, 9) - t0o);   // broadcast issued
                    m[5] += (double)(at(g, k, 0, 3) - t0);     // scales arrived (warp 0)
                    m[6] += (double)(at(g, k, 0, 5) - t0);     // average done
                    m[7] += (double)(tn - t0);                 // iteration
                    ++nk;
                }
                if (nk)
                    fprintf(stderr, "[kz cluster %d] dots %.0f partials %.0f owner %.0f xsum %.0f bcast %.0f scales %.0f "
                                    "avg %.0f | iteration %.0f cycles\n", g, m[0] / nk, m[1] / nk, m[2] / nk, m[3] / nk,
                            m[4] / nk, m[5] / nk, m[6] / nk, m[7] / nk);
            }
        }
        if (atoi(dbg_env("KZ_PHASE_TIMING")) >= 2) {  // per-warp mean stamps relative to the earliest warp start
            double pw[8][16] = {{0}};
            int nk = 0;
            for (int k = 4; k < 31; ++k) {
                long long t0 = -1;
                for (int w = 0; w < 8; ++w) {
                    const long long v = h[(k * 8 + w) * SL];
                    if (v && (t0 < 0 || v < t0)) t0 = v;
                }
                if (t0 < 0) continue;
                for (int w = 0; w < 8; ++w)
                    for (int ph = 0; ph < SL; ++ph) {
                        const long long v = h[(k * 8 + w) * SL + ph];
                        pw[w][ph] += v ? (double)(v - t0) : 0.0;
                    }
                ++nk;
            }
            for (int w = 0; w < 8 && nk; ++w) {
                fprintf(stderr, "[kz warp %d]", w);
                for (int ph = 0; ph < SL; ++ph) fprintf(stderr, " %6.0f", pw[w][ph] / nk);
                fprintf(stderr, "\n");
            }
        }
    }
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// CGLS on the resident matrix (cgls.py:42-75): x_LS of min ||A x - b|| with the
// reference's stopping rule ||A^T (A x - b)|| <= tol ||A^T b|| and one restart.
// ---------------------------------------------------------------------------
extern "C" int32_t kz_cgls(kz_system* s, const double* b_host, double tol, int64_t max_it, double* x_out,
                           int64_t* iterations, void* stream) {
    NvtxScope nvtx_("kz_cgls");
    if (!s || !x_out) return fail(KZ_EINVAL, "null argument");
    if (!(tol > 0)) return fail(KZ_EINVAL, "tol must be > 0, got %g", tol);
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    const int64_t m = s->m, n = s->n, ld = s->ld;
    if (max_it <= 0) max_it = 10 * n + 100;
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>((int64_t)s->sms * 4, (m + 255) / 256));
    const int64_t rpc = (m + nchunks - 1) / nchunks;
    // layout: x | p | s (ld each) | r | t | b (m each) | partial (nchunks x ld) | scalars (8)
    const size_t need = 3 * (size_t)ld + 3 * (size_t)m + (size_t)nchunks * ld + 8;
    KZ_TRY(s->cg.ensure(need));
    double* x = s->cg.p;
    double* pv = x + ld;
    double* sv = pv + ld;
    double* r = sv + ld;
    double* t = r + m;
    double* bb = t + m;
    double* part = bb + m;
    double* scal = part + (size_t)nchunks * ld;  // [0] gamma, [1] delta, [2] gamma_new, [3] scratch
    if (b_host)
        KZ_CUDA(cudaMemcpyAsync(bb, b_host, m * sizeof(double), cudaMemcpyHostToDevice, st));
    else
        KZ_CUDA(cudaMemcpyAsync(bb, s->b.p, m * sizeof(double), cudaMemcpyDeviceToDevice, st));
    const unsigned rows_blocks = (unsigned)((m + 7) / 8);
    const dim3 tgrid((unsigned)((n + 255) / 256), (unsigned)nchunks);
    const unsigned eblocks = (unsigned)std::min<int64_t>(1024, (std::max(n, m) + 255) / 256);
    auto gemv_t = [&](const double* vec, double* out) -> int {  // out = A^T vec
        cg_gemv_t_partial_kernel<<<tgrid, 256, 0, st>>>(s->A.p, vec, m, n, ld, rpc, part);
        KZ_TRY(check_launch("cg_gemv_t_partial_kernel"));
        cg_gemv_t_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nchunks, n, ld, out);
        return check_launch("cg_gemv_t_reduce_kernel");
    };
    auto dot = [&](const double* u, const double* v, int64_t len, int slot, double* host) -> int {
        cg_dot_kernel<<<1, 1024, 0, st>>>(u, v, len, scal + slot);
        KZ_TRY(check_launch("cg_dot_kernel"));
        if (host) {
            KZ_CUDA(cudaMemcpyAsync(host, scal + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
            KZ_CUDA(cudaStreamSynchronize(st));
        }
        return KZ_OK;
    };
    KZ_CUDA(cudaMemsetAsync(x, 0, ld * sizeof(double), st));
    double ref2 = 0.0;
    KZ_TRY(gemv_t(bb, sv));
    KZ_TRY(dot(sv, sv, n, 3, &ref2));
    const double ref = std::sqrt(ref2);
    int64_t used = 0;
    bool ok = ref == 0.0;
    if (!ok) {
        const double abs_tol = tol * ref;
        for (int pass = 0; pass < 2; ++pass) {
            cg_gemv_n_kernel<<<rows_blocks, 256, 0, st>>>(s->A.p, x, bb, m, n, ld, 1, r);  // r = b - A x
            KZ_TRY(check_launch("cg_gemv_n_kernel"));
            KZ_TRY(gemv_t(r, sv));
            KZ_CUDA(cudaMemcpyAsync(pv, sv, ld * sizeof(double), cudaMemcpyDeviceToDevice, st));
            double gamma = 0.0;
            KZ_TRY(dot(sv, sv, n, 0, &gamma));
            int64_t it_used = max_it - used;
            for (int64_t it = 1; it <= max_it - used; ++it) {
                if (std::sqrt(gamma) <= abs_tol) {
                    it_used = it - 1;
                    break;
                }
                cg_gemv_n_kernel<<<rows_blocks, 256, 0, st>>>(s->A.p, pv, nullptr, m, n, ld, 0, t);  // t = A p
                KZ_TRY(check_launch("cg_gemv_n_kernel"));
                double delta = 0.0;
                KZ_TRY(dot(t, t, m, 1, &delta));
                if (delta == 0.0) {
                    it_used = it - 1;
                    break;
                }
                cg_update_xr_kernel<<<eblocks, 256, 0, st>>>(x, pv, r, t, scal, n, m);
                KZ_TRY(check_launch("cg_update_xr_kernel"));
                KZ_TRY(gemv_t(r, sv));
                double gamma_new = 0.0;
                KZ_TRY(dot(sv, sv, n, 2, &gamma_new));
                cg_update_p_kernel<<<eblocks, 256, 0, st>>>(pv, sv, scal, n);
                KZ_TRY(check_launch("cg_update_p_kernel"));
                KZ_CUDA(cudaMemcpyAsync(scal, scal + 2, sizeof(double), cudaMemcpyDeviceToDevice, st));
                gamma = gamma_new;
            }
            used += it_used;
            // verify on a freshly computed normal-equations residual (cgls.py:66-68)
            cg_gemv_n_kernel<<<rows_blocks, 256, 0, st>>>(s->A.p, x, bb, m, n, ld, 1, r);
            KZ_TRY(check_launch("cg_gemv_n_kernel"));
            KZ_TRY(gemv_t(r, sv));
            double tr2 = 0.0;
            KZ_TRY(dot(sv, sv, n, 3, &tr2));
            if (std::sqrt(tr2) <= abs_tol) {
                ok = true;
                break;
            }
            if (used >= max_it) break;
        }
    }
    KZ_CUDA(cudaMemcpyAsync(x_out, x, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    if (iterations) *iterations = used;
    if (!ok) return fail(KZ_ENOCONV, "CGLS did not reach tol=%g within %lld iterations", tol, (long long)max_it);
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// Extreme singular values of the row block [row_lo, row_hi] (spectral.py:66-121):
// lambda_max by power iteration on A^T A, lambda_min by inverse iteration with a
// matrix-free CG inner solve; the start vectors (Prng(0x5EED, 0/1), normalised)
// come from the host.  out[0] = lambda_max, out[1] = lambda_min.
// ---------------------------------------------------------------------------
extern "C" int32_t kz_spectral(kz_system* s, int64_t row_lo, int64_t row_hi, const double* v0_host,
                               const double* v1_host, double tol, int64_t max_it, double* out, void* stream) {
    NvtxScope nvtx_("kz_spectral");
    if (!s || !v0_host || !v1_host || !out) return fail(KZ_EINVAL, "null argument");
    if (row_lo < 0 || row_hi >= s->m || row_hi < row_lo) return fail(KZ_EINVAL, "bad row range");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    const int64_t m = row_hi - row_lo + 1, n = s->n, ld = s->ld;
    const double* A = s->A.p + row_lo * ld;
    const int64_t nchunks = std::max<int64_t>(1, std::min<int64_t>((int64_t)s->sms * 4, (m + 255) / 256));
    const int64_t rpc = (m + nchunks - 1) / nchunks;
    // v | w | y | r | p | mp (ld each) | t (m) | partial (nchunks x ld) | scalars (8)
    const size_t need = 6 * (size_t)ld + (size_t)m + (size_t)nchunks * ld + 8;
    KZ_TRY(s->cg.ensure(need));
    double* v = s->cg.p;
    double* w = v + ld;
    double* y = w + ld;
    double* r = y + ld;
    double* p = r + ld;
    double* mp = p + ld;
    double* t = mp + ld;
    double* part = t + m;
    double* scal = part + (size_t)nchunks * ld;  // [0] rs, [1] denom, [2] rs_new, [3] scratch, [4] norm
    const unsigned rows_blocks = (unsigned)((m + 7) / 8);
    const dim3 tgrid((unsigned)((n + 255) / 256), (unsigned)nchunks);
    const unsigned eblocks = (unsigned)std::min<int64_t>(1024, (n + 255) / 256);
    auto Av = [&](const double* x, double* out_m) -> int {
        cg_gemv_n_kernel<<<rows_blocks, 256, 0, st>>>(A, x, nullptr, m, n, ld, 0, out_m);
        return check_launch("cg_gemv_n_kernel");
    };
    auto ATv = [&](const double* vec, double* out_n) -> int {
        cg_gemv_t_partial_kernel<<<tgrid, 256, 0, st>>>(A, vec, m, n, ld, rpc, part);
        KZ_TRY(check_launch("cg_gemv_t_partial_kernel"));
        cg_gemv_t_reduce_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(part, nchunks, n, ld, out_n);
        return check_launch("cg_gemv_t_reduce_kernel");
    };
    auto dot = [&](const double* u, const double* x, int64_t len, int slot, double* host) -> int {
        cg_dot_kernel<<<1, 1024, 0, st>>>(u, x, len, scal + slot);
        KZ_TRY(check_launch("cg_dot_kernel"));
        if (host) {
            KZ_CUDA(cudaMemcpyAsync(host, scal + slot, sizeof(double), cudaMemcpyDeviceToHost, st));
            KZ_CUDA(cudaStreamSynchronize(st));
        }
        return KZ_OK;
    };
    auto rayleigh = [&](const double* x, double* val) -> int {  // ||A x||^2
        KZ_TRY(Av(x, t));
        return dot(t, t, m, 3, val);
    };
    // ---- lambda_max: power iteration (spectral.py:75-95)
    KZ_CUDA(cudaMemcpyAsync(v, v0_host, n * sizeof(double), cudaMemcpyHostToDevice, st));
    double lam = 0.0;
    KZ_TRY(rayleigh(v, &lam));
    bool ok = false;
    for (int64_t it = 0; it < max_it; ++it) {
        KZ_TRY(Av(v, t));
        KZ_TRY(ATv(t, w));
        double nw2 = 0.0;
        KZ_TRY(dot(w, w, n, 4, &nw2));
        const double nw = std::sqrt(nw2);
        if (nw == 0.0) return fail(KZ_ESPECTRAL, "sigma_max: power iteration hit a null vector");
        KZ_CUDA(cudaMemcpyAsync(scal + 4, &nw, sizeof(double), cudaMemcpyHostToDevice, st));
        cg_scale_div_kernel<<<eblocks, 256, 0, st>>>(w, scal + 4, n, v);
        KZ_TRY(check_launch("cg_scale_div_kernel"));
        double lam_new = 0.0;
        KZ_TRY(rayleigh(v, &lam_new));
        const bool done = std::fabs(lam_new - lam) <= tol * lam_new;
        lam = lam_new;
        if (done) {
            ok = true;
            break;
        }
    }
    if (!ok) return fail(KZ_ESPECTRAL, "sigma_max: power iteration did not converge");
    out[0] = lam;
    // ---- lambda_min: inverse iteration, CG on A^T A y = v (spectral.py:97-115, 36-57)
    KZ_CUDA(cudaMemcpyAsync(v, v1_host, n * sizeof(double), cudaMemcpyHostToDevice, st));
    double theta = 0.0;
    KZ_TRY(rayleigh(v, &theta));
    const int64_t cg_max = 20 * n + 200;
    ok = false;
    for (int64_t it = 0; it < max_it; ++it) {
        // y = 0, r = v, p = v, rs = <r, r>, stop = (tol ||v||)^2
        KZ_CUDA(cudaMemsetAsync(y, 0, ld * sizeof(double), st));
        KZ_CUDA(cudaMemcpyAsync(r, v, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        KZ_CUDA(cudaMemcpyAsync(p, v, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
        double rs = 0.0;
        KZ_TRY(dot(r, r, n, 0, &rs));
        const double stop = (tol * std::sqrt(rs)) * (tol * std::sqrt(rs));
        bool cg_ok = false;
        for (int64_t k = 0; k < cg_max; ++k) {
            if (rs <= stop) {
                cg_ok = true;
                break;
            }
            KZ_TRY(Av(p, t));
            KZ_TRY(ATv(t, mp));
            double den = 0.0;
            KZ_TRY(dot(p, mp, n, 1, &den));
            if (den <= 0.0) break;
            cg_update_xr_kernel<<<eblocks, 256, 0, st>>>(y, p, r, mp, scal, n, n);  // alpha = rs / den
            KZ_TRY(check_launch("cg_update_xr_kernel"));
            double rs_new = 0.0;
            KZ_TRY(dot(r, r, n, 2, &rs_new));
            cg_update_p_kernel<<<eblocks, 256, 0, st>>>(p, r, scal, n);  // p = r + (rs_new / rs) p
            KZ_TRY(check_launch("cg_update_p_kernel"));
            KZ_CUDA(cudaMemcpyAsync(scal, scal + 2, sizeof(double), cudaMemcpyDeviceToDevice, st));
            rs = rs_new;
        }
        if (!cg_ok && !(rs <= stop)) return fail(KZ_ESPECTRAL, "sigma_min: inner CG solve failed");
        double ny2 = 0.0;
        KZ_TRY(dot(y, y, n, 4, &ny2));
        const double ny = std::sqrt(ny2);
        if (ny == 0.0) return fail(KZ_ESPECTRAL, "sigma_min: inverse iteration collapsed");
        KZ_CUDA(cudaMemcpyAsync(scal + 4, &ny, sizeof(double), cudaMemcpyHostToDevice, st));
        cg_scale_div_kernel<<<eblocks, 256, 0, st>>>(y, scal + 4, n, v);
        KZ_TRY(check_launch("cg_scale_div_kernel"));
        double theta_new = 0.0;
        KZ_TRY(rayleigh(v, &theta_new));
        const bool done = it >= 2 && std::fabs(theta_new - theta) <= tol * theta_new;
        theta = theta_new;
        if (done) {
            ok = true;
            break;
        }
    }
    if (!ok) return fail(KZ_ESPECTRAL, "sigma_min: inverse iteration did not converge");
    out[1] = theta;
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// KZSYS v1 system files (sysgen.py:190-271 save_system / load_system), read
// straight into device memory.  Layout: "KZSYS", u8 version = 1, u64 m, u64 n,
// u32 flags (1 consistent, 2 x_star, 4 x_ls, 8 generator metadata), [u64 seed,
// f64 mu_lo, mu_hi, sigma_lo, sigma_hi], A (m x n f64 LE, row-major), b (m),
// [x_star (n)], [x_ls (n)].  Rows [row_lo, row_hi] (a GPU's shard) stream from
// the file through two pinned buffers: pread of chunk c+1 overlaps the H2D copy
// and the device repack of chunk c into the 128-byte row pitch.
// ---------------------------------------------------------------------------
extern "C" int32_t kz_system_load_file(int32_t device, const char* path, int64_t row_lo, int64_t row_hi,
                                       kz_system** out, int64_t* m_total, int64_t* n_out, uint32_t* flags_out,
                                       double* meta5) {
    NvtxScope nvtx_("kz_system_load_file");
    if (!path || !out) return fail(KZ_EINVAL, "null argument");
    *out = nullptr;
    const int fd = open(path, O_RDONLY);
    if (fd < 0) return fail(KZ_EINVAL, "cannot open %s", path);
    struct Closer {
        int fd;
        ~Closer() { close(fd); }
    } closer{fd};
    auto read_at = [&](void* dst, size_t bytes, off_t off) -> bool {
        size_t got = 0;
        while (got < bytes) {
            const ssize_t r = pread(fd, (char*)dst + got, bytes - got, off + (off_t)got);
            if (r <= 0) return false;
            got += (size_t)r;
        }
        return true;
    };
    unsigned char head[26];
    if (!read_at(head, 5, 0)) return fail(KZ_EFORMAT, "truncated file while reading magic (offset 0)");
    if (memcmp(head, "KZSYS", 5) != 0) return fail(KZ_EFORMAT, "bad magic (offset 0)");
    if (!read_at(head + 5, 1, 5)) return fail(KZ_EFORMAT, "truncated file while reading version (offset 5)");
    if (head[5] != 1) return fail(KZ_EVERSION, "unsupported system file version %d (expected 1) (offset 5)", head[5]);
    if (!read_at(head + 6, 20, 6)) return fail(KZ_EFORMAT, "truncated file while reading header (offset 6)");
    uint64_t m, n;
    uint32_t flags;
    memcpy(&m, head + 6, 8);
    memcpy(&n, head + 14, 8);
    memcpy(&flags, head + 22, 4);
    if (m < 1 || n < 1) return fail(KZ_EFORMAT, "bad dimensions %llux%llu (offset 6)", (unsigned long long)m,
                                    (unsigned long long)n);
    off_t off = 26;
    double meta[5] = {-1.0, -5.0, 5.0, 1.0, 20.0};
    if (flags & 8u) {
        unsigned char g[40];
        if (!read_at(g, 40, off)) return fail(KZ_EFORMAT, "truncated file while reading generator metadata (offset %lld)",
                                              (long long)off);
        uint64_t seed;
        memcpy(&seed, g, 8);
        meta[0] = (double)seed;
        memcpy(meta + 1, g + 8, 32);
        off += 40;
    }
    if (row_hi < 0) row_hi = (int64_t)m - 1;
    if (row_lo < 0 || row_lo > row_hi || row_hi >= (int64_t)m) return fail(KZ_EINVAL, "bad row range");
    const int64_t rows = row_hi - row_lo + 1;
    const off_t a_off = off, b_off = a_off + (off_t)(m * n * 8), xs_off = b_off + (off_t)(m * 8);
    const off_t xl_off = xs_off + ((flags & 2u) ? (off_t)(n * 8) : 0);
    const off_t end = xl_off + ((flags & 4u) ? (off_t)(n * 8) : 0);
    if (lseek(fd, 0, SEEK_END) < end) return fail(KZ_EFORMAT, "truncated file (needs %lld bytes)", (long long)end);
    kz_system* s = nullptr;
    KZ_TRY(kz_system_create(device, rows, (int64_t)n, &s));
    struct Guard {
        kz_system*& s;
        bool keep = false;
        ~Guard() {
            if (!keep && s) kz_system_destroy(s);
        }
    } guard{s};
    cudaStream_t st = nullptr;
    // chunked rows: <= 64 MiB per chunk
    const int64_t chunk_rows = std::max<int64_t>(1, std::min<int64_t>(rows, ((int64_t)64 << 20) / (int64_t)(n * 8)));
    double* pin[2] = {nullptr, nullptr};
    for (auto& p : pin)
        if (cudaMallocHost(&p, (size_t)chunk_rows * n * 8) != cudaSuccess) {
            cudaGetLastError();
            for (auto& q : pin)
                if (q) cudaFreeHost(q);
            return fail(KZ_ENOMEM, "pinned staging allocation failed");
        }
    struct PinFree {
        double** p;
        ~PinFree() {
            for (int i = 0; i < 2; ++i)
                if (p[i]) cudaFreeHost(p[i]);
        }
    } pinfree{pin};
    KZ_TRY(s->stage.ensure((size_t)2 * chunk_rows * n));
    cudaEvent_t done[2];
    cudaEventCreate(&done[0]);
    cudaEventCreate(&done[1]);
    int rc = KZ_OK;
    int64_t c = 0;
    for (int64_t r0 = 0; r0 < rows && rc == KZ_OK; r0 += chunk_rows, ++c) {
        const int64_t nr = std::min<int64_t>(chunk_rows, rows - r0);
        const int k = (int)(c & 1);
        cudaEventSynchronize(done[k]);  // the copy out of this pinned buffer two chunks ago is done
        if (!read_at(pin[k], (size_t)nr * n * 8, a_off + (off_t)((row_lo + r0) * (int64_t)n * 8))) {
            rc = fail(KZ_EFORMAT, "truncated file while reading matrix rows");
            break;
        }
        double* dst = s->stage.p + (size_t)k * chunk_rows * n;
        if (cudaMemcpyAsync(dst, pin[k], (size_t)nr * n * 8, cudaMemcpyHostToDevice, st) != cudaSuccess) {
            rc = fail(KZ_ECUDA, "H2D copy failed");
            break;
        }
        const int64_t total = nr * s->ld;
        repack_rows_kernel<<<(unsigned)std::min<int64_t>((total + 255) / 256, (int64_t)s->sms * 32), 256, 0, st>>>(
            dst, nr, (int64_t)n, s->ld, s->A.p + r0 * s->ld);
        cudaEventRecord(done[k], st);
    }
    cudaStreamSynchronize(st);
    cudaEventDestroy(done[0]);
    cudaEventDestroy(done[1]);
    KZ_TRY(rc);
    KZ_TRY(check_launch("repack_rows_kernel"));
    std::vector<double> hb((size_t)rows), hx((size_t)n);
    if (!read_at(hb.data(), (size_t)rows * 8, b_off + (off_t)(row_lo * 8)))
        return fail(KZ_EFORMAT, "truncated file while reading constants");
    KZ_CUDA(cudaMemcpy(s->b.p, hb.data(), (size_t)rows * 8, cudaMemcpyHostToDevice));
    s->has_xref = false;
    if (flags & 6u) {  // x_ref: x_star if present, else x_ls (LinearSystem.x_ref)
        if (!read_at(hx.data(), (size_t)n * 8, (flags & 2u) ? xs_off : xl_off))
            return fail(KZ_EFORMAT, "truncated file while reading the solution vector");
        KZ_CUDA(cudaMemcpy(s->xref.p, hx.data(), (size_t)n * 8, cudaMemcpyHostToDevice));
        s->has_xref = true;
    }
    s->norms_valid = false;
    s->bs2_valid = false;
    s->sampler_scheme = -1;
    if (m_total) *m_total = (int64_t)m;
    if (n_out) *n_out = (int64_t)n;
    if (flags_out) *flags_out = flags;
    if (meta5) memcpy(meta5, meta, sizeof(meta));
    guard.keep = true;
    *out = s;
    return KZ_OK;
}


// ---------------------------------------------------------------------------
// Row-sharded multi-GPU solve (distributed.py:282-363 generalised to q workers
// per rank; BASELINE config 3).  One process per GPU; the ranks' worker sums
// are all-reduced in place by NCCL over NVLink on the solve stream.
// ---------------------------------------------------------------------------
namespace {
struct NcclApi {
    bool tried = false, ok = false;
    std::string why;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};
NcclApi g_nccl;

int nccl_load() {
    if (g_nccl.tried) return g_nccl.ok ? KZ_OK : fail(KZ_ENODEV, "%s", g_nccl.why.c_str());
    g_nccl.tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_nccl.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
        return fail(KZ_ENODEV, "%s", g_nccl.why.c_str());
    }
    g_nccl.get_unique_id = (decltype(g_nccl.get_unique_id))dlsym(h, "ncclGetUniqueId");
    g_nccl.comm_init_rank = (decltype(g_nccl.comm_init_rank))dlsym(h, "ncclCommInitRank");
    g_nccl.all_reduce = (decltype(g_nccl.all_reduce))dlsym(h, "ncclAllReduce");
    g_nccl.comm_destroy = (decltype(g_nccl.comm_destroy))dlsym(h, "ncclCommDestroy");
    g_nccl.error_string = (decltype(g_nccl.error_string))dlsym(h, "ncclGetErrorString");
    if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.all_reduce || !g_nccl.comm_destroy ||
        !g_nccl.error_string) {
        g_nccl.why = "libnccl.so.2 lacks the NCCL 2 entry points";
        return fail(KZ_ENODEV, "%s", g_nccl.why.c_str());
    }
    g_nccl.ok = true;
    return KZ_OK;
}

#define KZ_NCCL(call)                                                                                   \
    do {                                                                                                \
        ncclResult_t r_ = (call);                                                                       \
        if (r_ != ncclSuccess) return fail(KZ_ECUDA, "%s failed: %s", #call, g_nccl.error_string(r_)); \
    } while (0)
}  // namespace

struct kz_comm {
    int device = 0, world = 1, rank = 0;
    ncclComm_t nccl = nullptr;
    // cross-rank exchange of the fused row-sharded kernel (rka kernel mode 2): every rank's buffer
    // of tagged column sums [parity][rank][column], reachable from every GPU over NVLink
    unsigned long long* xbuf = nullptr;  // this rank's buffer (cudaMalloc, exported by IPC)
    int64_t xld = 0;                     // row pitch the buffers are sized for
    std::vector<void*> opened;           // peers' buffers mapped with cudaIpcOpenMemHandle
    unsigned long long** peers_dev = nullptr;  // device array of the world's buffers
    bool xr_ready = false;
    unsigned tag_next = 1;  // next tag: advanced identically on every rank, never reused
};

extern "C" int32_t kz_comm_unique_id(uint8_t* id_out) {
    if (!id_out) return fail(KZ_EINVAL, "null argument");
    static_assert(sizeof(ncclUniqueId) == KZ_COMM_ID_BYTES, "NCCL unique id size");
    KZ_TRY(nccl_load());
    ncclUniqueId id;
    KZ_NCCL(g_nccl.get_unique_id(&id));
    memcpy(id_out, &id, sizeof(id));
    return KZ_OK;
}

extern "C" int32_t kz_comm_create(int32_t device, const uint8_t* id, int32_t world, int32_t rank, kz_comm** out) {
    NvtxScope nvtx_("kz_comm_create");
    if (!id || !out) return fail(KZ_EINVAL, "null argument");
    if (world < 1 || rank < 0 || rank >= world) return fail(KZ_EINVAL, "rank %d out of range for world %d", rank, world);
    *out = nullptr;
    KZ_TRY(nccl_load());
    KZ_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    kz_comm* c = new kz_comm;
    c->device = device;
    c->world = world;
    c->rank = rank;
    ncclResult_t r = g_nccl.comm_init_rank(&c->nccl, world, uid, rank);
    if (r != ncclSuccess) {
        delete c;
        return fail(KZ_ECUDA, "ncclCommInitRank failed: %s", g_nccl.error_string(r));
    }
    *out = c;
    return KZ_OK;
}

extern "C" int32_t kz_comm_exchange_handle(kz_comm* c, int64_t ld, uint8_t* handle_out) {
    if (!c || !handle_out) return fail(KZ_EINVAL, "null argument");
    if (ld < 1) return fail(KZ_EINVAL, "ld must be >= 1");
    if (c->world > RKA_MAXR) return fail(KZ_EINVAL, "the fused exchange covers up to %d ranks", RKA_MAXR);
    static_assert(sizeof(cudaIpcMemHandle_t) == KZ_COMM_HANDLE_BYTES, "IPC handle size");
    KZ_CUDA(cudaSetDevice(c->device));
    if (c->xbuf && c->xld != ld) return fail(KZ_EINVAL, "exchange buffer already sized for pitch %lld", (long long)c->xld);
    if (!c->xbuf) {
        const size_t words = 4 * (size_t)c->world * (size_t)ld;  // [2 parities][world][ld] x 2 words
        KZ_CUDA(cudaMalloc(&c->xbuf, words * sizeof(unsigned long long)));
        KZ_CUDA(cudaMemset(c->xbuf, 0, words * sizeof(unsigned long long)));  // tag 0 is never used
        c->xld = ld;
    }
    cudaIpcMemHandle_t h;
    KZ_CUDA(cudaIpcGetMemHandle(&h, c->xbuf));
    memcpy(handle_out, &h, sizeof(h));
    return KZ_OK;
}

extern "C" int32_t kz_comm_exchange_connect(kz_comm* c, const uint8_t* handles) {
    NvtxScope nvtx_("kz_comm_exchange_connect");
    if (!c || !handles) return fail(KZ_EINVAL, "null argument");
    if (!c->xbuf) return fail(KZ_EINVAL, "kz_comm_exchange_handle first");
    KZ_CUDA(cudaSetDevice(c->device));
    std::vector<unsigned long long*> ptrs(c->world);
    for (int r = 0; r < c->world; ++r) {
        if (r == c->rank) {
            ptrs[r] = c->xbuf;
            continue;
        }
        cudaIpcMemHandle_t h;
        memcpy(&h, handles + (size_t)r * KZ_COMM_HANDLE_BYTES, sizeof(h));
        void* p = nullptr;
        KZ_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->opened.push_back(p);
        ptrs[r] = reinterpret_cast<unsigned long long*>(p);
    }
    if (!c->peers_dev) KZ_CUDA(cudaMalloc(&c->peers_dev, RKA_MAXR * sizeof(unsigned long long*)));
    KZ_CUDA(cudaMemcpy(c->peers_dev, ptrs.data(), c->world * sizeof(unsigned long long*), cudaMemcpyHostToDevice));
    c->xr_ready = true;
    return KZ_OK;
}

extern "C" int32_t kz_comm_destroy(kz_comm* c) {
    if (!c) return KZ_OK;
    cudaSetDevice(c->device);
    for (void* p : c->opened) cudaIpcCloseMemHandle(p);
    if (c->peers_dev) cudaFree(c->peers_dev);
    if (c->xbuf) cudaFree(c->xbuf);
    if (c->nccl && g_nccl.ok) {
        cudaSetDevice(c->device);
        g_nccl.comm_destroy(c->nccl);
    }
    delete c;
    return KZ_OK;
}

extern "C" int32_t kz_solve_sharded(kz_system* s, kz_comm* comm, const kz_params* p, kz_result* r, double* x_host,
                                    void* stream) {
    NvtxScope nvtx_("kz_solve_sharded");
    if (!s || !p || !r) return fail(KZ_EINVAL, "null argument");
    memset(r, 0, sizeof(*r));
    r->final_error_sq = NAN;
    r->final_residual = NAN;
    if (p->variant != KZ_RKA && p->variant != KZ_RKAB)
        return fail(KZ_EINVAL, "row-sharded solves run RKA or RKAB (variant %d)", p->variant);
    if (p->trace_step > 0) return fail(KZ_EINVAL, "row-sharded solves have no trace mode");
    if (p->ckpt_every > 0 && comm) return fail(KZ_EINVAL, "row-sharded solves have no checkpoint mode");
    if (comm && comm->device != s->device)
        return fail(KZ_EINVAL, "communicator on device %d, shard on device %d", comm->device, s->device);
    const int world = comm ? comm->world : 1;
    if (!comm && !(p->flags & KZ_FLAG_SHARDED_LOOP)) {
        // one rank and no communicator: the local sum is the whole sum, x = S / q is kz_solve's
        // in-kernel average, so the chunked single-GPU driver runs the identical iteration
        kz_params pp = *p;
        pp.partial_dev = nullptr;
        pp.k_start = 0;
        pp.keep_x = 0;
        return kz_solve(s, &pp, r, x_host, stream);
    }
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    KZ_TRY(s->S.ensure(2 * s->ld));  // two worker-sum buffers: step k writes S[k % 2], reads S[(k - 1) % 2]
    KZ_CUDA(cudaMemsetAsync(s->S.p, 0, 2 * s->ld * sizeof(double), st));  // the padded tails stay zero
    kz_params pp = *p;
    pp.partial_dev = s->S.p;
    SolveCtx cx;
    cx.sharded = true;
    KZ_TRY(solve_setup(s, &pp, r, st, cx));
    SolveArgs& args = cx.args;
    args.use_stop = 0;  // the stop rule runs on the averaged x, after the collective
    args.final_check = 0;
    args.count = 1;
    const bool stop_mode = cx.stop_mode, chain = cx.pl.kernel == KZ_KERNEL_CHAIN;
    const int64_t q = cx.q, bs = cx.bs, Q = q * world;
    const int64_t limit = cx.budget_mode ? p->budget : p->max_iterations;
    const int64_t chunk_max = std::min<int64_t>(cx.chunk_cap, 1024);
    KZ_TRY(s->errs.ensure(chunk_max + 1));
    KZ_TRY(s->halt.ensure(1));
    KZ_CUDA(cudaMemsetAsync(s->halt.p, 0, sizeof(int), st));
    args.halt = s->halt.p;
    std::vector<double> herr(chunk_max + 1);
    int hhalt = 0;
    int32_t* const idx0 = s->idx.p;
    const long long launches0 = g_launches.load();

    int64_t k = 0, evals = 0;
    bool converged = false;
    double err = NAN;
    // fused cross-rank path (RKA on the rka kernel, communicator connected): the step kernel runs a
    // whole chunk of outer iterations, exchanging column sums with the other ranks over NVLink peer
    // memory every iteration and applying the stop rule itself -- like kz_solve's chunked loop
    const bool xr = cx.pl.tma && comm && comm->xr_ready && bs == 1 && comm->xld == s->ld &&
                    !(p->flags & KZ_FLAG_NO_FUSED_EXCHANGE);
    if (xr) {
        Plan& pl = cx.pl;
        pl.xr = true;
        void* fn = rka_fn(pl.lg, pl.epl, pl.sr, 2);
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem));
        KZ_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        KZ_CUDA(cudaMemsetAsync(&s->status.p->aborted, 0, sizeof(int), st));
        args.partial = nullptr;
        args.x_sum = nullptr;
        args.halt = nullptr;
        args.use_stop = stop_mode ? 1 : 0;
        args.x_div = (double)Q;
        args.xr_peers = comm->peers_dev;
        args.xr_ranks = world;
        args.xr_rank = comm->rank;
        args.idx = idx0;
        args.idx_stride = q;
        KZ_CUDA(cudaEventRecord(s->ev[0], st));
        int64_t chunkf = stop_mode ? std::min<int64_t>(cx.chunk_cap, 4096) : cx.chunk_cap;
        for (;;) {
            const int64_t remaining = limit - k;
            if (remaining <= 0 && !stop_mode) break;
            const int64_t c = std::min<int64_t>(chunkf, remaining);
            if (c > 0) KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, q, p->k_start + k, c, idx0, 1, q, st));
            args.k0 = k;
            args.count = c;
            args.final_check = (stop_mode && k + c == p->max_iterations) ? 1 : 0;
            args.xr_tag0 = comm->tag_next;  // every rank launches the same counts: tags agree
            comm->tag_next += (unsigned)c + 1u;
            KZ_TRY(launch_step(s, &pp, r, cx, k == 0, st));
            KZ_CUDA(cudaMemcpyAsync(s->h_status, s->status.p, sizeof(SolveStatus), cudaMemcpyDeviceToHost, st));
            KZ_CUDA(cudaStreamSynchronize(st));
            const SolveStatus hs = *s->h_status;
            if (hs.aborted) return fail(KZ_ECUDA, "cross-rank exchange timed out (a rank stopped launching)");
            k += hs.iters_done;
            evals += hs.checks;
            if (hs.checks > 0) err = hs.err;
            if (hs.converged) {
                converged = true;
                break;
            }
            if (hs.iters_done != c)
                return fail(KZ_ECUDA, "solve kernel stopped early (%lld of %lld iterations)", (long long)hs.iters_done,
                            (long long)c);
            if (stop_mode && k >= p->max_iterations) break;
            if (stop_mode) chunkf = std::min<int64_t>(cx.chunk_cap, chunkf * 2);
        }
    } else if (stop_mode) {  // _drive's check before iteration 0 (x_0 = 0 or the kept iterate)
        KZ_TRY(error_sq_dev(s, &err, st));
        evals = 1;
        converged = err < p->epsilon;
    }
    if (!xr) KZ_CUDA(cudaEventRecord(s->ev[0], st));
    // rka kernel: x_k = S / Q, the stop rule and the halt flag live in the step kernel itself (one
    // kernel + one collective per outer iteration); chain kernel (RKAB): separate average kernel
    const bool fused = cx.pl.tma;
    if (fused) {
        args.use_stop = stop_mode ? 1 : 0;
        args.x_div = (double)Q;
    }
    // chunks never exceed chunk_max: the row-index buffer holds chunk_cap iterations of draws and
    // the error buffers chunk_max + 1 values
    int64_t chunk = stop_mode ? std::min<int64_t>(64, chunk_max) : chunk_max;
    const int64_t ck_cap = (!comm && p->ckpt_every > 0) ? cx.n_ck_cap : 0;  // waves of one GPU: checkpoints
    if (ck_cap > 0 && fused) return fail(KZ_EINVAL, "checkpoints of the per-iteration rka loop");
    while (!xr && !converged && k < limit) {
        const int64_t c = std::min<int64_t>(chunk, limit - k);
        // row draws of the whole chunk: one sampler launch (x-independent)
        const int64_t count = c * bs;
        if (chain)
            KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, q, (p->k_start + k) * bs, count, idx0, count, 1,
                                  st));
        else
            KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, q, (p->k_start + k) * bs, count, idx0, 1, q, st));
        for (int64_t i = 0; i < c; ++i) {
            const int64_t kk = k + i;
            double* Sk = s->S.p + (kk & 1) * s->ld;
            args.k0 = kk;
            args.idx = chain ? idx0 + i * bs : idx0 + i * q;
            args.idx_stride = chain ? count : q;
            args.partial = Sk;
            if (fused) args.x_sum = kk == 0 ? nullptr : s->S.p + ((kk - 1) & 1) * s->ld;  // x_0: resident
            KZ_TRY(launch_waves(s, &pp, r, cx, kk == 0, st));
            if (comm) KZ_NCCL(g_nccl.all_reduce(Sk, Sk, (size_t)s->ld, ncclFloat64, ncclSum, comm->nccl, st));
            if (!fused) {
                shard_average_kernel<<<1, 1024, 0, st>>>(Sk, (double)Q, s->n, s->ld, s->xref.p, s->x.p, p->epsilon,
                                                         stop_mode ? 1 : 0, kk + 1, s->errs.p + i, s->halt.p);
                KZ_TRY(check_launch("shard_average_kernel"));
                if (ck_cap > 0 && (kk + 1) % p->ckpt_every == 0 && (kk + 1) / p->ckpt_every <= ck_cap)
                    KZ_CUDA(cudaMemcpyAsync(s->ckpt.p + ((kk + 1) / p->ckpt_every - 1) * s->n, s->x.p,
                                            s->n * sizeof(double), cudaMemcpyDeviceToDevice, st));
            }
        }
        const bool last_chunk = k + c >= limit;
        if (fused && last_chunk) {  // x_K = S / Q and the check before iteration K
            shard_average_kernel<<<1, 1024, 0, st>>>(s->S.p + ((k + c - 1) & 1) * s->ld, (double)Q, s->n, s->ld,
                                                     s->xref.p, s->x.p, p->epsilon, stop_mode ? 1 : 0, k + c,
                                                     s->errs.p + c - 1, s->halt.p);
            KZ_TRY(check_launch("shard_average_kernel"));
        }
        // one host synchronisation per chunk: the errors, the stop flag and the kernel status
        KZ_CUDA(cudaMemcpyAsync(herr.data(), s->errs.p, c * sizeof(double), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaMemcpyAsync(&hhalt, s->halt.p, sizeof(int), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaMemcpyAsync(s->h_status, s->status.p, sizeof(SolveStatus), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        if (cx.pl.tma && cx.pl.ctas > cx.pl.cluster && s->h_status->aborted)
            return fail(KZ_ECUDA, "cross-cluster exchange timed out (clusters not co-resident)");
        if (hhalt != 0) {  // x_{hhalt - 1} met the rule; the launches after it were no-ops
            const int64_t ks = hhalt - 1;
            // the stopping kernel's own error total, or the average kernel's
            err = (fused && ks < k + c) ? s->h_status->err : herr[ks - k - 1];
            if (fused && ks < k + c && ks > 0) {
                // the stopping step kernel left x alone: x_ks = S[(ks - 1) % 2] / Q (intact -- that
                // kernel wrote S[ks % 2]); no stop check, no flag
                shard_average_kernel<<<1, 1024, 0, st>>>(s->S.p + ((ks - 1) & 1) * s->ld, (double)Q, s->n, s->ld,
                                                         s->xref.p, s->x.p, p->epsilon, 0, ks, s->errs.p + chunk_max,
                                                         nullptr);
                KZ_TRY(check_launch("shard_average_kernel"));
            }
            k = ks;
            evals = k + 1;
            converged = true;
            break;
        }
        k += c;
        if (!fused || last_chunk) err = herr[c - 1];
        if (stop_mode) evals = k + 1;
        chunk = std::min<int64_t>(chunk_max, chunk * 2);
    }
    KZ_CUDA(cudaEventRecord(s->ev[1], st));
    KZ_CUDA(cudaEventSynchronize(s->ev[1]));
    float loop_ms = 0.f;
    cudaEventElapsedTime(&loop_ms, s->ev[0], s->ev[1]);
    r->iterations = k;
    r->converged = converged ? 1 : 0;
    r->error_evals = stop_mode ? evals : 0;
    r->final_error_sq = stop_mode ? err : NAN;
    r->rows_projected = k * q * bs;  // this rank's projections
    r->loop_ms = loop_ms;
    r->kernel_ms = loop_ms;  // steps, collectives and averages interleave on one stream
    r->kernel_used = cx.pl.tma ? KZ_KERNEL_RKA : cx.pl.kernel;
    r->ctas = cx.pl.ctas;
    r->threads = cx.pl.threads;
    if (ck_cap > 0) {
        r->n_ckpt = std::min<int64_t>(ck_cap, k / p->ckpt_every);
        if (r->n_ckpt > 0 && p->ckpt_host)
            KZ_CUDA(cudaMemcpyAsync(p->ckpt_host, s->ckpt.p, (size_t)r->n_ckpt * s->n * sizeof(double),
                                    cudaMemcpyDeviceToHost, st));
    }
    r->plan_ep = cx.pl.kernel == KZ_KERNEL_CHAIN ? cx.pl.ep : cx.pl.epl;
    r->plan_rows = cx.pl.kernel == KZ_KERNEL_CHAIN ? cx.pl.rows : 1;
    r->plan_cluster = cx.pl.kernel == KZ_KERNEL_CHAIN ? cx.pl.pair : cx.pl.cluster;
    r->plan_stages = cx.pl.stages;
    r->plan_waves = cx.pl.waves;
    if (x_host) KZ_CUDA(cudaMemcpyAsync(x_host, s->x.p, s->n * sizeof(double), cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    r->kernel_launches = g_launches.load() - launches0;
    return KZ_OK;
}

// ---------------------------------------------------------------------------
// Many seeds of one RK configuration in one launch per chunk (the 10 seeds of BASELINE config 0:
// harness.measure_iterations, harness.py:127-149).  Each seed is one block of the one-warp RK
// kernel with its own iterate, row draws (stream Prng(seed, 0)), status and stop flag; a seed
// that meets the stop rule drops out of later launches.  Short rows only (the warp kernel).
// ---------------------------------------------------------------------------
extern "C" int32_t kz_solve_seeds(kz_system* s, const kz_params* p, const uint64_t* seeds, int64_t S,
                                  kz_result* results, double* x_host, void* stream) {
    NvtxScope nvtx_("kz_solve_seeds");
    if (!s || !p || !seeds || !results) return fail(KZ_EINVAL, "null argument");
    if (S < 1) return fail(KZ_EINVAL, "need at least one seed");
    if (p->variant != KZ_RK) return fail(KZ_EINVAL, "kz_solve_seeds runs RK (variant %d)", p->variant);
    if (s->ld > 256) return fail(KZ_EINVAL, "kz_solve_seeds covers rows of at most 256 columns");
    if (p->trace_step > 0 || p->ckpt_every > 0 || p->partial_dev)
        return fail(KZ_EINVAL, "kz_solve_seeds has no trace, checkpoint or partial mode");
    if (!(p->epsilon > 0)) return fail(KZ_EINVAL, "epsilon must be > 0, got %g", p->epsilon);
    if (p->max_iterations < 1) return fail(KZ_EINVAL, "max_iterations must be >= 1, got %lld", (long long)p->max_iterations);
    const bool budget_mode = p->budget > 0, stop_mode = !budget_mode;
    if (stop_mode && !s->has_xref) return fail(KZ_EINVAL, "system carries no reference solution");
    cudaStream_t st = pick_stream(s, stream);
    KZ_CUDA(cudaSetDevice(s->device));
    for (int64_t i = 0; i < S; ++i) {
        memset(&results[i], 0, sizeof(kz_result));
        results[i].final_error_sq = NAN;
        results[i].final_residual = NAN;
    }
    // one full-access range per seed: the RK sampler (q = 1) for every stream
    KZ_TRY(ensure_sampler(s, KZ_FULL_ACCESS, S, st));
    KZ_TRY(ensure_bs2(s, st));
    {
        std::vector<PcgPod> pods(S);
        for (int64_t i = 0; i < S; ++i) pods[i] = seed_stream(seeds[i], (uint64_t)p->worker_offset);
        KZ_TRY(s->states.ensure(S));
        KZ_CUDA(cudaMemcpyAsync(s->states.p, pods.data(), S * sizeof(PcgPod), cudaMemcpyHostToDevice, st));
        s->pods_q = -1;  // kz_solve's cached streams are overwritten
    }
    const double alpha = p->alphas_host ? p->alphas_host[0] : 1.0;
    KZ_TRY(s->alphas.ensure(1));
    KZ_CUDA(cudaMemcpyAsync(s->alphas.p, &alpha, sizeof(double), cudaMemcpyHostToDevice, st));
    s->alphas_cache.clear();
    const int64_t chunk_max = 4096;
    KZ_TRY(s->xs.ensure((size_t)S * s->ld));
    KZ_CUDA(cudaMemsetAsync(s->xs.p, 0, (size_t)S * s->ld * sizeof(double), st));
    KZ_TRY(s->idx.ensure((size_t)S * chunk_max));
    KZ_TRY(s->status.ensure(S));
    KZ_TRY(s->halt.ensure(S));
    KZ_CUDA(cudaMemsetAsync(s->halt.p, 0, S * sizeof(int), st));
    std::vector<SolveStatus> hs(S);
    std::vector<int> hh(S, 0);
    std::vector<int64_t> iters(S, 0), evals(S, 0);
    std::vector<double> errv(S, NAN);
    std::vector<int> conv(S, 0);

    const int epl = s->ld <= 64 ? 1 : (s->ld <= 128 ? 2 : 4);
    void* fn = rkw_fn(epl);
    SolveArgs args = {};
    args.A = s->A.p;
    args.b = s->b.p;
    args.sq = s->sq.p;
    args.bs2 = s->bs2.p;
    args.xref = s->xref.p;
    args.x = s->xs.p;
    args.idx = s->idx.p;
    args.alphas = s->alphas.p;
    args.status = s->status.p;
    args.halt = s->halt.p;
    args.n = s->n;
    args.ld = s->ld;
    args.q = 1;
    args.bs = 1;
    args.eps = p->epsilon;
    args.use_stop = stop_mode ? 1 : 0;
    const long long launches0 = g_launches.load();
    const int64_t limit = budget_mode ? p->budget : p->max_iterations;
    KZ_CUDA(cudaEventRecord(s->ev[0], st));
    int64_t k = 0, active = S;
    for (;;) {
        const int64_t remaining = limit - k;
        if (remaining <= 0 && !stop_mode) break;
        const int64_t c = std::min<int64_t>(chunk_max, remaining);
        if (c > 0) KZ_TRY(launch_sampler(s, s->states.p, s->lo.p, s->len.p, S, k, c, s->idx.p, c, 1, st));
        args.k0 = k;
        args.count = c;
        args.idx_stride = c;
        args.final_check = (stop_mode && k + c == p->max_iterations) ? 1 : 0;
        void* kargs[] = {&args};
        KZ_CUDA(cudaLaunchKernel(fn, dim3((unsigned)S), dim3(32), kargs, 0, st));
        g_launches.fetch_add(1, std::memory_order_relaxed);
        KZ_CUDA(cudaMemcpyAsync(hs.data(), s->status.p, S * sizeof(SolveStatus), cudaMemcpyDeviceToHost, st));
        KZ_CUDA(cudaStreamSynchronize(st));
        bool newly = false;
        for (int64_t i = 0; i < S; ++i) {
            if (hh[i]) continue;
            iters[i] = k + hs[i].iters_done;
            evals[i] += hs[i].checks;
            if (hs[i].checks > 0) errv[i] = hs[i].err;
            if (hs[i].converged) {
                conv[i] = 1;
                hh[i] = 1;
                --active;
                newly = true;
            } else if (hs[i].iters_done != c) {
                return fail(KZ_ECUDA, "seed %lld stopped early (%lld of %lld iterations)", (long long)i,
                            (long long)hs[i].iters_done, (long long)c);
            }
        }
        k += c;
        if (active == 0 || (stop_mode && k >= p->max_iterations)) break;
        if (newly) KZ_CUDA(cudaMemcpyAsync(s->halt.p, hh.data(), S * sizeof(int), cudaMemcpyHostToDevice, st));
    }
    KZ_CUDA(cudaEventRecord(s->ev[1], st));
    KZ_CUDA(cudaEventSynchronize(s->ev[1]));
    float loop_ms = 0.f;
    cudaEventElapsedTime(&loop_ms, s->ev[0], s->ev[1]);
    for (int64_t i = 0; i < S; ++i) {
        kz_result& r = results[i];
        r.iterations = iters[i];
        r.converged = conv[i];
        r.error_evals = stop_mode ? evals[i] : 0;
        r.final_error_sq = stop_mode ? errv[i] : NAN;
        r.rows_projected = iters[i];
        r.loop_ms = loop_ms;
        r.kernel_ms = loop_ms;
        r.kernel_used = KZ_KERNEL_WARP;
        r.ctas = (int32_t)S;
        r.threads = 32;
        r.kernel_launches = g_launches.load() - launches0;
    }
    if (x_host)
        KZ_CUDA(cudaMemcpy2DAsync(x_host, s->n * sizeof(double), s->xs.p, s->ld * sizeof(double), s->n * sizeof(double),
                                  S, cudaMemcpyDeviceToHost, st));
    KZ_CUDA(cudaStreamSynchronize(st));
    return KZ_OK;
}
