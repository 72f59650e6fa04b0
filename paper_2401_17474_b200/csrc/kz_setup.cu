// kz_setup.cu -- one-time-per-system kernels: row norms, CDFs, row sampling,
// and the residual/error norms used by traces.
//
//   row_sqnorm_kernel  <- row_norm_cache  (linalg.py:80-88), bit-exact einsum order
//   cdf_scan_kernel    <- make_sampler    (sampling.py:108: np.cumsum, sequential)
//   cdf_div_kernel     <- make_sampler    (sampling.py:109: cdf /= cdf[-1])
//   sample_rows_kernel <- RowSampler.sample x Prng.random (sampling.py:50-52, 177-182)
//   residual kernels   <- _trace_record / final residual (solvers.py:174-179, 246)
#include "kz_kernels.cuh"

namespace kz {

// ---------------------------------------------------------------------------
// Row norms.  numpy 2.3.5's einsum "ij,ij->i" sum-of-products kernel keeps two
// f64 lanes; every full chunk of 8 elements updates lane l as
//     acc_l = e_l^2 + (e_{2+l}^2 + (e_{4+l}^2 + (e_{6+l}^2 + acc_l)))
// with separately rounded products and sums (no FMA), then consumes the tail
// in zero-filled pairs from low to high, and returns acc_0 + acc_1.
// One thread per row; a CTA stages a 128-row x 32-column tile in shared
// memory with coalesced loads (row pitch 33 doubles: 2-way = conflict-free
// for 8-byte lanes).  128 x 33 x 8 B = 33 KB of static shared memory.
// ---------------------------------------------------------------------------
constexpr int NORM_ROWS = 128;
constexpr int NORM_COLS = 32;

__global__ void __launch_bounds__(NORM_ROWS) row_sqnorm_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                                                int64_t ld, double* __restrict__ sq,
                                                                unsigned long long* __restrict__ first_zero) {
    __shared__ double tile[NORM_ROWS][NORM_COLS + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t row0 = (int64_t)blockIdx.x * NORM_ROWS;
    const int64_t my_row = row0 + tid;
    double l0 = 0.0, l1 = 0.0;
    const int64_t full_end = (n / 8) * 8;  // columns consumed by full chunks
    for (int64_t c0 = 0; c0 < n; c0 += NORM_COLS) {
        // coalesced tile load: warp w loads rows w, w+4, ...; lane = column
        for (int r = warp; r < NORM_ROWS; r += NORM_ROWS / 32) {
            const int64_t gr = row0 + r;
            tile[r][lane] = (gr < m && c0 + lane < ld) ? A[gr * ld + c0 + lane] : 0.0;
        }
        __syncthreads();
        if (my_row < m) {
            const double* e = tile[tid];
            const int64_t cend = (c0 + NORM_COLS < full_end) ? c0 + NORM_COLS : full_end;
            for (int64_t c = c0; c < cend; c += 8) {
                const int j = (int)(c - c0);
                l0 = __dadd_rn(__dmul_rn(e[j], e[j]),
                               __dadd_rn(__dmul_rn(e[j + 2], e[j + 2]),
                                         __dadd_rn(__dmul_rn(e[j + 4], e[j + 4]),
                                                   __dadd_rn(__dmul_rn(e[j + 6], e[j + 6]), l0))));
                l1 = __dadd_rn(__dmul_rn(e[j + 1], e[j + 1]),
                               __dadd_rn(__dmul_rn(e[j + 3], e[j + 3]),
                                         __dadd_rn(__dmul_rn(e[j + 5], e[j + 5]),
                                                   __dadd_rn(__dmul_rn(e[j + 7], e[j + 7]), l1))));
            }
            // tail pairs (zero-filled), only in the tile that holds them
            for (int64_t c = (full_end > c0 ? full_end : c0); c < n && c < c0 + NORM_COLS; c += 2) {
                const int j = (int)(c - c0);
                const double e0 = e[j];
                const double e1 = (c + 1 < n) ? e[j + 1] : 0.0;
                l0 = __dadd_rn(__dmul_rn(e0, e0), l0);
                l1 = __dadd_rn(__dmul_rn(e1, e1), l1);
            }
        }
        __syncthreads();
    }
    if (my_row < m) {
        const double s = __dadd_rn(l0, l1);
        sq[my_row] = s;
        if (s == 0.0) atomicMin(first_zero, (unsigned long long)my_row);
    }
}

// ---------------------------------------------------------------------------
// CDF: the sequential np.cumsum order (c_j = fl(c_{j-1} + sq_j)) per support
// range; ranges run in parallel (one CTA each).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(CDF_SCAN_THREADS) cdf_scan_kernel(const double* __restrict__ sq,
                                                                     const int64_t* __restrict__ lo,
                                                                     const int64_t* __restrict__ len, int64_t nranges,
                                                                     double* __restrict__ cdf) {
    // one CTA per support range.  The sum is strictly sequential (np.cumsum), so
    // one thread adds; the CTA streams the range through shared memory in
    // chunks (coalesced loads of chunk i+1 overlap the adds of chunk i) and
    // writes the partial sums back coalesced.  ~8 cycles per element (the DADD
    // latency) instead of one global-load latency per 8 elements.
    constexpr int CH = 2048;
    __shared__ double buf[2][CH];
    const int64_t r = blockIdx.x;
    if (r >= nranges) return;
    const int tid = threadIdx.x;
    const int64_t base = lo[r], L = len[r];
    const double* s = sq + base;
    double* c = cdf + base;
    for (int64_t j = tid; j < CH && j < L; j += CDF_SCAN_THREADS) buf[0][j] = s[j];
    __syncthreads();
    double acc = 0.0;
    int cur = 0;
    for (int64_t c0 = 0; c0 < L; c0 += CH) {
        const int n = (int)(L - c0 < CH ? L - c0 : CH);
        if (tid == 0) {
            double* b = buf[cur];
            int j = 0;
            for (; j + 8 <= n; j += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = b[j + u];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    acc = __dadd_rn(acc, v[u]);
                    b[j + u] = acc;
                }
            }
            for (; j < n; ++j) {
                acc = __dadd_rn(acc, b[j]);
                b[j] = acc;
            }
        } else {  // the other threads stage the next chunk
            const int64_t c1 = c0 + CH;
            for (int64_t j = tid - 1; j < CH && c1 + j < L; j += CDF_SCAN_THREADS - 1) buf[cur ^ 1][j] = s[c1 + j];
        }
        __syncthreads();
        for (int j = tid; j < n; j += CDF_SCAN_THREADS) c[c0 + j] = buf[cur][j];
        __syncthreads();  // buf[cur] is refilled two chunks on
        cur ^= 1;
    }
}

// cdf_j /= cdf[last of its range]  (IEEE division, sampling.py:109)
__global__ void cdf_div_kernel(double* __restrict__ cdf, const int64_t* __restrict__ lo,
                               const int64_t* __restrict__ len) {
    const int64_t r = blockIdx.y;
    const int64_t base = lo[r], L = len[r];
    const double last = cdf[base + L - 1];
    __syncthreads();  // every thread has read `last` before anyone overwrites it
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < L; j += (int64_t)gridDim.x * blockDim.x) {
        if (j == L - 1) continue;  // divided last, below
        cdf[base + j] = __ddiv_rn(cdf[base + j], last);
    }
}

__global__ void cdf_div_last_kernel(double* __restrict__ cdf, const int64_t* __restrict__ lo,
                                    const int64_t* __restrict__ len, int64_t nranges) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= nranges) return;
    const int64_t i = lo[r] + len[r] - 1;
    cdf[i] = __ddiv_rn(cdf[i], cdf[i]);
}

// ---------------------------------------------------------------------------
// Row sampling.  Thread (run r, worker w) produces draws d0 + r*R ...
// d0 + r*R + R - 1 of worker w: jump the worker's PCG64 stream ahead by the
// draw offset, then R steps; the R binary searches run in lock-step for ILP.
// out index = w * stride_w + (d - d0) * stride_d.
// ---------------------------------------------------------------------------
constexpr int SAMPLE_R = 8;

__global__ void __launch_bounds__(256) sample_rows_kernel(const double* __restrict__ cdf,
                                                          const int64_t* __restrict__ lo,
                                                          const int64_t* __restrict__ len,
                                                          const PcgPod* __restrict__ base_states,
                                                          int64_t q, int64_t d0, int64_t count,
                                                          int32_t* __restrict__ out, int64_t stride_w,
                                                          int64_t stride_d) {
    const int64_t runs = (count + SAMPLE_R - 1) / SAMPLE_R;
    const int64_t total = runs * q;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < total;
         g += (int64_t)gridDim.x * blockDim.x) {
        const int64_t w = g % q, r = g / q;
        Pcg st = pcg_from_pod(base_states[w]);
        const int64_t first = r * SAMPLE_R;
        pcg_advance(st, (uint64_t)(d0 + first));
        const int64_t L = len[w], base = lo[w];
        const double* c = cdf + base;
        double u[SAMPLE_R];
        int64_t a[SAMPLE_R], b[SAMPLE_R];
#pragma unroll
        for (int k = 0; k < SAMPLE_R; ++k) {
            u[k] = pcg_u01(st);
            a[k] = 0;
            b[k] = L;
        }
        // lock-step binary searches (searchsorted side="right")
        bool busy = true;
        while (busy) {
            busy = false;
#pragma unroll
            for (int k = 0; k < SAMPLE_R; ++k) {
                if (a[k] < b[k]) {
                    const int64_t mid = a[k] + ((b[k] - a[k]) >> 1);
                    if (__ldg(c + mid) <= u[k])
                        a[k] = mid + 1;
                    else
                        b[k] = mid;
                    busy |= a[k] < b[k];
                }
            }
        }
#pragma unroll
        for (int k = 0; k < SAMPLE_R; ++k) {
            const int64_t d = first + k;
            if (d < count) {
                const int64_t j = a[k] >= L ? L - 1 : a[k];
                out[w * stride_w + d * stride_d] = (int32_t)(base + j);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Norms for traces / reports: ||A x - b||^2 per row block and ||x - x_ref||^2.
// Deterministic: per-row squares written out, reduced in fixed order by one
// CTA.  (Tolerance-level quantities; not on the iteration path.)
// ---------------------------------------------------------------------------
__global__ void residual_rows_kernel(const double* __restrict__ A, const double* __restrict__ b,
                                     const double* __restrict__ x, int64_t m, int64_t n, int64_t ld,
                                     double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= m) return;
    const double* a = A + row * ld;
    double d = 0.0;
    for (int64_t j = lane; j < n; j += 32) d = fma(a[j], x[j], d);
    d = warp_sum(d);
    if (lane == 0) {
        const double r = d - b[row];
        out[row] = r * r;
    }
}

// Trace residuals of K iterate snapshots (the trace records of one solve) in one pass over A:
// out[j * m + i] = (<a_i, X_j> - b_i)^2, X_j = X + j * ld.  harness trace semantics
// (solvers.py:210-224: every record carries ||Ax - b||) cost one GEMV over A per record; a
// 32-row x 32-snapshot tile per CTA reads A once for up to 32 records (fp64 FMAs on the CUDA
// cores, A and X staged 32 columns at a time through shared memory).  The dot of row i with
// snapshot j runs over the columns in ascending order, so a record's value does not depend on
// which other records share its batch.
__global__ void __launch_bounds__(256) residual_batch_kernel(const double* __restrict__ A,
                                                             const double* __restrict__ b,
                                                             const double* __restrict__ X, int64_t m, int64_t n,
                                                             int64_t ld, int K, double* __restrict__ out) {
    constexpr int TM = 32, KB = 32, TK = 32;
    __shared__ double As[TK][TM + 1];
    __shared__ __align__(16) double Xs[TK][KB];
    const int tid = threadIdx.x, ty = tid >> 4, tx = tid & 15;
    const int64_t row0 = (int64_t)blockIdx.x * TM;
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    for (int64_t c0 = 0; c0 < n; c0 += TK) {
#pragma unroll
        for (int t = 0; t < (TM * TK) / 256; ++t) {
            const int e = tid + 256 * t, r = e / TK, c = e % TK;
            const int64_t gr = row0 + r, gc = c0 + c;
            As[c][r] = (gr < m && gc < n) ? __ldg(A + gr * ld + gc) : 0.0;
            Xs[c][r] = (r < K && gc < n) ? __ldg(X + (int64_t)r * ld + gc) : 0.0;  // r = snapshot here
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            const double a0 = As[kk][2 * ty], a1 = As[kk][2 * ty + 1];
            const double2 xv = *reinterpret_cast<const double2*>(&Xs[kk][2 * tx]);
            acc[0][0] = fma(a0, xv.x, acc[0][0]);
            acc[0][1] = fma(a0, xv.y, acc[0][1]);
            acc[1][0] = fma(a1, xv.x, acc[1][0]);
            acc[1][1] = fma(a1, xv.y, acc[1][1]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 2; ++i) {
        const int64_t gr = row0 + 2 * ty + i;
        if (gr >= m) continue;
        const double bi = b[gr];
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const int sj = 2 * tx + j;
            if (sj < K) {
                const double r = acc[i][j] - bi;
                out[(int64_t)sj * m + gr] = r * r;
            }
        }
    }
}

__global__ void diff_sq_kernel(const double* __restrict__ x, const double* __restrict__ y, int64_t n,
                               double* __restrict__ out) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) {
        const double d = x[j] - y[j];
        out[j] = d * d;
    }
}

// x = S / Q (IEEE division by the worker count, solvers.py:137 / distributed.py:300)
__global__ void scale_copy_kernel(const double* __restrict__ S, double div, int64_t n, double* __restrict__ x) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) x[j] = __ddiv_rn(S[j], div);
}

// (b_i, ||a_i||^2) packed for one 16-byte copy per sampled row
__global__ void pack_bs2_kernel(const double* __restrict__ b, const double* __restrict__ sq, int64_t m,
                                double* __restrict__ out) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < m) {  // 32-byte record (b_i, ||a_i||^2, RN(1 / ||a_i||^2), 0)
        out[4 * i] = b[i];
        out[4 * i + 1] = sq[i];
        out[4 * i + 2] = sq[i] > 0.0 ? __drcp_rn(sq[i]) : 0.0;
        out[4 * i + 3] = 0.0;
    }
}

__global__ void __launch_bounds__(1024) sum_kernel(const double* __restrict__ v, int64_t n, double* __restrict__ out) {
    __shared__ double part[32];
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s += v[j];
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) out[0] = t;
    }
}

// Closing half of one row-sharded iteration on the device (distributed.py:296-301, solvers.py:137):
// x = S / Q, then ||x - x_ref||^2 in exactly diff_sq_kernel + sum_kernel's order (so the native loop
// and the host-driven one agree bitwise), written to *err_out.  In stop mode err < eps raises the halt
// flag (halt = k_next + 1: x_{k_next} met the rule): every later launch of the stream that reads the
// flag is a no-op, so x_{k_next} stands (_drive's check before iteration k, solvers.py:229-243).
__global__ void __launch_bounds__(1024) shard_average_kernel(const double* __restrict__ S, double Q, int64_t n,
                                                             int64_t ld, const double* __restrict__ xref,
                                                             double* __restrict__ x, double eps, int use_stop,
                                                             int64_t k_next, double* __restrict__ err_out,
                                                             int* __restrict__ halt) {
    if (halt != nullptr && *(volatile int*)halt != 0) return;  // stopped earlier: uniform over the block
    __shared__ double part[32];
    double s = 0.0;
#pragma unroll 4
    for (int64_t j = threadIdx.x; j < ld; j += blockDim.x) {
        const double v = __ddiv_rn(S[j], Q);
        x[j] = v;
        if (j < n) {
            const double d = __dsub_rn(v, xref[j]);
            s = __dadd_rn(s, __dmul_rn(d, d));
        }
    }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double t = (threadIdx.x < (blockDim.x >> 5)) ? part[threadIdx.x] : 0.0;
        t = warp_sum(t);
        if (threadIdx.x == 0) {
            *err_out = t;
            if (use_stop && halt != nullptr && t < eps) *halt = (int)(k_next + 1);
        }
    }
}

// Cyclic Kaczmarz rows (solvers.py:286-287): idx[j] = (k0 + j) mod m.
__global__ void cyclic_rows_kernel(int32_t* __restrict__ idx, int64_t k0, int64_t count, int64_t m) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < count; j += (int64_t)gridDim.x * blockDim.x)
        idx[j] = (int32_t)((k0 + j) % m);
}

// Dense rows (pitch n) -> pitched rows (pitch ld, zero padding).
__global__ void repack_rows_kernel(const double* __restrict__ src, int64_t m, int64_t n, int64_t ld,
                                   double* __restrict__ dst) {
    const int64_t total = m * ld;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = e / ld, j = e - i * ld;
        dst[e] = j < n ? src[i * n + j] : 0.0;
    }
}

}  // namespace kz
