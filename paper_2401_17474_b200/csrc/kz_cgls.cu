// kz_cgls.cu -- CGLS on the resident system (reference: cgls.py:18-75), device side.
//
// The reference's x_LS for the convergence-horizon experiments (c4) comes from
// CGLS on the normal equations: per iteration one product with A and one with
// A^T, two dot products and three vector updates.  All of it is HBM-bound
// GEMV work on the matrix that is already resident for the solves:
//   gemv_n  : y = A p (warp per row, fixed lane order + shuffle tree)
//   gemv_t  : s = A^T r in two deterministic passes: CTA (column tile, row
//             chunk) partial sums with coalesced row loads, then a fixed-order
//             sum over the chunks
//   dot     : one CTA, fixed tree
// Results are deterministic run to run; they match numpy's CGLS to rounding
// (tolerance parity; the reference's own x_LS is pinned that way).
#include "kz_kernels.cuh"

namespace kz {

// y = A x  (mode 0)   or   y = b - A x  (mode 1)
__global__ void cg_gemv_n_kernel(const double* __restrict__ A, const double* __restrict__ x,
                                 const double* __restrict__ b, int64_t m, int64_t n, int64_t ld, int mode,
                                 double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (row >= m) return;
    const double* a = A + row * ld;
    double acc = 0.0;
    for (int64_t j = lane; j < n; j += 32) acc = fma(a[j], x[j], acc);
    acc = warp_sum(acc);
    if (lane == 0) y[row] = mode ? b[row] - acc : acc;
}

// partial[c][j] = sum_{i in chunk c} A[i][j] r[i]
__global__ void cg_gemv_t_partial_kernel(const double* __restrict__ A, const double* __restrict__ r, int64_t m,
                                         int64_t n, int64_t ld, int64_t rows_per_chunk,
                                         double* __restrict__ partial) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t c = blockIdx.y;
    const int64_t i0 = c * rows_per_chunk;
    const int64_t i1 = i0 + rows_per_chunk < m ? i0 + rows_per_chunk : m;
    if (j >= n) return;
    double acc = 0.0;
    for (int64_t i = i0; i < i1; ++i) acc = fma(A[i * ld + j], __ldg(r + i), acc);
    partial[c * ld + j] = acc;
}

__global__ void cg_gemv_t_reduce_kernel(const double* __restrict__ partial, int64_t nchunks, int64_t n, int64_t ld,
                                        double* __restrict__ s) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    double acc = 0.0;
    for (int64_t c = 0; c < nchunks; ++c) acc += partial[c * ld + j];
    s[j] = acc;
}

// out = <x, y> (one CTA of 1024 threads, fixed order)
__global__ void __launch_bounds__(1024) cg_dot_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                     int64_t n, double* __restrict__ out) {
    __shared__ double part[32];
    double s = 0.0;
    for (int64_t j = threadIdx.x; j < n; j += blockDim.x) s = fma(x[j], y[j], s);
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        double v = threadIdx.x < (blockDim.x >> 5) ? part[threadIdx.x] : 0.0;
        v = warp_sum(v);
        if (threadIdx.x == 0) *out = v;
    }
}

// x += alpha p ; r -= alpha t   (alpha = gamma / delta read on the device)
__global__ void cg_update_xr_kernel(double* __restrict__ x, const double* __restrict__ p, double* __restrict__ r,
                                    const double* __restrict__ t, const double* __restrict__ scal, int64_t n,
                                    int64_t m) {
    const double alpha = scal[0] / scal[1];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < (n > m ? n : m);
         j += (int64_t)gridDim.x * blockDim.x) {
        if (j < n) x[j] = __dadd_rn(x[j], __dmul_rn(alpha, p[j]));
        if (j < m) r[j] = __dsub_rn(r[j], __dmul_rn(alpha, t[j]));
    }
}

// v = w / nw  (numpy `w / nw`: correctly rounded division per element)
__global__ void cg_scale_div_kernel(const double* __restrict__ w, const double* __restrict__ nw, int64_t n,
                                    double* __restrict__ v) {
    const double d = *nw;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        v[j] = __ddiv_rn(w[j], d);
}

// p = s + (gamma_new / gamma) p
__global__ void cg_update_p_kernel(double* __restrict__ p, const double* __restrict__ s,
                                   const double* __restrict__ scal, int64_t n) {
    const double beta = scal[2] / scal[0];
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        p[j] = __dadd_rn(__dmul_rn(p[j], beta), s[j]);
}

}  // namespace kz
