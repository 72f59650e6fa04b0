// kz_chain.cu -- worker-per-CTA persistent kernel for RK and RKAB.
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   kaczmarz_step      solvers.py:107-117   scale = alpha*(b_i - <a_i,v>)/sq_i ; v += scale*a_i
//   rkab_worker_block  solvers.py:140-145   bs chained projections on the private v
//   RKAB advance       solvers.py:361-367   v_t = x ; chain ; x = (sum_t v_t) / q, t ascending
//   solve_rk           solvers.py:294-310   (= q 1, bs 1)
//   _drive stop rule   solvers.py:229-243   ||x - x_ref||^2 < eps checked before every iteration
//
// Layout: CTA w runs worker w.  Its estimate v lives in registers: thread
// `tid` owns the 16-byte column pairs col = 2*(p*T + tid), p < EP.  Rows are
// streamed HBM -> shared memory by per-thread cp.async (16 B, each thread
// copies exactly the pairs it later reads, so no CTA barrier guards the
// data) through a `stages`-deep ring; row indices are x-independent and are
// read from a shared-memory window, so the ring runs stages-1 rows ahead.
// One CTA reduction (warp shuffles + one bar.sync on a parity-double-
// buffered scratch) per projection; the stop-rule error is fused into the
// first projection of each iteration when q == 1.
//
// Arithmetic: the axpy is __dmul_rn then __dadd_rn (two roundings, as numpy's
// `x += scale * row`); the scale is computed in the reference's order; the
// average is a strictly ordered sum over workers then an IEEE division.  Only
// the dot product's summation order differs from OpenBLAS (tolerance parity).
#include "kz_kernels.cuh"

namespace kz {

namespace {

struct ChainSmem {
    double* ring;   // stages x ld
    double* bsq;    // (stages + 1) x 2 : b_i, sq_i per in-flight row
    int32_t* win;   // IDX_WINDOW row indices
    double* red;    // 2 parities x 2 values x 32 warps
};

__device__ __forceinline__ ChainSmem carve(unsigned char* raw, int stages, int64_t ld) {
    ChainSmem s;
    s.ring = reinterpret_cast<double*>(raw);
    s.bsq = s.ring + (size_t)stages * ld;
    s.win = reinterpret_cast<int32_t*>(s.bsq + 2 * (stages + 1));
    s.red = reinterpret_cast<double*>(s.win + IDX_WINDOW);
    return s;
}

// Sum of one (or two) per-thread values over the CTA; every thread returns
// the same bits (fixed shuffle tree, fixed warp order).
template <bool TWO>
__device__ __forceinline__ void cta_reduce(double& v0, double& v1, double* red, int& par, int lane, int warp, int nw) {
    v0 = warp_sum(v0);
    if (TWO) v1 = warp_sum(v1);
    double* r = red + par * 64;
    if (lane == 0) {
        r[warp] = v0;
        if (TWO) r[32 + warp] = v1;
    }
    __syncthreads();
    v0 = warp_sum(lane < nw ? r[lane] : 0.0);
    if (TWO) v1 = warp_sum(lane < nw ? r[32 + lane] : 0.0);
    par ^= 1;
}

}  // namespace

// Largest CTA each pair count is launched with (keeps v register-resident).
template <int EP>
struct ChainMaxThreads {
    static constexpr int value = EP <= 4 ? 256 : (EP <= 8 ? 512 : 640);
};

template <int EP>
__global__ void __launch_bounds__(ChainMaxThreads<EP>::value, 1) chain_kernel(SolveArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
    const int D = a.stages;
    const int64_t ld = a.ld, q = a.q, bs = a.bs;
    ChainSmem sm = carve(smem_raw, D, ld);

    const int64_t w = blockIdx.x;  // worker id
    const int32_t* idx = a.idx + w * a.idx_stride;
    const double alpha = a.alphas[w];
    const int64_t total = a.count * bs;  // draws of this worker in the launch

    // v = x (x0 = 0 on the first launch, the carried iterate afterwards)
    double v[2 * EP];
#pragma unroll
    for (int p = 0; p < EP; ++p) {
        const int64_t col = 2 * ((int64_t)p * T + tid);
        double2 xv = make_double2(0.0, 0.0);
        if (col < ld) xv = __ldcg(reinterpret_cast<const double2*>(a.x + col));
        v[2 * p] = xv.x;
        v[2 * p + 1] = xv.y;
    }
    for (int64_t e = tid; e < IDX_WINDOW && e < total; e += T) sm.win[e] = idx[e];
    __syncthreads();

    // ring bookkeeping in 32-bit: row d lives in stage d % D, its (b_i, sq_i)
    // in slot d % (D + 1); both advance incrementally (no 64-bit modulo).
    auto issue = [&](int64_t d, int stage, int slot) {
        if (d < total) {
            const int64_t i = sm.win[d & (IDX_WINDOW - 1)];
            const double* src = a.A + i * ld;
            double* dst = sm.ring + (size_t)stage * ld;
#pragma unroll
            for (int p = 0; p < EP; ++p) {
                const int64_t col = 2 * ((int64_t)p * T + tid);
                if (col < ld) cp_async16(dst + col, src + col);
            }
            if (tid == 0) {
                double* bs_slot = sm.bsq + 2 * slot;
                cp_async8(bs_slot, a.b + i);
                cp_async8(bs_slot + 1, a.sq + i);
            }
        }
        cp_async_commit();
    };

    // stop-rule error of the current v (= x), every CTA computes the same bits
    auto err_partial = [&]() {
        double e = 0.0;
#pragma unroll
        for (int p = 0; p < EP; ++p) {
            const int64_t col = 2 * ((int64_t)p * T + tid);
            if (col < ld) {
                const double2 r = __ldg(reinterpret_cast<const double2*>(a.xref + col));
                const double d0 = v[2 * p] - r.x, d1 = v[2 * p + 1] - r.y;
                e = fma(d0, d0, e);
                e = fma(d1, d1, e);
            }
        }
        return e;
    };

    for (int j = 0; j < D - 1; ++j) issue(j, j, j);
    int stage = 0, slot = 0;  // consumption position of draw d

    int par = 0;
    unsigned epoch = 0;
    int64_t d = 0;
    long long done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;
    const double inv_q_d = (double)q;

    for (int64_t kk = 0;; ++kk) {
        const bool last = (kk == a.count);
        const bool want_check = a.use_stop && (!last || a.final_check);
        if (last || q > 1) {
            if (want_check) {
                double e = err_partial(), dummy = 0.0;
                cta_reduce<false>(e, dummy, sm.red, par, lane, warp, nw);
                ++checks;
                err_last = e;
                if (e < a.eps) {
                    conv = 1;
                    break;
                }
            }
            if (last) break;
        }
        for (int64_t s = 0; s < bs; ++s, ++d) {
            const bool chk = want_check && q == 1 && s == 0;
            if ((d & 511) == 0 && d > 0) {  // refill the index window half we are leaving
                for (int64_t e = d + 512 + tid; e < d + IDX_WINDOW && e < total; e += T)
                    sm.win[e & (IDX_WINDOW - 1)] = idx[e];
            }
            issue(d + D - 1, stage == 0 ? D - 1 : stage - 1, slot >= 2 ? slot - 2 : slot + D - 1);
            cp_async_wait_dyn(D - 1);
            const double* row = sm.ring + (size_t)stage * ld;
            double dot = 0.0, e2 = 0.0;
#pragma unroll
            for (int p = 0; p < EP; ++p) {
                const int64_t col = 2 * ((int64_t)p * T + tid);
                if (col < ld) {
                    const double2 r = *reinterpret_cast<const double2*>(row + col);
                    dot = fma(r.x, v[2 * p], dot);
                    dot = fma(r.y, v[2 * p + 1], dot);
                }
            }
            if (chk) {
                e2 = err_partial();
                cta_reduce<true>(dot, e2, sm.red, par, lane, warp, nw);
                ++checks;
                err_last = e2;
                if (e2 < a.eps) {
                    conv = 1;
                    goto finish;
                }
            } else {
                cta_reduce<false>(dot, e2, sm.red, par, lane, warp, nw);
            }
            {
                const double* bq = sm.bsq + 2 * slot;
                const double scale = __ddiv_rn(__dmul_rn(alpha, __dsub_rn(bq[0], dot)), bq[1]);
#pragma unroll
                for (int p = 0; p < EP; ++p) {
                    const int64_t col = 2 * ((int64_t)p * T + tid);
                    if (col < ld) {
                        const double2 r = *reinterpret_cast<const double2*>(row + col);
                        v[2 * p] = __dadd_rn(v[2 * p], __dmul_rn(scale, r.x));
                        v[2 * p + 1] = __dadd_rn(v[2 * p + 1], __dmul_rn(scale, r.y));
                    }
                }
            }
            stage = (stage + 1 == D) ? 0 : stage + 1;
            slot = (slot == D) ? 0 : slot + 1;
        }
        const int64_t k = a.k0 + kk;
        const bool ck = a.ckpt_every > 0 && ((k + 1) % a.ckpt_every) == 0 && ((k + 1) / a.ckpt_every) <= a.ckpt_cap;
        const int64_t slot = ck ? (k + 1) / a.ckpt_every - 1 : 0;
        if (q == 1) {
            if (ck) {
#pragma unroll
                for (int p = 0; p < EP; ++p) {
                    const int64_t col = 2 * ((int64_t)p * T + tid);
                    if (col < a.n) a.ckpt[slot * a.n + col] = v[2 * p];
                    if (col + 1 < a.n) a.ckpt[slot * a.n + col + 1] = v[2 * p + 1];
                }
            }
        } else {
            // publish v_w, average column slices in worker order, redistribute x
            double* vw = a.V + w * ld;
#pragma unroll
            for (int p = 0; p < EP; ++p) {
                const int64_t col = 2 * ((int64_t)p * T + tid);
                if (col < ld) __stcg(reinterpret_cast<double2*>(vw + col), make_double2(v[2 * p], v[2 * p + 1]));
            }
            grid_barrier(a.barrier, (++epoch) * gridDim.x);
            const int64_t G = gridDim.x;
            const int64_t cw = ((ld + G - 1) / G + 1) & ~(int64_t)1;
            const int64_t c0 = blockIdx.x * cw, c1 = (c0 + cw < ld) ? c0 + cw : ld;
            for (int64_t col = c0 + tid; col < c1; col += T) {
                double acc = __ldcg(a.V + col);
                for (int64_t t = 1; t < q; ++t) acc = __dadd_rn(acc, __ldcg(a.V + t * ld + col));
                if (a.partial) {  // row-sharded step: the un-normalised local sum, x untouched
                    __stcg(a.partial + col, acc);
                    continue;
                }
                const double xn = __ddiv_rn(acc, inv_q_d);
                __stcg(a.x + col, xn);
                if (ck && col < a.n) a.ckpt[slot * a.n + col] = xn;
            }
            grid_barrier(a.barrier, (++epoch) * gridDim.x);
#pragma unroll
            for (int p = 0; p < EP; ++p) {
                const int64_t col = 2 * ((int64_t)p * T + tid);
                if (col < ld) {
                    const double2 xv = __ldcg(reinterpret_cast<const double2*>(a.x + col));
                    v[2 * p] = xv.x;
                    v[2 * p + 1] = xv.y;
                }
            }
        }
        done = kk + 1;
    }
finish:
    cp_async_wait<0>();
    if (q == 1) {
        double* dst = a.partial ? a.partial : a.x;
#pragma unroll
        for (int p = 0; p < EP; ++p) {
            const int64_t col = 2 * ((int64_t)p * T + tid);
            if (col < ld) __stcg(reinterpret_cast<double2*>(dst + col), make_double2(v[2 * p], v[2 * p + 1]));
        }
    }
    if (blockIdx.x == 0 && tid == 0) {
        a.status->iters_done = done;
        a.status->converged = conv;
        a.status->checks = checks;
        a.status->err = err_last;
    }
}

template __global__ void chain_kernel<1>(SolveArgs);
template __global__ void chain_kernel<2>(SolveArgs);
template __global__ void chain_kernel<4>(SolveArgs);
template __global__ void chain_kernel<8>(SolveArgs);
template __global__ void chain_kernel<16>(SolveArgs);

}  // namespace kz
