// kz_rkw.cu -- one-warp RK / CK kernel for short rows (n <= 64 * EPL columns).
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   kaczmarz_step   solvers.py:107-117   scale = alpha (b_i - <a_i, x>) / ||a_i||^2; x += scale a_i
//   solve_rk        solvers.py:294-310   one stream, one row per iteration
//   solve_ck        solvers.py:271-291   row k mod m (the indices come from cyclic_rows_kernel)
//   _drive          solvers.py:229-243   ||x - x_ref||^2 < eps checked before every iteration
//
// A short row (BASELINE config 0: 2000 x 50) is a few hundred bytes: the chain kernel's TMA
// ring, CTA reductions and block machinery cost more than the row.  Here one warp owns the
// whole iterate (lane l holds the column pairs l, l + 32, ... in registers) and runs the
// sequential chain directly:
//   * rows arrive by plain 16-byte loads issued one group (P rows) ahead into a register ring;
//     the row indices are x-independent (the sampler wrote the whole chunk) and are read two
//     groups ahead, each row's (b, ||a||^2, 1/||a||^2) record one group ahead in lane r;
//   * per row one pair of xor butterflies gives <a_i, x> and ||x - x_ref||^2 in every lane
//     bit-identically (IEEE addition is commutative, so partner lanes add the same operands);
//   * the scale is the IEEE quotient (Markstein correction of the precomputed reciprocal,
//     bit-identical to the division) and x += fl(s a) with the reference's rounding.
// (Gram-corrected blocks of 4 rows, as in the chain kernel, measured slower here: one warp
// issues the block's 15-value reduction and solve itself.)
#include "kz_kernels.cuh"

namespace kz {

template <int EPL, int P>
__global__ void __launch_bounds__(32, 1) rkw_kernel(SolveArgs a) {
    static_assert(P <= 32, "one record per lane");
    // block b = one independent solve (kz_solve_seeds: the seeds of a configuration side by
    // side, each with its own iterate, row draws, status and stop flag); one block otherwise
    const int64_t sb = blockIdx.x;
    if (a.halt != nullptr && a.halt[sb] != 0) return;
    const int lane = threadIdx.x;
    const int64_t ld = a.ld, n = a.n, total = a.count;
    double* const xg = a.x + sb * ld;
    const int32_t* const ix = a.idx + sb * a.idx_stride;
    SolveStatus* const stat = a.status + sb;
    const double alpha = a.alphas[0];
    const bool use_stop = a.use_stop != 0, final_check = a.final_check != 0;
    const bool ckpt_on = a.ckpt_every > 0;

    double2 x[EPL], xr[EPL];
    bool vld[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int64_t col = 2 * (int64_t)(lane + 32 * e);
        vld[e] = col < ld;
        x[e] = vld[e] ? __ldcg(reinterpret_cast<const double2*>(xg + col)) : make_double2(0.0, 0.0);
        xr[e] = vld[e] ? __ldg(reinterpret_cast<const double2*>(a.xref + col)) : make_double2(0.0, 0.0);
    }
    auto row_ptr = [&](int i, int e) {
        return reinterpret_cast<const double2*>(a.A + (int64_t)i * ld + 2 * (lane + 32 * e));
    };
    auto idx_at = [&](int64_t j) -> int { return (lane < P && j < total) ? ix[j] : 0; };
    auto load_rec = [&](int64_t j, int i, double& b, double& sq, double& rc) {
        if (lane < P && j < total) {
            const double2 r01 = __ldg(reinterpret_cast<const double2*>(a.bs2 + 4 * (int64_t)i));
            b = r01.x;
            sq = r01.y;
            rc = __ldg(a.bs2 + 4 * (int64_t)i + 2);
        }
    };

    // group g = rows [g P, (g+1) P): ring rows and records (lane r) of g, indices of g + 1, g + 2
    double2 rw[P][EPL];
    double rb = 0.0, rsq = 1.0, rrc = 1.0;
    int iv1 = idx_at(P + lane), iv2 = 0;
    {
        const int iv0 = idx_at(lane);
        load_rec(lane, iv0, rb, rsq, rrc);
#pragma unroll
        for (int r = 0; r < P; ++r) {
            const int i = __shfl_sync(0xffffffffu, iv0, r);
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                rw[r][e] = (r < total && vld[e]) ? __ldg(row_ptr(i, e)) : make_double2(0.0, 0.0);
        }
    }

    int conv = 0, checks = 0;
    double err_last = 0.0;
    int64_t done = 0;
    bool fin = false;
    for (int64_t base = 0; !fin; base += P) {
        iv2 = idx_at(base + 2 * P + lane);  // consumed one group from now: no stall on it here
        double nb = 0.0, nsq = 1.0, nrc = 1.0;
        load_rec(base + P + lane, iv1, nb, nsq, nrc);
#pragma unroll
        for (int r = 0; r < P; ++r) {
            const int64_t k = base + r;  // x_k is in registers: check, then project row k
            const bool need = use_stop && (k < total || final_check);
            if (k >= total && !need) {
                fin = true;
                break;
            }
            double dot = 0.0, err = 0.0;
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (vld[e]) {
                    dot = fma(rw[r][e].y, x[e].y, fma(rw[r][e].x, x[e].x, dot));
                    const double d0 = x[e].x - xr[e].x, d1 = x[e].y - xr[e].y;
                    err = fma(d1, d1, fma(d0, d0, err));
                }
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) {
                dot += __shfl_xor_sync(0xffffffffu, dot, o);
                err += __shfl_xor_sync(0xffffffffu, err, o);
            }
            if (need) {
                ++checks;
                err_last = err;
                if (err < a.eps) {
                    conv = 1;
                    fin = true;
                    break;
                }
            }
            if (k >= total) {
                fin = true;
                break;
            }
            const double bi = __shfl_sync(0xffffffffu, rb, r);
            const double sqi = __shfl_sync(0xffffffffu, rsq, r);
            const double rci = __shfl_sync(0xffffffffu, rrc, r);
            const double s = div_rn_fast(__dmul_rn(alpha, __dsub_rn(bi, dot)), sqi, rci);
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (vld[e]) {
                    x[e].x = __dadd_rn(x[e].x, __dmul_rn(s, rw[r][e].x));
                    x[e].y = __dadd_rn(x[e].y, __dmul_rn(s, rw[r][e].y));
                }
            done = k + 1;
            if (ckpt_on && ((a.k0 + k + 1) % a.ckpt_every) == 0) {
                const int64_t slot = (a.k0 + k + 1) / a.ckpt_every - 1;
                if (slot < a.ckpt_cap) {
#pragma unroll
                    for (int e = 0; e < EPL; ++e) {
                        const int64_t col = 2 * (int64_t)(lane + 32 * e);
                        if (col < n) a.ckpt[slot * n + col] = x[e].x;
                        if (col + 1 < n) a.ckpt[slot * n + col + 1] = x[e].y;
                    }
                }
            }
            // slot r is free: row k + P goes in
            const int in = __shfl_sync(0xffffffffu, iv1, r);
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (k + P < total && vld[e]) rw[r][e] = __ldg(row_ptr(in, e));
        }
        rb = nb;
        rsq = nsq;
        rrc = nrc;
        iv1 = iv2;
    }
#pragma unroll
    for (int e = 0; e < EPL; ++e)
        if (vld[e]) __stcg(reinterpret_cast<double2*>(xg + 2 * (lane + 32 * e)), x[e]);
    if (lane == 0) {
        stat->iters_done = done;
        stat->converged = conv;
        stat->checks = checks;
        stat->err = err_last;
    }
}

template __global__ void rkw_kernel<1, 8>(SolveArgs);
template __global__ void rkw_kernel<2, 8>(SolveArgs);
template __global__ void rkw_kernel<4, 8>(SolveArgs);

}  // namespace kz
