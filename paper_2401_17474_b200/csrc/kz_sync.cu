// kz_sync.cu -- column-sliced persistent kernel for RKA (and RKAB with bs = 1).
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   rka_combined_step  solvers.py:120-137   q projections from one snapshot of x;
//                                            x = (sum_t fl(x + fl(s_t a_t))) / q, t ascending
//   solve_rka_seq      solvers.py:313-334   rows of iteration k: one draw per worker stream
//   _drive stop rule   solvers.py:229-243
//
// Layout: P CTAs each own a contiguous column slice [c0, c1) of x (kept in
// shared memory) and of every sampled row.  Per iteration:
//   1. the q row slices (indices known ahead) stream HBM -> smem through a
//      cp.async ring `stages` iterations deep, with b_i and sq_i;
//   2. LPR lanes per row form partial dots <a_t[c0:c1], x[c0:c1]>; warp 0
//      adds the partial of ||x - x_ref||^2;
//   3. the P x (q+1) partials are exchanged -- through distributed shared
//      memory inside one thread-block cluster (CLUSTER) or through global
//      memory behind a grid barrier -- and every CTA sums them in the same
//      CTA order, so all CTAs hold bit-identical scales and stop decisions;
//   4. each column of the slice applies the reference's ordered average.
// Partials are double-buffered by iteration parity: one barrier/iteration.
#include <cooperative_groups.h>

#include "kz_kernels.cuh"

namespace cg = cooperative_groups;

namespace kz {

template <bool CLUSTER, int LPR>
__global__ void __launch_bounds__(256) sync_kernel(SolveArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int T = blockDim.x, tid = threadIdx.x, lane = tid & 31;
    const int D = a.stages;
    const int64_t ld = a.ld, q = a.q;
    const int P = CLUSTER ? (int)cg::this_cluster().num_blocks() : (int)gridDim.x;
    const int c = CLUSTER ? (int)cg::this_cluster().block_rank() : (int)blockIdx.x;
    const int64_t cw = (((ld + P - 1) / P) + 1) & ~(int64_t)1;  // even => 16-byte pairs
    const int64_t c0 = (int64_t)c * cw < ld ? (int64_t)c * cw : ld;
    const int64_t c1 = (c0 + cw < ld) ? c0 + cw : ld;
    const int64_t wdt = c1 - c0;  // this CTA's columns (may be 0)
    const int64_t npairs = cw / 2;

    // shared memory carve
    double* ring = reinterpret_cast<double*>(smem_raw);      // D x q x cw
    double* bsq = ring + (size_t)D * q * cw;                 // D x q x 2
    double* xs = bsq + (size_t)D * q * 2;                    // cw
    double* xrs = xs + cw;                                   // cw
    double* part = xrs + cw;                                 // 2 x (q + 1)
    double* tot = part + 2 * (q + 1);                        // q + 1
    double* alp = tot + (q + 1);                             // q
    int32_t* iring = reinterpret_cast<int32_t*>(alp + q);    // 4 x q

    for (int64_t j = tid; j < cw; j += T) {
        xs[j] = (j < wdt) ? __ldcg(a.x + c0 + j) : 0.0;
        xrs[j] = (j < wdt) ? a.xref[c0 + j] : 0.0;
    }
    for (int64_t t = tid; t < q; t += T) alp[t] = a.alphas[t];
    // indices of the first D iterations (4-slot ring, written D iterations ahead)
    for (int64_t u = tid; u < (int64_t)D * q; u += T) {
        const int64_t it = u / q, t = u % q;
        if (it < a.count) iring[(it & 3) * q + t] = a.idx[it * q + t];
    }
    __syncthreads();

    const unsigned np32 = (unsigned)npairs, work = (unsigned)(q * npairs);
    auto issue = [&](int64_t it, int st) {
        if (it < a.count) {
            const int32_t* ir = iring + (it & 3) * q;
            double* dst = ring + (size_t)st * q * cw;
            for (unsigned u = tid; u < work; u += T) {
                const unsigned t = u / np32, pp = u - t * np32;
                const int64_t col = c0 + 2 * pp;
                if (col < c1) cp_async16(dst + (size_t)t * cw + 2 * pp, a.A + (int64_t)ir[t] * ld + col);
            }
            for (int64_t t = tid; t < q; t += T) {
                cp_async8(bsq + ((size_t)st * q + t) * 2, a.b + ir[t]);
                cp_async8(bsq + ((size_t)st * q + t) * 2 + 1, a.sq + ir[t]);
            }
        }
        cp_async_commit();
    };

    for (int j = 0; j < D - 1; ++j) issue(j, j);
    int st = 0;  // ring stage of iteration kk

    unsigned epoch = 0;
    long long done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;
    const double qd = (double)q;
    const int groups = T / LPR;
    const int g = tid / LPR, gl = tid % LPR;

    for (int64_t kk = 0;; ++kk) {
        const bool last = (kk == a.count);
        const bool want_check = a.use_stop && (!last || a.final_check);
        if (last && !want_check) break;
        const double* rows = ring + (size_t)st * q * cw;
        if (!last) {
            cp_async_wait_dyn(D - 2);
        }
        __syncthreads();  // stage kk visible to all; iteration kk-1 fully retired
        if (!last) {
            issue(kk + D - 1, st == 0 ? D - 1 : st - 1);
            // index ring: iteration kk + D, consumed by issue() one iteration from now
            const int64_t itn = kk + D;
            if (itn < a.count)
                for (int64_t t = tid; t < q; t += T) iring[(itn & 3) * q + t] = a.idx[itn * q + t];
        }
        // ---- partial dots over the slice + partial error ---------------------------
        double* mypart = part + (kk & 1) * (q + 1);
        double* gpart = a.part + ((size_t)(kk & 1) * P + c) * (q + 1);
        if (!last) {
            // rounds of `groups` rows; every lane joins each round's shuffles
            for (int64_t t0 = 0; t0 < q; t0 += groups) {
                const int64_t t = t0 + g;
                double s = 0.0;
                if (t < q) {
                    const double* r = rows + t * cw;
                    for (int64_t j = gl; j < wdt; j += LPR) s = fma(r[j], xs[j], s);
                }
#pragma unroll
                for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LPR);
                if (gl == 0 && t < q) {
                    if (CLUSTER)
                        mypart[t] = s;
                    else
                        __stcg(gpart + t, s);
                }
            }
        }
        if (tid < 32) {
            double e = 0.0;
            if (want_check)
                for (int64_t j = lane; j < wdt; j += 32) {
                    const double dd = xs[j] - xrs[j];
                    e = fma(dd, dd, e);
                }
            e = warp_sum(e);
            if (lane == 0) {
                if (CLUSTER)
                    mypart[q] = e;
                else
                    __stcg(gpart + q, e);
            }
        }
        // ---- exchange -----------------------------------------------------------------
        if (CLUSTER) {
            cg::this_cluster().sync();
        } else {
            grid_barrier(a.barrier, (++epoch) * gridDim.x);
        }
        const int64_t nt = last ? 0 : q;
        for (int64_t t = tid; t <= q; t += T) {
            if (t < nt || t == q) {
                double s = 0.0;
                if (CLUSTER) {
                    // issue all remote (DSMEM) loads first, then add in CTA order
                    double pv[16];
#pragma unroll
                    for (int cc = 0; cc < 16; ++cc)
                        if (cc < P) pv[cc] = cg::this_cluster().map_shared_rank(part, cc)[(kk & 1) * (q + 1) + t];
                    s = pv[0];
#pragma unroll
                    for (int cc = 1; cc < 16; ++cc)
                        if (cc < P) s = __dadd_rn(s, pv[cc]);
                } else {
                    const double* gp = a.part + (size_t)(kk & 1) * P * (q + 1) + t;
                    s = __ldcg(gp);
                    for (int cc = 1; cc < P; ++cc) s = __dadd_rn(s, __ldcg(gp + (size_t)cc * (q + 1)));
                }
                if (t < q) {
                    const double* bs2 = bsq + ((size_t)st * q + t) * 2;
                    tot[t] = __ddiv_rn(__dmul_rn(alp[t], __dsub_rn(bs2[0], s)), bs2[1]);
                } else {
                    tot[q] = s;
                }
            }
        }
        __syncthreads();
        if (want_check) {
            ++checks;
            err_last = tot[q];
            if (err_last < a.eps) {
                conv = 1;
                break;
            }
        }
        if (last) break;
        st = (st + 1 == D) ? 0 : st + 1;
        // ---- ordered average over the q projections (solvers.py:131-137) -------------
        const int64_t k = a.k0 + kk;
        const bool ck = a.ckpt_every > 0 && ((k + 1) % a.ckpt_every) == 0 && ((k + 1) / a.ckpt_every) <= a.ckpt_cap;
        const int64_t slot = ck ? (k + 1) / a.ckpt_every - 1 : 0;
        for (int64_t j = tid; j < wdt; j += T) {
            const double xj = xs[j];
            double acc = __dadd_rn(xj, __dmul_rn(tot[0], rows[j]));
            for (int64_t t = 1; t < q; ++t) acc = __dadd_rn(acc, __dadd_rn(xj, __dmul_rn(tot[t], rows[t * cw + j])));
            const double xn = __ddiv_rn(acc, qd);
            xs[j] = xn;
            if (ck && c0 + j < a.n) a.ckpt[slot * a.n + c0 + j] = xn;
        }
        done = kk + 1;
    }
    cp_async_wait<0>();
    __syncthreads();
    for (int64_t j = tid; j < wdt; j += T) __stcg(a.x + c0 + j, xs[j]);
    if (CLUSTER) cg::this_cluster().sync();  // peers may still read our partials
    if (c == 0 && tid == 0) {
        a.status->iters_done = done;
        a.status->converged = conv;
        a.status->checks = checks;
        a.status->err = err_last;
    }
}

template __global__ void sync_kernel<true, 8>(SolveArgs);
template __global__ void sync_kernel<true, 32>(SolveArgs);
template __global__ void sync_kernel<false, 8>(SolveArgs);
template __global__ void sync_kernel<false, 32>(SolveArgs);

}  // namespace kz
