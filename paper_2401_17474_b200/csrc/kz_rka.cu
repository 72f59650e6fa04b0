// kz_rka.cu -- column-sliced RKA kernel (RKA, RKAB with bs = 1) with TMA row staging.
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   rka_combined_step  solvers.py:120-137   q projections from one snapshot of x;
//                                            x = (sum_t fl(x + fl(s_t a_t))) / q
//   solve_rka_seq      solvers.py:313-334   rows of iteration k: one draw per worker stream
//   _drive stop rule   solvers.py:229-243
//
// P = G x Pc CTAs (G thread-block clusters of Pc CTAs); CTA c owns the column
// slice [c0, c0 + cw) of x and of every sampled row.  Roles:
//   * producer warp (warp 8): for iteration k it gathers the q row slices with
//     TMA `tile::gather4` (four rows per instruction, box = slice width) and the
//     q packed (b_i, ||a_i||^2) pairs into ring stage k mod D, completing the
//     stage's `full` mbarrier; it refills a stage once the 8 compute warps have
//     arrived on its `empty` mbarrier.  Row indices are x-independent, so it
//     runs D iterations ahead of the arithmetic.
//   * compute warps (0..7): warp w owns the worker block [w QB, (w+1) QB).
//     x and x_ref live in registers (EPL column pairs per lane).  Per iteration:
//       1. dots: 8 rows per warp per round, LG lanes per row (NR = LG/4 rows
//          per lane group, independent FMA chains), a transposed shuffle
//          reduction (NR-1 + 2 shuffles per round);
//       2. push: every row partial goes to all Pc CTAs of the cluster with
//          st.async (completing the receiver's exchange mbarrier); warp 0 adds
//          the slice's ||x - x_ref||^2 piece as entry q;
//       3. wait on the local exchange mbarrier; 4 lanes per worker add the Pc
//          partials with one fixed tree (bit-identical in every CTA).  With
//          G > 1 the rank-0 CTA of each cluster publishes its cluster totals
//          as tagged 64-bit words and every CTA adds the G cluster totals in
//          cluster order;
//       4. scale s_t = alpha_t (b_t - d_t) / ||a_t||^2; stop rule on entry q;
//       5. average: each warp sums fl(x + fl(s_t a_t)) over its block; the 8
//          per-warp sums meet in shared memory behind one named barrier and
//          every warp forms x_{k+1} (fixed tree, / q) for its own lanes, so x
//          never leaves registers.
//   One named barrier per iteration; the exchange mbarrier orders everything
//   else (a CTA's exchange completes only after every warp of every peer has
//   pushed, i.e. finished the previous iteration).
#include "kz_kernels.cuh"

namespace kz {

namespace {
constexpr int NW = RKA_NW;
constexpr unsigned CBAR = 1;  // named barrier id of the compute warps
}  // namespace

template <int LG, int EPL, bool TIMING>
__global__ void __launch_bounds__(RKA_NT, 1) rka_kernel(const __grid_constant__ SolveArgs a,
                                                        const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB) {
    constexpr int NR = LG / 4;  // rows per lane group per round (8 rows per warp per round)
    static_assert(LG == 8 || LG == 16 || LG == 32, "lane group");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = a.stages;
    const int ld = (int)a.ld, q = (int)a.q;
    const int P = (int)gridDim.x, c = (int)blockIdx.x;
    const int Pc = (int)cluster_size(), cr = (int)cluster_rank();
    const int G = P / Pc, gid = c / Pc;
    const int cw = (((ld + P - 1) / P) + 1) & ~1;
    const int c0 = c * cw < ld ? c * cw : ld;
    const int wdt = (c0 + cw < ld ? c0 + cw : ld) - c0;  // even
    const int cwb = a.box;                               // >= cw, multiple of 4
    const int q4 = (q + 3) & ~3;
    const int q1 = q + 1, q1p = (q1 + 1) & ~1;
    const int QB = (q + NW - 1) / NW;
    const int nwv = (q + QB - 1) / QB;  // warps owning at least one worker
    const unsigned rows_bytes = (unsigned)(q4 * cwb * 8);
    const int stage_bytes = (int)rows_bytes + q4 * 32;  // rows, then (b, sq) pairs in 128-B groups of 4

    // shared memory carve (rka_smem() in kz_api.cu must match)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw);  // D <= 8
    unsigned long long* empty = full + 8;                                       // D
    unsigned long long* xbar = full + 16;                                       // 2
    volatile int* halt = reinterpret_cast<volatile int*>(smem_raw + 160);
    unsigned char* ring = smem_raw + 256;                                        // D x stage_bytes
    double* inbuf = reinterpret_cast<double*>(ring + D * stage_bytes);  // 2 x Pc x q1p
    double* upd = inbuf + 2 * Pc * q1p;                                          // NW x cwb
    double* scal = upd + NW * cwb;                                               // q4
    double* alp = scal + q4;                                                     // q

    if (tid == 0) {
        for (int i = 0; i < D; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
        }
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        *halt = 0;
        fence_mbarrier_init_cluster();
    }
    for (int t = tid; t < q; t += RKA_NT) alp[t] = a.alphas[t];
    __syncthreads();
    cluster_sync_all();  // peers' mbarriers exist before anyone pushes

    if (warp == NW) {
        // ================= producer warp =================
        const int ng = q4 / 4;
        const unsigned bytes = rows_bytes + (unsigned)q4 * 16u;  // gather4 of pairs lands 64 B per group
        const unsigned ring_u = smem_u32(ring);
        int64_t it = 0;
        int s = 0;
        for (; it < a.count; ++it) {
            if (it >= D) {  // stage s was last filled for iteration it - D: await that release
                const unsigned eph = (unsigned)((it / D - 1) & 1);
                bool ok = false;
                while (!(ok = mbar_try_wait(&empty[s], eph)))
                    if (*halt) break;
                if (!ok) break;
            }
            if (*halt) break;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
            __syncwarp();
            const unsigned dst = ring_u + (unsigned)(s * stage_bytes);
            const unsigned fb = smem_u32(&full[s]);
            const int32_t* ix = a.idx + it * q;
            for (int op = lane; op < 2 * ng; op += 32) {
                const int i = op < ng ? op : op - ng;
                int r[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) r[u] = __ldg(ix + (4 * i + u < q ? 4 * i + u : q - 1));
                if (op < ng)
                    tma_gather4(dst + (unsigned)(i * 4 * cwb * 8), &tmA, c0, r[0], r[1], r[2], r[3], fb);
                else
                    tma_gather4(dst + rows_bytes + (unsigned)(i * 128), &tmB, 0, r[0], r[1], r[2], r[3], fb);
            }
            if (++s == D) s = 0;
        }
        // drain: the last issued phase of every stage must land before exit
        if (lane == 0) {
            for (int st = 0; st < D && st < it; ++st) {
                const int64_t last_it = st + ((it - 1 - st) / D) * D;
                mbar_wait(&full[st], (unsigned)((last_it / D) & 1));
            }
        }
        __syncwarp();
        __syncthreads();
        cluster_sync_all();
        return;
    }

    // ================= compute warps =================
    const int gl = lane % LG, grp = lane / LG;
    double2 xv[EPL], xr[EPL];
    bool vld[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int j = 2 * (gl + LG * e);
        vld[e] = j < wdt;
        xv[e] = vld[e] ? make_double2(__ldcg(a.x + c0 + j), __ldcg(a.x + c0 + j + 1)) : make_double2(0.0, 0.0);
        xr[e] = vld[e] ? make_double2(a.xref[c0 + j], a.xref[c0 + j + 1]) : make_double2(0.0, 0.0);
    }
    // ||x - x_ref||^2 over the slice (warp 0, lane group 0), pushed as entry q
    auto slice_err = [&]() -> double {
        double e2 = 0.0;
        if (grp == 0) {
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (vld[e]) {
                    const double d0 = xv[e].x - xr[e].x, d1 = xv[e].y - xr[e].y;
                    e2 = fma(d0, d0, e2);
                    e2 = fma(d1, d1, e2);
                }
        }
        return warp_sum(e2);
    };
    double errp = (warp == 0) ? slice_err() : 0.0;

    // reduced-row bookkeeping: after the transposed reduction lane gl holds row ri
    // of its group; lanes differing in the low two bits hold the same value
    int ri = 0;
#pragma unroll
    for (int h = NR / 2, o = LG / 2; h >= 1; h >>= 1, o >>= 1)
        if (gl & o) ri += h;
    const int rho = gl & 3;
    unsigned rin[4], rbar[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int pk = rho + 4 * i;
        rin[i] = mapa_u32(smem_u32(inbuf), (unsigned)(pk < Pc ? pk : 0));
        rbar[i] = mapa_u32(smem_u32(xbar), (unsigned)(pk < Pc ? pk : 0));
    }
    const unsigned rin_e = mapa_u32(smem_u32(inbuf), (unsigned)(lane < Pc ? lane : 0));
    const unsigned rbar_e = mapa_u32(smem_u32(xbar), (unsigned)(lane < Pc ? lane : 0));

    const int wb = warp * QB < q ? warp * QB : q;
    const int we = wb + QB < q ? wb + QB : q;
    const int nb = we - wb;
    const bool gh = nb > grp * NR;  // this lane group owns at least one worker
    const bool qpow2 = (q & (q - 1)) == 0;
    const double invq = 1.0 / (double)q;
    const double qd = (double)q;
    const bool ckpt_on = a.ckpt_every > 0;
    const unsigned xfer_bytes = (unsigned)(Pc * q1 * (int)sizeof(double));
    const int count = (int)a.count;
    const int cnt2 = Pc >= 2 ? Pc / 2 : 1;  // partials per lane in the totals (2 lanes per worker)

    int st = 0;
    unsigned fph = 0;  // parity of stage st's current full phase
    int done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;

    for (int kk = 0;; ++kk) {
        const bool last = (kk == count);
        const bool want_check = a.use_stop && (!last || a.final_check);
        if (last && !want_check) break;
        const int par = kk & 1;
        const bool rec = TIMING && a.dbg != nullptr && c == 0 && lane == 0 && kk < 32;
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 0] = clock64();
        if (tid == 0) mbar_arrive_expect_tx(&xbar[par], last ? (unsigned)(Pc * (int)sizeof(double)) : xfer_bytes);
        const double* rows = reinterpret_cast<const double*>(ring + st * stage_bytes);
        const double2* bsq = reinterpret_cast<const double2*>(ring + st * stage_bytes + rows_bytes);
        if (!last) mbar_wait(&full[st], fph);
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 1] = clock64();
        const unsigned my_off = (unsigned)(((par * Pc + cr) * q1p) * (int)sizeof(double));
        // ---- 1-2. partial dots of this warp's rows, pushed to every CTA of the cluster --
        if (!last) {
            for (int rb = wb; rb < we; rb += 8) {
                double acc[NR];
#pragma unroll
                for (int r = 0; r < NR; ++r) {
                    acc[r] = 0.0;
                    const int t = rb + grp * NR + r;
                    if (t < we) {
                        const double* row = rows + t * cwb;
#pragma unroll
                        for (int e = 0; e < EPL; ++e)
                            if (vld[e]) {
                                const double2 rv = *reinterpret_cast<const double2*>(row + 2 * (gl + LG * e));
                                acc[r] = fma(rv.x, xv[e].x, acc[r]);
                                acc[r] = fma(rv.y, xv[e].y, acc[r]);
                            }
                    }
                }
#pragma unroll
                for (int h = NR / 2, o = LG / 2; h >= 1; h >>= 1, o >>= 1) {
                    const bool up = (gl & o) != 0;
#pragma unroll
                    for (int i = 0; i < h; ++i) {
                        const double send = up ? acc[i] : acc[i + h];
                        const double keep = up ? acc[i + h] : acc[i];
                        acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
                acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
                const int t = rb + grp * NR + ri;
                if (t < we) {
                    const unsigned off = my_off + (unsigned)(t * (int)sizeof(double));
#pragma unroll
                    for (int i = 0; i < 4; ++i)
                        if (rho + 4 * i < Pc) st_async_f64(rin[i] + off, acc[0], rbar[i] + 8u * par);
                }
            }
        }
        if (warp == 0 && lane < Pc)
            st_async_f64(rin_e + my_off + (unsigned)(q * (int)sizeof(double)), errp, rbar_e + 8u * par);
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 2] = clock64();
        // ---- 3. exchange (the st.async data lands with the mbarrier's tx count) -----------
        mbar_wait(&xbar[par], (unsigned)((kk >> 1) & 1));
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 3] = clock64();
        // ---- 3-4. totals (2 lanes per worker), scales, stop rule -------------------------
        double err = 0.0;
        {
            const double* ib = inbuf + par * Pc * q1p;
            const int nbr = last ? 0 : nb;  // the final check exchanges only entry q
            const int nitems = nbr + (want_check ? 1 : 0);
            const int u = lane & 1;
            double errv = 0.0;
            for (int i0 = 0; i0 < nitems; i0 += 16) {
                const int item = i0 + (lane >> 1);
                const bool live = item < nitems;
                const int t = item < nbr ? wb + item : q;
                double v[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const int cc = u * cnt2 + k;
                    v[k] = (live && k < cnt2 && cc < Pc) ? ib[cc * q1p + t] : 0.0;
                }
                double tot = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
                tot += __shfl_xor_sync(0xffffffffu, tot, 1);
                if (G > 1) {
                    // cluster totals -> tagged words [par][cluster][t]; sum over clusters in order
                    const unsigned tag = (unsigned)kk + 1u;
                    unsigned long long* ll = reinterpret_cast<unsigned long long*>(a.part) + (size_t)par * G * q1 * 2;
                    if (cr == 0 && u == 0 && live && (item < nbr || warp == 0))
                        ll_store(ll + ((size_t)gid * q1 + t) * 2, tot, tag);
                    if (u == 0 && live) tot = ll_sum<RKA_MAXG>(ll + 2 * t, 2 * q1, G, tag, &a.status->aborted);
                    tot = __shfl_sync(0xffffffffu, tot, lane & ~1);
                }
                if (live && u == 0 && item < nbr) {
                    const double2 bb = bsq[((t >> 2) << 3) + (t & 3)];
                    scal[t] = __ddiv_rn(__dmul_rn(alp[t], __dsub_rn(bb.x, tot)), bb.y);
                }
                if (item == nbr) errv = tot;
            }
            if (want_check) err = __shfl_sync(0xffffffffu, errv, 2 * (nbr & 15));
        }
        if (want_check) {
            ++checks;
            err_last = err;
            if (err < a.eps) {
                conv = 1;
                break;
            }
        }
        if (last) break;
        __syncwarp();
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 4] = clock64();
        // ---- 5. average over this warp's workers -----------------------------------------
        double2 acc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = make_double2(0.0, 0.0);
        for (int rb = wb; rb < we; rb += 8) {
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int t = rb + grp * NR + r;
                if (t < we) {
                    const double s = scal[t];
                    const double* row = rows + t * cwb;
                    const bool first = (r == 0) && (rb == wb);
#pragma unroll
                    for (int e = 0; e < EPL; ++e)
                        if (vld[e]) {
                            const double2 rv = *reinterpret_cast<const double2*>(row + 2 * (gl + LG * e));
                            const double v0 = __dadd_rn(xv[e].x, __dmul_rn(s, rv.x));
                            const double v1 = __dadd_rn(xv[e].y, __dmul_rn(s, rv.y));
                            acc[e].x = first ? v0 : __dadd_rn(acc[e].x, v0);
                            acc[e].y = first ? v1 : __dadd_rn(acc[e].y, v1);
                        }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);  // this warp is done with the stage
        bool have = gh;
#pragma unroll
        for (int o = LG; o < 32; o <<= 1) {  // lane groups of the warp, fixed order
            const bool oh = __shfl_xor_sync(0xffffffffu, have, o);
            const bool lo = (lane & o) == 0;
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                const double ox = __shfl_xor_sync(0xffffffffu, acc[e].x, o);
                const double oy = __shfl_xor_sync(0xffffffffu, acc[e].y, o);
                if (have && oh) {
                    acc[e].x = lo ? __dadd_rn(acc[e].x, ox) : __dadd_rn(ox, acc[e].x);
                    acc[e].y = lo ? __dadd_rn(acc[e].y, oy) : __dadd_rn(oy, acc[e].y);
                } else if (oh) {
                    acc[e] = make_double2(ox, oy);
                }
            }
            have = have || oh;
        }
        if (grp == 0 && warp < nwv) {
#pragma unroll
            for (int e = 0; e < EPL; ++e)
                if (vld[e]) *reinterpret_cast<double2*>(upd + warp * cwb + 2 * (gl + LG * e)) = acc[e];
        }
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 5] = clock64();
        named_sync(CBAR, NW * 32);
        // ---- combine: every warp forms x_{k+1} for its own lanes (fixed tree over warps) --
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            if (!vld[e]) continue;
            const int j = 2 * (gl + LG * e);
            double2 w[NW];
            if (nwv == NW) {
#pragma unroll
                for (int i = 0; i < NW; ++i) w[i] = *reinterpret_cast<const double2*>(upd + i * cwb + j);
#pragma unroll
                for (int h = 1; h < NW; h <<= 1)
#pragma unroll
                    for (int i = 0; i + h < NW; i += 2 * h) {
                        w[i].x = __dadd_rn(w[i].x, w[i + h].x);
                        w[i].y = __dadd_rn(w[i].y, w[i + h].y);
                    }
            } else {
#pragma unroll
                for (int i = 0; i < NW; ++i)
                    w[i] = i < nwv ? *reinterpret_cast<const double2*>(upd + i * cwb + j) : make_double2(0.0, 0.0);
#pragma unroll
                for (int h = 1; h < NW; h <<= 1)
#pragma unroll
                    for (int i = 0; i + h < NW; i += 2 * h)
                        if (i + h < nwv) {
                            w[i].x = __dadd_rn(w[i].x, w[i + h].x);
                            w[i].y = __dadd_rn(w[i].y, w[i + h].y);
                        }
            }
            if (a.partial) {  // row-sharded step: un-normalised local sum
                if (warp == 0 && grp == 0 && vld[e]) {
                    __stcg(a.partial + c0 + j, w[0].x);
                    __stcg(a.partial + c0 + j + 1, w[0].y);
                }
                continue;
            }
            xv[e].x = qpow2 ? __dmul_rn(w[0].x, invq) : __ddiv_rn(w[0].x, qd);
            xv[e].y = qpow2 ? __dmul_rn(w[0].y, invq) : __ddiv_rn(w[0].y, qd);
        }
        if (ckpt_on && warp == 0 && grp == 0) {
            const int64_t k = a.k0 + kk;
            if (((k + 1) % a.ckpt_every) == 0 && ((k + 1) / a.ckpt_every) <= a.ckpt_cap) {
                const int64_t slot = (k + 1) / a.ckpt_every - 1;
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (vld[e]) {
                        const int j = 2 * (gl + LG * e);
                        if (c0 + j < a.n) a.ckpt[slot * a.n + c0 + j] = xv[e].x;
                        if (c0 + j + 1 < a.n) a.ckpt[slot * a.n + c0 + j + 1] = xv[e].y;
                    }
            }
        }
        if (warp == 0) errp = slice_err();
        if (TIMING && rec) a.dbg[(kk * 8 + warp) * 8 + 6] = clock64();
        if (++st == D) {
            st = 0;
            fph ^= 1u;
        }
        done = kk + 1;
    }
    if (tid == 0) *halt = 1;
    if (!a.partial && warp == 0 && grp == 0) {
#pragma unroll
        for (int e = 0; e < EPL; ++e)
            if (vld[e]) {
                const int j = 2 * (gl + LG * e);
                __stcg(a.x + c0 + j, xv[e].x);
                __stcg(a.x + c0 + j + 1, xv[e].y);
            }
    }
    __syncthreads();
    cluster_sync_all();  // no DSMEM traffic may target an exited CTA
    if (c == 0 && tid == 0) {
        a.status->iters_done = done;
        a.status->converged = conv;
        a.status->checks = checks;
        a.status->err = err_last;
    }
}

template __global__ void rka_kernel<8, 1, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, true>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);

}  // namespace kz
