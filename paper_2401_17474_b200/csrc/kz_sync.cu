// kz_sync.cu -- column-sliced persistent kernel for RKA (and RKAB with bs = 1).
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   rka_combined_step  solvers.py:120-137   q projections from one snapshot of x;
//                                            x = (sum_t fl(x + fl(s_t a_t))) / q
//   solve_rka_seq      solvers.py:313-334   rows of iteration k: one draw per worker stream
//   _drive stop rule   solvers.py:229-243
//
// Layout: P CTAs each own a contiguous column slice [c0, c1) of x (shared
// memory) and of every sampled row.  Per iteration k:
//   1. the q row slices (indices are x-independent, known ahead) stream
//      HBM -> smem through a cp.async ring `stages` iterations deep, with the
//      packed (b_i, ||a_i||^2) pairs;
//   2. LPR lanes per row form the partial dot <a_t[c0:c1], x[c0:c1]>;
//   3. exchange (CLUSTER): each warp redistributes its rows' partials over
//      its lanes with shuffles and every lane pushes them (st.async, 16 B)
//      into one peer CTA's receive buffer, completing that CTA's mbarrier
//      transaction count; each CTA then waits on its own mbarrier -- no
//      cluster barrier, no GPU-scope fence.  With G > 1 clusters (column
//      slices over all G x Pc CTAs) each cluster's rank-0 CTA then publishes
//      its cluster totals as tagged 64-bit words (value halves + iteration
//      tag, single-copy atomic) and every CTA polls the G words of its
//      workers: one L2 round trip, no grid barrier, no fence.  Grid mode:
//      global memory and a grid barrier.  The partial of ||x - x_ref||^2
//      rides along as entry q (its per-warp pieces come from the previous
//      iteration's combine);
//   4. scales: warp w owns the w-th contiguous block of workers; its lanes
//      add that block's P partials with one fixed tree (bit-identical in
//      every CTA) and form s_t = alpha (b - d) / ||a||^2;
//   5. average: every lane (= column) sums fl(x + fl(s_t a_t)) over its
//      warp's worker block; one CTA barrier; the per-warp sums of a column
//      are added by a fixed shuffle tree and divided by q.  (The reference
//      adds the q terms strictly left to right; regrouping changes the mean
//      by a few ulp -- tolerance parity, like the dot product.)
// Two CTA barriers per iteration.  All shared-memory index math is 32-bit.
#include "kz_kernels.cuh"

namespace kz {

namespace {
constexpr int NT = 256;           // threads per CTA
constexpr int NW = NT / 32;       // warps per CTA
constexpr int MAXP_TREE = 16;     // cluster size bound for the partial-sum tree
constexpr int IDX_PER_THREAD = 4;
constexpr int CPW = 32 / NW;      // columns per warp per combine round
constexpr int SEG_MAX = 64;       // workers per warp block
constexpr int MAXG = 10;          // clusters exchanging through tagged global words
}  // namespace

template <bool CLUSTER, int LPR>
__global__ void __launch_bounds__(NT) sync_kernel(SolveArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.halt != nullptr && *a.halt != 0) return;  // stopped earlier in the stream: uniform over the grid
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = a.stages;
    const int ld = (int)a.ld, q = (int)a.q;
    const int P = (int)gridDim.x;  // column slices
    const int c = (int)blockIdx.x;
    // exchange group: the thread-block cluster (CLUSTER) or the whole grid; with
    // several clusters (G > 1) their totals meet through tagged global words
    const int Pc = CLUSTER ? (int)cluster_size() : P;
    const int cr = CLUSTER ? (int)cluster_rank() : c;
    const int G = P / Pc, gid = c / Pc;
    const int cw = (((ld + P - 1) / P) + 1) & ~1;  // even => 16-byte pairs
    const int c0 = c * cw < ld ? c * cw : ld;
    const int c1 = (c0 + cw < ld) ? c0 + cw : ld;
    const int wdt = c1 - c0;  // this CTA's columns (may be 0); even
    const int npairs = cw / 2;
    const int rs = cw + 2;    // smem row stride: +16 B staggers banks across rows
    const int q1 = q + 1;
    const int q1p = (q1 + 1) & ~1;  // receive-row stride, even => 16-byte pushes
    const int stage_elems = q * rs;

    // shared memory carve (sync_smem() in kz_api.cu must match)
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem_raw);  // 2 mbarriers
    double* ring = reinterpret_cast<double*>(smem_raw + 16);                      // D x q x rs
    double2* bq = reinterpret_cast<double2*>(ring + D * stage_elems);             // D x q (b_i, sq_i)
    double* xs = reinterpret_cast<double*>(bq + D * q);                           // cw
    double* xrs = xs + cw;                                                         // cw
    double* inbuf = xrs + cw;                                                      // 2 x Pc x q1p (cluster)
    double* upd = inbuf + (CLUSTER ? 2 * Pc * q1p : 0);                            // NW x cw
    double* scal = upd + NW * cw;                                                  // NW x SEG_MAX
    double* errw = scal + NW * SEG_MAX;                                            // NW
    double* alp = errw + NW;                                                       // q
    int32_t* iring = reinterpret_cast<int32_t*>(alp + q);                          // 8 x q

    for (int j = tid; j < cw; j += NT) {
        xs[j] = (j < wdt) ? __ldcg(a.x + c0 + j) : 0.0;
        xrs[j] = (j < wdt) ? a.xref[c0 + j] : 0.0;
    }
    for (int t = tid; t < q; t += NT) alp[t] = a.alphas[t];
    // row indices: iterations 0..D in the 8-slot ring; D+1 held in registers
    for (int u = tid; u < (D + 1) * q; u += NT) {
        const int it = u / q, t = u - it * q;
        if (it < a.count) iring[(it & 7) * q + t] = a.idx[(int64_t)it * q + t];
    }
    int32_t pend[IDX_PER_THREAD];
#pragma unroll
    for (int r = 0; r < IDX_PER_THREAD; ++r) {
        const int t = tid + r * NT;
        pend[r] = (t < q && D + 1 < a.count) ? a.idx[(int64_t)(D + 1) * q + t] : 0;
    }
    if (CLUSTER && tid == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        fence_mbarrier_init_cluster();
    }
    __syncthreads();
    // per-warp pieces of ||x - x_ref||^2 over the slice (combine-step layout)
    const int jo = lane / NW, w8 = lane % NW;
    {
        double e = 0.0;
        for (int j0 = warp * CPW; j0 < wdt; j0 += NW * CPW) {
            const int j = j0 + jo;
            if (w8 == 0 && j < wdt) {
                const double d = xs[j] - xrs[j];
                e = fma(d, d, e);
            }
        }
        e = warp_sum(e);
        if (lane == 0) errw[warp] = e;
    }
    __syncthreads();
    if (CLUSTER) cluster_sync_all();  // peers' mbarriers exist before anyone pushes

    // cp.async issue: tpr threads per row (power of two), pairs strided by tpr
    int tpr = 1;
    while (tpr < npairs && tpr < 32) tpr <<= 1;
    const int rows_per_pass = NT / tpr, my_r = tid / tpr, my_p = tid % tpr;
    const bool one_pair = npairs <= tpr;
    const bool pair_ok = my_p < npairs && 2 * my_p < wdt;
    const double* Ac0 = a.A + c0 + 2 * my_p;
    const double2* bs2 = reinterpret_cast<const double2*>(a.bs2);
    auto issue = [&](int64_t it, int st) {
        if (it < a.count) {
            const int32_t* ir = iring + (int)(it & 7) * q;
            double* dst = ring + st * stage_elems + 2 * my_p;
            if (one_pair) {
                if (pair_ok)
#pragma unroll 4
                    for (int t = my_r; t < q; t += rows_per_pass)
                        cp_async16(dst + t * rs, Ac0 + (int64_t)ir[t] * ld);
            } else {
                for (int t = my_r; t < q; t += rows_per_pass) {
                    const double* src = Ac0 + (int64_t)ir[t] * ld;
                    for (int p = 0; 2 * (my_p + p) < wdt; p += tpr) cp_async16(dst + t * rs + 2 * p, src + 2 * p);
                }
            }
            for (int t = tid; t < q; t += NT) cp_async16(bq + st * q + t, bs2 + 2 * ir[t]);
        }
        cp_async_commit();
    };

    // push layout: lane -> (peer r = lane % P, part = lane / P); each part of a
    // warp's G_w rows goes to peer r as 16-byte st.async pairs
    constexpr int G_w = 32 / LPR;                       // rows per warp per round
    const int parts = (Pc >= 32) ? 1 : 32 / Pc;
    const int vpp = (G_w + parts - 1) / parts;          // rows per lane
    const int peer = lane % Pc, part = lane / Pc;
    unsigned rin = 0, rbar = 0;
    if (CLUSTER) {
        rin = mapa_u32(smem_u32(inbuf), (unsigned)peer);
        rbar = mapa_u32(smem_u32(bars), (unsigned)peer);
    }

    for (int j = 0; j < D - 1; ++j) issue(j, j);
    int st = 0;  // ring stage of iteration kk

    unsigned epoch = 0;
    long long done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;
    const double qd = (double)q;
    constexpr int groups = NT / LPR;
    const int g = tid / LPR, gl = tid % LPR;
    const unsigned xfer_bytes = (unsigned)(Pc * q1 * sizeof(double));
    // worker block of this warp for the scale / average steps
    const int tb = (q * warp) / NW, te = (q * (warp + 1)) / NW, nseg = te - tb;
    const bool ckpt_on = a.ckpt_every > 0;
    const bool w8_live = (q * (w8 + 1)) / NW > (q * w8) / NW;

    for (int64_t kk = 0;; ++kk) {
        const bool last = (kk == a.count);
        const bool want_check = a.use_stop && (!last || a.final_check);
        if (last && !want_check) break;
        const int par = (int)(kk & 1);
        const double* rows = ring + st * stage_elems;
        if (!last) cp_async_wait_dyn(D - 2);
        __syncthreads();  // (A) stage kk visible; x, errw of iteration kk-1 complete
        const bool rec = a.dbg != nullptr && c == 0 && lane == 0 && kk < 32;
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 0] = clock64();
        if (CLUSTER && tid == 0) mbar_arrive_expect_tx(&bars[par], xfer_bytes);
        if (!last) {
            issue(kk + D - 1, st == 0 ? D - 1 : st - 1);
            const int64_t itn = kk + D + 1;  // registers -> ring; read by issue() two iterations on
#pragma unroll
            for (int r = 0; r < IDX_PER_THREAD; ++r) {
                const int t = tid + r * NT;
                if (t < q && itn < a.count) {
                    iring[(int)(itn & 7) * q + t] = pend[r];
                    if (itn + 1 < a.count) pend[r] = a.idx[(itn + 1) * q + t];
                }
            }
        }
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 1] = clock64();
        // ---- partial dots over the slice, pushed to every CTA -----------------------
        const unsigned my_off = (unsigned)(((par * Pc + cr) * q1p) * (int)sizeof(double));
        double* gpart = a.part + ((size_t)par * P + c) * q1;
        for (int t0 = 0; t0 < q; t0 += groups) {  // every lane joins each round's shuffles
            const int t = t0 + g;
            double s = 0.0;
            if (t < q && !last) {
                const double* r = rows + t * rs;
#pragma unroll 4
                for (int j = 2 * gl; j < wdt; j += 2 * LPR) {
                    const double2 rv = *reinterpret_cast<const double2*>(r + j);
                    const double2 xv = *reinterpret_cast<const double2*>(xs + j);
                    s = fma(rv.x, xv.x, s);
                    s = fma(rv.y, xv.y, s);
                }
            }
#pragma unroll
            for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LPR);
            if (CLUSTER) {
                const int wrow0 = t0 + warp * G_w;  // first row of this warp in this round
#pragma unroll
                for (int i = 0; i < G_w; i += 2) {
                    if (i >= vpp) break;
                    const int ra = part * vpp + i, rb = ra + 1;  // warp-local row numbers
                    const double va = __shfl_sync(0xffffffffu, s, (ra % G_w) * LPR);
                    const double vb = __shfl_sync(0xffffffffu, s, (rb % G_w) * LPR);
                    const int ta = wrow0 + ra;
                    if (part < parts && ra < G_w && ta < q) {
                        const unsigned off = my_off + (unsigned)(ta * (int)sizeof(double));
                        if (i + 1 < vpp && rb < G_w && ta + 1 < q)
                            st_async_v2_f64(rin + off, va, vb, rbar + 8u * par);
                        else
                            st_async_f64(rin + off, va, rbar + 8u * par);
                    }
                }
            } else if (gl == 0 && t < q) {
                __stcg(gpart + t, s);
            }
        }
        if (warp == 0) {  // error piece of x_k (pieces written by the previous combine)
            double e = errw[0];
#pragma unroll
            for (int w = 1; w < NW; ++w) e = __dadd_rn(e, errw[w]);
            if (CLUSTER) {
                if (lane < Pc) st_async_f64(rin + my_off + (unsigned)(q * (int)sizeof(double)), e, rbar + 8u * par);
            } else if (lane == 0) {
                __stcg(gpart + q, e);
            }
        }
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 2] = clock64();
        // ---- exchange -----------------------------------------------------------------
        if (CLUSTER)
            mbar_wait_cluster(&bars[par], (unsigned)((kk >> 1) & 1));
        else
            grid_barrier(a.barrier, (++epoch) * gridDim.x);
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 3] = clock64();
        auto total = [&](int t) -> double {
            if (CLUSTER) {
                const double* ib = inbuf + par * Pc * q1p + t;
                double v[MAXP_TREE];
#pragma unroll
                for (int cc = 0; cc < MAXP_TREE; ++cc) v[cc] = (cc < Pc) ? ib[cc * q1p] : 0.0;
#pragma unroll
                for (int w = 1; w < MAXP_TREE; w <<= 1)
#pragma unroll
                    for (int i = 0; i + w < MAXP_TREE; i += 2 * w) v[i] = __dadd_rn(v[i], v[i + w]);
                return v[0];
            }
            const double* gp = a.part + (size_t)par * P * q1 + t;
            double buf[8];
            double s = 0.0;
            for (int cc0 = 0; cc0 < P; cc0 += 8) {  // 8 independent loads in flight
#pragma unroll
                for (int u = 0; u < 8; ++u) buf[u] = (cc0 + u < P) ? __ldcg(gp + (size_t)(cc0 + u) * q1) : 0.0;
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (cc0 + u < P) s = (cc0 + u == 0) ? buf[u] : __dadd_rn(s, buf[u]);
            }
            return s;
        };
        // ---- scales of this warp's workers; lanes past the block form the error total --
        double err = 0.0;
        {
            const double2* bqs = bq + st * q;
            const int tA = (lane < nseg) ? tb + lane : q;
            const int tB = tb + 32 + lane;
            const bool needA = lane < nseg || (want_check && nseg < 32);
            const bool needB = nseg > 32 && 32 + lane < nseg;
            const bool needE = want_check && nseg >= 32;
            double vA = needA ? total(tA) : 0.0;
            double vB = needB ? total(tB) : 0.0;
            double vE = needE ? total(q) : 0.0;
            if (CLUSTER && G > 1) {
                // cluster totals -> tagged words [par][cluster][t]; every CTA adds the
                // G cluster totals in cluster order (bit-identical everywhere)
                const unsigned tag = (unsigned)kk + 1u;
                unsigned long long* ll = reinterpret_cast<unsigned long long*>(a.part) + (size_t)par * G * q1 * 2;
                if (cr == 0) {
                    unsigned long long* mine = ll + (size_t)gid * q1 * 2;
                    if (lane < nseg) ll_store(mine + 2 * tA, vA, tag);
                    if (needB) ll_store(mine + 2 * tB, vB, tag);
                    if (warp == 0 && want_check && lane == (nseg < 32 ? nseg : 0))
                        ll_store(mine + 2 * q, nseg < 32 ? vA : vE, tag);
                }
                int* abort = &a.status->aborted;
                if (needA) vA = ll_sum<MAXG>(ll + 2 * tA, 2 * q1, G, tag, abort);
                if (needB) vB = ll_sum<MAXG>(ll + 2 * tB, 2 * q1, G, tag, abort);
                if (needE) vE = ll_sum<MAXG>(ll + 2 * q, 2 * q1, G, tag, abort);
            }
            if (lane < nseg && !last) {
                const double2 bb = bqs[tA];
                scal[warp * SEG_MAX + lane] = __ddiv_rn(__dmul_rn(alp[tA], __dsub_rn(bb.x, vA)), bb.y);
            }
            if (needB && !last) {
                const double2 bb = bqs[tB];
                scal[warp * SEG_MAX + 32 + lane] = __ddiv_rn(__dmul_rn(alp[tB], __dsub_rn(bb.x, vB)), bb.y);
            }
            if (want_check) err = (nseg < 32) ? __shfl_sync(0xffffffffu, vA, 31) : vE;
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
        st = (st + 1 == D) ? 0 : st + 1;
        __syncwarp();
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 4] = clock64();
        // ---- average over the q projections (solvers.py:131-137) ----------------------
        {
            const double* sw = scal + warp * SEG_MAX;
            for (int j0 = 0; j0 < wdt; j0 += 32) {
                const int j = j0 + lane;
                const int jj = j < wdt ? j : 0;
                const double xj = xs[jj];
                const double* rj = rows + tb * rs + jj;
                double acc = 0.0;
                int u = 0;
                for (; u + 2 <= nseg; u += 2) {
                    const double2 s2 = *reinterpret_cast<const double2*>(sw + u);
                    const double v0 = __dadd_rn(xj, __dmul_rn(s2.x, rj[u * rs]));
                    const double v1 = __dadd_rn(xj, __dmul_rn(s2.y, rj[(u + 1) * rs]));
                    acc = (u == 0) ? __dadd_rn(v0, v1) : __dadd_rn(__dadd_rn(acc, v0), v1);
                }
                if (u < nseg) {
                    const double v = __dadd_rn(xj, __dmul_rn(sw[u], rj[u * rs]));
                    acc = (u == 0) ? v : __dadd_rn(acc, v);
                }
                if (j < wdt) upd[warp * cw + j] = acc;
            }
        }
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 5] = clock64();
        __syncthreads();  // (B) per-warp sums complete
        {
            const int64_t k = a.k0 + kk;
            bool ck = false;
            int64_t slot = 0;
            if (ckpt_on) {
                ck = ((k + 1) % a.ckpt_every) == 0 && ((k + 1) / a.ckpt_every) <= a.ckpt_cap;
                slot = (k + 1) / a.ckpt_every - 1;
            }
            double e = 0.0;
            for (int j0 = warp * CPW; j0 < wdt; j0 += NW * CPW) {
                const int j = j0 + jo;
                double v = (w8_live && j < wdt) ? upd[w8 * cw + j] : 0.0;
#pragma unroll
                for (int o = NW / 2; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o, NW));
                if (w8 == 0 && j < wdt && a.partial) {  // row-sharded step: un-normalised local sum
                    __stcg(a.partial + c0 + j, v);
                } else if (w8 == 0 && j < wdt) {
                    const double xn = __ddiv_rn(v, qd);
                    xs[j] = xn;
                    const double d = xn - xrs[j];
                    e = fma(d, d, e);
                    if (ck && c0 + j < a.n) a.ckpt[slot * a.n + c0 + j] = xn;
                }
            }
            e = warp_sum(e);
            if (lane == 0) errw[warp] = e;
        }
        if (rec) a.dbg[(kk * 8 + warp) * 8 + 6] = clock64();
        done = kk + 1;
    }
    cp_async_wait<0>();
    __syncthreads();
    if (!a.partial)
        for (int j = tid; j < wdt; j += NT) __stcg(a.x + c0 + j, xs[j]);
    if (CLUSTER) cluster_sync_all();  // no DSMEM traffic may target an exited CTA
    if (c == 0 && tid == 0) {
        a.status->iters_done = done;
        a.status->converged = conv;
        a.status->checks = checks;
        a.status->err = err_last;
    }
}

template __global__ void sync_kernel<true, 4>(SolveArgs);
template __global__ void sync_kernel<true, 8>(SolveArgs);
template __global__ void sync_kernel<true, 32>(SolveArgs);
template __global__ void sync_kernel<false, 4>(SolveArgs);
template __global__ void sync_kernel<false, 8>(SolveArgs);
template __global__ void sync_kernel<false, 32>(SolveArgs);

}  // namespace kz
