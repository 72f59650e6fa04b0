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
//       2. reduce-scatter: worker t's partial goes to its owner, cluster rank
//          t / RPO (16-byte st.async for row pairs, completing the owner's
//          mbarrier); warp 0 sends the slice's ||x - x_ref||^2 piece as item q;
//       3. the owner warp (7) adds the Pc partials of its items with one fixed
//          tree, forms s_t = alpha_t (b_t - d_t) / ||a_t||^2 and broadcasts the
//          scales (and the error total) to every CTA of the cluster -- two
//          DSMEM hops carrying q values each instead of an all-to-all of q x Pc.
//          With G > 1 clusters the owners first exchange their cluster totals
//          as tagged 64-bit words (value halves + iteration tag, single-copy
//          atomic; no grid barrier, no fence; one 128-byte L2 line per slot),
//          polled one word per lane, and add them in cluster order;
//       4. stop rule on the broadcast error total;
//       5. average: each warp sums fl(x + fl(s_t a_t)) over its block; the 8
//          per-warp sums meet in shared memory behind one named barrier and
//          every warp forms x_{k+1} (fixed tree, / q) for its own lanes, so x
//          never leaves registers.
//   One named barrier per iteration; the two mbarriers order everything else
//   (an owner's items complete only after every peer has finished the previous
//   iteration).
#include "kz_kernels.cuh"

namespace kz {

namespace {
constexpr int NW = RKA_NW;

constexpr unsigned XBAR = 2;  // named barrier: producer warp -> compute warps, x_k in place
constexpr unsigned CBAR = 1;  // named barrier id of the compute warps
}  // namespace

template <int LG, int EPL, bool TIMING, bool SR, int MODE>
__global__ void __launch_bounds__(RKA_NT, 1) rka_kernel(const __grid_constant__ SolveArgs a,
                                                        const __grid_constant__ CUtensorMap tmA,
                                                        const __grid_constant__ CUtensorMap tmB) {
    constexpr int NR = LG / 4;  // rows per lane group per round (8 rows per warp per round)
    // rows whose shared-memory loads are issued together (RB x EPL 16-byte loads in flight per lane)
#ifndef KZ_RKA_PF
#define KZ_RKA_PF 2  // worker groups: L2 prefetch distance in iterations (0 = off)
#endif
    constexpr int RBW = EPL <= 1 ? NR : (EPL == 2 ? 4 : (EPL == 3 ? 2 : 1));
    constexpr int RB = NR < RBW ? NR : RBW;
    static_assert(LG == 8 || LG == 16 || LG == 32, "lane group");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    if (a.halt != nullptr && *a.halt != 0) return;  // stopped earlier in the stream: uniform over the grid
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int D = a.stages;
    const int ld = (int)a.ld, qa = (int)a.q;
    const int P = (int)gridDim.x, c = (int)blockIdx.x;
    const int Pc = (int)cluster_size(), cr = (int)cluster_rank();
    const int G = P / Pc, gid = c / Pc;
    // worker-group mode (a.wg): cluster g runs workers [wlo, wlo + q) over all columns (split over its
    // Pc CTAs) and the clusters add their per-column sums through tagged words; otherwise every
    // cluster runs all workers over its share of the columns and the clusters add dot totals
    constexpr bool wg = MODE == 1;  // separate instantiations: the column-sliced kernel keeps its register budget
    constexpr bool xr = MODE == 2;  // cross-rank: local column slices, column sums exchanged between GPUs
    const int Gx = wg ? 1 : G;                      // clusters exchanging dot totals
    const int gx = wg ? 0 : gid;
    const int wlo = wg ? (int)((int64_t)gid * qa / G) : 0;
    const int q = wg ? (int)((int64_t)(gid + 1) * qa / G) - wlo : qa;  // this cluster's workers
    const int PC = wg ? Pc : P, cc = wg ? cr : c;   // CTAs splitting the columns, this CTA's slice
    const int cw = (((ld + PC - 1) / PC) + 1) & ~1;
    const int c0 = cc * cw < ld ? cc * cw : ld;
    const int wdt = (c0 + cw < ld ? c0 + cw : ld) - c0;  // even
    const int cwb = a.box;                               // >= cw, multiple of 4
    const int q4 = (q + 3) & ~3;
    const int q1 = q + 1, q1p = (q1 + 1) & ~1;
    const int RPO = (((q + Pc - 1) / Pc) + 1) & ~1;  // workers per owner, even; the error belongs to rank Pc-1
    const int my_lo = cr * RPO < q ? cr * RPO : q;
    const int n_own = (my_lo + RPO < q ? my_lo + RPO : q) - my_lo;  // workers this CTA owns
    const int QB = (((q + NW - 1) / NW) + 1) & ~1;  // even: rows pair up into 16-byte pushes
    const int nwv = (q + QB - 1) / QB;  // warps owning at least one worker
    const unsigned rows_bytes = (unsigned)(q4 * cwb * 8);
    const int RPO4 = (RPO + 3) & ~3;
    const int stage_bytes = (int)rows_bytes + RPO4 * 32;  // rows, then the owned workers' (b, sq, 1/sq, 0)

    // shared memory carve (rka_smem() in kz_api.cu must match)
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem_raw);  // D <= 8
    unsigned long long* empty = full + 8;                                       // D
    unsigned long long* xbar = full + 16;                                       // 2: partials at the owner
    unsigned long long* sbar = full + 18;                                       // 2: scales everywhere
    unsigned long long* ebin = full + 20;                                       // 2: error pieces at rank Pc-1
    unsigned long long* ebar = full + 22;                                       // 2: error total everywhere
    volatile int* halt = reinterpret_cast<volatile int*>(smem_raw + 192);
    unsigned char* ring = smem_raw + 256;                                // D x stage_bytes
    double* inbuf = reinterpret_cast<double*>(ring + D * stage_bytes);  // 2 x Pc x RPO (owner side)
    double* scal = inbuf + 2 * Pc * RPO;                                 // 2 x q4 scales
    double* ein = scal + 2 * q4;                                         // 2 x Pc error pieces (rank Pc-1)
    double* errs = ein + 2 * Pc;                                         // 2 error totals
    double* sout = errs + 2;                                             // RPO (owner staging)
    double* upd = sout + RPO;                                            // NW x cwb
    double* xrs = upd + NW * cwb;                                        // cwb: x_ref slice
    double* xs = xrs + cwb;                                              // cwb: x_{k+1} (split combine)
    double* alp = xs + cwb;                                              // q

    if (tid == 0) {
        for (int i = 0; i < D; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], NW);
        }
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        mbar_init(&sbar[0], 1);
        mbar_init(&sbar[1], 1);
        mbar_init(&ebin[0], 1);
        mbar_init(&ebin[1], 1);
        mbar_init(&ebar[0], 1);
        mbar_init(&ebar[1], 1);
        *halt = 0;
        fence_mbarrier_init_cluster();
    }
    for (int t = tid; t < q; t += RKA_NT) alp[t] = a.alphas[wlo + t];
    __syncthreads();
    cluster_sync_all();  // peers' mbarriers exist before anyone pushes

    if (warp == NW) {
        // ================= producer warp =================
        if (a.x_sum) {  // row-sharded step: x_k = the all-reduced worker sum / Q (kz_average_from's division)
            for (int j = lane; j < wdt; j += 32) a.x[c0 + j] = __ddiv_rn(__ldcg(a.x_sum + c0 + j), a.x_div);
            named_sync(XBAR, RKA_NT);
        }
        const int ng = q4 / 4, nbg = (n_own + 3) / 4;
        const unsigned bytes = rows_bytes + (unsigned)nbg * 128u;
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
            if (TIMING && (a.ablate & 32) && it >= D) {  // ablation: no refills (stale rows), the stage completes at once
                if (lane == 0) mbar_arrive(&full[s]);
                __syncwarp();
                if (++s == D) s = 0;
                continue;
            }
            const unsigned dst = ring_u + (unsigned)(s * stage_bytes);
            const int32_t* ix = a.idx + it * qa + wlo;
            if (lane == 0) mbar_arrive_expect_tx(&full[s], bytes);
            __syncwarp();
            const unsigned fb = smem_u32(&full[s]);
            // all q row slices; the (b, sq, 1/sq) records only of the workers this CTA owns
            // (its owner warps are their only readers): q/4 + RPO/4 gathers per iteration
            for (int op = lane; op < ng + nbg; op += 32) {
                int r[4];
                if (op < ng) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) r[u] = __ldg(ix + (4 * op + u < q ? 4 * op + u : q - 1));
                    tma_gather4(dst + (unsigned)(op * 4 * cwb * 8), &tmA, c0, r[0], r[1], r[2], r[3], fb);
                } else {
                    const int g = op - ng;
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        r[u] = __ldg(ix + my_lo + (4 * g + u < n_own ? 4 * g + u : n_own - 1));
                    tma_gather4(dst + rows_bytes + (unsigned)(g * 128), &tmB, 0, r[0], r[1], r[2], r[3], fb);
                }
            }
#if KZ_RKA_PF > 0
            // worker groups: the row slices of iteration it + KZ_RKA_PF into L2, so the ring's refills
            // (~q/G rows of every column box per CTA, two or three stages deep) hit L2 instead of HBM
            // (c4 q = 512: 5.03 -> 4.75 us per iteration; the column-sliced plans do not gain and the
            // one-cluster ones lose -- 64 more bulk instructions per 2 us iteration -- so they skip it)
            if (wg && it + KZ_RKA_PF < a.count) {
                const int32_t* ixp = a.idx + (it + KZ_RKA_PF) * qa + wlo;
                for (int t = lane; t < q; t += 32)
                    prefetch_l2_bulk(a.A + (size_t)__ldg(ixp + t) * (size_t)ld + c0, (unsigned)(wdt * 8));
            }
#endif
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
    constexpr int OW = NW - 1;    // owner warp of the error total
    constexpr int NOWN = 2;       // owner warps (NW - NOWN .. NW - 1) splitting the worker pairs
    const int gl = lane % LG, grp = lane / LG;
    double2 xv[EPL];
    for (int j = tid; j < cwb; j += NW * 32) xrs[j] = j < wdt ? a.xref[c0 + j] : 0.0;
    if (a.x_sum) named_sync(XBAR, RKA_NT);  // the producer warp formed x_k = x_sum / Q (row-sharded step)
    named_sync(CBAR, NW * 32);
    bool vld[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
        const int j = 2 * (gl + LG * e);
        vld[e] = j < wdt;
        xv[e] = vld[e] ? make_double2(__ldcg(a.x + c0 + j), __ldcg(a.x + c0 + j + 1)) : make_double2(0.0, 0.0);
    }

    // reduced-row bookkeeping: after the transposed reduction lane gl holds row ri
    // of its group; lanes differing in the low two bits hold the same value and
    // rows ri, ri ^ 1 sit on lanes gl, gl ^ 4
    int ri = 0;
#pragma unroll
    for (int h = NR / 2, o = LG / 2; h >= 1; h >>= 1, o >>= 1)
        if (gl & o) ri += h;
    const unsigned inbuf_u = smem_u32(inbuf), xbar_u = smem_u32(xbar), scal_u = smem_u32(scal),
                   sbar_u = smem_u32(sbar), ein_u = smem_u32(ein), ebin_u = smem_u32(ebin),
                   errs_u = smem_u32(errs), ebar_u = smem_u32(ebar);

    const int wb = warp * QB < q ? warp * QB : q;
    const int we = wb + QB < q ? wb + QB : q;
    const int eown = Pc - 1;                                          // owner of the error total
    const bool gh = we - wb > grp * NR;  // this lane group owns at least one worker
    // x = (sum over all workers) / their count: qa here, q x ranks across GPUs
    const double qd = xr ? a.x_div : (double)qa;
    const int64_t qall = (int64_t)qd;
    const bool qpow2 = (qall & (qall - 1)) == 0;
    const double invq = 1.0 / qd;  // RN(1/Q): exact for powers of two, Markstein otherwise
    const bool ckpt_on = a.ckpt_every > 0;
    const int count = (int)a.count;
    const bool use_stop = opaque_i32(a.use_stop) != 0, final_check = opaque_i32(a.final_check) != 0;
    const int cnt2 = Pc >= 2 ? Pc / 2 : 1;  // partials per lane in the owner's tree (2 lanes per item)
    bool unit_alpha = true;
    for (int t = 0; t < q; ++t) unit_alpha = unit_alpha && alp[t] == 1.0;
    const bool split = wg || xr || (TIMING && (a.ablate & 16)) || cwb >= 64 || LG == 8;  // combine layout
    const int ppw = ((wdt >> 1) + NW - 1) / NW;                      // column pairs per warp (split)
    const int u = lane & 1;

    // owner tree: item i's Pc partials (stride `stride`) added by lanes 2i, 2i+1 in one fixed order
    auto owner_total = [&](const double* base, int stride, bool live) -> double {
        double v[8];
        if (Pc == 16) {  // the common cluster: 8 partials per lane, no bounds
            const double* bp = base + u * 8 * stride;
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = live ? bp[k * stride] : 0.0;
        } else {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int cc = u * cnt2 + k;
                v[k] = (live && k < cnt2 && cc < Pc) ? base[cc * stride] : 0.0;
            }
        }
        double tot = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
        tot += __shfl_xor_sync(0xffffffffu, tot, 1);
        return tot;
    };

    // per-lane constants: element offsets of the lane's rows in round 0 (later rounds
    // add 8 rows), the round-0 reduce-scatter target, the owner's broadcast slots
    // (opaque copies: keeps them in registers instead of re-deriving from the parameter bank)
    int roff[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) roff[r] = opaque_i32((wb + grp * NR + r) * cwb + 2 * gl);
    const int rstep = opaque_i32(8 * cwb);
    const int t_push0 = wb + grp * NR + ri;
    const int o_push0 = opaque_i32(t_push0 / RPO), s_push0 = opaque_i32(t_push0 - (t_push0 / RPO) * RPO);
    int pcs = 0;
    while ((1 << pcs) < Pc) ++pcs;  // Pc is a power of two
    const bool pusher = (ri & 1) == 0 && (gl & 3) == 0;
    int rok = 0;  // SR: bit r = row wb + grp NR + r exists
#pragma unroll
    for (int r = 0; r < NR; ++r)
        if (wb + grp * NR + r < we) rok |= 1 << r;
    rok = opaque_i32(rok);
    const bool push_ok = pusher && t_push0 < we, push_pair = t_push0 + 1 < we;

    int st = 0;
    unsigned fph = 0;  // parity of stage st's current full phase
    bool ready = false;  // stage st already awaited (prefetched wait)
    int done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;

    for (int kk = 0;; ++kk) {
        const bool last = (kk == count);
        const bool want_check = use_stop && (!last || final_check);
        if (last && !want_check) break;
        const int par = kk & 1;
        const unsigned bpar = (unsigned)((kk >> 1) & 1);
        // phase stamps (KZ_PHASE_TIMING): rank 0 of every cluster, lane 0 of every warp, iterations < 32,
        // slot [cluster][iteration][warp][16]
        const bool rec = TIMING && a.dbg != nullptr && cr == 0 && lane == 0 && kk < 32;
        long long* const stamp = TIMING ? a.dbg + ((size_t)(gid * 32 + kk) * 8 + warp) * 16 : nullptr;
        // every CTA: globaltimer at 4 events of the iteration (dots done, owner total, cross-cluster sum,
        // scales arrived), slot [65536 + (c * 32 + kk) * 4 + event]
        const bool rec_all = TIMING && a.dbg != nullptr && lane == 0 && kk < 32;
        long long* const gstamp = TIMING ? a.dbg + 65536 + ((size_t)c * 32 + kk) * 4 : nullptr;
        if (TIMING && rec) {
            stamp[0] = clock64();
            stamp[14] = (long long)globaltimer_ns();
        }
        if (tid == 32) {  // warp 1: not on the producer warp's scheduler (warps 0, 4, 8 share one)
            if (!last) {
                if (n_own > 0) mbar_arrive_expect_tx(&xbar[par], (unsigned)(n_own * Pc * (int)sizeof(double)));
                mbar_arrive_expect_tx(&sbar[par], (unsigned)(q * (int)sizeof(double)));
            }
            if (want_check) {
                if (cr == eown) mbar_arrive_expect_tx(&ebin[par], (unsigned)(Pc * (int)sizeof(double)));
                mbar_arrive_expect_tx(&ebar[par], (unsigned)sizeof(double));
            }
        }
        const double* rows = reinterpret_cast<const double*>(ring + st * stage_bytes);
        const double* bsr = reinterpret_cast<const double*>(ring + st * stage_bytes + rows_bytes);
        if (!last && !ready) mbar_wait(&full[st], fph);
        if (TIMING && rec) stamp[1] = clock64();
        // ---- 1-2. partial dots of this warp's rows -> their owners ------------------------
        if (!last) {
            int o_push = o_push0, s_push = s_push0;  // owner, slot of round 0
            // SR (q <= 64): exactly one round of 8 rows per warp, row predicates precomputed
            for (int rb = wb, rofs = 0; SR ? rb == wb && wb < we : rb < we; rb += 8, rofs += rstep) {
                double acc[NR];
                if (SR ? rok == (1 << NR) - 1 : rb + grp * NR + NR <= we) {
                    // all NR rows of the lane group exist: straight-line code, the loads of RB rows issued
                    // together ahead of their FMA chains (per-row branches kept every load behind the
                    // previous row's arithmetic: one exposed shared-memory latency per load)
#pragma unroll
                    for (int r0 = 0; r0 < NR; r0 += RB) {
                        double2 rv[RB][EPL];
#pragma unroll
                        for (int r = 0; r < RB; ++r)
#pragma unroll
                            for (int e = 0; e < EPL; ++e)
                                rv[r][e] = vld[e] ? *reinterpret_cast<const double2*>(rows + roff[r0 + r] + rofs +
                                                                                       2 * LG * e)
                                                  : make_double2(0.0, 0.0);
#pragma unroll
                        for (int r = 0; r < RB; ++r) {
                            double d = 0.0;
#pragma unroll
                            for (int e = 0; e < EPL; ++e)
                                if (vld[e]) {
                                    d = fma(rv[r][e].x, xv[e].x, d);
                                    d = fma(rv[r][e].y, xv[e].y, d);
                                }
                            acc[r0 + r] = d;
                        }
                    }
                } else {
#pragma unroll
                    for (int r = 0; r < NR; ++r) {
                        acc[r] = 0.0;
                        const int t = rb + grp * NR + r;
                        if (SR ? ((rok >> r) & 1) != 0 : t < we) {
                            const double* row = rows + roff[r] + rofs;
#pragma unroll
                            for (int e = 0; e < EPL; ++e)
                                if (vld[e]) {
                                    const double2 rv = *reinterpret_cast<const double2*>(row + 2 * LG * e);
                                    acc[r] = fma(rv.x, xv[e].x, acc[r]);
                                    acc[r] = fma(rv.y, xv[e].y, acc[r]);
                                }
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
                const double odd = __shfl_xor_sync(0xffffffffu, acc[0], 4);
                const int t = rb + grp * NR + ri;
                if (SR ? push_ok : (t < we && pusher)) {
                    const unsigned off = (unsigned)(((par * Pc + cr) * RPO + s_push) * (int)sizeof(double));
                    const unsigned dst = mapa_u32(inbuf_u, (unsigned)o_push) + off;
                    const unsigned bar = mapa_u32(xbar_u + 8u * par, (unsigned)o_push);
                    if (SR ? push_pair : t + 1 < we)
                        st_async_v2_f64(dst, acc[0], odd, bar);
                    else
                        st_async_f64(dst, acc[0], bar);
                }
                if (!SR && rb + 8 < we)
                    for (s_push += 8; s_push >= RPO; s_push -= RPO) ++o_push;  // next round: 8 rows on
            }
        }
        if (TIMING && rec) stamp[13] = clock64();
        if (TIMING && rec_all && warp == 0) gstamp[0] = (long long)globaltimer_ns();
        // ---- error piece of x_k (needed only at the end of the iteration) -----------------
        if (want_check && warp == 0 && !(TIMING && (a.ablate & 1))) {
            double e2 = 0.0;
            if (grp == 0) {
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (vld[e]) {
                        const double2 xr = *reinterpret_cast<const double2*>(xrs + 2 * (gl + LG * e));
                        const double d0 = xv[e].x - xr.x, d1 = xv[e].y - xr.y;
                        e2 = fma(d0, d0, e2);
                        e2 = fma(d1, d1, e2);
                    }
            }
            e2 = warp_sum(e2);
            if (lane == 0)
                st_async_f64(mapa_u32(ein_u, (unsigned)eown) + (unsigned)((par * Pc + cr) * (int)sizeof(double)), e2,
                             mapa_u32(ebin_u + 8u * par, (unsigned)eown));
        } else if (want_check && warp == 0 && lane == 0) {
            st_async_f64(mapa_u32(ein_u, (unsigned)eown) + (unsigned)((par * Pc + cr) * (int)sizeof(double)), 0.0,
                         mapa_u32(ebin_u + 8u * par, (unsigned)eown));
        }
        if (TIMING && rec) stamp[2] = clock64();
        // the next stage's rows are awaited now, while the exchange is in flight
        ready = false;
        if (warp < NW - NOWN && kk + 1 < count) {
            const int st1 = st + 1 == D ? 0 : st + 1;
            mbar_wait(&full[st1], st + 1 == D ? fph ^ 1u : fph);
            ready = true;
        }
        // ---- 3. owner: totals of its workers, scales, broadcast; then the error total -------
        if (warp >= NW - NOWN) {
            // NOWN owner warps: warp ow takes the worker pairs ow, ow + NOWN, ... of this CTA
            const int ow = warp - (NW - NOWN);
            const unsigned tag = (unsigned)kk + 1u;  // the words are zeroed before every launch
            constexpr int lp = RKA_LL_PAD;  // u64 words per slot
            unsigned long long* ll = reinterpret_cast<unsigned long long*>(a.part) + (size_t)par * Gx * q1 * lp;
            const int npair = (n_own + 1) / 2;
            const int my_pairs = npair > ow ? (npair - ow + NOWN - 1) / NOWN : 0;
            if (!last && my_pairs > 0) {
                mbar_wait(&xbar[par], bpar);
                if (TIMING && rec) stamp[7] = clock64();
                const double* ib = inbuf + par * Pc * RPO;
                for (int l0 = 0; l0 < 2 * my_pairs; l0 += 16) {  // 16 items per pass, 2 lanes each
                    const int li = l0 + (lane >> 1);
                    const int i = 2 * (ow + NOWN * (li >> 1)) + (li & 1);
                    const bool live = li < 2 * my_pairs && i < n_own;
                    const int t = my_lo + i;
                    double tot = owner_total(ib + i, RPO, live);
                    if (TIMING && rec && warp == NW - NOWN && l0 == 0)
                        stamp[10] = clock64() + (long long)(tot * 0.0);
                    if (TIMING && rec_all && warp == NW - NOWN && l0 == 0)
                        gstamp[1] = (long long)globaltimer_ns() + (long long)(tot * 0.0);
                    if (Gx > 1) {
                        // cluster totals -> tagged words [par][cluster][t] (summed in the pass below)
                        if (u == 0 && live) ll_store(ll + ((size_t)gx * q1 + t) * lp, tot, tag);
                        continue;
                    }
                    if (live && u == 0) {
                        const double* rec4 = bsr + 4 * i;  // (b, sq, 1/sq, 0) of owned worker i
                        const double d = __dsub_rn(rec4[0], tot);
                        const double nume = unit_alpha ? d : __dmul_rn(alp[t], d);  // 1 * d == d exactly
                        sout[i] = div_rn_fast(nume, rec4[1], rec4[2]);
                        if (TIMING && rec && warp == NW - NOWN && l0 == 0)
                            stamp[11] = clock64() + (long long)(sout[i] * 0.0);
                        if (TIMING && rec_all && warp == NW - NOWN && l0 == 0)
                            gstamp[2] = (long long)globaltimer_ns() + (long long)(sout[i] * 0.0);
                    }
                }
                if (Gx > 1) {
                    // the clusters' totals of each item, LPI lanes per item (lane h polls cluster h's
                    // word), added in cluster order; then the scale
                    const int LPI = Gx <= 8 ? 8 : 16, ipr = 32 / LPI, h = lane & (LPI - 1);
                    for (int j0 = 0; j0 < 2 * my_pairs; j0 += ipr) {
                        const int li = j0 + lane / LPI;
                        const int i = 2 * (ow + NOWN * (li >> 1)) + (li & 1);
                        const bool live = li < 2 * my_pairs && i < n_own;
                        const int t = my_lo + i;
                        const double v = ll_poll_lane(ll + ((size_t)h * q1 + t) * lp, live && h < Gx, tag,
                                                      &a.status->aborted);
                        const double tot = ordered_group_sum(v, lane & ~(LPI - 1), Gx);
                        if (live && h == 0) {
                            const double* rec4 = bsr + 4 * i;  // (b, sq, 1/sq, 0) of owned worker i
                            const double d = __dsub_rn(rec4[0], tot);
                            const double nume = unit_alpha ? d : __dmul_rn(alp[t], d);  // 1 * d == d exactly
                            sout[i] = div_rn_fast(nume, rec4[1], rec4[2]);
                            if (TIMING && rec && warp == NW - NOWN && j0 == 0)
                                stamp[11] = clock64() + (long long)(sout[i] * 0.0);
                            if (TIMING && rec_all && warp == NW - NOWN && j0 == 0)
                                gstamp[2] = (long long)globaltimer_ns() + (long long)(sout[i] * 0.0);
                        }
                    }
                }
                __syncwarp();
                if (TIMING && rec) stamp[8] = clock64();
                // broadcast: this warp's worker pairs as 16-byte pushes to every CTA of the cluster
                for (int k = lane; k < my_pairs * Pc; k += 32) {
                    const int pi = ow + NOWN * (k >> pcs), peer = k & (Pc - 1);
                    const int i = 2 * pi, t = my_lo + i;
                    const unsigned dst =
                        mapa_u32(scal_u, (unsigned)peer) + (unsigned)((par * q4 + t) * (int)sizeof(double));
                    const unsigned bar = mapa_u32(sbar_u + 8u * par, (unsigned)peer);
                    if (i + 1 < n_own)
                        st_async_v2_f64(dst, sout[i], sout[i + 1], bar);
                    else
                        st_async_f64(dst, sout[i], bar);
                }
                if (TIMING && rec) stamp[9] = clock64();
            }
            if (warp == OW && want_check && cr == eown) {
                mbar_wait(&ebin[par], bpar);
                if (TIMING && rec) stamp[10] = clock64();
                double tot = owner_total(ein + par * Pc, 1, lane < 2);
                if (Gx > 1) {  // lane h polls cluster h's error total; added in cluster order
                    if (lane == 0) ll_store(ll + ((size_t)gx * q1 + q) * lp, tot, tag);
                    const double v = ll_poll_lane(ll + ((size_t)lane * q1 + q) * lp, lane < Gx, tag, &a.status->aborted);
                    tot = ordered_group_sum(v, 0, Gx);
                }
                tot = __shfl_sync(0xffffffffu, tot, 0);
                if (lane < Pc)
                    st_async_f64(mapa_u32(errs_u, (unsigned)lane) + (unsigned)(par * (int)sizeof(double)), tot,
                                 mapa_u32(ebar_u + 8u * par, (unsigned)lane));
            }
        }
        if (last) {  // final stop-rule evaluation only
            mbar_wait(&ebar[par], bpar);
            const double err = errs[par];
            ++checks;
            err_last = err;
            if (err < a.eps) conv = 1;
            break;
        }
        // ---- 4. scales arrive ------------------------------------------------------------
        mbar_wait(&sbar[par], bpar);
        if (TIMING && rec) stamp[3] = clock64();
        if (TIMING && rec_all && warp == 0) gstamp[3] = (long long)globaltimer_ns();
        const double* sc = scal + par * q4;
        if (TIMING && rec) stamp[4] = clock64();
        // ---- 5. average over this warp's workers -----------------------------------------
        double2 acc[EPL];
#pragma unroll
        for (int e = 0; e < EPL; ++e) acc[e] = make_double2(0.0, 0.0);
        for (int rb = wb; SR ? rb == wb && wb < we : rb < we; rb += 8) {
            if (SR ? rok == (1 << NR) - 1 : rb + grp * NR + NR <= we) {
                // all NR rows exist: the loads of RB rows (and their scales) ahead of the arithmetic,
                // the sums in the same row order as below
#pragma unroll
                for (int r0 = 0; r0 < NR; r0 += RB) {
                    double2 rv[RB][EPL];
                    double sv[RB];
#pragma unroll
                    for (int r = 0; r < RB; ++r) {
                        sv[r] = sc[rb + grp * NR + r0 + r];
#pragma unroll
                        for (int e = 0; e < EPL; ++e)
                            rv[r][e] = vld[e] ? *reinterpret_cast<const double2*>(rows + roff[r0 + r] +
                                                                                   (rb - wb) * cwb + 2 * LG * e)
                                              : make_double2(0.0, 0.0);
                    }
#pragma unroll
                    for (int r = 0; r < RB; ++r) {
                        const bool first = (r0 + r == 0) && (rb == wb);
#pragma unroll
                        for (int e = 0; e < EPL; ++e)
                            if (vld[e]) {
                                const double v0 = __dadd_rn(xv[e].x, __dmul_rn(sv[r], rv[r][e].x));
                                const double v1 = __dadd_rn(xv[e].y, __dmul_rn(sv[r], rv[r][e].y));
                                acc[e].x = first ? v0 : __dadd_rn(acc[e].x, v0);
                                acc[e].y = first ? v1 : __dadd_rn(acc[e].y, v1);
                            }
                    }
                }
                continue;
            }
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int t = rb + grp * NR + r;
                if (SR ? ((rok >> r) & 1) != 0 : t < we) {
                    const double s = sc[t];
                    const double* row = rows + roff[r] + (rb - wb) * cwb;
                    const bool first = (r == 0) && (rb == wb);
#pragma unroll
                    for (int e = 0; e < EPL; ++e)
                        if (vld[e]) {
                            const double2 rv = *reinterpret_cast<const double2*>(row + 2 * LG * e);
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
        if (TIMING && rec) stamp[5] = clock64();
        named_sync(CBAR, NW * 32);
        // ---- combine: x_{k+1} = (fixed tree over the warps' sums) / q ----------------------
        // narrow slices: every warp forms its own lanes' columns (no second barrier);
        // wide slices: warp w forms its share of the columns into xs, one more barrier,
        // every lane reads its columns back (8x less shared-memory traffic)
        auto combine_pair = [&](int j) -> double2 {
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
            return w[0];
        };
        auto scale_q = [&](double2 v) -> double2 {
            return qpow2 ? make_double2(__dmul_rn(v.x, invq), __dmul_rn(v.y, invq))
                         : make_double2(div_rn_fast(v.x, qd, invq), div_rn_fast(v.y, qd, invq));
        };
        double2 xn[EPL];
        if constexpr (!xr) {  // cross-rank mode forms xn after the exchange (fewer live registers there)
#pragma unroll
            for (int e = 0; e < EPL; ++e) xn[e] = xv[e];
        }
        const bool ck = ckpt_on && (((a.k0 + kk + 1) % a.ckpt_every) == 0) &&
                        (((a.k0 + kk + 1) / a.ckpt_every) <= a.ckpt_cap);
        const int64_t ck_slot = ck ? (a.k0 + kk + 1) / a.ckpt_every - 1 : 0;
        if (split) {
            const int np = wdt >> 1;
            for (int pp = warp * ppw + lane; pp < (warp + 1) * ppw && pp < np; pp += 32) {
                const int j = 2 * pp;
                const double2 v = combine_pair(j);
                if (wg && G > 1) {
                    // this cluster's column sums -> tagged words [par][cluster][column] (summed below)
                    unsigned long long* wl =
                        reinterpret_cast<unsigned long long*>(a.part) + (size_t)par * G * ld * 2;
                    const unsigned tag = (unsigned)kk + 1u;
                    ll_store(wl + ((size_t)gid * ld + c0 + j) * 2, v.x, tag);
                    ll_store(wl + ((size_t)gid * ld + c0 + j + 1) * 2, v.y, tag);
                    continue;
                }
                if (xr) {
                    // this GPU's column sums -> every rank's buffer, slot [par][this rank][column]
                    // (NVLink peer stores; summed below in rank order, identical on every rank)
                    // slot parity by the global iteration: consecutive launches keep alternating, so a
                    // rank one iteration ahead never overwrites a slot another rank still polls
                    const unsigned tag = a.xr_tag0 + (unsigned)kk;
                    const int xpar = (int)((a.k0 + kk) & 1);
                    const size_t off = ((size_t)(xpar * a.xr_ranks + a.xr_rank) * ld + c0 + j) * 2;
                    for (int r = 0; r < a.xr_ranks; ++r) {
                        unsigned long long* pb = a.xr_peers[r];
                        ll_store_sys(pb + off, v.x, tag);
                        ll_store_sys(pb + off + 2, v.y, tag);
                    }
                    continue;
                }
                if (a.partial) {  // row-sharded step: un-normalised local sum
                    __stcg(a.partial + c0 + j, v.x);
                    __stcg(a.partial + c0 + j + 1, v.y);
                    continue;
                }
                const double2 x2 = scale_q(v);
                *reinterpret_cast<double2*>(xs + j) = x2;
                if (ck) {
                    if (c0 + j < a.n) a.ckpt[ck_slot * a.n + c0 + j] = x2.x;
                    if (c0 + j + 1 < a.n) a.ckpt[ck_slot * a.n + c0 + j + 1] = x2.y;
                }
            }
            if (wg && G > 1 && tid < wdt) {
                // worker groups: thread j adds the G clusters' sums of column c0 + j in cluster order
                // (every cluster forms the same x bit for bit)
                const unsigned long long* wl =
                    reinterpret_cast<const unsigned long long*>(a.part) + (size_t)par * G * ld * 2;
                const double tot = ll_sum_inl<RKA_MAXG>(wl + (size_t)(c0 + tid) * 2, 2 * ld, G, (unsigned)kk + 1u,
                                                        &a.status->aborted);
                const double xj = qpow2 ? __dmul_rn(tot, invq) : div_rn_fast(tot, qd, invq);
                xs[tid] = xj;
                if (ck && gid == 0 && c0 + tid < a.n) a.ckpt[ck_slot * a.n + c0 + tid] = xj;
            }
            if (xr && tid < wdt) {
                // thread j adds the ranks' sums of column c0 + j in rank order
                const unsigned long long* own =
                    a.xr_peers[a.xr_rank] + (size_t)((a.k0 + kk) & 1) * a.xr_ranks * ld * 2;
                // ranks polled four at a time (register budget), summed in rank order
                const unsigned xtag = a.xr_tag0 + (unsigned)kk;
                const unsigned long long* pw = own + (size_t)(c0 + tid) * 2;
                double tot = ll_sum_inl<4, true>(pw, 2 * ld, a.xr_ranks < 4 ? a.xr_ranks : 4, xtag, &a.status->aborted);
                if (a.xr_ranks > 4)
                    tot = __dadd_rn(tot, ll_sum_inl<4, true>(pw + (size_t)8 * ld, 2 * ld, a.xr_ranks - 4, xtag,
                                                              &a.status->aborted));
                xs[tid] = qpow2 ? __dmul_rn(tot, invq) : div_rn_fast(tot, qd, invq);
            }
            named_sync(CBAR, NW * 32);
            if constexpr (xr) {
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    xn[e] = vld[e] ? *reinterpret_cast<const double2*>(xs + 2 * (gl + LG * e)) : xv[e];
            } else if (!a.partial) {
#pragma unroll
                for (int e = 0; e < EPL; ++e)
                    if (vld[e]) xn[e] = *reinterpret_cast<const double2*>(xs + 2 * (gl + LG * e));
            }
        } else {
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                if (!vld[e]) continue;
                const int j = 2 * (gl + LG * e);
                const double2 v = combine_pair(j);
                if (a.partial) {
                    if (warp == 0 && grp == 0) {
                        __stcg(a.partial + c0 + j, v.x);
                        __stcg(a.partial + c0 + j + 1, v.y);
                    }
                    continue;
                }
                xn[e] = scale_q(v);
                if (ck && warp == 0 && grp == 0) {
                    if (c0 + j < a.n) a.ckpt[ck_slot * a.n + c0 + j] = xn[e].x;
                    if (c0 + j + 1 < a.n) a.ckpt[ck_slot * a.n + c0 + j + 1] = xn[e].y;
                }
            }
        }
        // ---- stop rule on x_k (its error total arrived while x_{k+1} was formed) ----------
        if (want_check) {
            if (TIMING && rec) stamp[11] = clock64();
            mbar_wait(&ebar[par], bpar);
            if (TIMING && rec) stamp[12] = clock64();
            const double err = errs[par];
            ++checks;
            err_last = err;
            if (err < a.eps) {
                conv = 1;
                break;  // x_k stands; x_{k+1} is discarded
            }
        }
#pragma unroll
        for (int e = 0; e < EPL; ++e) xv[e] = xn[e];
        if (TIMING && rec) stamp[6] = clock64();
        if (++st == D) {
            st = 0;
            fph ^= 1u;
        }
        done = kk + 1;
    }
    if (tid == 0) *halt = 1;
    if (!a.partial && warp == 0 && grp == 0 && (!wg || gid == 0)) {
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
        if (conv && a.halt != nullptr) *a.halt = (int)(a.k0 + done + 1);  // later launches become no-ops
    }
}

template __global__ void rka_kernel<8, 1, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 1, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<8, 2, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<16, 1, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 1, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 2, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 3, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, true, false, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, true, true, 0>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, false, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, true, 1>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, false, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);
template __global__ void rka_kernel<32, 4, false, true, 2>(const __grid_constant__ SolveArgs,
    const __grid_constant__ CUtensorMap, const __grid_constant__ CUtensorMap);

}  // namespace kz
