// kz_chain.cu -- worker-per-CTA persistent kernel for RK and RKAB.
//
// Reference semantics (paths relative to /root/reference/pkg/src/kaczbench):
//   kaczmarz_step      solvers.py:107-117   s = alpha*(b_i - <a_i,v>)/sq_i ; v += s*a_i
//   rkab_worker_block  solvers.py:140-145   bs chained projections on the private v
//   RKAB advance       solvers.py:361-367   v_t = x ; chain ; x = (sum_t v_t) / q, t ascending
//   solve_rk           solvers.py:294-310   (q = 1, bs = 1)
//   _drive stop rule   solvers.py:229-243   ||x - x_ref||^2 < eps checked before every iteration
//
// Layout: CTA w runs worker w.  Its estimate v lives in registers: thread
// `tid` owns the 16-byte column pairs col = 2*(p*T + tid), p < EP.  Rows are
// streamed HBM -> shared memory by per-thread cp.async (each thread copies
// exactly the pairs it later reads) through a ring of `stages` rows; row
// indices are x-independent and come from a shared-memory window, so the
// ring runs ahead of the arithmetic.
//
// Row blocks (the latency lever).  A chain of projections is a dependent
// sequence -- dot, CTA-wide reduction, scale, axpy -- so one reduction per
// row leaves the memory system idle.  The kernel instead takes R consecutive
// rows a_1..a_R of a worker's chain and reduces, in ONE CTA reduction,
//     d_r = <a_r, v>   and   G_rl = <a_r, a_l> (l < r),
// then resolves the chain exactly as the reference orders it:
//     <a_r, v_{r-1}> = d_r + sum_{l<r} s_l G_rl,  s_r = alpha (b_r - <a_r, v_{r-1}>) / sq_r,
// and applies v += s_r a_r row by row: with the reference's rounding
// (__dmul_rn then __dadd_rn) when R = 1, as one FMA per element in blocks of
// R > 1 rows, whose scales are already rebracketed.  The dot products are
// rebracketed (tolerance parity, like any change of summation order); the
// averaging is the reference's.  1/sq_r replaces the division.
//
// The stop rule (RK and RKAB with q = 1 check between rows) rides along:
// the same reduction carries ||v - x_ref||^2 and <a_r, x_ref>, and
//     ||v_r - x_ref||^2 = ||v_{r-1} - x_ref||^2 + 2 s_r (<a_r, v_{r-1}> - <a_r, x_ref>) + s_r^2 sq_r
// gives the error before each row of the block.  A derived value that comes
// within 1e-6 (relative) of eps truncates the block, so every decision near
// the threshold is taken on a directly reduced ||x - x_ref||^2.
//
// RKAB with q > 1 averages the worker estimates in worker order behind two
// grid barriers (cooperative launch) and checks the averaged x directly.
//
// The threaded engine's combine (parallel.py:175-304, engine="threads") runs on
// the same machinery: its workers add increments to the shared x under a lock in
// arrival order; here the order is the worker order, one valid schedule.
//   RKA  (KZ_COMBINE_RKA_DELTA, bs = 1): s_t = alpha (b - <a, x>) / (q sq) (by the
//        reciprocal of fl(q sq), like every scale here); the worker publishes fl(s_t a_t) and
//        x_j <- fl(x_j + inc_tj), t ascending            (parallel.py:214-226)
//   RKAB (KZ_COMBINE_RKAB_DELTA): the worker publishes v_t; inc_tj = fl(fl(v_tj - x_j) / q)
//        against the pre-combine x, x_j <- fl(x_j + inc_tj)  (parallel.py:286-298)
#include "kz_kernels.cuh"

namespace kz {

namespace {

template <int R>
struct Blk {
    static constexpr int NG = R * (R - 1) / 2;  // Gram entries l < r
    static constexpr int NVN = R + NG;          // without stop-rule terms
    static constexpr int NVC = NVN + R + 1;     // + <a_r, x_ref>, ||v - x_ref||^2
};

__host__ __device__ constexpr int gidx(int r, int l) { return r * (r - 1) / 2 + l; }

struct ChainSmem {
    double* ring;   // stages x ld
    double2* bsq;   // stages + R slots of (b_i, sq_i)
    int32_t* win;   // IDX_WINDOW row indices
    double* scr;    // NVC x T reduction scratch (value-major)
    double* tot;    // NVC totals
};

// CTA-wide sums of NV per-thread values; every thread receives every total,
// bit-identical.  (1) Inside each warp a transposed shuffle reduction per 32
// values: they are halved across lanes at xor offsets 16, 8, 4, 2, 1 -- a lane
// keeps one half and adds its partner's copy -- so after 31 shuffles lane l
// holds the warp sum of value l (no shared-memory traffic, 5 dependent levels);
// more than 32 values take a second pass.  (2) Those land in scr[warp][NP]; one
// barrier; thread v < NV adds the nw warp sums in a fixed tree into tot[v]; one
// barrier; everyone reads tot.
template <int NV32>
__device__ __forceinline__ void warp_transpose32(const double* v, double* dst, int lane) {
    double w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = i < NV32 ? v[i] : 0.0;
#pragma unroll
    for (int h = 16, o = 16; o >= 1; h >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? w[i] : w[i + h];
            const double keep = up ? w[i + h] : w[i];
            w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    if (lane < NV32) dst[lane] = w[0];
}

// The same for at most 16 values in half the shuffles: the values are halved across lanes at xor
// offsets 16, 8, 4, 2 (8 + 4 + 2 + 1 shuffles), which leaves lane l with value (l >> 1) summed over
// the 16 lanes of its parity, and one butterfly step at xor 1 completes the warp sum (both lanes of
// a pair hold the same bits; the even one stores).
template <int NV16>
__device__ __forceinline__ void warp_transpose16(const double* v, double* dst, int lane) {
    double w[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) w[i] = i < NV16 ? v[i] : 0.0;
#pragma unroll
    for (int h = 8, o = 16; o >= 2; h >>= 1, o >>= 1) {
        const bool up = (lane & o) != 0;
#pragma unroll
        for (int i = 0; i < h; ++i) {
            const double send = up ? w[i] : w[i + h];
            const double keep = up ? w[i + h] : w[i];
            w[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
        }
    }
    const double tot = w[0] + __shfl_xor_sync(0xffffffffu, w[0], 1);
    if ((lane & 1) == 0 && (lane >> 1) < NV16) dst[lane >> 1] = tot;
}

template <int NV, typename OnTotal>
__device__ __forceinline__ void cta_reduce(double (&v)[NV], double* scr, double* tot, int tid, int T, int nw,
                                           OnTotal on_total) {
    constexpr int NP = NV <= 32 ? 32 : 64;
    static_assert(NV <= 64, "cta_reduce: at most 64 values");
    const int lane = tid & 31, warp = tid >> 5;
    if (NV <= 4) {  // few values: a butterfly per value (5 NV shuffles, no padding registers)
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            double x = v[i];
#pragma unroll
            for (int o = 16; o >= 1; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
            if (lane == i) scr[warp * NP + i] = x;
        }
    } else if (NV <= 12) {  // (the stop-rule blocks' 15 values measured faster on the 32-wide form)
        warp_transpose16<NV>(v, scr + warp * NP, lane);
    } else if (NV <= 32) {
        warp_transpose32<NV>(v, scr + warp * NP, lane);
    } else {  // two passes of 32: the padded 64-value transpose would hold 128 registers at once
        warp_transpose32<32>(v, scr + warp * NP, lane);
        warp_transpose32<NV - 32>(v + 32, scr + warp * NP + 32, lane);
    }
    named_sync(1, T);  // the compute threads (the producer warp is not in the reduction)
    for (int u = tid; u < NV; u += T) {
        double a[16];
#pragma unroll
        for (int k = 0; k < 16; ++k) a[k] = k < nw ? scr[k * NP + u] : 0.0;
#pragma unroll
        for (int hh = 1; hh < 16; hh <<= 1)
#pragma unroll
            for (int k = 0; k + hh < 16; k += 2 * hh) a[k] = __dadd_rn(a[k], a[k + hh]);
        tot[u] = a[0];
        on_total(u, a[0]);  // the cluster join's push leaves from the thread that formed the total
    }
    named_sync(1, T);
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = tot[i];
}

struct TrueT {
    static constexpr bool value = true;
};
struct FalseT {
    static constexpr bool value = false;
};

}  // namespace

template <int EP>
struct ChainMaxThreads {  // compute threads; the CTA adds one producer warp
    // the plan keeps CTAs <= 128 threads below EP 16.  Registers go to warps in groups of four,
    // so the 11 warps of an EP = 16 CTA get 168 registers per thread (an EP = 24 variant on 7 + 1
    // warps with 255 registers spilled more: 2 x 24 pairs of v and row leave too little)
    static constexpr int value = EP <= 8 ? 128 : 320;
};

// grid barrier over the compute threads of every CTA (the producer warps keep streaming)
__device__ __forceinline__ void grid_barrier_c(unsigned* counter, unsigned target, int T) {
    named_sync(1, T);
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(counter) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(counter) : "memory");
        } while (v < target);
    }
    named_sync(1, T);
}

template <int EP, int R, int C, bool DELTA, bool WIDE>
__global__ void __launch_bounds__(ChainMaxThreads<EP>::value + 32, 1) chain_kernel(SolveArgs a) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    if (a.halt != nullptr && *a.halt != 0) return;  // stopped earlier in the stream: uniform over the grid
    // compute threads T = blockDim - 32; the last warp is the producer (row ring issue)
    const int T = (int)blockDim.x - 32, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nw = T >> 5;
    const int D = a.stages;
    const int64_t ld = a.ld, q = a.q, bs = a.bs;
    // C >= 2: a worker is a thread-block cluster of C CTAs (a pair for RKAB's long rows, up to
    // 8 for one long RK chain); CTA h owns columns [h*ld/C, (h+1)*ld/C) and the C slices of
    // every reduction are joined through distributed shared memory (st.async + mbarrier).
    const int h = (C >= 2) ? (int)cluster_rank() : 0;
    const int ldc = (int)(ld / C);  // this CTA's columns [cb, cb + ldc): 32-bit offsets within the slice
    const int64_t cb = (int64_t)h * ldc;
    // ring row pitch: for EP < 16 every thread's EP pairs (2 EP T columns >= ldc), the tail past ldc
    // zero, so the row loops read and update without a bounds test (v stays 0 past ldc: s * 0):
    // c2 166 -> 153 us per outer iteration, c4-shape RKAB 748 -> 700.  EP = 16 keeps the exact
    // pitch: its tail (2.4 % at c3) costs more shared-memory traffic than the tests do.
    constexpr bool PADDED = EP < 16;
    const int ldr = PADDED ? 2 * EP * T : ldc;
    ChainSmem sm;
    unsigned long long* xbar = reinterpret_cast<unsigned long long*>(smem_raw);  // 2 exchange mbarriers
    unsigned long long* full = xbar + 2;                                         // 16 row-stage mbarriers
    unsigned long long* empty = full + 16;                                       // 16 stage releases
    volatile int* halt = reinterpret_cast<volatile int*>(smem_raw + 272);        // compute done
    double* xbuf = reinterpret_cast<double*>(smem_raw + 288);                     // 2 x C x NVC peer totals
    sm.ring = xbuf + 2 * C * Blk<R>::NVC + 2;
    sm.bsq = reinterpret_cast<double2*>(sm.ring + (size_t)D * ldr);
    sm.win = reinterpret_cast<int32_t*>(sm.bsq + D);
    sm.scr = reinterpret_cast<double*>(sm.win + IDX_WINDOW);
    sm.tot = sm.scr + (size_t)Blk<R>::NVC * T;
    if (tid == 0) {
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        for (int k = 0; k < D; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&empty[k], EP < 16 ? 1 : nw);  // EP = 16: one release per compute warp
        }
        *halt = 0;
        fence_mbarrier_init_cluster();
    }
    for (int k = 0; k < D; ++k)  // the ring rows' zero tails (TMA never writes them)
        for (int j = ldc + tid; j < ldr; j += blockDim.x) sm.ring[(size_t)k * ldr + j] = 0.0;
    __syncthreads();
    if (C >= 2) cluster_sync_all();
    int nex = 0;  // cluster exchanges done

    const int64_t w = blockIdx.x / C;  // worker id
    const int32_t* idx = a.idx + w * a.idx_stride;
    const double alpha = a.alphas[w];
    const int total = (int)(a.count * bs);  // draws of this worker in the launch (< 2^31, kz_solve checks)
    const double2* bs2 = reinterpret_cast<const double2*>(a.bs2);
    const unsigned row_bytes = (unsigned)(ldc * sizeof(double));

    if (warp == nw) {
        // ================= producer warp: the row ring =================
        // Row j goes into stage j mod D once row j - D has been released by the compute
        // threads; its slice by one bulk copy (TMA engine), its (b, sq) pair by a 16-byte
        // cp.async on the same mbarrier.  Indices are read 32 at a time, one per lane.
        // Rows go out up to four at a time on deep rings, one per lane: the per-row TMA and
        // mbarrier issue costs overlap; the compute threads release stages in row order, so the
        // release of a group's last predecessor covers the whole group.
        constexpr int GI = 4;
        int64_t j = 0;
        for (int64_t j0 = 0; j0 < total && !*halt; j0 += 32) {
            const int32_t my = (j0 + lane < total) ? idx[j0 + lane] : 0;
            const int cnt = (int)(total - j0 < 32 ? total - j0 : 32);
            bool stop = false;
            // groups only on deep rings: a group waits for its last row's stage, which would hold
            // back its first rows on a shallow ring (c3: two 80 KB stages)
            const int gmax = D >= 4 * GI ? GI : 1;
            for (int u0 = 0; u0 < cnt; u0 += gmax) {
                const int g = cnt - u0 < gmax ? cnt - u0 : gmax;
                const int64_t jl = j0 + u0 + g - 1;  // the group's last row
                if (jl >= D) {
                    const unsigned eph = (unsigned)(((jl / D) - 1) & 1);
                    bool ok = false;
                    while (!(ok = mbar_try_wait(&empty[jl % D], eph)))
                        if (*halt) break;
                    if (!ok) {
                        stop = true;
                        break;
                    }
                }
                const int64_t i = __shfl_sync(0xffffffffu, my, (u0 + lane) & 31);
                if (lane < g) {
                    const int st = (int)((j0 + u0 + lane) % D);
                    cp_async16(sm.bsq + st, bs2 + 2 * i);
                    cp_async_mbar_arrive(&full[st]);
                    mbar_arrive_expect_tx(&full[st], row_bytes);
                    bulk_g2s(sm.ring + (size_t)st * ldr, a.A + i * ld + cb, row_bytes, &full[st]);
                }
                __syncwarp();
                j = jl + 1;  // rows issued
            }
            if (stop || *halt) break;
        }
        // every issued copy must land before the CTA exits
        if (lane == 0)
            for (int k = 0; k < D && k < j; ++k) {
                const int64_t last = k + ((j - 1 - k) / D) * D;  // the last row issued into stage k
                mbar_wait(&full[k], (unsigned)((last / D) & 1));
            }
        __syncwarp();
        if (C >= 2) cluster_sync_all();
        return;
    }

    double v[2 * EP];
#pragma unroll
    for (int p = 0; p < EP; ++p) {
        const int lc = 2 * (p * T + tid);
        double2 xv = make_double2(0.0, 0.0);
        if (lc < ldc) xv = __ldcg(reinterpret_cast<const double2*>(a.x + cb + lc));
        v[2 * p] = xv.x;
        v[2 * p + 1] = xv.y;
    }
    named_sync(1, T);

    // direct ||v - x_ref||^2 over the CTA
    // join the C slices of a reduction: every CTA sends its totals to every peer (slot
    // [parity][sender][value]) and adds the C totals in CTA order, so all hold the same bits
    // (for a pair the order is immaterial: IEEE addition is commutative)
    // total u of the current reduction -> slot [parity][this CTA][u] of every peer, by the thread
    // that formed it (before the reduction's second barrier: the peers' waits end that much sooner)
    auto push_total = [&](int u, double val) {
        if (C < 2) return;
        const int xp = nex & 1;
        const int u_o = opaque_i32(u);  // slot arithmetic formed here, not hoisted out of the row loop
#pragma unroll
        for (int pk = 0; pk < C - 1; ++pk) {
            const unsigned peer = (unsigned)(pk < h ? pk : pk + 1);
            st_async_f64(mapa_u32(smem_u32(xbuf + (xp * C + h) * Blk<R>::NVC + u_o), peer), val,
                         mapa_u32(smem_u32(&xbar[xp]), peer));
        }
    };
    auto pair_join = [&](double* vals, int nv) {
        if (C < 2) return;
        const int xp = nex & 1;
        const unsigned ph = (unsigned)((nex >> 1) & 1);
        ++nex;
        if (tid == 0) mbar_arrive_expect_tx(&xbar[xp], (unsigned)((C - 1) * nv * sizeof(double)));
        // (the totals were pushed to the peers by push_total, from inside the reduction)
        // the peers' totals arrive by st.async into THIS CTA's shared memory and complete xbar's
        // bytes; a CTA-scope wait sees them (as in the rka kernel's exchanges) -- the cluster-scope
        // acquire form compiles to an L1 invalidate (CCTL.IVALL) after every join, 5.6 % of the
        // c4-shape RKAB kernel's stall samples, and evicts the row indices and (b, sq) lines
        mbar_wait(&xbar[xp], ph);
        for (int i = 0; i < nv; ++i) {
            double acc = h == 0 ? vals[i] : xbuf[(xp * C) * Blk<R>::NVC + i];
            for (int c = 1; c < C; ++c) acc = __dadd_rn(acc, c == h ? vals[i] : xbuf[(xp * C + c) * Blk<R>::NVC + i]);
            vals[i] = acc;
        }
    };

    // Cold paths (stop rule, checkpoints, publishing v, reloading x) form their column offsets from
    // an opaque tid: otherwise the compiler hoists EP 64-bit addresses out of the row loop and
    // keeps them live across it, which the EP = 16 kernels pay for in spills.
    auto err_direct = [&]() {
        double e[1] = {0.0};
        const int tid_o = opaque_i32(tid);
#pragma unroll
        for (int p = 0; p < EP; ++p) {
            const int lc = 2 * (p * T + tid_o);
            const int64_t col = cb + lc;
            if (lc < ldc) {
                const double2 r = __ldg(reinterpret_cast<const double2*>(a.xref + col));
                const double d0 = v[2 * p] - r.x, d1 = v[2 * p + 1] - r.y;
                e[0] = fma(d0, d0, e[0]);
                e[0] = fma(d1, d1, e[0]);
            }
        }
        cta_reduce<1>(e, sm.scr, sm.tot, tid, T, nw, push_total);
        pair_join(e, 1);
        return e[0];
    };

    unsigned epoch = 0;
    long long done = 0;
    int conv = 0, checks = 0;
    double err_last = 0.0;
    const double qd = (double)q;
    // the threaded engine's RKA has instantiations of its own (DELTA): a runtime switch in the row
    // loop cost the other engines 7 % (c2)
    const bool rka_delta = DELTA && q > 1 && a.combine == KZ_COMBINE_RKA_DELTA;
    const bool use_stop = a.use_stop != 0;
    const bool ckpt_on = a.ckpt_every > 0;
    int nblk = 0;                 // blocks processed (phase timing)
    int d = 0;                    // rows consumed
    int next_check = 0;           // q == 1: next row preceded by a stop-rule check (multiple of bs)
    int outer_end = (int)bs;      // q == 1: row count at which the current outer iteration completes
    int64_t kdone = a.k0;         // q == 1: outer iterations completed (global index)
    int64_t next_ck = ckpt_on ? (a.k0 / a.ckpt_every + 1) * a.ckpt_every : 0;
    int c_stage = 0;              // ring stage of row d
    unsigned c_par = 0;           // mbarrier phase parity of row d's stage

    // Process rows [d, d + Rp) of the chain (Rp <= R).  CHECK: stop rule before
    // rows with (d + r) % bs == 0 (q == 1 only).  Returns rows applied.
    auto block = [&](int Rp, auto check_tag) -> int {
        constexpr bool CHECK = decltype(check_tag)::value;
        constexpr int NV = CHECK ? Blk<R>::NVC : Blk<R>::NVN;
        const bool rec = a.dbg != nullptr && blockIdx.x == 0 && tid == 0 && nblk < 64;
        if (rec) a.dbg[nblk * 8 + 0] = clock64();
        if (rec) a.dbg[nblk * 8 + 1] = clock64();
        int stg[R];
        unsigned prs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            int s0 = c_stage + r;
            unsigned pr = c_par;
            if (s0 >= D) {
                s0 -= D;
                pr ^= 1u;
            }
            stg[r] = s0;
            prs[r] = pr;
        }
        // rows d .. d + Rp - 1 landed: the R barrier probes go out together (one ~90-cycle
        // round trip instead of R); only stragglers are re-polled
        {
            unsigned okm;
            if constexpr (R == 4)
                okm = mbar_test4(&full[stg[0]], prs[0], &full[stg[1]], prs[1], &full[stg[2]], prs[2], &full[stg[3]],
                                 prs[3]);
            else if constexpr (R == 2)
                okm = mbar_test2(&full[stg[0]], prs[0], &full[stg[1]], prs[1]);
            else
                okm = mbar_test(&full[stg[0]], prs[0]) ? 1u : 0u;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r < Rp && !((okm >> r) & 1u)) mbar_wait(&full[stg[r]], prs[r]);
        }
        if (rec) a.dbg[nblk * 8 + 2] = clock64();
        // rows -> registers (kept for the update), (b, sq) -> lane r.  EP = 16 (168 registers per
        // thread at 352 threads) cannot hold 16 pairs of v and 16 of the row across the reduction
        // without spilling: its update re-reads the row from the ring (the stage is released after
        // the update), a second pass over shared memory instead of local-memory traffic
        constexpr bool KEEP_ROW = EP < 16;
        constexpr int EPK = KEEP_ROW ? EP : 1;
        double2 rr[R][EPK];
        if constexpr (KEEP_ROW) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int p = 0; p < EP; ++p) {
                    const int lc = 2 * (p * T + tid);
                    rr[r][p < EPK ? p : 0] =
                        (r < Rp && (PADDED || lc < ldc)) ? *reinterpret_cast<const double2*>(sm.ring + (size_t)stg[r] * ldr + lc)
                                             : make_double2(0.0, 0.0);
                }
        }
        auto row = [&](int r, int p) -> double2 {  // the dot's read
            if constexpr (KEEP_ROW) return rr[r][p < EPK ? p : 0];
            const int lc = 2 * (p * T + tid);
            return r < Rp ? *reinterpret_cast<const double2*>(sm.ring + (size_t)stg[r] * ldr + lc)
                          : make_double2(0.0, 0.0);
        };
        auto row_again = [&](int r, int p) -> double2 {  // the update's read
            if constexpr (KEEP_ROW) return rr[r][p < EPK ? p : 0];
            const int lc = 2 * (p * T + tid);
            return lds_reread_f64x2(sm.ring + (size_t)stg[r] * ldr + lc);
        };
        double2 bq = make_double2(0.0, 1.0);
        if constexpr (R == 1) {
            // one row per reduction: every lane reads the (b, sq) pair and divides for itself (in the
            // shadow of the dot's shared-memory reads); no shuffle between the join and the scale
            if (Rp > 0) bq = sm.bsq[c_stage];
        } else if (lane < Rp) {
            int sl = c_stage + lane;
            if (sl >= D) sl -= D;
            bq = sm.bsq[sl];
        }
        // (b_r, sq_r) sit in lane r; 1/sq_r formed there now (off the critical path: the division
        // overlaps the partial dots and the reduction)
        // (the threaded engine's RKA divides by q sq, parallel.py:221: its reciprocal instead)
        const double inv_l = 1.0 / (rka_delta ? __dmul_rn(qd, bq.y) : bq.y);
        double vals[NV];
#pragma unroll
        for (int i = 0; i < NV; ++i) vals[i] = 0.0;
#pragma unroll
        for (int p = 0; p < EP; ++p) {
            const int lc = 2 * (p * T + tid);
            const int64_t col = cb + lc;
            if ((PADDED && !CHECK) || lc < ldc) {  // the stop-rule terms read x_ref: bounded
                const double vx = v[2 * p], vy = v[2 * p + 1];
#pragma unroll
                double2 ar[R];
#pragma unroll
                for (int r = 0; r < R; ++r) ar[r] = row(r, p);
#pragma unroll
                for (int r = 0; r < R; ++r) vals[r] = fma(ar[r].y, vy, fma(ar[r].x, vx, vals[r]));
#pragma unroll
                for (int r = 1; r < R; ++r)
#pragma unroll
                    for (int l = 0; l < r; ++l)
                        vals[R + gidx(r, l)] = fma(ar[r].y, ar[l].y, fma(ar[r].x, ar[l].x, vals[R + gidx(r, l)]));
                if (CHECK) {
                    const double2 xr = __ldg(reinterpret_cast<const double2*>(a.xref + col));
#pragma unroll
                    for (int r = 0; r < R; ++r)
                        vals[Blk<R>::NVN + r] = fma(ar[r].y, xr.y, fma(ar[r].x, xr.x, vals[Blk<R>::NVN + r]));
                    const double d0 = vx - xr.x, d1 = vy - xr.y;
                    vals[NV - 1] = fma(d1, d1, fma(d0, d0, vals[NV - 1]));
                }
            }
        }
        if (rec) a.dbg[nblk * 8 + 3] = clock64();
        // every row's (b, sq) to all lanes before the reduction (they need no division), alpha / sq
        // after it (the division in lane r overlaps the reduction): two of the three shuffle rounds
        // leave the path between the join and the scales
        double brs[R], sqrs[R], invrs[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            brs[r] = R == 1 ? bq.x : __shfl_sync(0xffffffffu, bq.x, r);
            sqrs[r] = R == 1 ? bq.y : __shfl_sync(0xffffffffu, bq.y, r);
        }
        cta_reduce<NV>(vals, sm.scr, sm.tot, tid, T, nw, push_total);
        pair_join(vals, NV);
        if (rec) a.dbg[nblk * 8 + 4] = clock64();
#pragma unroll
        for (int r = 0; r < R; ++r) invrs[r] = R == 1 ? inv_l : __shfl_sync(0xffffffffu, inv_l, r);
        double s[R];
        int Reff = Rp;
        double e = CHECK ? vals[NV - 1] : 0.0;
        // s_r = alpha (b_r - <a_r, v> - sum_{l<r} s_l <a_r, a_l>) / sq_r as c_r - sum_l s_l g_rl with
        // c_r = (b_r - <a_r, v>) (alpha / sq_r) and g_rl = <a_r, a_l> (alpha / sq_r) formed up front,
        // independent of the scales: the sequential chain s_0 -> s_1 -> ... is one FMA per row
        // instead of FMA, subtraction and two multiplications
        double cs[R], gs[Blk<R>::NG > 0 ? Blk<R>::NG : 1];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            const double ai = __dmul_rn(alpha, invrs[r]);
            cs[r] = __dmul_rn(__dsub_rn(brs[r], vals[r]), ai);
#pragma unroll
            for (int l = 0; l < r; ++l) gs[gidx(r, l)] = __dmul_rn(vals[R + gidx(r, l)], ai);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < Reff) {
                const double sqr = sqrs[r];
                double dr = vals[r];
                if (CHECK) {  // <a_r, v_r> itself: the error update below (off the scales' chain)
#pragma unroll
                    for (int l = 0; l < r; ++l) dr = fma(s[l], vals[R + gidx(r, l)], dr);
                }
                if (CHECK && d + r == next_check) {
                    if (r == 0) {
                        ++checks;
                        err_last = e;
                        if (e < a.eps) {
                            conv = 1;
                            Reff = 0;
                        }
                    } else if (e < a.eps * (1.0 + 1e-6)) {
                        Reff = r;  // decide on a direct reduction next block
                    } else {
                        ++checks;
                        err_last = e;
                    }
                }
                if (r < Reff) {
                    if (CHECK && d + r == next_check) next_check += bs;
                    double sr = cs[r];
#pragma unroll
                    for (int l = 0; l < r; ++l) sr = fma(-s[l], gs[gidx(r, l)], sr);
                    s[r] = sr;
                    if (CHECK) e = fma(s[r] * s[r], sqr, fma(2.0 * s[r], dr - vals[Blk<R>::NVN + r], e));
                }
            }
        }
        if (rec) a.dbg[nblk * 8 + 5] = clock64();
        // apply the Reff projections in order (R = 1: the reference's multiply-then-add rounding).  The threaded RKA
        // publishes the increment itself: v restarts from 0 (0 + fl(s a) is exact; v is reloaded
        // from x after the combine), so the row loop below is the same for every engine
        if (rka_delta) {
#pragma unroll
            for (int i = 0; i < 2 * EP; ++i) v[i] = 0.0;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            if (r < Reff) {
#pragma unroll
                for (int p = 0; p < EP; ++p) {
                    const int lc = 2 * (p * T + tid);
                    if (PADDED || lc < ldc) {  // padded: the zero tail leaves v past ldc at 0
                        const double2 ap = row_again(r, p);
                        if constexpr (R > 1) {
                            // Gram-corrected blocks already round differently from the reference's
                            // row-by-row arithmetic (within the 1e-10 parity bar): their update is one
                            // FMA per element, half the FP64 instructions of the block's apply phase
                            v[2 * p] = fma(s[r], ap.x, v[2 * p]);
                            v[2 * p + 1] = fma(s[r], ap.y, v[2 * p + 1]);
                        } else {
                            v[2 * p] = __dadd_rn(v[2 * p], __dmul_rn(s[r], ap.x));
                            v[2 * p + 1] = __dadd_rn(v[2 * p + 1], __dmul_rn(s[r], ap.y));
                        }
                    }
                }
                if (q == 1 && d + r + 1 == outer_end) {  // outer iteration kdone completes here
                    outer_end += bs;
                    ++kdone;
                    if (ckpt_on && kdone == next_ck) {
                        next_ck += a.ckpt_every;
                        const int64_t slot = kdone / a.ckpt_every - 1;
                        if (slot < a.ckpt_cap) {
                            const int tid_o = opaque_i32(tid);
#pragma unroll
                            for (int p = 0; p < EP; ++p) {
                                const int lc = 2 * (p * T + tid_o);
                                const int64_t col = cb + lc;
                                if (lc >= ldc) continue;  // lanes past this CTA's slice own nothing
                                if (col < a.n) a.ckpt[slot * a.n + col] = v[2 * p];
                                if (col + 1 < a.n) a.ckpt[slot * a.n + col + 1] = v[2 * p + 1];
                            }
                        }
                    }
                }
            }
        }
        if (rec) a.dbg[nblk * 8 + 6] = clock64();
        ++nblk;
        // the applied rows' stages go back to the producer.  Rows kept in registers: every thread
        // read them before the reduction's barriers, so one thread releases -- the last compute
        // thread, not thread 0, whose warp also runs the reduction's cross-warp pass and the cluster
        // join (RK n = 2000 0.382 -> 0.370 us per row, c2 146.9 -> 144.4 and c4-shape RKAB 664 ->
        // 649 us per outer iteration).  Rows re-read from the ring by the update (EP = 16): every
        // warp releases after its own re-reads (the stage barriers count the compute warps).
        if constexpr (KEEP_ROW) {
            if (tid == T - 1)
                for (int r = 0; r < Reff; ++r) {
                    int st = c_stage + r;
                    if (st >= D) st -= D;
                    mbar_arrive(&empty[st]);
                }
        } else {
            __syncwarp();
            if (lane == 0)
                for (int r = 0; r < Reff; ++r) {
                    int st = c_stage + r;
                    if (st >= D) st -= D;
                    mbar_arrive(&empty[st]);
                }
        }
        d += Reff;
        c_stage += Reff;
        if (c_stage >= D) {
            c_stage -= D;
            c_par ^= 1u;
        }
        return Reff;
    };

    // Which drivers an instantiation carries (the plan guarantees the pairing): one chain (q = 1)
    // never runs on a pair with EP >= 8 (rows of < 1536 columns) and workers averaged (q > 1)
    // never run on 4- or 8-CTA clusters.  Compiling the unused driver out leaves the register
    // allocator one loop to fit (the EP = 16 pair kernel then keeps v and the row without spilling).
    // (WIDE: averaged workers of 4 or 8 CTAs each, RKAB on rows beyond a pair's 20480 columns)
    constexpr bool ONE_CHAIN = !(C == 2 && EP >= 8) && !WIDE;
    constexpr bool AVERAGED = C <= 2 || WIDE;
    if (ONE_CHAIN && (q == 1 || !AVERAGED)) {
        // one chain: outer iteration k = rows [k*bs, (k+1)*bs); x = v after each
        while (d < total) {
            const int Rp = (int)((total - d) < R ? (total - d) : R);
            if (use_stop)
                block(Rp, TrueT{});
            else
                block(Rp, FalseT{});
            if (conv) break;
        }
        done = d / bs;
        if (!conv && use_stop && a.final_check) {
            const double e = err_direct();
            ++checks;
            err_last = e;
            if (e < a.eps) conv = 1;
        }
    } else if (AVERAGED) {
        for (int64_t kk = 0;; ++kk) {
            const bool last = (kk == a.count);
            if (use_stop && (!last || a.final_check)) {
                const double e = err_direct();  // identical in every CTA
                ++checks;
                err_last = e;
                if (e < a.eps) {
                    conv = 1;
                    break;
                }
            }
            if (last) break;
            const int end = (int)((kk + 1) * bs);
            while (d < end) block((int)((end - d) < R ? (end - d) : R), FalseT{});
            // publish v_w, average column slices in worker order, redistribute x
            const int64_t k = a.k0 + kk;
            const bool ck = ckpt_on && ((k + 1) % a.ckpt_every) == 0 && ((k + 1) / a.ckpt_every) <= a.ckpt_cap;
            const int64_t slot = ck ? (k + 1) / a.ckpt_every - 1 : 0;
            double* vw = a.V + w * ld;
            {
                const int tid_o = opaque_i32(tid);
#pragma unroll
                for (int p = 0; p < EP; ++p) {
                    const int lc = 2 * (p * T + tid_o);
                    if (lc < ldc)
                        __stcg(reinterpret_cast<double2*>(vw + cb + lc), make_double2(v[2 * p], v[2 * p + 1]));
                }
            }
            grid_barrier_c(a.barrier, (++epoch) * gridDim.x, T);
            const int64_t G = gridDim.x;
            const int64_t cw = ((ld + G - 1) / G + 1) & ~(int64_t)1;
            const int64_t c0 = blockIdx.x * cw, c1 = (c0 + cw < ld) ? c0 + cw : ld;
            if (a.combine != KZ_COMBINE_AVERAGE) {  // threaded engine: increments in worker order
                for (int64_t col = c0 + tid; col < c1; col += T) {
                    const double xp = __ldcg(a.x + col);
                    double acc = xp;
                    for (int64_t t = 0; t < q; ++t) {
                        const double vt = __ldcg(a.V + t * ld + col);
                        acc = __dadd_rn(acc, rka_delta ? vt : __ddiv_rn(__dsub_rn(vt, xp), qd));
                    }
                    __stcg(a.x + col, acc);
                    if (ck && col < a.n) a.ckpt[slot * a.n + col] = acc;
                }
            }
            for (int64_t col = c0 + tid; a.combine == KZ_COMBINE_AVERAGE && col < c1; col += T) {
                // ((S + v_0) + v_1) + ...: a later wave continues the earlier waves' ordered sum
                double acc = a.accumulate ? __dadd_rn(__ldcg(a.partial + col), __ldcg(a.V + col)) : __ldcg(a.V + col);
                for (int64_t t = 1; t < q; ++t) acc = __dadd_rn(acc, __ldcg(a.V + t * ld + col));
                if (a.partial) {  // row-sharded step: the un-normalised local sum, x untouched
                    __stcg(a.partial + col, acc);
                    continue;
                }
                const double xn = __ddiv_rn(acc, qd);
                __stcg(a.x + col, xn);
                if (ck && col < a.n) a.ckpt[slot * a.n + col] = xn;
            }
            grid_barrier_c(a.barrier, (++epoch) * gridDim.x, T);
            const int tid_o = opaque_i32(tid);
#pragma unroll
            for (int p = 0; p < EP; ++p) {
                const int lc = 2 * (p * T + tid_o);
                if (lc < ldc) {
                    const double2 xv = __ldcg(reinterpret_cast<const double2*>(a.x + cb + lc));
                    v[2 * p] = xv.x;
                    v[2 * p + 1] = xv.y;
                }
            }
            done = kk + 1;
        }
    }
    if (tid == 0) *halt = 1;  // the producer stops issuing and drains what it issued
    if (q == 1) {
        double* dst = a.partial ? a.partial : a.x;
#pragma unroll
        for (int p = 0; p < EP; ++p) {
            const int lc = 2 * (p * T + tid);
            if (lc < ldc) __stcg(reinterpret_cast<double2*>(dst + cb + lc), make_double2(v[2 * p], v[2 * p + 1]));
        }
    }
    if (C >= 2) cluster_sync_all();  // no DSMEM traffic may target an exited CTA
    if (blockIdx.x == 0 && tid == 0) {
        a.status->iters_done = done;
        a.status->converged = conv;
        a.status->checks = checks;
        a.status->err = err_last;
    }
}

#define KZ_CHAIN(EP, R, C) template __global__ void chain_kernel<EP, R, C, false, false>(SolveArgs);
#define KZ_CHAIN_DELTA(EP, R) template __global__ void chain_kernel<EP, R, 1, true, false>(SolveArgs);
#define KZ_CHAIN_WIDE(EP, R, C) template __global__ void chain_kernel<EP, R, C, false, true>(SolveArgs);
KZ_CHAIN(1, 1, 1)
KZ_CHAIN(1, 4, 1)
KZ_CHAIN(2, 1, 1)
KZ_CHAIN(2, 4, 1)
KZ_CHAIN(4, 1, 1)
KZ_CHAIN(4, 2, 1)
KZ_CHAIN(4, 4, 1)
KZ_CHAIN(8, 1, 1)
KZ_CHAIN(8, 2, 1)
KZ_CHAIN(16, 1, 1)
KZ_CHAIN(1, 4, 2)
KZ_CHAIN(2, 4, 2)
KZ_CHAIN(4, 2, 2)
KZ_CHAIN(4, 4, 2)
KZ_CHAIN(8, 1, 2)
KZ_CHAIN(8, 2, 2)
KZ_CHAIN(16, 1, 2)
// one long RK / CK chain over a cluster of 4 or 8 CTAs (q = 1); EP 8 / 16: n up to 40960
KZ_CHAIN(1, 4, 4)
KZ_CHAIN(2, 4, 4)
KZ_CHAIN(4, 4, 4)
KZ_CHAIN(8, 1, 4)
KZ_CHAIN(8, 2, 4)
KZ_CHAIN(16, 1, 4)
KZ_CHAIN(1, 4, 8)
KZ_CHAIN(2, 4, 8)
KZ_CHAIN(8, 1, 8)
KZ_CHAIN(8, 2, 8)
KZ_CHAIN(16, 1, 8)
// the threaded engine's RKA (one CTA per worker)
KZ_CHAIN_DELTA(1, 1)
KZ_CHAIN_DELTA(1, 4)
KZ_CHAIN_DELTA(2, 1)
KZ_CHAIN_DELTA(2, 4)
KZ_CHAIN_DELTA(4, 1)
KZ_CHAIN_DELTA(4, 2)
KZ_CHAIN_DELTA(4, 4)
KZ_CHAIN_DELTA(8, 1)
KZ_CHAIN_DELTA(8, 2)
KZ_CHAIN_DELTA(16, 1)
// averaged workers on clusters of 4 or 8 (RKAB with 20480 < n <= 81920)
KZ_CHAIN_WIDE(8, 1, 4)
KZ_CHAIN_WIDE(8, 2, 4)
KZ_CHAIN_WIDE(16, 1, 4)
KZ_CHAIN_WIDE(8, 1, 8)
KZ_CHAIN_WIDE(8, 2, 8)
KZ_CHAIN_WIDE(16, 1, 8)
#undef KZ_CHAIN
#undef KZ_CHAIN_DELTA
#undef KZ_CHAIN_WIDE

}  // namespace kz
