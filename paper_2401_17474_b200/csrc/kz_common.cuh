// kz_common.cuh -- shared device helpers for the sm_100a RK/RKA/RKAB kernels.
//
// PCG64 restatement (numpy's pcg64.h as used by Prng, sampling.py:132-140):
// 128-bit LCG, output = XSL-RR of the *stepped* state, random() =
// (out >> 11) * 2^-53.  Everything here is integer-exact.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace kz {

typedef unsigned __int128 u128;

struct Pcg {
    u128 s;
    u128 inc;
};

__host__ __device__ __forceinline__ u128 pcg_mult() {
    return (((u128)2549297995355413924ULL) << 64) | (u128)4865540595714422341ULL;
}

__host__ __device__ __forceinline__ uint64_t pcg_next(Pcg& g) {
    g.s = g.s * pcg_mult() + g.inc;
    const uint64_t hi = (uint64_t)(g.s >> 64), lo = (uint64_t)g.s;
    const uint64_t x = hi ^ lo;
    const unsigned r = (unsigned)(hi >> 58);
    return (x >> r) | (x << ((64u - r) & 63u));
}

__host__ __device__ __forceinline__ double pcg_u01(Pcg& g) {
    return (double)(pcg_next(g) >> 11) * (1.0 / 9007199254740992.0);
}

// Jump the LCG ahead by `delta` steps (Brown, "Random number generation
// with arbitrary strides"): O(log delta) 128-bit multiplies.
__host__ __device__ __forceinline__ void pcg_advance(Pcg& g, uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = g.inc;
    while (delta) {
        if (delta & 1u) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    g.s = acc_mult * g.s + acc_plus;
}

// Plain-old-data copy of a generator for kernel arguments / device arrays.
struct PcgPod {
    unsigned long long s_hi, s_lo, inc_hi, inc_lo;
};

__host__ __device__ __forceinline__ Pcg pcg_from_pod(const PcgPod& p) {
    Pcg g;
    g.s = ((u128)p.s_hi << 64) | p.s_lo;
    g.inc = ((u128)p.inc_hi << 64) | p.inc_lo;
    return g;
}

// searchsorted(cdf, u, side="right") clamped to len-1 (sampling.py:177-182).
__device__ __forceinline__ int64_t upper_bound_clamped(const double* __restrict__ cdf, int64_t len, double u) {
    int64_t lo = 0, hi = len;
    while (lo < hi) {
        const int64_t mid = lo + ((hi - lo) >> 1);
        if (__ldg(cdf + mid) <= u)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo >= len ? len - 1 : lo;
}

// ---- cp.async (LDGSTS) 16-byte helpers --------------------------------------
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async_wait_dyn(int n) {
    // wait_group needs an immediate; dispatch the small range we use.
    switch (n) {
        case 0: cp_async_wait<0>(); break;
        case 1: cp_async_wait<1>(); break;
        case 2: cp_async_wait<2>(); break;
        case 3: cp_async_wait<3>(); break;
        case 4: cp_async_wait<4>(); break;
        case 5: cp_async_wait<5>(); break;
        case 6: cp_async_wait<6>(); break;
        default: cp_async_wait<7>(); break;
    }
}

// ---- grid barrier on a monotonically increasing global counter ----------
// Valid only for cooperative launches (all CTAs co-resident).  `target` is
// the counter value after this barrier (epoch * gridDim.x).
__device__ __forceinline__ void grid_barrier(unsigned* counter, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;\n" ::"l"(counter) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(counter) : "memory");
        } while (v < target);
    }
    __syncthreads();
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

}  // namespace kz
