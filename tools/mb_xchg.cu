// Cluster exchange microbenchmark (16 CTAs): the rka kernel's two-hop pattern
// (64 partials -> owners of 4 items -> 64 totals broadcast) with
//   MODE 0: st.async + mbarrier complete_tx (current kernel)
//   MODE 1: tagged 64-bit words ({32-bit half, tag}) stored with st.relaxed.cluster
//           into the peer's shared memory, polled locally (no mbarrier)
// Cycles per exchange round (dependent rounds).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_xchg tools/mb_xchg.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2401_17474_b200/csrc/kz_common.cuh"
using namespace kz;

constexpr int PC = 16, Q = 64, RPO = 4;

__device__ __forceinline__ void st_cluster_v2(unsigned addr, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.cluster.shared::cluster.v2.b64 [%0], {%1, %2};" ::"r"(addr), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_local_v2(unsigned addr, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.relaxed.cluster.shared::cta.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(addr) : "memory");
}
__device__ __forceinline__ void pack(double v, unsigned tag, unsigned long long& w0, unsigned long long& w1) {
    const unsigned long long bits = (unsigned long long)__double_as_longlong(v);
    w0 = (bits & 0xffffffffull) | ((unsigned long long)tag << 32);
    w1 = (bits >> 32) | ((unsigned long long)tag << 32);
}
__device__ __forceinline__ double poll(unsigned addr, unsigned tag) {
    unsigned long long w0, w1;
    do {
        ld_local_v2(addr, w0, w1);
    } while ((unsigned)(w0 >> 32) != tag || (unsigned)(w1 >> 32) != tag);
    return __longlong_as_double((long long)((w1 << 32) | (w0 & 0xffffffffull)));
}

template <int MODE>
__global__ void __cluster_dims__(PC, 1, 1) __launch_bounds__(256, 1) xchg(long long* out, double* sink, int reps) {
    __shared__ __align__(16) double inb[2][PC][RPO];
    __shared__ __align__(16) double scal[2][Q];
    __shared__ __align__(16) unsigned long long inw[2][PC][RPO][2];
    __shared__ __align__(16) unsigned long long scw[2][Q][2];
    __shared__ unsigned long long xbar[2], sbar[2];
    __shared__ __align__(16) double all[2][PC][Q];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int cr = (int)cluster_rank();
    for (int i = tid; i < 2 * PC * RPO * 2; i += 256) (&inw[0][0][0][0])[i] = 0;
    for (int i = tid; i < 2 * Q * 2; i += 256) (&scw[0][0][0])[i] = 0;
    if (tid == 0) {
        mbar_init(&xbar[0], 1);
        mbar_init(&xbar[1], 1);
        mbar_init(&sbar[0], 1);
        mbar_init(&sbar[1], 1);
        fence_mbarrier_init_cluster();
    }
    __syncthreads();
    cluster_sync_all();
    double v = 1.0 + tid * 1e-3 + cr;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        const int par = it & 1;
        const unsigned bpar = (unsigned)((it >> 1) & 1), tag = (unsigned)it + 1u;
        if (MODE == 0 && tid == 0) {
            mbar_arrive_expect_tx(&xbar[par], RPO * PC * 8);
            mbar_arrive_expect_tx(&sbar[par], Q * 8);
        }
        if (MODE >= 2) {  // single-hop all-to-all: 64 partials to all 16 CTAs
            if (tid == 0) mbar_arrive_expect_tx(&xbar[par], Q * PC * 8);
            // warp w holds rows 8w..8w+7; lane l: row 8w + (l & 7) (MODE 2: scalar) -> peers (l >> 3) + 4j
            if (MODE == 2) {
                const int t = warp * 8 + (lane & 7);
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int peer = (lane >> 3) + 4 * j;
                    st_async_f64(mapa_u32(smem_u32(&all[par][cr][t]), (unsigned)peer), v,
                                 mapa_u32(smem_u32(&xbar[par]), (unsigned)peer));
                }
            } else {  // MODE 3: pairs (16 B), lanes 0..3 x 4 pairs... lane l: pair (l & 3), peers (l >> 2) + 8j
                const int t = warp * 8 + 2 * (lane & 3);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int peer = (lane >> 2) + 8 * j;
                    st_async_v2_f64(mapa_u32(smem_u32(&all[par][cr][t]), (unsigned)peer), v, v + 1.0,
                                    mapa_u32(smem_u32(&xbar[par]), (unsigned)peer));
                }
            }
            mbar_wait(&xbar[par], bpar);
            // totals of the warp's 8 rows: 4 lanes per row x 4 partials, two shuffle levels
            const int t = warp * 8 + (lane >> 2), u4 = lane & 3;
            double s = ((all[par][4 * u4][t] + all[par][4 * u4 + 1][t]) + (all[par][4 * u4 + 2][t] + all[par][4 * u4 + 3][t]));
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            s += __shfl_xor_sync(0xffffffffu, s, 2);
            v += s * 1e-20;
            continue;
        }
        // hop 1: threads 0..63 (warps 0, 1) each push row t's partial to owner t / RPO
        if (tid < Q) {
            const int t = tid, o = t / RPO;
            if (MODE == 0) {
                st_async_f64(mapa_u32(smem_u32(&inb[par][cr][t % RPO]), (unsigned)o), v,
                             mapa_u32(smem_u32(&xbar[par]), (unsigned)o));
            } else {
                unsigned long long w0, w1;
                pack(v, tag, w0, w1);
                st_cluster_v2(mapa_u32(smem_u32(&inw[par][cr][t % RPO][0]), (unsigned)o), w0, w1);
            }
        }
        // owner (warp 7): lanes 2i, 2i+1 add 8 partials each of item i, broadcast to all
        if (warp == 7) {
            double s = 0.0;
            const int i = lane >> 1, u = lane & 1;
            if (MODE == 0) {
                mbar_wait(&xbar[par], bpar);
                if (i < RPO)
                    for (int k = 0; k < 8; ++k) s += inb[par][u * 8 + k][i];
            } else {
                if (i < RPO)
                    for (int k = 0; k < 8; ++k) s += poll(smem_u32(&inw[par][u * 8 + k][i][0]), tag);
            }
            s += __shfl_xor_sync(0xffffffffu, s, 1);
            // lane l -> peer l % 16, items (l / 16) * 2, +1
            const int peer = lane % PC, i0 = (lane / PC) * 2;
            const double a0 = __shfl_sync(0xffffffffu, s, 2 * i0), a1 = __shfl_sync(0xffffffffu, s, 2 * i0 + 2);
            const int t = cr * RPO + i0;
            if (MODE == 0) {
                st_async_v2_f64(mapa_u32(smem_u32(&scal[par][t]), (unsigned)peer), a0, a1,
                                mapa_u32(smem_u32(&sbar[par]), (unsigned)peer));
            } else {
                unsigned long long w0, w1, w2, w3;
                pack(a0, tag, w0, w1);
                pack(a1, tag, w2, w3);
                st_cluster_v2(mapa_u32(smem_u32(&scw[par][t][0]), (unsigned)peer), w0, w1);
                st_cluster_v2(mapa_u32(smem_u32(&scw[par][t + 1][0]), (unsigned)peer), w2, w3);
            }
        }
        // everyone: the 8 scales of its warp's rows
        double sc;
        if (MODE == 0) {
            mbar_wait(&sbar[par], bpar);
            sc = scal[par][warp * 8 + (lane & 7)];
        } else {
            sc = poll(smem_u32(&scw[par][warp * 8 + (lane & 7)][0]), tag);
        }
        v += sc * 1e-20;
    }
    long long t1 = clock64();
    if (tid == 0 && cr == 0) out[0] = t1 - t0;
    sink[cr * 256 + tid] = v;
    cluster_sync_all();
}

int main() {
    long long* d_out;
    double* d_sink;
    cudaMalloc(&d_out, 8);
    cudaMalloc(&d_sink, PC * 256 * 8);
    const int reps = 4000;
    cudaFuncSetAttribute(xchg<0>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(xchg<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(xchg<2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(xchg<3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    const char* names[] = {"two-hop st.async + mbarrier", "two-hop tagged words + polling",
                           "all-to-all st.async f64 + mbarrier", "all-to-all st.async v2 + mbarrier"};
    for (int mode = 0; mode < 4; ++mode) {
        if (mode == 0) xchg<0><<<PC, 256>>>(d_out, d_sink, reps);
        else if (mode == 1) xchg<1><<<PC, 256>>>(d_out, d_sink, reps);
        else if (mode == 2) xchg<2><<<PC, 256>>>(d_out, d_sink, reps);
        else xchg<3><<<PC, 256>>>(d_out, d_sink, reps);
        cudaError_t e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        long long h = 0;
        cudaMemcpy(&h, d_out, 8, cudaMemcpyDeviceToHost);
        printf("mode %d (%s): %.1f cycles per exchange (%s)\n", mode, names[mode], (double)h / reps,
               cudaGetErrorString(e));
    }
    return 0;
}
