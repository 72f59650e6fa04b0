// Latency microbenchmarks on the B200 (cycles), to calibrate kernel design.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2401_17474_b200/csrc/kz_common.cuh"
using namespace kz;

__global__ void lat_kernel(long long* out, double* dsink, int n) {
    __shared__ double sm[1024];
    __shared__ unsigned long long bar;
    int tid = threadIdx.x;
    for (int i = tid; i < 1024; i += blockDim.x) sm[i] = 1.0 + i * 1e-9;
    __syncthreads();
    double x = dsink[0], y = dsink[1];
    long long t0, t1;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, y);
    t1 = clock64();
    if (tid == 0) out[0] = (t1 - t0);
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = fma(x, y, 1e-300);
    t1 = clock64();
    if (tid == 0) out[1] = (t1 - t0);
    // DMUL chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, y);
    t1 = clock64();
    if (tid == 0) out[2] = (t1 - t0);
    // shfl chain (double)
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __shfl_xor_sync(0xffffffffu, x, 1);
    t1 = clock64();
    if (tid == 0) out[3] = (t1 - t0);
    // LDS chain (pointer chase in smem)
    int idx = (int)(x * 0) + tid;
    t0 = clock64();
    for (int i = 0; i < n; ++i) idx = ((int)sm[idx & 1023]) + (idx & 7);
    t1 = clock64();
    if (tid == 0) out[4] = (t1 - t0);
    // ddiv chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) x = __ddiv_rn(y, x + 1.0);
    t1 = clock64();
    if (tid == 0) out[5] = (t1 - t0);
    // __syncthreads chain
    t0 = clock64();
    for (int i = 0; i < n; ++i) __syncthreads();
    t1 = clock64();
    if (tid == 0) out[6] = (t1 - t0);
    // dadd chain of 4 independent
    double a0 = x, a1 = y, a2 = x + 1, a3 = y + 1;
    t0 = clock64();
    for (int i = 0; i < n; ++i) { a0 = __dadd_rn(a0, y); a1 = __dadd_rn(a1, y); a2 = __dadd_rn(a2, y); a3 = __dadd_rn(a3, y); }
    t1 = clock64();
    if (tid == 0) out[7] = (t1 - t0);
    dsink[2 + tid] = x + a0 + a1 + a2 + a3 + idx;
}

// Cluster exchange round trip: CTA 0 bulk-copies 528 B into CTA 1, CTA 1 answers.
__global__ void __cluster_dims__(2, 1, 1) pingpong_kernel(long long* out, int n) {
    __shared__ __align__(16) double buf[2][66];
    __shared__ __align__(8) unsigned long long bars[1];
    unsigned rank = cluster_rank();
    if (threadIdx.x == 0) { mbar_init(&bars[0], 1); fence_mbarrier_init_cluster(); }
    for (int i = threadIdx.x; i < 132; i += blockDim.x) (&buf[0][0])[i] = i;
    __syncthreads();
    cluster_sync_all();
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
        if (threadIdx.x == 0) {
            unsigned par = it & 1;
            mbar_arrive_expect_tx(&bars[0], 528);
            if ((int)rank == (it & 1)) {
                fence_proxy_async_smem();
                unsigned peer = rank ^ 1;
                bulk_s2s_cluster(mapa_u32(smem_u32(&buf[1][0]), peer), smem_u32(&buf[0][0]), 528, mapa_u32(smem_u32(&bars[0]), peer));
                // self-complete my own phase with a zero-byte style: send to self too
                bulk_s2s_cluster(mapa_u32(smem_u32(&buf[1][0]), rank), smem_u32(&buf[0][0]), 528, mapa_u32(smem_u32(&bars[0]), rank));
            } else {
                // the receiver only waits; it also needs its own tx: peer sends both? keep symmetric below
            }
            (void)par;
        }
        break;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[8] = t1 - t0;
    cluster_sync_all();
}

// st.async ping-pong: CTA r sends one double to peer; waits for peer's message.
__global__ void __cluster_dims__(2, 1, 1) stasync_kernel(long long* out, int n) {
    __shared__ __align__(16) double buf[2];
    __shared__ __align__(8) unsigned long long bars[2];
    unsigned rank = cluster_rank(), peer = rank ^ 1;
    if (threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); fence_mbarrier_init_cluster(); }
    __syncthreads();
    cluster_sync_all();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < n; ++it) {
            int p = it & 1;
            mbar_arrive_expect_tx(&bars[p], 8);
            if ((int)rank == 0) {
                st_async_f64(mapa_u32(smem_u32(&buf[p]), peer), (double)it, mapa_u32(smem_u32(&bars[p]), peer));
                mbar_wait_cluster(&bars[p], (it >> 1) & 1);
            } else {
                mbar_wait_cluster(&bars[p], (it >> 1) & 1);
                st_async_f64(mapa_u32(smem_u32(&buf[p]), peer), (double)it, mapa_u32(smem_u32(&bars[p]), peer));
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[9] = (t1 - t0);
    cluster_sync_all();
}

// bulk-copy ping-pong with 528-byte payloads
__global__ void __cluster_dims__(2, 1, 1) bulkpp_kernel(long long* out, int n) {
    __shared__ __align__(16) double src[66];
    __shared__ __align__(16) double dst[2][66];
    __shared__ __align__(8) unsigned long long bars[2];
    unsigned rank = cluster_rank(), peer = rank ^ 1;
    for (int i = threadIdx.x; i < 66; i += blockDim.x) src[i] = i;
    if (threadIdx.x == 0) { mbar_init(&bars[0], 1); mbar_init(&bars[1], 1); fence_mbarrier_init_cluster(); }
    fence_proxy_async_smem();
    __syncthreads();
    cluster_sync_all();
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 0; it < n; ++it) {
            int p = it & 1;
            mbar_arrive_expect_tx(&bars[p], 528);
            if ((int)rank == 0) {
                bulk_s2s_cluster(mapa_u32(smem_u32(&dst[p][0]), peer), smem_u32(src), 528, mapa_u32(smem_u32(&bars[p]), peer));
                mbar_wait_cluster(&bars[p], (it >> 1) & 1);
            } else {
                mbar_wait_cluster(&bars[p], (it >> 1) & 1);
                bulk_s2s_cluster(mapa_u32(smem_u32(&dst[p][0]), peer), smem_u32(src), 528, mapa_u32(smem_u32(&bars[p]), peer));
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) out[10] = (t1 - t0);
    cluster_sync_all();
}

// global-memory flag ping-pong between two CTAs (grid barrier building block)
__global__ void flagpp_kernel(long long* out, unsigned* flags, int n) {
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        for (int it = 1; it <= n; ++it) {
            if (blockIdx.x == 0) {
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags), "r"((unsigned)it) : "memory");
                unsigned v;
                do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags + 32) : "memory"); } while (v < (unsigned)it);
            } else {
                unsigned v;
                do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(flags) : "memory"); } while (v < (unsigned)it);
                asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(flags + 32), "r"((unsigned)it) : "memory");
            }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[11] = (t1 - t0);
}

int main() {
    long long* d_out; double* d_sink; unsigned* d_flags;
    cudaMalloc(&d_out, 64 * sizeof(long long));
    cudaMalloc(&d_sink, 4096 * sizeof(double));
    cudaMalloc(&d_flags, 4096);
    cudaMemset(d_out, 0, 64 * 8); cudaMemset(d_flags, 0, 4096);
    double h2[2] = {1.0000001, 1e-12};
    cudaMemcpy(d_sink, h2, 16, cudaMemcpyHostToDevice);
    const int n = 1000;
    lat_kernel<<<1, 256>>>(d_out, d_sink, n);
    stasync_kernel<<<2, 32>>>(d_out, n);
    bulkpp_kernel<<<2, 32>>>(d_out, n);
    flagpp_kernel<<<2, 32>>>(d_out, d_flags, n);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[64];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    printf("status %s\n", cudaGetErrorString(e));
    const char* names[] = {"dadd", "dfma", "dmul", "shfl.f64", "lds(chase)", "ddiv", "bar.sync(8 warps)", "4x indep dadd/iter"};
    for (int i = 0; i < 8; ++i) printf("%-22s %.1f cycles/op\n", names[i], (double)h[i] / n);
    printf("%-22s %.1f cycles/round trip\n", "st.async ping-pong", (double)h[9] / n);
    printf("%-22s %.1f cycles/round trip\n", "bulk s2s 528B pp", (double)h[10] / n);
    printf("%-22s %.1f cycles/round trip\n", "gmem flag pp", (double)h[11] / n);
    return 0;
}
