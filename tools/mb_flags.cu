// Cross-SM signalling latency variants (cycles per round trip), B200.
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void pp(long long* out, unsigned* flags, double* data, int n) {
    long long t0 = clock64();
    if (threadIdx.x == 0) {
        unsigned* mine = flags + 32 * blockIdx.x;
        unsigned* peer = flags + 32 * (1 - blockIdx.x);
        for (int it = 1; it <= n; ++it) {
            const bool ping = blockIdx.x == 0;
            auto signal = [&]() {
                if (MODE == 0) {  // relaxed store, no fence
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"((unsigned)it) : "memory");
                } else if (MODE == 1) {  // data write + __threadfence + relaxed flag
                    data[blockIdx.x * 64] = it;
                    __threadfence();
                    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"((unsigned)it) : "memory");
                } else if (MODE == 2) {  // data write + st.release
                    data[blockIdx.x * 64] = it;
                    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(mine), "r"((unsigned)it) : "memory");
                } else {  // data write + red.release.gpu (grid-barrier style)
                    data[blockIdx.x * 64] = it;
                    asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(mine) : "memory");
                }
            };
            auto wait = [&]() {
                unsigned v;
                if (MODE <= 1) {
                    do { asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(peer) : "memory"); } while (v < (unsigned)it);
                    if (MODE == 1) __threadfence();
                } else {
                    do { asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(peer) : "memory"); } while (v < (unsigned)it);
                }
            };
            if (ping) { signal(); wait(); } else { wait(); signal(); }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) out[MODE] = t1 - t0;
}

int main() {
    long long* d_out; unsigned* d_flags; double* d_data;
    cudaMalloc(&d_out, 64 * 8); cudaMalloc(&d_flags, 4096); cudaMalloc(&d_data, 4096 * 8);
    const int n = 2000;
    const char* names[] = {"relaxed st/ld, no fence", "fence + relaxed", "st.release / ld.acquire", "red.release / ld.acquire"};
    long long h[8];
    for (int mode = 0; mode < 4; ++mode) {
        cudaMemset(d_flags, 0, 4096);
        if (mode == 0) pp<0><<<2, 32>>>(d_out, d_flags, d_data, n);
        if (mode == 1) pp<1><<<2, 32>>>(d_out, d_flags, d_data, n);
        if (mode == 2) pp<2><<<2, 32>>>(d_out, d_flags, d_data, n);
        if (mode == 3) pp<3><<<2, 32>>>(d_out, d_flags, d_data, n);
        cudaDeviceSynchronize();
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        printf("%-28s %.0f cycles / round trip\n", names[mode], (double)h[mode] / n);
    }
    return 0;
}
