// Global-memory ping-pong between two CTAs on different SMs: cycles per round trip
// (store a tagged word, the peer polls it and answers) for several store / load flavours.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_l2ping tools/mb_l2ping.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__device__ __forceinline__ void put(unsigned long long* p, unsigned long long v) {
    if (MODE == 0) asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 1) asm volatile("st.volatile.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 2) asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 3) asm volatile("st.relaxed.gpu.global.L1::no_allocate.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
    if (MODE == 4) asm volatile("atom.relaxed.gpu.global.exch.b64 _, [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <int MODE>
__device__ __forceinline__ unsigned long long get(const unsigned long long* p) {
    unsigned long long v;
    if (MODE == 2)
        asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else if (MODE == 1)
        asm volatile("ld.volatile.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    else
        asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

template <int MODE>
__global__ void ping(unsigned long long* words, int a, int b, int reps, long long* out) {
    const int c = blockIdx.x;
    if ((c != a && c != b) || threadIdx.x != 0) return;
    unsigned long long* wa = words;       // a -> b
    unsigned long long* wb = words + 64;  // b -> a (another 512-byte line)
    if (c == a) {
        long long t0 = 0;
        for (int k = 1; k <= reps; ++k) {
            if (k == 11) t0 = clock64();
            put<MODE>(wa, (unsigned long long)k);
            while (get<MODE>(wb) != (unsigned long long)k) {
            }
        }
        out[0] = (clock64() - t0) / (reps - 10);
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        out[1] = smid;
    } else {
        for (int k = 1; k <= reps; ++k) {
            while (get<MODE>(wa) != (unsigned long long)k) {
            }
            put<MODE>(wb, (unsigned long long)k);
        }
        unsigned smid;
        asm("mov.u32 %0, %%smid;" : "=r"(smid));
        out[2] = smid;
    }
}

template <int MODE>
void run(const char* name, unsigned long long* w, long long* o, int a, int b) {
    cudaMemset(w, 0, 4096);
    ping<MODE><<<148, 32>>>(w, a, b, 2000, o);
    cudaDeviceSynchronize();
    long long h[3];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("%-34s CTAs %3d,%3d (SM %3lld,%3lld): %lld cycles per round trip\n", name, a, b, h[1], h[2], h[0]);
}

int main() {
    unsigned long long* w;
    long long* o;
    cudaMalloc(&w, 4096);
    cudaMalloc(&o, 64);
    const int pairs[][2] = {{0, 1}, {0, 2}, {0, 16}, {0, 74}, {0, 100}, {0, 147}, {5, 90}};
    for (auto& p : pairs) {
        run<0>("st.relaxed.gpu / ld.relaxed.gpu", w, o, p[0], p[1]);
        run<1>("st.volatile / ld.volatile", w, o, p[0], p[1]);
        run<2>("st.release.gpu / ld.acquire.gpu", w, o, p[0], p[1]);
        run<3>("st.relaxed L1::no_allocate", w, o, p[0], p[1]);
        run<4>("atom.exch / ld.relaxed", w, o, p[0], p[1]);
    }
    return 0;
}
