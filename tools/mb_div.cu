// Exhaustive-ish check of kz::div_rn_fast against __ddiv_rn on random operands,
// plus its dependent-chain latency.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb_div tools/mb_div.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2401_17474_b200/csrc/kz_common.cuh"
using namespace kz;

__device__ unsigned long long mix(unsigned long long z) {
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void check(unsigned long long seed, long long per_thread, unsigned long long* bad, double* ex) {
    const unsigned long long tid = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    unsigned long long nbad = 0;
    for (long long i = 0; i < per_thread; ++i) {
        const unsigned long long h1 = mix(seed ^ (tid * 0x100000001b3ull + i * 2));
        const unsigned long long h2 = mix(seed ^ (tid * 0x100000001b3ull + i * 2 + 1));
        // mantissas uniform; exponents: mostly near 0 (the solver's range), 1/8 spread wide
        const int mode = (int)(h1 & 7);
        const int en = mode == 0 ? (int)((h1 >> 3) % 2046) + 1 : 1023 + (int)((h1 >> 3) % 80) - 40;
        const int ey = mode == 0 ? (int)((h2 >> 3) % 2046) + 1 : 1023 + (int)((h2 >> 3) % 60) - 10;
        const unsigned long long bn = ((h1 >> 12) & 0xfffffffffffffull) | ((unsigned long long)en << 52) |
                                      ((h2 & 1ull) << 63);
        const unsigned long long by = ((h2 >> 12) & 0xfffffffffffffull) | ((unsigned long long)ey << 52);
        const double n = __longlong_as_double((long long)bn), y = __longlong_as_double((long long)by);
        const double r = __drcp_rn(y);
        const double a = div_rn_fast(n, y, r), b = __ddiv_rn(n, y);
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
            if (nbad == 0) {
                ex[0] = n;
                ex[1] = y;
            }
            ++nbad;
        }
    }
    atomicAdd(bad, nbad);
}

__global__ void latency(long long* out, double* sink, int reps) {
    double n = sink[0] + 1.2345, y = sink[1] + 3.21, r = __drcp_rn(y);
    long long t0 = clock64();
    for (int i = 0; i < reps; ++i) n = div_rn_fast(n + 7.0, y, r);
    long long t1 = clock64();
    out[0] = t1 - t0;
    sink[2] = n;
}

int main() {
    unsigned long long* bad;
    double* ex;
    long long* out;
    double* sink;
    cudaMalloc(&bad, 8);
    cudaMalloc(&ex, 16);
    cudaMalloc(&out, 8);
    cudaMalloc(&sink, 64);
    cudaMemset(bad, 0, 8);
    cudaMemset(sink, 0, 64);
    const long long per = 4096;
    const int blocks = 148 * 8, threads = 256;
    for (int s = 0; s < 4; ++s) check<<<blocks, threads>>>(0x1234567ull + s * 977, per, bad, ex);
    unsigned long long h = 0;
    double hex[2] = {0, 0};
    cudaMemcpy(&h, bad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(hex, ex, 16, cudaMemcpyDeviceToHost);
    printf("samples %.3e mismatches %llu (first n=%.17g y=%.17g)\n", 4.0 * per * blocks * threads, h, hex[0], hex[1]);
    latency<<<1, 1>>>(out, sink, 1000);
    long long c = 0;
    cudaMemcpy(&c, out, 8, cudaMemcpyDeviceToHost);
    printf("div_rn_fast dependent latency %.1f cycles\n", c / 1000.0);
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
