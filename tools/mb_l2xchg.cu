// The rka kernel's cross-cluster exchange in isolation: G groups x 16 CTAs, CTA (g, r) owns
// workers 4r..4r+3; per round each owner stores its 4 group totals as tagged 16-byte words and
// polls the G groups' words of its workers (sum in group order).  Rounds are back to back, so the
// time per round is the exchange latency with every CTA polling -- the floor of the rka kernel's
// cross-cluster step.  PAD = u64 words per slot (2: 16-byte slots sharing lines, 16: a line each).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_l2xchg tools/mb_l2xchg.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st2(unsigned long long* p, unsigned long long a, unsigned long long b) {
    asm volatile("st.relaxed.gpu.global.v2.b64 [%0], {%1, %2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld2(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

__device__ __forceinline__ void ld2v(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.volatile.global.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
__device__ __forceinline__ void ld2cg(const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
    asm volatile("ld.global.cg.v2.b64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}

// MODE 0: one lane per worker polls the G groups in a loop over a runtime-indexed word array (local
// memory: each load waits for the previous one's register -- the slow case); 1: lane (h, item) polls
// one word, completion by ballot, the sum in group order by shuffles; 2: as 0 with ld.volatile;
// 3: as 0 with ld.global.cg; 4: the 7 loads issued together into registers (G = 7); 5: volatile C++
// loads
template <int PAD, int MODE>
__global__ void xchg(unsigned long long* words, int G, int rounds, long long* out) {
    const int c = blockIdx.x, g = c / 16, r = c % 16, lane = threadIdx.x;
    const int Q1 = 65;
    long long t0 = 0;
    double acc = 0;
    for (int k = 1; k <= rounds; ++k) {
        if (k == 11) t0 = clock64();
        const int par = k & 1;
        unsigned long long* base = words + (size_t)par * G * Q1 * PAD;
        const unsigned long long kk = (unsigned long long)k;
        if (MODE == 1) {
            const int item = lane >> 3, h = lane & 7;  // 4 items x up to 8 groups
            const int t = 4 * r + item;
            if (h == 0) st2(base + ((size_t)g * Q1 + t) * PAD, (kk << 32) | 1u, (kk << 32) | 2u);
            unsigned long long w0 = kk << 32, w1 = kk << 32;
            const bool mine = h < G;
            bool ok = !mine;
            while (!__all_sync(0xffffffffu, ok)) {
                if (!ok) {
                    ld2(base + ((size_t)h * Q1 + t) * PAD, w0, w1);
                    ok = (w0 >> 32) == kk && (w1 >> 32) == kk;
                }
            }
            double v = mine ? (double)(w0 & 0xffffffffull) : 0.0;
            for (int o = 1; o < 8; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc += v;
        } else if (MODE == 4 && lane < 4) {  // all 7 words in one asm statement (G == 7)
            const int t = 4 * r + lane;
            st2(base + ((size_t)g * Q1 + t) * PAD, (kk << 32) | 1u, (kk << 32) | 2u);
            unsigned long long w[14];
            for (;;) {
                const unsigned long long* q0 = base + (size_t)t * PAD;
                const size_t st = (size_t)Q1 * PAD;
                asm volatile(
                    "ld.relaxed.gpu.global.v2.b64 {%0, %1}, [%14];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%2, %3}, [%15];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%4, %5}, [%16];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%6, %7}, [%17];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%8, %9}, [%18];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%10, %11}, [%19];\n"
                    "ld.relaxed.gpu.global.v2.b64 {%12, %13}, [%20];\n"
                    : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3]), "=l"(w[4]), "=l"(w[5]), "=l"(w[6]),
                      "=l"(w[7]), "=l"(w[8]), "=l"(w[9]), "=l"(w[10]), "=l"(w[11]), "=l"(w[12]), "=l"(w[13])
                    : "l"(q0), "l"(q0 + st), "l"(q0 + 2 * st), "l"(q0 + 3 * st), "l"(q0 + 4 * st), "l"(q0 + 5 * st),
                      "l"(q0 + 6 * st)
                    : "memory");
                bool all = true;
                for (int h = 0; h < 14; ++h)
                    if ((w[h] >> 32) != kk) all = false;
                if (all) break;
            }
            for (int h = 0; h < 14; h += 2) acc += (double)(w[h] & 0xffffffffull);
        } else if (MODE == 5 && lane < 4) {  // plain volatile C++ loads (compiler-scheduled)
            const int t = 4 * r + lane;
            st2(base + ((size_t)g * Q1 + t) * PAD, (kk << 32) | 1u, (kk << 32) | 2u);
            volatile const unsigned long long* vb = base;
            for (;;) {
                unsigned long long w0[16], w1[16];
                for (int h = 0; h < G; ++h) {
                    w0[h] = vb[((size_t)h * Q1 + t) * PAD];
                    w1[h] = vb[((size_t)h * Q1 + t) * PAD + 1];
                }
                bool all = true;
                for (int h = 0; h < G; ++h)
                    if ((w0[h] >> 32) != kk || (w1[h] >> 32) != kk) all = false;
                if (all) {
                    for (int h = 0; h < G; ++h) acc += (double)(w0[h] & 0xffffffffull);
                    break;
                }
            }
        } else if (MODE <= 3 && lane < 4) {
            const int t = 4 * r + lane;
            st2(base + ((size_t)g * Q1 + t) * PAD, (kk << 32) | 1u, (kk << 32) | 2u);
            unsigned long long w0[16], w1[16];
            auto ld = [&](const unsigned long long* p, unsigned long long& a, unsigned long long& b) {
                if (MODE == 2) ld2v(p, a, b);
                else if (MODE == 3) ld2cg(p, a, b);
                else ld2(p, a, b);
            };
            for (int h = 0; h < G; ++h) ld(base + ((size_t)h * Q1 + t) * PAD, w0[h], w1[h]);
            for (;;) {
                bool all = true;
                for (int h = 0; h < G; ++h)
                    if ((w0[h] >> 32) != kk || (w1[h] >> 32) != kk) all = false;
                if (all) break;
                for (int h = 0; h < G; ++h)
                    if ((w0[h] >> 32) != kk || (w1[h] >> 32) != kk) ld(base + ((size_t)h * Q1 + t) * PAD, w0[h], w1[h]);
            }
            for (int h = 0; h < G; ++h) acc += (double)(w0[h] & 0xffffffffull);
        }
        __syncthreads();
    }
    if (lane == 0) out[c] = (clock64() - t0) / (rounds - 10);
    if (acc < 0) out[0] = 0;
}

template <int PAD, int MODE>
void run(unsigned long long* w, long long* o, int G) {
    cudaMemset(w, 0, 16 << 20);
    xchg<PAD, MODE><<<G * 16, 32>>>(w, G, 2000, o);
    cudaDeviceSynchronize();
    long long h[128];
    cudaMemcpy(h, o, G * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0, sum = 0;
    for (int i = 0; i < G * 16; ++i) { mx = h[i] > mx ? h[i] : mx; sum += h[i]; }
    printf("G=%d (%3d CTAs) pad=%2d mode=%d: %lld cycles per exchange round (mean over CTAs %lld)\n", G, G * 16, PAD,
           MODE, mx, sum / (G * 16));
}

int main() {
    unsigned long long* w;
    long long* o;
    cudaMalloc(&w, 16 << 20);
    cudaMalloc(&o, 4096);
    for (int G : {1, 4, 7}) {
        run<2, 0>(w, o, G);
        run<16, 0>(w, o, G);
        run<2, 1>(w, o, G);
        run<16, 1>(w, o, G);
        run<2, 2>(w, o, G);
        run<2, 3>(w, o, G);
        run<16, 5>(w, o, G);
    }
    run<16, 4>(w, o, 7);
    return 0;
}
