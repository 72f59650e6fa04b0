// (1) Does the latency of a coherent (gpu-scope) load depend on which L2 partition homes the line?
//     One thread on each of a few SMs times dependent ld.relaxed.gpu loads to N lines (4 KB + 128 B
//     apart); per SM: the latency distribution and a near/far bit string of the first 64 lines.
// (2) Ping-pong between two CTAs on different dies (complementary near/far patterns) with the two flag
//     lines homed on the reader's or the writer's die: does the placement of a polled word matter?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_l2home tools/mb_l2home.cu
#include <algorithm>
#include <cstdio>
#include <vector>
#include <cuda_runtime.h>

constexpr int N = 256, R = 16, STRIDE = (4096 + 128) / 8;

__global__ void probe(const unsigned long long* base, const int* ctas, int nprobe, int* lat, int* smids) {
    int slot = -1;
    for (int i = 0; i < nprobe; ++i)
        if (ctas[i] == (int)blockIdx.x) slot = i;
    if (slot < 0 || threadIdx.x != 0) return;
    unsigned smid;
    asm("mov.u32 %0, %%smid;" : "=r"(smid));
    smids[slot] = (int)smid;
    for (int pass = 0; pass < 2; ++pass)  // pass 0 warms the TLB
        for (int i = 0; i < N; ++i) {
            const unsigned long long* p = base + (size_t)i * STRIDE;
            unsigned long long v = 0;
            const long long t0 = clock64();
            for (int r = 0; r < R; ++r) {
                unsigned long long w;
                asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(w) : "l"(p + (v & 1)) : "memory");
                v = w;  // the words are zero: the next address depends on this load
            }
            const long long t1 = clock64();
            if (pass == 1) lat[slot * N + i] = (int)((t1 - t0) / R) + (int)(v & 1);
        }
}

__global__ void ping(unsigned long long* wa, unsigned long long* wb, int a, int b, int reps, long long* out) {
    const int c = blockIdx.x;
    if ((c != a && c != b) || threadIdx.x != 0) return;
    if (c == a) {
        long long t0 = 0;
        for (int k = 1; k <= reps; ++k) {
            if (k == 11) t0 = clock64();
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(wa), "l"((unsigned long long)k) : "memory");
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(wb) : "memory");
            } while (v != (unsigned long long)k);
        }
        out[0] = (clock64() - t0) / (reps - 10);
    } else {
        for (int k = 1; k <= reps; ++k) {
            unsigned long long v;
            do {
                asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(wa) : "memory");
            } while (v != (unsigned long long)k);
            asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(wb), "l"((unsigned long long)k) : "memory");
        }
    }
}

int main() {
    unsigned long long* w;
    int *lat, *smids, *ctas;
    long long* o;
    const std::vector<int> probe_ctas = {0, 1, 2, 16, 40, 74, 100, 120, 147};
    const int np = (int)probe_ctas.size();
    const size_t bytes = (size_t)N * STRIDE * 8 + 4096;
    cudaMalloc(&w, bytes);
    cudaMemset(w, 0, bytes);
    cudaMalloc(&lat, np * N * sizeof(int));
    cudaMalloc(&smids, np * sizeof(int));
    cudaMalloc(&ctas, np * sizeof(int));
    cudaMalloc(&o, 64);
    cudaMemcpy(ctas, probe_ctas.data(), np * sizeof(int), cudaMemcpyHostToDevice);
    probe<<<148, 32>>>(w, ctas, np, lat, smids);
    cudaDeviceSynchronize();
    std::vector<int> h(np * N), sm(np);
    cudaMemcpy(h.data(), lat, h.size() * sizeof(int), cudaMemcpyDeviceToHost);
    cudaMemcpy(sm.data(), smids, np * sizeof(int), cudaMemcpyDeviceToHost);
    std::vector<std::vector<int>> farbit(np, std::vector<int>(N));
    for (int s = 0; s < np; ++s) {
        std::vector<int> v(h.begin() + s * N, h.begin() + (s + 1) * N);
        std::vector<int> srt = v;
        std::sort(srt.begin(), srt.end());
        const int thr = (srt[N / 10] + srt[N - 1 - N / 10]) / 2;
        int far = 0;
        for (int i = 0; i < N; ++i) far += farbit[s][i] = v[i] > thr;
        printf("CTA %3d SM %3d: load latency min %d p10 %d median %d p90 %d max %d; threshold %d -> %d of %d lines far; ",
               probe_ctas[s], sm[s], srt[0], srt[N / 10], srt[N / 2], srt[N - 1 - N / 10], srt[N - 1], thr, far, N);
        for (int i = 0; i < 64; ++i) putchar(farbit[s][i] ? 'F' : 'n');
        putchar('\n');
    }
    // a pair of probed CTAs on different dies: the most complementary patterns; and a same-die pair
    int pa = 0, pb = 1, best = -1, sa = 0, sb = 1, same = N + 1;
    for (int x = 0; x < np; ++x)
        for (int y = x + 1; y < np; ++y) {
            int diff = 0;
            for (int i = 0; i < N; ++i) diff += farbit[x][i] != farbit[y][i];
            if (diff > best) best = diff, pa = x, pb = y;
            if (diff < same) same = diff, sa = x, sb = y;
        }
    printf("different dies: CTAs %d, %d (%d of %d lines differ); same die: CTAs %d, %d (%d differ)\n", probe_ctas[pa],
           probe_ctas[pb], best, N, probe_ctas[sa], probe_ctas[sb], same);
    // lines both agree on: near for a (far for b) and near for b (far for a)
    std::vector<int> nearA, nearB;
    for (int i = 0; i < N; ++i) {
        if (!farbit[pa][i] && farbit[pb][i]) nearA.push_back(i);
        if (farbit[pa][i] && !farbit[pb][i]) nearB.push_back(i);
    }
    auto run = [&](const char* name, int la, int lb, int a, int b) {
        cudaMemset(w, 0, bytes);
        ping<<<148, 32>>>(w + (size_t)la * STRIDE, w + (size_t)lb * STRIDE, a, b, 2000, o);
        cudaDeviceSynchronize();
        long long r;
        cudaMemcpy(&r, o, sizeof(r), cudaMemcpyDeviceToHost);
        printf("%-64s %lld cycles per round trip\n", name, r);
    };
    if (nearA.size() >= 2 && nearB.size() >= 2) {
        const int a = probe_ctas[pa], b = probe_ctas[pb];
        run("cross-die, both flags homed on a's die", nearA[0], nearA[1], a, b);
        run("cross-die, both flags homed on b's die", nearB[0], nearB[1], a, b);
        run("cross-die, each flag homed on its READER's die", nearB[0], nearA[0], a, b);  // wa read by b, wb read by a
        run("cross-die, each flag homed on its WRITER's die", nearA[0], nearB[0], a, b);
        const int c = probe_ctas[sa], d = probe_ctas[sb];
        const bool cA = same == 0 ? farbit[sa][nearA[0]] == 0 : true;
        run("same die, flags homed on that die", cA ? nearA[0] : nearB[0], cA ? nearA[1] : nearB[1], c, d);
        run("same die, flags homed on the other die", cA ? nearB[0] : nearA[0], cA ? nearB[1] : nearA[1], c, d);
    }
    return 0;
}
