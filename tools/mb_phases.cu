// Microbenchmark of the rka kernel's per-iteration phases in isolation (one CTA,
// 8 warps, c1 shape: LG = 16 lanes per row group, 4 rows per group, 1 pair per lane).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_phases tools/mb_phases.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "../paper_2401_17474_b200/csrc/kz_common.cuh"
using namespace kz;

constexpr int LG = 16, NR = 4, CWB = 32;

template <int MODE>
__global__ void __launch_bounds__(256, 1) phase_kernel(long long* out, double* sink, int reps) {
    __shared__ __align__(16) double rows[64 * CWB];
    __shared__ __align__(16) double upd[8 * CWB];
    __shared__ double scal[64];
    __shared__ unsigned long long mb[4];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gl = lane % LG, grp = lane / LG;
    for (int i = tid; i < 64 * CWB; i += 256) rows[i] = 1.0 + 1e-3 * (i % 97);
    for (int i = tid; i < 64; i += 256) scal[i] = 1e-3 * i;
    if (tid == 0) {
        mbar_init(&mb[0], 1);
        mbar_init(&mb[1], 1);
        mbar_arrive(&mb[0]);  // phase 0 of mb[0] complete
    }
    __syncthreads();
    double2 xv = make_double2(sink[0] + gl, sink[1] - gl);
    const int wb = warp * 8;
    double keep_sum = 0.0;
    long long t0 = clock64();
    for (int it = 0; it < reps; ++it) {
        if (MODE == 0 || MODE == 1) {  // dots (+ reduction when MODE 0)
            double acc[NR];
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const double2 rv = *reinterpret_cast<const double2*>(rows + (wb + grp * NR + r) * CWB + 2 * gl);
                acc[r] = fma(rv.x, xv.x, 0.0);
                acc[r] = fma(rv.y, xv.y, acc[r]);
            }
            if (MODE == 0) {
#pragma unroll
                for (int h = NR / 2, o = LG / 2; h >= 1; h >>= 1, o >>= 1) {
                    const bool up = (gl & o) != 0;
#pragma unroll
                    for (int i = 0; i < h; ++i) {
                        const double send = up ? acc[i] : acc[i + h];
                        const double kp = up ? acc[i + h] : acc[i];
                        acc[i] = kp + __shfl_xor_sync(0xffffffffu, send, o);
                    }
                }
                acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 2);
                acc[0] += __shfl_xor_sync(0xffffffffu, acc[0], 1);
            } else {
                acc[0] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
            }
            xv.x += acc[0] * 1e-30;  // dependence across repetitions
        } else if (MODE == 2) {  // average + group combine + upd store + named barrier + combine
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int t = wb + grp * NR + r;
                const double s = scal[t];
                const double2 rv = *reinterpret_cast<const double2*>(rows + t * CWB + 2 * gl);
                const double v0 = __dadd_rn(xv.x, __dmul_rn(s, rv.x));
                const double v1 = __dadd_rn(xv.y, __dmul_rn(s, rv.y));
                acc.x = r == 0 ? v0 : __dadd_rn(acc.x, v0);
                acc.y = r == 0 ? v1 : __dadd_rn(acc.y, v1);
            }
            const double ox = __shfl_xor_sync(0xffffffffu, acc.x, 16);
            const double oy = __shfl_xor_sync(0xffffffffu, acc.y, 16);
            acc.x = __dadd_rn(acc.x, ox);
            acc.y = __dadd_rn(acc.y, oy);
            if (grp == 0) *reinterpret_cast<double2*>(upd + warp * CWB + 2 * gl) = acc;
            named_sync(1, 256);
            double2 w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const double2*>(upd + i * CWB + 2 * gl);
#pragma unroll
            for (int h = 1; h < 8; h <<= 1)
#pragma unroll
                for (int i = 0; i + h < 8; i += 2 * h) {
                    w[i].x = __dadd_rn(w[i].x, w[i + h].x);
                    w[i].y = __dadd_rn(w[i].y, w[i + h].y);
                }
            xv.x = __dmul_rn(w[0].x, 0.015625);
            xv.y = __dmul_rn(w[0].y, 0.015625);
            named_sync(1, 256);  // upd reuse (in the kernel the exchange orders this)
        } else if (MODE == 3) {  // average only (no barrier, no combine)
            double2 acc = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 0; r < NR; ++r) {
                const int t = wb + grp * NR + r;
                const double s = scal[t];
                const double2 rv = *reinterpret_cast<const double2*>(rows + t * CWB + 2 * gl);
                const double v0 = __dadd_rn(xv.x, __dmul_rn(s, rv.x));
                const double v1 = __dadd_rn(xv.y, __dmul_rn(s, rv.y));
                acc.x = r == 0 ? v0 : __dadd_rn(acc.x, v0);
                acc.y = r == 0 ? v1 : __dadd_rn(acc.y, v1);
            }
            xv.x = acc.x * 1e-3;
            xv.y = acc.y * 1e-3;
        } else if (MODE == 4) {  // warp_sum of a double (err piece)
            keep_sum += warp_sum(xv.x);
            xv.x += keep_sum * 1e-30;
        } else if (MODE == 6) {  // named barrier alone
            named_sync(1, 256);
        } else if (MODE == 7) {  // STS + barrier + 8 LDS.128 + tree (double-buffered upd)
            double* u = upd + (it & 1) * 0;  // same buffer; ordering by the barrier of the next rep
            if (grp == 0) *reinterpret_cast<double2*>(u + warp * CWB + 2 * gl) = xv;
            named_sync(1, 256);
            double2 w[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) w[i] = *reinterpret_cast<const double2*>(u + i * CWB + 2 * gl);
#pragma unroll
            for (int h = 1; h < 8; h <<= 1)
#pragma unroll
                for (int i = 0; i + h < 8; i += 2 * h) {
                    w[i].x = __dadd_rn(w[i].x, w[i + h].x);
                    w[i].y = __dadd_rn(w[i].y, w[i + h].y);
                }
            xv.x = __dmul_rn(w[0].x, 0.015625);
            xv.y = __dmul_rn(w[0].y, 0.015625);
        } else if (MODE == 8) {  // ddiv alone (dependent)
            xv.x = __ddiv_rn(xv.y, xv.x + 3.0);
        } else if (MODE == 9) {  // one double shuffle-add level
            xv.x += __shfl_xor_sync(0xffffffffu, xv.x, 1);
        } else if (MODE == 10) {  // try_wait on an already completed phase
            mbar_wait(&mb[0], 0u);
            xv.x += 1e-30;
        } else if (MODE == 11) {  // arrive + wait on a count-1 barrier (one warp)
            if (lane == 0) mbar_arrive(&mb[1]);
            mbar_wait(&mb[1], (unsigned)(it & 1));
        } else if (MODE == 12) {  // clock64 stamp to global
            if (lane == 0) sink[512 + warp] = (double)clock64();
        } else if (MODE == 13) {  // the in-kernel probe: 16 dependent LDS then 32 dependent DADD/DMUL
            int zi = ((int)xv.x) & 1;
#pragma unroll
            for (int zz = 0; zz < 16; ++zz) zi = (int)scal[zi] & 1;
            double z = xv.y + zi;
#pragma unroll
            for (int zz = 0; zz < 32; ++zz) z = __dadd_rn(z, z * 1e-3);
            xv.x += z * 1e-30;
            xv.y = z;
        } else if (MODE == 5) {  // owner: 8 smem loads, tree, shfl, division
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) v[k] = rows[((lane & 1) * 8 + k) * 66 + (lane >> 1)];
            double tot = ((v[0] + v[1]) + (v[2] + v[3])) + ((v[4] + v[5]) + (v[6] + v[7]));
            tot += __shfl_xor_sync(0xffffffffu, tot, 1);
            const double s = __ddiv_rn(__dmul_rn(1.0, __dsub_rn(xv.x, tot)), xv.y + 3.0);
            rows[lane] = s;
            __syncwarp();
            xv.x += rows[(lane + 1) & 31] * 1e-30;
        }
    }
    long long t1 = clock64();
    if (lane == 0) out[warp] = (t1 - t0);
    sink[2 + tid] = xv.x + xv.y + keep_sum;
}

int main() {
    long long* d_out;
    double* d_sink;
    cudaMalloc(&d_out, 64 * sizeof(long long));
    cudaMalloc(&d_sink, 1024 * sizeof(double));
    cudaMemset(d_sink, 0, 1024 * sizeof(double));
    const int reps = 2000;
    const char* names[] = {"dots+reduce", "dots only", "avg+barrier+combine", "avg only", "warp_sum", "owner",
                           "named barrier", "sts+bar+lds8+tree", "ddiv", "shfl-add level", "try_wait done",
                           "arrive+wait", "clock stamp", "probe 16 LDS + 32 DADD/DMUL"};
    for (int mode = 0; mode < 14; ++mode) {
        for (int nw : {1, 8}) {
            switch (mode) {
                case 0: phase_kernel<0><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 1: phase_kernel<1><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 2: if (nw == 8) phase_kernel<2><<<1, 256>>>(d_out, d_sink, reps); break;
                case 3: phase_kernel<3><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 4: phase_kernel<4><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 5: phase_kernel<5><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 6: if (nw == 8) phase_kernel<6><<<1, 256>>>(d_out, d_sink, reps); break;
                case 7: if (nw == 8) phase_kernel<7><<<1, 256>>>(d_out, d_sink, reps); break;
                case 8: phase_kernel<8><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 9: phase_kernel<9><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 10: phase_kernel<10><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 11: if (nw == 1) phase_kernel<11><<<1, 32>>>(d_out, d_sink, reps); break;
                case 12: phase_kernel<12><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
                case 13: phase_kernel<13><<<1, 32 * nw>>>(d_out, d_sink, reps); break;
            }
            if ((mode == 2 || mode == 6 || mode == 7) && nw == 1) continue;
            if (mode == 11 && nw == 8) continue;
            cudaDeviceSynchronize();
            long long h[8];
            cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
            double mx = 0;
            for (int w = 0; w < nw; ++w) mx = h[w] > mx ? h[w] : mx;
            printf("%-22s warps=%d  %.1f cycles/rep\n", names[mode], nw, mx / reps);
        }
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
