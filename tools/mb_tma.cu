// TMA tile::gather4 throughput on one SM: K gathers of 4 random rows x W doubles
// from a 20000 x 512 fp64 matrix into shared memory, issued by 1 or 32 lanes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o mb_tma tools/mb_tma.cu -lcuda
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#include "../paper_2401_17474_b200/csrc/kz_common.cuh"
using namespace kz;

__global__ void gather_kernel(const __grid_constant__ CUtensorMap tm, int K, int W, int lanes, int reps,
                              long long* out) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ unsigned long long bar;
    const int lane = threadIdx.x;
    if (lane == 0) mbar_init(&bar, 1);
    __syncwarp();
    const unsigned bytes = (unsigned)(K * 4 * W * 8);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        if (lane == 0) mbar_arrive_expect_tx(&bar, bytes);
        __syncwarp();
        for (int k = lane; k < K; k += lanes) {
            if (lane >= lanes) break;
            const int base = (k * 7919 + r * 104729) % 19990;
            tma_gather4(smem_u32(sm + (size_t)k * 4 * W * 8), &tm, 0, base, base + 3, base + 5, base + 9, smem_u32(&bar));
        }
        mbar_wait(&bar, (unsigned)(r & 1));
    }
    long long t1 = clock64();
    if (lane == 0) out[0] = t1 - t0;
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    const int m = 20000, n = 512;
    double* A;
    cudaMalloc(&A, (size_t)m * n * 8);
    cudaMemset(A, 0, (size_t)m * n * 8);
    long long* out;
    cudaMalloc(&out, 8);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
    EncFn enc = (EncFn)fp;
    cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int W : {16, 32, 64, 128, 256}) {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {(cuuint64_t)n, (cuuint64_t)m};
        const cuuint64_t strides[1] = {(cuuint64_t)n * 8};
        const cuuint32_t box[2] = {(cuuint32_t)W, 1};
        const cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, A, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int lanes : {1, 32}) {
            const int K = W <= 64 ? 64 : (W <= 128 ? 48 : 24);
            const int reps = 200;
            gather_kernel<<<1, 32, K * 4 * W * 8>>>(tm, K, W, lanes, reps, out);
            cudaError_t e = cudaDeviceSynchronize();
            long long h = 0;
            cudaMemcpy(&h, out, 8, cudaMemcpyDeviceToHost);
            printf("W=%3d lanes=%2d K=%d: %.1f cycles per gather4 (%.0f B per op, %s)\n", W, lanes, K,
                   (double)h / reps / K, 4.0 * W * 8, cudaGetErrorString(e));
        }
    }
    return 0;
}
