// TMA streaming microbenchmark (sm_100a): how many bytes in flight per SM,
// and which box shapes, does a 1-producer TMA ring need to reach HBM peak?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tma_stream tools/tma_stream.cu
//   ./tma_stream
// Reads an fp32 matrix [M x 128] (512 MB) once per launch: box = 32 cols x R rows
// (128-byte rows, SWIZZLE_128B), 4 boxes per stage (all 128 columns of R rows),
// S stages, C CTAs per SM; the consumer warp releases a stage as soon as it lands.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* b, int c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* b, uint32_t ph) {
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(done) : "r"(su32(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ void bar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void bar_expect(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void tma2d(uint32_t dst, const CUtensorMap* m, int x, int y, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
        ::"r"(dst), "l"((uint64_t)m), "r"(x), "r"(y), "r"(su32(b)) : "memory");
}

__global__ void __launch_bounds__(64) k_stream(const __grid_constant__ CUtensorMap tm, int M, int R, int S,
                                              unsigned long long* sink) {
    extern __shared__ uint8_t raw[];
    uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t full[16], empty[16];
    const int stage_bytes = R * 512;
    if (threadIdx.x == 0) {
        for (int i = 0; i < S; ++i) { bar_init(&full[i], 1); bar_init(&empty[i], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int tiles = (M + R - 1) / R;
    const int my = (tiles - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    if (threadIdx.x == 0) {
        for (int it = 0; it < my; ++it) {
            const int st = it % S;
            if (it >= S) bar_wait(&empty[st], ((it / S) - 1) & 1);
            const int y = ((int)blockIdx.x + it * (int)gridDim.x) * R;
            bar_expect(&full[st], stage_bytes);
            for (int g = 0; g < 4; ++g) tma2d(su32(sm + st * stage_bytes + g * R * 128), &tm, g * 32, y, &full[st]);
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (int it = 0; it < my; ++it) {
            const int st = it % S;
            bar_wait(&full[st], (it / S) & 1);
            acc += sm[st * stage_bytes + (it & 127)];
            bar_arrive(&empty[st]);
        }
        if (acc == 0xdeadbeef) *sink = acc;
    }
}

typedef CUresult (*EncFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                          const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                          CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
    // argv[1]: logical columns (<= 128; the 4th 32-column box is partly out of bounds when < 128),
    // argv[2]: row stride in floats
    const int M = 1 << 20;
    const int NC = argc > 1 ? atoi(argv[1]) : 128, COLS = argc > 2 ? atoi(argv[2]) : 128;
    float* d;
    cudaMalloc(&d, (size_t)M * COLS * 4);
    cudaMemset(d, 1, (size_t)M * COLS * 4);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    EncFn enc = (EncFn)p;
    cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024); cudaGetLastError();
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int Rs[] = {32, 128};
    printf("cols %d ld %d (GB/s counts the %d logical columns)\nR rows/box  stage_KB  S  CTAs/SM  inflight_KB/SM   GB/s\n", NC, COLS, NC);
    for (int R : Rs) {
        CUtensorMap tm;
        cuuint64_t dims[2] = {(cuuint64_t)NC, (cuuint64_t)M};
        cuuint64_t str[1] = {(cuuint64_t)COLS * 4};
        cuuint32_t box[2] = {32, (cuuint32_t)(R > 256 ? 256 : R)};
        cuuint32_t es[2] = {1, 1};
        enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        for (int S : {2, 4, 6}) {
            for (int C : {1, 2}) {
                const int stage = R * 512;
                const int smem = S * stage + 1024;
                if (smem > 226 * 1024 || smem * C > 226 * 1024 || S > 16) continue;
                const int grid = 148 * C;
                k_stream<<<grid, 64, smem>>>(tm, M, R, S, sink);
                cudaEventRecord(a);
                for (int r = 0; r < 5; ++r) k_stream<<<grid, 64, smem>>>(tm, M, R, S, sink);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                const double gbs = 5.0 * M * NC * 4 / (ms * 1e-3) / 1e9;
                printf("%4d  %8d  %2d  %d  %8d   %7.0f%s\n", R, stage / 1024, S, C, S * stage * C / 1024, gbs,
                       cudaGetLastError() == cudaSuccess ? "" : "  (error)");
            }
        }
    }
    return 0;
}
