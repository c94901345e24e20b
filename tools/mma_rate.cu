// tcgen05.mma kind::tf32 issue-rate microbenchmark (sm_100a): back-to-back MMAs
// with operands resident in shared memory (SS) or A in TMEM (TS), no loads, one
// CTA per SM; reports cycles per instruction and the implied dense tf32 rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2311_13225_b200/csrc -o tools/mma_rate tools/mma_rate.cu && tools/mma_rate
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "hg_tc.cuh"
using namespace hgtc;

template <int N, bool TS, bool BMN = false>
__global__ void __launch_bounds__(128, 1) k_rate(int iters, unsigned long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t done;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    constexpr uint32_t IDESC = idesc_tf32(128, N, 0, BMN ? 1 : 0);
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = a + 16384;
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                // B K-major (SWIZZLE_128B) or MN-major (SWIZZLE_128B_BASE32B, as the wgrad's G operand)
                const uint64_t db = BMN ? sdesc(b + s * 1024, 4096, 512, 1) : sdesc(b + s * 32, 16, 1024);
                if (TS) {
                    mma_tf32_ts(tmem, tmem + 256 + s * 8, db, IDESC, (i | s) ? 1u : 0u);
                } else {
                    const uint64_t da = sdesc(a + s * 32, 16, 1024);
                    mma_tf32(tmem, da, db, IDESC, (i | s) ? 1u : 0u);
                }
            }
        }
        mma_commit(&done);
        mbar_wait(&done, 0);
        const unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int N, bool TS, bool BMN = false>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 16384 + 256 * 128 + 1024;
    cudaFuncSetAttribute(k_rate<N, TS, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    k_rate<N, TS, BMN><<<148, 128, smem>>>(16, d);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a);
    k_rate<N, TS, BMN><<<148, 128, smem>>>(iters, d);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    const double n_mma = 4.0 * iters;
    const double flops = 148.0 * n_mma * 2.0 * 128 * N * 8;
    printf("%-28s N=%3d: %6.1f cycles/MMA, %7.1f TFLOP/s tf32 (%s)\n", name, N, cyc / n_mma, flops / (ms * 1e-3) / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<64, false>("SS (A, B from smem)");
    run<128, false>("SS (A, B from smem)");
    run<192, false>("SS (A, B from smem)");
    run<256, false>("SS (A, B from smem)");
    run<64, true>("TS (A from TMEM)");
    run<128, true>("TS (A from TMEM)");
    run<192, true>("TS (A from TMEM)");
    run<256, true>("TS (A from TMEM)");
    run<64, true, true>("TS, B MN-major");
    run<128, true, true>("TS, B MN-major");
    run<64, false, true>("SS, B MN-major");
    run<128, false, true>("SS, B MN-major");
    return 0;
}
