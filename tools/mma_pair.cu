// tcgen05.mma kind::tf32 rate of the 3xTF32 K-slice SEQUENCES the GEMMs issue
// (sm_100a), operands resident (no loads), one CTA per SM, 148 CTAs:
//   pair    A_hi x [B_hi;B_lo] (N=128) then A_lo x B_hi (N=64), same accumulator
//   pair2   A_hi x [B_hi;B_lo] (N=128) then A_lo x [B_hi;B_lo] (N=128, extra lo*lo term)
//   three   A_hi x B_hi, A_hi x B_lo, A_lo x B_hi (N=64 each)
//   split   pair, but A_lo x B_hi into a SEPARATE accumulator (no back-to-back
//           dependency on the same TMEM columns)
// each with / without a tcgen05.commit every 4 slices (the GEMMs commit per K tile).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -I paper_2311_13225_b200/csrc -o tools/mma_pair tools/mma_pair.cu && tools/mma_pair
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include "hg_tc.cuh"
using namespace hgtc;

template <int SEQ, bool COMMIT>
__global__ void __launch_bounds__(128, 1) k_seq(int iters, unsigned long long* cycles) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t done, step;
    __shared__ uint32_t s_tmem;
    const int warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        mbar_init(&step, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    constexpr uint32_t I64 = idesc_tf32(128, 64, 0, 0), I128 = idesc_tf32(128, 128, 0, 0);
    if (threadIdx.x == 0) {
        const uint32_t b = smem_u32(smem);  // [B_hi ; B_lo]: 128 K-major rows, SWIZZLE_128B
        const uint32_t ta = tmem + 256;     // A_hi cols 256.., A_lo cols 288..
        const unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint64_t dbh = sdesc(b + s * 32, 16, 1024);
                const uint64_t dbl = sdesc(b + 8192 + s * 32, 16, 1024);
                const uint32_t acc = (i | s) ? 1u : 0u;
                if (SEQ == 0) {
                    mma_tf32_ts(tmem, ta + s * 8, dbh, I128, acc);
                    mma_tf32_ts(tmem, ta + 32 + s * 8, dbh, I64, 1u);
                } else if (SEQ == 1) {
                    mma_tf32_ts(tmem, ta + s * 8, dbh, I128, acc);
                    mma_tf32_ts(tmem, ta + 32 + s * 8, dbh, I128, 1u);
                } else if (SEQ == 2) {
                    mma_tf32_ts(tmem, ta + s * 8, dbh, I64, acc);
                    mma_tf32_ts(tmem, ta + s * 8, dbl, I64, 1u);
                    mma_tf32_ts(tmem, ta + 32 + s * 8, dbh, I64, 1u);
                } else {
                    mma_tf32_ts(tmem, ta + s * 8, dbh, I128, acc);
                    mma_tf32_ts(tmem + 128, ta + 32 + s * 8, dbh, I64, acc);
                }
            }
            if (COMMIT) mma_commit(&step);
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

template <int SEQ, bool COMMIT>
void run(const char* name) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 16384 + 1024;
    cudaFuncSetAttribute(k_seq<SEQ, COMMIT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 4096;
    k_seq<SEQ, COMMIT><<<148, 128, smem>>>(16, d);
    cudaDeviceSynchronize();
    k_seq<SEQ, COMMIT><<<148, 128, smem>>>(iters, d);
    cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    // ideal: 64 cycles per N=128, 48 per N=64 (profiles/r01_mma_rate.txt)
    printf("%-34s commit/4 %d: %6.1f cycles per K slice (%s)\n", name, (int)COMMIT, cyc / (4.0 * iters),
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    run<0, false>("pair  (N128 + N64, same acc)");
    run<0, true>("pair  (N128 + N64, same acc)");
    run<1, false>("pair2 (N128 + N128)");
    run<1, true>("pair2 (N128 + N128)");
    run<2, false>("three (3 x N64)");
    run<2, true>("three (3 x N64)");
    run<3, false>("split (N128 + N64, separate acc)");
    run<3, true>("split (N128 + N64, separate acc)");
    return 0;
}
