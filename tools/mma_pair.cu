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

// Interference: the paired sequence issued by warp 1 while the other warps of the
// CTA (320 threads, as the GEMMs) either spin on an mbarrier that never completes
// (MODE 1, as waiting split / epilogue warps), keep storing to other TMEM columns
// (MODE 2, as the split warps' tcgen05.st), or stream TMA bulk copies into other
// shared memory (MODE 3, as the producer), or all three (MODE 4).
template <int MODE>
__global__ void __launch_bounds__(320, 1) k_interf(int iters, unsigned long long* cycles, const float* __restrict__ src,
                                                   int src_bytes) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t done, never, tbar[2], step;
    __shared__ uint32_t s_tmem;
    __shared__ volatile int s_stop;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&done, 1);
        mbar_init(&never, 1);
        mbar_init(&tbar[0], 1);
        mbar_init(&tbar[1], 1);
        mbar_init(&step, 1);
        s_stop = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    constexpr uint32_t I64 = idesc_tf32(128, 64, 0, 0), I128 = idesc_tf32(128, 128, 0, 0);
    if (warp == 1) {
        if (lane == 0) {
            const uint32_t b = smem_u32(smem);
            const uint32_t ta = tmem + 256;
            const unsigned long long t0 = clock64();
            for (int i = 0; i < iters; ++i) {
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const uint64_t dbh = sdesc(b + s * 32, 16, 1024);
                    mma_tf32_ts(tmem, ta + s * 8, dbh, I128, (i | s) ? 1u : 0u);
                    mma_tf32_ts(tmem, ta + 32 + s * 8, dbh, I64, 1u);
                }
                mma_commit(&step);
            }
            mma_commit(&done);
            mbar_wait(&done, 0);
            const unsigned long long t1 = clock64();
            if (blockIdx.x == 0) *cycles = t1 - t0;
            s_stop = 1;
        }
    } else if (warp == 0 && (MODE == 3 || MODE == 4)) {
        if (lane == 0) {  // TMA bulk stream: 32 KB per copy into a separate region, 2 in flight
            uint32_t ph[2] = {0, 0};
            for (int k = 0; !s_stop; ++k) {
                const int st = k & 1;
                if (k >= 2) { mbar_wait(&tbar[st] + 0, ph[st]); ph[st] ^= 1; }
                mbar_expect_tx(&tbar[st], 32768);
                bulk_load(smem_u32(smem + 16384 + st * 32768), reinterpret_cast<const uint8_t*>(src) +
                          ((int64_t)k * 32768) % src_bytes, 32768, &tbar[st]);
            }
        }
    } else if (warp >= 2 && warp < 6 && (MODE == 2 || MODE == 4)) {
        uint32_t v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = j;
        const uint32_t ta = tmem + ((uint32_t)((warp & 3) * 32) << 16) + 384;
        while (!s_stop) {
            tmem_st32(ta, v);
            tmem_wait_st();
        }
    } else if (MODE == 1 || MODE == 4) {
        while (!s_stop) {
            uint32_t ok = 0;
            asm volatile(
                "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                : "=r"(ok)
                : "r"(smem_u32(&never)), "r"(0u)
                : "memory");
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

template <int MODE>
void run_interf(const char* name, const float* src, int src_bytes) {
    unsigned long long* d;
    cudaMalloc(&d, 8);
    const int smem = 16384 + 65536 + 1024;
    cudaFuncSetAttribute(k_interf<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_interf<MODE><<<148, 320, smem>>>(16, d, src, src_bytes);
    cudaDeviceSynchronize();
    const int iters = 4096;
    k_interf<MODE><<<148, 320, smem>>>(iters, d, src, src_bytes);
    cudaDeviceSynchronize();
    unsigned long long cyc = 0;
    cudaMemcpy(&cyc, d, 8, cudaMemcpyDeviceToHost);
    printf("%-40s: %6.1f cycles per K slice (%s)\n", name, cyc / (4.0 * iters), cudaGetErrorString(cudaGetLastError()));
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
    const int src_bytes = 256 << 20;
    float* src;
    cudaMalloc(&src, src_bytes);
    cudaMemset(src, 0, src_bytes);
    run_interf<0>("pair, 320 threads, others idle", src, src_bytes);
    run_interf<1>("pair + 8 warps spinning on try_wait", src, src_bytes);
    run_interf<2>("pair + 4 warps tcgen05.st", src, src_bytes);
    run_interf<3>("pair + TMA bulk stream into smem", src, src_bytes);
    run_interf<4>("pair + all three", src, src_bytes);
    return 0;
}
