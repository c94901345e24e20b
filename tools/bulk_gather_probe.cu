// Is the random-row gather bound per SM (L1 miss tracking) or globally (DRAM)?
// Gathers R uniformly random 400-byte rows of a 2.4M x 100 fp32 table on G SMs:
//   ldg   one warp per row, 25 lanes x 16 B __ldg, U rows in flight per warp
//         (what k_agg_fwd does), 4 CTAs x 256 threads per SM
//   bulk  cp.async.bulk global -> shared per row (the TMA engine, not L1), one
//         issuing lane per warp, S-row ring per warp with an mbarrier per slot,
//         the warp sums each landed row from shared memory; 1 CTA x 8 warps per SM
// If bulk on 74 SMs matches ldg on 148, the aggregation could leave half the GPU
// to the concurrent training half.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2311_13225_b200/csrc \
//        -o tools/bulk_gather_probe tools/bulk_gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#include "hg_tc.cuh"
using namespace hgtc;

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const float* __restrict__ x, int ld, int F4, const int* __restrict__ idx,
                                            int R, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int r0 = warp * U; r0 < R; r0 += nw * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + u;
            v[u] = (r < R && lane < F4) ? __ldg(reinterpret_cast<const float4*>(x + (int64_t)idx[r] * ld) + lane)
                                        : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 123.456f) out[warp] = acc;
}

constexpr int BW = 8;  // warps per CTA (bulk)

__global__ void __launch_bounds__(BW * 32, 1) k_bulk(const float* __restrict__ x, int ld, int F4,
                                                     const int* __restrict__ idx, int R, int S,
                                                     float* __restrict__ out) {
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rb = (uint32_t)F4 * 16u;
    const int stride = (int)((rb + 127) & ~127u);
    uint8_t* ring = sm + (size_t)warp * S * stride;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)BW * S * stride) + warp * S;
    if (lane == 0) {
        for (int i = 0; i < S; ++i) mbar_init(&bar[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    const int gw = blockIdx.x * BW + warp, nw = gridDim.x * BW;
    // this warp's rows: gw, gw + nw, ...
    const int mine = gw < R ? (R - 1 - gw) / nw + 1 : 0;
    float acc = 0.f;
    int issued = 0;
    auto issue = [&](int k) {
        if (lane == 0) {
            const int st = k % S;
            const int r = idx[gw + k * nw];
            mbar_expect_tx(&bar[st], rb);
            bulk_load(smem_u32(ring + (size_t)st * stride), x + (int64_t)r * ld, rb, &bar[st]);
        }
    };
    for (; issued < mine && issued < S; ++issued) issue(issued);
    for (int k = 0; k < mine; ++k) {
        const int st = k % S;
        mbar_wait(&bar[st], (uint32_t)((k / S) & 1));
        if (lane < F4) {
            const float4 v = *reinterpret_cast<const float4*>(ring + (size_t)st * stride + lane * 16);
            acc += v.x + v.y + v.z + v.w;
        }
        __syncwarp();
        if (issued < mine) {
            fence_proxy_async();
            issue(issued);
            ++issued;
        }
    }
    if (acc == 123.456f) out[gw] = acc;
}

int main(int argc, char** argv) {
    const int V = 2400000, F = 100, ld = 100, R = 738000;
    float* x;
    cudaMalloc(&x, (size_t)V * ld * 4);
    cudaMemset(x, 0, (size_t)V * ld * 4);
    int* idx;
    cudaMalloc(&idx, R * 4);
    int* h = (int*)malloc(R * 4);
    srand(1);
    for (int i = 0; i < R; ++i) h[i] = (int)(((uint64_t)rand() * 2654435761ull) % V);
    cudaMemcpy(idx, h, R * 4, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 1 << 22);
    char* fl;
    cudaMalloc(&fl, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    auto timeit = [&](auto launch) {
        float best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
            cudaMemset(fl, rep, 256 << 20);
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        return best * 1e3f;
    };
    printf("%d random 400-B rows of a 2.4M-row table (L2 flushed)\n", R);
    for (int G : {148, 111, 74, 37}) {
        const float t = timeit([&] { k_ldg<16><<<G * 4, 256>>>(x, ld, F / 4, idx, R, out); });
        printf("ldg   SMs %3d (4 x 256 thr)        : %6.1f us  %6.1f rows/us/SM  %s\n", G, t, R / t / G,
               cudaGetErrorString(cudaGetLastError()));
    }
    for (int G : {148, 74, 37}) {
        for (int S : {8, 16, 32, 48}) {
            const int stride = 512;
            const int smem = BW * S * stride + BW * S * 8;
            if (smem > 220 * 1024) continue;
            const float t = timeit([&] { k_bulk<<<G, BW * 32, smem>>>(x, ld, F / 4, idx, R, S, out); });
            printf("bulk  SMs %3d (8 warps, %2d rows/warp): %6.1f us  %6.1f rows/us/SM  %s\n", G, S, t, R / t / G,
                   cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
