// Random-row gather ceiling on B200: read R random rows of a [V x ld] fp32 table
// (row bytes = 4*F), one warp per row group with U rows in flight, reduce into
// a per-warp sum (no writes besides one float per warp).  Compares with the
// bottom aggregation's DRAM rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_probe tools/gather_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

template <int U>
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ x, int ld, int F4, const int* __restrict__ idx,
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

int main(int argc, char** argv) {
    const int V = 2400000, F = argc > 1 ? atoi(argv[1]) : 100, ld = argc > 2 ? atoi(argv[2]) : 100;
    const int R = 738000;
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
    cudaMalloc(&out, 1 << 20);
    // L2 flush buffer
    char* fl;
    cudaMalloc(&fl, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    printf("F=%d ld=%d rows=%d (%.1f MB of row data)\n", F, ld, R, R * F * 4 / 1e6);
    for (int ctas : {4, 8, 16}) {
        for (int U : {4, 8, 16}) {
            float best = 1e9;
            for (int rep = 0; rep < 5; ++rep) {
                cudaMemset(fl, rep, 256 << 20);
                const int grid = 148 * ctas;
                cudaEventRecord(a);
                if (U == 4) k_gather<4><<<grid, 256>>>(x, ld, F / 4, idx, R, out);
                else if (U == 8) k_gather<8><<<grid, 256>>>(x, ld, F / 4, idx, R, out);
                else k_gather<16><<<grid, 256>>>(x, ld, F / 4, idx, R, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = ms < best ? ms : best;
            }
            printf("ctas/SM %2d  rows in flight/warp %2d : %6.1f us  %6.0f GB/s of row data\n", ctas, U, best * 1e3,
                   (double)R * F * 4 / (best * 1e-3) / 1e9);
        }
    }
    return 0;
}
