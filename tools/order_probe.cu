// Does the ORDER of the bottom block's row fetches decide its DRAM traffic?
// Reads a fetch list (int32 row ids, the C2 bottom block: every destination's
// self row + its drawn neighbours, written by tools/order_probe.py) and gathers
// the rows of a 2.4M x 100 fp32 table in several orders, L2 flushed before each
// run: as listed (destination order, what k_agg_fwd does), stably bucketed into
// K source-id ranges (all warps walk the list in order, so a range's duplicate
// rows are fetched close together in time), and fully sorted.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/order_probe tools/order_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include <algorithm>

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
    const char* path = argc > 1 ? argv[1] : "tools/fetch_list.i32";
    FILE* fp = fopen(path, "rb");
    if (!fp) { printf("no %s\n", path); return 1; }
    fseek(fp, 0, SEEK_END);
    const int R = (int)(ftell(fp) / 4);
    fseek(fp, 0, SEEK_SET);
    std::vector<int> base(R);
    if (fread(base.data(), 4, R, fp) != (size_t)R) return 1;
    fclose(fp);
    const int V = 2400000, F = 100, ld = 100;
    float* x;
    cudaMalloc(&x, (size_t)V * ld * 4);
    cudaMemset(x, 0, (size_t)V * ld * 4);
    int* idx;
    cudaMalloc(&idx, (size_t)R * 4);
    float* out;
    cudaMalloc(&out, 1 << 20);
    char* fl;
    cudaMalloc(&fl, 512 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    std::vector<int> uniq(base);
    std::sort(uniq.begin(), uniq.end());
    uniq.erase(std::unique(uniq.begin(), uniq.end()), uniq.end());
    printf("fetches %d unique %zu\n", R, uniq.size());
    auto run = [&](const char* name, const std::vector<int>& order) {
        cudaMemcpy(idx, order.data(), (size_t)R * 4, cudaMemcpyHostToDevice);
        float best = 1e9;
        for (int rep = 0; rep < 7; ++rep) {
            cudaMemset(fl, rep, 512 << 20);
            cudaEventRecord(a);
            k_gather<16><<<148 * 8, 256>>>(x, ld, F / 4, idx, R, out);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%-28s %7.1f us  %6.0f GB/s of fetched row data, %6.0f GB/s of unique rows\n", name, best * 1e3,
               (double)R * F * 4 / (best * 1e-3) / 1e9, (double)uniq.size() * F * 4 / (best * 1e-3) / 1e9);
    };
    run("destination order", base);
    for (int K : {2, 3, 4, 6, 8, 16, 32}) {
        // K ranges holding equal numbers of unique rows; stable bucket of the list
        std::vector<int> bnd(K + 1);
        for (int k = 0; k <= K; ++k) bnd[k] = k == K ? V : uniq[(size_t)k * uniq.size() / K];
        std::vector<int> order;
        order.reserve(R);
        for (int k = 0; k < K; ++k)
            for (int v : base) if (v >= bnd[k] && v < bnd[k + 1]) order.push_back(v);
        char name[64];
        snprintf(name, sizeof name, "bucketed, K=%d ranges", K);
        run(name, order);
    }
    std::vector<int> s(base);
    std::sort(s.begin(), s.end());
    run("fully sorted", s);
    run("unique rows only (sorted)", [&] { std::vector<int> u(uniq); u.resize(R, uniq.back()); return u; }());
    return 0;
}
