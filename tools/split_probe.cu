// Does splitting each 400-byte feature row into a line-aligned 384-byte body and
// a 16-byte tail (kept in a separate, L2-persisting [V x 4] table) cut the bottom
// gather's DRAM time?  Random rows cost per 128-byte LINE touched
// (profiles/r02s_gather_rowsize.txt: 1/2/4/5-line rows take 33/43/72-74/86 us per
// 738K rows), and a 400-byte row touches 4 lines for 3.125 lines of data; the
// body of the split row is exactly 3 aligned lines.
// Input: the C2 bottom block's fetch list (tools/order_probe.py), destination
// order, gathered the way k_agg_fwd does (one warp per row, U rows in flight).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/split_probe tools/split_probe.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>

template <int U, int MODE>  // MODE 0: one table (ld, F4 lanes); 1: body (B4 lanes, ldb) + tail (T4 lanes, ldt)
__global__ void __launch_bounds__(256) k_gather(const float* __restrict__ x, int ld, int F4, const float* __restrict__ t,
                                               int ldt, int B4, const int* __restrict__ idx, int R, float* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    float acc = 0.f;
    for (int r0 = warp * U; r0 < R; r0 += nw * U) {
        float4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int r = r0 + u;
            const int64_t row = r < R ? idx[r] : 0;
            if (MODE == 0) {
                v[u] = (r < R && lane < F4) ? __ldg(reinterpret_cast<const float4*>(x + row * ld) + lane)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
                const float4* p = lane < B4 ? reinterpret_cast<const float4*>(x + row * ld) + lane
                                            : reinterpret_cast<const float4*>(t + row * ldt) + (lane - B4);
                v[u] = (r < R && lane < F4) ? __ldg(p) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) acc += v[u].x + v[u].y + v[u].z + v[u].w;
    }
    if (acc == 123.456f) out[warp] = acc;
}

static void set_window(cudaStream_t s, const void* base, size_t bytes) {
    cudaStreamAttrValue a = {};
    if (base) {
        a.accessPolicyWindow.base_ptr = const_cast<void*>(base);
        a.accessPolicyWindow.num_bytes = bytes;
        a.accessPolicyWindow.hitRatio = 1.0f;
        a.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        a.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    }
    cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &a);
}

int main(int argc, char** argv) {
    const char* path = argc > 1 ? argv[1] : "tools/fetch_list.i32";
    FILE* fp = fopen(path, "rb");
    if (!fp) { printf("no %s\n", path); return 1; }
    fseek(fp, 0, SEEK_END);
    const int R = (int)(ftell(fp) / 4);
    fseek(fp, 0, SEEK_SET);
    std::vector<int> h(R);
    if (fread(h.data(), 4, R, fp) != (size_t)R) return 1;
    fclose(fp);
    const int V = 2400000, F = 100;
    int maxp = 0;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, maxp);
    printf("rows %d  persisting L2 max %.1f MB\n", R, maxp / 1e6);
    float *x, *xb, *xt;
    cudaMalloc(&x, (size_t)V * F * 4);
    // one allocation: the tail table, then the bodies (hub rows first), so one
    // access-policy window can cover the tails and the hottest bodies
    cudaMalloc(&xt, (size_t)V * 100 * 4);
    xb = xt + (size_t)V * 4;
    cudaMemset(x, 0, (size_t)V * F * 4);
    cudaMemset(xt, 0, (size_t)V * 100 * 4);
    int* idx;
    cudaMalloc(&idx, (size_t)R * 4);
    cudaMemcpy(idx, h.data(), (size_t)R * 4, cudaMemcpyHostToDevice);
    float* out;
    cudaMalloc(&out, 1 << 20);
    char* fl;
    cudaMalloc(&fl, 512 << 20);
    cudaStream_t s;
    cudaStreamCreate(&s);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, int mode, const void* wbase, size_t wbytes) {
        set_window(s, wbase, wbytes);
        float best = 1e9;
        for (int rep = 0; rep < 8; ++rep) {
            cudaMemsetAsync(fl, rep, 512 << 20, s);
            cudaEventRecord(a, s);
            if (mode == 0) k_gather<16, 0><<<148 * 8, 256, 0, s>>>(x, F, F / 4, nullptr, 0, 0, idx, R, out);
            else k_gather<16, 1><<<148 * 8, 256, 0, s>>>(xb, 96, F / 4, xt, 4, 24, idx, R, out);
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;  // rep 0 warms the persisting lines
        }
        set_window(s, nullptr, 0);
        cudaCtxResetPersistingL2Cache();
        printf("%-44s %7.1f us  %6.0f GB/s of row data\n", name, best * 1e3, (double)R * F * 4 / (best * 1e-3) / 1e9);
    };
    run("400-B rows, no window", 0, nullptr, 0);
    run("400-B rows, 32 MB hub window", 0, x, 32u << 20);
    run("400-B rows, max hub window", 0, x, (size_t)maxp);
    run("384-B body + 16-B tail, no window", 1, nullptr, 0);
    run("384-B body + 16-B tail, tail table window", 1, xt, (size_t)V * 16);
    run("384-B body + 16-B tail, tails + 32 MB hub bodies", 1, xt, (size_t)V * 16 + (32u << 20));
    run("384-B body + 16-B tail, tails + hub bodies to max", 1, xt, (size_t)maxp);
    return 0;
}
