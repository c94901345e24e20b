// Shared device helpers for the hg_gnn sm_100a library.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define HG_GOLDEN 0x9E3779B97F4A7C15ULL  // reference kernels.py:21
#define HG_MIX1 0xBF58476D1CE4E5B9ULL    // kernels.py:22
#define HG_MIX2 0x94D049BB133111EBULL    // kernels.py:23
#define HG_PHI 0x2545F4914F6CDD1DULL     // kernels.py:24
#define HG_SAMPLE_TAG 0x5AULL            // sampler.py:19

#define HG_NUM_SMS 148
#define HG_INT_MAX 0x7fffffff

// error codes returned through the C-ABI (0 ok)
#define HG_OK 0
#define HG_EINVAL -1
#define HG_ECUDA -2
#define HG_EUNSUPPORTED -3

__host__ __device__ __forceinline__ uint64_t hg_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * HG_MIX1;
    x = (x ^ (x >> 27)) * HG_MIX2;
    return x ^ (x >> 31);
}

// derive_seed(seed, a, b) — kernels.py:61-70 with two parts (the sampler's
// per-layer stream derive_seed(rng_seed, 0x5A, layer), sampler.py:143).
__host__ __device__ __forceinline__ uint64_t hg_derive2(uint64_t seed, uint64_t a, uint64_t b) {
    uint64_t st = hg_mix64(seed + HG_GOLDEN);
    st = hg_mix64((st + HG_GOLDEN) ^ a);
    st = hg_mix64((st + HG_GOLDEN) ^ b);
    return st;
}

__device__ __forceinline__ unsigned hg_lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// element count held in device memory (null => the static capacity)
__device__ __forceinline__ int hg_load_count(const int* d_n, int cap) {
    if (!d_n) return cap;
    int n = *d_n;
    return n < cap ? n : cap;
}

static inline int hg_ceil_div(long long a, long long b) { return (int)((a + b - 1) / b); }

// grid size for a grid-stride kernel over `work` items with `per_block` each
static inline int hg_grid(long long work, int per_block, int max_blocks_per_sm = 16) {
    long long g = (work + per_block - 1) / per_block;
    long long cap = (long long)HG_NUM_SMS * max_blocks_per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return (int)g;
}

// ---------------------------------------------------------------------------
// Programmatic dependent launch (PDL): step kernels are launched with
// cudaLaunchAttributeProgrammaticStreamSerialization (programmatic edges once
// captured into a graph), so a kernel's CTAs are scheduled while its
// predecessor drains.  Every such kernel calls hg_pdl_begin() first:
// griddepcontrol.wait blocks until the predecessor grid has completed and its
// writes are visible (so correctness never depends on the trigger), then
// launch_dependents lets the next kernel start launching.  No-ops when the
// kernel was launched without the attribute.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void hg_pdl_begin() {
    asm volatile("griddepcontrol.wait;\n" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory");
}

bool hg_pdl_enabled();

template <typename... KArgs, typename... Args>
inline cudaError_t hg_launch(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                             Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute a[1];
    a[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    a[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = a;
    cfg.numAttrs = hg_pdl_enabled() ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// set by every entry point; read through hg_last_error()
void hg_set_error(const char* fmt, ...);
int hg_check_launch(const char* what);
