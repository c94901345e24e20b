#include <cuda.h>
// Error plumbing, device-wide exclusive scan and stable LSD radix sort.
//
// Both primitives are deterministic (no float atomics; stable ordering) and
// read their element count from device memory so a whole training step can be
// captured in one CUDA graph without host round trips.
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "hg_common.cuh"
#include "hg_gnn_internal.h"

static thread_local char g_err[512] = "";

void hg_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int hg_check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        hg_set_error("%s: %s", what, cudaGetErrorString(e));
        return HG_ECUDA;
    }
    return HG_OK;
}

extern "C" int hg_last_error(char* buf, int len) {
    if (!buf || len <= 0) return (int)strlen(g_err);
    snprintf(buf, (size_t)len, "%s", g_err);
    return (int)strlen(g_err);
}

extern "C" uint64_t hg_mix64_host(uint64_t x) { return hg_mix64(x); }

extern "C" uint64_t hg_derive_seed(uint64_t seed, const uint64_t* parts, int n_parts) {
    uint64_t st = hg_mix64(seed + HG_GOLDEN);
    for (int i = 0; i < n_parts; ++i) st = hg_mix64((st + HG_GOLDEN) ^ parts[i]);
    return st;
}

extern "C" int hg_abi_version(void) { return HG_ABI_VERSION; }

// Number of kernel nodes in a captured CUDA graph (cudaGraph_t as void*):
// the bench's evidence of how many of this library's kernels one step launches.
extern "C" int64_t hg_graph_kernel_count(void* graph) {
    if (!graph) return -1;
    size_t n = 0;
    if (cudaGraphGetNodes((cudaGraph_t)graph, nullptr, &n) != cudaSuccess) return -1;
    cudaGraphNode_t* nodes = (cudaGraphNode_t*)malloc(sizeof(cudaGraphNode_t) * (n ? n : 1));
    if (!nodes) return -1;
    int64_t k = -1;
    if (cudaGraphGetNodes((cudaGraph_t)graph, nodes, &n) == cudaSuccess) {
        k = 0;
        for (size_t i = 0; i < n; ++i) {
            cudaGraphNodeType t;
            if (cudaGraphNodeGetType(nodes[i], &t) == cudaSuccess && t == cudaGraphNodeTypeKernel) ++k;
        }
    }
    free(nodes);
    return k;
}

// ---------------------------------------------------------------------------
// exclusive scan over int32 (reduce -> scan tile sums -> apply)
// ---------------------------------------------------------------------------
namespace {
constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 8;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

__device__ __forceinline__ long long scan_len(const int* d_n, long long mult, long long cap) {
    long long n = d_n ? (long long)(*d_n) * mult : cap;
    return n < cap ? n : cap;
}

template <int NT>
__device__ __forceinline__ int block_excl_scan(int v, int* s_warp, int& total) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < NT / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < NT / 32) s_warp[lane] = w;
    }
    __syncthreads();
    total = s_warp[NT / 32 - 1];
    int base = wid ? s_warp[wid - 1] : 0;
    __syncthreads();
    return base + x - v;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_reduce(const int* __restrict__ in,
                                                              const int* d_n, long long mult,
                                                              long long cap, int* __restrict__ tile_sums) {
    __shared__ int s_warp[SCAN_THREADS / 32];
    const long long n = scan_len(d_n, mult, cap);
    const long long t0 = (long long)blockIdx.x * SCAN_TILE;
    int acc = 0;
    if (t0 < n) {
#pragma unroll
        for (int k = 0; k < SCAN_ITEMS; ++k) {
            long long p = t0 + (long long)k * SCAN_THREADS + threadIdx.x;
            if (p < n) acc += in[p];
        }
    }
    int tot;
    block_excl_scan<SCAN_THREADS>(acc, s_warp, tot);
    if (threadIdx.x == 0) tile_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(1024) k_scan_tiles(int* __restrict__ tile_sums, int n_tiles,
                                                      int* __restrict__ d_total) {
    __shared__ int s_warp[32];
    int carry = 0;
    for (int base = 0; base < n_tiles; base += 1024) {
        int i = base + threadIdx.x;
        int v = i < n_tiles ? tile_sums[i] : 0;
        int tot;
        int ex = block_excl_scan<1024>(v, s_warp, tot);
        if (i < n_tiles) tile_sums[i] = carry + ex;
        carry += tot;
    }
    if (threadIdx.x == 0 && d_total) *d_total = carry;
}

__global__ void __launch_bounds__(SCAN_THREADS) k_scan_apply(const int* in, int* out, const int* d_n,
                                                             long long mult, long long cap,
                                                             const int* __restrict__ tile_sums) {
    __shared__ int s_warp[SCAN_THREADS / 32];
    const long long n = scan_len(d_n, mult, cap);
    const long long t0 = (long long)blockIdx.x * SCAN_TILE;
    if (t0 >= n) return;
    // each thread owns SCAN_ITEMS consecutive items (blocked arrangement)
    int v[SCAN_ITEMS];
    int acc = 0;
    const long long my0 = t0 + (long long)threadIdx.x * SCAN_ITEMS;
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        long long p = my0 + k;
        v[k] = p < n ? in[p] : 0;
        acc += v[k];
    }
    int tot;
    int ex = block_excl_scan<SCAN_THREADS>(acc, s_warp, tot) + tile_sums[blockIdx.x];
#pragma unroll
    for (int k = 0; k < SCAN_ITEMS; ++k) {
        long long p = my0 + k;
        if (p < n) out[p] = ex;
        ex += v[k];
    }
}
}  // namespace

size_t hg_scan_ws_ints(long long cap) { return (size_t)hg_ceil_div(cap, SCAN_TILE) + 1; }

// out[p] = sum(in[0..p)) for p < n, n = min(*d_n * mult, cap) (or cap when d_n
// is null).  in == out is allowed.  *d_total (optional) = sum of all n items.
int hg_scan_launch(const int* in, int* out, const int* d_n, long long mult, long long cap,
                   int* d_total, int* ws, cudaStream_t s) {
    if (cap <= 0) {
        if (d_total) cudaMemsetAsync(d_total, 0, sizeof(int), s);
        return hg_check_launch("scan(empty)");
    }
    int tiles = hg_ceil_div(cap, SCAN_TILE);
    k_scan_reduce<<<tiles, SCAN_THREADS, 0, s>>>(in, d_n, mult, cap, ws);
    k_scan_tiles<<<1, 1024, 0, s>>>(ws, tiles, d_total);
    k_scan_apply<<<tiles, SCAN_THREADS, 0, s>>>(in, out, d_n, mult, cap, ws);
    return hg_check_launch("scan");
}

extern "C" int hg_scan_exclusive(const int32_t* in, int32_t* out, const int32_t* d_n, int64_t cap,
                                 int32_t* d_total, int32_t* ws, void* stream) {
    return hg_scan_launch(in, out, d_n, 1, cap, d_total, ws, (cudaStream_t)stream);
}

extern "C" int64_t hg_scan_ws_size(int64_t cap) { return (int64_t)hg_scan_ws_ints(cap); }

// ---------------------------------------------------------------------------
// stable LSD radix sort: uint32 keys (low `key_bits` significant), int32 values
// ---------------------------------------------------------------------------
namespace {
constexpr int RS_THREADS = 256;
constexpr int RS_CHUNKS = 8;  // chunks of RS_THREADS items per tile
constexpr int RS_TILE = RS_THREADS * RS_CHUNKS;
constexpr int RS_BITS = 8;
constexpr int RS_RADIX = 1 << RS_BITS;

__global__ void __launch_bounds__(RS_THREADS) k_rs_hist(const uint32_t* __restrict__ keys, long long n,
                                                        int shift, int n_tiles, int* __restrict__ hist) {
    __shared__ int s_h[RS_RADIX];
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) s_h[d] = 0;
    __syncthreads();
    const long long t0 = (long long)blockIdx.x * RS_TILE;
    for (int c = 0; c < RS_CHUNKS; ++c) {
        long long p = t0 + (long long)c * RS_THREADS + threadIdx.x;
        if (p < n) atomicAdd(&s_h[(keys[p] >> shift) & (RS_RADIX - 1)], 1);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) hist[(long long)d * n_tiles + blockIdx.x] = s_h[d];
}

__global__ void __launch_bounds__(RS_THREADS) k_rs_scatter(const uint32_t* __restrict__ kin,
                                                           const int* __restrict__ vin, uint32_t* __restrict__ kout,
                                                           int* __restrict__ vout, long long n, int shift,
                                                           int n_tiles, const int* __restrict__ offs) {
    constexpr int NW = RS_THREADS / 32;
    __shared__ int s_base[RS_RADIX];       // running per-digit base inside the tile
    __shared__ int s_wcnt[NW][RS_RADIX];   // per-warp digit counts of the current chunk
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS)
        s_base[d] = offs[(long long)d * n_tiles + blockIdx.x];
    const long long t0 = (long long)blockIdx.x * RS_TILE;
    for (int c = 0; c < RS_CHUNKS; ++c) {
        for (int d = threadIdx.x; d < RS_RADIX * NW; d += RS_THREADS) (&s_wcnt[0][0])[d] = 0;
        __syncthreads();
        long long p = t0 + (long long)c * RS_THREADS + threadIdx.x;
        bool ok = p < n;
        uint32_t key = ok ? kin[p] : 0u;
        int val = ok ? vin[p] : 0;
        int dig = ok ? (int)((key >> shift) & (RS_RADIX - 1)) : RS_RADIX;  // sentinel group
        unsigned peers = __match_any_sync(0xffffffffu, dig);
        int in_warp = __popc(peers & hg_lanemask_lt());
        int leader = __ffs(peers) - 1;
        if (ok && lane == leader) s_wcnt[wid][dig] = __popc(peers);
        __syncthreads();
        // exclusive prefix across warps for each digit; then advance the running base
        for (int d = threadIdx.x; d < RS_RADIX; d += RS_THREADS) {
            int run = s_base[d];
            for (int w = 0; w < NW; ++w) {
                int cnt = s_wcnt[w][d];
                s_wcnt[w][d] = run;
                run += cnt;
            }
            s_base[d] = run;
        }
        __syncthreads();
        if (ok) {
            int pos = s_wcnt[wid][dig] + in_warp;
            kout[pos] = key;
            vout[pos] = val;
        }
        __syncthreads();
    }
}
}  // namespace

// Sorts (keys, vals) of length n by the low key_bits bits, stable.  The result
// lands in (k_alt, v_alt) if an odd number of passes ran, else back in (keys,
// vals); *out_in_alt tells which.  ws >= hg_radix_ws_ints(n) ints.
int hg_radix_sort_launch(uint32_t* keys, int* vals, uint32_t* k_alt, int* v_alt, long long n, int key_bits,
                         int* ws, int* out_in_alt, cudaStream_t s) {
    int passes = (key_bits + RS_BITS - 1) / RS_BITS;
    if (passes < 1) passes = 1;
    int n_tiles = hg_ceil_div(n, RS_TILE);
    if (n_tiles < 1) n_tiles = 1;
    uint32_t *ka = keys, *kb = k_alt;
    int *va = vals, *vb = v_alt;
    int* hist = ws;
    int* scan_ws = ws + (size_t)RS_RADIX * n_tiles;
    for (int pss = 0; pss < passes; ++pss) {
        int shift = pss * RS_BITS;
        k_rs_hist<<<n_tiles, RS_THREADS, 0, s>>>(ka, n, shift, n_tiles, hist);
        hg_scan_launch(hist, hist, nullptr, 1, (long long)RS_RADIX * n_tiles, nullptr, scan_ws, s);
        k_rs_scatter<<<n_tiles, RS_THREADS, 0, s>>>(ka, va, kb, vb, n, shift, n_tiles, hist);
        uint32_t* tk = ka; ka = kb; kb = tk;
        int* tv = va; va = vb; vb = tv;
    }
    *out_in_alt = (passes & 1);
    return hg_check_launch("radix_sort");
}

extern "C" int hg_radix_sort_pairs(uint32_t* keys, int32_t* vals, uint32_t* k_alt, int32_t* v_alt,
                                   int64_t n, int32_t key_bits, int32_t* ws, int32_t* out_in_alt,
                                   void* stream) {
    return hg_radix_sort_launch(keys, vals, k_alt, v_alt, n, key_bits, ws, out_in_alt,
                                (cudaStream_t)stream);
}

size_t hg_radix_ws_ints(long long n) {
    // histogram + the scan workspace of the histogram
    long long h = (long long)RS_RADIX * (hg_ceil_div(n, RS_TILE) > 0 ? hg_ceil_div(n, RS_TILE) : 1);
    return (size_t)(h + (long long)hg_scan_ws_ints(h) + 16);
}

extern "C" int64_t hg_radix_ws_size(int64_t n) { return (int64_t)hg_radix_ws_ints(n); }

// ---------------------------------------------------------------------------
// L2 residency for the hot rows of the feature table (process-wide): kernels
// that gather feature rows attach an access-policy window so accesses inside it
// persist in L2 across batches (hub rows are re-read by most batches).
// ---------------------------------------------------------------------------
namespace {
const void* g_l2_base = nullptr;
size_t g_l2_bytes = 0;
float g_l2_hit = 0.f;
}  // namespace

bool hg_l2_window_attr(cudaLaunchAttribute* a) {
    if (!g_l2_base || !g_l2_bytes) return false;
    a->id = cudaLaunchAttributeAccessPolicyWindow;
    a->val.accessPolicyWindow.base_ptr = const_cast<void*>(g_l2_base);
    a->val.accessPolicyWindow.num_bytes = g_l2_bytes;
    a->val.accessPolicyWindow.hitRatio = g_l2_hit;
    a->val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    a->val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    return true;
}

extern "C" int64_t hg_l2_persist_max(void) {
    int dev = 0, a = 0, b = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceGetAttribute(&a, cudaDevAttrMaxPersistingL2CacheSize, dev);
    cudaDeviceGetAttribute(&b, cudaDevAttrMaxAccessPolicyWindowSize, dev);
    return (int64_t)(a < b ? a : b);
}

extern "C" int hg_set_l2_persist(const void* base, int64_t bytes, float hit_ratio) {
    if (!base || bytes <= 0) {
        g_l2_base = nullptr;
        g_l2_bytes = 0;
        cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, 0);
        return hg_check_launch("set_l2_persist(off)");
    }
    const int64_t mx = hg_l2_persist_max();
    if (mx <= 0) { hg_set_error("set_l2_persist: device has no persisting L2"); return HG_EUNSUPPORTED; }
    if (bytes > mx) bytes = mx;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)bytes) != cudaSuccess)
        return hg_check_launch("set_l2_persist");
    g_l2_base = base;
    g_l2_bytes = (size_t)bytes;
    g_l2_hit = hit_ratio < 0.f ? 0.f : (hit_ratio > 1.f ? 1.f : hit_ratio);
    return HG_OK;
}

// PDL switch (hg_set_tuning key 5; env HG_PDL=0 turns it off at load)
namespace {
int g_pdl = -1;
}
bool hg_pdl_enabled() {
    if (g_pdl < 0) {
        const char* e = getenv("HG_PDL");
        g_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    return g_pdl == 1;
}
void hg_set_pdl(int v) { g_pdl = v ? 1 : 0; }

// ---------------------------------------------------------------------------
// CUDA IPC: export / import device allocations between the per-GPU processes
// (NVLink peer pointers for the row-sharded feature table)
// ---------------------------------------------------------------------------
// The handle names the whole allocation (a caching allocator may sub-allocate):
// *out_offset = dptr - allocation base, to add to the importer's mapping.
extern "C" int hg_ipc_get_handle(const void* dptr, uint8_t* out_handle64, int64_t* out_offset) {
    typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = nullptr;
    if (!range) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            range = reinterpret_cast<RangeFn>(p);
    }
    if (!range) { hg_set_error("ipc_get_handle: cuMemGetAddressRange unavailable"); return HG_ECUDA; }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)dptr) != CUDA_SUCCESS) { hg_set_error("ipc_get_handle: address range"); return HG_ECUDA; }
    cudaIpcMemHandle_t h;
    if (cudaIpcGetMemHandle(&h, (void*)base) != cudaSuccess) return hg_check_launch("ipc_get_handle");
    memcpy(out_handle64, &h, sizeof(h));
    *out_offset = (int64_t)((CUdeviceptr)dptr - base);
    return HG_OK;
}

extern "C" int hg_ipc_open_handle(const uint8_t* handle64, void** out_ptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    if (cudaIpcOpenMemHandle(out_ptr, h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess)
        return hg_check_launch("ipc_open_handle");
    return HG_OK;
}

extern "C" int hg_ipc_close(void* ptr) {
    if (cudaIpcCloseMemHandle(ptr) != cudaSuccess) return hg_check_launch("ipc_close");
    return HG_OK;
}

extern "C" int hg_enable_peer_access(int32_t peer_device) {
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e == cudaSuccess || e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
        return HG_OK;
    }
    return hg_check_launch("enable_peer_access");
}

// ---------------------------------------------------------------------------
// Device-to-device copy of a small buffer as a kernel node (the per-batch input
// block the sample half hands to the train half): inside a captured graph a
// kernel node chains like its neighbours, a memcpy node does not.
// ---------------------------------------------------------------------------
namespace {
__global__ void k_copy_words(uint4* __restrict__ dst, const uint4* __restrict__ src, int64_t n16,
                             uint8_t* __restrict__ dtail, const uint8_t* __restrict__ stail, int tail) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
    if (blockIdx.x == 0 && threadIdx.x < tail) dtail[threadIdx.x] = stail[threadIdx.x];
}
}  // namespace

extern "C" int hg_copy_bytes(void* dst, const void* src, int64_t nbytes, void* stream) {
    if (nbytes <= 0) return HG_OK;
    if ((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src)) & 15) {
        hg_set_error("copy_bytes: dst and src must be 16-byte aligned");
        return HG_EINVAL;
    }
    const int64_t n16 = nbytes / 16;
    const int tail = (int)(nbytes - n16 * 16);
    const int grid = (int)((n16 + 255) / 256) < 1 ? 1 : (int)((n16 + 255) / 256);
    k_copy_words<<<grid < 64 ? grid : 64, 256, 0, (cudaStream_t)stream>>>(
        (uint4*)dst, (const uint4*)src, n16, (uint8_t*)dst + n16 * 16, (const uint8_t*)src + n16 * 16, tail);
    return hg_check_launch("copy_bytes");
}
