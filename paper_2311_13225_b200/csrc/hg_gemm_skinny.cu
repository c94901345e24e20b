// K8, latency path: fp32 SIMT kernels for the SMALL dense transforms of the
// upper layers (M = a few thousand destination rows, K, N <= 128).
//
// At those sizes a tensor-core tile pipeline is a serial chain per CTA (TMA ->
// split -> 96 MMAs -> epilogue) spread over only M/128 SMs, ~8 us however fast
// its stages are.  These kernels spread the same work over many warps with
// short dependency chains instead:
//
//   k_gemm_skinny   one warp per 2 output rows; the CTA decodes op(B) once from
//                   the tensor-core B image (its "hi" words are the exact fp32
//                   weights) into shared memory; each lane owns columns
//                   lane + 32 j and accumulates over k in order (fp32 FMA).
//   k_wgrad_skinny  CTA = (64-row chunk, source): the chunk's A and G rows in
//                   shared memory, every thread a float4 of outputs for a strided
//                   set of k; partials reduced over chunks in a fixed order.
//
// Same contracts and determinism as hg_gemm_tc / hg_wgrad_tc (which dispatch
// here when M_cap <= HG_SKINNY_MAX_M and K, N <= 128).
#include "hg_common.cuh"
#include "hg_gnn_internal.h"
#include "hg_tc.cuh"

namespace {
using namespace hgtc;

constexpr int SK_THREADS = 256;
constexpr int SK_RPW = 2;      // output rows per warp (fwd)
constexpr int WG_R = 64;       // rows per wgrad chunk

// Decode op(B) (its hi words) from the B image (hg_gemm_tc_prep_b) into a plain
// [K][NP] shared array: the image is read linearly (coalesced, 8 words in
// flight per thread) and each word's (n, k) recovered by inverting the
// K-major SWIZZLE_128B offset; tile (nt, kt) = hi words of BN columns x 32 k.
__device__ __forceinline__ void decode_b(const uint8_t* __restrict__ img, int K1, int K2, int nk1, int nk, int n_nt,
                                         int bn, int N, float* sB, int NP) {
    const int words_per_tile = bn * 32;
    const int total = n_nt * nk * words_per_tile;
    for (int e0 = threadIdx.x; e0 < total; e0 += 8 * SK_THREADS) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * SK_THREADS;
            v[u] = 0.f;
            if (e < total) {
                const int tile = e / words_per_tile, w = e - tile * words_per_tile;
                v[u] = *reinterpret_cast<const float*>(img + (int64_t)tile * (2 * bn * 128) + w * 4);
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * SK_THREADS;
            if (e >= total) break;
            const int tile = e / words_per_tile, w = e - tile * words_per_tile;
            const int nt = tile / nk, kt = tile - nt * nk;
            const int o = w * 4;
            const int r = ((o >> 10) << 3) + ((o >> 7) & 7);
            const int c = ((o >> 4) & 7) ^ (r & 7);
            const int kk = c * 4 + ((o >> 2) & 3);
            const int n = nt * bn + r;
            int k;
            if (kt < nk1) {
                k = kt * 32 + kk;
                if (k >= K1) continue;  // zero padding of source 1's last tile
            } else {
                const int k2 = (kt - nk1) * 32 + kk;
                if (k2 >= K2) continue;
                k = K1 + k2;
            }
            if (n < NP) sB[k * NP + n] = n < N ? v[u] : 0.f;
        }
    }
}

// C[M x N] = act(A1 op(B)[:K1] + A2 op(B)[K1:]); NPL = columns per lane (N <= 32 NPL),
// KC = 32-wide k chunks per source held in registers (K1, K2 <= 32 KC).
// Persistent CTAs: B decoded once per CTA, warps stride over row pairs.
template <int NPL, int KC>
__global__ void __launch_bounds__(SK_THREADS) k_gemm_skinny(
    const float* __restrict__ A1, int lda1, int K1, const float* __restrict__ A2, int lda2, int K2,
    const uint8_t* __restrict__ img, int bn, int nk1, int nk, int n_nt, float* __restrict__ C, int ldc, int N,
    const int* __restrict__ d_M, int M_cap, int act) {
    constexpr int NP = 32 * NPL;
    extern __shared__ float sB[];  // [K1 + K2][NP]
    const int M = hg_load_count(d_M, M_cap);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if ((int)blockIdx.x * (SK_THREADS / 32) * SK_RPW >= M) return;
    decode_b(img, K1, K2, nk1, nk, n_nt, bn, N, sB, NP);
    __syncthreads();
    const int row_stride = gridDim.x * (SK_THREADS / 32) * SK_RPW;
    for (int row0 = (blockIdx.x * (SK_THREADS / 32) + warp) * SK_RPW; row0 < M; row0 += row_stride) {
        float acc[SK_RPW][NPL];
#pragma unroll
        for (int r = 0; r < SK_RPW; ++r)
#pragma unroll
            for (int j = 0; j < NPL; ++j) acc[r][j] = 0.f;
#pragma unroll
        for (int src = 0; src < 2; ++src) {
            const float* A = src ? A2 : A1;
            const int Ks = src ? K2 : K1, lda = src ? lda2 : lda1, kb = src ? K1 : 0;
            if (!A || Ks <= 0) continue;
            float a[SK_RPW][KC];  // lane holds A[row][c*32 + lane]
#pragma unroll
            for (int r = 0; r < SK_RPW; ++r) {
                const int row = row0 + r;
#pragma unroll
                for (int c = 0; c < KC; ++c) {
                    const int k = c * 32 + lane;
                    a[r][c] = (row < M && k < Ks) ? __ldg(A + (int64_t)row * lda + k) : 0.f;
                }
            }
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                if (c * 32 >= Ks) break;
                const int kend = min(32, Ks - c * 32);
#pragma unroll 4
                for (int kk = 0; kk < kend; ++kk) {
                    const float* brow = sB + (kb + c * 32 + kk) * NP + lane;
                    float b[NPL];
#pragma unroll
                    for (int j = 0; j < NPL; ++j) b[j] = brow[32 * j];
#pragma unroll
                    for (int r = 0; r < SK_RPW; ++r) {
                        const float av = __shfl_sync(0xffffffffu, a[r][c], kk);
#pragma unroll
                        for (int j = 0; j < NPL; ++j) acc[r][j] = fmaf(av, b[j], acc[r][j]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < SK_RPW; ++r) {
            const int row = row0 + r;
            if (row >= M) break;
#pragma unroll
            for (int j = 0; j < NPL; ++j) {
                const int n = lane + 32 * j;
                if (n < N) C[(int64_t)row * ldc + n] = act ? fmaxf(acc[r][j], 0.f) : acc[r][j];
            }
        }
    }
}

// partial[src][chunk][K x N] = A_src[chunk rows]^T G[chunk rows]; KPT = max k per thread
template <int KPT>
__global__ void __launch_bounds__(SK_THREADS) k_wgrad_skinny(
    const float* __restrict__ A1, int lda1, const float* __restrict__ A2, int lda2, int K,
    const float* __restrict__ G, int ldg, int N, const int* __restrict__ d_M, int M_cap, float* __restrict__ partial,
    int n_chunks) {
    extern __shared__ float sm[];
    const int N4 = (N + 3) >> 2, NP = N4 * 4;
    const int K4 = (K + 3) >> 2, KP = K4 * 4;
    float* sA = sm;              // [WG_R][KP]
    float* sG = sm + WG_R * KP;  // [WG_R][NP]
    const int M = hg_load_count(d_M, M_cap);
    const int chunk = blockIdx.x, src = blockIdx.y;
    const int m0 = chunk * WG_R;
    if (m0 >= M) return;
    const int rows = min(WG_R, M - m0);
    const float* A = src ? A2 : A1;
    const int lda = src ? lda2 : lda1;
    // 16-byte loads, 4 in flight per thread (row strides are multiples of 4 floats)
    const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int e0 = threadIdx.x; e0 < WG_R * K4; e0 += 4 * SK_THREADS) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * SK_THREADS;
            const int r = e / K4, c = e - r * K4;
            v[u] = (e < WG_R * K4 && r < rows) ? __ldg(reinterpret_cast<const float4*>(A + (int64_t)(m0 + r) * lda) + c) : z4;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * SK_THREADS;
            if (e >= WG_R * K4) break;
            const int r = e / K4, c = e - r * K4;
            float4 w = v[u];
            if (c * 4 + 3 >= K) {  // padding columns of the last chunk
                if (c * 4 + 1 >= K) w.y = 0.f;
                if (c * 4 + 2 >= K) w.z = 0.f;
                if (c * 4 + 3 >= K) w.w = 0.f;
            }
            *reinterpret_cast<float4*>(sA + r * KP + c * 4) = w;
        }
    }
    for (int e0 = threadIdx.x; e0 < WG_R * N4; e0 += 4 * SK_THREADS) {
        float4 v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * SK_THREADS;
            const int r = e / N4, c = e - r * N4;
            v[u] = (e < WG_R * N4 && r < rows) ? __ldg(reinterpret_cast<const float4*>(G + (int64_t)(m0 + r) * ldg) + c) : z4;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int e = e0 + u * SK_THREADS;
            if (e >= WG_R * N4) break;
            const int r = e / N4, c = e - r * N4;
            float4 w = v[u];
            if (c * 4 + 3 >= N) {
                if (c * 4 + 1 >= N) w.y = 0.f;
                if (c * 4 + 2 >= N) w.z = 0.f;
                if (c * 4 + 3 >= N) w.w = 0.f;
            }
            *reinterpret_cast<float4*>(sG + r * NP + c * 4) = w;
        }
    }
    __syncthreads();
    const int KG = SK_THREADS / N4;
    const int t = threadIdx.x;
    if (t >= KG * N4) return;
    const int n4 = t % N4, kg = t / N4;
    float4 acc[KPT];
#pragma unroll
    for (int i = 0; i < KPT; ++i) acc[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int r = 0; r < rows; ++r) {
        const float4 g = *reinterpret_cast<const float4*>(sG + r * NP + n4 * 4);
        const float* ar = sA + r * KP;
#pragma unroll
        for (int i = 0; i < KPT; ++i) {
            const int k = kg + i * KG;
            if (k < K) {
                const float a = ar[k];
                acc[i].x = fmaf(a, g.x, acc[i].x);
                acc[i].y = fmaf(a, g.y, acc[i].y);
                acc[i].z = fmaf(a, g.z, acc[i].z);
                acc[i].w = fmaf(a, g.w, acc[i].w);
            }
        }
    }
    float* P = partial + ((int64_t)src * n_chunks + chunk) * (int64_t)K * N;
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
        const int k = kg + i * KG;
        if (k >= K) break;
        float* p = P + (int64_t)k * N + n4 * 4;
        const float v[4] = {acc[i].x, acc[i].y, acc[i].z, acc[i].w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (n4 * 4 + q < N) p[q] = v[q];
    }
}

// out_s = sum over the active chunks (ceil(M / WG_R)) in chunk order, then the
// 8 warp sums in order: deterministic.
__global__ void __launch_bounds__(256) k_wgrad_skinny_reduce(const float* __restrict__ partial, int KN, int n_chunks,
                                                             const int* __restrict__ d_M, int M_cap,
                                                             float* __restrict__ out1, float* __restrict__ out2) {
    __shared__ float s_part[8][33];
    const int M = hg_load_count(d_M, M_cap);
    const int chunks = (M + WG_R - 1) / WG_R;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per_src = (KN + 31) / 32;
    const int s = blockIdx.x / per_src;
    const int e = (blockIdx.x - s * per_src) * 32 + lane;
    float acc = 0.f;
    if (e < KN) {
        const float* p = partial + (int64_t)s * n_chunks * KN + e;
        for (int c = w; c < chunks; c += 8) acc += p[(int64_t)c * KN];
    }
    s_part[w][lane] = acc;
    __syncthreads();
    if (w == 0 && e < KN) {
        float t = 0.f;
#pragma unroll
        for (int k = 0; k < 8; ++k) t += s_part[k][lane];
        (s ? out2 : out1)[e] = t;
    }
}

template <int NPL, int KC>
int launch_skinny(int M_cap, cudaStream_t s, const float* A1, int lda1, int K1, const float* A2, int lda2, int K2,
                  const uint8_t* img, int bn, int nk1, int nk, float* C, int ldc, int N, const int* d_M, int act) {
    const int smem = (K1 + K2) * 32 * NPL * 4;
    static int attr = 0;
    if (smem > 48 * 1024 && attr < smem) {
        cudaFuncSetAttribute(k_gemm_skinny<NPL, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        attr = 128 * 1024;
    }
    const int rows_per_cta = (SK_THREADS / 32) * SK_RPW;
    int grid = hg_ceil_div(M_cap, rows_per_cta);
    grid = grid < 2 * HG_NUM_SMS ? grid : 2 * HG_NUM_SMS;
    k_gemm_skinny<NPL, KC><<<grid, SK_THREADS, smem, s>>>(A1, lda1, K1, A2, lda2, K2, img, bn, nk1, nk,
                                                          hg_ceil_div(N, bn), C, ldc, N, d_M, M_cap, act);
    return hg_check_launch("gemm_skinny");
}

}  // namespace

bool hg_skinny_gemm_ok(int M_cap, int K1, int K2, int N) {
    return M_cap <= HG_SKINNY_MAX_M && K1 <= 128 && K2 <= 128 && N <= 128;
}

bool hg_skinny_wgrad_ok(int M_cap, int K, int N) { return M_cap <= HG_SKINNY_MAX_M && K <= 128 && N <= 128; }
// (callers guarantee row strides that are multiples of 4 floats and 16-byte aligned rows)

int hg_gemm_skinny_launch(const float* A1, int lda1, int K1, const float* A2, int lda2, int K2, const uint8_t* img,
                          float* C, int ldc, int N, const int* d_M, int M_cap, int act, cudaStream_t s) {
    const int bn = hg_tma_gemm_bn(N);
    const int nk1 = hg_ceil_div(K1, 32);
    const int k2 = (A2 && K2 > 0) ? K2 : 0;
    const int nk = nk1 + (k2 ? hg_ceil_div(k2, 32) : 0);
    const int npl = N <= 32 ? 1 : N <= 64 ? 2 : 4;
    const int kc = (K1 > k2 ? K1 : k2) <= 64 ? 2 : 4;
#define HG_SK(NPL, KC) \
    return launch_skinny<NPL, KC>(M_cap, s, A1, lda1, K1, k2 ? A2 : nullptr, lda2, k2, img, bn, nk1, nk, C, ldc, N, d_M, act)
    if (npl == 1) { if (kc == 2) HG_SK(1, 2); HG_SK(1, 4); }
    if (npl == 2) { if (kc == 2) HG_SK(2, 2); HG_SK(2, 4); }
    if (kc == 2) HG_SK(4, 2);
    HG_SK(4, 4);
#undef HG_SK
}

int64_t hg_wgrad_skinny_ws_floats(int K, int N, int M_cap, int n_src) {
    return (int64_t)n_src * hg_ceil_div(M_cap > 0 ? M_cap : 1, WG_R) * K * N;
}

int hg_wgrad_skinny_launch(const float* A1, int lda1, const float* A2, int lda2, int K, const float* G, int ldg, int N,
                           const int* d_M, int M_cap, float* out1, float* out2, float* ws, cudaStream_t s) {
    const int n_src = A2 ? 2 : 1;
    const int n_chunks = hg_ceil_div(M_cap > 0 ? M_cap : 1, WG_R);
    const int N4 = (N + 3) / 4;
    const int KG = SK_THREADS / N4;
    const int kpt = hg_ceil_div(K, KG);
    const int smem = (WG_R * ((K + 3) / 4) * 4 + WG_R * N4 * 4) * 4;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_wgrad_skinny<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_wgrad_skinny<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        cudaFuncSetAttribute(k_wgrad_skinny<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
        attr = true;
    }
    if (M_cap > 0) {
        dim3 grid(n_chunks, n_src);
        if (kpt <= 4) k_wgrad_skinny<4><<<grid, SK_THREADS, smem, s>>>(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, ws, n_chunks);
        else if (kpt <= 8) k_wgrad_skinny<8><<<grid, SK_THREADS, smem, s>>>(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, ws, n_chunks);
        else k_wgrad_skinny<16><<<grid, SK_THREADS, smem, s>>>(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, ws, n_chunks);
        int rc = hg_check_launch("wgrad_skinny");
        if (rc) return rc;
    }
    k_wgrad_skinny_reduce<<<n_src * hg_ceil_div((long long)K * N, 32), 256, 0, s>>>(ws, K * N, n_chunks, d_M, M_cap,
                                                                                   out1, out2);
    return hg_check_launch("wgrad_skinny_reduce");
}
