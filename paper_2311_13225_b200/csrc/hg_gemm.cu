// K8 (portable path): fp32 SIMT GEMMs for the dense layer transforms.
//
//   forward   Z  = act(A1 B1 + A2 B2)        SAGE: [h_self | mean] [W_self; W_neigh]
//                                            GCN : agg W           (gnnmath.py:121,173)
//   backward  dA = dZ W^T                    (gnnmath.py:139,194-198)
//             dW = A^T dZ  (split-M, fixed-order reduction; gnnmath.py:135,190-191)
//
// M (rows = destinations) is read from device memory so the kernels can sit in
// a captured CUDA graph.  This is the correctness baseline and the fallback for
// shapes the tcgen05 path (hg_gemm_tc.cu) does not take; both are deterministic.
#include "hg_common.cuh"
#include "hg_gnn_internal.h"

namespace {
constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <bool TRANS_B>
__device__ __forceinline__ void gemm_accumulate(const float* __restrict__ A, int lda, int K,
                                                const float* __restrict__ B, int ldb, int N, int m0, int n0,
                                                int M, float (&acc)[4][4], float (*As)[BM + 4],
                                                float (*Bs)[BN + 4]) {
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    for (int k0 = 0; k0 < K; k0 += BK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + q * NT;
            const int r = e >> 4, c = e & 15;  // A tile: 64 rows x 16 k
            const int gm = m0 + r, gk = k0 + c;
            As[c][r] = (gm < M && gk < K) ? __ldg(A + (int64_t)gm * lda + gk) : 0.f;
            const int kb = e >> 6, nb = e & 63;  // B tile: 16 k x 64 n
            const int bk = k0 + kb, bn = n0 + nb;
            float bv = 0.f;
            if (bk < K && bn < N) bv = TRANS_B ? __ldg(B + (int64_t)bn * ldb + bk) : __ldg(B + (int64_t)bk * ldb + bn);
            Bs[kb][nb] = bv;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < BK; ++kk) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
}

template <bool TRANS_B>
__global__ void __launch_bounds__(NT) k_gemm(const float* __restrict__ A1, int lda1, int K1,
                                             const float* __restrict__ B1, int ldb1, const float* __restrict__ A2,
                                             int lda2, int K2, const float* __restrict__ B2, int ldb2,
                                             float* __restrict__ C, int ldc, int N, const int* d_M, int M_cap,
                                             int act) {
    __shared__ float As[BK][BM + 4];
    __shared__ float Bs[BK][BN + 4];
    const int M = hg_load_count(d_M, M_cap);
    const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
    if (m0 >= M) return;
    float acc[4][4] = {};
    gemm_accumulate<TRANS_B>(A1, lda1, K1, B1, ldb1, N, m0, n0, M, acc, As, Bs);
    if (A2) gemm_accumulate<TRANS_B>(A2, lda2, K2, B2, ldb2, N, m0, n0, M, acc, As, Bs);
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty * 4 + i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int nn = n0 + tx * 4 + j;
            if (nn < N) C[(int64_t)m * ldc + nn] = act ? fmaxf(acc[i][j], 0.f) : acc[i][j];
        }
    }
}

// partial[c] = A[rows of chunk c]^T G[rows of chunk c]   (K x N per chunk)
constexpr int MC = 512;  // rows per chunk
__global__ void __launch_bounds__(NT) k_wgrad_partial(const float* __restrict__ A, int lda, int K,
                                                      const float* __restrict__ G, int ldg, int N, const int* d_M,
                                                      int M_cap, float* __restrict__ partial) {
    __shared__ float As[BK][BM + 4];  // [m][k]
    __shared__ float Gs[BK][BN + 4];  // [m][n]
    const int M = hg_load_count(d_M, M_cap);
    const int k0 = blockIdx.x * BM, n0 = blockIdx.y * BN, c = blockIdx.z;
    const int mbeg = c * MC;
    if (mbeg >= M) return;
    const int mend = min(M, mbeg + MC);
    const int t = threadIdx.x, tx = t & 15, ty = t >> 4;
    float acc[4][4] = {};
    for (int ms = mbeg; ms < mend; ms += BK) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int e = t + q * NT;
            const int r = e >> 6, col = e & 63;  // 16 m x 64 cols
            const int gm = ms + r;
            As[r][col] = (gm < mend && k0 + col < K) ? __ldg(A + (int64_t)gm * lda + k0 + col) : 0.f;
            Gs[r][col] = (gm < mend && n0 + col < N) ? __ldg(G + (int64_t)gm * ldg + n0 + col) : 0.f;
        }
        __syncthreads();
#pragma unroll
        for (int mm = 0; mm < BK; ++mm) {
            float a[4], b[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[mm][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) b[j] = Gs[mm][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
        }
        __syncthreads();
    }
    float* P = partial + (int64_t)c * K * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int k = k0 + ty * 4 + i;
        if (k >= K) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int nn = n0 + tx * 4 + j;
            if (nn < N) P[(int64_t)k * N + nn] = acc[i][j];
        }
    }
}

__global__ void k_wgrad_reduce(const float* __restrict__ partial, int KN, const int* d_M, int M_cap,
                               float* __restrict__ out, float scale) {
    const int M = hg_load_count(d_M, M_cap);
    const int chunks = (M + MC - 1) / MC;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < KN; idx += gridDim.x * blockDim.x) {
        float s = 0.f;
        for (int c = 0; c < chunks; ++c) s += partial[(int64_t)c * KN + idx];
        out[idx] = s * scale;
    }
}
}  // namespace

// C[M x N] = act(A1[M x K1] op(B1) + A2[M x K2] op(B2)); op(B) = B ([K x N], ldb)
// or, with trans_b, B^T where B is stored [N x K] (ldb).  A2/B2 may be null.
extern "C" int hg_gemm_f32(const float* A1, int32_t lda1, int32_t K1, const float* B1, int32_t ldb1,
                           const float* A2, int32_t lda2, int32_t K2, const float* B2, int32_t ldb2,
                           int32_t trans_b, float* C, int32_t ldc, int32_t N, const int32_t* d_M, int32_t M_cap,
                           int32_t act, void* stream) {
    if (M_cap <= 0 || N <= 0) return HG_OK;
    dim3 grid(hg_ceil_div(M_cap, BM), hg_ceil_div(N, BN));
    cudaStream_t s = (cudaStream_t)stream;
    if (trans_b)
        k_gemm<true><<<grid, NT, 0, s>>>(A1, lda1, K1, B1, ldb1, A2, lda2, K2, B2, ldb2, C, ldc, N, d_M, M_cap, act);
    else
        k_gemm<false><<<grid, NT, 0, s>>>(A1, lda1, K1, B1, ldb1, A2, lda2, K2, B2, ldb2, C, ldc, N, d_M, M_cap, act);
    return hg_check_launch("gemm_f32");
}

extern "C" int64_t hg_wgrad_ws_size(int32_t K, int32_t N, int32_t M_cap) {
    return (int64_t)hg_ceil_div(M_cap > 0 ? M_cap : 1, MC) * K * N;
}

// out[K x N] = scale * A[M x K]^T G[M x N]; deterministic split-M.
// ws: >= hg_wgrad_ws_size(K, N, M_cap) floats.
extern "C" int hg_wgrad_f32(const float* A, int32_t lda, int32_t K, const float* G, int32_t ldg, int32_t N,
                            const int32_t* d_M, int32_t M_cap, float* out, float scale, float* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (K <= 0 || N <= 0) return HG_OK;
    const int chunks = hg_ceil_div(M_cap > 0 ? M_cap : 1, MC);
    dim3 grid(hg_ceil_div(K, BM), hg_ceil_div(N, BN), chunks);
    if (M_cap > 0) k_wgrad_partial<<<grid, NT, 0, s>>>(A, lda, K, G, ldg, N, d_M, M_cap, ws);
    k_wgrad_reduce<<<hg_grid((long long)K * N, 256, 4), 256, 0, s>>>(ws, K * N, d_M, M_cap, out, scale);
    return hg_check_launch("wgrad_f32");
}
