// K8: the dense layer transforms on the 5th-generation tensor cores (tcgen05).
//
//   hg_gemm_tc   C[M x N] = act(A1 op(B)[:K1] + A2 op(B)[K1:])   (fwd; dX = dZ W^T)
//   hg_wgrad_tc  dW_s[K x N] = A_s^T G  (s = 1, 2; split-M, fixed-order reduction)
//
// fp32 accuracy from tf32 tensor cores ("3xTF32"): every operand x is fed as
// x (the MMA reads its top 19 bits, i.e. hi = trunc_tf32(x)) and lo = x - hi
// (exact in fp32), and D += A_hi B_hi + A_hi B_lo + A_lo B_hi, so the product
// error is ~2^-21 relative instead of tf32's 2^-10.  The GEMMs here are small
// and HBM-bound (K <= 2F, N <= 256), so the 3x MMA count is free.
//
#include "hg_common.cuh"
#ifndef HG_GEMM_MAX_BN
#define HG_GEMM_MAX_BN 128  // widest N tile of the forward / dX GEMMs: wider N runs as several 128-wide TS-form
                            // N tiles (C3: 3.61 -> 3.82 M seeds/s vs one 256-wide SS-form tile, 2 stages)
#endif
#include "hg_gnn_internal.h"
#include "hg_tc.cuh"

namespace {
using namespace hgtc;

int g_mn_swap = 0;  // tuning knob (hg_set_tuning key 1): MN-major descriptor offset assignment

// ---------------------------------------------------------------------------
// Several B images in one launch (blockIdx.z = image): the per-step rebuild of
// every layer's forward / dX images costs one kernel node instead of five.
struct PrepDesc {
    const float* B;
    uint8_t* img;
    int ldb, trans_b, K1, K2, N, bn, nk1, nk, nnt;
};
constexpr int MAX_PREP = 8;
struct PrepBatch {
    PrepDesc d[MAX_PREP];
};

__global__ void k_prep_b_many(const __grid_constant__ PrepBatch pb) {
    const PrepDesc& d = pb.d[blockIdx.z];
    const int kt = blockIdx.x, nt = blockIdx.y;
    if (kt >= d.nk || nt >= d.nnt) return;
    const int BN = d.bn;
    uint8_t* base = d.img + ((int64_t)nt * d.nk + kt) * (2 * BN * 128);
    const int K = kt < d.nk1 ? d.K1 : d.K2;
    const int k0 = kt < d.nk1 ? kt * 32 : (kt - d.nk1) * 32;
    const int kb = kt < d.nk1 ? k0 : d.K1 + k0;
    for (int e = threadIdx.x; e < BN * 32; e += blockDim.x) {
        int n, k;
        if (d.trans_b) { k = e / BN; n = e - k * BN; }
        else { n = e >> 5; k = e & 31; }
        const int gn = nt * BN + n, gk = k0 + k;
        float v = 0.f;
        if (gn < d.N && gk < K)
            v = d.trans_b ? d.B[(int64_t)(kb + k) * d.ldb + gn] : d.B[(int64_t)gn * d.ldb + kb + k];
        const uint32_t off = off_k(n, k >> 2) + (k & 3) * 4;
        *reinterpret_cast<float*>(base + off) = v;
        *reinterpret_cast<float*>(base + BN * 128 + off) = tf32_lo(v);
    }
}

// ---------------------------------------------------------------------------
// One launch at the end of a training step: SGD on the flat parameter buffer
// (gnnmath.py:277-283) + max |w_new - w_old| (orchestrator.py:246-255), the
// tensor-core B images of the UPDATED weights written in the same pass (each
// weight lands at its swizzled hi/lo positions of every image built from it;
// padding positions were zeroed by the initial full build and never change),
// and — by the last block to finish — the per-batch record (loss, max delta
// into the epoch arrays, orchestrator.py:527-544).  Replaces hg_sgd +
// hg_gemm_tc_prep_b_many + hg_record_batch (three dependent launches).
__device__ __forceinline__ void img_put(const PrepDesc& d, int64_t e, float v) {
    const int64_t rows_ld = (int64_t)d.ldb;
    const int row = (int)(e / rows_ld), col = (int)(e - (int64_t)row * rows_ld);
    int k, n;
    if (d.trans_b) { k = row; n = col; } else { n = row; k = col; }
    if (n >= d.N || k >= d.K1 + d.K2) return;
    int kt, kk;
    if (k < d.K1) { kt = k >> 5; kk = k & 31; }
    else { const int k2 = k - d.K1; kt = d.nk1 + (k2 >> 5); kk = k2 & 31; }
    const int nt = n / d.bn, nn = n - nt * d.bn;
    uint8_t* base = d.img + ((int64_t)nt * d.nk + kt) * (2 * d.bn * 128);
    const uint32_t off = off_k(nn, kk >> 2) + (kk & 3) * 4;
    *reinterpret_cast<float*>(base + off) = v;
    *reinterpret_cast<float*>(base + d.bn * 128 + off) = tf32_lo(v);
}

struct FusedImages {
    PrepDesc d[MAX_PREP];
    int64_t lo[MAX_PREP], hi[MAX_PREP];  // [lo, hi): flat weight indices each image is built from
};

__global__ void __launch_bounds__(256) k_sgd_fused(const __grid_constant__ FusedImages pb, int n_img,
                                                   float* __restrict__ w, const float* __restrict__ g, long long n,
                                                   float lr, unsigned* __restrict__ ctl, const int64_t* __restrict__ bp,
                                                   const float* __restrict__ d_loss, float* __restrict__ loss_arr,
                                                   float* __restrict__ md_arr) {
    hg_pdl_begin();
    __shared__ float s_m[8];
    __shared__ bool s_last;
    float md = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float old = w[i];
        const float nw = old - lr * g[i];
        w[i] = nw;
        md = fmaxf(md, fabsf(nw - old));
        for (int j = 0; j < n_img; ++j)
            if (i >= pb.lo[j] && i < pb.hi[j]) img_put(pb.d[j], i - pb.lo[j], nw);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) md = fmaxf(md, __shfl_xor_sync(0xffffffffu, md, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = md;
    __syncthreads();
    if (threadIdx.x == 0) {
        float m = 0.f;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) m = fmaxf(m, s_m[k]);
        atomicMax(&ctl[0], __float_as_uint(m));  // non-negative floats order like their bits
        __threadfence();
        s_last = atomicAdd(&ctl[1], 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
        __threadfence();
        const int bi = (int)bp[3];  // BP_BATCH_IN_EPOCH
        loss_arr[bi] = *d_loss;
        md_arr[bi] = __uint_as_float(atomicExch(&ctl[0], 0u));
        ctl[1] = 0u;
    }
}

// B image: for every (N tile, K tile) the exact swizzled smem bytes of the
// operand tile, hi then lo (2 * BN * 128 bytes), so CTAs stage B with plain
// 16-byte cp.async copies.  Built once per weight update by k_prep_b.
template <int BN>
__global__ void k_prep_b(const float* __restrict__ B, int ldb, int trans_b, int K1, int K2, int N, int nk1, int nk,
                         uint8_t* __restrict__ img) {
    const int nt = blockIdx.y, kt = blockIdx.x;
    uint8_t* base = img + ((int64_t)nt * nk + kt) * (2 * BN * 128);
    const int K = kt < nk1 ? K1 : K2;
    const int k0 = kt < nk1 ? kt * 32 : (kt - nk1) * 32;
    const int kb = kt < nk1 ? k0 : K1 + k0;
    for (int e = threadIdx.x; e < BN * 32; e += blockDim.x) {
        int n, k;
        if (trans_b) { k = e / BN; n = e - k * BN; }
        else { n = e >> 5; k = e & 31; }
        const int gn = nt * BN + n, gk = k0 + k;
        float v = 0.f;
        if (gn < N && gk < K) v = trans_b ? B[(int64_t)(kb + k) * ldb + gn] : B[(int64_t)gn * ldb + kb + k];
        const uint32_t off = off_k(n, k >> 2) + (k & 3) * 4;
        *reinterpret_cast<float*>(base + off) = v;
        *reinterpret_cast<float*>(base + BN * 128 + off) = tf32_lo(v);
    }
}


int gemm_bn(int N) {
    const int Nr = (N + 15) & ~15;
    return Nr <= 32 ? 32 : Nr <= 64 ? 64 : (Nr <= 128 || HG_GEMM_MAX_BN <= 128) ? 128 : 256;
}


}  // namespace

// Byte size of the B operand image for (K1, K2, N).
extern "C" int64_t hg_gemm_tc_bimg_size(int32_t K1, int32_t K2, int32_t N) {
    const int bn = gemm_bn(N);
    const int nk = hg_ceil_div(K1, 32) + (K2 > 0 ? hg_ceil_div(K2, 32) : 0);
    return (int64_t)hg_ceil_div(N, bn) * nk * 2 * bn * 128;
}

// Build the B image: op(B)(k, n) = B[k*ldb + n] with trans_b (B stored
// [K x N], the forward weights [W_self; W_neigh]) or B[n*ldb + k] without (B
// stored [N x K], dX = dZ W^T); rows K1.. of op(B) feed the second A source.
extern "C" int hg_gemm_tc_prep_b(const float* B, int32_t ldb, int32_t trans_b, int32_t K1, int32_t K2, int32_t N,
                                 void* img, void* stream) {
    if (N <= 0 || K1 <= 0) return HG_OK;
    const int bn = gemm_bn(N);
    const int nk1 = hg_ceil_div(K1, 32);
    const int nk = nk1 + (K2 > 0 ? hg_ceil_div(K2, 32) : 0);
    dim3 g(nk, hg_ceil_div(N, bn));
    cudaStream_t s = (cudaStream_t)stream;
    uint8_t* p = (uint8_t*)img;
    switch (bn) {
        case 32: k_prep_b<32><<<g, 256, 0, s>>>(B, ldb, trans_b, K1, K2, N, nk1, nk, p); break;
        case 64: k_prep_b<64><<<g, 256, 0, s>>>(B, ldb, trans_b, K1, K2, N, nk1, nk, p); break;
        case 128: k_prep_b<128><<<g, 256, 0, s>>>(B, ldb, trans_b, K1, K2, N, nk1, nk, p); break;
        default: k_prep_b<256><<<g, 256, 0, s>>>(B, ldb, trans_b, K1, K2, N, nk1, nk, p); break;
    }
    return hg_check_launch("gemm_tc_prep_b");
}

// Batched hg_gemm_tc_prep_b: host_desc holds n rows of 7 int64
// (B, ldb, trans_b, K1, K2, N, img); n <= 8.
extern "C" int hg_gemm_tc_prep_b_many(int32_t n, const int64_t* host_desc, void* stream) {
    if (n <= 0) return HG_OK;
    if (n > MAX_PREP) { hg_set_error("gemm_tc_prep_b_many: at most %d images", MAX_PREP); return HG_EINVAL; }
    PrepBatch pb{};
    int gx = 1, gy = 1;
    for (int i = 0; i < n; ++i) {
        const int64_t* r = host_desc + 7 * i;
        PrepDesc& d = pb.d[i];
        d.B = reinterpret_cast<const float*>(r[0]);
        d.ldb = (int)r[1];
        d.trans_b = (int)r[2];
        d.K1 = (int)r[3];
        d.K2 = (int)r[4];
        d.N = (int)r[5];
        d.img = reinterpret_cast<uint8_t*>(r[6]);
        d.bn = gemm_bn(d.N);
        d.nk1 = hg_ceil_div(d.K1, 32);
        d.nk = d.nk1 + (d.K2 > 0 ? hg_ceil_div(d.K2, 32) : 0);
        d.nnt = hg_ceil_div(d.N, d.bn);
        gx = d.nk > gx ? d.nk : gx;
        gy = d.nnt > gy ? d.nnt : gy;
    }
    k_prep_b_many<<<dim3(gx, gy, n), 256, 0, (cudaStream_t)stream>>>(pb);
    return hg_check_launch("gemm_tc_prep_b_many");
}

// C[M x N] = act(A1[M x K1] op(B)[0:K1] + A2[M x K2] op(B)[K1:K1+K2]) with the
// B image from hg_gemm_tc_prep_b.  Requirements: lda % 4 == 0, 16-byte aligned A.
extern "C" int hg_gemm_tc(const float* A1, int32_t lda1, int32_t K1, const float* A2, int32_t lda2, int32_t K2,
                          const void* bimg, float* C, int32_t ldc, int32_t N, const int32_t* d_M, int32_t M_cap,
                          int32_t act, void* stream) {
    if (M_cap <= 0 || N <= 0) return HG_OK;
    if ((lda1 & 3) || (A2 && (lda2 & 3)) || (reinterpret_cast<uintptr_t>(A1) & 15) ||
        (A2 && (reinterpret_cast<uintptr_t>(A2) & 15)) || (reinterpret_cast<uintptr_t>(bimg) & 15)) {
        hg_set_error("gemm_tc: A rows and the B image must be 16-byte aligned (lda %% 4 == 0)");
        return HG_EINVAL;
    }
    return hg_gemm_tma_launch(A1, lda1, K1, A2, lda2, K2, (const uint8_t*)bimg, C, ldc, N, d_M, M_cap, act,
                              (cudaStream_t)stream);
}

// process-wide tuning knobs of the kernel forms (see each setter); measured-slower
// alternates (cp.async GEMMs, SIMT small-M GEMMs, resident-B, the cooperative block
// sampler, the CSC backward) were removed from the library in round 2.
extern "C" int hg_set_tuning(int32_t key, int32_t value) {
    if (key == 1) { g_mn_swap = value ? 1 : 0; return HG_OK; }
    if (key == 3) { hg_tma_set_fwd_form(value ? 1 : 0); return HG_OK; }
    if (key == 5) { hg_set_pdl(value); return HG_OK; }
    if (key == 7) { hg_tma_set_pair(value); return HG_OK; }
    if (key == 9) { hg_tma_set_dbg(value); return HG_OK; }
    if (key == 11) { hg_tma_set_wg_tsa(value); return HG_OK; }
    if (key == 12) { hg_set_agg_bulk(value); return HG_OK; }
    hg_set_error("set_tuning: unknown key %d", key);
    return HG_EINVAL;
}

extern "C" int64_t hg_wgrad_tc_ws_size(int32_t K, int32_t N, int32_t M_cap, int32_t n_src) {
    return (int64_t)n_src * hg_wgrad_tma_chunks(K, n_src, M_cap) * K * N;
}

// out_s[K x N] = A_s[M x K]^T G[M x N] for s = 1 (A1) and, if A2, s = 2.
// ws >= hg_wgrad_tc_ws_size(K, N, M_cap, n_src) floats.  N <= 256.
extern "C" int hg_wgrad_tc(const float* A1, int32_t lda1, const float* A2, int32_t lda2, int32_t K, const float* G,
                           int32_t ldg, int32_t N, const int32_t* d_M, int32_t M_cap, float* out1, float* out2,
                           float* ws, void* stream) {
    if (K <= 0 || N <= 0) return HG_OK;
    if (N > 256) { hg_set_error("wgrad_tc: N > 256"); return HG_EUNSUPPORTED; }
    if ((lda1 & 3) || (A2 && (lda2 & 3)) || (ldg & 3)) {
        hg_set_error("wgrad_tc: row strides must be multiples of 4");
        return HG_EINVAL;
    }
    const uint32_t lbo = g_mn_swap ? 512u : 4096u, sbo = g_mn_swap ? 4096u : 512u;
    return hg_wgrad_tma_launch(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, out1, out2, ws, lbo, sbo,
                               (cudaStream_t)stream);
}

// hg_sgd + hg_gemm_tc_prep_b_many + hg_record_batch in one launch (see
// k_sgd_fused).  host_desc: n_img rows of int64 {B, ldb, trans_b, K1, K2, N, img}
// whose B lie inside w; ctl: 2 uint32 (max |dw| bits, last-block ticket), zero
// at rest; bp/d_loss/loss_arr/md_arr as hg_record_batch.
extern "C" int hg_sgd_fused(float* w, const float* g, int64_t n, float lr, int32_t n_img, const int64_t* host_desc,
                            uint32_t* ctl, const int64_t* bp, const float* d_loss, float* loss_arr, float* md_arr,
                            void* stream) {
    if (n <= 0) return HG_OK;
    if (n_img < 0 || n_img > MAX_PREP) { hg_set_error("sgd_fused: at most %d images", MAX_PREP); return HG_EINVAL; }
    FusedImages pb{};
    for (int i = 0; i < n_img; ++i) {
        const int64_t* r = host_desc + 7 * i;
        PrepDesc& d = pb.d[i];
        d.B = reinterpret_cast<const float*>(r[0]);
        d.ldb = (int)r[1];
        d.trans_b = (int)r[2];
        d.K1 = (int)r[3];
        d.K2 = (int)r[4];
        d.N = (int)r[5];
        d.img = reinterpret_cast<uint8_t*>(r[6]);
        d.bn = gemm_bn(d.N);
        d.nk1 = hg_ceil_div(d.K1, 32);
        d.nk = d.nk1 + (d.K2 > 0 ? hg_ceil_div(d.K2, 32) : 0);
        d.nnt = hg_ceil_div(d.N, d.bn);
        const int64_t off = (reinterpret_cast<const char*>(d.B) - reinterpret_cast<const char*>(w)) / 4;
        const int64_t rows = d.trans_b ? (int64_t)(d.K1 + d.K2) : (int64_t)d.N;
        if (off < 0 || off + rows * d.ldb > n) { hg_set_error("sgd_fused: image source outside w"); return HG_EINVAL; }
        pb.lo[i] = off;
        pb.hi[i] = off + rows * d.ldb;
    }
    cudaStream_t s = (cudaStream_t)stream;
    hg_launch(k_sgd_fused, hg_grid(n, 256, 4), 256, 0, s, pb, n_img, w, g, n, lr, ctl, bp, d_loss, loss_arr, md_arr);
    return hg_check_launch("sgd_fused");
}
