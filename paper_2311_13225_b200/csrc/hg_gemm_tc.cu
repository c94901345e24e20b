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
// Structure (one CTA = 128 output rows x BN columns, 4 warps):
//   cp.async (16 B, zero-filled beyond M/K) stages 128-byte-swizzled operand
//   tiles (the canonical SWIZZLE_128B layouts of the UMMA smem descriptors),
//   threads split lo = x - trunc(x) in place, fence.proxy.async + barrier,
//   one elected thread issues tcgen05.mma (M=128, kind::tf32, accumulator in
//   TMEM) and tcgen05.commit's to the stage's mbarrier, which gates the reuse
//   of that smem stage (2-stage ring: loads of tile k+1 overlap MMAs of tile k).
//   The epilogue reads the accumulator with tcgen05.ld (32x32b: warp w owns
//   TMEM lanes 32w..32w+31 = output rows) and applies the ReLU.
// The wgrad kernel feeds both operands MN-major (A^T and G are read as stored,
// row-major over the reduction dimension), which tf32 UMMA supports.
#include "hg_common.cuh"
#include "hg_gnn_internal.h"
#include "hg_tc.cuh"

namespace {
using namespace hgtc;

int g_mn_swap = 0;  // tuning knob (hg_set_tuning key 1): MN-major descriptor offset assignment
int g_skinny = 0;   // tuning knob (hg_set_tuning key 4): SIMT latency path for small M (hg_gemm_skinny.cu; measured slower than the TMA pipelines on B200, kept selectable)
int g_legacy = 0;   // tuning knob (hg_set_tuning key 2): 1 = the cp.async kernels below instead of hg_gemm_tma.cu

constexpr int TC_THREADS = 256;    // wgrad CTAs
constexpr int GEMM_THREADS = 256;  // forward / dX CTAs (8 warps: more loads and splits in flight)
constexpr int A_TILE = 128 * 128;  // 128 rows x 32 fp32

template <int BN>
__host__ __device__ constexpr int gemm_stage_bytes() { return 2 * A_TILE + 2 * BN * 128; }

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

template <int BN>
__host__ __device__ constexpr int gemm_stages() { return BN <= 64 ? 4 : (BN <= 128 ? 3 : 2); }
template <int BN>
__host__ __device__ constexpr int wgrad_stages() { return BN <= 64 ? 4 : (BN <= 128 ? 3 : 2); }

// Persistent CTAs: CTA b walks M tiles b, b+G, ... and the flattened (tile, k)
// iteration space streams through an S-stage cp.async ring (loads run S-1
// iterations ahead, a stage is refilled once the MMAs that read it committed).
// Two TMEM accumulators alternate between tiles, so the epilogue of tile t
// (tcgen05.ld + ReLU + stores) runs while tile t+1's MMAs are in flight.
template <int BN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
k_gemm_tc(const float* __restrict__ A1, int lda1, int K1, const float* __restrict__ A2, int lda2, int K2,
          const uint8_t* __restrict__ Bimg, float* __restrict__ C, int ldc, int N,
          const int* __restrict__ d_M, int M_cap, int act) {
    constexpr int S = gemm_stages<BN>();
    constexpr int STAGE = gemm_stage_bytes<BN>();
    constexpr int B_TILE = BN * 128;
    constexpr uint32_t NCOLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    constexpr uint32_t IDESC = idesc_tf32(128, BN, 0, 0);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[S];
    __shared__ uint64_t accbar[2];
    __shared__ uint32_t s_tmem;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int M = hg_load_count(d_M, M_cap);
    const int n_mt = (M + 127) >> 7;
    if ((int)blockIdx.x >= n_mt) return;
    const int n_my = (n_mt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int n0 = blockIdx.y * BN;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int nk1 = (K1 + 31) >> 5;
    const int nk2 = A2 ? (K2 + 31) >> 5 : 0;
    const int nk = nk1 + nk2;
    const int iters = n_my * nk;

    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
        mbar_init(&accbar[0], 1);
        mbar_init(&accbar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&s_tmem, NCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    const uint8_t* bimg = Bimg + (int64_t)blockIdx.y * nk * (2 * B_TILE);
    auto load_iter = [&](int it) {
        const int tile = it / nk, kt = it - tile * nk;
        const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
        uint8_t* base = smem + (it % S) * STAGE;
        const float* A;
        int lda, K, k0;
        if (kt < nk1) { A = A1; lda = lda1; K = K1; k0 = kt * 32; }
        else { A = A2; lda = lda2; K = K2; k0 = (kt - nk1) * 32; }
#pragma unroll
        for (int i = 0; i < 1024 / GEMM_THREADS; ++i) {  // A: 128 rows x 8 chunks of 16 B
            const int q = tid + GEMM_THREADS * i;
            const int r = q >> 3, c = q & 7;
            const int gm = m0 + r, gk = k0 + c * 4;
            int bytes = gm < M ? (K - gk) * 4 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            const float* src = bytes > 0 ? A + (int64_t)gm * lda + gk : A;
            cp_async16(smem_u32(base + off_k(r, c)), src, bytes);
        }
        // B: the prebuilt swizzled hi|lo image of this K tile (contiguous bytes)
        const uint8_t* bsrc = bimg + (int64_t)kt * (2 * B_TILE);
        const uint32_t bdst = smem_u32(base + 2 * A_TILE);
        for (int q = tid; q < (2 * B_TILE) / 16; q += GEMM_THREADS) cp_async16(bdst + q * 16, bsrc + q * 16, 16);
    };
    auto epilogue = [&](int tile) {
        const int acc = tile & 1;
        mbar_wait(&accbar[acc], (uint32_t)((tile >> 1) & 1));
        tc_fence_after();
        const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
        // warp w reads TMEM lanes 32*(w%4).. (its rows); warps w and w+4 split the columns
        const int gm = m0 + (warp & 3) * 32 + lane;
        const int cbeg = (warp >> 2) * (BN / 2);
#pragma unroll
        for (int c0 = cbeg; c0 < cbeg + BN / 2; c0 += 16) {
            float v[16];
            tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(acc * BN + c0), v);
            if (gm < M) {
                float* crow = C + (int64_t)gm * ldc + n0 + c0;
                const int lim = N - (n0 + c0);
                if (lim >= 16 && ((reinterpret_cast<uintptr_t>(crow) & 15) == 0)) {
#pragma unroll
                    for (int j = 0; j < 16; j += 4) {
                        float4 o = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
                        if (act) { o.x = fmaxf(o.x, 0.f); o.y = fmaxf(o.y, 0.f); o.z = fmaxf(o.z, 0.f); o.w = fmaxf(o.w, 0.f); }
                        *reinterpret_cast<float4*>(crow + j) = o;
                    }
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (j < lim) crow[j] = act ? fmaxf(v[j], 0.f) : v[j];
                }
            }
        }
        tc_fence_before();
    };

#pragma unroll
    for (int p = 0; p < S - 1; ++p) {
        if (p < iters) load_iter(p);
        cp_async_commit();
    }
    for (int it = 0; it < iters; ++it) {
        const int st = it % S;
        const int tile = it / nk, kt = it - tile * nk;
        cp_async_wait<S - 2>();  // the group of iteration `it` has landed
        uint8_t* base = smem + st * STAGE;
#pragma unroll
        for (int i = 0; i < 1024 / GEMM_THREADS; ++i) {
            const int q = tid + GEMM_THREADS * i;
            const uint32_t off = off_k(q >> 3, q & 7);
            split_lo16(base + off, base + A_TILE + off);
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t d = tmem + (uint32_t)((tile & 1) * BN);
            const uint32_t a_hi = smem_u32(base), a_lo = a_hi + A_TILE;
            const uint32_t b_hi = a_hi + 2 * A_TILE, b_lo = b_hi + B_TILE;
#pragma unroll
            for (int s = 0; s < 4; ++s) {
                const uint64_t dah = sdesc(a_hi + s * 32, 16, 1024), dal = sdesc(a_lo + s * 32, 16, 1024);
                const uint64_t dbh = sdesc(b_hi + s * 32, 16, 1024), dbl = sdesc(b_lo + s * 32, 16, 1024);
                mma_tf32(d, dah, dbh, IDESC, (kt | s) ? 1u : 0u);
                mma_tf32(d, dah, dbl, IDESC, 1u);
                mma_tf32(d, dal, dbh, IDESC, 1u);
            }
            mma_commit(&bars[st]);
            if (kt == nk - 1) mma_commit(&accbar[tile & 1]);
        }
        __syncwarp();
        // refill the stage consumed by iteration it-1 with iteration it+S-1
        const int nxt = it + S - 1;
        if (nxt < iters && it >= 1)  // use number (it-1)/S of that stage's barrier
            mbar_wait(&bars[(it - 1) % S], (uint32_t)(((it - 1) / S) & 1));
        if (nxt < iters) load_iter(nxt);
        cp_async_commit();
        // epilogue of the previous tile overlaps this tile's MMAs
        if (kt == 0 && tile > 0) epilogue(tile - 1);
    }
    if (iters > 0) epilogue(n_my - 1);
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, NCOLS);
}

// ---------------------------------------------------------------------------
// wgrad: partial[src][chunk][K x N] = A_src[rows of chunk]^T G[rows of chunk]
template <int BN>
__global__ void __launch_bounds__(TC_THREADS, 1)
k_wgrad_tc(const float* __restrict__ A1, int lda1, const float* __restrict__ A2, int lda2, int K,
           const float* __restrict__ G, int ldg, int N, const int* __restrict__ d_M, int M_cap, int rows_per_chunk,
           int n_chunks, float* __restrict__ partial, uint32_t lbo, uint32_t sbo) {
    constexpr int G_TILE = BN * 128;  // 32 rows x BN fp32
    constexpr int STAGE = 2 * A_TILE + 2 * G_TILE;
    constexpr int WS = wgrad_stages<BN>();
    constexpr uint32_t NCOLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
    constexpr uint32_t IDESC = idesc_tf32(128, BN, 1, 1);
    constexpr int GCH = BN / 4;  // 16-byte chunks per G row
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bars[WS];
    __shared__ uint32_t s_tmem;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int M = hg_load_count(d_M, M_cap);
    const int k0 = blockIdx.x * 128;
    const int src = blockIdx.y;
    const int chunk = blockIdx.z;
    const int mbeg = chunk * rows_per_chunk;
    float* P = partial + ((int64_t)src * n_chunks + chunk) * (int64_t)K * N;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (mbeg >= M) return;  // reduction skips chunks past M
    const int mend = min(M, mbeg + rows_per_chunk);
    const float* A = src ? A2 : A1;
    const int lda = src ? lda2 : lda1;
    const int nk = (mend - mbeg + 31) >> 5;

    if (tid == 0) {
#pragma unroll
        for (int i = 0; i < WS; ++i) mbar_init(&bars[i], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 0) tmem_alloc(&s_tmem, NCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;

    auto load_tile = [&](int kt, int st) {
        uint8_t* base = smem + st * STAGE;
        const int r0 = mbeg + kt * 32;
#pragma unroll
        for (int i = 0; i < 1024 / TC_THREADS; ++i) {  // A: 32 rows x 32 chunks (128 k)
            const int q = tid + TC_THREADS * i;
            const int r = q >> 5, cg = q & 31;
            const int gm = r0 + r, gk = k0 + cg * 4;
            int bytes = gm < mend ? (K - gk) * 4 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            const float* s = bytes > 0 ? A + (int64_t)gm * lda + gk : A;
            cp_async16(smem_u32(base + off_mn(r, cg)), s, bytes);
        }
        uint8_t* gb = base + 2 * A_TILE;
        for (int q = tid; q < 32 * GCH; q += TC_THREADS) {  // G: 32 rows x BN/4 chunks
            const int r = q / GCH, cg = q - r * GCH;
            const int gm = r0 + r, gn = cg * 4;
            int bytes = gm < mend ? (N - gn) * 4 : 0;
            bytes = bytes < 0 ? 0 : (bytes > 16 ? 16 : bytes);
            const float* s = bytes > 0 ? G + (int64_t)gm * ldg + gn : G;
            cp_async16(smem_u32(gb + off_mn(r, cg)), s, bytes);
        }
        cp_async_commit();
    };

#pragma unroll
    for (int p = 0; p < WS - 1; ++p) {
        if (p < nk) load_tile(p, p);
        else cp_async_commit();
    }
    for (int kt = 0; kt < nk; ++kt) {
        const int st = kt % WS;
        cp_async_wait<WS - 2>();  // tile kt landed
        uint8_t* base = smem + st * STAGE;
#pragma unroll
        for (int i = 0; i < 1024 / TC_THREADS; ++i) {
            const int q = tid + TC_THREADS * i;
            const uint32_t off = off_mn(q >> 5, q & 31);
            split_lo16(base + off, base + A_TILE + off);
        }
        uint8_t* gb = base + 2 * A_TILE;
        for (int q = tid; q < 32 * GCH; q += TC_THREADS) {
            const uint32_t off = off_mn(q / GCH, q % GCH);
            split_lo16(gb + off, gb + G_TILE + off);
        }
        fence_proxy_async();
        __syncthreads();
        if (tid == 0) {
            tc_fence_after();
            const uint32_t a_hi = smem_u32(base), a_lo = a_hi + A_TILE;
            const uint32_t g_hi = a_hi + 2 * A_TILE, g_lo = g_hi + G_TILE;
#pragma unroll
            for (int s = 0; s < 4; ++s) {  // 8 reduction rows (two 4-row K atoms) per MMA
                const uint64_t dah = sdesc(a_hi + s * 1024, lbo, sbo, 1), dal = sdesc(a_lo + s * 1024, lbo, sbo, 1);
                const uint64_t dgh = sdesc(g_hi + s * 1024, lbo, sbo, 1), dgl = sdesc(g_lo + s * 1024, lbo, sbo, 1);
                mma_tf32(tmem, dah, dgh, IDESC, (kt | s) ? 1u : 0u);
                mma_tf32(tmem, dah, dgl, IDESC, 1u);
                mma_tf32(tmem, dal, dgh, IDESC, 1u);
            }
            mma_commit(&bars[st]);
        }
        __syncwarp();
        const int nxt = kt + WS - 1;  // refill the stage tile kt-1 used
        if (nxt < nk) {
            if (kt >= 1) mbar_wait(&bars[(kt - 1) % WS], (uint32_t)(((kt - 1) / WS) & 1));
            load_tile(nxt, nxt % WS);
        } else {
            cp_async_commit();
        }
    }
    mbar_wait(&bars[(nk - 1) % WS], (uint32_t)(((nk - 1) / WS) & 1));  // all MMAs done
    tc_fence_after();
    const int r = (warp & 3) * 32 + lane;  // TMEM lane quarter of this warp
    const int gk = k0 + r;
    const int cbeg = (warp >> 2) * (BN / (TC_THREADS / 128));
#pragma unroll
    for (int c0 = cbeg; c0 < cbeg + BN / (TC_THREADS / 128); c0 += 16) {
        float v[16];
        tmem_ld16(tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0, v);
        if (gk < K) {
            float* prow = P + (int64_t)gk * N + c0;
            const int lim = N - c0;
#pragma unroll
            for (int j = 0; j < 16; ++j)
                if (j < lim) prow[j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) tmem_dealloc(tmem, NCOLS);
}

// Fixed-order reduction of the per-chunk partials: block = 32 consecutive
// outputs x 8 warps; warp w sums chunks w, w+8, ... (coalesced 128-byte rows),
// then warp 0 adds the 8 warp sums in order.  Deterministic.
__global__ void __launch_bounds__(256) k_wgrad_tc_reduce(const float* __restrict__ partial, int KN, int n_src,
                                                         int n_chunks, int rows_per_chunk, const int* __restrict__ d_M,
                                                         int M_cap, float* __restrict__ out1, float* __restrict__ out2) {
    __shared__ float s_part[8][33];
    const int M = hg_load_count(d_M, M_cap);
    const int chunks = min(n_chunks, (M + rows_per_chunk - 1) / rows_per_chunk);
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

template <int BN>
int launch_gemm(dim3 grid, cudaStream_t s, const float* A1, int lda1, int K1, const float* A2, int lda2, int K2,
                const uint8_t* bimg, float* C, int ldc, int N, const int* d_M, int M_cap, int act) {
    const int smem = gemm_stages<BN>() * gemm_stage_bytes<BN>() + 1024;
    grid.x = grid.x < (unsigned)HG_NUM_SMS ? grid.x : (unsigned)HG_NUM_SMS;  // persistent: <= 1 CTA per SM
    static bool attr = false;  // idempotent; set before first launch (outside graph capture via warm-up)
    if (!attr) {
        cudaFuncSetAttribute(k_gemm_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    k_gemm_tc<BN><<<grid, GEMM_THREADS, smem, s>>>(A1, lda1, K1, A2, lda2, K2, bimg, C, ldc, N, d_M, M_cap, act);
    return hg_check_launch("gemm_tc");
}

int gemm_bn(int N) {
    const int Nr = (N + 15) & ~15;
    return Nr <= 32 ? 32 : Nr <= 64 ? 64 : Nr <= 128 ? 128 : 256;
}

template <int BN>
int launch_wgrad(dim3 grid, cudaStream_t s, const float* A1, int lda1, const float* A2, int lda2, int K,
                 const float* G, int ldg, int N, const int* d_M, int M_cap, int rpc, int n_chunks, float* partial) {
    const int smem = wgrad_stages<BN>() * (2 * A_TILE + 2 * BN * 128) + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_wgrad_tc<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    // MN-major SWIZZLE_128B_BASE32B: LBO steps between 32-element MN atoms
    // (4 KB apart here), SBO between 4-row K atoms (512 B apart)
    const uint32_t lbo = g_mn_swap ? 512u : 4096u, sbo = g_mn_swap ? 4096u : 512u;
    k_wgrad_tc<BN><<<grid, TC_THREADS, smem, s>>>(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, rpc, n_chunks, partial,
                                                  lbo, sbo);
    return hg_check_launch("wgrad_tc");
}

int wgrad_rows_per_chunk(int M_cap, int ktiles, int n_src) {
    // aim for ~2 CTAs per SM over (k-tiles x sources x chunks), 32-row multiples, >= 128 rows
    long long want_chunks = (2LL * HG_NUM_SMS) / (ktiles * n_src);
    if (want_chunks < 1) want_chunks = 1;
    long long rpc = (M_cap + want_chunks - 1) / want_chunks;
    rpc = ((rpc + 31) / 32) * 32;
    if (rpc < 128) rpc = 128;
    return (int)rpc;
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
    cudaStream_t s = (cudaStream_t)stream;
    const int bn = gemm_bn(N);
    const uint8_t* b = (const uint8_t*)bimg;
    if (g_skinny && hg_skinny_gemm_ok(M_cap, K1, A2 ? K2 : 0, N))
        return hg_gemm_skinny_launch(A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act, s);
    if (!g_legacy) return hg_gemm_tma_launch(A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act, s);
    dim3 g(hg_ceil_div(M_cap, 128), hg_ceil_div(N, bn));
    switch (bn) {
        case 32: return launch_gemm<32>(g, s, A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act);
        case 64: return launch_gemm<64>(g, s, A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act);
        case 128: return launch_gemm<128>(g, s, A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act);
        default: return launch_gemm<256>(g, s, A1, lda1, K1, A2, lda2, K2, b, C, ldc, N, d_M, M_cap, act);
    }
}

// process-wide tuning knobs (key 1: MN-major descriptor LBO/SBO assignment)
extern "C" int hg_set_tuning(int32_t key, int32_t value) {
    if (key == 1) { g_mn_swap = value ? 1 : 0; return HG_OK; }
    if (key == 2) { g_legacy = value ? 1 : 0; return HG_OK; }
    if (key == 3) { hg_tma_set_fwd_form(value ? 1 : 0); return HG_OK; }
    if (key == 4) { g_skinny = value ? 1 : 0; return HG_OK; }
    if (key == 5) { hg_set_pdl(value); return HG_OK; }
    if (key == 6) { hg_tma_set_resb(value); return HG_OK; }
    if (key == 7) { hg_tma_set_pair(value); return HG_OK; }
    if (key == 8) { hg_set_block_coop(value); return HG_OK; }
    if (key == 9) { hg_tma_set_dbg(value); return HG_OK; }
    if (key == 11) { hg_tma_set_wg_tsa(value); return HG_OK; }
    if (key == 12) { hg_set_agg_bulk(value); return HG_OK; }
    hg_set_error("set_tuning: unknown key %d", key);
    return HG_EINVAL;
}

extern "C" int64_t hg_wgrad_tc_ws_size(int32_t K, int32_t N, int32_t M_cap, int32_t n_src) {
    const int kt = hg_ceil_div(K > 0 ? K : 1, 128);
    const int rpc = wgrad_rows_per_chunk(M_cap > 0 ? M_cap : 1, kt, n_src);
    const int chunks = hg_ceil_div(M_cap > 0 ? M_cap : 1, rpc);
    const int tchunks = hg_wgrad_tma_chunks(K, n_src);
    const int64_t tc = (int64_t)n_src * (chunks > tchunks ? chunks : tchunks) * K * N;
    const int64_t sk = hg_wgrad_skinny_ws_floats(K, N, M_cap, n_src);
    return tc > sk ? tc : sk;
}

// out_s[K x N] = A_s[M x K]^T G[M x N] for s = 1 (A1) and, if A2, s = 2.
// ws >= hg_wgrad_tc_ws_size(K, N, M_cap, n_src) floats.  N <= 256.
extern "C" int hg_wgrad_tc(const float* A1, int32_t lda1, const float* A2, int32_t lda2, int32_t K, const float* G,
                           int32_t ldg, int32_t N, const int32_t* d_M, int32_t M_cap, float* out1, float* out2,
                           float* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (K <= 0 || N <= 0) return HG_OK;
    if (N > 256) { hg_set_error("wgrad_tc: N > 256"); return HG_EUNSUPPORTED; }
    if ((lda1 & 3) || (A2 && (lda2 & 3)) || (ldg & 3)) {
        hg_set_error("wgrad_tc: row strides must be multiples of 4");
        return HG_EINVAL;
    }
    const uint32_t lbo = g_mn_swap ? 512u : 4096u, sbo = g_mn_swap ? 4096u : 512u;
    const bool al16 = ((reinterpret_cast<uintptr_t>(A1) | reinterpret_cast<uintptr_t>(A2) |
                        reinterpret_cast<uintptr_t>(G)) & 15) == 0;
    if (g_skinny && al16 && hg_skinny_wgrad_ok(M_cap, K, N))
        return hg_wgrad_skinny_launch(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, out1, out2, ws, s);
    if (!g_legacy) return hg_wgrad_tma_launch(A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, out1, out2, ws, lbo, sbo, s);
    const int n_src = A2 ? 2 : 1;
    const int kt = hg_ceil_div(K, 128);
    const int Mc = M_cap > 0 ? M_cap : 1;
    const int rpc = wgrad_rows_per_chunk(Mc, kt, n_src);
    const int chunks = hg_ceil_div(Mc, rpc);
    const int Nr = (N + 15) & ~15;
    dim3 grid(kt, n_src, chunks);
    int rc = HG_OK;
    if (M_cap > 0) {
        if (Nr <= 32) rc = launch_wgrad<32>(grid, s, A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, rpc, chunks, ws);
        else if (Nr <= 64) rc = launch_wgrad<64>(grid, s, A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, rpc, chunks, ws);
        else if (Nr <= 128) rc = launch_wgrad<128>(grid, s, A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, rpc, chunks, ws);
        else rc = launch_wgrad<256>(grid, s, A1, lda1, A2, lda2, K, G, ldg, N, d_M, M_cap, rpc, chunks, ws);
        if (rc) return rc;
    }
    k_wgrad_tc_reduce<<<n_src * hg_ceil_div(K * N, 32), 256, 0, s>>>(ws, K * N, n_src, chunks, rpc, d_M, M_cap, out1,
                                                                     out2);
    return hg_check_launch("wgrad_tc_reduce");
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
