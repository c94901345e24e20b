#include <type_traits>
// K8, warp-specialised TMA pipelines for the dense layer transforms.
//
// Same contracts as hg_gemm_tc.cu (fwd / dX: C = act(A1 op(B)[:K1] + A2 op(B)[K1:]);
// wgrad: dW_s = A_s^T G) and the same 3xTF32 arithmetic (x fed raw = its
// truncated tf32 "hi", lo = x - hi split in shared memory, D += AhBh + AhBl + AlBh),
// but the GEMMs here are HBM streams (K <= 2F, N <= 256), so the kernels are
// built to keep the memory system busy:
//
//   warp 0 (one lane)  TMA producer: cp.async.bulk.tensor 2-D tiles of A (and G)
//                      straight into the 128-byte-swizzled UMMA layouts, the
//                      prebuilt B image with one cp.async.bulk; completion via
//                      mbarrier transaction counts; runs up to S stages ahead.
//   warp 1 (one lane)  MMA issuer: tcgen05.mma kind::tf32 into TMEM, commits free
//                      the stage (and, per output tile, hand the accumulator to
//                      the epilogue).
//   4 split warps      lo = x - trunc_tf32(x) of each landed stage (layout-agnostic,
//                      linear 16-byte chunks), zeroing reduction rows past M (wgrad).
//   4 epilogue warps   (fwd) tcgen05.ld of the previous tile's accumulator + ReLU +
//                      stores, overlapping the next tile's loads and MMAs (two TMEM
//                      accumulators).
//
// No __syncthreads inside the main loops: every hand-off is an mbarrier
// (full -> split -> MMA -> empty -> producer; tfull -> epilogue -> tempty -> MMA).
// wgrad splits the reduction over M into a fixed number of chunks sized from the
// device-side row count, then reduces the partials in a fixed order
// (deterministic).
#include <cuda.h>

#include "hg_common.cuh"
#ifndef HG_GEMM_MAX_BN
#define HG_GEMM_MAX_BN 128  // widest N tile of the forward / dX GEMMs: wider N runs as several 128-wide TS-form
                            // N tiles (C3: 3.61 -> 3.82 M seeds/s vs one 256-wide SS-form tile, 2 stages)
#endif
#include "hg_gnn_internal.h"
#include "hg_tc.cuh"

namespace {
using namespace hgtc;

constexpr int FWD_THREADS = 320;  // w0 TMA, w1 MMA, w2-5 split, w6-9 epilogue
constexpr int WG_THREADS = 320;   // w0 TMA, w1 MMA, w2-9 split (w2-5 also the final epilogue)
constexpr int WG_SPLIT = WG_THREADS - 64;
constexpr int A_BYTES = 128 * 128;  // 128 rows x 32 fp32 (fwd) / 32 rows x 128 fp32 (wgrad)
// pipeline depths (shared memory per CTA also decides what else fits on the SM
// while these persistent kernels run)
#ifndef HG_WG_STAGES64
#define HG_WG_STAGES64 5
#endif
#ifndef HG_TS_PAIR_STAGES
#define HG_TS_PAIR_STAGES 6
#endif

template <int BN>
__host__ __device__ constexpr int fwd_stages() { return BN <= 32 ? 5 : BN <= 64 ? 4 : BN <= 128 ? 3 : 2; }
template <int BN>
__host__ __device__ constexpr int fwd_stage_bytes() { return 2 * A_BYTES + 2 * BN * 128; }
template <int BN, bool TSA>  // TS-form stages are 16 KB smaller (below): one more fits at BN <= 64
__host__ __device__ constexpr int wg_stages() { return BN <= 64 ? (TSA ? HG_WG_STAGES64 : 4) : BN <= 128 ? 3 : 2; }
// wgrad stage: [A | A lo (SS form only) | G hi | G lo]; the TS form (A^T through
// TMEM) never writes A lo to shared memory, so its stages are 16 KB smaller
template <int BN, bool TSA>
__host__ __device__ constexpr int wg_goff() { return (TSA ? 1 : 2) * A_BYTES; }
template <int BN, bool TSA>
__host__ __device__ constexpr int wg_stage_bytes() { return wg_goff<BN, TSA>() + 2 * BN * 128; }
template <int C>
__host__ __device__ constexpr uint32_t tmem_cols() { return C <= 32 ? 32 : C <= 64 ? 64 : C <= 128 ? 128 : C <= 256 ? 256 : 512; }

// profiling knob (hg_set_tuning key 9): bit 0 skips the MMAs, bit 1 the split
// work (pipelines still run; results are wrong) — isolates the bound stage
__constant__ int c_dbg;
// timeline probe (c_dbg bit 3): globaltimer stamps of CTA 0's first 64 iterations
__device__ unsigned long long g_tl[8][64];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#define TL(ev, it) do { if ((c_dbg & 8) && blockIdx.x == 0 && blockIdx.y == 0 && (it) < 64) g_tl[ev][it] = gtime(); } while (0)

__device__ __forceinline__ void mbar_init_fence() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }

// Epilogue store of 32 columns of this thread's output row (TMEM lane = row;
// float4 stores when aligned).  A shared-memory staged form that turns the
// row-per-thread stores into 128-byte row segments was measured slower in the
// step (+18 KB of shared memory per CTA costs co-residency).
__device__ __forceinline__ void epi_row32(const uint32_t (&r0)[16], const uint32_t (&r1)[16], int act,
                                          float* __restrict__ crow, int lim, bool vec) {
    auto val = [&](int j) {
        const float v = __uint_as_float(j < 16 ? r0[j] : r1[j - 16]);
        return act ? fmaxf(v, 0.f) : v;
    };
    if (vec && lim >= 32) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
            *reinterpret_cast<float4*>(crow + j) = make_float4(val(j), val(j + 1), val(j + 2), val(j + 3));
    } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
            if (j < lim) crow[j] = val(j);
    }
}

// ---------------------------------------------------------------------------
// forward / dX: persistent CTAs over 128-row M tiles (blockIdx.y = BN-wide N tile)
template <int BN>
__global__ void __launch_bounds__(FWD_THREADS, 1)
k_gemm_tma(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2, int nk1, int nk2, int ls1, int ls2,
           const uint8_t* __restrict__ Bimg, float* __restrict__ C, int ldc, int N, const int* __restrict__ d_M,
           int M_cap, int act) {
    constexpr int S = fwd_stages<BN>();
    constexpr int STAGE = fwd_stage_bytes<BN>();
    constexpr int B_BYTES = 2 * BN * 128;
    constexpr int B_TILE = BN * 128;
    constexpr uint32_t NCOLS = tmem_cols<2 * BN>();
    constexpr uint32_t IDESC = idesc_tf32(128, BN, 0, 0);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[S], splt[S], empty[S], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nk = nk1 + nk2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.y * BN;

    // prologue before griddepcontrol.wait (overlaps the previous kernel's tail)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&splt[i], 4);
            mbar_init(&empty[i], 1);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init_fence();
        tma_prefetch_desc(&tmA1);
        if (nk2) tma_prefetch_desc(&tmA2);
    }
    if (warp == 1) tmem_alloc(&s_tmem, NCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    hg_pdl_begin();
    const int M = hg_load_count(d_M, M_cap);
    const int n_mt = (M + 127) >> 7;
    if ((int)blockIdx.x >= n_mt) {
        if (warp == 1) tmem_dealloc(tmem, NCOLS);
        return;
    }
    const int n_my = (n_mt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int iters = n_my * nk;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const uint8_t* bimg = Bimg + (int64_t)blockIdx.y * nk * B_BYTES;
            for (int it = 0; it < iters; ++it) {
                const int st = it % S;
                if (it >= S) mbar_wait(&empty[st], (uint32_t)(((it / S) - 1) & 1));
                const int tile = it / nk, kt = it - tile * nk;
                const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
                uint8_t* base = smem + st * STAGE;
                mbar_expect_tx(&full[st], A_BYTES + B_BYTES);
                if (kt < nk1) tma_load_2d(smem_u32(base), &tmA1, kt * 32, m0, &full[st]);
                else tma_load_2d(smem_u32(base), &tmA2, (kt - nk1) * 32, m0, &full[st]);
                bulk_load(smem_u32(base + 2 * A_BYTES), bimg + (int64_t)kt * B_BYTES, B_BYTES, &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            int it = 0;
            for (int tile = 0; tile < n_my; ++tile) {
                const int acc = tile & 1;
                if (tile >= 2) mbar_wait(&tempty[acc], (uint32_t)(((tile >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * BN);
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int st = it % S;
                    mbar_wait(&splt[st], (uint32_t)((it / S) & 1));
                    tc_fence_after();
                    const uint32_t a_hi = smem_u32(smem + st * STAGE), a_lo = a_hi + A_BYTES;
                    const uint32_t b_hi = a_hi + 2 * A_BYTES, b_lo = b_hi + B_TILE;
                    // 8-wide K slices past the source's K hold TMA zero fill: skipped
                    const int ns = kt == nk1 - 1 ? ls1 : (kt == nk1 + nk2 - 1 ? ls2 : 4);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if (s >= ns) break;
                        const uint64_t dah = sdesc(a_hi + s * 32, 16, 1024), dal = sdesc(a_lo + s * 32, 16, 1024);
                        const uint64_t dbh = sdesc(b_hi + s * 32, 16, 1024), dbl = sdesc(b_lo + s * 32, 16, 1024);
                        mma_tf32(d, dah, dbh, IDESC, (kt | s) ? 1u : 0u);
                        mma_tf32(d, dah, dbl, IDESC, 1u);
                        mma_tf32(d, dal, dbh, IDESC, 1u);
                    }
                    mma_commit(&empty[st]);
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else if (warp < 6) {  // ---- split warps
        const int t = threadIdx.x - 64;
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            mbar_wait(&full[st], (uint32_t)((it / S) & 1));
            uint8_t* base = smem + st * STAGE;
#pragma unroll
            for (int i = 0; i < A_BYTES / 16 / 128; ++i) {
                const int off = (t + 128 * i) * 16;
                split_lo16(base + off, base + A_BYTES + off);
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&splt[st]);
        }
    } else {  // ---- epilogue warps: TMEM lane quarter = warp % 4
        const int q = warp & 3;
        const bool vec = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
        for (int tile = 0; tile < n_my; ++tile) {
            const int acc = tile & 1;
            mbar_wait(&tfull[acc], (uint32_t)((tile >> 1) & 1));
            tc_fence_after();
            const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
            const int gm = m0 + q * 32 + lane;
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r0[16], r1[16];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * BN + c0);
                tmem_ld16_nowait(ta, r0);
                tmem_ld16_nowait(ta + 16, r1);
                tmem_wait_ld();
                if (gm < M && n0 + c0 < N && !(c_dbg & 4))
                    epi_row32(r0, r1, act, C + (int64_t)gm * ldc + n0 + c0, N - (n0 + c0), vec);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, NCOLS);
    }
}

// ---------------------------------------------------------------------------
// forward / dX, "TS" form (BN <= 128): the split warps read each landed A tile
// once from shared memory (one 128-byte row per thread), and write hi and lo
// straight into TMEM with tcgen05.st; the MMAs take A from TMEM and only B from
// shared memory.  Shared-memory traffic per K tile drops from ~136 KB (A hi/lo
// written, A read by 8 of 12 MMAs, lo written) to ~72 KB, which is what bounds
// the SS form at N = 64.  TMEM: 2 accumulators (2*BN columns) + S A stages of
// 64 columns (hi 32 | lo 32).
template <int BN>
__host__ __device__ constexpr int ts_stages() { return BN <= 64 ? 6 : 4; }
template <int BN>
__host__ __device__ constexpr int ts_stage_bytes() { return A_BYTES + 2 * BN * 128; }

// PAIR: the B image's hi and lo tiles are adjacent 64-row blocks of one K-major
// tile, i.e. one N = 2*BN operand [B_hi ; B_lo]: per K slice the MMAs become
// A_hi x [B_hi ; B_lo] (N = 2*BN, into two accumulator halves) + A_lo x B_hi
// (N = BN), two instructions instead of three, and the epilogue adds the halves.
// (The tensor pipe, not memory, bounds the three-MMA form at N = 64.)
template <int BN, bool PAIR>
__host__ __device__ constexpr int ts_acc_cols() { return PAIR ? 2 * BN : BN; }
template <int BN, bool PAIR>
__host__ __device__ constexpr int ts_nstages() {
    return PAIR ? ((512 - 2 * ts_acc_cols<BN, PAIR>()) / 64 < HG_TS_PAIR_STAGES ? (512 - 2 * ts_acc_cols<BN, PAIR>()) / 64
                                                                                : HG_TS_PAIR_STAGES)
                : ts_stages<BN>();
}

template <int BN, bool PAIR>
__global__ void __launch_bounds__(FWD_THREADS, 1)
k_gemm_tma_ts(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2, int nk1, int nk2, int ls1, int ls2,
              const uint8_t* __restrict__ Bimg, float* __restrict__ C, int ldc, int N, const int* __restrict__ d_M,
              int M_cap, int act) {
    constexpr int S = ts_nstages<BN, PAIR>();
    constexpr int STAGE = ts_stage_bytes<BN>();
    constexpr int B_BYTES = 2 * BN * 128;
    constexpr int B_TILE = BN * 128;
    constexpr int ACC = ts_acc_cols<BN, PAIR>();  // accumulator columns per output tile
    constexpr uint32_t A_COL0 = 2 * ACC;           // first TMEM column of the A stages
    static_assert(2 * ACC + S * 64 <= 512, "TMEM budget");
    static_assert(S >= 2, "stages");
    constexpr uint32_t IDESC = idesc_tf32(128, BN, 0, 0);
    constexpr uint32_t IDESC2 = idesc_tf32(128, 2 * BN, 0, 0);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[S], splt[S], empty[S], tfull[2], tempty[2];
    __shared__ uint32_t s_tmem;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int nk = nk1 + nk2;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int n0 = blockIdx.y * BN;

    // prologue (barriers, TMEM, descriptor prefetch) touches nothing the previous
    // kernel writes: it runs before griddepcontrol.wait, overlapping that kernel's tail
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&splt[i], 4);
            mbar_init(&empty[i], 1);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);
        }
        mbar_init_fence();
        tma_prefetch_desc(&tmA1);
        if (nk2) tma_prefetch_desc(&tmA2);
    }
    if (warp == 1) tmem_alloc(&s_tmem, 512);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    hg_pdl_begin();
    const int M = hg_load_count(d_M, M_cap);
    const int n_mt = (M + 127) >> 7;
    if ((int)blockIdx.x >= n_mt) {  // nothing to do: give the TMEM back
        if (warp == 1) tmem_dealloc(tmem, 512);
        return;
    }
    const int n_my = (n_mt - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
    const int iters = n_my * nk;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer
            const uint8_t* bimg = Bimg + (int64_t)blockIdx.y * nk * B_BYTES;
            for (int it = 0; it < iters; ++it) {
                const int st = it % S;
                if (it >= S) mbar_wait(&empty[st], (uint32_t)(((it / S) - 1) & 1));
                TL(0, it);
                const int tile = it / nk, kt = it - tile * nk;
                const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
                uint8_t* base = smem + st * STAGE;
                mbar_expect_tx(&full[st], A_BYTES + B_BYTES);
                if (kt < nk1) tma_load_2d(smem_u32(base), &tmA1, kt * 32, m0, &full[st]);
                else tma_load_2d(smem_u32(base), &tmA2, (kt - nk1) * 32, m0, &full[st]);
                bulk_load(smem_u32(base + A_BYTES), bimg + (int64_t)kt * B_BYTES, B_BYTES, &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer (A from TMEM)
            int it = 0;
            for (int tile = 0; tile < n_my; ++tile) {
                const int acc = tile & 1;
                if (tile >= 2) mbar_wait(&tempty[acc], (uint32_t)(((tile >> 1) - 1) & 1));
                tc_fence_after();
                const uint32_t d = tmem + (uint32_t)(acc * ACC);
                for (int kt = 0; kt < nk; ++kt, ++it) {
                    const int st = it % S;
                    mbar_wait(&splt[st], (uint32_t)((it / S) & 1));
                    TL(3, it);
                    tc_fence_after();
                    const uint32_t ta = tmem + A_COL0 + (uint32_t)(st * 64);
                    const uint32_t b_hi = smem_u32(smem + st * STAGE + A_BYTES);
                    const uint32_t b_lo = b_hi + B_TILE;
                    // 8-wide K slices past the source's K hold TMA zero fill: skipped
                    const int ns = kt == nk1 - 1 ? ls1 : (kt == nk1 + nk2 - 1 ? ls2 : 4);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if ((c_dbg & 1) || s >= ns) break;
                        const uint64_t dbh = sdesc(b_hi + s * 32, 16, 1024), dbl = sdesc(b_lo + s * 32, 16, 1024);
                        if (PAIR) {  // [B_hi ; B_lo] is one N = 2*BN operand starting at b_hi
                            mma_tf32_ts(d, ta + s * 8, dbh, IDESC2, (kt | s) ? 1u : 0u);
                            mma_tf32_ts(d, ta + 32 + s * 8, dbh, IDESC, 1u);
                        } else {
                            mma_tf32_ts(d, ta + s * 8, dbh, IDESC, (kt | s) ? 1u : 0u);
                            mma_tf32_ts(d, ta + s * 8, dbl, IDESC, 1u);
                            mma_tf32_ts(d, ta + 32 + s * 8, dbh, IDESC, 1u);
                        }
                    }
                    mma_commit(&empty[st]);
                    TL(4, it);
                }
                mma_commit(&tfull[acc]);
            }
        }
    } else if (warp < 6) {  // ---- split warps: one tile row per thread, hi|lo -> TMEM
        const int q = warp & 3;
        const int r = q * 32 + lane;
        for (int it = 0; it < iters; ++it) {
            const int st = it % S;
            mbar_wait(&full[st], (uint32_t)((it / S) & 1));
            if (warp == 2 && lane == 0) TL(1, it);
            const uint8_t* base = smem + st * STAGE;
            if (c_dbg & 2) {  // profiling: no split work (same hand-offs)
                __syncwarp();
                if (lane == 0) mbar_arrive(&splt[st]);
                continue;
            }
            uint32_t hi[32], lo[32];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const float4 v = *reinterpret_cast<const float4*>(base + off_k(r, c));
                hi[4 * c + 0] = __float_as_uint(v.x);
                hi[4 * c + 1] = __float_as_uint(v.y);
                hi[4 * c + 2] = __float_as_uint(v.z);
                hi[4 * c + 3] = __float_as_uint(v.w);
            }
#pragma unroll
            for (int k = 0; k < 32; ++k) lo[k] = __float_as_uint(tf32_lo(__uint_as_float(hi[k])));
            const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + A_COL0 + (uint32_t)(st * 64);
            tmem_st32(ta, hi);
            tmem_st32(ta + 32, lo);
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&splt[st]);
            if (warp == 2 && lane == 0) TL(2, it);
        }
    } else {  // ---- epilogue warps: TMEM lane quarter = warp % 4
        const int q = warp & 3;
        const bool vec = ((ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(C) & 15) == 0);
        for (int tile = 0; tile < n_my; ++tile) {
            const int acc = tile & 1;
            mbar_wait(&tfull[acc], (uint32_t)((tile >> 1) & 1));
            tc_fence_after();
            const int m0 = ((int)blockIdx.x + tile * (int)gridDim.x) * 128;
            const int gm = m0 + q * 32 + lane;
#pragma unroll
            for (int c0 = 0; c0 < BN; c0 += 32) {
                uint32_t r0[16], r1[16];
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(acc * ACC + c0);
                tmem_ld16_nowait(ta, r0);
                tmem_ld16_nowait(ta + 16, r1);
                if (PAIR) {  // + the A_hi x B_lo half
                    uint32_t p0[16], p1[16];
                    tmem_ld16_nowait(ta + BN, p0);
                    tmem_ld16_nowait(ta + BN + 16, p1);
                    tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        r0[j] = __float_as_uint(__uint_as_float(r0[j]) + __uint_as_float(p0[j]));
                        r1[j] = __float_as_uint(__uint_as_float(r1[j]) + __uint_as_float(p1[j]));
                    }
                }
                tmem_wait_ld();
                if (gm < M && n0 + c0 < N && !(c_dbg & 4))
                    epi_row32(r0, r1, act, C + (int64_t)gm * ldc + n0 + c0, N - (n0 + c0), vec);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

// ---------------------------------------------------------------------------
// wgrad: CTA (unit = (src, 128-row K tile), chunk) accumulates
//   partial[src][chunk][K x N] = A_src[rows of chunk]^T G[rows of chunk]
// with both operands MN-major (SWIZZLE_128B_BASE32B atoms: 32 MN elements x 4
// reduction rows, loaded by TMA with the matching 32-byte-atom swizzle).
__device__ __forceinline__ int wg_rows_per_chunk(int M, int n_chunks) {
    int r = (M + n_chunks - 1) / n_chunks;
    return ((r + 31) / 32) * 32;
}

// PAIR (BN <= 64): the G hi and lo tiles are consecutive MN groups of one
// MN-major operand [G_hi | G_lo] (N = 2*BN): A_hi x [G_hi | G_lo] + A_lo x G_hi,
// two MMAs per K slice instead of three; the epilogue adds the halves.
// TSA: A^T through TMEM — A is loaded unswizzled (32 rows x 128 k, one TMA box),
// the split warps write its hi / lo columns straight into TMEM (lane = k,
// column = reduction row) and the MMAs read only G from shared memory: the
// per-step smem traffic drops from ~128 KB (A lo written back, A read by the
// MMAs) to ~80 KB, which is what paces the SS form.
template <int BN, bool PAIR, bool TSA>
__global__ void __launch_bounds__(WG_THREADS, 1)
k_wgrad_tma(const __grid_constant__ CUtensorMap tmA1, const __grid_constant__ CUtensorMap tmA2,
            const __grid_constant__ CUtensorMap tmG, int K, int N, int ktiles, const int* __restrict__ d_M, int M_cap,
            int n_chunks, float* __restrict__ partial, uint32_t lbo, uint32_t sbo) {
    constexpr int S = wg_stages<BN, TSA>();
    constexpr int STAGE = wg_stage_bytes<BN, TSA>();
    constexpr int GOFF = wg_goff<BN, TSA>();
    constexpr int G_TILE = BN * 128;  // 32 rows x BN fp32
    constexpr int NG = BN / 32;       // G boxes (32 columns each) per stage
    constexpr uint32_t ACC = PAIR ? 2 * BN : BN;
    constexpr uint32_t NCOLS = TSA ? 512u : tmem_cols<ACC>();
    static_assert(!TSA || ACC + S * 64 <= 512, "TMEM budget");
    constexpr uint32_t IDESC = idesc_tf32(128, BN, TSA ? 0 : 1, 1);
    constexpr uint32_t IDESC2 = idesc_tf32(128, 2 * BN, TSA ? 0 : 1, 1);
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t full[S], splt[S], empty[S], done;
    __shared__ uint32_t s_tmem;
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int chunk = blockIdx.y;
    const int src = blockIdx.x / ktiles, kt = blockIdx.x - src * ktiles;
    const CUtensorMap* tmA = src ? &tmA2 : &tmA1;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    // prologue before griddepcontrol.wait (overlaps the previous kernel's tail)
    if (threadIdx.x == 0) {
#pragma unroll
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&splt[i], WG_SPLIT / 32);
            mbar_init(&empty[i], 1);
        }
        mbar_init(&done, 1);
        mbar_init_fence();
        tma_prefetch_desc(tmA);
        tma_prefetch_desc(&tmG);
    }
    if (warp == 1) tmem_alloc(&s_tmem, NCOLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = s_tmem;
    hg_pdl_begin();
    const int M = hg_load_count(d_M, M_cap);
    const int rpc = wg_rows_per_chunk(M, n_chunks);
    const int mbeg = chunk * rpc;
    if (mbeg >= M) {  // the reduction skips chunks past M
        if (warp == 1) tmem_dealloc(tmem, NCOLS);
        return;
    }
    const int mend = min(M, mbeg + rpc);
    const int nsteps = (mend - mbeg + 31) >> 5;

    if (warp == 0) {
        if (lane == 0) {  // ---- TMA producer: 4 A boxes (32 k x 32 rows) + NG G boxes per step
            for (int j = 0; j < nsteps; ++j) {
                const int st = j % S;
                if (j >= S) mbar_wait(&empty[st], (uint32_t)(((j / S) - 1) & 1));
                TL(0, j);
                uint8_t* base = smem + st * STAGE;
                const int y = mbeg + 32 * j;
                mbar_expect_tx(&full[st], A_BYTES + G_TILE);
                if (TSA) {
                    tma_load_2d(smem_u32(base), tmA, kt * 128, y, &full[st]);  // [32 rows][128 k], row-major
                } else {
#pragma unroll
                    for (int g = 0; g < 4; ++g)
                        tma_load_2d(smem_u32(base + g * 4096), tmA, kt * 128 + g * 32, y, &full[st]);
                }
#pragma unroll
                for (int g = 0; g < NG; ++g)
                    tma_load_2d(smem_u32(base + GOFF + g * 4096), &tmG, g * 32, y, &full[st]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {  // ---- MMA issuer
            for (int j = 0; j < nsteps; ++j) {
                const int st = j % S;
                mbar_wait(&splt[st], (uint32_t)((j / S) & 1));
                TL(3, j);
                tc_fence_after();
                const uint32_t a_hi = smem_u32(smem + st * STAGE), a_lo = a_hi + A_BYTES;
                const uint32_t g_hi = a_hi + GOFF, g_lo = g_hi + G_TILE;
#pragma unroll
                for (int s = 0; s < 4; ++s) {  // 8 reduction rows (two 4-row K atoms) per MMA
                    if (c_dbg & 1) break;
                    const uint64_t dah = sdesc(a_hi + s * 1024, lbo, sbo, 1), dal = sdesc(a_lo + s * 1024, lbo, sbo, 1);
                    const uint64_t dgh = sdesc(g_hi + s * 1024, lbo, sbo, 1), dgl = sdesc(g_lo + s * 1024, lbo, sbo, 1);
                    if (TSA) {  // A^T hi / lo columns of this stage in TMEM, 8 reduction rows per slice
                        const uint32_t ta = tmem + ACC + (uint32_t)(st * 64) + (uint32_t)(s * 8);
                        if (PAIR) {
                            mma_tf32_ts(tmem, ta, dgh, IDESC2, (j | s) ? 1u : 0u);
                            mma_tf32_ts(tmem, ta + 32, dgh, IDESC, 1u);
                        } else {
                            mma_tf32_ts(tmem, ta, dgh, IDESC, (j | s) ? 1u : 0u);
                            mma_tf32_ts(tmem, ta, dgl, IDESC, 1u);
                            mma_tf32_ts(tmem, ta + 32, dgh, IDESC, 1u);
                        }
                    } else if (PAIR) {
                        mma_tf32(tmem, dah, dgh, IDESC2, (j | s) ? 1u : 0u);
                        mma_tf32(tmem, dal, dgh, IDESC, 1u);
                    } else {
                        mma_tf32(tmem, dah, dgh, IDESC, (j | s) ? 1u : 0u);
                        mma_tf32(tmem, dah, dgl, IDESC, 1u);
                        mma_tf32(tmem, dal, dgh, IDESC, 1u);
                    }
                }
                mma_commit(&empty[st]);
                TL(4, j);
            }
            mma_commit(&done);
        }
    } else {  // ---- split warps (reduction rows past M are zeroed in hi and lo)
        const int t = threadIdx.x - 64;
        for (int j = 0; j < nsteps; ++j) {
            const int st = j % S;
            mbar_wait(&full[st], (uint32_t)((j / S) & 1));
            if (warp == 2 && lane == 0) TL(1, j);
            uint8_t* base = smem + st * STAGE;
            const int valid = mend - (mbeg + 32 * j);  // rows < valid are real
            if (TSA && !(c_dbg & 2)) {
                // A^T into TMEM: warp w writes lanes 32*(w%4).. (k), columns 16*half.. (rows)
                const int q = warp & 3, half = (warp - 2) >> 2;
                const int k = q * 32 + lane;
                uint32_t hi[16], lo[16];
#pragma unroll
                for (int c = 0; c < 16; ++c) {
                    const int m = half * 16 + c;
                    const float x = m < valid ? *reinterpret_cast<const float*>(base + m * 512 + k * 4) : 0.f;
                    hi[c] = __float_as_uint(x);
                    lo[c] = __float_as_uint(tf32_lo(x));
                }
                const uint32_t ta = tmem + ((uint32_t)(q * 32) << 16) + ACC + (uint32_t)(st * 64) + (uint32_t)(half * 16);
                tmem_st16(ta, hi);
                tmem_st16(ta + 32, lo);
            }
            if (!(c_dbg & 2)) {
                // all loads of the stage first (ILP: the split is latency-bound with
                // 4 warps), then lo = x - hi and the stores; rows past M -> zeros
                constexpr int NA = TSA ? 0 : A_BYTES / 16 / WG_SPLIT;
                constexpr int NGC = (G_TILE / 16 + WG_SPLIT - 1) / WG_SPLIT;
                float4 va[NA > 0 ? NA : 1], vg[NGC];
#pragma unroll
                for (int i = 0; i < NA; ++i) va[i] = *reinterpret_cast<const float4*>(base + (t + WG_SPLIT * i) * 16);
                uint8_t* gb = base + GOFF;
#pragma unroll
                for (int i = 0; i < NGC; ++i)
                    if (t + WG_SPLIT * i < G_TILE / 16) vg[i] = *reinterpret_cast<const float4*>(gb + (t + WG_SPLIT * i) * 16);
                const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int i = 0; i < NA; ++i) {
                    const int off = (t + WG_SPLIT * i) * 16;
                    if (((off & 4095) >> 7) < valid) {
                        const float4 v = va[i];
                        *reinterpret_cast<float4*>(base + A_BYTES + off) =
                            make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
                    } else {
                        *reinterpret_cast<float4*>(base + off) = z;
                        *reinterpret_cast<float4*>(base + A_BYTES + off) = z;
                    }
                }
#pragma unroll
                for (int i = 0; i < NGC; ++i) {
                    if (t + WG_SPLIT * i >= G_TILE / 16) break;
                    const int off = (t + WG_SPLIT * i) * 16;
                    if (((off & 4095) >> 7) < valid) {
                        const float4 v = vg[i];
                        *reinterpret_cast<float4*>(gb + G_TILE + off) =
                            make_float4(tf32_lo(v.x), tf32_lo(v.y), tf32_lo(v.z), tf32_lo(v.w));
                    } else {
                        *reinterpret_cast<float4*>(gb + off) = z;
                        *reinterpret_cast<float4*>(gb + G_TILE + off) = z;
                    }
                }
            }
            if (TSA) {
                tmem_wait_st();
                tc_fence_before();
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&splt[st]);
            if (warp == 2 && lane == 0) TL(2, j);
        }
        // ---- epilogue (warps 2-5, one per TMEM lane quarter): partial rows k of this K tile
        if (warp < 6) {
        mbar_wait(&done, 0u);
        tc_fence_after();
        const int q = warp & 3;
        const int gk = kt * 128 + q * 32 + lane;
        float* P = partial + ((int64_t)src * n_chunks + chunk) * (int64_t)K * N;
#pragma unroll
        for (int c0 = 0; c0 < BN; c0 += 16) {
            uint32_t r[16];
            tmem_ld16_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)c0, r);
            if (PAIR) {  // + the A_hi x G_lo half
                uint32_t p[16];
                tmem_ld16_nowait(tmem + ((uint32_t)(q * 32) << 16) + (uint32_t)(BN + c0), p);
                tmem_wait_ld();
#pragma unroll
                for (int jj = 0; jj < 16; ++jj) r[jj] = __float_as_uint(__uint_as_float(r[jj]) + __uint_as_float(p[jj]));
            }
            tmem_wait_ld();
            if (gk < K && c0 < N) {  // partials are N-major: lanes (consecutive k) store one 128-byte line
                float* pcol = P + (int64_t)c0 * K + gk;
                const int lim = N - c0;
#pragma unroll
                for (int jj = 0; jj < 16; ++jj)
                    if (jj < lim) pcol[(int64_t)jj * K] = __uint_as_float(r[jj]);
            }
        }
        tc_fence_before();
        }
    }
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc(tmem, NCOLS);
    }
}

// Fixed-order reduction of the active chunks' partials (chunk order within each
// of the 8 warps, then the 8 warp sums in order): deterministic for a given M.
// Partials are N-major ([n][k], element e = n*K + k); the result is written
// row-major dW[k][n].  A block covers 32*VEC consecutive elements, VEC per lane
// (VEC = 4: 16-byte loads, four chunk rows in flight per warp).
template <int VEC>
__global__ void __launch_bounds__(256) k_wgrad_tma_reduce(const float* __restrict__ partial, int K, int N, int n_chunks,
                                                          const int* __restrict__ d_M, int M_cap,
                                                          float* __restrict__ out1, float* __restrict__ out2) {
    constexpr int BE = 32 * VEC;  // elements per block
    using VT = typename std::conditional<VEC == 4, float4, float>::type;
    const int KN = K * N;
    hg_pdl_begin();
    __shared__ float s_part[8][BE + 1];
    const int M = hg_load_count(d_M, M_cap);
    const int rpc = M > 0 ? wg_rows_per_chunk(M, n_chunks) : 1;
    const int chunks = M > 0 ? (M + rpc - 1) / rpc : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int per_src = (KN + BE - 1) / BE;
    const int s = blockIdx.x / per_src;
    const int e0 = (blockIdx.x - s * per_src) * BE;
    const int e = e0 + lane * VEC;  // KN % VEC == 0: a lane's VEC elements are all in range or all out
    float acc[VEC];
#pragma unroll
    for (int v = 0; v < VEC; ++v) acc[v] = 0.f;
    if (e < KN) {
        const float* p = partial + (int64_t)s * n_chunks * KN + e;
        // G chunk rows per batch, all loads issued before the in-order sums: one
        // memory latency per batch instead of one per chunk
        constexpr int G = 16 / VEC;
        for (int c0 = w; c0 < chunks; c0 += 8 * G) {
            VT x[G];
#pragma unroll
            for (int u = 0; u < G; ++u) {
                const int c = c0 + 8 * u;
                if (c < chunks) x[u] = *reinterpret_cast<const VT*>(p + (int64_t)c * KN);
            }
#pragma unroll
            for (int u = 0; u < G; ++u) {
                if (c0 + 8 * u >= chunks) break;
                const float* xf = reinterpret_cast<const float*>(&x[u]);
#pragma unroll
                for (int v = 0; v < VEC; ++v) acc[v] += xf[v];
            }
        }
    }
#pragma unroll
    for (int v = 0; v < VEC; ++v) s_part[w][lane * VEC + v] = acc[v];
    __syncthreads();
    for (int i = threadIdx.x; i < BE; i += blockDim.x) {
        const int ei = e0 + i;
        if (ei >= KN) break;
        float t = 0.f;
#pragma unroll
        for (int r = 0; r < 8; ++r) t += s_part[r][i];
        const int n = ei / K, k = ei - n * K;
        (s ? out2 : out1)[(int64_t)k * N + n] = t;
    }
}

int g_pair = 1;  // paired hi|lo MMA form for BN <= 64, fwd and wgrad (hg_set_tuning key 7)
int g_wg_tsa = 1;  // wgrad with A^T through TMEM (hg_set_tuning key 11)

// ---------------------------------------------------------------------------
// host: tensor maps through the driver entry point (no libcuda link needed)
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeTiledFn>(p);
    }
    return fn;
}

// fp32 matrix [rows x cols] with row stride ld (elements); box = box_cols x box_rows
int make_map(CUtensorMap* m, const float* base, int cols, int rows, int ld, int box_cols, int box_rows,
             CUtensorMapSwizzle sw) {
    EncodeTiledFn enc = encode_fn();
    if (!enc) {
        hg_set_error("gemm_tma: cuTensorMapEncodeTiled unavailable");
        return HG_ECUDA;
    }
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)(rows > 0 ? rows : 1)};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
        hg_set_error("gemm_tma: cuTensorMapEncodeTiled failed (%d): cols %d rows %d ld %d", (int)r, cols, rows, ld);
        return HG_ECUDA;
    }
    return HG_OK;
}

template <int BN>
int launch_fwd(int M_cap, int n_nt, cudaStream_t s, const CUtensorMap& m1, const CUtensorMap& m2, int nk1, int nk2,
               int ls1, int ls2,
               const uint8_t* bimg, float* C, int ldc, int N, const int* d_M, int act) {
    const int smem = fwd_stages<BN>() * fwd_stage_bytes<BN>() + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm_tma<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        attr = true;
    }
    int gx = hg_ceil_div(M_cap, 128);
    gx = gx < HG_NUM_SMS ? gx : HG_NUM_SMS;
    hg_launch(k_gemm_tma<BN>, dim3(gx, n_nt), FWD_THREADS, smem, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, M_cap, act);
    return hg_check_launch("gemm_tma");
}

template <int BN>
int launch_fwd_ts(int M_cap, int n_nt, cudaStream_t s, const CUtensorMap& m1, const CUtensorMap& m2, int nk1,
                  int nk2, int ls1, int ls2, const uint8_t* bimg, float* C, int ldc, int N, const int* d_M, int act) {
    const int smem = ts_stages<BN>() * ts_stage_bytes<BN>() + 1024;
    const bool pair = g_pair && BN <= 64;
    constexpr bool PB = BN <= 64;
    const int smem_pair = ts_nstages<BN, PB>() * ts_stage_bytes<BN>() + 1024;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_gemm_tma_ts<BN, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_gemm_tma_ts<BN, PB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_pair);
        attr = true;
    }
    int gx = hg_ceil_div(M_cap, 128);
    gx = gx < HG_NUM_SMS ? gx : HG_NUM_SMS;
    if (pair)
        hg_launch(k_gemm_tma_ts<BN, (BN <= 64)>, dim3(gx, n_nt), FWD_THREADS, smem_pair, s, m1, m2, nk1, nk2, ls1, ls2,
                  bimg, C, ldc, N, d_M, M_cap, act);
    else
        hg_launch(k_gemm_tma_ts<BN, false>, dim3(gx, n_nt), FWD_THREADS, smem, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C,
                  ldc, N, d_M, M_cap, act);
    return hg_check_launch("gemm_tma_ts");
}

int g_fwd_form = 1;  // 1: TS form for BN <= 128 (hg_set_tuning key 3), 0: SS form everywhere

template <int BN>
int launch_wg(dim3 grid, cudaStream_t s, const CUtensorMap& m1, const CUtensorMap& m2, const CUtensorMap& mg, int K,
              int N, int ktiles, const int* d_M, int M_cap, int n_chunks, float* partial, uint32_t lbo, uint32_t sbo,
              bool tsa) {
    const int smem_ss = wg_stages<BN, false>() * wg_stage_bytes<BN, false>() + 1024;
    const int smem_ts = wg_stages<BN, true>() * wg_stage_bytes<BN, true>() + 1024;
    constexpr bool PB = BN <= 64;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_wgrad_tma<BN, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ss);
        cudaFuncSetAttribute(k_wgrad_tma<BN, PB, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ss);
        cudaFuncSetAttribute(k_wgrad_tma<BN, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ts);
        cudaFuncSetAttribute(k_wgrad_tma<BN, PB, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_ts);
        attr = true;
    }
#define HG_WG(P, T)                                                                                                  \
    hg_launch(k_wgrad_tma<BN, P, T>, grid, WG_THREADS, T ? smem_ts : smem_ss, s, m1, m2, mg, K, N, ktiles, d_M, M_cap, \
              n_chunks, partial, lbo, sbo)
    const bool pair = g_pair && PB;
    if (pair && tsa) HG_WG(PB, true);
    else if (pair) HG_WG(PB, false);
    else if (tsa) HG_WG(false, true);
    else HG_WG(false, false);
#undef HG_WG
    return hg_check_launch("wgrad_tma");
}

}  // namespace

void hg_tma_set_fwd_form(int v) { g_fwd_form = v; }
void hg_tma_set_wg_tsa(int v) { g_wg_tsa = v ? 1 : 0; }
void hg_tma_set_pair(int v) { g_pair = v ? 1 : 0; }
void hg_tma_set_dbg(int v) { cudaMemcpyToSymbol(c_dbg, &v, sizeof(int)); }
// timeline probe read-back: 8 x 64 globaltimer stamps (ns)
extern "C" int hg_debug_timeline(uint64_t* out) {
    return cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)) == cudaSuccess ? HG_OK : HG_ECUDA;
}

int hg_tma_gemm_bn(int N) {
    const int Nr = (N + 15) & ~15;
    return Nr <= 32 ? 32 : Nr <= 64 ? 64 : (Nr <= 128 || HG_GEMM_MAX_BN <= 128) ? 128 : 256;
}

int hg_gemm_tma_launch(const float* A1, int lda1, int K1, const float* A2, int lda2, int K2, const uint8_t* bimg,
                       float* C, int ldc, int N, const int* d_M, int M_cap, int act, cudaStream_t s) {
    CUtensorMap m1, m2;
    int rc = make_map(&m1, A1, K1, M_cap, lda1, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    if (rc) return rc;
    if (A2 && K2 > 0) {
        rc = make_map(&m2, A2, K2, M_cap, lda2, 32, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        if (rc) return rc;
    } else {
        m2 = m1;
    }
    const int nk1 = hg_ceil_div(K1, 32), nk2 = (A2 && K2 > 0) ? hg_ceil_div(K2, 32) : 0;
    const int ls1 = (K1 - 1) % 32 / 8 + 1, ls2 = nk2 ? (K2 - 1) % 32 / 8 + 1 : 4;  // live 8-wide slices of each last tile
    const int bn = hg_tma_gemm_bn(N);
    const int n_nt = hg_ceil_div(N, bn);
    if (g_fwd_form == 1 && bn <= 128) {
        switch (bn) {
            case 32: return launch_fwd_ts<32>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
            case 64: return launch_fwd_ts<64>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
            default: return launch_fwd_ts<128>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
        }
    }
    switch (bn) {
        case 32: return launch_fwd<32>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
        case 64: return launch_fwd<64>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
        case 128: return launch_fwd<128>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
        default: return launch_fwd<256>(M_cap, n_nt, s, m1, m2, nk1, nk2, ls1, ls2, bimg, C, ldc, N, d_M, act);
    }
}

// Split-M chunk count: one CTA per (source, K tile, chunk), one wave.  (Capping
// it by the layer's row count — >= 128/256/512 rows per chunk for the small
// upper layers — measured slower in the pipelined step: 178.5/179.4/185.4 vs
// 178.1 us; the side-stream weight gradients are latency-, not SM-time-bound.)
int hg_wgrad_tma_chunks(int K, int n_src, int M_cap) {
    (void)M_cap;
    const int units = hg_ceil_div(K > 0 ? K : 1, 128) * n_src;
    const int c = HG_NUM_SMS / units;
    return c < 1 ? 1 : c;
}

int hg_wgrad_tma_launch(const float* A1, int lda1, const float* A2, int lda2, int K, const float* G, int ldg, int N,
                        const int* d_M, int M_cap, float* out1, float* out2, float* ws, uint32_t lbo, uint32_t sbo,
                        cudaStream_t s) {
    const int n_src = A2 ? 2 : 1;
    const int ktiles = hg_ceil_div(K, 128);
    const int n_chunks = hg_wgrad_tma_chunks(K, n_src, M_cap);
    if (M_cap > 0) {
        CUtensorMap m1, m2, mg;
        const CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;
        // TS form: A as plain [32 rows][128 k] boxes (read by the split warps, never by the MMA)
        const bool tsa = g_wg_tsa != 0;
        const int abox = tsa ? 128 : 32;
        const CUtensorMapSwizzle asw = tsa ? CU_TENSOR_MAP_SWIZZLE_NONE : sw;
        int rc = make_map(&m1, A1, K, M_cap, lda1, abox, 32, asw);
        if (!rc && A2) rc = make_map(&m2, A2, K, M_cap, lda2, abox, 32, asw);
        if (!A2) m2 = m1;
        if (!rc) rc = make_map(&mg, G, N, M_cap, ldg, 32, 32, sw);
        if (rc) return rc;
        const int Nr = (N + 15) & ~15;
        dim3 grid(ktiles * n_src, n_chunks);
        if (Nr <= 32) rc = launch_wg<32>(grid, s, m1, m2, mg, K, N, ktiles, d_M, M_cap, n_chunks, ws, lbo, sbo, tsa);
        else if (Nr <= 64) rc = launch_wg<64>(grid, s, m1, m2, mg, K, N, ktiles, d_M, M_cap, n_chunks, ws, lbo, sbo, tsa);
        else if (Nr <= 128) rc = launch_wg<128>(grid, s, m1, m2, mg, K, N, ktiles, d_M, M_cap, n_chunks, ws, lbo, sbo, tsa);
        else rc = launch_wg<256>(grid, s, m1, m2, mg, K, N, ktiles, d_M, M_cap, n_chunks, ws, lbo, sbo, tsa);
        if (rc) return rc;
    }
    // 16-byte lanes only when that still leaves >= 2 blocks per SM (C3's bottom layer:
    // 1,204 blocks); the small C2 layers keep one float per lane and 4x the blocks
    const long long blocks4 = n_src * hg_ceil_div((long long)K * N, 128);
    if (((K * N) & 3) == 0 && !(reinterpret_cast<uintptr_t>(ws) & 15) && blocks4 >= 2 * HG_NUM_SMS)
        hg_launch(k_wgrad_tma_reduce<4>, n_src * hg_ceil_div((long long)K * N, 128), 256, 0, s, ws, K, N, n_chunks, d_M,
                  M_cap, out1, out2);
    else
        hg_launch(k_wgrad_tma_reduce<1>, n_src * hg_ceil_div((long long)K * N, 32), 256, 0, s, ws, K, N, n_chunks, d_M,
                  M_cap, out1, out2);
    return hg_check_launch("wgrad_tma_reduce");
}
