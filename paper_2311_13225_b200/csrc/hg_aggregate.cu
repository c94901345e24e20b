#include <cstdlib>
// K4-K7: gather + mean/GCN aggregation forward, transposed aggregation backward.
//
// Forward replaces, for one sampled block,
//   feature gather  data.features[stack.bottom_src()]        (orchestrator.py:239)
//   SAGE            _sage_neighbor_edges + segment_weighted_rows (gnnmath.py:145-154,171)
//   GCN             gcn_norm_weights   + segment_weighted_rows (gnnmath.py:89-97,120)
// in ONE pass: the bottom layer reads feature rows straight from the
// HBM-resident table by global id (no materialised [n_src x F] gather buffer)
// and writes [self rows | aggregate] for the dense transform; rows of
// destinations whose output will be replaced by a historical embedding
// (gnnmath.py:240-245) are skipped (zero-filled) — the reduced gather of
// transfer.needed_bottom_rows (transfer.py:59-73).
//
// Each destination is served by a group of LPR lanes; lane l of the group owns
// float4 columns l, l+LPR, ...  Edges are consumed in slot order (ascending
// local src = the reference's (dst, src) order) with four rows in flight per
// step, so accumulation order per column is fixed: deterministic, no atomics.
//
// Backward (layers >= 1 only, need_dx = l > 0, gnnmath.py:256) replaces the
// transposed scatter segment_weighted_rows(ed, es, ...) (gnnmath.py:140,199)
// with k_bwd_scatter + k_bwd_finish below: a deterministic two-word fixed-point
// scatter (integer atomics, order-independent), then the SAGE self-term
// gradient and the lower layer's ReLU' and injected-row masks
// (gnnmath.py:130-134,183-188) before dZ of the layer below is written.
#include "hg_common.cuh"
#include "hg_gnn_internal.h"
#include "hg_tc.cuh"

namespace {

enum { M_SAGE_LOCAL = 0, M_SAGE_GLOBAL = 1, M_GCN_LOCAL = 2, M_GCN_GLOBAL = 3 };

__device__ __forceinline__ float4 f4_fma(float w, float4 r, float4 a) {
    a.x = fmaf(w, r.x, a.x);
    a.y = fmaf(w, r.y, a.y);
    a.z = fmaf(w, r.z, a.z);
    a.w = fmaf(w, r.w, a.w);
    return a;
}

__device__ __forceinline__ float gcn_w(int outdeg_s, int indeg_d) {
    return (float)(1.0 / sqrt((double)outdeg_s * (double)indeg_d));
}

// Feature table row-sharded over devices (C4: features larger than one GPU's
// HBM): row v lives in shard v / rows_per_shard, at row v % rows_per_shard; the
// bases are NVLink peer pointers (CUDA IPC) or slices of one local table.
constexpr int HG_MAX_SHARDS = 8;
struct FeatShards {
    const float* base[HG_MAX_SHARDS];
    int n;
    int rows_per_shard;
    // split rows (AD_SPLIT): columns [0, 4*body4) in the line-aligned body table
    // (hin, stride ld_in), columns [4*body4, F) in the tail table (stride tail_ld)
    const float* tail;
    int tail_ld;
    int body4;
};
// Row addressing of the feature gather: one table, row-sharded tables, or split rows.
enum { AD_PLAIN = 0, AD_SHARDED = 1, AD_SPLIT = 2 };

// Rows in flight per warp when a whole row is one float4 per lane (F <= 128, LPR 32):
// 8, not 16 — the kernel then needs 48 registers instead of 64, five 256-thread
// CTAs fit on an SM (agg_ctas_per_sm() = 5, one wave) and the bottom aggregation
// of the C2 step runs in 61 instead of 67.5 us with the step at 172.7 instead of
// 177.2 us (4 CTAs x 16 rows, 3 CTAs, 6 CTAs at 40 registers with
// spills, 10/12 rows in flight measured slower).
#ifndef HG_AGG_U1
#define HG_AGG_U1 8
#endif
// L2 prefetch of a destination's edge rows as soon as its edge list is known
// (one prefetch.global.L2 per 128-byte line, no registers held): the rows past
// the first U in flight are already on their way when the warp loads them.
// Bottom aggregation 61.2 -> 60.3 us, C2 step -1 to -3 us (profiles/
// r02s_occupancy_sweep.md); prefetching the next destination's rows or its
// metadata, or before the self row copy, measured slower.
#ifndef HG_AGG_PF
#define HG_AGG_PF 1
#endif
__device__ __forceinline__ void prefetch_row_l2(const float4* p, int F4) {
    const uintptr_t a0 = reinterpret_cast<uintptr_t>(p), a1 = a0 + (uintptr_t)F4 * 16;
    for (uintptr_t a = a0 & ~uintptr_t(127); a < a1; a += 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
}
#if defined(HG_AGG_MINB) && HG_AGG_MINB > 0  // experiment knob: register cap via min CTAs per SM
#define HG_AGG_BOUNDS __launch_bounds__(256, HG_AGG_MINB)
#else
#define HG_AGG_BOUNDS __launch_bounds__(256)
#endif
template <int LPR, int NV, int MODE, int AD = AD_PLAIN>
__global__ void HG_AGG_BOUNDS k_agg_fwd(
    const float* __restrict__ hin, int ld_in, int F4, const int* __restrict__ frontier, const int* d_n, int cap,
    int f, const int* __restrict__ counts, const int* __restrict__ slot_g, const int* __restrict__ slot_local,
    const int* __restrict__ nself, const int* __restrict__ outdeg, const uint8_t* __restrict__ inj,
    float* __restrict__ self_out, int ld_self, float* __restrict__ agg_out, int ld_agg, const FeatShards shards) {
    hg_pdl_begin();
    constexpr bool SH = AD == AD_SHARDED, SPLIT = AD == AD_SPLIT;
    auto rowp = [&](int v) -> const float4* {
        if (SH) {
            const int k = v / shards.rows_per_shard;
            return reinterpret_cast<const float4*>(shards.base[k] + (int64_t)(v - k * shards.rows_per_shard) * ld_in);
        }
        return reinterpret_cast<const float4*>(hin + (int64_t)v * ld_in);
    };
    // float4 column c of row v.  Split rows (one float4 per lane, c == lane's column):
    // the lane's column lives in the body's whole 128-byte lines or in the tail
    // table, fixed per lane, so the address is one base + v * stride as for a plain row.
    static_assert(!SPLIT || NV == 1, "split rows: one float4 column per lane");
    const int lr0 = threadIdx.x & (LPR - 1);
    const bool in_tail = SPLIT && lr0 >= shards.body4;
    const float* lbase = in_tail ? shards.tail + (lr0 - shards.body4) * 4 : hin + lr0 * 4;
    const int64_t lstride = in_tail ? shards.tail_ld : ld_in;
    auto colp = [&](int v, int c) -> const float4* {
        if (SPLIT) return reinterpret_cast<const float4*>(lbase + (int64_t)v * lstride);
        return rowp(v) + c;
    };
    constexpr bool GLOBAL = (MODE == M_SAGE_GLOBAL || MODE == M_GCN_GLOBAL);
    constexpr bool GCN = (MODE == M_GCN_LOCAL || MODE == M_GCN_GLOBAL);
    const int n = hg_load_count(d_n, cap);
    const int lane = threadIdx.x & 31;
    const int lr = lane & (LPR - 1);
    const int g0 = lane & ~(LPR - 1);
    const unsigned gmask = (LPR == 32) ? 0xffffffffu : (((1u << LPR) - 1u) << g0);
    const int groups_per_block = blockDim.x / LPR;
    for (int i0 = blockIdx.x * groups_per_block; i0 < n; i0 += gridDim.x * groups_per_block) {
        const int i = i0 + threadIdx.x / LPR;
        if (i >= n) continue;
        float4 acc[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        const bool skip = inj && inj[i];
        const int v = frontier[i];
        const int64_t sbase = (int64_t)i * f;
        if (!skip) {
            if (GLOBAL && self_out) {  // self row gather (the SAGE/GCN-free "gather" part)
                float4* dst = reinterpret_cast<float4*>(self_out + (int64_t)i * ld_self);
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int c = lr + k * LPR;
                    if (c < F4) dst[c] = __ldg(colp(v, c));
                }
            }
            const int cnt = counts[i];
            float wd = 0.f;
            if (!GCN) { const int ns = nself[i]; wd = ns > 0 ? 1.0f / (float)ns : 0.f; }
            for (int j0 = 0; j0 < cnt; j0 += LPR) {
                // lanes fetch up to LPR edge descriptors, then broadcast
                int my_row = -1;
                float my_w = 0.f;
                if (j0 + lr < cnt) {
                    const int sg = slot_g[sbase + j0 + lr];
                    const int sl = (GLOBAL && !GCN) ? 0 : slot_local[sbase + j0 + lr];  // SAGE bottom: global ids only
                    if (GCN) { my_row = GLOBAL ? sg : sl; my_w = gcn_w(outdeg[sl], cnt); }
                    else if (sg != v) { my_row = GLOBAL ? sg : sl; my_w = wd; }  // non-self edge
                }
                if (HG_AGG_PF && NV == 1 && !SH && my_row >= 0)
                    prefetch_row_l2(rowp(my_row), SPLIT ? shards.body4 : F4);  // split: tails are L2-persisting
                const int m = min(LPR, cnt - j0);
                // U rows in flight (a whole fanout-15 segment in one batch for F <= 128),
                // consumed in edge order; slots past m are masked
                constexpr int U = NV >= 8 ? 2 : (NV == 1 && LPR == 32) ? HG_AGG_U1 : 16 / NV;
                for (int j = 0; j < m; j += U) {
                    int r[U]; float w[U];
#pragma unroll
                    for (int t = 0; t < U; ++t) {
                        const int src = j + t < LPR ? j + t : LPR - 1;
                        const int rr = __shfl_sync(gmask, my_row, src, LPR);
                        w[t] = __shfl_sync(gmask, my_w, src, LPR);
                        r[t] = j + t < m ? rr : -1;
                    }
                    float4 x[U][NV];
#pragma unroll
                    for (int t = 0; t < U; ++t) {
                        const int rv = r[t] < 0 ? 0 : r[t];
#pragma unroll
                        for (int k = 0; k < NV; ++k) {
                            const int c = lr + k * LPR;
                            x[t][k] = (r[t] >= 0 && c < F4) ? __ldg(colp(rv, c)) : make_float4(0.f, 0.f, 0.f, 0.f);
                        }
                    }
#pragma unroll
                    for (int t = 0; t < U; ++t)
                        if (r[t] >= 0) {
#pragma unroll
                            for (int k = 0; k < NV; ++k) acc[k] = f4_fma(w[t], x[t][k], acc[k]);
                        }
                }
            }
        } else if (GLOBAL && self_out) {
            float4* dst = reinterpret_cast<float4*>(self_out + (int64_t)i * ld_self);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int c = lr + k * LPR;
                if (c < F4) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float4* out = reinterpret_cast<float4*>(agg_out + (int64_t)i * ld_agg);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lr + k * LPR;
            if (c < F4) out[c] = acc[k];
        }
    }
}

__global__ void k_swr_keys(const int64_t* __restrict__ edge_dst, long long n, uint32_t* __restrict__ keys,
                           int* __restrict__ vals) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
        keys[e] = (uint32_t)edge_dst[e];
        vals[e] = (int)e;
    }
}

__global__ void k_swr_bounds(const uint32_t* __restrict__ keys, long long n, int* __restrict__ beg,
                             int* __restrict__ end) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x) {
        const uint32_t key = keys[k];
        if (k == 0 || keys[k - 1] != key) beg[key] = (int)k;
        if (k == n - 1 || keys[k + 1] != key) end[key] = (int)(k + 1);
    }
}

__global__ void k_swr_rows(const int64_t* __restrict__ edge_src, const double* __restrict__ w,
                           const double* __restrict__ rows, int d, const int* __restrict__ order,
                           const int* __restrict__ beg, const int* __restrict__ end, int n_out,
                           double* __restrict__ out) {
    const int warps = (gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (int o = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; o < n_out; o += warps) {
        const int b = beg[o], e = end[o];
        for (int c = lane; c < d; c += 32) {
            double acc = 0.0;
            for (int k = b; k < e; ++k) {
                const int ed = order[k];
                acc = __dadd_rn(acc, __dmul_rn(w[ed], rows[edge_src[ed] * (int64_t)d + c]));
            }
            out[(int64_t)o * d + c] = acc;
        }
    }
}

// The bottom (global-id) aggregation grid is sized as one wave of CTAs
// (agg_ctas_per_sm() per SM); a wide-row instantiation whose registers allow
// fewer resident CTAs (k_agg_fwd<32,5,..> for C3's 602-float rows: 113
// registers, 2 per SM) is clamped to what fits, so it too runs as one wave:
// C3 bottom aggregation 80.9 -> 75.1 us (profiles/r02s_occupancy_sweep.md).
template <typename K>
void clamp_to_resident(cudaLaunchConfig_t& cfg, K kernel, int& per_sm) {  // per_sm: per-instantiation cache
    if (per_sm == 0) {
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, (int)cfg.blockDim.x,
                                                          cfg.dynamicSmemBytes) != cudaSuccess) {
            (void)cudaGetLastError();
            per_sm = -1;
        }
    }
    if (per_sm < 1) return;
    const unsigned cap = (unsigned)per_sm * HG_NUM_SMS;
    if (cfg.gridDim.x > cap) cfg.gridDim.x = cap;
}

template <int MODE, int AD = AD_PLAIN>
int launch_fwd(int LPR, int NV, dim3 g, cudaStream_t s, const float* hin, int ld_in, int F4, const int* frontier,
               const int* d_n, int cap, int f, const int* counts, const int* slot_g, const int* slot_local,
               const int* nself, const int* outdeg, const uint8_t* inj, float* self_out, int ld_self,
               float* agg_out, int ld_agg, const FeatShards& shards = FeatShards{}) {
    // bottom layer (rows by global id): persisting L2 window over the hot feature rows
    cudaLaunchAttribute attr[2];
    int na = 0;
    if ((MODE == M_SAGE_GLOBAL || MODE == M_GCN_GLOBAL) && hg_l2_window_attr(&attr[na])) ++na;
    if (hg_pdl_enabled()) {  // programmatic dependent launch (see hg_common.cuh)
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = g;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = s;
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
#define HG_FWD(L, V)                                                                                      \
    if (LPR == L && NV == V) {                                                                            \
        static int per_sm = 0;                                                                            \
        if (MODE == M_SAGE_GLOBAL || MODE == M_GCN_GLOBAL)                                                \
            clamp_to_resident(cfg, k_agg_fwd<L, V, MODE, AD>, per_sm);                                    \
        cudaLaunchKernelEx(&cfg, k_agg_fwd<L, V, MODE, AD>, hin, ld_in, F4, frontier, d_n, cap, f, counts, \
                           slot_g, slot_local, nself, outdeg, inj, self_out, ld_self, agg_out, ld_agg,    \
                           shards);                                                                        \
        return HG_OK;                                                                                     \
    }
    if constexpr (AD == AD_SPLIT) {  // split rows: one float4 per lane (F <= 128)
        HG_FWD(8, 1) HG_FWD(16, 1) HG_FWD(32, 1)
    } else {
        HG_FWD(8, 1) HG_FWD(16, 1) HG_FWD(32, 1) HG_FWD(32, 2) HG_FWD(32, 4) HG_FWD(32, 5) HG_FWD(32, 6)
        HG_FWD(32, 8)
    }
#undef HG_FWD
    return HG_EUNSUPPORTED;
}


// ---------------------------------------------------------------------------
// Wide rows (F > 128: C3's 602 features = 2.4 KB rows): the rows of a
// destination's edges are staged into shared memory by the TMA engine
// (cp.async.bulk global -> shared, one mbarrier per stage, complete_tx) instead
// of per-lane 128-bit loads.  One lane per warp keeps up to S rows in flight
// (S * 2.4 KB per warp, no register cost: the LDG loop holds 2 rows per warp in
// ~96 registers), running ahead into the warp's next destination; the warp
// consumes the rows in edge order from shared memory.  Same items, weights
// and FMA order as k_agg_fwd, so the outputs are bit-identical.
// ---------------------------------------------------------------------------
constexpr int BULK_WARPS = 4;

struct BulkDesc {
    int i, cnt, v, n_items;
    bool skip, self_item;
    unsigned valid;  // lanes j < cnt holding a consumed edge
    int row;         // this lane's edge row (slot j = lane), -1 if none
    float w;
};

template <int NV, int MODE>
__global__ void __launch_bounds__(BULK_WARPS * 32) k_agg_fwd_bulk(
    const float* __restrict__ hin, int ld_in, int F4, const int* __restrict__ frontier, const int* d_n, int cap,
    int f, const int* __restrict__ counts, const int* __restrict__ slot_g, const int* __restrict__ slot_local,
    const int* __restrict__ nself, const int* __restrict__ outdeg, const uint8_t* __restrict__ inj,
    float* __restrict__ self_out, int ld_self, float* __restrict__ agg_out, int ld_agg, int S, int stage_bytes) {
    using namespace hgtc;
    constexpr bool GLOBAL = (MODE == M_SAGE_GLOBAL || MODE == M_GCN_GLOBAL);
    constexpr bool GCN = (MODE == M_GCN_LOCAL || MODE == M_GCN_GLOBAL);
    extern __shared__ __align__(128) uint8_t sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* ring = sm + (size_t)warp * S * stage_bytes;
    uint64_t* bar = reinterpret_cast<uint64_t*>(sm + (size_t)BULK_WARPS * S * stage_bytes) + warp * S;
    if (lane == 0) {
        for (int st = 0; st < S; ++st) mbar_init(&bar[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncwarp();
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const uint32_t row_bytes = (uint32_t)F4 * 16u;

    auto load_desc = [&](int i, BulkDesc& d) {
        d.i = i < n ? i : -1;
        d.row = -1;
        d.w = 0.f;
        d.cnt = 0;
        d.skip = true;
        d.self_item = false;
        d.valid = 0u;
        d.n_items = 0;
        if (d.i < 0) return;
        d.skip = inj && inj[i];
        d.v = frontier[i];
        d.self_item = GLOBAL && self_out && !d.skip;
        if (!d.skip) {
            d.cnt = counts[i];
            const int64_t sbase = (int64_t)i * f;
            float wd = 0.f;
            if (!GCN) { const int ns = nself[i]; wd = ns > 0 ? 1.0f / (float)ns : 0.f; }
            if (lane < d.cnt) {
                const int sg = slot_g[sbase + lane];
                const int sl = (GLOBAL && !GCN) ? 0 : slot_local[sbase + lane];
                if (GCN) { d.row = GLOBAL ? sg : sl; d.w = gcn_w(outdeg[sl], d.cnt); }
                else if (sg != d.v) { d.row = GLOBAL ? sg : sl; d.w = wd; }
            }
        }
        d.valid = __ballot_sync(0xffffffffu, d.row >= 0);
        d.n_items = (d.self_item ? 1 : 0) + __popc(d.valid);
    };
    // row id of item t of descriptor d (uniform across the warp)
    auto item_row = [&](const BulkDesc& d, int t) -> int {
        if (d.self_item) {
            if (t == 0) return d.v;
            --t;
        }
        const int src = __fns(d.valid, 0, t + 1);
        return __shfl_sync(0xffffffffu, d.row, src);
    };
    auto issue = [&](const BulkDesc& d, int t, long long k) {
        const int r = item_row(d, t);
        if (lane == 0) {
            const int st = (int)(k % S);
            fence_proxy_async();  // the stage's previous generic reads before the async write
            mbar_expect_tx(&bar[st], row_bytes);
            bulk_load(smem_u32(ring + (size_t)st * stage_bytes), hin + (int64_t)r * ld_in, row_bytes, &bar[st]);
        }
    };

    const int gw = blockIdx.x * BULK_WARPS + warp, nw = gridDim.x * BULK_WARPS;
    BulkDesc cur, nxt;
    load_desc(gw, cur);
    load_desc(gw + nw, nxt);
    long long kp = 0, kc = 0;  // items produced / consumed by this warp
    int pd = 0, pt = 0;        // producer: descriptor (0 = cur, 1 = nxt), next item
    while (cur.i >= 0) {
        float4 acc[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) acc[k] = make_float4(0.f, 0.f, 0.f, 0.f);
        for (int t = 0; t < cur.n_items; ++t) {
            while (kp - kc < S) {  // keep up to S rows in flight, into the next destination
                if (pd == 0) {
                    if (pt < cur.n_items) { issue(cur, pt++, kp++); continue; }
                    pd = 1;
                    pt = 0;
                }
                if (pt < nxt.n_items) { issue(nxt, pt++, kp++); continue; }
                break;
            }
            const int st = (int)(kc % S);
            mbar_wait(&bar[st], (uint32_t)((kc / S) & 1));
            const float4* x = reinterpret_cast<const float4*>(ring + (size_t)st * stage_bytes);
            if (cur.self_item && t == 0) {  // the destination's own row (SAGE self term input)
                float4* dst = reinterpret_cast<float4*>(self_out + (int64_t)cur.i * ld_self);
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int c = lane + k * 32;
                    if (c < F4) dst[c] = x[c];
                }
            } else {
                const int te = t - (cur.self_item ? 1 : 0);
                const float w = __shfl_sync(0xffffffffu, cur.w, __fns(cur.valid, 0, te + 1));
#pragma unroll
                for (int k = 0; k < NV; ++k) {
                    const int c = lane + k * 32;
                    if (c < F4) acc[k] = f4_fma(w, x[c], acc[k]);
                }
            }
            __syncwarp();
            ++kc;
        }
        if (GLOBAL && self_out && cur.skip) {
            float4* dst = reinterpret_cast<float4*>(self_out + (int64_t)cur.i * ld_self);
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int c = lane + k * 32;
                if (c < F4) dst[c] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
        float4* out = reinterpret_cast<float4*>(agg_out + (int64_t)cur.i * ld_agg);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lane + k * 32;
            if (c < F4) out[c] = acc[k];
        }
        // the next destination becomes current; the producer keeps its position
        if (pd == 1) pd = 0;
        else pt = 0;
        cur = nxt;
        load_desc(cur.i < 0 ? n : cur.i + nw, nxt);
    }
}

// wide-row gather: bulk-copy staging on (hg_set_tuning key 12 = 1 or env
// HG_AGG_BULK=1) / the per-lane LDG loop (default: measured 2.4x faster at C3,
// profiles/r02_c3_wide_rows.md)
int g_agg_bulk = -1;
bool agg_bulk_enabled() {
    if (g_agg_bulk < 0) {
        const char* e = getenv("HG_AGG_BULK");
        g_agg_bulk = e ? (atoi(e) != 0) : 0;
    }
    return g_agg_bulk != 0;
}

// stages per warp for rows of row_bytes: fill ~2 CTAs x 100 KB per SM (env HG_BULK_STAGES)
int bulk_stages(int stage_bytes) {
    int S = (100 * 1024) / (BULK_WARPS * stage_bytes);
    if (const char* e = getenv("HG_BULK_STAGES")) S = atoi(e);
    return S < 2 ? 2 : (S > 32 ? 32 : S);
}

template <int MODE>
int launch_fwd_bulk(int F4, cudaStream_t s, const float* hin, int ld_in, const int* frontier, const int* d_n,
                    int cap, int f, const int* counts, const int* slot_g, const int* slot_local, const int* nself,
                    const int* outdeg, const uint8_t* inj, float* self_out, int ld_self, float* agg_out, int ld_agg) {
    const int stage_bytes = (F4 * 16 + 127) / 128 * 128;
    const int S = bulk_stages(stage_bytes);
    const size_t smem = (size_t)BULK_WARPS * S * stage_bytes + (size_t)BULK_WARPS * S * 8;
    if (smem > 227 * 1024) return HG_EUNSUPPORTED;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if ((MODE == M_SAGE_GLOBAL || MODE == M_GCN_GLOBAL) && hg_l2_window_attr(&attr[na])) ++na;
    if (hg_pdl_enabled()) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    cudaLaunchConfig_t cfg = {};
    const int per_sm = (int)((227 * 1024) / (smem + 1024));
    const long long need = ((long long)cap + BULK_WARPS - 1) / BULK_WARPS;
    long long grid = (long long)HG_NUM_SMS * (per_sm < 1 ? 1 : per_sm);
    cfg.gridDim = dim3((unsigned)(need < grid ? (need < 1 ? 1 : need) : grid));
    cfg.blockDim = dim3(BULK_WARPS * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cfg.attrs = na ? attr : nullptr;
    cfg.numAttrs = na;
#define HG_FWDB(V)                                                                                           \
    if (F4 <= 32 * V) {                                                                                      \
        static bool attr_set = false;                                                                        \
        if (!attr_set) {                                                                                     \
            cudaFuncSetAttribute(k_agg_fwd_bulk<V, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                                 227 * 1024);                                                                \
            attr_set = true;                                                                                 \
        }                                                                                                    \
        cudaLaunchKernelEx(&cfg, k_agg_fwd_bulk<V, MODE>, hin, ld_in, F4, frontier, d_n, cap, f, counts,      \
                           slot_g, slot_local, nself, outdeg, inj, self_out, ld_self, agg_out, ld_agg, S,    \
                           stage_bytes);                                                                     \
        return HG_OK;                                                                                        \
    }
    HG_FWDB(2) HG_FWDB(4) HG_FWDB(6) HG_FWDB(8)
#undef HG_FWDB
    return HG_EUNSUPPORTED;
}

// CTAs per SM of the bottom (global-id) aggregation grid: env HG_AGG_CTAS_PER_SM
// (default 5 = what fits at 48 registers: one wave, no tail)
int agg_ctas_per_sm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HG_AGG_CTAS_PER_SM");
        v = e ? atoi(e) : 5;
        v = v < 1 ? 1 : (v > 8 ? 8 : v);
    }
    return v;
}

void pick_lanes(int F4, int& LPR, int& NV);

// forward aggregation: wide rows (128 < F4 <= 192) get exactly the float4 columns
// they need per lane (C3's 602 features: 5 instead of 8), so each warp keeps 3
// rows in flight instead of 2 in about the same registers (C3 bottom aggregation
// 81.6 -> 79.0 us, profiles/r02_c3_tight_nv.txt)
void pick_lanes_fwd(int F4, int& LPR, int& NV) {
    pick_lanes(F4, LPR, NV);
    if (F4 > 128 && F4 <= 192) NV = F4 <= 160 ? 5 : 6;
}

void pick_lanes(int F4, int& LPR, int& NV) {
    if (F4 <= 8) { LPR = 8; NV = 1; }
    else if (F4 <= 16) { LPR = 16; NV = 1; }
    else if (F4 <= 32) { LPR = 32; NV = 1; }
    else if (F4 <= 64) { LPR = 32; NV = 2; }
    else if (F4 <= 128) { LPR = 32; NV = 4; }
    else { LPR = 32; NV = 8; }
}

}  // namespace

void hg_set_agg_bulk(int v) { g_agg_bulk = v ? 1 : 0; }

// model: 0 = SAGE (mean over non-self sampled neighbours), 1 = GCN (block sym-norm).
// global_src: 1 = rows addressed by global id (bottom layer, reads the feature
// table), 0 = by local src id (upper layers, reads the previous activation).
// F: columns (multiple of 4; pad the row stride ld_* to a multiple of 4).
extern "C" int hg_aggregate_fwd(int32_t model, int32_t global_src, const float* hin, int32_t ld_in, int32_t F,
                                const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                                const int32_t* counts, const int32_t* slot_g, const int32_t* slot_local,
                                const int32_t* nself, const int32_t* outdeg, const uint8_t* inj_mask,
                                float* self_out, int32_t ld_self, float* agg_out, int32_t ld_agg, void* stream) {
    if (F % 4 || ld_in % 4 || ld_agg % 4 || (self_out && ld_self % 4)) {
        hg_set_error("aggregate_fwd: F and row strides must be multiples of 4");
        return HG_EINVAL;
    }
    if (F > 1024) { hg_set_error("aggregate_fwd: F > 1024 unsupported"); return HG_EUNSUPPORTED; }
    if (cap_dst == 0) return HG_OK;
    const int F4 = F / 4;
    int LPR, NV;
    pick_lanes_fwd(F4, LPR, NV);
    dim3 g(hg_grid((long long)cap_dst * LPR, 256, global_src ? agg_ctas_per_sm() : 8));
    cudaStream_t s = (cudaStream_t)stream;
    int rc;
    const int mode = (model ? 2 : 0) + (global_src ? 1 : 0);
    if (F4 > 32 && F4 <= 256 && fanout <= 32 && agg_bulk_enabled()) {  // wide rows: TMA bulk-copy staging
        switch (mode) {
            case M_SAGE_LOCAL: rc = launch_fwd_bulk<M_SAGE_LOCAL>(F4, s, hin, ld_in, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
            case M_SAGE_GLOBAL: rc = launch_fwd_bulk<M_SAGE_GLOBAL>(F4, s, hin, ld_in, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
            case M_GCN_LOCAL: rc = launch_fwd_bulk<M_GCN_LOCAL>(F4, s, hin, ld_in, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
            default: rc = launch_fwd_bulk<M_GCN_GLOBAL>(F4, s, hin, ld_in, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
        }
        if (rc == HG_OK) return hg_check_launch("aggregate_fwd(bulk)");
    }
    switch (mode) {
        case M_SAGE_LOCAL: rc = launch_fwd<M_SAGE_LOCAL>(LPR, NV, g, s, hin, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
        case M_SAGE_GLOBAL: rc = launch_fwd<M_SAGE_GLOBAL>(LPR, NV, g, s, hin, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
        case M_GCN_LOCAL: rc = launch_fwd<M_GCN_LOCAL>(LPR, NV, g, s, hin, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
        default: rc = launch_fwd<M_GCN_GLOBAL>(LPR, NV, g, s, hin, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg); break;
    }
    if (rc) { hg_set_error("aggregate_fwd: unsupported width"); return rc; }
    return hg_check_launch("aggregate_fwd");
}

// hg_aggregate_fwd for the bottom layer with the feature table row-sharded over
// devices: shard_ptrs (host array of n_shards device pointers: peer pointers from
// hg_ipc_open_handle, or slices of one table) each hold rows_per_shard rows of
// stride ld_in.  Same outputs, bit for bit, as the unsharded call.
extern "C" int hg_aggregate_fwd_sharded(int32_t model, const float* const* shard_ptrs, int32_t n_shards,
                                        int32_t rows_per_shard, int32_t ld_in, int32_t F, const int32_t* frontier,
                                        const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                                        const int32_t* counts, const int32_t* slot_g, const int32_t* slot_local,
                                        const int32_t* nself, const int32_t* outdeg, const uint8_t* inj_mask,
                                        float* self_out, int32_t ld_self, float* agg_out, int32_t ld_agg,
                                        void* stream) {
    if (n_shards < 1 || n_shards > HG_MAX_SHARDS || rows_per_shard < 1) {
        hg_set_error("aggregate_fwd_sharded: 1..%d shards with rows_per_shard >= 1", HG_MAX_SHARDS);
        return HG_EINVAL;
    }
    if (F % 4 || ld_in % 4 || ld_agg % 4 || (self_out && ld_self % 4)) {
        hg_set_error("aggregate_fwd_sharded: F and row strides must be multiples of 4");
        return HG_EINVAL;
    }
    if (F > 1024) { hg_set_error("aggregate_fwd_sharded: F > 1024 unsupported"); return HG_EUNSUPPORTED; }
    if (cap_dst == 0) return HG_OK;
    FeatShards sh{};
    for (int i = 0; i < n_shards; ++i) {
        if (!shard_ptrs[i] || (reinterpret_cast<uintptr_t>(shard_ptrs[i]) & 15)) {
            hg_set_error("aggregate_fwd_sharded: shard %d pointer null or not 16-byte aligned", i);
            return HG_EINVAL;
        }
        sh.base[i] = shard_ptrs[i];
    }
    sh.n = n_shards;
    sh.rows_per_shard = rows_per_shard;
    const int F4 = F / 4;
    int LPR, NV;
    pick_lanes_fwd(F4, LPR, NV);
    dim3 g(hg_grid((long long)cap_dst * LPR, 256, agg_ctas_per_sm()));
    cudaStream_t s = (cudaStream_t)stream;
    const int rc = model ? launch_fwd<M_GCN_GLOBAL, AD_SHARDED>(LPR, NV, g, s, nullptr, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg, sh)
                         : launch_fwd<M_SAGE_GLOBAL, AD_SHARDED>(LPR, NV, g, s, nullptr, ld_in, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg, sh);
    if (rc) { hg_set_error("aggregate_fwd_sharded: unsupported width"); return rc; }
    return hg_check_launch("aggregate_fwd_sharded");
}

// hg_aggregate_fwd for the bottom layer over a split-row copy of the feature
// table: columns [0, body_cols) of row v at body + v * ld_body (ld_body a
// multiple of 32 floats and body 128-byte aligned, so a row's body is whole
// 128-byte lines), columns [body_cols, F) at tail + v * ld_tail.  A 100-float
// (400-byte) row otherwise always touches four 128-byte lines; split, it
// touches three lines of the body plus a 16-byte tail whose table (V x 16 B)
// is held in L2 by the persisting window (DeviceGraph.persist_hot_rows).  The
// gather's DRAM cost is per line touched (profiles/r02s_gather_rowsize.txt).
// Same items, weights and FMA order as hg_aggregate_fwd: bit-identical outputs.
extern "C" int hg_aggregate_fwd_split(int32_t model, const float* body, int32_t ld_body, const float* tail,
                                      int32_t ld_tail, int32_t body_cols, int32_t F, const int32_t* frontier,
                                      const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                                      const int32_t* counts, const int32_t* slot_g, const int32_t* slot_local,
                                      const int32_t* nself, const int32_t* outdeg, const uint8_t* inj_mask,
                                      float* self_out, int32_t ld_self, float* agg_out, int32_t ld_agg,
                                      void* stream) {
    if (F % 4 || body_cols % 4 || ld_body % 4 || ld_tail % 4 || ld_agg % 4 || (self_out && ld_self % 4)) {
        hg_set_error("aggregate_fwd_split: F, body_cols and row strides must be multiples of 4");
        return HG_EINVAL;
    }
    if (body_cols <= 0 || body_cols >= F || ld_body < body_cols || ld_tail < F - body_cols || !body || !tail ||
        (reinterpret_cast<uintptr_t>(body) & 15) || (reinterpret_cast<uintptr_t>(tail) & 15)) {
        hg_set_error("aggregate_fwd_split: need 0 < body_cols < F, ld_body >= body_cols, ld_tail >= F - body_cols, "
                     "16-byte aligned tables");
        return HG_EINVAL;
    }
    if (F > 128) { hg_set_error("aggregate_fwd_split: F > 128 unsupported"); return HG_EUNSUPPORTED; }
    if (cap_dst == 0) return HG_OK;
    FeatShards sh{};
    sh.tail = tail;
    sh.tail_ld = ld_tail;
    sh.body4 = body_cols / 4;
    const int F4 = F / 4;
    int LPR, NV;
    pick_lanes_fwd(F4, LPR, NV);
    dim3 g(hg_grid((long long)cap_dst * LPR, 256, agg_ctas_per_sm()));
    cudaStream_t s = (cudaStream_t)stream;
    const int rc = model ? launch_fwd<M_GCN_GLOBAL, AD_SPLIT>(LPR, NV, g, s, body, ld_body, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg, sh)
                         : launch_fwd<M_SAGE_GLOBAL, AD_SPLIT>(LPR, NV, g, s, body, ld_body, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, inj_mask, self_out, ld_self, agg_out, ld_agg, sh);
    if (rc) { hg_set_error("aggregate_fwd_split: unsupported width"); return rc; }
    return hg_check_launch("aggregate_fwd_split");
}

extern "C" int64_t hg_swr_ws_size(int64_t n_edges, int32_t n_out) {
    return (int64_t)(4 * n_edges + 2 * (long long)n_out + (long long)hg_radix_ws_ints(n_edges) + 16);
}

// fp64 segment_weighted_rows (kernels.py:121-144), bit-identical to the
// reference's numba loop / np.add.at for any edge order.
extern "C" int hg_segment_weighted_rows_f64(const int64_t* edge_src, const int64_t* edge_dst, const double* w,
                                            int64_t n_edges, const double* rows, int32_t d, int32_t n_out,
                                            double* out, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    cudaMemsetAsync(out, 0, sizeof(double) * (size_t)n_out * d, s);
    if (n_edges == 0 || n_out == 0 || d == 0) return hg_check_launch("swr(empty)");
    const long long n = n_edges;
    uint32_t* keys = (uint32_t*)ws;
    int* vals = ws + n;
    uint32_t* k_alt = (uint32_t*)(ws + 2 * n);
    int* beg = ws + 3 * n;
    int* end = beg + n_out;
    int* rws = end + n_out;
    int* v_alt = rws + hg_radix_ws_ints(n);
    cudaMemsetAsync(beg, 0, sizeof(int) * 2 * (size_t)n_out, s);
    int bits = 1;
    while ((1u << bits) < (uint32_t)n_out && bits < 32) ++bits;
    k_swr_keys<<<hg_grid(n, 256, 8), 256, 0, s>>>(edge_dst, n, keys, vals);
    int in_alt = 0;
    int rc = hg_radix_sort_launch(keys, vals, k_alt, v_alt, n, bits, rws, &in_alt, s);
    if (rc) return rc;
    const uint32_t* sk = in_alt ? k_alt : keys;
    const int* sv = in_alt ? v_alt : vals;
    k_swr_bounds<<<hg_grid(n, 256, 8), 256, 0, s>>>(sk, n, beg, end);
    k_swr_rows<<<hg_grid((long long)n_out * 32, 256, 8), 256, 0, s>>>(edge_src, w, rows, d, sv, beg, end, n_out, out);
    return hg_check_launch("segment_weighted_rows_f64");
}

// ---------------------------------------------------------------------------
// Transposed aggregation by deterministic scatter (layers >= 1; replaces the
// CSC gather above on the default path).  The reference scatters
// segment_weighted_rows(ed, es, w, dz W^T) over the edges (gnnmath.py:140,199);
// here every destination row of dagg is read once (coalesced, in the slot
// form the forward uses) and its weighted copies are added into a FIXED-POINT
// int64 accumulator per (src, column) with integer atomics.  Integer addition
// is associative, so the result is bit-identical for any execution order
// (eager = graph replay = pipelined) with no sort and no src-major view: the
// whole per-layer CSC build (radix sort + scans + bounds + weights, ~10
// kernels) leaves the sampling graph.
//
// Two-word fixed point: a contribution v (fp32) is split exactly into
// hi = round(v * 2^20) and lo = round((v - hi * 2^-20) * 2^60), accumulated in
// two independent int64 words (the row's hi words, then its lo words: an
// accumulator row is 2F words).  Range |sum| < 2^43, resolution 2^-60 (every
// fp32 contribution >= 2^-37 in magnitude is represented exactly, smaller ones
// to 2^-61 absolute), so the sum is the exact sum of the contributions up to
// one final rounding, for any gradient scale that fp32 itself represents.
// d_flags bit 0: a non-finite contribution (the reference's non-finite guard,
// gnnmath.py:100-102); bit 1: outdeg(s) * |v| >= 2^42, i.e. the source's sum
// could leave the accumulator's range (|v| of order 1e12 — a diverged run).
// The finish pass converts, adds the SAGE self term, applies the lower
// layer's ReLU' / injected-row masks, writes dx, and clears the accumulator
// for the next step.
// ---------------------------------------------------------------------------
namespace {
constexpr double FX_HI = 1048576.0;                 // 2^20
constexpr double FX_HI_INV = 1.0 / 1048576.0;
constexpr double FX_LO = 1152921504606846976.0;     // 2^60
constexpr double FX_LO_INV = 1.0 / 1152921504606846976.0;
constexpr float FX_RANGE = 4398046511104.0f;        // 2^42: bound on outdeg * |v|

// row = the source's accumulator row (2F words), k = column
__device__ __forceinline__ void fx_add(unsigned long long* row, int F, int k, float v, int od, int& flags) {
    if (!isfinite(v)) { flags |= 1; return; }
    if (!(fabsf(v) * (float)od < FX_RANGE)) flags |= 2;
    const double d = (double)v;
    const long long hi = __double2ll_rn(d * FX_HI);
    const long long lo = __double2ll_rn((d - (double)hi * FX_HI_INV) * FX_LO);
    atomicAdd(row + k, (unsigned long long)hi);
    if (lo) atomicAdd(row + F + k, (unsigned long long)lo);
}

__device__ __forceinline__ float fx_value(unsigned long long hi, unsigned long long lo) {
    return (float)((double)(long long)hi * FX_HI_INV + (double)(long long)lo * FX_LO_INV);
}

__device__ __forceinline__ int finite_flag(float4 a) {
    return (isfinite(a.x) && isfinite(a.y) && isfinite(a.z) && isfinite(a.w)) ? 0 : 1;
}

// Sources s >= n_dst with exactly one incoming transposed edge (outdeg[s] == 1;
// most of them: ~1.15 edges per source at C2) take the single-contribution fast
// path: the final dx row (ReLU' and injected-row masks applied) is stored
// directly, with no accumulator round trip.  Everything else accumulates in
// fixed point and is finished by k_bwd_finish.
__device__ __forceinline__ float4 bwd_mask(float4 a, const float* __restrict__ hmask, int ld_hmask, int s, int c,
                                           bool zero_row) {
    if (hmask) {  // ReLU' of the layer below: z > 0  <=>  relu(z) > 0
        const float4 h = __ldg(reinterpret_cast<const float4*>(hmask + (int64_t)s * ld_hmask) + c);
        a.x = h.x > 0.f ? a.x : 0.f; a.y = h.y > 0.f ? a.y : 0.f;
        a.z = h.z > 0.f ? a.z : 0.f; a.w = h.w > 0.f ? a.w : 0.f;
    }
    if (zero_row) a = make_float4(0.f, 0.f, 0.f, 0.f);
    return a;
}

template <int LPR, int NV, bool GCN>
__global__ void __launch_bounds__(256) k_bwd_scatter(
    const float* __restrict__ dagg, int ld_dagg, int F4, const int* __restrict__ frontier, const int* d_n_dst,
    int cap_dst, int f, const int* __restrict__ counts, const int* __restrict__ slot_g,
    const int* __restrict__ slot_local, const int* __restrict__ nself, const int* __restrict__ outdeg,
    unsigned long long* __restrict__ acc, int* __restrict__ d_flags, const float* __restrict__ hmask, int ld_hmask,
    const uint8_t* __restrict__ inj, float* __restrict__ dx, int ld_dx) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n_dst, cap_dst);
    const int lane = threadIdx.x & 31;
    const int lr = lane & (LPR - 1);
    const int groups_per_block = blockDim.x / LPR;
    const int F = F4 * 4;
    int bad = 0;
    // one lane group per SLOT (edge), not per destination: the ~f dependent
    // loads of a destination's edge loop (slot -> outdeg / mask -> store) run in
    // parallel across groups; the destination's dagg row is re-read per edge
    // from L2.
    const long long Q = (long long)n * f;
    for (long long q0 = (long long)blockIdx.x * groups_per_block; q0 < Q; q0 += (long long)gridDim.x * groups_per_block) {
        const long long q = q0 + threadIdx.x / LPR;
        if (q >= Q) continue;
        const int d = (int)(q / f), j = (int)(q - (long long)d * f);
        // round 1: everything that depends only on the slot (issued before any
        // branch; slots past the destination's count hold stale ids, unused)
        const int cnt = counts[d];
        const int s = slot_local[q];
        const int sg = GCN ? 0 : slot_g[q];
        const int fd = GCN ? 0 : frontier[d];
        const int ns = GCN ? 0 : nself[d];
        float4 x[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lr + k * LPR;
            x[k] = c < F4 ? __ldg(reinterpret_cast<const float4*>(dagg + (int64_t)d * ld_dagg) + c)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        if (j >= cnt) continue;
        if (!GCN && sg == fd) continue;  // SAGE drops self edges (gnnmath.py:148)
        // round 2: the source's out-degree, ReLU' mask row and injected flag together
        const int od = outdeg[s];
        const bool zero_row = inj && inj[s];
        float4 h[NV];
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lr + k * LPR;
            h[k] = (hmask && c < F4) ? __ldg(reinterpret_cast<const float4*>(hmask + (int64_t)s * ld_hmask) + c)
                                     : make_float4(1.f, 1.f, 1.f, 1.f);
        }
        const float w = GCN ? gcn_w(od, cnt) : (ns > 0 ? 1.0f / (float)ns : 0.f);
        if (s >= n && od == 1) {  // single contribution: final row, no accumulator
#pragma unroll
            for (int k = 0; k < NV; ++k) {
                const int c = lr + k * LPR;
                if (c < F4) {
                    float4 a = make_float4(w * x[k].x, w * x[k].y, w * x[k].z, w * x[k].w);
                    bad |= finite_flag(a);
                    a.x = h[k].x > 0.f ? a.x : 0.f; a.y = h[k].y > 0.f ? a.y : 0.f;
                    a.z = h[k].z > 0.f ? a.z : 0.f; a.w = h[k].w > 0.f ? a.w : 0.f;
                    if (zero_row) a = make_float4(0.f, 0.f, 0.f, 0.f);
                    reinterpret_cast<float4*>(dx + (int64_t)s * ld_dx)[c] = a;
                }
            }
            continue;
        }
        unsigned long long* row = acc + (int64_t)s * 2 * F;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lr + k * LPR;
            if (c < F4) {
                fx_add(row, F, 4 * c + 0, w * x[k].x, od, bad);
                fx_add(row, F, 4 * c + 1, w * x[k].y, od, bad);
                fx_add(row, F, 4 * c + 2, w * x[k].z, od, bad);
                fx_add(row, F, 4 * c + 3, w * x[k].w, od, bad);
            }
        }
    }
    if (bad && d_flags) atomicOr(d_flags, bad);
}

template <int LPR, int NV>
__global__ void __launch_bounds__(256) k_bwd_finish(
    unsigned long long* __restrict__ acc, int F4, const float* __restrict__ dself, int ld_dself, const int* d_n_dst,
    int cap_dst, const int* d_n_src, int cap_src, const int* __restrict__ outdeg, const float* __restrict__ hmask,
    int ld_hmask, const uint8_t* __restrict__ inj, float* __restrict__ dx, int ld_dx) {
    hg_pdl_begin();
    const int n_src = hg_load_count(d_n_src, cap_src);
    const int n_dst = hg_load_count(d_n_dst, cap_dst);
    const int lane = threadIdx.x & 31;
    const int lr = lane & (LPR - 1);
    const int groups_per_block = blockDim.x / LPR;
    const int F = F4 * 4;
    for (int s0 = blockIdx.x * groups_per_block; s0 < n_src; s0 += gridDim.x * groups_per_block) {
        const int s = s0 + threadIdx.x / LPR;
        if (s >= n_src) continue;
        if (s >= n_dst && outdeg[s] == 1) continue;  // written by the scatter's fast path
        const bool zero_row = inj && inj[s];
        ulonglong4* arow = reinterpret_cast<ulonglong4*>(acc + (int64_t)s * 2 * F);
        ulonglong4* lrow = arow + F4;
        float4* out = reinterpret_cast<float4*>(dx + (int64_t)s * ld_dx);
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            const int c = lr + k * LPR;
            if (c >= F4) continue;
            const ulonglong4 q = arow[c], r = lrow[c];
            arow[c] = make_ulonglong4(0ull, 0ull, 0ull, 0ull);
            lrow[c] = make_ulonglong4(0ull, 0ull, 0ull, 0ull);
            float4 a = make_float4(fx_value(q.x, r.x), fx_value(q.y, r.y), fx_value(q.z, r.z), fx_value(q.w, r.w));
            if (dself && s < n_dst) {  // dx[:n_dst] = dz W_self^T + scatter (gnnmath.py:195-199)
                const float4 ds = __ldg(reinterpret_cast<const float4*>(dself + (int64_t)s * ld_dself) + c);
                a.x = ds.x + a.x; a.y = ds.y + a.y; a.z = ds.z + a.z; a.w = ds.w + a.w;
            }
            out[c] = bwd_mask(a, hmask, ld_hmask, s, c, zero_row);
        }
    }
}

template <bool GCN>
int launch_scatter(int LPR, int NV, dim3 g, dim3 g2, cudaStream_t s, const float* dagg, int ld_dagg,
                   const float* dself, int ld_dself, int F4, const int* frontier, const int* d_n_dst, int cap_dst,
                   int f, const int* counts, const int* slot_g, const int* slot_local, const int* nself,
                   const int* outdeg, const int* d_n_src, int cap_src, const float* hmask, int ld_hmask,
                   const uint8_t* inj, unsigned long long* acc, float* dx, int ld_dx, int* d_flags) {
#define HG_SC(L, V)                                                                                            \
    if (LPR == L && NV == V) {                                                                                 \
        hg_launch(k_bwd_scatter<L, V, GCN>, g, 256, 0, s, dagg, ld_dagg, F4, frontier, d_n_dst, cap_dst, f, counts,   \
                                                   slot_g, slot_local, nself, outdeg, acc, d_flags, hmask,     \
                                                   ld_hmask, inj, dx, ld_dx);                                  \
        hg_launch(k_bwd_finish<L, V>, g2, 256, 0, s, acc, F4, dself, ld_dself, d_n_dst, cap_dst, d_n_src, cap_src,    \
                                              outdeg, hmask, ld_hmask, inj, dx, ld_dx);                        \
        return HG_OK;                                                                                          \
    }
    HG_SC(8, 1) HG_SC(16, 1) HG_SC(32, 1) HG_SC(32, 2) HG_SC(32, 4) HG_SC(32, 8)
#undef HG_SC
    return HG_EUNSUPPORTED;
}
}  // namespace

extern "C" int hg_aggregate_bwd_scatter(int32_t model, const float* dagg, int32_t ld_dagg, const float* dself,
                                        int32_t ld_dself, int32_t F, const int32_t* frontier, const int32_t* d_n_dst,
                                        int32_t cap_dst, int32_t fanout, const int32_t* counts, const int32_t* slot_g,
                                        const int32_t* slot_local, const int32_t* nself, const int32_t* outdeg,
                                        const int32_t* d_n_src, int32_t cap_src, const float* hmask,
                                        int32_t ld_hmask, const uint8_t* inj_mask, int64_t* acc_ws, float* dx,
                                        int32_t ld_dx, int32_t* d_flags, void* stream) {
    if (F % 4 || ld_dagg % 4 || ld_dx % 4 || (dself && ld_dself % 4) || (hmask && ld_hmask % 4)) {
        hg_set_error("aggregate_bwd_scatter: widths must be multiples of 4");
        return HG_EINVAL;
    }
    if (F > 1024) { hg_set_error("aggregate_bwd_scatter: F > 1024 unsupported"); return HG_EUNSUPPORTED; }
    if (cap_src == 0) return HG_OK;
    if (!outdeg) { hg_set_error("aggregate_bwd_scatter: needs the per-source edge counts (outdeg)"); return HG_EINVAL; }
    const int F4 = F / 4;
    int LPR, NV;
    pick_lanes(F4, LPR, NV);
    dim3 g(hg_grid((long long)(cap_dst > 0 ? cap_dst : 1) * fanout * LPR, 256, 8));  // one group per slot
    dim3 g2(hg_grid((long long)cap_src * LPR, 256, 8));
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(acc_ws);
    const int rc = model ? launch_scatter<true>(LPR, NV, g, g2, s, dagg, ld_dagg, dself, ld_dself, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, d_n_src, cap_src, hmask, ld_hmask, inj_mask, acc, dx, ld_dx, d_flags)
                         : launch_scatter<false>(LPR, NV, g, g2, s, dagg, ld_dagg, dself, ld_dself, F4, frontier, d_n_dst, cap_dst, fanout, counts, slot_g, slot_local, nself, outdeg, d_n_src, cap_src, hmask, ld_hmask, inj_mask, acc, dx, ld_dx, d_flags);
    if (rc) { hg_set_error("aggregate_bwd_scatter: unsupported width"); return rc; }
    return hg_check_launch("aggregate_bwd_scatter");
}

// ---------------------------------------------------------------------------
// Top SAGE layer in ONE kernel (the chain agg -> transform -> softmax-CE ->
// dX -> transposed scatter of the top layer, gnnmath.py:157-200 +
// 263-274, one warp per seed row): each warp gathers the mean of its
// destination's non-self neighbours (local ids) and its self row, computes the
// logits against [W_self; W_neigh] held in shared memory (fp32 FMA, k order),
// the softmax / loss / dlogits, then dself = dlogits W_self^T and
// dmean = dlogits W_neigh^T, and scatters w * dmean into the layer below
// (single-contribution fast path / fixed-point accumulator, as k_bwd_scatter).
// Outputs: mean rows and dlogits (for the weight gradients), dself rows (for the
// finish pass), logits, per-row losses with a last-block fixed-order mean.
// Replaces five dependent launches on the training critical path.
// ---------------------------------------------------------------------------
namespace {
constexpr int TOP_THREADS = 256;

// W [rows x N] (row-major, global) -> shared memory with row stride NS, 8 loads
// in flight per thread (a CTA-wide staging that otherwise costs one L2 round trip
// per element slot)
__device__ __forceinline__ void stage_w(float* sW, const float* __restrict__ W, int rows, int N, int NS) {
    const int total = rows * N;
    for (int e0 = threadIdx.x; e0 < total; e0 += 8 * TOP_THREADS) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * TOP_THREADS;
            v[u] = e < total ? __ldg(W + e) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int e = e0 + u * TOP_THREADS;
            if (e < total) sW[(e / N) * NS + e % N] = v[u];
        }
    }
}

__global__ void __launch_bounds__(TOP_THREADS) k_sage_top(
    const float* __restrict__ hin, int ld_in, int K, const int* __restrict__ frontier, const int* d_n, int cap, int f,
    const int* __restrict__ counts, const int* __restrict__ slot_g, const int* __restrict__ slot_local,
    const int* __restrict__ nself, const int* __restrict__ outdeg, const float* __restrict__ W, int C,
    const int* __restrict__ labels, const int* __restrict__ seeds, const int* __restrict__ d_div,
    float* __restrict__ logits, int ld_c, float* __restrict__ dlogits, float* __restrict__ agg_out, int ld_agg,
    float* __restrict__ dself_out, int ld_dself, const float* __restrict__ hmask, int ld_hmask,
    const uint8_t* __restrict__ inj, unsigned long long* __restrict__ acc, int F_acc, float* __restrict__ dx,
    int ld_dx, int* __restrict__ d_flags, float* __restrict__ row_loss, float* __restrict__ d_loss) {
    extern __shared__ float sW[];  // [2K][C]: W_self rows then W_neigh rows
    __shared__ double s_part[TOP_THREADS / 32];
    __shared__ bool s_last;
    const int CS = C | 1;  // odd row stride: conflict-free column walks in the dX loop
    // the weights were last written by the previous step's update, long complete:
    // staged before griddepcontrol.wait, overlapping the previous kernel's tail
    stage_w(sW, W, 2 * K, C, CS);
    __syncthreads();
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const float grad_scale = 1.0f / (float)(d_div ? *d_div : (n > 0 ? n : 1));
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * TOP_THREADS) >> 5;
    const float* Ws = sW;
    const float* Wn = sW + K * CS;
    int bad = 0;
    for (int i = (blockIdx.x * TOP_THREADS + threadIdx.x) >> 5; i < n; i += nw) {
        const int y = labels[seeds ? seeds[i] : i];  // issued early: two dependent loads
        const int cnt = counts[i];
        const int v = frontier[i];
        const int ns = nself[i];
        const float wd = ns > 0 ? 1.0f / (float)ns : 0.f;
        const int64_t sb = (int64_t)i * f;
        // ---- self row (local id i) and the mean of the non-self neighbours, edge order
        const int k0 = lane, k1 = lane + 32;
        const float s0 = k0 < K ? hin[(int64_t)i * ld_in + k0] : 0.f;
        const float s1 = k1 < K ? hin[(int64_t)i * ld_in + k1] : 0.f;
        // lane j < cnt holds edge j: local source (-1 for the self edge) and its out-degree
        int my_s = -1, my_od = 0;
        if (lane < cnt) {
            my_s = slot_local[sb + lane];
            if (slot_g[sb + lane] == v) my_s = -1;  // SAGE drops self edges (gnnmath.py:148)
            else my_od = outdeg[my_s];
        }
        float m0 = 0.f, m1 = 0.f;
        for (int j0 = 0; j0 < cnt; j0 += 8) {  // 8 neighbour rows in flight, summed in edge order
            float x0[8], x1[8];
            int sj[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                sj[u] = __shfl_sync(0xffffffffu, my_s, (j0 + u) & 31);
                if (j0 + u >= cnt) sj[u] = -1;
                x0[u] = (sj[u] >= 0 && k0 < K) ? hin[(int64_t)sj[u] * ld_in + k0] : 0.f;
                x1[u] = (sj[u] >= 0 && k1 < K) ? hin[(int64_t)sj[u] * ld_in + k1] : 0.f;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u)
                if (sj[u] >= 0) { m0 = fmaf(wd, x0[u], m0); m1 = fmaf(wd, x1[u], m1); }
        }
        if (k0 < K) agg_out[(int64_t)i * ld_agg + k0] = m0;
        if (k1 < K) agg_out[(int64_t)i * ld_agg + k1] = m1;
        // ---- logits: z[c] = sum_k self[k] W_self[k][c] + sum_k mean[k] W_neigh[k][c]
        const int c0 = lane, c1 = lane + 32;
        float z0 = 0.f, z1 = 0.f;
        const int cc0 = c0 < C ? c0 : 0, cc1 = c1 < C ? c1 : 0;  // clamped smem columns (results masked)
#pragma unroll 8
        for (int k = 0; k < K; ++k) {
            const float a = __shfl_sync(0xffffffffu, k < 32 ? s0 : s1, k & 31);
            z0 = fmaf(a, Ws[k * CS + cc0], z0);
            z1 = fmaf(a, Ws[k * CS + cc1], z1);
        }
#pragma unroll 8
        for (int k = 0; k < K; ++k) {
            const float b = __shfl_sync(0xffffffffu, k < 32 ? m0 : m1, k & 31);
            z0 = fmaf(b, Wn[k * CS + cc0], z0);
            z1 = fmaf(b, Wn[k * CS + cc1], z1);
        }
        if (c0 < C) logits[(int64_t)i * ld_c + c0] = z0;
        if (c1 < C) logits[(int64_t)i * ld_c + c1] = z1;
        // ---- softmax cross-entropy (gnnmath.py:263-274)
        float mx = fmaxf(c0 < C ? z0 : -INFINITY, c1 < C ? z1 : -INFINITY);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float e0 = c0 < C ? expf(z0 - mx) : 0.f, e1 = c1 < C ? expf(z1 - mx) : 0.f;
        float se = e0 + e1;
#pragma unroll
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const float zy = __shfl_sync(0xffffffffu, y < 32 ? z0 : z1, y & 31);
        const float inv = 1.f / se;
        const float d0 = c0 < C ? (e0 * inv - (c0 == y ? 1.f : 0.f)) * grad_scale : 0.f;
        const float d1 = c1 < C ? (e1 * inv - (c1 == y ? 1.f : 0.f)) * grad_scale : 0.f;
        if (c0 < C) dlogits[(int64_t)i * ld_c + c0] = d0;
        if (c1 < C) dlogits[(int64_t)i * ld_c + c1] = d1;
        if (lane == 0) row_loss[i] = logf(se) - (zy - mx);
        // ---- dself = dlogits W_self^T, dmean = dlogits W_neigh^T (lane owns k0, k1)
        float ds0 = 0.f, ds1 = 0.f, dm0 = 0.f, dm1 = 0.f;
        const int kk0 = k0 < K ? k0 : 0, kk1 = k1 < K ? k1 : 0;
#pragma unroll 8
        for (int c = 0; c < C; ++c) {
            const float dl = __shfl_sync(0xffffffffu, c < 32 ? d0 : d1, c & 31);
            ds0 = fmaf(dl, Ws[kk0 * CS + c], ds0);
            dm0 = fmaf(dl, Wn[kk0 * CS + c], dm0);
            ds1 = fmaf(dl, Ws[kk1 * CS + c], ds1);
            dm1 = fmaf(dl, Wn[kk1 * CS + c], dm1);
        }
        if (k0 < K) dself_out[(int64_t)i * ld_dself + k0] = ds0;
        if (k1 < K) dself_out[(int64_t)i * ld_dself + k1] = ds1;
        // ---- transposed scatter of w * dmean into the layer below (as k_bwd_scatter)
        const float a0 = wd * dm0, a1 = wd * dm1;
        if (cnt > 0 && !(isfinite(a0) && isfinite(a1))) bad |= 1;
        for (int j0 = 0; j0 < cnt; j0 += 8) {  // 8 edges at a time: their masks load together
            int sj[8], od[8];
            float h0[8], h1[8];
            bool zr[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                sj[u] = __shfl_sync(0xffffffffu, my_s, (j0 + u) & 31);
                od[u] = __shfl_sync(0xffffffffu, my_od, (j0 + u) & 31);
                if (j0 + u >= cnt) sj[u] = -1;
                const bool fast = sj[u] >= n && od[u] == 1;
                h0[u] = (fast && hmask && k0 < K) ? hmask[(int64_t)sj[u] * ld_hmask + k0] : 1.f;
                h1[u] = (fast && hmask && k1 < K) ? hmask[(int64_t)sj[u] * ld_hmask + k1] : 1.f;
                zr[u] = fast && inj && inj[sj[u]];
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int sv = sj[u];
                if (sv < 0) continue;
                if (sv >= n && od[u] == 1) {  // single contribution: final masked row
                    if (k0 < K) dx[(int64_t)sv * ld_dx + k0] = (zr[u] || !(h0[u] > 0.f)) ? 0.f : a0;
                    if (k1 < K) dx[(int64_t)sv * ld_dx + k1] = (zr[u] || !(h1[u] > 0.f)) ? 0.f : a1;
                } else {
                    unsigned long long* row = acc + (int64_t)sv * 2 * F_acc;
                    if (k0 < K) fx_add(row, F_acc, k0, a0, od[u], bad);
                    if (k1 < K) fx_add(row, F_acc, k1, a1, od[u], bad);
                }
            }
        }
    }
    if (bad && d_flags) atomicOr(d_flags, bad);
    // ---- last block: fixed-order mean of the row losses (ticket in row_loss[cap])
    unsigned* ticket = reinterpret_cast<unsigned*>(row_loss + cap);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double part = 0.0;
    for (int r = threadIdx.x; r < n; r += TOP_THREADS) part += (double)__ldcg(row_loss + r);
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int k = 0; k < TOP_THREADS / 32; ++k) tot += s_part[k];
        *d_loss = n > 0 ? (float)(tot / (double)n) : 0.f;
        *ticket = 0u;
    }
}
}  // namespace

extern "C" int hg_sage_top_fused(const float* hin, int32_t ld_in, int32_t K, const int32_t* frontier,
                                 const int32_t* d_n, int32_t cap, int32_t fanout, const int32_t* counts,
                                 const int32_t* slot_g, const int32_t* slot_local, const int32_t* nself,
                                 const int32_t* outdeg, const float* W, int32_t C, const int32_t* labels,
                                 const int32_t* seeds, const int32_t* d_div, float* logits, int32_t ld_c,
                                 float* dlogits, float* agg_out, int32_t ld_agg, float* dself_out, int32_t ld_dself,
                                 const float* hmask, int32_t ld_hmask, const uint8_t* inj_mask, int64_t* acc_ws,
                                 int32_t F_acc, float* dx, int32_t ld_dx, int32_t* d_flags, float* row_ws,
                                 float* d_loss, void* stream) {
    if (K < 1 || K > 64 || C < 1 || C > 64) {
        hg_set_error("sage_top_fused: needs K, C in [1, 64] (got %d, %d)", K, C);
        return HG_EUNSUPPORTED;
    }
    if (cap <= 0) { hg_set_error("sage_top_fused: empty batch"); return HG_EINVAL; }
    if (fanout > 32) { hg_set_error("sage_top_fused: fanout > 32"); return HG_EUNSUPPORTED; }
    int grid = hg_ceil_div(cap, TOP_THREADS / 32);
    grid = grid < 2 * HG_NUM_SMS ? grid : 2 * HG_NUM_SMS;
    const int smem = 2 * K * (C | 1) * 4;
    hg_launch(k_sage_top, dim3(grid), dim3(TOP_THREADS), (size_t)smem, (cudaStream_t)stream, hin, ld_in, K, frontier,
              d_n, cap, fanout, counts, slot_g, slot_local, nself, outdeg, W, C, labels, seeds, d_div, logits, ld_c,
              dlogits, agg_out, ld_agg, dself_out, ld_dself, hmask, ld_hmask, inj_mask,
              reinterpret_cast<unsigned long long*>(acc_ws), F_acc, dx, ld_dx, d_flags, row_ws, d_loss);
    return hg_check_launch("sage_top_fused");
}

// finish pass of hg_aggregate_bwd_scatter alone (after a fused scatter)
extern "C" int hg_aggregate_bwd_finish(const float* dself, int32_t ld_dself, int32_t F, const int32_t* d_n_dst,
                                       int32_t cap_dst, const int32_t* d_n_src, int32_t cap_src,
                                       const int32_t* outdeg, const float* hmask, int32_t ld_hmask,
                                       const uint8_t* inj_mask, int64_t* acc_ws, float* dx, int32_t ld_dx,
                                       void* stream) {
    if (F % 4 || ld_dx % 4 || (dself && ld_dself % 4) || (hmask && ld_hmask % 4)) {
        hg_set_error("aggregate_bwd_finish: widths must be multiples of 4");
        return HG_EINVAL;
    }
    if (cap_src == 0) return HG_OK;
    const int F4 = F / 4;
    int LPR, NV;
    pick_lanes(F4, LPR, NV);
    dim3 g2(hg_grid((long long)cap_src * LPR, 256, 8));
    cudaStream_t s = (cudaStream_t)stream;
    unsigned long long* acc = reinterpret_cast<unsigned long long*>(acc_ws);
#define HG_FIN(L, V)                                                                                              \
    if (LPR == L && NV == V) {                                                                                    \
        hg_launch(k_bwd_finish<L, V>, g2, dim3(256), 0, s, acc, F4, dself, ld_dself, d_n_dst, cap_dst, d_n_src,     \
                  cap_src, outdeg, hmask, ld_hmask, inj_mask, dx, ld_dx);                                         \
        return hg_check_launch("aggregate_bwd_finish");                                                          \
    }
    HG_FIN(8, 1) HG_FIN(16, 1) HG_FIN(32, 1) HG_FIN(32, 2) HG_FIN(32, 4) HG_FIN(32, 8)
#undef HG_FIN
    hg_set_error("aggregate_bwd_finish: unsupported width");
    return HG_EUNSUPPORTED;
}
