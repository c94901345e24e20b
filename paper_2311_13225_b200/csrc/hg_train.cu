// K9-K12 + the device embedding store: loss, optimiser updates, historical
// embedding put/lookup/inject, queue construction helpers and evaluation.
#include "hg_common.cuh"
#include "hg_gnn_internal.h"

// Per-batch device parameter block (int64 slots), written by the host before a
// captured step is replayed.  Index names mirror the reference's batch loop
// variables (orchestrator.py:456-545).
enum {
    BP_RNG_SEED = 0,      // runplan.batch_sample_seed (derive_seed(seed, 0x22, epoch, b))
    BP_N_SEEDS = 1,       // |batch|
    BP_READING_BATCH = 2, // global batch index (the store's reading_batch)
    BP_BATCH_IN_EPOCH = 3,
    BP_CPU_TAG = 4,       // tag of the current super-batch's cpu_set (-1: none)
    BP_TABLE_SEL = 5,     // which of the two store buffers is "current"
    BP_CUR_STAMP = 6,     // stamp of entries readable in this super-batch
    BP_WARMUP = 7,        // 1 in super-batch 0 of a layer-based epoch with a hot set
};

namespace {

// --------------------------------------------------------------------------
// softmax cross-entropy (gnnmath.py:263-274): mean loss + dlogits
// --------------------------------------------------------------------------
// n rows (device count, <= cap); dlogits = (p - onehot) / div where div =
// *d_div (the global batch size; == n on one GPU, gnnmath.py:273)
// one warp per row; per-row losses land in row_loss, reduced in fixed order by
// k_xent_reduce (deterministic, no float atomics)
// One launch: per-row warps write dlogits and the row losses; the last block
// to finish (threadfence + ticket in row_ws[cap]) reduces the row losses in a
// fixed order (fp64), so the batch loss is deterministic, and re-arms the ticket.
__global__ void __launch_bounds__(256) k_xent(const float* __restrict__ logits, int ld, int C, const int* d_n,
                                              int cap, const int* __restrict__ labels, const int* __restrict__ seeds,
                                              const int* __restrict__ d_div, float* __restrict__ dlogits, int ldd,
                                              float* __restrict__ row_loss, float* __restrict__ d_loss) {
    hg_pdl_begin();
    __shared__ double s_part[8];
    __shared__ bool s_last;
    const int n = hg_load_count(d_n, cap);
    const float grad_scale = 1.0f / (float)(d_div ? *d_div : (n > 0 ? n : 1));
    const int lane = threadIdx.x & 31;
    const int nw = (gridDim.x * blockDim.x) >> 5;
    for (int r = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < n; r += nw) {
        const float* z = logits + (int64_t)r * ld;
        float mx = -INFINITY;
        for (int c = lane; c < C; c += 32) mx = fmaxf(mx, z[c]);
#pragma unroll
        for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        float se = 0.f;
        for (int c = lane; c < C; c += 32) se += expf(z[c] - mx);
#pragma unroll
        for (int o = 16; o; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const int y = labels[seeds ? seeds[r] : r];
        const float inv = 1.f / se;
        for (int c = lane; c < C; c += 32) {
            const float p = expf(z[c] - mx) * inv;
            dlogits[(int64_t)r * ldd + c] = (p - (c == y ? 1.f : 0.f)) * grad_scale;
        }
        if (lane == 0) row_loss[r] = logf(se) - (z[y] - mx);  // -log softmax_y
    }
    // ---- last block: fixed-order mean of the row losses ----
    unsigned* ticket = reinterpret_cast<unsigned*>(row_loss + cap);
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    double part = 0.0;
    for (int r = threadIdx.x; r < n; r += blockDim.x) part += (double)__ldcg(row_loss + r);
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_part[threadIdx.x >> 5] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int k = 0; k < (int)(blockDim.x >> 5); ++k) tot += s_part[k];
        *d_loss = n > 0 ? (float)(tot / (double)n) : 0.f;
        *ticket = 0u;
    }
}

// per-batch record (orchestrator.py:527-544 row fields): loss and max |dw|
// land at [batch_in_epoch]; the max-delta accumulator is reset for the next step
__global__ void k_record(const int64_t* __restrict__ bp, const float* __restrict__ d_loss,
                         unsigned* __restrict__ d_maxdelta, float* __restrict__ loss_arr,
                         float* __restrict__ md_arr) {
    const int bi = (int)bp[BP_BATCH_IN_EPOCH];
    loss_arr[bi] = *d_loss;
    md_arr[bi] = __uint_as_float(*d_maxdelta);
    *d_maxdelta = 0u;
}

// --------------------------------------------------------------------------
// SGD (gnnmath.py:277-283) + max |w_new - w_old| (orchestrator.py:246-255)
// --------------------------------------------------------------------------
__device__ __forceinline__ void block_max_to(float v, unsigned* d_max) {
    __shared__ float s_m[32];
#pragma unroll
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if ((threadIdx.x & 31) == 0) s_m[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x < 32) {
        float x = threadIdx.x < (blockDim.x >> 5) ? s_m[threadIdx.x] : 0.f;
#pragma unroll
        for (int o = 16; o; o >>= 1) x = fmaxf(x, __shfl_xor_sync(0xffffffffu, x, o));
        if (threadIdx.x == 0 && d_max) atomicMax(d_max, __float_as_uint(x));  // x >= 0
    }
}

__global__ void k_sgd(float* __restrict__ w, const float* __restrict__ g, long long n, float lr,
                      unsigned* __restrict__ d_maxdelta) {
    float md = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float old = w[i];
        const float nw = old - lr * g[i];
        w[i] = nw;
        md = fmaxf(md, fabsf(nw - old));
    }
    block_max_to(md, d_maxdelta);
}

// Adam (gnnmath.py:286-312); step counter t lives on the device
__global__ void k_adam(float* __restrict__ w, const float* __restrict__ g, float* __restrict__ m,
                       float* __restrict__ v, long long n, float lr, float b1, float b2, float eps,
                       const int* __restrict__ d_t, unsigned* __restrict__ d_maxdelta) {
    const int t = *d_t;
    const float c1 = (float)(1.0 - pow((double)b1, (double)t));
    const float c2 = (float)(1.0 - pow((double)b2, (double)t));
    float md = 0.f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const float gi = g[i];
        const float mi = m[i] * b1 + (1.f - b1) * gi;
        const float vi = v[i] * b2 + (1.f - b2) * gi * gi;
        m[i] = mi;
        v[i] = vi;
        const float old = w[i];
        const float nw = old - lr * (mi / c1) / (sqrtf(vi / c2) + eps);
        w[i] = nw;
        md = fmaxf(md, fabsf(nw - old));
    }
    block_max_to(md, d_maxdelta);
}

__global__ void k_incr(int* c) { *c += 1; }

// --------------------------------------------------------------------------
// historical-embedding store (store.py:24-146) on device
// --------------------------------------------------------------------------
// put (store.py:53-65): staging[slot_of[v]] = (emb, version, stamp)
__global__ void k_store_put(const int* __restrict__ ids, const int* d_n, int cap, const float* __restrict__ emb,
                            int ld_emb, int H, const int* __restrict__ slot_of, float* __restrict__ tab,
                            int* __restrict__ ver, int* __restrict__ stamp, int version, int stamp_val,
                            int* __restrict__ d_puts) {
    hg_pdl_begin();
    __shared__ int s_puts;
    if (threadIdx.x == 0) s_puts = 0;
    __syncthreads();
    const int n = hg_load_count(d_n, cap);
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    int puts = 0;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        const int slot = slot_of[ids[i]];
        if (slot < 0) continue;  // not a hot vertex: caller bug, ignored
        for (int c = lane; c < H; c += 32) tab[(int64_t)slot * H + c] = emb[(int64_t)i * ld_emb + c];
        if (lane == 0) {
            ver[slot] = version;
            stamp[slot] = stamp_val;
            ++puts;
        }
    }
    // one counter atomic per CTA (a per-row atomic on the single counter serialised
    // ~23 K updates per producer chunk: 27 us of the 28 us kernel, ncu)
    if (lane == 0 && puts) atomicAdd(&s_puts, puts);
    __syncthreads();
    if (threadIdx.x == 0 && s_puts && d_puts) atomicAdd(d_puts, s_puts);
}

// lookup (store.py:67-98) for every bottom destination in the current cpu_set
// (orchestrator.py:486-500): sets inj_mask / inj_slot, counts hits, misses
// (fallbacks), warm-up rows, tracks the max version gap and flags violations.
// stats[0]=max (gap<<32 | ~batch) packed, stats[1]=violations.
__global__ void k_store_lookup(const int* __restrict__ dst, const int* d_n, int cap, const int64_t* __restrict__ bp,
                               const int* __restrict__ cpu_tag_of, const int* __restrict__ slot_of,
                               const int* __restrict__ ver0, const int* __restrict__ ver1,
                               const int* __restrict__ stamp0, const int* __restrict__ stamp1, int gap_bound,
                               uint8_t* __restrict__ inj_mask, int* __restrict__ inj_slot,
                               int* __restrict__ batch_hits, int* __restrict__ batch_miss,
                               int* __restrict__ batch_warm, unsigned long long* __restrict__ stats) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const int cpu_tag = (int)bp[BP_CPU_TAG];
    const int sel = (int)bp[BP_TABLE_SEL];
    const int cur_stamp = (int)bp[BP_CUR_STAMP];
    const int rb = (int)bp[BP_READING_BATCH];
    const int bi = (int)bp[BP_BATCH_IN_EPOCH];
    const bool warm = bp[BP_WARMUP] != 0;
    const int* ver = sel ? ver1 : ver0;
    const int* stamp = sel ? stamp1 : stamp0;
    int hits = 0, miss = 0, wc = 0;
    unsigned long long best = 0ULL;
    int viol = 0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int v = dst[i];
        uint8_t m = 0;
        if (cpu_tag >= 0 && cpu_tag_of[v] == cpu_tag) {
            const int slot = slot_of[v];
            if (slot >= 0 && stamp[slot] == cur_stamp) {
                const int gap = rb - ver[slot];
                if (gap > gap_bound) {
                    // StalenessViolation (store.py:85-92): counted, never injected — the
                    // row is computed from features; the host raises at the next check
                    ++viol;
                } else {
                    ++hits;
                    m = 1;
                    inj_slot[i] = slot;
                    const unsigned long long key = ((unsigned long long)(unsigned)gap << 32) | (0xffffffffu - (unsigned)rb);
                    best = best > key ? best : key;
                }
            } else {
                ++miss;
            }
        } else if (warm && slot_of[v] >= 0) {
            ++wc;
        }
        inj_mask[i] = m;
    }
    // warp-aggregate then one atomic per warp
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        hits += __shfl_xor_sync(0xffffffffu, hits, o);
        miss += __shfl_xor_sync(0xffffffffu, miss, o);
        wc += __shfl_xor_sync(0xffffffffu, wc, o);
        viol += __shfl_xor_sync(0xffffffffu, viol, o);
        unsigned long long ob = __shfl_xor_sync(0xffffffffu, best, o);
        best = best > ob ? best : ob;
    }
    if ((threadIdx.x & 31) == 0) {
        if (hits) atomicAdd(&batch_hits[bi], hits);
        if (miss) atomicAdd(&batch_miss[bi], miss);
        if (wc) atomicAdd(&batch_warm[bi], wc);
        if (best) atomicMax(&stats[0], best);
        if (viol) atomicAdd(&stats[1], (unsigned long long)viol);
    }
}

// overwrite injected rows of the bottom layer's OUTPUT (gnnmath.py:240-245)
__global__ void k_inject(const uint8_t* __restrict__ inj_mask, const int* __restrict__ inj_slot, const int* d_n,
                         int cap, const int64_t* __restrict__ bp, const float* __restrict__ tab0,
                         const float* __restrict__ tab1, int H, float* __restrict__ h, int ldh) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const float* tab = bp[BP_TABLE_SEL] ? tab1 : tab0;
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int i = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += warps) {
        if (!inj_mask[i]) continue;
        const int slot = inj_slot[i];
        for (int c = lane; c < H; c += 32) h[(int64_t)i * ldh + c] = tab[(int64_t)slot * H + c];
    }
}

// --------------------------------------------------------------------------
// queue construction (orchestrator.py:211-228) helpers
// --------------------------------------------------------------------------
__global__ void k_tag(const int* __restrict__ ids, const int* d_n, int cap, int* __restrict__ tag_of, int tag) {
    const int n = hg_load_count(d_n, cap);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) tag_of[ids[k]] = tag;
}

// sample_khop_skip_hot (sampler.py:150-163): flags[i] = values[i] is in the tagged set
__global__ void k_member_flags(const int* __restrict__ values, const int* d_n, int cap, const int* __restrict__ tag_of,
                               int tag, uint8_t* __restrict__ flags) {
    const int n = hg_load_count(d_n, cap);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        flags[k] = tag_of[values[k]] == tag;
}

__global__ void k_filter_flags(const int* __restrict__ list, int n, const int* __restrict__ tag_of, int tag,
                               int* __restrict__ flags) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        flags[k] = tag_of[list[k]] == tag;
}

__global__ void k_filter_emit(const int* __restrict__ list, int n, const int* __restrict__ tag_of, int tag,
                              const int* __restrict__ rank, int* __restrict__ out) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        if (tag_of[list[k]] == tag) out[rank[k]] = list[k];
}

// --------------------------------------------------------------------------
// full-graph aggregation for evaluate (orchestrator.py:662-680): the block is
// the whole CSR (edge_src = targets, edge_dst = row), same layer semantics.
// --------------------------------------------------------------------------
__global__ void k_full_agg(int model, const float* __restrict__ hin, int ld_in, int F4,
                           const int64_t* __restrict__ offsets, const int* __restrict__ targets, int V,
                           const int* __restrict__ outdeg, float* __restrict__ out, int ld_out) {
    const int lane = threadIdx.x & 31;
    const int warps = (gridDim.x * blockDim.x) >> 5;
    for (int v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < V; v += warps) {
        const int64_t b = offsets[v], e = offsets[v + 1];
        int ns = 0;
        if (model == 0)
            for (int64_t k = b + lane; k < e; k += 32) ns += targets[k] != v;
#pragma unroll
        for (int o = 16; o; o >>= 1) ns += __shfl_xor_sync(0xffffffffu, ns, o);
        const float wd = ns > 0 ? 1.0f / (float)ns : 0.f;
        const int indeg = (int)(e - b);
        for (int c0 = 0; c0 < F4; c0 += 32) {
            const int c = c0 + lane;
            float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
            for (int64_t k = b; k < e; ++k) {
                const int u = targets[k];
                float w;
                if (model == 0) { if (u == v) continue; w = wd; }
                else w = (float)(1.0 / sqrt((double)outdeg[u] * (double)indeg));
                if (c < F4) {
                    const float4 r = __ldg(reinterpret_cast<const float4*>(hin + (int64_t)u * ld_in) + c);
                    acc.x = fmaf(w, r.x, acc.x); acc.y = fmaf(w, r.y, acc.y);
                    acc.z = fmaf(w, r.z, acc.z); acc.w = fmaf(w, r.w, acc.w);
                }
            }
            if (c < F4) reinterpret_cast<float4*>(out + (int64_t)v * ld_out)[c] = acc;
        }
    }
}

__global__ void k_target_hist(const int* __restrict__ targets, long long E, int* __restrict__ cnt) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < E; k += (long long)gridDim.x * blockDim.x)
        atomicAdd(&cnt[targets[k]], 1);
}

// number of masked rows whose argmax (first max, np.argmax) equals the label
__global__ void k_argmax_correct(const float* __restrict__ logits, int ld, int C, int V,
                                 const int* __restrict__ labels, const uint8_t* __restrict__ mask,
                                 unsigned long long* __restrict__ d_correct) {
    int corr = 0;
    for (int v = blockIdx.x * blockDim.x + threadIdx.x; v < V; v += gridDim.x * blockDim.x) {
        if (!mask[v]) continue;
        const float* z = logits + (int64_t)v * ld;
        int best = 0;
        float bv = z[0];
        for (int c = 1; c < C; ++c)
            if (z[c] > bv) { bv = z[c]; best = c; }
        corr += best == labels[v];
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) corr += __shfl_xor_sync(0xffffffffu, corr, o);
    if ((threadIdx.x & 31) == 0 && corr) atomicAdd(d_correct, (unsigned long long)corr);
}

}  // namespace

extern "C" int hg_softmax_xent(const float* logits, int32_t ld, int32_t C, const int32_t* d_n, int32_t cap,
                               const int32_t* labels, const int32_t* seeds, const int32_t* d_div, float* dlogits,
                               int32_t ldd, float* d_loss, float* row_ws, void* stream) {
    if (cap <= 0) { hg_set_error("softmax_xent: empty batch"); return HG_EINVAL; }
    cudaStream_t s = (cudaStream_t)stream;
    hg_launch(k_xent, hg_ceil_div(cap, 8), 256, 0, s, logits, ld, C, d_n, cap, labels, seeds, d_div, dlogits, ldd, row_ws,
                                               d_loss);
    return hg_check_launch("softmax_xent");
}

extern "C" int hg_record_batch(const int64_t* bp, const float* d_loss, uint32_t* d_maxdelta, float* loss_arr,
                               float* md_arr, void* stream) {
    k_record<<<1, 1, 0, (cudaStream_t)stream>>>(bp, d_loss, d_maxdelta, loss_arr, md_arr);
    return hg_check_launch("record_batch");
}

extern "C" int hg_sgd(float* w, const float* g, int64_t n, float lr, uint32_t* d_maxdelta, void* stream) {
    if (n <= 0) return HG_OK;
    k_sgd<<<hg_grid(n, 256, 4), 256, 0, (cudaStream_t)stream>>>(w, g, n, lr, d_maxdelta);
    return hg_check_launch("sgd");
}

extern "C" int hg_adam(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2,
                       float eps, int32_t* d_t, uint32_t* d_maxdelta, void* stream) {
    if (n <= 0) return HG_OK;
    cudaStream_t s = (cudaStream_t)stream;
    k_incr<<<1, 1, 0, s>>>(d_t);
    k_adam<<<hg_grid(n, 256, 4), 256, 0, s>>>(w, g, m, v, n, lr, b1, b2, eps, d_t, d_maxdelta);
    return hg_check_launch("adam");
}

extern "C" int hg_store_put(const int32_t* ids, const int32_t* d_n, int32_t cap, const float* emb, int32_t ld_emb,
                            int32_t H, const int32_t* slot_of, float* tab, int32_t* ver, int32_t* stamp,
                            int32_t version, int32_t stamp_val, int32_t* d_puts, void* stream) {
    if (cap <= 0) return HG_OK;
    hg_launch(k_store_put, hg_grid((long long)cap * 32, 256, 8), 256, 0, (cudaStream_t)stream, 
        ids, d_n, cap, emb, ld_emb, H, slot_of, tab, ver, stamp, version, stamp_val, d_puts);
    return hg_check_launch("store_put");
}

extern "C" int hg_store_lookup(const int32_t* dst, const int32_t* d_n, int32_t cap, const int64_t* bp,
                               const int32_t* cpu_tag_of, const int32_t* slot_of, const int32_t* ver0,
                               const int32_t* ver1, const int32_t* stamp0, const int32_t* stamp1, int32_t gap_bound,
                               uint8_t* inj_mask, int32_t* inj_slot, int32_t* batch_hits, int32_t* batch_miss,
                               int32_t* batch_warm, uint64_t* stats, void* stream) {
    if (cap <= 0) return HG_OK;
    hg_launch(k_store_lookup, hg_grid(cap, 256, 8), 256, 0, (cudaStream_t)stream, 
        dst, d_n, cap, bp, cpu_tag_of, slot_of, ver0, ver1, stamp0, stamp1, gap_bound, inj_mask, inj_slot, batch_hits,
        batch_miss, batch_warm, (unsigned long long*)stats);
    return hg_check_launch("store_lookup");
}

extern "C" int hg_inject_rows(const uint8_t* inj_mask, const int32_t* inj_slot, const int32_t* d_n, int32_t cap,
                              const int64_t* bp, const float* tab0, const float* tab1, int32_t H, float* h,
                              int32_t ldh, void* stream) {
    if (cap <= 0) return HG_OK;
    hg_launch(k_inject, hg_grid((long long)cap * 32, 256, 8), 256, 0, (cudaStream_t)stream, inj_mask, inj_slot, d_n, cap, bp,
                                                                                     tab0, tab1, H, h, ldh);
    return hg_check_launch("inject_rows");
}

extern "C" int hg_tag_vertices(const int32_t* ids, const int32_t* d_n, int32_t cap, int32_t* tag_of, int32_t tag,
                               void* stream) {
    if (cap <= 0) return HG_OK;
    k_tag<<<hg_grid(cap, 256, 8), 256, 0, (cudaStream_t)stream>>>(ids, d_n, cap, tag_of, tag);
    return hg_check_launch("tag_vertices");
}

extern "C" int hg_member_flags(const int32_t* values, const int32_t* d_n, int32_t cap, const int32_t* tag_of,
                               int32_t tag, uint8_t* flags, void* stream) {
    if (cap <= 0) return HG_OK;
    k_member_flags<<<hg_grid(cap, 256, 8), 256, 0, (cudaStream_t)stream>>>(values, d_n, cap, tag_of, tag, flags);
    return hg_check_launch("member_flags");
}

extern "C" int64_t hg_filter_ws_size(int32_t n) { return (int64_t)(n + (long long)hg_scan_ws_ints(n) + 16); }

// out = [x for x in list if tag_of[x] == tag], order kept; *d_n_out = count
extern "C" int hg_filter_tagged(const int32_t* list, int32_t n, const int32_t* tag_of, int32_t tag, int32_t* out,
                                int32_t* d_n_out, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) { cudaMemsetAsync(d_n_out, 0, sizeof(int), s); return hg_check_launch("filter(empty)"); }
    const int g = hg_grid(n, 256, 8);
    k_filter_flags<<<g, 256, 0, s>>>(list, n, tag_of, tag, ws);
    int rc = hg_scan_launch(ws, ws, nullptr, 1, n, d_n_out, ws + n, s);
    if (rc) return rc;
    k_filter_emit<<<g, 256, 0, s>>>(list, n, tag_of, tag, ws, out);
    return hg_check_launch("filter_tagged");
}

extern "C" int hg_full_aggregate(int32_t model, const float* hin, int32_t ld_in, int32_t F, const int64_t* offsets,
                                 const int32_t* targets, int32_t V, const int32_t* outdeg, float* out, int32_t ld_out,
                                 void* stream) {
    if (F % 4 || ld_in % 4 || ld_out % 4) { hg_set_error("full_aggregate: widths must be multiples of 4"); return HG_EINVAL; }
    k_full_agg<<<hg_grid((long long)V * 32, 256, 8), 256, 0, (cudaStream_t)stream>>>(model, hin, ld_in, F / 4, offsets,
                                                                                     targets, V, outdeg, out, ld_out);
    return hg_check_launch("full_aggregate");
}

extern "C" int hg_target_histogram(const int32_t* targets, int64_t E, int32_t* cnt, void* stream) {
    if (E <= 0) return HG_OK;
    k_target_hist<<<hg_grid(E, 256, 8), 256, 0, (cudaStream_t)stream>>>(targets, E, cnt);
    return hg_check_launch("target_histogram");
}

extern "C" int hg_argmax_correct(const float* logits, int32_t ld, int32_t C, int32_t V, const int32_t* labels,
                                 const uint8_t* mask, uint64_t* d_correct, void* stream) {
    k_argmax_correct<<<hg_grid(V, 256, 8), 256, 0, (cudaStream_t)stream>>>(logits, ld, C, V, labels, mask,
                                                                           (unsigned long long*)d_correct);
    return hg_check_launch("argmax_correct");
}

// --------------------------------------------------------------------------
// Per-batch transfer accounting (transfer.py:59-73 needed_bottom_rows, reported
// as the batch CSV's raw_rows, reporting.py:23-27): the number of distinct
// bottom-block source vertices feeding a computed (non-injected) destination,
// plus the computed destinations' own self rows.  First-writer counting on a
// per-vertex tag table (atomicExch(tag_of[v], tag) != tag counts v once) gives
// the exact distinct count in any order; tag = reading batch + 1, so the table
// is never reset.  out[bp[BATCH_IN_EPOCH]] += count.
// --------------------------------------------------------------------------
namespace {
__global__ void __launch_bounds__(256) k_count_needed(const int* __restrict__ frontier, const int* d_n, int cap, int f,
                                                      const int* __restrict__ counts, const int* __restrict__ slots,
                                                      const uint8_t* __restrict__ inj, const int64_t* __restrict__ bp,
                                                      const uint8_t* __restrict__ cached, int* __restrict__ tag_of,
                                                      int* __restrict__ out, int* __restrict__ out_hits) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const int tag = (int)bp[BP_READING_BATCH] + 1;
    const long long Q = (long long)n * (f + 1);
    int c = 0, h = 0;
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < Q; q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / (f + 1)), j = (int)(q - (long long)i * (f + 1));
        if (inj && inj[i]) continue;  // injected destination: nothing of it is computed
        int v;
        if (j == f) v = frontier[i];  // the destination's own self row
        else if (j < counts[i]) v = slots[(int64_t)i * f + j];
        else continue;
        if (atomicExch(&tag_of[v], tag) != tag) {
            // a needed row is a raw transfer unless it sits in the static feature
            // cache (transfer.py:103-114, cache_hit_rows)
            if (cached && cached[v]) ++h;
            else ++c;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        c += __shfl_xor_sync(0xffffffffu, c, o);
        h += __shfl_xor_sync(0xffffffffu, h, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (c) atomicAdd(&out[(int)bp[BP_BATCH_IN_EPOCH]], c);
        if (h && out_hits) atomicAdd(&out_hits[(int)bp[BP_BATCH_IN_EPOCH]], h);
    }
}
}  // namespace

extern "C" int hg_count_needed_rows(const int32_t* frontier, const int32_t* d_n, int32_t cap, int32_t fanout,
                                    const int32_t* counts, const int32_t* slots, const uint8_t* inj_mask,
                                    const int64_t* bp, const uint8_t* cached, int32_t* tag_of, int32_t* out,
                                    int32_t* out_hits, void* stream) {
    if (cap <= 0) return HG_OK;
    hg_launch(k_count_needed, hg_grid((long long)cap * (fanout + 1), 256, 8), 256, 0, (cudaStream_t)stream, frontier,
              d_n, cap, fanout, counts, slots, inj_mask, bp, cached, tag_of, out, out_hits);
    return hg_check_launch("count_needed_rows");
}
