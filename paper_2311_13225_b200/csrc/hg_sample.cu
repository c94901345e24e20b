#include <cstdlib>
// K1-K3: bit-exact k-hop block sampling on an HBM-resident CSR.
//
// Replaces the reference's per-layer block construction
//   sampler._expand_frontier (sampler.py:104-118)
//     = kernels._sample_layer (kernels.py:77-118)      -> k_sample_seg / k_sample_seq
//     + kernels.stable_unique (kernels.py:166-180)     -> k_mark + scan + k_emit_src
//     + np.lexsort((src_local, dst_local))             -> k_relabel_sort_seg
//
// Layout ("slot" form, what the training step consumes): destination i owns
// the fixed-stride slot range [i*f, i*f + counts[i]); slots hold the sampled
// global ids and, after relabel, the local src ids sorted ascending — exactly
// the reference's (dst, src) edge order.  No prefix sum is needed to address a
// segment, so the aggregation kernels index segments directly.  A compacted
// CSR (the reference's Block.edge_src/edge_dst) is produced only on request
// (hg_block_to_edges).
//
// RNG: the reference's splitmix64 per-(stream, vertex) partial Fisher–Yates.
// Draw j of vertex v uses r_j = mix64(s_v + (j+1)*GOLDEN), which is counter
// based, so the lanes of a segment compute all r_j and picks in parallel; the
// swap chain of the partial Fisher–Yates is then resolved with a shared-memory
// "last writer" table, pointer jumping and __match_any_sync (see k_sample_seg).
//
// Dedup: positions follow the reference's emission order (frontier first,
// then draws in (dst, draw) order).  A dense uint64 first-occurrence table
// minpos[V] receives atomicMin((tag << 32) | position) for every emitted id; an
// id's first occurrence is the position that won.  The tag decreases with every
// use of the table (a device counter bumped by the relabel kernel), so entries
// left by earlier blocks always lose and the table never needs resetting.
#include "hg_common.cuh"
#include "hg_gnn_internal.h"

namespace {

// CTAs per SM for the draw / relabel grids (env HG_SAMPLE_CTAS_PER_SM, default 8):
// fewer leaves SM room for the training stream's kernels that run concurrently
int hg_sample_ctas_per_sm() {
    static int v = -1;
    if (v < 0) {
        const char* e = getenv("HG_SAMPLE_CTAS_PER_SM");
        v = e ? atoi(e) : 8;
        if (v < 1) v = 1;
        if (v > 8) v = 8;
    }
    return v;
}

constexpr unsigned long long FO_RANKED = 0xFFFFFFFF00000000ull;  // tag of rewritten (ranked) entries

__device__ __forceinline__ uint32_t fo_tag(const int* ctr) { return 0xFFFFFFFEu - (uint32_t)(*ctr); }
__device__ __forceinline__ unsigned long long fo_key(uint32_t tag, long long pos) {
    return ((unsigned long long)tag << 32) | (unsigned long long)(uint32_t)pos;
}

// --------------------------------------------------------------------------
// draw kernel, fanout <= 32: one W-lane segment per destination
// --------------------------------------------------------------------------
template <int W>
__device__ __forceinline__ void draw_seg_body(const int64_t* __restrict__ offsets, const int* __restrict__ targets,
                                              const int* __restrict__ frontier, const int* d_n, int cap, int f,
                                              const uint64_t* __restrict__ d_seed, int layer,
                                              int* __restrict__ counts, int* __restrict__ slots,
                                              unsigned long long* __restrict__ minpos, const int* __restrict__ tag_ctr,
                                              int* __restrict__ nself, int* s_last) {
    const int n = hg_load_count(d_n, cap);
    const uint32_t tag = minpos ? fo_tag(tag_ctr) : 0u;
    const uint64_t stream = layer >= 0 ? hg_derive2(*d_seed, HG_SAMPLE_TAG, (uint64_t)layer) : *d_seed;
    const uint64_t base = hg_mix64(stream + HG_GOLDEN);  // kernels.py:153
    const int lane = threadIdx.x & 31;
    const int sub = lane & (W - 1);
    const int seg0 = lane & ~(W - 1);  // first lane of my segment
    const unsigned segmask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << seg0);
    const int segs_per_block = blockDim.x / W;
    int* last = s_last + (threadIdx.x & ~(W - 1));
    for (int i0 = blockIdx.x * segs_per_block; i0 < n; i0 += gridDim.x * segs_per_block) {
        const int i = i0 + threadIdx.x / W;
        if (i >= n) continue;  // segment-uniform
        const int v = frontier[i];
        if (sub == 0 && minpos) atomicMin(&minpos[v], fo_key(tag, i));  // frontier position i
        const int64_t off = offsets[v];
        const int64_t deg = offsets[v + 1] - off;
        const int cnt = deg < f ? (int)deg : f;
        if (sub == 0) counts[i] = cnt;
        int u = -1;
        if (deg <= f) {  // kernels.py:100-103: every neighbour, CSR order
            if (sub < deg) u = targets[off + sub];
        } else {  // kernels.py:104-117
            int pick = -1 - sub;  // distinct sentinels for idle lanes
            if (sub < f) {
                const uint64_t st = hg_mix64(base ^ ((uint64_t)(int64_t)v * HG_PHI)) +
                                    (uint64_t)(sub + 1) * HG_GOLDEN;
                const uint64_t r = hg_mix64(st);
                pick = sub + (int)(r % (uint64_t)(deg - sub));
            }
            // last[p] = latest earlier draw m (< p) whose pick was position p
            last[sub] = -1;
            __syncwarp(segmask);
            if (sub < f && pick < f && pick != sub) atomicMax(&last[pick], sub);
            __syncwarp(segmask);
            // before(p) = value held at position p right before draw p:
            // follow last[] down to a position never overwritten (pointer jumping)
            int root = (sub < f && last[sub] >= 0) ? last[sub] : sub;
#pragma unroll
            for (int k = 1; k < W; k <<= 1) root = __shfl_sync(segmask, root, root, W);
            // draw j emits the current content of position pick_j: the value the
            // latest earlier draw k with the same pick moved there (before(k)),
            // or pick_j itself if untouched
            const unsigned peers = __match_any_sync(segmask, pick) & hg_lanemask_lt();
            const int k = peers ? (31 - __clz(peers)) - seg0 : sub;
            const int moved = __shfl_sync(segmask, root, k, W);
            if (sub < f) u = targets[off + (peers ? moved : pick)];
        }
        if (sub < cnt) {
            slots[(int64_t)i * f + sub] = u;
            if (minpos) atomicMin(&minpos[u], fo_key(tag, (long long)n + (long long)i * f + sub));
        }
        if (nself) {  // SAGE non-self count (gnnmath.py:145-154) when no relabel pass follows
            const unsigned ns = __ballot_sync(segmask, sub < cnt && u != v);
            if (sub == 0) nself[i] = __popc(ns);
        }
    }
}

template <int W>
__global__ void __launch_bounds__(256) k_sample_seg(const int64_t* __restrict__ offsets,
                                                    const int* __restrict__ targets,
                                                    const int* __restrict__ frontier, const int* d_n,
                                                    int cap, int f, const uint64_t* __restrict__ d_seed,
                                                    int layer, int* __restrict__ counts,
                                                    int* __restrict__ slots, unsigned long long* __restrict__ minpos,
                                                    const int* __restrict__ tag_ctr, int* __restrict__ nself) {
    hg_pdl_begin();
    __shared__ int s_last[256];
    draw_seg_body<W>(offsets, targets, frontier, d_n, cap, f, d_seed, layer, counts, slots, minpos, tag_ctr, nself,
                     s_last);
}

// --------------------------------------------------------------------------
// draw kernel, fanout > 32: one thread per destination, sequential partial
// Fisher–Yates with a small swap map in scratch (pos, val pairs; O(f^2))
// --------------------------------------------------------------------------
__global__ void k_sample_seq(const int64_t* __restrict__ offsets, const int* __restrict__ targets,
                             const int* __restrict__ frontier, const int* d_n, int cap, int f,
                             const uint64_t* __restrict__ d_seed, int layer, int* __restrict__ counts,
                             int* __restrict__ slots, unsigned long long* __restrict__ minpos,
                             const int* __restrict__ tag_ctr, int* __restrict__ scratch, int* __restrict__ nself) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    const uint32_t tag = minpos ? fo_tag(tag_ctr) : 0u;
    const uint64_t stream = layer >= 0 ? hg_derive2(*d_seed, HG_SAMPLE_TAG, (uint64_t)layer) : *d_seed;
    const uint64_t base = hg_mix64(stream + HG_GOLDEN);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int v = frontier[i];
        if (minpos) atomicMin(&minpos[v], fo_key(tag, i));
        const int64_t off = offsets[v];
        const int64_t deg = offsets[v + 1] - off;
        const int cnt = deg < f ? (int)deg : f;
        counts[i] = cnt;
        int* sp = slots + (int64_t)i * f;
        if (deg <= f) {
            for (int j = 0; j < cnt; ++j) sp[j] = targets[off + j];
        } else {
            int* mp = scratch + (int64_t)i * 2 * f;  // map entries: position, value
            int m = 0;
            uint64_t st = hg_mix64(base ^ ((uint64_t)(int64_t)v * HG_PHI));
            for (int j = 0; j < f; ++j) {
                st += HG_GOLDEN;
                const uint64_t r = hg_mix64(st);
                const int pick = j + (int)(r % (uint64_t)(deg - j));
                int vj = j, vp = pick, ip = -1;
                for (int t = 0; t < m; ++t) {
                    if (mp[2 * t] == j) vj = mp[2 * t + 1];
                    if (mp[2 * t] == pick) { vp = mp[2 * t + 1]; ip = t; }
                }
                // swap(idx[j], idx[pick]); emit idx[j].  Position j is never read
                // again (later picks are > j), so only position pick is recorded.
                if (pick != j) {
                    if (ip >= 0) mp[2 * ip + 1] = vj;
                    else { mp[2 * m] = pick; mp[2 * m + 1] = vj; ++m; }
                }
                sp[j] = targets[off + vp];
            }
        }
        if (minpos)
            for (int j = 0; j < cnt; ++j) atomicMin(&minpos[sp[j]], fo_key(tag, (long long)n + (long long)i * f + j));
        if (nself) {
            int ns = 0;
            for (int j = 0; j < cnt; ++j) ns += sp[j] != v;
            nself[i] = ns;
        }
    }
}

// ---------------------------------------------------------------------------
// Single-pass first-occurrence compaction (replaces flag -> 3-kernel scan ->
// emit): each 2048-position tile marks its first occurrences (minpos[u] == p),
// scans them in the block, resolves its global offset by decoupled look-back
// over the predecessors' published (aggregate | inclusive prefix) words, then
// writes rank[p] and src_vertices[rank] = u.  The tile that holds position P-1
// writes n_src.  Status words carry a generation (bits 34..63) so the array
// never needs clearing: generation = *d_gen + 1, bumped by the relabel kernel.
// ---------------------------------------------------------------------------
constexpr int MS_THREADS = 256;
constexpr int MS_ITEMS = 8;
constexpr int MS_TILE = MS_THREADS * MS_ITEMS;

__device__ __forceinline__ unsigned long long ms_word(uint32_t gen, uint32_t flag, uint32_t v) {
    return ((unsigned long long)gen << 34) | ((unsigned long long)flag << 32) | v;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// one tile t of the mark/scan/emit pass (t = blockIdx.x in k_markscan)
__device__ __forceinline__ void markscan_tile(int t, const int* __restrict__ frontier, const int* d_n, int cap,
                                              int f, const int* __restrict__ counts, const int* __restrict__ slots,
                                              unsigned long long* __restrict__ minpos,
                                              const int* __restrict__ tag_ctr, int* __restrict__ rank,
                                              int* __restrict__ src_vertices, int* __restrict__ d_n_src,
                                              unsigned long long* __restrict__ status,
                                              const int* __restrict__ d_gen, int* __restrict__ outdeg) {
    __shared__ int s_warp[MS_THREADS / 32];
    __shared__ int s_prefix;
    const int n = hg_load_count(d_n, cap);
    const uint32_t tag = fo_tag(tag_ctr);
    const uint32_t gen = (uint32_t)(*d_gen) + 1u;  // issued with the two loads above
    const long long P = (long long)n * (f + 1);
    const long long p0 = (long long)t * MS_TILE;
    if (p0 >= P) {
        if (t == 0 && threadIdx.x == 0) *d_n_src = 0;
        return;  // no later tile waits on this one
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    int u[MS_ITEMS];
    unsigned flags = 0;
    int cnt = 0;
    const long long my0 = p0 + (long long)threadIdx.x * MS_ITEMS;
    // three rounds of independent loads (ids and counts, then the table) instead
    // of a dependent counts -> slots -> minpos chain per item; the (dst, draw)
    // coordinates of the thread's contiguous positions are stepped, one division
    int si = 0, sj = 0;
    if (my0 > n) {
        const long long q0 = my0 - n;
        si = (int)(q0 / f);
        sj = (int)(q0 - (long long)si * f);
    }
    int jk[MS_ITEMS], ck[MS_ITEMS];
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        const long long p = my0 + k;
        u[k] = -1;
        jk[k] = 0;
        ck[k] = 1;
        if (p < P) {
            if (p < n) {
                u[k] = frontier[p];
            } else {
                u[k] = slots[p - n];
                ck[k] = counts[si];
                jk[k] = sj;
                if (++sj == f) { sj = 0; ++si; }
            }
        }
    }
    unsigned long long mk[MS_ITEMS];
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        mk[k] = 0;
        if (u[k] >= 0 && jk[k] < ck[k]) mk[k] = minpos[u[k]];
    }
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        const long long p = my0 + k;
        if (p < P && jk[k] < ck[k] && mk[k] == fo_key(tag, p)) {
            flags |= 1u << k;
            ++cnt;
        }
    }
    // block exclusive scan of per-thread counts
    int x = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[wid] = x;
    __syncthreads();
    if (wid == 0) {
        int w = lane < MS_THREADS / 32 ? s_warp[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        if (lane < MS_THREADS / 32) s_warp[lane] = w;
    }
    __syncthreads();
    const int tile_total = s_warp[MS_THREADS / 32 - 1];
    int local = (wid ? s_warp[wid - 1] : 0) + x - cnt;
    if (wid == 0) {  // decoupled look-back
        int excl = 0;
        if (t == 0) {
            if (lane == 0) st_release_u64(&status[0], ms_word(gen, 2, (uint32_t)tile_total));
        } else {
            if (lane == 0) st_release_u64(&status[t], ms_word(gen, 1, (uint32_t)tile_total));
            int idx = t - 1;
            while (true) {
                const int j = idx - lane;
                unsigned long long w = 0;
                uint32_t fl = 2, val = 0;
                if (j >= 0) {
                    do {
                        w = ld_acquire_u64(&status[j]);
                    } while ((uint32_t)(w >> 34) != gen || ((w >> 32) & 3u) == 0u);
                    fl = (uint32_t)((w >> 32) & 3u);
                    val = (uint32_t)w;
                }
                const unsigned incl = __ballot_sync(0xffffffffu, fl == 2u);
                const int stop = incl ? (__ffs(incl) - 1) : 32;
                int contrib = lane <= stop ? (int)val : 0;  // lanes past the first inclusive word ignored
#pragma unroll
                for (int o = 16; o; o >>= 1) contrib += __shfl_xor_sync(0xffffffffu, contrib, o);
                excl += contrib;
                if (incl) break;
                idx -= 32;
            }
            if (lane == 0) st_release_u64(&status[t], ms_word(gen, 2, (uint32_t)(excl + tile_total)));
        }
        if (lane == 0) s_prefix = excl;
    }
    __syncthreads();
    local += s_prefix;
#pragma unroll
    for (int k = 0; k < MS_ITEMS; ++k) {
        if (flags & (1u << k)) {
            // the first occurrence's table entry becomes its local id under the
            // reserved tag 0xFFFFFFFF: larger than every live key (tags count down),
            // so later atomicMin's always win, never equal to a position key that
            // another tile compares against, and the relabel pass reads local ids
            // with one load instead of minpos -> rank
            minpos[u[k]] = FO_RANKED | (unsigned)local;
            src_vertices[local] = u[k];
            if (outdeg) outdeg[local] = 0;  // counted by the relabel kernel that follows
            ++local;
        }
    }
    if (p0 + MS_TILE >= P && threadIdx.x == 0) *d_n_src = s_prefix + tile_total;
    __syncthreads();  // s_warp / s_prefix are reused by the CTA's next tile
}

__global__ void __launch_bounds__(MS_THREADS) k_markscan(const int* __restrict__ frontier, const int* d_n, int cap,
                                                         int f, const int* __restrict__ counts,
                                                         const int* __restrict__ slots,
                                                         unsigned long long* __restrict__ minpos,
                                                         const int* __restrict__ tag_ctr, int* __restrict__ rank,
                                                         int* __restrict__ src_vertices, int* __restrict__ d_n_src,
                                                         unsigned long long* __restrict__ status,
                                                         const int* __restrict__ d_gen, int* __restrict__ outdeg) {
    hg_pdl_begin();
    markscan_tile(blockIdx.x, frontier, d_n, cap, f, counts, slots, minpos, tag_ctr, rank, src_vertices, d_n_src,
                  status, d_gen, outdeg);
}

// per destination: local id = rank[minpos[id]]; sort the segment by local id
// (stable on draw order, = np.lexsort((src_local, dst_local))); write sorted
// global ids back into slots and local ids into slot_local; per-dst non-self
// count (SAGE, gnnmath.py:145-154) and block out-degree (GCN, gnnmath.py:96).
template <int W>
__device__ __forceinline__ void relabel_seg_body(const int* __restrict__ frontier, const int* d_n, int cap, int f,
                                                 const int* __restrict__ counts, int* __restrict__ slots,
                                                 int* __restrict__ slot_local,
                                                 const unsigned long long* __restrict__ minpos,
                                                 int* __restrict__ nself, int* __restrict__ outdeg,
                                                 int* __restrict__ tag_ctr, int* __restrict__ d_gen) {
    const int n = hg_load_count(d_n, cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // retire this use of the table and of the scan status
        *tag_ctr += 1;
        *d_gen += 1;
    }
    const int lane = threadIdx.x & 31;
    const int sub = lane & (W - 1);
    const int seg0 = lane & ~(W - 1);
    const unsigned segmask = (W == 32) ? 0xffffffffu : (((1u << W) - 1u) << seg0);
    const int segs_per_block = blockDim.x / W;
    for (int i0 = blockIdx.x * segs_per_block; i0 < n; i0 += gridDim.x * segs_per_block) {
        const int i = i0 + threadIdx.x / W;
        if (i >= n) continue;
        const int cnt = counts[i];
        const int v = frontier[i];
        int u = -1, loc = HG_INT_MAX;
        if (sub < cnt) {
            u = slots[(int64_t)i * f + sub];
            loc = (int)(uint32_t)minpos[u];  // local id (rewritten by k_markscan)
        }
        int r = 0;
        for (int k = 0; k < cnt; ++k) {
            const int lk = __shfl_sync(segmask, loc, k, W);
            r += (lk < loc) || (lk == loc && k < sub);
        }
        const unsigned nonself = __ballot_sync(segmask, sub < cnt && u != v);
        __syncwarp(segmask);
        if (sub < cnt) {
            slots[(int64_t)i * f + r] = u;
            slot_local[(int64_t)i * f + r] = loc;
            if (outdeg) atomicAdd(&outdeg[loc], 1);
        }
        if (sub == 0 && nself) nself[i] = __popc(nonself);
    }
}

template <int W>
__global__ void __launch_bounds__(256) k_relabel_sort_seg(const int* __restrict__ frontier, const int* d_n,
                                                          int cap, int f, const int* __restrict__ counts,
                                                          int* __restrict__ slots, int* __restrict__ slot_local,
                                                          const unsigned long long* __restrict__ minpos,
                                                          const int* __restrict__ rank,
                                                          int* __restrict__ nself, int* __restrict__ outdeg,
                                                          int* __restrict__ tag_ctr, int* __restrict__ d_gen) {
    hg_pdl_begin();
    relabel_seg_body<W>(frontier, d_n, cap, f, counts, slots, slot_local, minpos, nself, outdeg, tag_ctr, d_gen);
}


__global__ void k_relabel_sort_seq(const int* __restrict__ frontier, const int* d_n, int cap, int f,
                                   const int* __restrict__ counts, int* __restrict__ slots,
                                   int* __restrict__ slot_local, const unsigned long long* __restrict__ minpos,
                                   const int* __restrict__ rank, int* __restrict__ nself,
                                   int* __restrict__ outdeg, int* __restrict__ tag_ctr, int* __restrict__ d_gen) {
    hg_pdl_begin();
    const int n = hg_load_count(d_n, cap);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *tag_ctr += 1;
        *d_gen += 1;
    }
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int cnt = counts[i];
        const int v = frontier[i];
        int* sp = slots + (int64_t)i * f;
        int* lp = slot_local + (int64_t)i * f;
        int ns = 0;
        for (int j = 0; j < cnt; ++j) {
            lp[j] = (int)(uint32_t)minpos[sp[j]];
            ns += sp[j] != v;
        }
        for (int j = 1; j < cnt; ++j) {  // stable insertion sort by local id
            int l = lp[j], u = sp[j], k = j - 1;
            while (k >= 0 && lp[k] > l) { lp[k + 1] = lp[k]; sp[k + 1] = sp[k]; --k; }
            lp[k + 1] = l;
            sp[k + 1] = u;
        }
        if (outdeg) for (int j = 0; j < cnt; ++j) atomicAdd(&outdeg[lp[j]], 1);
        if (nself) nself[i] = ns;
    }
}

__global__ void k_fo_advance(int* __restrict__ tag_ctr) { *tag_ctr += 1; }

// compacted edges (Block.edge_src / edge_dst) from the slot form; starts =
// exclusive scan of counts
__global__ void k_block_edges(const int* d_n, int cap, int f, const int* __restrict__ counts,
                              const int* __restrict__ starts, const int* __restrict__ slot_local,
                              int* __restrict__ edge_src, int* __restrict__ edge_dst) {
    const int n = hg_load_count(d_n, cap);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)n * f;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / f), j = (int)(q - (long long)i * f);
        if (j < counts[i]) {
            edge_src[starts[i] + j] = slot_local[q];
            edge_dst[starts[i] + j] = i;
        }
    }
}

// raw-sample emission (kernels.sample_layer): edges in (dst, draw) order
__global__ void k_emit_raw(const int* d_n, int cap, int f, const int* __restrict__ counts,
                           const int* __restrict__ starts, const int* __restrict__ slots,
                           int* __restrict__ edge_dst, int* __restrict__ edge_src) {
    const int n = hg_load_count(d_n, cap);
    for (long long q = blockIdx.x * (long long)blockDim.x + threadIdx.x; q < (long long)n * f;
         q += (long long)gridDim.x * blockDim.x) {
        const int i = (int)(q / f), j = (int)(q - (long long)i * f);
        if (j < counts[i]) {
            edge_dst[starts[i] + j] = i;
            edge_src[starts[i] + j] = slots[q];
        }
    }
}

int seg_width(int f) { return f <= 4 ? 4 : f <= 8 ? 8 : f <= 16 ? 16 : 32; }

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================

// Draw step of one layer (kernels.py:77-118).  d_seed: the batch rng seed when
// layer >= 0 (stream = derive_seed(seed, 0x5A, layer), sampler.py:143), else the
// stream seed itself (kernels.sample_layer).  scratch: cap*2*fanout ints, only
// touched when fanout > 32.
static int sample_layer_impl(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                             const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                             int32_t layer, int32_t* counts, int32_t* slots, uint64_t* minpos, int32_t* tag_ctr,
                             int32_t* scratch, int32_t* nself, cudaStream_t s) {
    if (fanout < 1 || cap_dst < 0) { hg_set_error("sample_layer: bad fanout/cap"); return HG_EINVAL; }
    if ((long long)cap_dst * (fanout + 1) >= 0x7fffffffLL) { hg_set_error("sample_layer: cap too large"); return HG_EINVAL; }
    if (cap_dst == 0) return HG_OK;
    unsigned long long* mp = (unsigned long long*)minpos;
    if (fanout <= 32) {
        const int W = seg_width(fanout);
        const int grid = hg_grid((long long)cap_dst * W, 256, hg_sample_ctas_per_sm());
        switch (W) {
            case 4: hg_launch(k_sample_seg<4>, grid, 256, 0, s, offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots, mp, tag_ctr, nself); break;
            case 8: hg_launch(k_sample_seg<8>, grid, 256, 0, s, offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots, mp, tag_ctr, nself); break;
            case 16: hg_launch(k_sample_seg<16>, grid, 256, 0, s, offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots, mp, tag_ctr, nself); break;
            default: hg_launch(k_sample_seg<32>, grid, 256, 0, s, offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots, mp, tag_ctr, nself); break;
        }
    } else {
        if (!scratch) { hg_set_error("sample_layer: fanout > 32 needs scratch"); return HG_EINVAL; }
        hg_launch(k_sample_seq, hg_grid(cap_dst, 128, 8), 128, 0, s, offsets, targets, frontier, d_n_dst, cap_dst,
                  fanout, d_seed, layer, counts, slots, mp, tag_ctr, scratch, nself);
    }
    return hg_check_launch("sample_layer");
}

// Draw step of one layer (kernels.py:77-118).  d_seed: the batch rng seed when
// layer >= 0 (stream = derive_seed(seed, 0x5A, layer), sampler.py:143), else the
// stream seed itself (kernels.sample_layer).  scratch: cap*2*fanout ints, only
// touched when fanout > 32.
extern "C" int hg_sample_layer(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                               const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                               const uint64_t* d_seed, int32_t layer, int32_t* counts, int32_t* slots,
                               uint64_t* minpos, int32_t* tag_ctr, int32_t* scratch, void* stream) {
    if (fanout >= 1 && cap_dst > 0 && !minpos) {
        hg_set_error("sample_layer: minpos required (see hg_sample_layer_draws)");
        return HG_EINVAL;
    }
    return sample_layer_impl(offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots,
                             minpos, tag_ctr, scratch, nullptr, (cudaStream_t)stream);
}

// Draws only, for a block whose sources are consumed by GLOBAL id (the SAGE
// bottom layer: the fused gather reads feature rows directly, and no backward
// transposed aggregation exists below it): no first-occurrence marks and no
// dedup/relabel pass; per-destination non-self counts come from the draw kernel.
extern "C" int hg_sample_layer_draws(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                                     const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                                     int32_t layer, int32_t* counts, int32_t* slots, int32_t* nself,
                                     int32_t* scratch, void* stream) {
    return sample_layer_impl(offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots,
                             nullptr, nullptr, scratch, nself, (cudaStream_t)stream);
}

// Retire a first-occurrence tag without a dedup pass (a bare draw).
extern "C" int hg_first_occurrence_advance(int32_t* tag_ctr, void* stream) {
    k_fo_advance<<<1, 1, 0, (cudaStream_t)stream>>>(tag_ctr);
    return hg_check_launch("first_occurrence_advance");
}

// Dedup + relabel + per-dst sort (kernels.py:166-180, sampler.py:106-118).
// ws: >= hg_dedup_ws_size(cap_dst, fanout) ints.  Produces src_vertices[0..n_src),
// *d_n_src, sorted slots / slot_local, nself (nullable), outdeg (nullable; entries
// [0, n_src) reset by the mark/scan pass), and retires the first-occurrence tag.
// ws layout (ints): rank[P] | pad | status (uint64)[tiles] | generation counter.
// The workspace must be zero-filled once when allocated and then kept.
extern "C" int64_t hg_dedup_ws_size(int32_t cap_dst, int32_t fanout) {
    long long P = (long long)cap_dst * (fanout + 1);
    long long tiles = (P + MS_TILE - 1) / MS_TILE;
    return (int64_t)(((P + 1) & ~1LL) + 2 * tiles + 4);
}

// First half of hg_dedup_relabel: the mark/scan/emit pass alone.  Produces
// src_vertices[0..n_src), *d_n_src and resets outdeg[0..n_src); the table
// entries of first occurrences now hold local ids for hg_block_relabel.
extern "C" int hg_dedup_mark(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                             const int32_t* counts, const int32_t* slots, uint64_t* minpos, const int32_t* tag_ctr,
                             int32_t* src_vertices, int32_t* d_n_src, int32_t* outdeg, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cap_dst == 0) { cudaMemsetAsync(d_n_src, 0, sizeof(int), s); return hg_check_launch("dedup(empty)"); }
    const long long P = (long long)cap_dst * (fanout + 1);
    const long long tiles = (P + MS_TILE - 1) / MS_TILE;
    int* flags = ws;  // rank of each first-occurrence position
    unsigned long long* status = reinterpret_cast<unsigned long long*>(ws + ((P + 1) & ~1LL));
    int* d_gen = ws + ((P + 1) & ~1LL) + 2 * tiles;
    hg_launch(k_markscan, (unsigned)tiles, MS_THREADS, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots,
                                                      (unsigned long long*)minpos, tag_ctr, flags, src_vertices,
                                                      d_n_src, status, d_gen, outdeg);
    return hg_check_launch("dedup_mark");
}

// Second half: per-destination local ids + segment sort, nself / outdeg, and the
// retirement of the table's tag and the workspace's scan generation.  Nothing in
// the next layer's draw / mark reads its outputs, so it may run on another stream
// concurrently with them provided they use a DIFFERENT first-occurrence table.
extern "C" int hg_block_relabel(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                                const int32_t* counts, int32_t* slots, int32_t* slot_local, const uint64_t* minpos,
                                int32_t* tag_ctr, int32_t* nself, int32_t* outdeg, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cap_dst == 0) return HG_OK;
    const long long P = (long long)cap_dst * (fanout + 1);
    const long long tiles = (P + MS_TILE - 1) / MS_TILE;
    int* flags = ws;
    int* d_gen = ws + ((P + 1) & ~1LL) + 2 * tiles;
    if (fanout <= 32) {
        const int W = seg_width(fanout);
        const int grid = hg_grid((long long)cap_dst * W, 256, hg_sample_ctas_per_sm());
        switch (W) {
            case 4: hg_launch(k_relabel_sort_seg<4>, grid, 256, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, (const unsigned long long*)minpos, flags, nself, outdeg, tag_ctr, d_gen); break;
            case 8: hg_launch(k_relabel_sort_seg<8>, grid, 256, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, (const unsigned long long*)minpos, flags, nself, outdeg, tag_ctr, d_gen); break;
            case 16: hg_launch(k_relabel_sort_seg<16>, grid, 256, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, (const unsigned long long*)minpos, flags, nself, outdeg, tag_ctr, d_gen); break;
            default: hg_launch(k_relabel_sort_seg<32>, grid, 256, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, (const unsigned long long*)minpos, flags, nself, outdeg, tag_ctr, d_gen); break;
        }
    } else {
        hg_launch(k_relabel_sort_seq, hg_grid(cap_dst, 128, 8), 128, 0, s, frontier, d_n_dst, cap_dst, fanout, counts, slots,
                                                                    slot_local, (const unsigned long long*)minpos,
                                                                    flags, nself, outdeg, tag_ctr, d_gen);
    }
    return hg_check_launch("block_relabel");
}

extern "C" int hg_dedup_relabel(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                                const int32_t* counts, int32_t* slots, int32_t* slot_local, uint64_t* minpos,
                                int32_t* tag_ctr, int32_t* src_vertices, int32_t* d_n_src, int32_t cap_src, int32_t* nself,
                                int32_t* outdeg, int32_t* ws, void* stream) {
    int rc = hg_dedup_mark(frontier, d_n_dst, cap_dst, fanout, counts, slots, minpos, tag_ctr, src_vertices, d_n_src,
                           outdeg, ws, stream);
    if (rc) return rc;
    return hg_block_relabel(frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, minpos, tag_ctr, nself,
                            outdeg, ws, stream);
}

// Draw + dedup + relabel of one layer (hg_sample_layer followed by
// hg_dedup_relabel).
extern "C" int hg_sample_block(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                               const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                               int32_t layer, int32_t* counts, int32_t* slots, int32_t* slot_local, uint64_t* minpos,
                               int32_t* tag_ctr, int32_t* src_vertices, int32_t* d_n_src, int32_t cap_src,
                               int32_t* nself, int32_t* outdeg, int32_t* ws, int32_t* scratch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (fanout < 1 || cap_dst < 0) { hg_set_error("sample_block: bad fanout/cap"); return HG_EINVAL; }
    if (cap_dst == 0) { cudaMemsetAsync(d_n_src, 0, sizeof(int), s); return hg_check_launch("sample_block(empty)"); }
    int rc = sample_layer_impl(offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots,
                               minpos, tag_ctr, scratch, nullptr, s);
    if (rc) return rc;
    return hg_dedup_relabel(frontier, d_n_dst, cap_dst, fanout, counts, slots, slot_local, minpos, tag_ctr,
                            src_vertices, d_n_src, cap_src, nself, outdeg, ws, stream);
}

extern "C" int hg_sample_block_mark(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                                    const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                                    int32_t layer, int32_t* counts, int32_t* slots, uint64_t* minpos,
                                    int32_t* tag_ctr, int32_t* src_vertices, int32_t* d_n_src, int32_t* outdeg,
                                    int32_t* ws, int32_t* scratch, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (fanout < 1 || cap_dst < 0) { hg_set_error("sample_block_mark: bad fanout/cap"); return HG_EINVAL; }
    if (!minpos) { hg_set_error("sample_block_mark: minpos required"); return HG_EINVAL; }
    if (cap_dst == 0) { cudaMemsetAsync(d_n_src, 0, sizeof(int), s); return hg_check_launch("sample_block_mark(empty)"); }
    int rc = sample_layer_impl(offsets, targets, frontier, d_n_dst, cap_dst, fanout, d_seed, layer, counts, slots,
                               minpos, tag_ctr, scratch, nullptr, s);
    if (rc) return rc;
    return hg_dedup_mark(frontier, d_n_dst, cap_dst, fanout, counts, slots, minpos, tag_ctr, src_vertices, d_n_src,
                         outdeg, ws, stream);
}

// Compacted Block edges; starts: cap_dst ints workspace (+ scan ws after it).
extern "C" int64_t hg_block_edges_ws_size(int32_t cap_dst) {
    return (int64_t)(cap_dst + (long long)hg_scan_ws_ints(cap_dst) + 16);
}

extern "C" int hg_block_to_edges(const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const int32_t* counts,
                                 const int32_t* slot_local, int32_t* edge_src, int32_t* edge_dst,
                                 int32_t* d_n_edges, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cap_dst == 0) { cudaMemsetAsync(d_n_edges, 0, sizeof(int), s); return HG_OK; }
    int rc = hg_scan_launch(counts, ws, d_n_dst, 1, cap_dst, d_n_edges, ws + cap_dst, s);
    if (rc) return rc;
    k_block_edges<<<hg_grid((long long)cap_dst * fanout, 256, 8), 256, 0, s>>>(d_n_dst, cap_dst, fanout, counts,
                                                                               ws, slot_local, edge_src, edge_dst);
    return hg_check_launch("block_to_edges");
}

extern "C" int hg_raw_edges(const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const int32_t* counts,
                            const int32_t* slots, int32_t* edge_dst, int32_t* edge_src, int32_t* d_n_edges,
                            int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (cap_dst == 0) { cudaMemsetAsync(d_n_edges, 0, sizeof(int), s); return HG_OK; }
    int rc = hg_scan_launch(counts, ws, d_n_dst, 1, cap_dst, d_n_edges, ws + cap_dst, s);
    if (rc) return rc;
    k_emit_raw<<<hg_grid((long long)cap_dst * fanout, 256, 8), 256, 0, s>>>(d_n_dst, cap_dst, fanout, counts, ws,
                                                                            slots, edge_dst, edge_src);
    return hg_check_launch("raw_edges");
}

// ---------------------------------------------------------------------------
// generic first-occurrence dedup of int64 values (kernels.stable_unique):
// open-addressing hash (key, min position) + flags/scan/emit
// ---------------------------------------------------------------------------
namespace {
__device__ __forceinline__ uint32_t hash_slot(unsigned long long key, uint32_t mask) {
    return (uint32_t)hg_mix64(key) & mask;
}
constexpr unsigned long long EMPTY_KEY = 0xffffffffffffffffULL;

__global__ void k_uq_insert(const long long* __restrict__ vals, long long n, unsigned long long* __restrict__ hkeys,
                            int* __restrict__ hpos, uint32_t mask) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const unsigned long long key = (unsigned long long)vals[p];
        if (key == EMPTY_KEY) { atomicMin(&hpos[mask + 1], (int)p); continue; }  // sentinel-valued id
        uint32_t h = hash_slot(key, mask);
        while (true) {
            unsigned long long prev = atomicCAS(&hkeys[h], EMPTY_KEY, key);
            if (prev == EMPTY_KEY || prev == key) { atomicMin(&hpos[h], (int)p); break; }
            h = (h + 1) & mask;
        }
    }
}

__device__ __forceinline__ uint32_t uq_find(unsigned long long key, const unsigned long long* hkeys, uint32_t mask) {
    if (key == EMPTY_KEY) return mask + 1;
    uint32_t h = hash_slot(key, mask);
    while (hkeys[h] != key) h = (h + 1) & mask;
    return h;
}

__global__ void k_uq_flags(const long long* __restrict__ vals, long long n, const unsigned long long* __restrict__ hkeys,
                           const int* __restrict__ hpos, uint32_t mask, int* __restrict__ flags,
                           int* __restrict__ slot_of) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const uint32_t h = uq_find((unsigned long long)vals[p], hkeys, mask);
        slot_of[p] = (int)h;
        flags[p] = hpos[h] == (int)p;
    }
}

__global__ void k_uq_emit(const long long* __restrict__ vals, long long n, const int* __restrict__ hpos,
                          const int* __restrict__ slot_of, const int* __restrict__ rank,
                          long long* __restrict__ uniq, long long* __restrict__ inverse) {
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n; p += (long long)gridDim.x * blockDim.x) {
        const int first = hpos[slot_of[p]];
        if (first == (int)p) uniq[rank[p]] = vals[p];
        inverse[p] = rank[first];
    }
}
}  // namespace

extern "C" int64_t hg_unique_ws_size(int64_t n) {
    long long cap = 16;
    while (cap < 2 * n) cap <<= 1;
    return (int64_t)(2 * cap + cap + 1 + 2 * n + (long long)hg_scan_ws_ints(n) + 16);
}

// uniq (n) / inverse (n) int64; *d_n_uniq = unique count.
extern "C" int hg_unique_first_i64(const int64_t* vals, int64_t n, int64_t* uniq, int64_t* inverse,
                                   int32_t* d_n_uniq, int32_t* ws, void* stream) {
    cudaStream_t s = (cudaStream_t)stream;
    if (n <= 0) { cudaMemsetAsync(d_n_uniq, 0, sizeof(int), s); return HG_OK; }
    if (n >= 0x7fffffffLL) { hg_set_error("unique_first: n too large"); return HG_EINVAL; }
    long long cap = 16;
    while (cap < 2 * n) cap <<= 1;
    unsigned long long* hkeys = (unsigned long long*)ws;
    int* hpos = ws + 2 * cap;
    int* flags = hpos + cap + 1;
    int* slot_of = flags + n;
    int* scan_ws = slot_of + n;
    cudaMemsetAsync(hkeys, 0xff, sizeof(unsigned long long) * cap, s);
    cudaMemsetAsync(hpos, 0x7f, sizeof(int) * (cap + 1), s);
    const int g = hg_grid(n, 256, 8);
    const uint32_t mask = (uint32_t)(cap - 1);
    k_uq_insert<<<g, 256, 0, s>>>((const long long*)vals, n, hkeys, hpos, mask);
    k_uq_flags<<<g, 256, 0, s>>>((const long long*)vals, n, hkeys, hpos, mask, flags, slot_of);
    int rc = hg_scan_launch(flags, flags, nullptr, 1, n, d_n_uniq, scan_ws, s);
    if (rc) return rc;
    k_uq_emit<<<g, 256, 0, s>>>((const long long*)vals, n, hpos, slot_of, flags, (long long*)uniq,
                                (long long*)inverse);
    return hg_check_launch("unique_first_i64");
}

// counter[v] += 1 for every v in ids (kernels.py:161-163), int64 counters
namespace {
__global__ void k_count_into(long long* __restrict__ counter, const int* __restrict__ ids, const int* d_n, int cap) {
    const int n = hg_load_count(d_n, cap);
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&counter[ids[k]], 1ULL);
}
__global__ void k_count_into64(long long* __restrict__ counter, const long long* __restrict__ ids, long long n) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        atomicAdd((unsigned long long*)&counter[ids[k]], 1ULL);
}
}  // namespace

extern "C" int hg_count_into(int64_t* counter, const int32_t* ids, const int32_t* d_n, int32_t cap, void* stream) {
    if (cap <= 0) return HG_OK;
    k_count_into<<<hg_grid(cap, 256, 8), 256, 0, (cudaStream_t)stream>>>((long long*)counter, ids, d_n, cap);
    return hg_check_launch("count_into");
}

extern "C" int hg_count_into_i64(int64_t* counter, const int64_t* ids, int64_t n, void* stream) {
    if (n <= 0) return HG_OK;
    k_count_into64<<<hg_grid(n, 256, 8), 256, 0, (cudaStream_t)stream>>>((long long*)counter, (const long long*)ids, n);
    return hg_check_launch("count_into_i64");
}
