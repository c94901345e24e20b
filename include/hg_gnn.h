/*
 * hg_gnn — C ABI of the B200-native sample-based GNN training hot path
 * (NeutronOrch, arXiv 2311.13225; reference package `hetgnn` v0.1.0).
 *
 * Conventions
 *  - Plain pointers and sizes only.  Every pointer argument is DEVICE memory
 *    unless the parameter name says `host_`; the caller allocates every buffer
 *    including workspaces (sizes from the *_ws_size functions, in elements of
 *    the pointer's type).  The library keeps no allocations and no global
 *    mutable state; all entry points are reentrant.
 *  - `stream` is a cudaStream_t (CUstream) passed as void*; work is enqueued
 *    asynchronously on it.  Nothing synchronises the host.
 *  - Counts that are produced by a previous step (frontier sizes, edge counts)
 *    are passed as `const int32_t* d_n` device pointers together with a host
 *    upper bound `cap`; a NULL d_n means "exactly cap".  This lets a whole
 *    training step be captured into one CUDA graph.
 *  - Vertex ids are int32 on device (V < 2^31); CSR offsets are int64.
 *  - Return value: 0 on success, < 0 on error (-1 invalid argument, -2 CUDA
 *    launch error, -3 unsupported shape); hg_last_error() has the message
 *    (thread-local).  The Python layer maps these onto the reference's
 *    exception classes (SamplerError, ShapeError, ...).
 *
 * Each entry point names the reference interface it replaces (file:line in
 * /root/reference/pkg/src/hetgnn).
 */
#ifndef HG_GNN_H
#define HG_GNN_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HG_GNN_ABI_VERSION 1

int hg_abi_version(void);
int hg_last_error(char* buf, int len);
/* kernel nodes in a captured cudaGraph_t (passed as void*); -1 on error */
int64_t hg_graph_kernel_count(void* graph);

/* ---- splitmix64 streams: kernels.py:51-70 (_mix64, derive_seed) -------- */
uint64_t hg_mix64_host(uint64_t x);
uint64_t hg_derive_seed(uint64_t seed, const uint64_t* host_parts, int n_parts);

/* ---- K1 neighbour draw: kernels.py:77-118,147-158 (_sample_layer /
 *      sample_layer).  layer >= 0: *d_seed is the batch rng seed and the
 *      stream is derive_seed(seed, 0x5A, layer) (sampler.py:143); layer < 0:
 *      *d_seed is the stream seed itself.  Writes counts[i] = min(deg, f) and
 *      the drawn global ids into slots[i*f + j] (emission order), and
 *      atomicMin's (tag << 32 | position) into the first-occurrence table
 *      minpos[V] (all ~0 when allocated, never reset; tag = 0xFFFFFFFE -
 *      *tag_ctr).  scratch: cap_dst*2*fanout ints, used only when fanout > 32. */
int hg_sample_layer(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                    const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                    int32_t layer, int32_t* counts, int32_t* slots, uint64_t* minpos, int32_t* tag_ctr,
                    int32_t* scratch, void* stream);
/* Draws only (same draws, counts and slot contents as hg_sample_layer) for a
 * block consumed by global source ids (the SAGE bottom layer of the training
 * step): no first-occurrence marks, no dedup pass; nself (nullable) receives the
 * per-destination non-self counts (gnnmath.py:145-154). */
int hg_sample_layer_draws(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                          const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                          int32_t layer, int32_t* counts, int32_t* slots, int32_t* nself, int32_t* scratch,
                          void* stream);

/* Retires the current first-occurrence tag after a draw that is not followed
 * by hg_dedup_relabel (which retires it itself). */
int hg_first_occurrence_advance(int32_t* tag_ctr, void* stream);

/* ---- K2/K3 dedup + relabel + (dst, src) order: kernels.py:166-180
 *      (stable_unique) and sampler.py:104-118 (_expand_frontier lexsort).
 *      Produces src_vertices (first-occurrence order, dst prefix first),
 *      *d_n_src, slots re-ordered by local src id with slot_local, per-dst
 *      non-self counts `nself` (gnnmath.py:145-154; nullable) and block
 *      out-degrees `outdeg` (gnnmath.py:96; nullable; entries [0, n_src) are reset by the call), and
 *      bumps *tag_ctr so the next use of minpos starts clean (first-occurrence
 *      entries are left holding their local id under the reserved tag 0xFFFFFFFF). */
int64_t hg_dedup_ws_size(int32_t cap_dst, int32_t fanout);
/* hg_sample_layer + hg_dedup_relabel in one call (same arguments, same outputs). */
int hg_sample_block(const int64_t* offsets, const int32_t* targets, const int32_t* frontier, const int32_t* d_n_dst,
                    int32_t cap_dst, int32_t fanout, const uint64_t* d_seed, int32_t layer, int32_t* counts,
                    int32_t* slots, int32_t* slot_local, uint64_t* minpos, int32_t* tag_ctr, int32_t* src_vertices,
                    int32_t* d_n_src, int32_t cap_src, int32_t* nself, int32_t* outdeg, int32_t* ws,
                    int32_t* scratch, void* stream);
int hg_dedup_relabel(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                     const int32_t* counts, int32_t* slots, int32_t* slot_local, uint64_t* minpos,
                     int32_t* tag_ctr, int32_t* src_vertices, int32_t* d_n_src, int32_t cap_src, int32_t* nself,
                     int32_t* outdeg, int32_t* ws, void* stream);
/* hg_dedup_relabel in two halves.  hg_dedup_mark: src_vertices, *d_n_src, outdeg
 * reset (what the NEXT layer's draw needs).  hg_block_relabel: slots order,
 * slot_local, nself, outdeg, tag retirement (what only the training step needs);
 * it may run on a second stream concurrently with the next layer's sampling when
 * that layer uses a different first-occurrence table.  hg_sample_block_mark =
 * hg_sample_layer + hg_dedup_mark. */
int hg_dedup_mark(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                  const int32_t* counts, const int32_t* slots, uint64_t* minpos, const int32_t* tag_ctr,
                  int32_t* src_vertices, int32_t* d_n_src, int32_t* outdeg, int32_t* ws, void* stream);
int hg_block_relabel(const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                     const int32_t* counts, int32_t* slots, int32_t* slot_local, const uint64_t* minpos,
                     int32_t* tag_ctr, int32_t* nself, int32_t* outdeg, int32_t* ws, void* stream);
int hg_sample_block_mark(const int64_t* offsets, const int32_t* targets, const int32_t* frontier,
                         const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const uint64_t* d_seed,
                         int32_t layer, int32_t* counts, int32_t* slots, uint64_t* minpos, int32_t* tag_ctr,
                         int32_t* src_vertices, int32_t* d_n_src, int32_t* outdeg, int32_t* ws, int32_t* scratch,
                         void* stream);

/* Block.edge_src / edge_dst (sampler.py:45-78) from the slot form. */
int64_t hg_block_edges_ws_size(int32_t cap_dst);
int hg_block_to_edges(const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const int32_t* counts,
                      const int32_t* slot_local, int32_t* edge_src, int32_t* edge_dst, int32_t* d_n_edges,
                      int32_t* ws, void* stream);
/* Raw emission (edge_dst_local, edge_src_global) of kernels.sample_layer. */
int hg_raw_edges(const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout, const int32_t* counts,
                 const int32_t* slots, int32_t* edge_dst, int32_t* edge_src, int32_t* d_n_edges, int32_t* ws,
                 void* stream);

/* ---- generic plug-in kernels (numpy-shaped API) ------------------------- */
/* kernels.stable_unique (kernels.py:166-180) for arbitrary int64 values. */
int64_t hg_unique_ws_size(int64_t n);
int hg_unique_first_i64(const int64_t* vals, int64_t n, int64_t* uniq, int64_t* inverse, int32_t* d_n_uniq,
                        int32_t* ws, void* stream);
/* kernels.count_into (kernels.py:161-163). */
int hg_count_into(int64_t* counter, const int32_t* ids, const int32_t* d_n, int32_t cap, void* stream);
int hg_count_into_i64(int64_t* counter, const int64_t* ids, int64_t n, void* stream);
/* kernels.segment_weighted_rows (kernels.py:121-144), fp64, bit-exact. */
int64_t hg_swr_ws_size(int64_t n_edges, int32_t n_out);
int hg_segment_weighted_rows_f64(const int64_t* edge_src, const int64_t* edge_dst, const double* w,
                                 int64_t n_edges, const double* rows, int32_t d, int32_t n_out, double* out,
                                 int32_t* ws, void* stream);

/* ---- K4-K7 gather + aggregation (orchestrator.py:239; gnnmath.py:89-200) --
 *  model 0 = SAGE mean of non-self neighbours, 1 = GCN block sym-norm.
 *  global_src 1: rows addressed by global id (bottom layer: reads the feature
 *  table and also writes the gathered self rows to self_out); 0: by local id. */
int hg_aggregate_fwd(int32_t model, int32_t global_src, const float* hin, int32_t ld_in, int32_t F,
                     const int32_t* frontier, const int32_t* d_n_dst, int32_t cap_dst, int32_t fanout,
                     const int32_t* counts, const int32_t* slot_g, const int32_t* slot_local, const int32_t* nself,
                     const int32_t* outdeg, const uint8_t* inj_mask, float* self_out, int32_t ld_self,
                     float* agg_out, int32_t ld_agg, void* stream);
/* Bottom-layer hg_aggregate_fwd over a feature table row-sharded across devices
 * (C4, features larger than one GPU): shard_ptrs is a HOST array of n_shards (<= 8)
 * device pointers (NVLink peer pointers from hg_ipc_open_handle, or slices of one
 * table), each holding rows_per_shard rows of stride ld_in; row v lives in shard
 * v / rows_per_shard.  Outputs are bit-identical to the unsharded call. */
int hg_aggregate_fwd_sharded(int32_t model, const float* const* shard_ptrs, int32_t n_shards, int32_t rows_per_shard,
                             int32_t ld_in, int32_t F, const int32_t* frontier, const int32_t* d_n_dst,
                             int32_t cap_dst, int32_t fanout, const int32_t* counts, const int32_t* slot_g,
                             const int32_t* slot_local, const int32_t* nself, const int32_t* outdeg,
                             const uint8_t* inj_mask, float* self_out, int32_t ld_self, float* agg_out,
                             int32_t ld_agg, void* stream);
/* Bottom-layer hg_aggregate_fwd (orchestrator.py:239) over a split-row copy of the
 * feature table: columns [0, body_cols) of row v at body + v*ld_body (128-byte
 * aligned, ld_body a multiple of 32: whole 128-byte lines), columns [body_cols, F)
 * at tail + v*ld_tail (the small tail table is kept in L2).  F <= 128.  Outputs are
 * bit-identical to hg_aggregate_fwd on the unsplit table. */
int hg_aggregate_fwd_split(int32_t model, const float* body, int32_t ld_body, const float* tail, int32_t ld_tail,
                           int32_t body_cols, int32_t F, const int32_t* frontier, const int32_t* d_n_dst,
                           int32_t cap_dst, int32_t fanout, const int32_t* counts, const int32_t* slot_g,
                           const int32_t* slot_local, const int32_t* nself, const int32_t* outdeg,
                           const uint8_t* inj_mask, float* self_out, int32_t ld_self, float* agg_out,
                           int32_t ld_agg, void* stream);
/* CUDA IPC between the per-GPU processes (64-byte cudaIpcMemHandle_t blobs); the
 * handle names dptr's whole allocation and *out_offset locates dptr inside it */
int hg_ipc_get_handle(const void* dptr, uint8_t* out_handle64, int64_t* out_offset);
int hg_ipc_open_handle(const uint8_t* handle64, void** out_ptr);
int hg_ipc_close(void* ptr);
int hg_enable_peer_access(int32_t peer_device);
/* Transposed aggregation by deterministic fixed-point scatter (layers >= 1): dx[s] = mask(dself[s] (s < n_dst) + sum_e w_e dagg[dst_e]) with
 * the sum accumulated in two-word fixed point (hi = v*2^20, lo = remainder*2^60, two
 * int64 words; order-independent, bit-exact across runs, exact for every fp32
 * contribution >= 2^-37) in acc_ws (int64 [cap_src x 2F]: a row's F hi words then its
 * F lo words; zero on first use, left zeroed);
 * outdeg (required): sampled edges per local source (hg_dedup_relabel's outdeg);
 * sources s >= n_dst with outdeg 1 get their final row stored directly;
 * d_flags[0] |= 1 if a contribution is non-finite, |= 2 if outdeg * |v| >= 2^42. */
int hg_aggregate_bwd_scatter(int32_t model, const float* dagg, int32_t ld_dagg, const float* dself,
                             int32_t ld_dself, int32_t F, const int32_t* frontier, const int32_t* d_n_dst,
                             int32_t cap_dst, int32_t fanout, const int32_t* counts, const int32_t* slot_g,
                             const int32_t* slot_local, const int32_t* nself, const int32_t* outdeg,
                             const int32_t* d_n_src, int32_t cap_src, const float* hmask, int32_t ld_hmask,
                             const uint8_t* inj_mask, int64_t* acc_ws, float* dx, int32_t ld_dx, int32_t* d_flags,
                             void* stream);
/* Top SAGE layer fused (K = d_in <= 64, C = classes <= 64, fanout <= 32): mean of the
 * non-self neighbours (local ids into hin) -> logits = [h_self | mean] [W_self; W_neigh]
 * (W: the layer's flat [2K x C] weights) -> softmax-CE (loss into *d_loss, dlogits)
 * -> dself = dlogits W_self^T (into dself_out) -> dmean = dlogits W_neigh^T scattered
 * into the layer below exactly like hg_aggregate_bwd_scatter's scatter pass (fast path
 * into dx, else the two-word fixed-point acc_ws of row stride 2 * F_acc); follow with
 * hg_aggregate_bwd_finish.  row_ws: cap + 1 floats as hg_softmax_xent's. */
int hg_sage_top_fused(const float* hin, int32_t ld_in, int32_t K, const int32_t* frontier, const int32_t* d_n,
                      int32_t cap, int32_t fanout, const int32_t* counts, const int32_t* slot_g,
                      const int32_t* slot_local, const int32_t* nself, const int32_t* outdeg, const float* W,
                      int32_t C, const int32_t* labels, const int32_t* seeds, const int32_t* d_div, float* logits,
                      int32_t ld_c, float* dlogits, float* agg_out, int32_t ld_agg, float* dself_out,
                      int32_t ld_dself, const float* hmask, int32_t ld_hmask, const uint8_t* inj_mask,
                      int64_t* acc_ws, int32_t F_acc, float* dx, int32_t ld_dx, int32_t* d_flags, float* row_ws,
                      float* d_loss, void* stream);
/* the finish pass of hg_aggregate_bwd_scatter alone (convert the fixed-point sums, add
 * dself for s < n_dst, ReLU' / injected-row masks, clear the accumulator) */
int hg_aggregate_bwd_finish(const float* dself, int32_t ld_dself, int32_t F, const int32_t* d_n_dst, int32_t cap_dst,
                            const int32_t* d_n_src, int32_t cap_src, const int32_t* outdeg, const float* hmask,
                            int32_t ld_hmask, const uint8_t* inj_mask, int64_t* acc_ws, float* dx, int32_t ld_dx,
                            void* stream);
/* ---- K8 dense transforms (gnnmath.py:121,135,139,173,190-198) ---------- */
/* tcgen05 (5th-gen tensor core, kind::tf32, 3xTF32 split => fp32-class accuracy).
 *  C = act(A1 op(B)[0:K1] + A2 op(B)[K1:K1+K2]); op(B)(k,n) = B[k*ldb+n] if trans_b
 *  (forward: B = [W_self; W_neigh] stacked [K x N]) else B[n*ldb+k] (dX = dZ W^T).
 *  B is consumed as a prebuilt swizzled hi/lo image (hg_gemm_tc_prep_b, once per
 *  weight update; hg_gemm_tc_bimg_size bytes, 16-byte aligned). */
int64_t hg_gemm_tc_bimg_size(int32_t K1, int32_t K2, int32_t N);
int hg_gemm_tc_prep_b(const float* B, int32_t ldb, int32_t trans_b, int32_t K1, int32_t K2, int32_t N, void* img,
                      void* stream);
/* up to 8 images in one launch; host_desc: n rows of int64 {B, ldb, trans_b, K1, K2, N, img} */
int hg_gemm_tc_prep_b_many(int32_t n, const int64_t* host_desc, void* stream);
int hg_gemm_tc(const float* A1, int32_t lda1, int32_t K1, const float* A2, int32_t lda2, int32_t K2,
               const void* bimg, float* C, int32_t ldc, int32_t N, const int32_t* d_M, int32_t M_cap, int32_t act,
               void* stream);
/* process-wide tuning knobs for the tensor-core kernels (key 1: MN-major descriptor offsets;
 * key 3: forward GEMM form, 1 = A operand through TMEM (default), 0 = both operands from smem;
 * key 5: programmatic dependent launch of the step kernels, 1 (default; env HG_PDL=0 at load turns it off) / 0;
 * key 7: paired hi|lo MMAs (N = 2*BN operand, two instructions per K slice instead of three) for BN <= 64 (1, default) / 0;
 * key 11: weight gradient with A^T's hi/lo written to TMEM by the split warps, MMAs reading only G from
 *        shared memory (1, default) / both operands from shared memory (0);
 * key 12: wide-row (F > 128) aggregation stages rows into shared memory with TMA bulk copies
 *        (cp.async.bulk + mbarrier; 1) / per-lane 128-bit loads (0, default: measured 2.4x faster at
 *        C3's 2.4 KB rows) — bit-identical results */
int hg_set_tuning(int32_t key, int32_t value);
/* profiling aid: the 8 x 64 globaltimer stamps (ns) of the tensor-core GEMM's
 * pipeline timeline probe (hg_set_tuning key 9, bit 3) */
int hg_debug_timeline(uint64_t* out);
/* L2 residency: feature-gathering kernels launched after this call attach an
 * access-policy window [base, base+bytes) with persisting hits (hit_ratio of the
 * window's lines), and the device's persisting-L2 carve-out is set to bytes
 * (clamped to hg_l2_persist_max()).  base NULL / bytes 0 turns it off. */
int64_t hg_l2_persist_max(void);
int hg_set_l2_persist(const void* base, int64_t bytes, float hit_ratio);
/* out_s[K x N] = A_s^T G (s = 1, 2; A2 may be NULL), deterministic split-M. */
int64_t hg_wgrad_tc_ws_size(int32_t K, int32_t N, int32_t M_cap, int32_t n_src);
int hg_wgrad_tc(const float* A1, int32_t lda1, const float* A2, int32_t lda2, int32_t K, const float* G,
                int32_t ldg, int32_t N, const int32_t* d_M, int32_t M_cap, float* out1, float* out2, float* ws,
                void* stream);

/* Per-batch needed bottom rows (transfer.py:59-73, 87-115; the batch CSV's raw_rows and
 * cache_hit_rows): distinct sources of non-injected destinations + their self rows;
 * rows whose vertex is flagged in cached[V] (the case3/case4 static feature cache,
 * nullable) are added to out_hits[bp[3]], the rest to out[bp[3]]; tag_of: int32[V]
 * (any initial contents below 0 / never equal to a future reading_batch + 1),
 * tag = bp[2] + 1. */
int hg_count_needed_rows(const int32_t* frontier, const int32_t* d_n, int32_t cap, int32_t fanout,
                         const int32_t* counts, const int32_t* slots, const uint8_t* inj_mask, const int64_t* bp,
                         const uint8_t* cached, int32_t* tag_of, int32_t* out, int32_t* out_hits, void* stream);

/* ---- K9/K10 loss and updates (gnnmath.py:263-312; orchestrator.py:246-255) */
/* dlogits = (softmax - onehot) / *d_div (d_div NULL: / n); *d_loss = mean CE over
 * the n = min(*d_n, cap) rows; labels indexed by seeds[r] (seeds NULL: by r).
 * row_ws: cap + 1 floats, zero-filled once and then kept (per-row losses, reduced
 * in a fixed order by the last block to finish; row_ws[cap] is its ticket). */
int hg_softmax_xent(const float* logits, int32_t ld, int32_t C, const int32_t* d_n, int32_t cap,
                    const int32_t* labels, const int32_t* seeds, const int32_t* d_div, float* dlogits,
                    int32_t ldd, float* d_loss, float* row_ws, void* stream);
/* per-batch row record: loss_arr[bp[3]] = *d_loss, md_arr[bp[3]] = max|dw|; resets *d_maxdelta */
int hg_record_batch(const int64_t* bp, const float* d_loss, uint32_t* d_maxdelta, float* loss_arr,
                    float* md_arr, void* stream);
int hg_sgd(float* w, const float* g, int64_t n, float lr, uint32_t* d_maxdelta, void* stream);
/* hg_sgd + hg_gemm_tc_prep_b_many + hg_record_batch in ONE launch: the tensor-core
 * B images (host_desc: n_img <= 8 rows of int64 {B, ldb, trans_b, K1, K2, N, img},
 * every B inside w, images fully built once before) are rewritten from the updated
 * weights in the same pass; the last block records loss / max |dw| of the batch.
 * ctl: 2 uint32 zero at rest (max |dw| bits, last-block ticket). */
int hg_sgd_fused(float* w, const float* g, int64_t n, float lr, int32_t n_img, const int64_t* host_desc,
                 uint32_t* ctl, const int64_t* bp, const float* d_loss, float* loss_arr, float* md_arr, void* stream);
int hg_adam(float* w, const float* g, float* m, float* v, int64_t n, float lr, float b1, float b2, float eps,
            int32_t* d_t, uint32_t* d_maxdelta, void* stream);

/* Device-to-device copy of nbytes (16-byte aligned pointers) as one small kernel
 * (a graph kernel node; the sample half's hand-off of the batch inputs). */
int hg_copy_bytes(void* dst, const void* src, int64_t nbytes, void* stream);

/* ---- native step driver: the per-batch loop of Trainer.train_batches
 *      (orchestrator.py:520-560) over captured half-step graphs.  For step k:
 *      pack host_stage[k*slot_bytes, +slot_bytes) = bp_rows[k] (8 int64) at 0 |
 *      {n_seeds[k], n_div[k]} (int32) at counts_offset | the n_seeds[k] int64 seed ids
 *      at host_seed_ptrs[k] narrowed to int32 at seeds_offset (engine.stage_views),
 *      right before the step's launches; H2D of the packed bytes into dev_stage[k % n_sets]
 *      + sample_execs[k % n_sets] on sample_stream (after batch k - n_sets
 *      trained); train_execs[k % n_sets] on train_stream (after that sample half),
 *      which records batch k's loss at d_loss_arr[k] (bp[3] = k); at the end one
 *      D2H of d_loss_arr[0, n_steps) into host_loss.  Execs are cudaGraphExec_t; host_stage
 *      and host_loss pinned; both streams start after caller_stream, which waits
 *      for both at the end (asynchronous: synchronise caller_stream to read). */
int hg_pipeline_run(int32_t n_steps, int32_t n_sets, const int64_t* sample_execs, const int64_t* train_execs,
                    void* caller_stream, void* sample_stream, void* train_stream, const int64_t* dev_stage,
                    uint8_t* host_stage, int64_t slot_bytes, int32_t counts_offset, int32_t seeds_offset,
                    const int64_t* bp_rows, const int64_t* host_seed_ptrs, const int32_t* n_seeds,
                    const int32_t* n_div, const float* d_loss_arr, float* host_loss);

/* ---- K11 historical-embedding store (store.py:24-146; orchestrator.py:259-271,
 *      381-395 producer, 480-504 consumer, gnnmath.py:240-245 injection).
 *  bp: per-batch int64 parameter block (see hg_train.cu BP_* indices). */
int hg_store_put(const int32_t* ids, const int32_t* d_n, int32_t cap, const float* emb, int32_t ld_emb, int32_t H,
                 const int32_t* slot_of, float* tab, int32_t* ver, int32_t* stamp, int32_t version,
                 int32_t stamp_val, int32_t* d_puts, void* stream);
int hg_store_lookup(const int32_t* dst, const int32_t* d_n, int32_t cap, const int64_t* bp,
                    const int32_t* cpu_tag_of, const int32_t* slot_of, const int32_t* ver0, const int32_t* ver1,
                    const int32_t* stamp0, const int32_t* stamp1, int32_t gap_bound, uint8_t* inj_mask,
                    int32_t* inj_slot, int32_t* batch_hits, int32_t* batch_miss, int32_t* batch_warm,
                    uint64_t* stats, void* stream);
int hg_inject_rows(const uint8_t* inj_mask, const int32_t* inj_slot, const int32_t* d_n, int32_t cap,
                   const int64_t* bp, const float* tab0, const float* tab1, int32_t H, float* h, int32_t ldh,
                   void* stream);

/* ---- epoch planning helpers (orchestrator.py:200-229 queue replay) ------ */
int hg_tag_vertices(const int32_t* ids, const int32_t* d_n, int32_t cap, int32_t* tag_of, int32_t tag,
                    void* stream);
/* sample_khop_skip_hot hot flags (sampler.py:150-163: np.isin(bottom src, hot)):
 * flags[i] = (tag_of[values[i]] == tag) for i < *d_n (or cap when d_n is NULL) */
int hg_member_flags(const int32_t* values, const int32_t* d_n, int32_t cap, const int32_t* tag_of, int32_t tag,
                    uint8_t* flags, void* stream);
int64_t hg_filter_ws_size(int32_t n);
int hg_filter_tagged(const int32_t* list, int32_t n, const int32_t* tag_of, int32_t tag, int32_t* out,
                     int32_t* d_n_out, int32_t* ws, void* stream);

/* ---- evaluation (orchestrator.py:662-680) -------------------------------- */
int hg_full_aggregate(int32_t model, const float* hin, int32_t ld_in, int32_t F, const int64_t* offsets,
                      const int32_t* targets, int32_t V, const int32_t* outdeg, float* out, int32_t ld_out,
                      void* stream);
int hg_target_histogram(const int32_t* targets, int64_t E, int32_t* cnt, void* stream);
int hg_argmax_correct(const float* logits, int32_t ld, int32_t C, int32_t V, const int32_t* labels,
                      const uint8_t* mask, uint64_t* d_correct, void* stream);

/* ---- primitives ---------------------------------------------------------- */
int64_t hg_scan_ws_size(int64_t cap);
int hg_scan_exclusive(const int32_t* in, int32_t* out, const int32_t* d_n, int64_t cap, int32_t* d_total,
                      int32_t* ws, void* stream);
int64_t hg_radix_ws_size(int64_t n);
int hg_radix_sort_pairs(uint32_t* keys, int32_t* vals, uint32_t* k_alt, int32_t* v_alt, int64_t n,
                        int32_t key_bits, int32_t* ws, int32_t* host_out_in_alt, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* HG_GNN_H */
