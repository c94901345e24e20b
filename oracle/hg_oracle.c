/*
 * ORACLE — test infrastructure only.
 *
 * Plain-C restatement of the two compiled (numba @njit) loops of the
 * reference's operator plug-in layer, hetgnn/kernels.py.  It is the checker
 * for the CUDA path and the CPU baseline in bench.py; nothing in the product
 * package links or calls it.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Parity pinned by tests/test_oracle_golden.py against fixtures produced by
 * the reference itself (tests/golden/make_golden.py).
 *
 * Build: oracle/Makefile  ->  oracle/libhg_oracle.so   (gcc -O2, single thread,
 * the same execution model as the reference's numba kernels, kernels.py:139-141)
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define GOLDEN 0x9E3779B97F4A7C15ULL /* kernels.py:21 */
#define MIX1 0xBF58476D1CE4E5B9ULL   /* kernels.py:22 */
#define MIX2 0x94D049BB133111EBULL   /* kernels.py:23 */
#define PHI 0x2545F4914F6CDD1DULL    /* kernels.py:24 */

/* splitmix64 finaliser — kernels.py:51-55 */
uint64_t oracle_mix64(uint64_t x) {
    x = (x ^ (x >> 30)) * MIX1;
    x = (x ^ (x >> 27)) * MIX2;
    return x ^ (x >> 31);
}

/* derive_seed — kernels.py:61-70 */
uint64_t oracle_derive_seed(uint64_t seed, const uint64_t *parts, int n_parts) {
    uint64_t st = oracle_mix64(seed + GOLDEN);
    for (int i = 0; i < n_parts; ++i) st = oracle_mix64((st + GOLDEN) ^ parts[i]);
    return st;
}

/* Per-dst emission counts and total — kernels.py:82-92. */
int64_t oracle_sample_counts(const int64_t *offsets, const int64_t *dst, int64_t n_dst,
                             int64_t fanout, int64_t *counts) {
    int64_t total = 0;
    for (int64_t i = 0; i < n_dst; ++i) {
        int64_t v = dst[i];
        int64_t deg = offsets[v + 1] - offsets[v];
        counts[i] = deg < fanout ? deg : fanout;
        total += counts[i];
    }
    return total;
}

/* _sample_layer — kernels.py:77-118 (stream base already mixed, as in
 * sample_layer kernels.py:147-158).  Outputs pre-sized by oracle_sample_counts. */
void oracle_sample_layer(const int64_t *offsets, const int64_t *targets, const int64_t *dst,
                         int64_t n_dst, int64_t fanout, uint64_t stream_seed,
                         int64_t *edge_dst, int64_t *edge_src) {
    uint64_t base = oracle_mix64(stream_seed + GOLDEN);
    int64_t pos = 0;
    int64_t *idx = NULL;
    int64_t idx_cap = 0;
    for (int64_t i = 0; i < n_dst; ++i) {
        int64_t v = dst[i];
        int64_t off = offsets[v];
        int64_t deg = offsets[v + 1] - off;
        if (deg <= fanout) {
            for (int64_t j = 0; j < deg; ++j) {
                edge_dst[pos + j] = i;
                edge_src[pos + j] = targets[off + j];
            }
            pos += deg;
        } else {
            uint64_t state = oracle_mix64(base ^ ((uint64_t)v * PHI));
            if (deg > idx_cap) {
                free(idx);
                idx_cap = deg;
                idx = (int64_t *)malloc(sizeof(int64_t) * (size_t)idx_cap);
            }
            for (int64_t j = 0; j < deg; ++j) idx[j] = j;
            for (int64_t j = 0; j < fanout; ++j) {
                state += GOLDEN;
                uint64_t r = oracle_mix64(state);
                int64_t pick = j + (int64_t)(r % (uint64_t)(deg - j));
                int64_t tmp = idx[j];
                idx[j] = idx[pick];
                idx[pick] = tmp;
                edge_dst[pos + j] = i;
                edge_src[pos + j] = targets[off + idx[j]];
            }
            pos += fanout;
        }
    }
    free(idx);
}

/* _segment_weighted_rows_loop — kernels.py:121-129: out[d] += w*rows[s] in
 * the given edge order (out must be zeroed by the caller). */
void oracle_segment_weighted_rows(const int64_t *edge_src, const int64_t *edge_dst,
                                  const double *w, int64_t n_edges, const double *rows,
                                  int64_t d, double *out) {
    for (int64_t e = 0; e < n_edges; ++e) {
        /* rows and out never overlap; restrict lets the compiler vectorise the
         * column loop like numba's LLVM does (per-element arithmetic unchanged) */
        const double *restrict r = rows + edge_src[e] * d;
        double *restrict o = out + edge_dst[e] * d;
        const double we = w[e];
        for (int64_t c = 0; c < d; ++c) o[c] += we * r[c];
    }
}
