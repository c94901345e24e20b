// Internal (non-ABI) prototypes shared by the hg_gnn translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#define HG_ABI_VERSION 1

// int64 words of the per-batch parameter block (hg_train.cu BP_*; engine.BP_SIZE)
#define HG_BP_WORDS 8

size_t hg_scan_ws_ints(long long cap);
int hg_scan_launch(const int* in, int* out, const int* d_n, long long mult, long long cap, int* d_total,
                   int* ws, cudaStream_t s);
size_t hg_radix_ws_ints(long long n);
int hg_radix_sort_launch(uint32_t* keys, int* vals, uint32_t* k_alt, int* v_alt, long long n,
                         int key_bits, int* ws, int* out_in_alt, cudaStream_t s);

// warp-specialised TMA tensor-core GEMMs (hg_gemm_tma.cu)
int hg_tma_gemm_bn(int N);
void hg_tma_set_fwd_form(int v);
void hg_tma_set_pair(int v);
void hg_tma_set_dbg(int v);
void hg_tma_set_wg_tsa(int v);
int hg_gemm_tma_launch(const float* A1, int lda1, int K1, const float* A2, int lda2, int K2, const uint8_t* bimg,
                       float* C, int ldc, int N, const int* d_M, int M_cap, int act, cudaStream_t s);
int hg_wgrad_tma_chunks(int K, int n_src, int M_cap);
int hg_wgrad_tma_launch(const float* A1, int lda1, const float* A2, int lda2, int K, const float* G, int ldg, int N,
                        const int* d_M, int M_cap, float* out1, float* out2, float* ws, uint32_t lbo, uint32_t sbo,
                        cudaStream_t s);

// access-policy window of the persisting feature rows (hg_util.cu); false if unset
bool hg_l2_window_attr(cudaLaunchAttribute* a);

void hg_set_pdl(int v);

// wide-row bottom gather: TMA bulk-copy staging on/off (hg_aggregate.cu)
void hg_set_agg_bulk(int v);
