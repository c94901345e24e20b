// Internal (non-ABI) prototypes shared by the hg_gnn translation units.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#define HG_ABI_VERSION 1

size_t hg_scan_ws_ints(long long cap);
int hg_scan_launch(const int* in, int* out, const int* d_n, long long mult, long long cap, int* d_total,
                   int* ws, cudaStream_t s);
size_t hg_radix_ws_ints(long long n);
int hg_radix_sort_launch(uint32_t* keys, int* vals, uint32_t* k_alt, int* v_alt, long long n,
                         int key_bits, int* ws, int* out_in_alt, cudaStream_t s);
