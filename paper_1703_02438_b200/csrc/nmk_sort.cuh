// nmk_sort.cuh — host launchers of the 64-bit radix sort and prefix sums (k_sort.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace nmk {
// Stable ascending sort of n 64-bit keys (and, with vals_in, their values) into
// the outputs; the inputs are left untouched, outputs must not alias them.
size_t sort64_ws_bytes(uint64_t n, bool with_vals);
void sort64(const unsigned long long* keys_in, unsigned long long* keys_out, const unsigned long long* vals_in,
            unsigned long long* vals_out, uint64_t n, void* ws, cudaStream_t s);
// out[i] = sum(in[0..i)) (exclusive) or sum(in[0..i]) (inclusive); in-place allowed.
size_t scan64_ws_bytes(uint64_t n);
void scan64(const unsigned long long* in, unsigned long long* out, uint64_t n, bool inclusive, void* ws,
            cudaStream_t s);
}  // namespace nmk
