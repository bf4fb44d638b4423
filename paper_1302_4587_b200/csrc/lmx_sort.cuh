// lmx_sort.cuh -- radix sorts of the load path through CUB's double-buffer
// interface: the temporary storage is a few MB instead of another copy of
// the keys and values (the plain interface keeps its alternate buffers in
// the temporary storage), which is what sets the load's memory peak.
#pragma once
#include <cub/cub.cuh>

#include "lmx_internal.cuh"

// Sort (*ka, *va) by key bits [b0, b1).  On return *kb / *vb hold the sorted
// pairs and *ka / *va the scratch (the pointer pairs are swapped when the
// passes end in the input buffers); both pairs must be caller-owned buffers
// of the same size.
template <typename K, typename V>
int lmx_sort_pairs(lmx_ctx *ctx, K **ka, K **kb, V **va, V **vb, long long n, int b0, int b1, cudaStream_t st,
                   const char *what) {
    if (n <= 0) return LMX_OK;
    cub::DoubleBuffer<K> dk(*ka, *kb);
    cub::DoubleBuffer<V> dv(*va, *vb);
    size_t tb = 0;
    cudaError_t e = cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, n, b0, b1, st);
    if (e != cudaSuccess) return lmx_cuda_check(ctx, e, what);
    void *tmp = nullptr;
    LMX_TRY(lmx_alloc(ctx, &tmp, tb, what));
    e = cub::DeviceRadixSort::SortPairs(tmp, tb, dk, dv, n, b0, b1, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);   // the scratch block goes back to the cache
    lmx_free(ctx, &tmp, tb);
    if (e != cudaSuccess) return lmx_cuda_check(ctx, e, what);
    if (dk.Current() != *kb) std::swap(*ka, *kb);
    if (dv.Current() != *vb) std::swap(*va, *vb);
    return LMX_OK;
}
