// lmx_pram.cu -- the PRAM restatement's cross pointers and exclusive-write
// check on the device (pram.py:28-51 WriteLog, :54-124 PramState layout,
// :127-166 compute_cross_pointers, Lemma 2 of PAPER.md:233-257).
//
// The reference's incidence layout (graph.py:108-115: slots sorted by
// (vertex, edge id), caller ids) is rebuilt by a stable radix sort of the
// edge-ordered slot stream by vertex.  The cross pointer of every slot (the
// other slot of its edge) is then computed by the reference's two write/read
// step pairs through a per-edge scratch cell: the min-id endpoint's slots
// write their index, the max-id endpoint's slots read it, then the roles
// swap.  Every step counts its writes and, with a per-cell counter, the
// writes that hit a cell already written in the same step (WriteLog.record's
// conflict rule).  Then the layout is checked as PramState.check_consistent
// does: cross is an involution, stays on its edge, switches endpoints.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "lmx_internal.cuh"

using namespace lmx;

namespace lmx {

__global__ void k_pram_stream(const uint32_t *eu, const uint32_t *ev, unsigned long long m, uint32_t *sv,
                              uint32_t *se) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        sv[2 * e] = eu[e];
        se[2 * e] = (uint32_t)e;
        sv[2 * e + 1] = ev[e];
        se[2 * e + 1] = (uint32_t)e;
    }
}

// One write step: every slot of the given side writes its index into its
// edge's scratch cell (write) or reads the cell into its cross pointer (read).
// stats: [0] writes, [1] conflicts.  cnt: per-cell write counters of this step.
template <bool WRITE>
__global__ void k_pram_step(const uint32_t *sv, const uint32_t *se, unsigned long long S, const uint32_t *eu,
                            const uint32_t *ev, bool min_side, uint32_t *scratch, uint32_t *cross, uint32_t *cnt,
                            unsigned long long *stats) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long writes = 0, conflicts = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += stride) {
        const uint32_t e = se[i];
        const uint32_t lo = min(eu[e], ev[e]);
        if ((sv[i] == lo) != min_side) continue;
        const unsigned long long cell = WRITE ? e : i;   // edge.scratch / slot.cross
        if (atomicAdd(cnt + cell, 1u) != 0u) ++conflicts;
        ++writes;
        if (WRITE) scratch[e] = (uint32_t)i;
        else cross[i] = scratch[e];
    }
    for (int off = 16; off > 0; off >>= 1) {
        writes += __shfl_xor_sync(0xffffffffu, writes, off);
        conflicts += __shfl_xor_sync(0xffffffffu, conflicts, off);
    }
    if ((threadIdx.x & 31) == 0) {
        if (writes) atomicAdd(stats, writes);
        if (conflicts) atomicAdd(stats + 1, conflicts);
    }
}

// PramState.check_consistent on the cross pointers (pram.py:115-124).
__global__ void k_pram_check(const uint32_t *sv, const uint32_t *se, const uint32_t *cross, unsigned long long S,
                             unsigned long long *bad) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < S; i += stride) {
        const uint32_t c = cross[i];
        const bool ok = c < S && cross[c] == (uint32_t)i && se[c] == se[i] && sv[c] != sv[i];
        if (!ok) atomicMin(bad, i);
    }
}

}  // namespace lmx

static int pgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    return (int)std::max<unsigned long long>(1, std::min(b, cap));
}

extern "C" int lmx_pram_cross(lmx_ctx *ctx, int64_t *cross_out, int64_t *log_out, int out_where) {
    if (!ctx || !log_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (ctx->dist_local) return lmx_fail(ctx, LMX_ESTATE, "cross pointers need the whole graph (not a partition)");
    if (!ctx->eu && ctx->m) return lmx_fail(ctx, LMX_ESTATE, "no graph loaded");
    cudaStream_t st = ctx->stream;
    const unsigned long long n = (unsigned long long)ctx->n, m = (unsigned long long)ctx->m, S = 2 * m;
    const size_t S1 = std::max<unsigned long long>(S, 1), m1 = std::max<unsigned long long>(m, 1);
    uint32_t *sv = nullptr, *se = nullptr, *sv2 = nullptr, *se2 = nullptr, *scratch = nullptr, *cross = nullptr,
             *cnt = nullptr;
    unsigned long long *stats = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    unsigned long long h[4] = {0, 0, ~0ULL, 0};   // writes, conflicts, first bad slot
    int steps = 0;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&sv, S1 * 4, "pram slot vertex")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&se, S1 * 4, "pram slot edge")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&sv2, S1 * 4, "pram slot vertex2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&se2, S1 * 4, "pram slot edge2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&scratch, m1 * 4, "pram scratch")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cross, S1 * 4, "pram cross")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cnt, S1 * 4, "pram write counters")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&stats, 32, "pram stats")) != LMX_OK) break;
        e = cudaMemcpyAsync(stats, h, 32, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess || m == 0) break;
        // graph.py:108-115 layout: stable sort of the edge-ordered slots by vertex
        k_pram_stream<<<pgrid(ctx, m), kBlock, 0, st>>>(ctx->eu, ctx->ev, m, sv, se);
        int bits = 1;
        while (bits < 32 && (1ULL << bits) < n) ++bits;
        e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, sv, sv2, se, se2, (long long)S, 0, bits, st);
        if (e != cudaSuccess) break;
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "pram sort tmp")) != LMX_OK) break;
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, sv, sv2, se, se2, (long long)S, 0, bits, st);
        if (e != cudaSuccess) break;
        // pram.py:150-165: min writes, max reads, max writes, min reads
        const bool sides[4] = {true, false, false, true};
        for (int k = 0; k < 4 && e == cudaSuccess; ++k) {
            e = cudaMemsetAsync(cnt, 0, S1 * 4, st);
            if (e != cudaSuccess) break;
            if (k == 0 || k == 2)
                k_pram_step<true><<<pgrid(ctx, S), kBlock, 0, st>>>(sv2, se2, S, ctx->eu, ctx->ev, sides[k], scratch,
                                                                   cross, cnt, stats);
            else
                k_pram_step<false><<<pgrid(ctx, S), kBlock, 0, st>>>(sv2, se2, S, ctx->eu, ctx->ev, sides[k],
                                                                    scratch, cross, cnt, stats);
            e = cudaGetLastError();
            ++steps;
        }
        if (e != cudaSuccess) break;
        k_pram_check<<<pgrid(ctx, S), kBlock, 0, st>>>(sv2, se2, cross, S, stats + 2);
        e = cudaGetLastError();
        if (e == cudaSuccess && cross_out) {
            // int64 cross pointers for the caller (device: via the counters' buffer)
            if (out_where == LMX_DEVICE) {
                e = cudaMemsetAsync(cross_out, 0, S * 8, st);
                if (e == cudaSuccess) e = cudaMemcpy2DAsync(cross_out, 8, cross, 4, 4, S, cudaMemcpyDeviceToDevice, st);
            } else {
                std::vector<uint32_t> hc(S);
                e = cudaMemcpyAsync(hc.data(), cross, S * 4, cudaMemcpyDeviceToHost, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                for (unsigned long long i = 0; i < S && e == cudaSuccess; ++i) cross_out[i] = (int64_t)hc[i];
            }
        }
    } while (0);
    if (e == cudaSuccess && rc == LMX_OK) e = cudaMemcpyAsync(h, stats, 32, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&sv, S1 * 4);
    lmx_free(ctx, (void **)&se, S1 * 4);
    lmx_free(ctx, (void **)&sv2, S1 * 4);
    lmx_free(ctx, (void **)&se2, S1 * 4);
    lmx_free(ctx, (void **)&scratch, m1 * 4);
    lmx_free(ctx, (void **)&cross, S1 * 4);
    lmx_free(ctx, (void **)&cnt, S1 * 4);
    lmx_free(ctx, (void **)&stats, 32);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, e);
    log_out[0] = steps;
    log_out[1] = (int64_t)h[0];
    log_out[2] = (int64_t)h[1];
    log_out[3] = h[2] == ~0ULL ? -1 : (int64_t)h[2];   // first slot failing check_consistent
    return LMX_OK;
}
