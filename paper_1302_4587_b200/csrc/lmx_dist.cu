// lmx_dist.cu -- the reference's boundary-message accounting for the
// 1D-partitioned engine (bsp.py:29-41 RoundMessages, :148-170).
//
// bsp_local_max counts, per round r, (a) candidate records: one per (vertex x,
// receiving worker w != owner(x)) such that x has a live cut edge to a vertex
// of w, and (b) the surviving cut edges (status records = 2 per edge).  Both
// follow from the edges' death rounds: an edge is live in round r iff
// r <= death(e) = min(mround(u), mround(v)) (matchers.py:111).  So after the
// loop, with the match rounds of all vertices (all-gathered), each partition
// histograms, over its owned vertices x:
//   rec[D(x, s, w)]  with D = max death over the edges to worker w at which x
//                 is the edge_u (s = 0) or the edge_v (s = 1) end: bsp.py:152-154
//                 dedupes the two sides separately; a record is sent in every
//                 round r <= D
//   cut[death(e)] for each cut edge once (from its lower end)
// and the host turns the summed suffix sums into RoundMessages.
#include <algorithm>
#include <vector>

#include "lmx_internal.cuh"

using namespace lmx;

namespace lmx {

constexpr int kMaxP = 64;

__global__ void __launch_bounds__(kBlock) k_dist_messages(const unsigned long long *vbeg, const uint2 *ids,
                                                          unsigned long long nl, uint32_t lo, uint32_t nbr_mask,
                                                          const uint32_t *mround, const unsigned long long *bounds,
                                                          int p, int rank, uint32_t R, const uint32_t *side_bits,
                                                          unsigned long long *rec,
                                                          unsigned long long *cut) {
    __shared__ unsigned long long s_b[kMaxP + 1];
    __shared__ int s_D[kWarps][2 * kMaxP];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i <= p; i += kBlock) s_b[i] = bounds[i];
    __syncthreads();
    const unsigned long long gw = ((unsigned long long)blockIdx.x * kBlock + tid) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * kBlock) >> 5;
    for (unsigned long long v = gw; v < nl; v += nw) {
        for (int w = lane; w < 2 * p; w += 32) s_D[warp][w] = -1;
        __syncwarp();
        const uint32_t x = lo + (uint32_t)v;
        const uint32_t mx = mround[x];
        for (unsigned long long i = vbeg[v] + lane; i < vbeg[v + 1]; i += 32) {
            const uint2 sl = ids[i];
            const uint32_t y = sl.x & nbr_mask;
            int w = 0;
            while (w + 1 < p && y >= s_b[w + 1]) ++w;
            if (w == rank) continue;
            const uint32_t d = min(min(mx, mround[y]), R);
            const int side = (side_bits[i >> 5] >> (i & 31)) & 1u;   // x is the edge's u (0) or v (1) end
            atomicMax(&s_D[warp][side * p + w], (int)d);
            if (x < y) atomicAdd(cut + d, 1ULL);
        }
        __syncwarp();
        for (int w = lane; w < 2 * p; w += 32)
            if (s_D[warp][w] >= 0) atomicAdd(rec + s_D[warp][w], 1ULL);
        __syncwarp();
    }
}

}  // namespace lmx

extern "C" int lmx_dist_messages(lmx_ctx *ctx, int n_rounds, void **hist_dev) {
    if (!ctx || !hist_dev || n_rounds < 0) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (!ctx->mround || !ctx->vbeg || !ctx->slot_side)
        return lmx_fail(ctx, LMX_ESTATE, "no partitioned matching to account");
    if (ctx->dist_p > kMaxP) return lmx_fail(ctx, LMX_ELIMIT, "message accounting supports p <= 64");
    const size_t nb = (size_t)n_rounds + 1;
    const size_t need = 2 * nb;
    if (ctx->hist_cap < need) {
        lmx_free(ctx, (void **)&ctx->hist, (ctx->hist_cap + 1) * 8);
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->hist, (need + 1) * 8, "message histograms"));
        ctx->hist_cap = need;
    }
    cudaStream_t st = ctx->stream;
    unsigned long long *bdev = reinterpret_cast<unsigned long long *>(ctx->hist + need);   // p + 1 <= 65 words
    std::vector<unsigned long long> hb(ctx->bounds.begin(), ctx->bounds.end());
    unsigned long long *bounds = nullptr;
    LMX_TRY(lmx_alloc(ctx, (void **)&bounds, hb.size() * 8, "bounds"));
    LMX_CUDA(ctx, cudaMemcpyAsync(bounds, hb.data(), hb.size() * 8, cudaMemcpyHostToDevice, st));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->hist, 0, need * 8, st));
    (void)bdev;
    const unsigned long long nl = (unsigned long long)ctx->n_local;
    if (nl) {
        k_dist_messages<<<ctx->num_sms * 8, kBlock, 0, st>>>(
            ctx->vbeg, ctx->ids0, nl, (uint32_t)ctx->lo, ctx->algo == 1 ? kSlotNbr : 0xFFFFFFFFu, ctx->mround, bounds,
            ctx->dist_p, ctx->dist_rank, (uint32_t)n_rounds, ctx->slot_side, ctx->hist, ctx->hist + nb);
        LMX_CUDA(ctx, cudaGetLastError());
    }
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    lmx_free(ctx, (void **)&bounds, hb.size() * 8);
    *hist_dev = ctx->hist;
    return LMX_OK;
}
