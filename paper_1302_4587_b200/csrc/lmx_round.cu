// lmx_round.cu -- the local max round loop on sm_100a (K1..K4 of SURVEY.md §2.4).
//
// One round r of local_max_seq (matchers.py:87-119) is two kernels:
//
//   lmx_round_kernel<MODE>  (K3 of round r-1 fused with K1 of round r)
//     for every vertex v of this round's live lists: stream v's live slots,
//     drop those whose neighbour was matched in round r-1 (matchers.py:111),
//     compact the survivors to the front of v's segment (pram.py:248-272's
//     compaction, done per segment so no global scan is needed), and take the
//     lexicographic max of (weight rank, mix64(eid ^ rs_r)) over them
//     (matchers.py:93-103; the edge id never decides because mix64 is a
//     bijection, so distinct edges have distinct salts).
//       MODE 0 = round 0: no filter, no writes, identity vertex list
//       MODE 1 = round 1: filter ids0 -> ids1 (pristine copy stays intact)
//       MODE 2 = round >= 2: filter ids1 in place
//     Work mapping: hubs (live degree >= kHubMin) one block each, grabbed
//     dynamically first; the rest in warp chunks of 256 vertices, each vertex
//     thread-per-vertex (degree <= kThreadMax) or warp-per-vertex.
//
//   lmx_match_kernel  (K2 + K4)
//     v is matched iff cand[cand[v].nbr] is the same edge (matchers.py:105);
//     sets the matched bitmap and mate, emits the edge id once, and appends
//     every unmatched vertex with live edges to the next round's lists.
//
// The host enqueues rounds in batches without waiting; kernels of rounds past
// the end find empty lists and exit, so the loop syncs once per batch.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "lmx_internal.cuh"

namespace lmx {

struct Best {
    uint32_t wk;
    uint32_t nbr;   // kNone = no candidate
    uint32_t eid;
    uint64_t salt;
};

__device__ __forceinline__ void best_init(Best &b) {
    b.wk = 0;
    b.nbr = kNone;
    b.eid = kNone;
    b.salt = 0;
}

// Offer one live slot; the salt is only hashed when the weight rank can win.
__device__ __forceinline__ void best_offer(Best &b, uint32_t k, uint32_t eid, uint32_t nbr,
                                           uint64_t rs) {
    if (b.nbr == kNone || k >= b.wk) {
        uint64_t s = mix64((uint64_t)eid ^ rs);
        if (b.nbr == kNone || k > b.wk || s > b.salt) {
            b.wk = k;
            b.salt = s;
            b.nbr = nbr;
            b.eid = eid;
        }
    }
}

__device__ __forceinline__ void best_merge(Best &b, const Best &o) {
    if (o.nbr == kNone) return;
    if (b.nbr == kNone || o.wk > b.wk || (o.wk == b.wk && o.salt > b.salt)) b = o;
}

__device__ __forceinline__ Best best_shfl_xor(const Best &b, int off) {
    Best o;
    o.wk = __shfl_xor_sync(0xffffffffu, b.wk, off);
    o.nbr = __shfl_xor_sync(0xffffffffu, b.nbr, off);
    o.eid = __shfl_xor_sync(0xffffffffu, b.eid, off);
    o.salt = __shfl_xor_sync(0xffffffffu, (unsigned long long)b.salt, off);
    return o;
}

__device__ __forceinline__ void best_warp_reduce(Best &b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) best_merge(b, best_shfl_xor(b, off));
}

struct RoundArgs {
    const unsigned long long *vbeg;
    uint32_t *vdeg;
    uint2 *cand;
    const uint2 *src_ids;
    const uint32_t *src_wk;
    uint2 *dst_ids;
    uint32_t *dst_wk;
    const uint32_t *matched;
    const uint32_t *L;   // unused in MODE 0 (identity over [0, n))
    const uint32_t *H;
    RoundCtr *ctr;       // this round's counters
    uint64_t rs;         // round seed (tiebreak.py:40-52)
    uint32_t n;
};

template <int MODE>
__device__ __forceinline__ uint2 ld_slot(const uint2 *p) {
    if (MODE < 2) return __ldcs(p);   // pristine records: streamed, evict-first
    return *p;                        // in-place working copy
}
template <int MODE>
__device__ __forceinline__ uint32_t ld_wk(const uint32_t *p) {
    if (MODE < 2) return __ldcs(p);
    return *p;
}

__device__ __forceinline__ bool is_matched(const uint32_t *bits, uint32_t v) {
    return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- thread per vertex -------------------------------------------------
template <int MODE, bool WK>
__device__ __forceinline__ uint32_t thread_vertex(const RoundArgs &a, uint32_t v, uint32_t d,
                                                  Best &b) {
    const unsigned long long beg = a.vbeg[v];
    const uint2 *s = a.src_ids + beg;
    const uint32_t *sk = WK ? a.src_wk + beg : nullptr;
    uint2 *o = a.dst_ids + beg;
    uint32_t *ok = WK ? a.dst_wk + beg : nullptr;
    uint32_t w = 0;
    for (uint32_t i = 0; i < d; i += 4) {
        uint2 x[4];
        uint32_t k[4];
        bool alive[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (i + j < d) {
                x[j] = ld_slot<MODE>(s + i + j);
                k[j] = WK ? ld_wk<MODE>(sk + i + j) : 0u;
            } else {
                x[j] = make_uint2(kNone, kNone);
                k[j] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            alive[j] = (i + j < d) && (MODE == 0 || !is_matched(a.matched, x[j].x));
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (alive[j]) {
                if (MODE == 1 || (MODE == 2 && w != i + j)) {
                    o[w] = x[j];
                    if (WK) ok[w] = k[j];
                }
                ++w;
                best_offer(b, k[j], x[j].y, x[j].x, a.rs);
            }
        }
    }
    return w;
}

// ---- warp per vertex (v, d warp-uniform) ------------------------------
template <int MODE, bool WK>
__device__ __forceinline__ uint32_t warp_vertex(const RoundArgs &a, uint32_t v, uint32_t d,
                                                Best &b, int lane) {
    const unsigned long long beg = a.vbeg[v];
    const uint2 *s = a.src_ids + beg;
    const uint32_t *sk = WK ? a.src_wk + beg : nullptr;
    uint2 *o = a.dst_ids + beg;
    uint32_t *ok = WK ? a.dst_wk + beg : nullptr;
    const uint32_t lt = lanemask_lt();
    uint32_t w = 0;
    for (uint32_t c = 0; c < d; c += 128) {
        uint2 x[4];
        uint32_t k[4];
        bool alive[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = c + j * 32 + lane;
            if (i < d) {
                x[j] = ld_slot<MODE>(s + i);
                k[j] = WK ? ld_wk<MODE>(sk + i) : 0u;
            } else {
                x[j] = make_uint2(kNone, kNone);
                k[j] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            alive[j] = (c + j * 32 + lane < d) && (MODE == 0 || !is_matched(a.matched, x[j].x));
        if (MODE == 2) __syncwarp();   // every read of this chunk precedes its writes
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            if (MODE != 0) {
                const uint32_t bal = __ballot_sync(0xffffffffu, alive[j]);
                const uint32_t pos = w + __popc(bal & lt);
                if (alive[j] && (MODE == 1 || pos != c + j * 32 + lane)) {
                    o[pos] = x[j];
                    if (WK) ok[pos] = k[j];
                }
                w += __popc(bal);
            }
            if (alive[j]) best_offer(b, k[j], x[j].y, x[j].x, a.rs);
        }
    }
    if (MODE == 0) w = d;
    return w;
}

// ---- block per vertex (hubs) --------------------------------------------
template <int MODE, bool WK>
__device__ __forceinline__ uint32_t block_vertex(const RoundArgs &a, uint32_t v, uint32_t d,
                                                 Best &b, uint32_t (*s_cnt)[kWarps]) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long beg = a.vbeg[v];
    const uint2 *s = a.src_ids + beg;
    const uint32_t *sk = WK ? a.src_wk + beg : nullptr;
    uint2 *o = a.dst_ids + beg;
    uint32_t *ok = WK ? a.dst_wk + beg : nullptr;
    const uint32_t lt = lanemask_lt();
    uint32_t w = 0;
    for (uint32_t c = 0; c < d; c += 4 * kBlock) {
        uint2 x[4];
        uint32_t k[4];
        bool alive[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const uint32_t i = c + j * kBlock + tid;
            if (i < d) {
                x[j] = ld_slot<MODE>(s + i);
                k[j] = WK ? ld_wk<MODE>(sk + i) : 0u;
            } else {
                x[j] = make_uint2(kNone, kNone);
                k[j] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            alive[j] = (c + j * kBlock + tid < d) && (MODE == 0 || !is_matched(a.matched, x[j].x));
        if (MODE != 0) {
            uint32_t bal[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                bal[j] = __ballot_sync(0xffffffffu, alive[j]);
                if (lane == 0) s_cnt[j][warp] = __popc(bal[j]);
            }
            __syncthreads();   // counts visible; also orders all reads before writes
            uint32_t total = 0, before[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t acc = 0;
#pragma unroll
                for (int q = 0; q < kWarps; ++q) {
                    const uint32_t cq = s_cnt[j][q];
                    acc += (q < warp) ? cq : 0u;
                    total += cq;
                }
                before[j] = acc;   // within (j), warps before me
            }
            // prefix over j: survivors of earlier j blocks come first
            uint32_t jbase = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                uint32_t cj = 0;
#pragma unroll
                for (int q = 0; q < kWarps; ++q) cj += s_cnt[j][q];
                const uint32_t pos = w + jbase + before[j] + __popc(bal[j] & lt);
                if (alive[j] && (MODE == 1 || pos != c + j * kBlock + tid)) {
                    o[pos] = x[j];
                    if (WK) ok[pos] = k[j];
                }
                jbase += cj;
            }
            w += total;
            __syncthreads();   // s_cnt reuse
        }
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (alive[j]) best_offer(b, k[j], x[j].y, x[j].x, a.rs);
    }
    if (MODE == 0) w = d;
    return w;
}

template <int MODE, bool WK>
__global__ void __launch_bounds__(kBlock) lmx_round_kernel(RoundArgs a) {
    __shared__ uint32_t s_cnt[4][kWarps];
    __shared__ Best s_best[kWarps];
    __shared__ uint32_t s_item;
    __shared__ unsigned long long s_red[2][kWarps];

    const uint32_t nH = a.ctr->nH;
    const uint32_t nL = a.ctr->nL;
    if (nH == 0 && nL == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long live = 0, reads = 0;

    // phase 1: hubs, one block each, grabbed dynamically
    for (;;) {
        if (tid == 0) s_item = atomicAdd(&a.ctr->cur_hub, 1u);
        __syncthreads();
        const uint32_t i = s_item;
        __syncthreads();
        if (i >= nH) break;
        const uint32_t v = a.H[i];
        const uint32_t d = a.vdeg[v];
        Best b;
        best_init(b);
        const uint32_t w = block_vertex<MODE, WK>(a, v, d, b, s_cnt);
        best_warp_reduce(b);
        if (lane == 0) s_best[warp] = b;
        __syncthreads();
        if (tid == 0) {
            Best t = s_best[0];
            for (int q = 1; q < kWarps; ++q) best_merge(t, s_best[q]);
            if (MODE != 0) a.vdeg[v] = w;
            a.cand[v] = (w > 0) ? make_uint2(t.nbr, t.eid) : make_uint2(kNone, kNone);
            live += w;
            reads += d;
        }
        __syncthreads();
    }

    // phase 2: warp chunks of the vertex list
    for (;;) {
        uint32_t chunk = 0;
        if (lane == 0) chunk = atomicAdd(&a.ctr->cur_L, 1u);
        chunk = __shfl_sync(0xffffffffu, chunk, 0);
        const unsigned long long base = (unsigned long long)chunk * kWarpChunk;
        if (base >= nL) break;
#pragma unroll 1
        for (int jj = 0; jj < kLanesItems; ++jj) {
            const unsigned long long idx = base + (unsigned long long)jj * 32 + lane;
            uint32_t v = kNone, d = 0;
            if (idx < nL) {
                v = (MODE == 0) ? (uint32_t)idx : a.L[idx];
                d = a.vdeg[v];
                if (MODE == 0 && d >= kHubMin) d = 0;   // done in phase 1
            }
            if (d > 0 && d <= kThreadMax) {
                Best b;
                best_init(b);
                const uint32_t w = thread_vertex<MODE, WK>(a, v, d, b);
                if (MODE != 0) a.vdeg[v] = w;
                a.cand[v] = (w > 0) ? make_uint2(b.nbr, b.eid) : make_uint2(kNone, kNone);
                live += w;
                reads += d;
            }
            uint32_t big = __ballot_sync(0xffffffffu, d > kThreadMax);
            while (big) {
                const int src = __ffs(big) - 1;
                big &= big - 1;
                const uint32_t vv = __shfl_sync(0xffffffffu, v, src);
                const uint32_t dd = __shfl_sync(0xffffffffu, d, src);
                Best b;
                best_init(b);
                const uint32_t w = warp_vertex<MODE, WK>(a, vv, dd, b, lane);
                best_warp_reduce(b);
                if (lane == src) {
                    if (MODE != 0) a.vdeg[vv] = w;
                    a.cand[vv] = (w > 0) ? make_uint2(b.nbr, b.eid) : make_uint2(kNone, kNone);
                    live += w;
                    reads += dd;
                }
            }
        }
    }

    // block totals -> one atomic per block
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        live += __shfl_xor_sync(0xffffffffu, live, off);
        reads += __shfl_xor_sync(0xffffffffu, reads, off);
    }
    if (lane == 0) {
        s_red[0][warp] = live;
        s_red[1][warp] = reads;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long tl = 0, tr = 0;
        for (int q = 0; q < kWarps; ++q) {
            tl += s_red[0][q];
            tr += s_red[1][q];
        }
        if (tl) atomicAdd(&a.ctr->live_slots, tl);
        if (tr) atomicAdd(&a.ctr->slot_reads, tr);
    }
}

struct MatchArgs {
    const uint32_t *vdeg;
    const uint2 *cand;
    uint32_t *matched;
    long long *mate;
    const uint32_t *L;      // null = identity (round 0)
    const uint32_t *H;
    uint32_t *L_next;
    uint32_t *H_next;
    uint32_t *mids;
    unsigned long long *mcount;
    RoundCtr *ctr;          // this round
    RoundCtr *ctr_next;     // next round (list sizes)
};

constexpr int kMatchItems = 4;

__global__ void __launch_bounds__(kBlock) lmx_match_kernel(MatchArgs a) {
    __shared__ uint32_t s_cnt[3][kWarps];
    __shared__ unsigned long long s_base[3];
    const uint32_t nH = a.ctr->nH, nL = a.ctr->nL;
    const unsigned long long total = (unsigned long long)nH + nL;
    if (total == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    unsigned long long matched_v = 0;
    const unsigned long long tile = (unsigned long long)kBlock * kMatchItems;
    for (unsigned long long t0 = (unsigned long long)blockIdx.x * tile; t0 < total;
         t0 += (unsigned long long)gridDim.x * tile) {
        uint32_t vv[kMatchItems], kind[kMatchItems], eid[kMatchItems];
        uint32_t bal[kMatchItems][3];
        uint32_t wc[3] = {0, 0, 0};
#pragma unroll
        for (int j = 0; j < kMatchItems; ++j) {
            const unsigned long long i = t0 + (unsigned long long)j * kBlock + tid;
            uint32_t v = kNone, d = 0;
            if (i < total) {
                v = (i < nH) ? a.H[i] : (a.L ? a.L[i - nH] : (uint32_t)(i - nH));
                d = a.vdeg[v];
                // round 0 lists hubs twice (hub list + identity range): skip the second
                if (!a.L && i >= nH && d >= kHubMin) d = 0;
            }
            uint32_t kd = 3;   // 0 = L_next, 1 = H_next, 2 = matched (emit eid), 3 = none
            uint32_t e = 0;
            if (d > 0) {
                const uint2 c = a.cand[v];
                const uint2 cx = a.cand[c.x];
                if (cx.x == v && cx.y == c.y) {
                    atomicOr(a.matched + (v >> 5), 1u << (v & 31));
                    a.mate[v] = (long long)c.x;
                    ++matched_v;
                    if (v < c.x) {
                        kd = 2;
                        e = c.y;
                    }
                } else {
                    kd = (d >= kHubMin) ? 1u : 0u;
                }
            }
            vv[j] = v;
            kind[j] = kd;
            eid[j] = e;
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                bal[j][q] = __ballot_sync(0xffffffffu, kd == (uint32_t)q);
                wc[q] += __popc(bal[j][q]);
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < 3; ++q) s_cnt[q][warp] = wc[q];
        }
        __syncthreads();
        if (tid < 3) {
            uint32_t sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += s_cnt[tid][w];
            unsigned long long base = 0;
            if (sum) {
                if (tid == 0) base = atomicAdd(&a.ctr_next->nL, sum);
                else if (tid == 1) base = atomicAdd(&a.ctr_next->nH, sum);
                else base = atomicAdd(a.mcount, (unsigned long long)sum);
            }
            s_base[tid] = base;
        }
        __syncthreads();
        unsigned long long pos[3];
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            unsigned long long p = s_base[q];
            for (int w = 0; w < warp; ++w) p += s_cnt[q][w];
            pos[q] = p;
        }
#pragma unroll
        for (int j = 0; j < kMatchItems; ++j) {
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                if (kind[j] == (uint32_t)q) {
                    const unsigned long long p = pos[q] + __popc(bal[j][q] & lt);
                    if (q == 0) a.L_next[p] = vv[j];
                    else if (q == 1) a.H_next[p] = vv[j];
                    else a.mids[p] = eid[j];
                }
                pos[q] += __popc(bal[j][q]);
            }
        }
        __syncthreads();   // s_cnt / s_base reuse
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) matched_v += __shfl_xor_sync(0xffffffffu, matched_v, off);
    if (lane == 0 && matched_v) atomicAdd(&a.ctr->matched_v, matched_v);
}

// Per-match initialisation: live degrees, mates, matched bitmap.
__global__ void lmx_init_kernel(uint32_t n, const uint32_t *deg0, uint32_t *vdeg, long long *mate,
                                uint32_t *matched) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        vdeg[v] = deg0[v];
        mate[v] = -1;
        if ((v & 31) == 0) matched[v >> 5] = 0;
    }
}

__global__ void lmx_widen_kernel(const uint32_t *src, long long *dst, unsigned long long k) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride)
        dst[i] = src[i];
}

}  // namespace lmx

using namespace lmx;

template <int MODE>
static void launch_round(lmx_ctx *ctx, const RoundArgs &a) {
    if (ctx->has_wk)
        lmx_round_kernel<MODE, true><<<ctx->round_blocks, kBlock, 0, ctx->stream>>>(a);
    else
        lmx_round_kernel<MODE, false><<<ctx->round_blocks, kBlock, 0, ctx->stream>>>(a);
}

int lmx_alloc_match_state(lmx_ctx *ctx) {
    const size_t n = (size_t)std::max<int64_t>(ctx->n, 1);
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->vdeg, n * 4, "vdeg"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->cand, n * 8, "cand"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mate, n * 8, "mate"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->matched, ((n + 31) / 32) * 4, "matched"));
    for (int i = 0; i < 2; ++i) {
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->L[i], n * 4, "L"));
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->H[i], n * 4, "H"));
    }
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mids, (n / 2 + 1) * 4, "mids"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mids_sorted, (n / 2 + 1) * 4, "mids_sorted"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mcount, 8, "mcount"));
    size_t tmp = 0;
    LMX_CUDA(ctx, cub::DeviceRadixSort::SortKeys(nullptr, tmp, ctx->mids, ctx->mids_sorted,
                                                 (int)(n / 2 + 1)));
    ctx->sort_tmp_bytes = tmp + 256;
    LMX_TRY(lmx_alloc(ctx, &ctx->sort_tmp, ctx->sort_tmp_bytes, "sort_tmp"));
    return LMX_OK;
}

// Ensure ctr has room for rounds [0, need].  Only called with the stream idle.
static int ensure_ctr(lmx_ctx *ctx, int need) {
    if (need < ctx->ctr_cap) return LMX_OK;
    const int ncap = std::max(ctx->ctr_cap * 2, need + 64);
    RoundCtr *nc = nullptr, *nh = nullptr;
    LMX_CUDA(ctx, cudaMalloc(&nc, sizeof(RoundCtr) * (size_t)ncap));
    LMX_CUDA(ctx, cudaMemsetAsync(nc, 0, sizeof(RoundCtr) * (size_t)ncap, ctx->stream));
    LMX_CUDA(ctx, cudaMallocHost(&nh, sizeof(RoundCtr) * (size_t)ncap));
    if (ctx->ctr) {
        LMX_CUDA(ctx, cudaMemcpyAsync(nc, ctx->ctr, sizeof(RoundCtr) * (size_t)ctx->ctr_cap,
                                      cudaMemcpyDeviceToDevice, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        std::copy(ctx->ctr_host, ctx->ctr_host + ctx->ctr_cap, nh);
        cudaFree(ctx->ctr);
        cudaFreeHost(ctx->ctr_host);
    }
    ctx->ctr = nc;
    ctx->ctr_host = nh;
    ctx->ctr_cap = ncap;
    return LMX_OK;
}

// The round loop of local_max_seq (matchers.py:87-119) on the device.
// Leaves mate in ctx->mate, matched ids (unsorted) in ctx->mids.
int lmx_run_rounds(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                   std::vector<lmx_round_stats> &stats, unsigned long long &n_matched) {
    const uint32_t n = (uint32_t)ctx->n;
    stats.clear();
    n_matched = 0;
    ctx->timing.round_launches = 0;
    ctx->timing.slot_reads = 0;
    LMX_TRY(ensure_ctr(ctx, 64));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ctr, 0, sizeof(RoundCtr) * (size_t)ctx->ctr_cap, ctx->stream));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->mcount, 0, 8, ctx->stream));
    ctx->ctr_host[0] = RoundCtr{};
    ctx->ctr_host[0].nL = n;
    ctx->ctr_host[0].nH = ctx->n_hubs0;
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr, ctx->ctr_host, sizeof(RoundCtr), cudaMemcpyHostToDevice,
                                  ctx->stream));
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    // optional per-kernel timeline: tl[0] after init, then (after round r, after match r)
    int tl_used = 0;
    auto tl_mark = [&](void) -> int {
        if (!ctx->kernel_timing) return LMX_OK;
        if (tl_used >= (int)ctx->tl_events.size()) {
            cudaEvent_t e;
            LMX_CUDA(ctx, cudaEventCreate(&e));
            ctx->tl_events.push_back(e);
        }
        LMX_CUDA(ctx, cudaEventRecord(ctx->tl_events[tl_used++], ctx->stream));
        return LMX_OK;
    };
    ctx->timing.round_kernel_ms = 0;
    ctx->timing.match_kernel_ms = 0;
    if (n > 0) {
        lmx_init_kernel<<<ctx->num_sms * 8, kBlock, 0, ctx->stream>>>(n, ctx->deg0, ctx->vdeg,
                                                                     ctx->mate, ctx->matched);
        LMX_CUDA(ctx, cudaGetLastError());
        ctx->timing.round_launches += 1;
    }
    LMX_TRY(tl_mark());
    int r = 0;
    int n_rounds = -1;
    int batch = 6;
    while (n_rounds < 0 && ctx->m > 0) {
        LMX_TRY(ensure_ctr(ctx, r + batch + 1));
        const int r0 = r;
        for (int b = 0; b < batch; ++b, ++r) {
            const int mode = r == 0 ? 0 : (r == 1 ? 1 : 2);
            RoundArgs a;
            a.vbeg = ctx->vbeg;
            a.vdeg = ctx->vdeg;
            a.cand = ctx->cand;
            a.src_ids = mode < 2 ? ctx->ids0 : ctx->ids1;
            a.src_wk = mode < 2 ? ctx->wk0 : ctx->wk1;
            a.dst_ids = ctx->ids1;
            a.dst_wk = ctx->wk1;
            a.matched = ctx->matched;
            a.L = ctx->L[r & 1];
            a.H = r == 0 ? ctx->hubs0 : ctx->H[r & 1];
            a.ctr = ctx->ctr + r;
            a.rs = round_seed(seed_masked, (uint64_t)r, rerandomize);
            a.n = n;
            if (mode == 0) launch_round<0>(ctx, a);
            else if (mode == 1) launch_round<1>(ctx, a);
            else launch_round<2>(ctx, a);
            LMX_CUDA(ctx, cudaGetLastError());
            LMX_TRY(tl_mark());
            MatchArgs ma;
            ma.vdeg = ctx->vdeg;
            ma.cand = ctx->cand;
            ma.matched = ctx->matched;
            ma.mate = ctx->mate;
            ma.L = r == 0 ? nullptr : ctx->L[r & 1];
            ma.H = a.H;
            ma.L_next = ctx->L[(r + 1) & 1];
            ma.H_next = ctx->H[(r + 1) & 1];
            ma.mids = ctx->mids;
            ma.mcount = ctx->mcount;
            ma.ctr = ctx->ctr + r;
            ma.ctr_next = ctx->ctr + r + 1;
            lmx_match_kernel<<<ctx->match_blocks, kBlock, 0, ctx->stream>>>(ma);
            LMX_CUDA(ctx, cudaGetLastError());
            LMX_TRY(tl_mark());
            ctx->timing.round_launches += 2;
        }
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host + r0, ctx->ctr + r0, sizeof(RoundCtr) * (size_t)batch,
                                      cudaMemcpyDeviceToHost, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        for (int i = r0; i < r; ++i) {
            if (ctx->ctr_host[i].live_slots == 0) {
                n_rounds = i;
                break;
            }
        }
        batch = 4;
    }
    if (ctx->kernel_timing && tl_used > 1) {
        for (int i = 1; i < tl_used; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->tl_events[i - 1], ctx->tl_events[i]);
            if (i & 1) ctx->timing.round_kernel_ms += ms;
            else ctx->timing.match_kernel_ms += ms;
        }
    }
    ctx->timing.rounds_executed = r;
    if (n_rounds < 0) n_rounds = 0;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    unsigned long long total_matched_v = 0;
    for (int i = 0; i < n_rounds; ++i) {
        const RoundCtr &c = ctx->ctr_host[i];
        if ((c.live_slots & 1ULL) || (c.matched_v & 1ULL))
            return lmx_fail(ctx, LMX_ECUDA, "internal: odd slot or matched-vertex count");
        lmx_round_stats s;
        s.edges_before = (int64_t)(c.live_slots / 2);
        s.edges_matched = (int64_t)(c.matched_v / 2);
        const unsigned long long nxt = (i + 1 < n_rounds) ? ctx->ctr_host[i + 1].live_slots / 2 : 0;
        s.edges_removed = s.edges_before - (int64_t)nxt;
        stats.push_back(s);
        total_matched_v += c.matched_v;
        ctx->timing.slot_reads += (int64_t)c.slot_reads;
    }
    n_matched = total_matched_v / 2;
    return LMX_OK;
}

// Sort the matched edge ids (K5) and copy mate / ids out.
int lmx_emit_outputs(lmx_ctx *ctx, unsigned long long n_matched, int64_t *mate_out,
                     int64_t *ids_out, int out_where) {
    const size_t n = (size_t)ctx->n;
    if (n_matched > 0) {
        size_t tmp = ctx->sort_tmp_bytes;
        LMX_CUDA(ctx, cub::DeviceRadixSort::SortKeys(ctx->sort_tmp, tmp, ctx->mids, ctx->mids_sorted,
                                                     (int)n_matched, 0, 32, ctx->stream));
    }
    if (out_where == LMX_DEVICE) {
        if (mate_out && n)
            LMX_CUDA(ctx, cudaMemcpyAsync(mate_out, ctx->mate, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        if (ids_out && n_matched) {
            lmx_widen_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(
                ctx->mids_sorted, (long long *)ids_out, n_matched);
            LMX_CUDA(ctx, cudaGetLastError());
            ctx->timing.round_launches += 1;
        }
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev2, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    } else {
        if (mate_out && n)
            LMX_CUDA(ctx, cudaMemcpyAsync(mate_out, ctx->mate, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
        std::vector<uint32_t> tmp32((size_t)n_matched);
        if (ids_out && n_matched)
            LMX_CUDA(ctx, cudaMemcpyAsync(tmp32.data(), ctx->mids_sorted, (size_t)n_matched * 4,
                                          cudaMemcpyDeviceToHost, ctx->stream));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev2, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
        if (ids_out)
            for (size_t i = 0; i < (size_t)n_matched; ++i) ids_out[i] = (int64_t)tmp32[i];
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.rounds_ms = ms;
    cudaEventElapsedTime(&ms, ctx->ev1, ctx->ev2);
    ctx->timing.output_ms = ms;
    return LMX_OK;
}

// Persistent grid sizes: every resident block slot of the device.
int lmx_configure_grids(lmx_ctx *ctx) {
    int occ = 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lmx_round_kernel<2, true>, kBlock, 0));
    ctx->round_blocks = ctx->num_sms * std::max(occ, 1);
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lmx_match_kernel, kBlock, 0));
    ctx->match_blocks = ctx->num_sms * std::max(occ, 1);
    return LMX_OK;
}
