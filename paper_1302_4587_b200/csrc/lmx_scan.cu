// lmx_scan.cu -- the weight-ordered round loop ("scan" algorithm) for the
// DISTINCT weight-key layout on one GPU.
//
// Same result as local_max_seq (matchers.py:61-122) and as the compacting
// round loop of lmx_round.cu, reached with O(m) total slot traffic instead of
// O(sum_r m_r + m):
//
//   * At load time every vertex segment of ids0 is sorted by weight rank,
//     descending (lmx_setup.cu).  With (almost) distinct weights the key order
//     of a vertex's edges is then fixed across rounds: only edges of one tied
//     weight need the per-round salt (tiebreak.py:55-80), and those sit next to
//     each other in the segment.
//   * ptr[v] marks the first slot of v not yet known to be dead.  Edges only
//     ever die (matchers.py:111), so v's candidate in round r is the first live
//     slot at or after ptr[v] (or the salt-max of its tie run): one probe for
//     most vertices, and each slot is skipped at most once over all rounds.
//   * The per-round statistics (edges_before, RoundStats of matchers.py:113-118)
//     come from the vertices matched in round r: every edge that dies in round
//     r has an endpoint in M_r, so m_{r+1} = m_r - |{e : e touches M_r}|,
//     counted by one scan of each matched vertex's remaining slots:
//     weight 2 for an unmatched neighbour, 1 for a neighbour also matched in
//     round r (that edge is seen from both sides), 0 for an older match.
//     Every vertex's slots are streamed once, when it is matched.
//
// Per round r, two kernels:
//   lmx_scan_round_kernel: removal count of M_{r-1} (block / warp / 8-lane /
//     thread per vertex by remaining length) and the candidate probe of every
//     active vertex A_r (thread per vertex);
//   lmx_scan_match_kernel: mutual candidates -> matched/fresh bits, mate, the
//     edge bit; appends M_r (bucketed by remaining length) and A_{r+1}.
// The vertex state word mf[v / 32] = {matched bits, fresh bits}: fresh marks
// M_r until the next match kernel clears it.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "lmx_internal.cuh"

#ifndef LMX_SCAN_MINB
#define LMX_SCAN_MINB 4
#endif

namespace lmx {

struct ScanArgs {
    const unsigned long long *vbeg;
    const uint32_t *deg0;
    uint32_t *ptr;              // first possibly-live slot of each vertex (segment offset)
    uint32_t *cand_nbr;
    uint32_t *cand_id;
    const uint2 *ids;           // ids0, weight-descending per segment
    const uint2 *mf;            // {matched, fresh} per 32 vertices
    const uint32_t *alist;      // A_r
    const uint32_t *mlist;      // M_{r-1}: kBuckets regions of capacity cap
    unsigned long long cap;
    RoundCtr *ctr;              // ctr[r]: pad[0] = |A_r|, n[q] = |M_{r-1} bucket q|
    uint64_t rs;                // round seed (tiebreak.py:40-52)
    uint32_t D;                 // distinct weight values; x >= D is a tied edge
    const uint32_t *tie_rank;
    const uint32_t *eid_of_x;
};

__device__ __forceinline__ bool mf_matched(const uint2 *mf, uint32_t u) {
    return (mf[u >> 5].x >> (u & 31)) & 1u;
}

// Removal weight of slot neighbour u for a vertex matched in the last round.
__device__ __forceinline__ uint32_t removal_weight(const uint2 *mf, uint32_t u) {
    const uint2 w = mf[u >> 5];
    const uint32_t s = u & 31;
    const uint32_t m = (w.x >> s) & 1u, f = (w.y >> s) & 1u;
    return m ? f : 2u;
}

// Removal count over [beg, beg + len) by a team of TEAM threads (t = rank in
// the team): unaligned head slot, 16-byte slot pairs, tail slot.
template <int TEAM>
__device__ __forceinline__ uint32_t team_removal(const ScanArgs &a, unsigned long long beg, uint32_t len, uint32_t t,
                                                 unsigned long long &reads) {
    uint32_t acc = 0;
    const uint32_t head = (uint32_t)(beg & 1ULL) < len ? (uint32_t)(beg & 1ULL) : len;
    if (head && t == 0) acc += removal_weight(a.mf, __ldcs(a.ids + beg).x);
    const uint32_t rest = len - head;
    const uint32_t npairs = rest >> 1;
    const uint4 *pp = reinterpret_cast<const uint4 *>(a.ids + beg + head);
    constexpr int U = 4;
    for (uint32_t c = t; c < npairs; c += TEAM * U) {
        uint4 q[U];
#pragma unroll
        for (int j = 0; j < U; ++j) {
            const uint32_t i = c + j * TEAM;
            q[j] = i < npairs ? __ldcs(pp + i) : make_uint4(kNone, 0, kNone, 0);
        }
#pragma unroll
        for (int j = 0; j < U; ++j)
            if (q[j].x != kNone) acc += removal_weight(a.mf, q[j].x) + removal_weight(a.mf, q[j].z);
    }
    if ((rest & 1u) && t == 0) acc += removal_weight(a.mf, __ldcs(a.ids + beg + len - 1).x);
    if (t == 0) reads += len;
    return acc;
}

// First live slot at or after p (p is left on it).  False when v has none.
template <bool FIRST>
__device__ __forceinline__ bool advance(const ScanArgs &a, unsigned long long b, uint32_t &p, uint32_t d,
                                        uint2 &out, unsigned long long &reads) {
    while (p < d) {
        const uint32_t cnt = min(4u, d - p);
        uint2 s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] = (uint32_t)j < cnt ? a.ids[b + p + j] : make_uint2(kNone, kNone);
        reads += cnt;
        uint32_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((uint32_t)j < cnt && (FIRST || !mf_matched(a.mf, s[j].x))) live |= 1u << j;
        if (live) {
            const int j0 = __ffs(live) - 1;
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (j == j0) out = s[j];
            p += (uint32_t)j0;
            return true;
        }
        p += cnt;
    }
    return false;
}

// `out` (at p) is live and tied: every live slot of its run of equal weight
// competes on the edge salt (tiebreak.py:55-80).
template <bool FIRST>
__device__ __forceinline__ void resolve_tie(const ScanArgs &a, unsigned long long b, uint32_t p, uint32_t d,
                                            uint2 &out, unsigned long long &reads) {
    const uint32_t r0 = __ldg(a.tie_rank + (out.y - a.D));
    uint64_t best = mix64((uint64_t)__ldg(a.eid_of_x + out.y) ^ a.rs);
    for (uint32_t q = p + 1; q < d; ++q) {
        const uint2 t = a.ids[b + q];
        ++reads;
        if (t.y < a.D || __ldg(a.tie_rank + (t.y - a.D)) != r0) break;
        if (!FIRST && mf_matched(a.mf, t.x)) continue;
        const uint64_t s = mix64((uint64_t)__ldg(a.eid_of_x + t.y) ^ a.rs);
        if (s > best) {
            best = s;
            out = t;
        }
    }
}

template <bool FIRST>
__global__ void __launch_bounds__(kBlock, LMX_SCAN_MINB) lmx_scan_round_kernel(ScanArgs a) {
    __shared__ uint32_t s_item;
    __shared__ unsigned long long s_red[2][kWarps];
    uint32_t nb[kBuckets];
    uint32_t any = 0;
#pragma unroll
    for (int q = 0; q < kBuckets; ++q) {
        nb[q] = FIRST ? 0u : a.ctr->n[q];
        any |= nb[q];
    }
    const uint32_t na = a.ctr->pad[0];
    if ((any | na) == 0) return;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long removed2 = 0, reads = 0;

    if (!FIRST) {
        // removal of M_{r-1}: buckets 4 and 3, one block per vertex
#pragma unroll 1
        for (int q = kBuckets - 1; q >= 3; --q) {
            for (;;) {
                if (tid == 0) s_item = atomicAdd(&a.ctr->cur[q], 1u);
                __syncthreads();
                const uint32_t i = s_item;
                __syncthreads();
                if (i >= nb[q]) break;
                const uint32_t v = a.mlist[(unsigned long long)q * a.cap + i];
                const uint32_t p = a.ptr[v];
                removed2 += team_removal<kBlock>(a, a.vbeg[v] + p, a.deg0[v] - p, tid, reads);
            }
        }
        // bucket 2: warp per vertex, 8 per grab
        for (;;) {
            uint32_t i0 = 0;
            if (lane == 0) i0 = atomicAdd(&a.ctr->cur[2], 8u);
            i0 = __shfl_sync(0xffffffffu, i0, 0);
            if (i0 >= nb[2]) break;
            unsigned long long mb = 0;
            uint32_t ml = 0;
            if (lane < 8 && i0 + lane < nb[2]) {
                const uint32_t v = a.mlist[2 * a.cap + i0 + lane];
                const uint32_t p = a.ptr[v];
                mb = a.vbeg[v] + p;
                ml = a.deg0[v] - p;
            }
            const uint32_t cnt = min(8u, nb[2] - i0);
            for (uint32_t k = 0; k < cnt; ++k) {
                const unsigned long long beg = __shfl_sync(0xffffffffu, mb, k);
                const uint32_t len = __shfl_sync(0xffffffffu, ml, k);
                removed2 += team_removal<32>(a, beg, len, lane, reads);
            }
        }
        // bucket 1: 8 lanes per vertex (<= 32 slots), 4 vertices per warp pass
        for (;;) {
            uint32_t i0 = 0;
            if (lane == 0) i0 = atomicAdd(&a.ctr->cur[1], 16u);
            i0 = __shfl_sync(0xffffffffu, i0, 0);
            if (i0 >= nb[1]) break;
            unsigned long long mb = 0;
            uint32_t ml = 0;
            if (lane < 16 && i0 + lane < nb[1]) {
                const uint32_t v = a.mlist[a.cap + i0 + lane];
                const uint32_t p = a.ptr[v];
                mb = a.vbeg[v] + p;
                ml = a.deg0[v] - p;
            }
#pragma unroll 1
            for (int it = 0; it < 4; ++it) {
                const int src = it * 4 + (lane >> 3);
                const unsigned long long beg = __shfl_sync(0xffffffffu, mb, src);
                const uint32_t len = __shfl_sync(0xffffffffu, ml, src);
                const uint32_t gl = lane & 7;
                uint32_t u[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t i = gl + 8 * j;
                    u[j] = i < len ? __ldcs(a.ids + beg + i).x : kNone;
                }
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (u[j] != kNone) removed2 += removal_weight(a.mf, u[j]);
                if (gl == 0) reads += len;
            }
        }
        // bucket 0: thread per vertex (<= 4 slots), 128 per grab
        for (;;) {
            uint32_t i0 = 0;
            if (lane == 0) i0 = atomicAdd(&a.ctr->cur[0], 128u);
            i0 = __shfl_sync(0xffffffffu, i0, 0);
            if (i0 >= nb[0]) break;
#pragma unroll 1
            for (int it = 0; it < 4; ++it) {
                const uint32_t i = i0 + it * 32 + lane;
                if (i >= nb[0]) continue;
                const uint32_t v = a.mlist[i];
                const uint32_t p = a.ptr[v];
                const unsigned long long beg = a.vbeg[v] + p;
                const uint32_t len = a.deg0[v] - p;
                uint32_t u[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) u[j] = (uint32_t)j < len ? __ldcs(a.ids + beg + j).x : kNone;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (u[j] != kNone) removed2 += removal_weight(a.mf, u[j]);
                reads += len;
            }
        }
    }

    // candidate probe of A_r: thread per vertex, 4 vertices per lane per grab
    for (;;) {
        uint32_t i0 = 0;
        if (lane == 0) i0 = atomicAdd(&a.ctr->pad[1], 128u);
        i0 = __shfl_sync(0xffffffffu, i0, 0);
        if (i0 >= na) break;
        uint32_t v[4], p[4], d[4];
        unsigned long long b[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t i = i0 + it * 32 + lane;
            v[it] = i < na ? a.alist[i] : kNone;
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            if (v[it] != kNone) {
                p[it] = FIRST ? 0u : a.ptr[v[it]];
                d[it] = a.deg0[v[it]];
                b[it] = a.vbeg[v[it]];
            } else {
                p[it] = d[it] = 0;
                b[it] = 0;
            }
        }
        // first probe of all four vertices at once (their chains overlap)
        uint2 s[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) s[it] = p[it] < d[it] ? a.ids[b[it] + p[it]] : make_uint2(kNone, kNone);
        bool live[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) live[it] = s[it].x != kNone && (FIRST || !mf_matched(a.mf, s[it].x));
        // fast path: the probed slot is live and of a unique weight
        uint32_t slow = 0;
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            if (v[it] == kNone) continue;
            reads += 1;
            if (live[it] && s[it].y < a.D) {
                a.cand_nbr[v[it]] = s[it].x;
                a.cand_id[v[it]] = s[it].y;
            } else {
                slow |= 1u << it;
            }
        }
        // slow path (dead probe or tied weight), one vertex at a time
        while (slow) {
            const int k = __ffs(slow) - 1;
            slow &= slow - 1;
            uint32_t vk = 0, pk = 0, dk = 0;
            unsigned long long bk = 0;
            uint2 c = make_uint2(kNone, kNone);
            bool found = false;
#pragma unroll
            for (int it = 0; it < 4; ++it) {
                if (it == k) {
                    vk = v[it];
                    pk = p[it];
                    dk = d[it];
                    bk = b[it];
                    c = s[it];
                    found = live[it];
                }
            }
            uint32_t pp = pk;
            if (!found && pk < dk) {
                pp = pk + 1;
                found = advance<FIRST>(a, bk, pp, dk, c, reads);
            }
            if (found && c.y >= a.D) resolve_tie<FIRST>(a, bk, pp, dk, c, reads);
            a.cand_nbr[vk] = found ? c.x : kNone;
            a.cand_id[vk] = found ? c.y : kNone;
            if (pp != pk) a.ptr[vk] = pp;
        }
    }

#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        removed2 += __shfl_xor_sync(0xffffffffu, removed2, off);
        reads += __shfl_xor_sync(0xffffffffu, reads, off);
    }
    const int warp = tid >> 5;
    if (lane == 0) {
        s_red[0][warp] = removed2;
        s_red[1][warp] = reads;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long t0 = 0, t1 = 0;
        for (int q = 0; q < kWarps; ++q) {
            t0 += s_red[0][q];
            t1 += s_red[1][q];
        }
        if (t0) atomicAdd(&a.ctr->live_slots, t0);
        if (t1) atomicAdd(&a.ctr->slot_reads, t1);
    }
}

struct ScanMatchArgs {
    const uint32_t *cand_nbr;
    const uint32_t *cand_id;
    const uint32_t *ptr;
    const uint32_t *deg0;
    uint32_t *mf;                 // uint2 words viewed as u32 pairs
    long long *mate;
    const uint32_t *oldid;
    const uint32_t *alist;        // A_r
    uint32_t *anext;              // A_{r+1}
    const uint32_t *mprev;        // M_{r-1} (fresh bits cleared here)
    uint32_t *mnext;              // M_r, kBuckets regions
    unsigned long long cap;
    uint32_t *ebits;
    const uint32_t *eid_of_x;
    RoundCtr *ctr;
    RoundCtr *ctr_next;
};

constexpr int kScanTargets = kBuckets + 1;   // M_r buckets, then A_{r+1}

__device__ __forceinline__ uint32_t lanemask_lt_u32() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__global__ void __launch_bounds__(kBlock, 8) lmx_scan_match_kernel(ScanMatchArgs a) {
    __shared__ uint32_t s_cnt[kScanTargets][kWarps];
    __shared__ uint32_t s_base[kScanTargets];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const unsigned long long gtid = (unsigned long long)blockIdx.x * kBlock + tid;
    const unsigned long long gstride = (unsigned long long)gridDim.x * kBlock;
    // fresh bits of M_{r-1} end here (disjoint from the M_r bits set below)
#pragma unroll 1
    for (int q = 0; q < kBuckets; ++q) {
        const uint32_t c = a.ctr->n[q];
        for (unsigned long long i = gtid; i < c; i += gstride) {
            const uint32_t v = a.mprev[(unsigned long long)q * a.cap + i];
            atomicAnd(a.mf + 2 * (v >> 5) + 1, ~(1u << (v & 31)));
        }
    }
    const uint32_t total = a.ctr->pad[0];
    if (total == 0) return;
    const uint32_t lt = lanemask_lt_u32();
    unsigned long long matched_v = 0;
    constexpr int kItems = 4;
    const uint32_t tile = kBlock * kItems;
    for (uint32_t t0 = blockIdx.x * tile; t0 < total; t0 += gridDim.x * tile) {
        uint32_t vv[kItems], kind[kItems];
        uint32_t wc[kScanTargets];
#pragma unroll
        for (int q = 0; q < kScanTargets; ++q) wc[q] = 0;
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t i = t0 + j * kBlock + tid;
            const uint32_t v = i < total ? a.alist[i] : kNone;
            uint32_t kd = kScanTargets;   // dropped
            if (v != kNone) {
                const uint32_t x = a.cand_nbr[v];
                if (x != kNone) {
                    const uint32_t id = a.cand_id[v];
                    if (a.cand_id[x] == id) {   // weight keys are unique per edge
                        atomicOr(a.mf + 2 * (v >> 5), 1u << (v & 31));
                        atomicOr(a.mf + 2 * (v >> 5) + 1, 1u << (v & 31));
                        if (a.oldid) a.mate[a.oldid[v]] = (long long)a.oldid[x];
                        else a.mate[v] = (long long)x;
                        ++matched_v;
                        if (v < x) {
                            const uint32_t e = a.eid_of_x[id];
                            atomicOr(a.ebits + (e >> 5), 1u << (e & 31));
                        }
                        kd = (uint32_t)bucket_of(a.deg0[v] - a.ptr[v]);
                    } else {
                        kd = kBuckets;   // stays active
                    }
                }
            }
            vv[j] = v;
            kind[j] = kd;
#pragma unroll
            for (int q = 0; q < kScanTargets; ++q) wc[q] += __popc(__ballot_sync(0xffffffffu, kd == (uint32_t)q));
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < kScanTargets; ++q) s_cnt[q][warp] = wc[q];
        }
        __syncthreads();
        if (tid < kScanTargets) {
            uint32_t sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += s_cnt[tid][w];
            uint32_t base = 0;
            if (sum) base = atomicAdd(tid < kBuckets ? &a.ctr_next->n[tid] : &a.ctr_next->pad[0], sum);
            s_base[tid] = base;
        }
        __syncthreads();
        uint32_t pos[kScanTargets];
#pragma unroll
        for (int q = 0; q < kScanTargets; ++q) {
            uint32_t p = s_base[q];
            for (int w = 0; w < warp; ++w) p += s_cnt[q][w];
            pos[q] = p;
        }
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
#pragma unroll
            for (int q = 0; q < kScanTargets; ++q) {
                const uint32_t bal = __ballot_sync(0xffffffffu, kind[j] == (uint32_t)q);
                if (kind[j] == (uint32_t)q) {
                    const uint32_t p = pos[q] + __popc(bal & lt);
                    if (q < kBuckets) a.mnext[(unsigned long long)q * a.cap + p] = vv[j];
                    else a.anext[p] = vv[j];
                }
                pos[q] += __popc(bal);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) matched_v += __shfl_xor_sync(0xffffffffu, matched_v, off);
    if (lane == 0 && matched_v) atomicAdd(&a.ctr->matched_v, matched_v);
}

}  // namespace lmx

using namespace lmx;

int lmx_scan_configure_grids(lmx_ctx *ctx) {
    int occ0 = 0, occ1 = 0, occm = 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, lmx_scan_round_kernel<true>, kBlock, 0));
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, lmx_scan_round_kernel<false>, kBlock, 0));
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occm, lmx_scan_match_kernel, kBlock, 0));
    ctx->scan_grid[0] = ctx->num_sms * std::max(occ0, 1);
    ctx->scan_grid[1] = ctx->num_sms * std::max(occ1, 1);
    ctx->scan_match_grid = ctx->num_sms * std::max(occm, 1);
    return LMX_OK;
}

int lmx_scan_alloc(lmx_ctx *ctx) {
    const size_t n = (size_t)std::max<int64_t>(ctx->n, 1);
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mf, ((n + 31) / 32) * 8, "matched/fresh"));
    for (int i = 0; i < 2; ++i) LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mlists[i], nl * 4 * kBuckets, "mlists"));
    return LMX_OK;
}

int lmx_run_rounds_scan(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                        std::vector<lmx_round_stats> &stats, unsigned long long &n_matched) {
    stats.clear();
    n_matched = 0;
    ctx->timing.round_launches = 0;
    ctx->timing.slot_reads = 0;
    ctx->timing.round_kernel_ms = 0;
    ctx->timing.match_kernel_ms = 0;
    const size_t n = (size_t)ctx->n;
    const size_t cap = (size_t)std::max<int64_t>(ctx->n_local, 1);
    cudaStream_t st = ctx->stream;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    LMX_TRY(lmx_ensure_ctr(ctx, 64));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ctr, 0, sizeof(RoundCtr) * (size_t)ctx->ctr_cap, st));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ebits, 0, ((size_t)std::max<int64_t>(ctx->m, 1) + 31) / 32 * 4, st));
    if (n) {
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mate_target, 0xFF, n * 8, st));   // -1
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mf, 0, (n + 31) / 32 * 8, st));
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->vdeg, 0, cap * 4, st));
    }
    ctx->ctr_host[0] = RoundCtr{};
    ctx->ctr_host[0].pad[0] = ctx->n_bins0[0];
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr, ctx->ctr_host, sizeof(RoundCtr), cudaMemcpyHostToDevice, st));

    int tl_used = 0;
    auto tl_mark = [&]() -> int {
        if (!ctx->kernel_timing) return LMX_OK;
        if (tl_used >= (int)ctx->tl_events.size()) {
            cudaEvent_t e;
            LMX_CUDA(ctx, cudaEventCreate(&e));
            ctx->tl_events.push_back(e);
        }
        LMX_CUDA(ctx, cudaEventRecord(ctx->tl_events[tl_used++], st));
        return LMX_OK;
    };
    LMX_TRY(tl_mark());

    uint32_t *cand_nbr = reinterpret_cast<uint32_t *>(ctx->cand);
    uint32_t *cand_id = cand_nbr + cap;
    std::vector<long long> live_m(1, (long long)ctx->m);   // m_r
    int r = 0, n_rounds = -1, batch = 6;
    while (n_rounds < 0 && ctx->m > 0) {
        LMX_TRY(lmx_ensure_ctr(ctx, r + batch + 1));
        const int r0 = r;
        for (int b = 0; b < batch; ++b, ++r) {
            const uint32_t *alist = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
            ScanArgs a;
            a.vbeg = ctx->vbeg;
            a.deg0 = ctx->deg0;
            a.ptr = ctx->vdeg;
            a.cand_nbr = cand_nbr;
            a.cand_id = cand_id;
            a.ids = ctx->ids0;
            a.mf = ctx->mf;
            a.alist = alist;
            a.mlist = ctx->mlists[(r + 1) & 1];   // M_{r-1}
            a.cap = cap;
            a.ctr = ctx->ctr + r;
            a.rs = round_seed(seed_masked, (uint64_t)r, rerandomize);
            a.D = ctx->n_distinct;
            a.tie_rank = ctx->tie_rank;
            a.eid_of_x = ctx->eid_of_x;
            if (r == 0) lmx_scan_round_kernel<true><<<ctx->scan_grid[0], kBlock, 0, st>>>(a);
            else lmx_scan_round_kernel<false><<<ctx->scan_grid[1], kBlock, 0, st>>>(a);
            LMX_CUDA(ctx, cudaGetLastError());
            LMX_TRY(tl_mark());
            ScanMatchArgs ma;
            ma.cand_nbr = cand_nbr;
            ma.cand_id = cand_id;
            ma.ptr = ctx->vdeg;
            ma.deg0 = ctx->deg0;
            ma.mf = reinterpret_cast<uint32_t *>(ctx->mf);
            ma.mate = ctx->mate_target;
            ma.oldid = ctx->relabeled ? ctx->oldid : nullptr;
            ma.alist = alist;
            ma.anext = ctx->lists[(r + 1) & 1];
            ma.mprev = ctx->mlists[(r + 1) & 1];
            ma.mnext = ctx->mlists[r & 1];
            ma.cap = cap;
            ma.ebits = ctx->ebits;
            ma.eid_of_x = ctx->eid_of_x;
            ma.ctr = ctx->ctr + r;
            ma.ctr_next = ctx->ctr + r + 1;
            lmx_scan_match_kernel<<<ctx->scan_match_grid, kBlock, 0, st>>>(ma);
            LMX_CUDA(ctx, cudaGetLastError());
            LMX_TRY(tl_mark());
            ctx->timing.round_launches += 2;
        }
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host + r0, ctx->ctr + r0, sizeof(RoundCtr) * (size_t)batch,
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        for (int i = std::max(r0, 1); i < r; ++i) {
            const unsigned long long rem2 = ctx->ctr_host[i].live_slots;
            if (rem2 & 1ULL) return lmx_fail(ctx, LMX_ECUDA, "internal: odd removal count");
            live_m.push_back(live_m.back() - (long long)(rem2 / 2));
            if (live_m.back() < 0) return lmx_fail(ctx, LMX_ECUDA, "internal: negative live edge count");
        }
        for (int i = r0; i < r; ++i) {
            if (live_m[(size_t)i] == 0) {
                n_rounds = i;
                break;
            }
        }
        batch = 4;
    }
    if (ctx->kernel_timing && tl_used > 1) {
        ctx->kernel_ms.clear();
        for (int i = 1; i < tl_used; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->tl_events[i - 1], ctx->tl_events[i]);
            ctx->kernel_ms.push_back(ms);
            if (i & 1) ctx->timing.round_kernel_ms += ms;
            else ctx->timing.match_kernel_ms += ms;
        }
    } else {
        ctx->kernel_ms.clear();
    }
    ctx->timing.rounds_executed = r;
    if (n_rounds < 0) n_rounds = 0;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
    unsigned long long total_matched_v = 0;
    for (int i = 0; i < n_rounds; ++i) {
        const RoundCtr &c = ctx->ctr_host[i];
        if (c.matched_v & 1ULL) return lmx_fail(ctx, LMX_ECUDA, "internal: odd matched-vertex count");
        lmx_round_stats s;
        s.edges_before = (int64_t)live_m[(size_t)i];
        s.edges_matched = (int64_t)(c.matched_v / 2);
        s.edges_removed = (int64_t)(live_m[(size_t)i] - live_m[(size_t)i + 1]);
        stats.push_back(s);
        total_matched_v += c.matched_v;
    }
    for (int i = 0; i < r; ++i) ctx->timing.slot_reads += (int64_t)ctx->ctr_host[i].slot_reads;
    n_matched = total_matched_v / 2;
    return LMX_OK;
}
