// lmx_round.cu -- the local max round loop on sm_100a (K1..K4 of SURVEY.md §2.4).
//
// One round r of local_max_seq (matchers.py:87-119) is two kernels:
//
//   lmx_round_kernel<MODE, LAYOUT>  (K3 of round r-1 fused with K1 of round r)
//     for every vertex v of this round's live lists: stream v's live slots,
//     drop those whose neighbour was matched in round r-1 (matchers.py:111),
//     compact the survivors to the front of v's segment (pram.py:248-272's
//     compaction, done per segment so no global scan is needed), and take the
//     lexicographic max of (weight, mix64(eid ^ rs_r)) over them
//     (matchers.py:93-103; the edge id never decides because mix64 is a
//     bijection, so distinct edges have distinct salts).
//       MODE 0 = round 0: no filter, no writes
//       MODE 1 = round 1: filter ids0 -> ids1 (the pristine copy stays intact)
//       MODE 2 = round >= 2: filter ids1 in place
//     Work mapping by live-degree bucket (lmx_internal.cuh): hubs one block
//     each (largest bucket first), then warp-, 8-lane-group- and
//     thread-per-vertex, every unit grabbed dynamically so no warp owns more
//     than a few thousand slots of work.
//
//   lmx_match_kernel  (K2 + K4)
//     v is matched iff cand[cand[v].nbr] is the same edge (matchers.py:105);
//     sets the matched bitmap and mate, emits the edge once, and appends every
//     unmatched vertex with live edges to the next round's bucket lists.
//
// The host enqueues rounds in batches without waiting; kernels of rounds past
// the end find empty lists and exit, so the loop syncs once per batch.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "lmx_internal.cuh"

// Tuning (measured on RMAT-26, profiles/): full occupancy beats per-thread
// memory-level parallelism for this latency-chained workload.
#ifndef LMX_MINB
#define LMX_MINB 8
#endif

namespace lmx {

struct Best {
    uint32_t hi;    // weight key (rank), 0 for UNIFORM
    uint32_t nbr;   // kNone = no candidate
    uint32_t id;
    uint64_t salt;
};

__device__ __forceinline__ void best_init(Best &b) {
    b.hi = 0;
    b.nbr = kNone;
    b.id = kNone;
    b.salt = 0;
}

__device__ __forceinline__ void best_merge(Best &b, const Best &o) {
    if (o.nbr == kNone) return;
    if (b.nbr == kNone || o.hi > b.hi || (o.hi == b.hi && o.salt > b.salt)) b = o;
}

__device__ __forceinline__ Best best_shfl_xor(const Best &b, int off) {
    Best o;
    o.hi = __shfl_xor_sync(0xffffffffu, b.hi, off);
    o.nbr = __shfl_xor_sync(0xffffffffu, b.nbr, off);
    o.id = __shfl_xor_sync(0xffffffffu, b.id, off);
    o.salt = __shfl_xor_sync(0xffffffffu, (unsigned long long)b.salt, off);
    return o;
}

template <int G>
__device__ __forceinline__ void best_group_reduce(Best &b) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) best_merge(b, best_shfl_xor(b, off));
}

struct RoundArgs {
    const unsigned long long *vbeg;
    uint32_t *vdeg;
    uint32_t *cand_nbr;   // candidate edge of v: neighbour ...
    uint32_t *cand_id;    // ... and edge id / weight key (split: the match kernel's
                          // random read of the partner touches only cand_id)
    const uint2 *ids0;
    const uint32_t *wk0;
    uint2 *ids1;
    uint32_t *wk1;
    const uint32_t *matched;
    const uint32_t *list[kBuckets];
    RoundCtr *ctr;             // this round's counters
    uint64_t rs;               // round seed (tiebreak.py:40-52)
    uint32_t n_distinct;       // DISTINCT layout: D
    const uint32_t *tie_rank;  // DISTINCT layout
    const uint32_t *eid_of_x;  // DISTINCT layout
    int round;
};

#ifdef LMX_PHASE_TIMING   // profiling builds only: warp-cycles spent in each phase per round
__device__ unsigned long long g_phase_cycles[64][5];
#define PHASE_MARK(k)                                                                       \
    do {                                                                                    \
        const long long _t = clock64();                                                     \
        if ((threadIdx.x & 31) == 0 && a.round < 64)                                        \
            atomicAdd(&g_phase_cycles[a.round][k], (unsigned long long)(_t - phase_t0));    \
        phase_t0 = _t;                                                                      \
    } while (0)
#else
#define PHASE_MARK(k) \
    do {              \
    } while (0)
#endif

// Offer one live slot {nbr, id} (+ weight rank k for GENERAL) to the running max.
template <int L>
__device__ __forceinline__ void offer(Best &b, uint32_t nbr, uint32_t id, uint32_t k, const RoundArgs &a) {
    if (L == kUniform) {
        const uint64_t s = mix64((uint64_t)id ^ a.rs);
        if (b.nbr == kNone || s > b.salt) {
            b.salt = s;
            b.nbr = nbr;
            b.id = id;
        }
    } else if (L == kGeneral) {
        if (b.nbr == kNone || k >= b.hi) {   // hash only when the weight can win
            const uint64_t s = mix64((uint64_t)id ^ a.rs);
            if (b.nbr == kNone || k > b.hi || s > b.salt) {
                b.hi = k;
                b.salt = s;
                b.nbr = nbr;
                b.id = id;
            }
        }
    } else {   // DISTINCT: id is the weight key x
        if (id < a.n_distinct) {   // unique weight: rank decides alone
            if (b.nbr == kNone || id > b.hi) {
                b.hi = id;
                b.salt = 0;
                b.nbr = nbr;
                b.id = id;
            }
        } else {                   // tied weight: rank, then salt of the edge id
            const uint32_t r = __ldg(a.tie_rank + (id - a.n_distinct));
            if (b.nbr == kNone || r >= b.hi) {
                const uint64_t s = mix64((uint64_t)__ldg(a.eid_of_x + id) ^ a.rs);
                if (b.nbr == kNone || r > b.hi || s > b.salt) {
                    b.hi = r;
                    b.salt = s;
                    b.nbr = nbr;
                    b.id = id;
                }
            }
        }
    }
}

template <int MODE, int L>
__device__ __forceinline__ void load_slot(const RoundArgs &a, unsigned long long p, uint2 &x, uint32_t &k) {
    if (MODE < 2) {
        x = __ldcs(a.ids0 + p);   // pristine records: streamed once, evict-first
        k = (L == kGeneral) ? __ldcs(a.wk0 + p) : 0u;
    } else {
        x = a.ids1[p];            // working copy, compacted in place
        k = (L == kGeneral) ? a.wk1[p] : 0u;
    }
}

template <int L>
__device__ __forceinline__ void store_slot(const RoundArgs &a, unsigned long long p, uint2 x, uint32_t k) {
    a.ids1[p] = x;
    if (L == kGeneral) a.wk1[p] = k;
}

__device__ __forceinline__ bool is_matched(const uint32_t *bits, uint32_t v) {
    return (__ldg(bits + (v >> 5)) >> (v & 31)) & 1u;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---- G lanes per vertex (G in {1, 8, 32}); every lane of the warp calls it.
// For G < 32 a single pass covers d <= G * ITEMS; for G == 32 (v, d) are
// warp-uniform and the loop runs ceil(d / (32 * ITEMS)) passes.
template <int MODE, int L, int G, int ITEMS>
__device__ __forceinline__ uint32_t group_vertex(const RoundArgs &a, unsigned long long beg, uint32_t d,
                                                 int lane, Best &b) {
    const int gl = lane & (G - 1);
    const uint32_t gmask = (G == 32) ? 0xffffffffu : (((1u << G) - 1u) << (lane & ~(G - 1)));
    const uint32_t lt = lanemask_lt() & gmask;
    const uint32_t span = G * ITEMS;
    const uint32_t npass = (G == 32) ? (d + span - 1) / span : 1u;
    uint32_t w = 0;
    for (uint32_t pass = 0; pass < npass; ++pass) {
        const uint32_t c = pass * span;
        uint2 x[ITEMS];
        uint32_t k[ITEMS];
        bool alive[ITEMS];
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            const uint32_t i = c + j * G + gl;
            if (i < d) {
                load_slot<MODE, L>(a, beg + i, x[j], k[j]);
            } else {
                x[j] = make_uint2(kNone, kNone);
                k[j] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < ITEMS; ++j)
            alive[j] = (c + j * G + gl < d) && (MODE == 0 || !is_matched(a.matched, x[j].x));
        if (MODE == 2) __syncwarp();   // every read of this pass precedes its writes
#pragma unroll
        for (int j = 0; j < ITEMS; ++j) {
            if (MODE != 0) {
                const uint32_t bal = __ballot_sync(0xffffffffu, alive[j]) & gmask;
                const uint32_t pos = w + __popc(bal & lt);
                if (alive[j] && (MODE == 1 || pos != c + j * G + gl)) store_slot<L>(a, beg + pos, x[j], k[j]);
                w += __popc(bal);
            }
            if (alive[j]) offer<L>(b, x[j].x, x[j].y, k[j], a);
        }
    }
    best_group_reduce<G>(b);
    return MODE == 0 ? d : w;
}

// ---- vectorised team paths (a warp or a whole block per vertex) ------------
// The segment [beg, beg + d) is split into an unaligned head slot, 16-byte
// aligned slot pairs loaded as uint4, and a tail slot.  Survivors are
// compacted in item order (any order inside a segment is valid: the key order
// is total); every read of a pass precedes its writes, and writes only land
// below the slots already read, so in-place compaction is race-free.
#ifndef LMX_PAIRS
#define LMX_PAIRS 2
#endif
constexpr int kPairs = LMX_PAIRS;         // uint4 pairs per thread per pass
constexpr int kBlockItems = 2 * kPairs;   // slot items per thread per pass

template <int MODE, int L>
__device__ __forceinline__ void load_pair(const RoundArgs &a, unsigned long long p, uint2 &x0, uint2 &x1,
                                          uint32_t &k0, uint32_t &k1) {
    uint4 q;
    if (MODE < 2) q = __ldcs(reinterpret_cast<const uint4 *>(a.ids0 + p));
    else q = *reinterpret_cast<const uint4 *>(a.ids1 + p);
    x0 = make_uint2(q.x, q.y);
    x1 = make_uint2(q.z, q.w);
    if (L == kGeneral) {
        uint2 kk;
        if (MODE < 2) kk = __ldcs(reinterpret_cast<const uint2 *>(a.wk0 + p));
        else kk = *reinterpret_cast<const uint2 *>(a.wk1 + p);
        k0 = kk.x;
        k1 = kk.y;
    } else {
        k0 = k1 = 0;
    }
}

// Compact + offer NI items per thread of a TEAM (32 = warp, kBlock = block).
// rd[j] is the segment index item j was read from; w is team-uniform.
template <int MODE, int L, int TEAM, int NI>
__device__ __forceinline__ void team_commit(const RoundArgs &a, unsigned long long beg, const uint2 *x,
                                            const uint32_t *k, const bool *alive, const uint32_t *rd,
                                            uint32_t &w, Best &b, uint32_t (*s_cnt)[kWarps]) {
    if (MODE != 0) {
        const uint32_t lt = lanemask_lt();
        if (TEAM == 32) {
            if (MODE == 2) __syncwarp();
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                const uint32_t bal = __ballot_sync(0xffffffffu, alive[j]);
                const uint32_t pos = w + __popc(bal & lt);
                if (alive[j] && (MODE == 1 || pos != rd[j])) store_slot<L>(a, beg + pos, x[j], k[j]);
                w += __popc(bal);
            }
        } else {
            const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
            uint32_t bal[NI];
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                bal[j] = __ballot_sync(0xffffffffu, alive[j]);
                if (lane == 0) s_cnt[j][warp] = __popc(bal[j]);
            }
            __syncthreads();   // counts visible; also orders all reads before writes
            uint32_t base = w;
#pragma unroll
            for (int j = 0; j < NI; ++j) {
                uint32_t before = 0, cj = 0;
#pragma unroll
                for (int q = 0; q < kWarps; ++q) {
                    const uint32_t cq = s_cnt[j][q];
                    before += (q < warp) ? cq : 0u;
                    cj += cq;
                }
                const uint32_t pos = base + before + __popc(bal[j] & lt);
                if (alive[j] && (MODE == 1 || pos != rd[j])) store_slot<L>(a, beg + pos, x[j], k[j]);
                base += cj;
            }
            w = base;
            __syncthreads();   // s_cnt reuse
        }
    }
#pragma unroll
    for (int j = 0; j < NI; ++j)
        if (alive[j]) offer<L>(b, x[j].x, x[j].y, k[j], a);
}

// One scalar slot (segment index i) handled by thread 0 of the team.
template <int MODE, int L, int TEAM>
__device__ __forceinline__ void team_single(const RoundArgs &a, unsigned long long beg, uint32_t i, uint32_t &w,
                                            Best &b, uint32_t (*s_cnt)[kWarps]) {
    uint2 x = make_uint2(kNone, kNone);
    uint32_t k = 0;
    bool alive = false;
    if (threadIdx.x % TEAM == 0) {
        load_slot<MODE, L>(a, beg + i, x, k);
        alive = MODE == 0 || !is_matched(a.matched, x.x);
    }
    team_commit<MODE, L, TEAM, 1>(a, beg, &x, &k, &alive, &i, w, b, s_cnt);
}

// (A cp.async per-thread double buffer of the next pass was measured slower:
// its 24 KB of shared memory per block squeezes the L1 that serves the
// matched-bitmap lookups.  Register loads at full occupancy win.)
template <int MODE, int L, int TEAM>
__device__ __forceinline__ uint32_t team_vertex(const RoundArgs &a, unsigned long long beg, uint32_t d,
                                                Best &b, uint32_t (*s_cnt)[kWarps]) {
    const uint32_t t = threadIdx.x % TEAM;
    uint32_t w = 0;
    const uint32_t head = (uint32_t)(beg & 1ULL);
    if (head) team_single<MODE, L, TEAM>(a, beg, 0, w, b, s_cnt);
    const uint32_t rem = d - head;
    const uint32_t npairs = rem >> 1;
    for (uint32_t c = 0; c < npairs; c += kPairs * TEAM) {
        uint2 x[kBlockItems];
        uint32_t k[kBlockItems], rd[kBlockItems];
        bool alive[kBlockItems];
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
            const uint32_t p = c + j * TEAM + t;
            rd[2 * j] = head + 2 * p;
            rd[2 * j + 1] = head + 2 * p + 1;
            if (p < npairs) {
                load_pair<MODE, L>(a, beg + head + 2ULL * p, x[2 * j], x[2 * j + 1], k[2 * j], k[2 * j + 1]);
            } else {
                x[2 * j] = x[2 * j + 1] = make_uint2(kNone, kNone);
                k[2 * j] = k[2 * j + 1] = 0;
            }
        }
#pragma unroll
        for (int j = 0; j < kPairs; ++j) {
            const bool in = c + j * TEAM + t < npairs;
            alive[2 * j] = in && (MODE == 0 || !is_matched(a.matched, x[2 * j].x));
            alive[2 * j + 1] = in && (MODE == 0 || !is_matched(a.matched, x[2 * j + 1].x));
        }
        team_commit<MODE, L, TEAM, kBlockItems>(a, beg, x, k, alive, rd, w, b, s_cnt);
    }
    if (rem & 1u) team_single<MODE, L, TEAM>(a, beg, d - 1, w, b, s_cnt);
    best_group_reduce<32>(b);
    return MODE == 0 ? d : w;
}

__device__ __forceinline__ void put_result(const RoundArgs &a, int mode, uint32_t v, uint32_t w, const Best &b) {
    if (mode != 0) a.vdeg[v] = w;
    a.cand_nbr[v] = (w > 0) ? b.nbr : kNone;
    a.cand_id[v] = (w > 0) ? b.id : kNone;
}

// Buckets 1 and 5: a group of G lanes per vertex (live degree <= 4 G), 4
// rounds of 32 / G vertices per grab.
template <int MODE, int L, int G>
__device__ __forceinline__ void group_bucket(const RoundArgs &a, int q, uint32_t n, int lane,
                                             unsigned long long &live, unsigned long long &reads) {
    constexpr int kVpi = 32 / G, kIters = kVpi > 8 ? 32 / kVpi : 4, kGrab = kIters * kVpi;
    static_assert(G >= 2 && G <= 32 && (G & (G - 1)) == 0 && kGrab <= 32, "a grab's vertices are one per lane");
    for (;;) {
        uint32_t i0 = 0;
        if (lane == 0) i0 = atomicAdd(&a.ctr->cur[q], (uint32_t)kGrab);
        i0 = __shfl_sync(0xffffffffu, i0, 0);
        if (i0 >= n) break;
        uint32_t mv = kNone, md = 0;
        unsigned long long mb = 0;
        if (lane < kGrab && i0 + lane < n) {
            mv = a.list[q][i0 + lane];
            md = a.vdeg[mv];
            mb = a.vbeg[mv];
        }
#pragma unroll 1
        for (int it = 0; it < kIters; ++it) {
            const int src = it * kVpi + lane / G;
            const uint32_t v = __shfl_sync(0xffffffffu, mv, src);
            const uint32_t d = __shfl_sync(0xffffffffu, md, src);
            const unsigned long long beg = __shfl_sync(0xffffffffu, mb, src);
            Best b;
            best_init(b);
            const uint32_t w = group_vertex<MODE, L, G, 4>(a, beg, d, lane, b);
            if ((lane & (G - 1)) == 0 && d) {
                put_result(a, MODE, v, w, b);
                live += w;
                reads += d;
            }
        }
    }
}

template <int MODE, int L>
__global__ void __launch_bounds__(kBlock, LMX_MINB) lmx_round_kernel(RoundArgs a) {
    __shared__ uint32_t s_cnt[kBlockItems][kWarps];
    __shared__ Best s_best[kWarps];
    __shared__ uint32_t s_item;
    __shared__ unsigned long long s_red[2][kWarps];

    uint32_t nb[kBuckets];
    uint32_t any = 0;
#pragma unroll
    for (int q = 0; q < kBuckets; ++q) {
        nb[q] = a.ctr->n[q];
#ifdef LMX_ONLY_BUCKET   // profiling experiments only: time one bucket's mapping
        if (q != LMX_ONLY_BUCKET) nb[q] = 0;
#endif
        any |= nb[q];
    }
    if (any == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    unsigned long long live = 0, reads = 0;
#ifdef LMX_PHASE_TIMING
    long long phase_t0 = clock64();
#endif

    // phase 1: buckets 4 then 3, one block per vertex
#pragma unroll
    for (int q = 4; q >= 3; --q) {
        for (;;) {
            if (tid == 0) s_item = atomicAdd(&a.ctr->cur[q], 1u);
            __syncthreads();
            const uint32_t i = s_item;
            __syncthreads();
            if (i >= nb[q]) break;
            const uint32_t v = a.list[q][i];
            const uint32_t d = a.vdeg[v];
            Best b;
            best_init(b);
            const uint32_t w = team_vertex<MODE, L, kBlock>(a, a.vbeg[v], d, b, s_cnt);
            if (lane == 0) s_best[warp] = b;
            __syncthreads();
            if (tid == 0) {
                Best t = s_best[0];
                for (int z = 1; z < kWarps; ++z) best_merge(t, s_best[z]);
                put_result(a, MODE, v, w, t);
                live += w;
                reads += d;
            }
            __syncthreads();
        }
    }

    PHASE_MARK(0);
    // The small-vertex phases below fetch the per-vertex metadata (list entry,
    // live degree, segment start) of a whole grab at once, one vertex per
    // lane, and broadcast it: the list -> vdeg/vbeg -> slots dependency chain
    // is paid once per grab instead of once per vertex.

    // phase 2: bucket 2, warp per vertex, 8 vertices per grab
    for (;;) {
        uint32_t i0 = 0;
        if (lane == 0) i0 = atomicAdd(&a.ctr->cur[2], 8u);
        i0 = __shfl_sync(0xffffffffu, i0, 0);
        if (i0 >= nb[2]) break;
        uint32_t mv = kNone, md = 0;
        unsigned long long mb = 0;
        if (lane < 8 && i0 + lane < nb[2]) {
            mv = a.list[2][i0 + lane];
            md = a.vdeg[mv];
            mb = a.vbeg[mv];
        }
        const uint32_t cnt = min(8u, nb[2] - i0);
        for (uint32_t k = 0; k < cnt; ++k) {
            const uint32_t v = __shfl_sync(0xffffffffu, mv, k);
            const uint32_t d = __shfl_sync(0xffffffffu, md, k);
            const unsigned long long beg = __shfl_sync(0xffffffffu, mb, k);
            Best b;
            best_init(b);
            const uint32_t w = team_vertex<MODE, L, 32>(a, beg, d, b, s_cnt);
            if (lane == 0) {
                put_result(a, MODE, v, w, b);
                live += w;
                reads += d;
            }
        }
    }

    PHASE_MARK(1);
    // phase 3: buckets 1 (8 lanes per vertex) and 5 (4 lanes per vertex)
    group_bucket<MODE, L, 8>(a, 1, nb[1], lane, live, reads);
    group_bucket<MODE, L, 4>(a, 5, nb[5], lane, live, reads);


    PHASE_MARK(2);
    // phase 4: bucket 0, thread per vertex, 128 vertices per grab
    for (;;) {
        uint32_t i0 = 0;
        if (lane == 0) i0 = atomicAdd(&a.ctr->cur[0], 128u);
        i0 = __shfl_sync(0xffffffffu, i0, 0);
        if (i0 >= nb[0]) break;
        uint32_t mv[4], md[4];
#pragma unroll
        for (int it = 0; it < 4; ++it) {
            const uint32_t i = i0 + it * 32 + lane;
            mv[it] = (i < nb[0]) ? a.list[0][i] : kNone;
        }
#pragma unroll
        for (int it = 0; it < 4; ++it) md[it] = (mv[it] != kNone) ? a.vdeg[mv[it]] : 0u;
#pragma unroll 1
        for (int it = 0; it < 4; ++it) {
            const uint32_t v = mv[it], d = md[it];
            const unsigned long long beg = d ? a.vbeg[v] : 0ULL;
            Best b;
            best_init(b);
            const uint32_t w = group_vertex<MODE, L, 1, 4>(a, beg, d, lane, b);
            if (d) {
                put_result(a, MODE, v, w, b);
                live += w;
                reads += d;
            }
        }
    }

    PHASE_MARK(3);
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
    const uint32_t *cand_nbr;
    const uint32_t *cand_id;
    uint32_t *matched;
    long long *mate;
    const uint32_t *oldid;   // device id -> caller id (null: identity)
    const uint32_t *list;    // kBuckets regions of capacity `cap`
    uint32_t *next;          // kBuckets regions of capacity `cap`
    unsigned long long cap;
    uint32_t *ebits;            // matched edge-id bitmap (m bits)
    const uint32_t *eid_of_x;   // DISTINCT layout: weight key -> edge id (else null)
    uint32_t lo, nl;            // owned device-id range [lo, lo + nl)
    uint32_t *remote_ok;        // [nl] the remote partner's owner confirmed the edge
    uint32_t *mround;           // partitions: round each vertex was matched in (device ids), or null
    int round;
    RoundCtr *ctr;        // this round
    RoundCtr *ctr_next;   // next round (list sizes)
};

#ifndef LMX_MATCH_ITEMS
#define LMX_MATCH_ITEMS 4
#endif
#ifndef LMX_MATCH_MINB
#define LMX_MATCH_MINB 8
#endif
constexpr int kMatchItems = LMX_MATCH_ITEMS;
constexpr int kTargets = kBuckets;   // next-round bucket lists

__global__ void __launch_bounds__(kBlock, LMX_MATCH_MINB) lmx_match_kernel(MatchArgs a) {
    __shared__ uint32_t s_cnt[kTargets][kWarps];
    __shared__ uint32_t s_base[kTargets];
    uint32_t nb[kBuckets], pre[kBuckets + 1];
    pre[0] = 0;
#pragma unroll
    for (int q = 0; q < kBuckets; ++q) {
        nb[q] = a.ctr->n[q];
        pre[q + 1] = pre[q] + nb[q];
    }
    const uint32_t total = pre[kBuckets];
    if (total == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt();
    unsigned long long matched_v = 0;
    const uint32_t tile = kBlock * kMatchItems;
    for (uint32_t t0 = blockIdx.x * tile; t0 < total; t0 += gridDim.x * tile) {
        uint32_t vv[kMatchItems], kind[kMatchItems];
        uint32_t wc[kTargets];
#pragma unroll
        for (int q = 0; q < kTargets; ++q) wc[q] = 0;
#pragma unroll
        for (int j = 0; j < kMatchItems; ++j) {
            const uint32_t i = t0 + j * kBlock + tid;
            uint32_t v = kNone, d = 0;
            if (i < total) {
                int q = 0;
#pragma unroll
                for (int z = 1; z < kBuckets; ++z) q += (i >= pre[z]) ? 1 : 0;
                v = a.list[(unsigned long long)q * a.cap + (i - pre[q])];
                d = a.vdeg[v];
            }
            uint32_t kd = kTargets;   // none
            if (d > 0) {
                const uint32_t x = a.cand_nbr[v];   // global id
                const uint32_t id = a.cand_id[v];
                const uint32_t gv = v + a.lo;
                bool mutual;
                if (x - a.lo < a.nl) {
                    // edge ids / weight keys are unique per edge: same id at x <=> same edge
                    mutual = a.cand_id[x - a.lo] == id;
                } else {
                    // partner owned by another rank: its owner sent the edge back (exchange A)
                    mutual = a.remote_ok[v] != 0;
                    if (mutual) a.remote_ok[v] = 0;
                }
                if (mutual) {
                    atomicOr(a.matched + (gv >> 5), 1u << (gv & 31));
                    if (a.mround) a.mround[gv] = (uint32_t)a.round;
                    if (a.oldid) a.mate[a.oldid[gv]] = (long long)a.oldid[x];
                    else a.mate[gv] = (long long)x;
                    ++matched_v;
                    if (gv < x) {   // the lower endpoint records the edge (graph.py:195-203)
                        const uint32_t e = a.eid_of_x ? a.eid_of_x[id] : id;
                        atomicOr(a.ebits + (e >> 5), 1u << (e & 31));
                    }
                } else {
                    kd = (uint32_t)bucket_of(d);
                }
            }
            vv[j] = v;
            kind[j] = kd;
#pragma unroll
            for (int q = 0; q < kTargets; ++q) wc[q] += __popc(__ballot_sync(0xffffffffu, kd == (uint32_t)q));
        }
        if (lane == 0) {
#pragma unroll
            for (int q = 0; q < kTargets; ++q) s_cnt[q][warp] = wc[q];
        }
        __syncthreads();
        if (tid < kTargets) {
            uint32_t sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += s_cnt[tid][w];
            uint32_t base = 0;
            if (sum) base = atomicAdd(&a.ctr_next->n[tid], sum);
            s_base[tid] = base;
        }
        __syncthreads();
        uint32_t pos[kTargets];
#pragma unroll
        for (int q = 0; q < kTargets; ++q) {
            uint32_t p = s_base[q];
            for (int w = 0; w < warp; ++w) p += s_cnt[q][w];
            pos[q] = p;
        }
#pragma unroll
        for (int j = 0; j < kMatchItems; ++j) {
#pragma unroll
            for (int q = 0; q < kTargets; ++q) {
                const uint32_t bal = __ballot_sync(0xffffffffu, kind[j] == (uint32_t)q);
                if (kind[j] == (uint32_t)q) {
                    const uint32_t p = pos[q] + __popc(bal & lt);
                    a.next[(unsigned long long)q * a.cap + p] = vv[j];
                }
                pos[q] += __popc(bal);
            }
        }
        __syncthreads();   // s_cnt / s_base reuse
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) matched_v += __shfl_xor_sync(0xffffffffu, matched_v, off);
    if (lane == 0 && matched_v) atomicAdd(&a.ctr->matched_v, matched_v);
}

// Per-match initialisation: live degrees (owned), mates and matched bitmap (global).
__global__ void lmx_init_kernel(uint32_t n, uint32_t nl, const uint32_t *deg0, uint32_t *vdeg, long long *mate,
                                uint32_t *matched) {
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        if (v < nl) vdeg[v] = deg0[v];
        mate[v] = -1;
        if ((v & 31) == 0) matched[v >> 5] = 0;
    }
}

// ---- multi-GPU exchange A (bsp.py:148-167 as a minimal record exchange) ----
struct ProposeArgs {
    const uint32_t *vdeg;
    const uint32_t *cand_nbr;
    const uint32_t *cand_id;
    const uint32_t *list;
    unsigned long long cap;
    const RoundCtr *ctr;
    const uint32_t *eid_of_x;
    const unsigned long long *bounds;   // p + 1 cut points (global ids)
    int p;
    uint32_t lo, nl;
    uint32_t *cnt;      // [p] records per destination
    uint2 *region;      // p regions of capacity nl: {global target vertex, edge id}
};

// For every owned live vertex whose candidate partner is owned elsewhere, send
// {partner, edge id} to the partner's owner.  Pass 0 counts per destination,
// pass 1 writes the records grouped by destination.
__global__ void lmx_propose_kernel(ProposeArgs a) {
    uint32_t total = 0;
#pragma unroll
    for (int q = 0; q < kBuckets; ++q) total += a.ctr->n[q];
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        uint32_t q = 0, base = 0;
        while (q + 1 < (uint32_t)kBuckets && i >= base + a.ctr->n[q]) base += a.ctr->n[q++];
        const uint32_t v = a.list[(unsigned long long)q * a.cap + (i - base)];
        if (a.vdeg[v] == 0) continue;
        const uint32_t x = a.cand_nbr[v];
        if (x - a.lo < a.nl) continue;   // local partner
        int k = 0;
        while (k + 1 < a.p && x >= a.bounds[k + 1]) ++k;
        const uint32_t id = a.cand_id[v];
        const uint32_t e = a.eid_of_x ? a.eid_of_x[id] : id;
        const uint32_t pos = atomicAdd(a.cnt + k, 1u);
        a.region[(unsigned long long)k * a.nl + pos] = make_uint2(x, e);
    }
}

// Pack the p regions back to back (destination order) and publish the counts
// as int64 for the collective; no host round trip.
__global__ void lmx_pack_kernel(const uint2 *region, const uint32_t *cnt, int p, uint32_t nl, uint2 *packed,
                                long long *counts64) {
    const uint32_t stride = gridDim.x * blockDim.x;
    const uint32_t tid0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid0 < (uint32_t)p) counts64[tid0] = cnt[tid0];
    uint32_t cmax = 0;   // no region holds more records than this
    for (int k = 0; k < p; ++k) cmax = max(cmax, cnt[k]);
    for (uint32_t i = tid0; i < min(nl, cmax); i += stride) {
        uint32_t off = 0;
        for (int k = 0; k < p; ++k) {
            const uint32_t c = cnt[k];
            if (i < c) packed[off + i] = region[(unsigned long long)k * nl + i];
            off += c;
        }
    }
}

// Received {x, e}: x (owned) is matched across the cut iff its own candidate is edge e.
__global__ void lmx_accept_kernel(const uint2 *rec, unsigned long long k, const uint32_t *vdeg,
                                  const uint32_t *cand_id, const uint32_t *eid_of_x, uint32_t lo,
                                  uint32_t *remote_ok) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint2 r = rec[i];
        const uint32_t xl = r.x - lo;
        if (vdeg[xl] == 0) continue;
        const uint32_t id = cand_id[xl];
        const uint32_t e = eid_of_x ? eid_of_x[id] : id;
        if (e == r.y) remote_ok[xl] = 1u;
    }
}

// K5: matched edge ids, ascending, from the edge-id bitmap.
__global__ void lmx_word_counts(const uint32_t *ebits, unsigned long long words, uint32_t *cnt) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += stride)
        cnt[i] = __popc(ebits[i]);
}

template <typename T>
__global__ void lmx_emit_ids(const uint32_t *ebits, const uint32_t *off, unsigned long long words, T *out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < words;
         i += stride) {
        uint32_t bits = ebits[i];
        uint32_t p = off[i];
        while (bits) {
            const int b = __ffs(bits) - 1;
            bits &= bits - 1;
            out[p++] = (T)(i * 32 + b);
        }
    }
}

}  // namespace lmx

using namespace lmx;

template <int MODE, int L>
static void launch_round_l(lmx_ctx *ctx, const RoundArgs &a) {
    lmx_round_kernel<MODE, L><<<ctx->round_grid[MODE][L], kBlock, 0, ctx->stream>>>(a);
}

template <int MODE>
static void launch_round(lmx_ctx *ctx, const RoundArgs &a) {
    if (ctx->layout == kUniform) launch_round_l<MODE, kUniform>(ctx, a);
    else if (ctx->layout == kDistinct) launch_round_l<MODE, kDistinct>(ctx, a);
    else launch_round_l<MODE, kGeneral>(ctx, a);
}

int lmx_alloc_match_state(lmx_ctx *ctx) {
    const size_t n = (size_t)std::max<int64_t>(ctx->n, 1);          // global ids
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);   // owned vertices
    // per-vertex state of the owned vertices (local index v - lo)
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->vdeg, nl * 4, "vdeg"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->cand, nl * 8, "cand"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->remote_ok, nl * 4, "remote_ok"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mate, n * 8, "mate"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->matched, ((n + 31) / 32) * 4, "matched"));
    // the scan loop keeps one list per round; the compacting loop one per live-degree bucket
    const size_t regions = ctx->algo == 1 ? 1 : kBuckets;
    for (int i = 0; i < 2; ++i) LMX_TRY(lmx_alloc(ctx, (void **)&ctx->lists[i], nl * 4 * regions, "lists"));
    const size_t words = (size_t)(std::max<int64_t>(ctx->m, 1) + 31) / 32;
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mids, (n / 2 + 1) * 8, "mids"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ebits, words * 4, "ebits"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ebits_off, words * 4, "ebits_off"));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->remote_ok, 0, nl * 4, ctx->stream));
    size_t tmp = 0;
    LMX_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->ebits_off, ctx->ebits_off, (long long)words));
    ctx->sort_tmp_bytes = tmp + 256;
    LMX_TRY(lmx_alloc(ctx, &ctx->sort_tmp, ctx->sort_tmp_bytes, "sort_tmp"));
    return LMX_OK;
}

// Ensure ctr has room for rounds [0, need].  Only called with the stream idle.
int lmx_ensure_ctr(lmx_ctx *ctx, int need) {
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
    // the persistent scan loop's round count + per-phase stamps
    if (ctx->loop_aux) cudaFree(ctx->loop_aux);
    if (ctx->loop_host) cudaFreeHost(ctx->loop_host);
    ctx->loop_aux = ctx->loop_host = nullptr;
    LMX_CUDA(ctx, cudaMalloc(&ctx->loop_aux, lmx_loop_aux_bytes(ncap)));
    LMX_CUDA(ctx, cudaMallocHost(&ctx->loop_host, lmx_loop_aux_bytes(ncap)));
    return LMX_OK;
}

// ---- round-loop building blocks (shared by the single-GPU loop and the
// stepped multi-GPU protocol) ------------------------------------------------

// Reset per-match state: counters, edge bitmap, live degrees, mates, bitmap.
static int begin_match(lmx_ctx *ctx) {
    const uint32_t nl = (uint32_t)ctx->n_local;
    LMX_TRY(lmx_ensure_ctr(ctx, 64));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ctr, 0, sizeof(RoundCtr) * (size_t)ctx->ctr_cap, ctx->stream));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ebits, 0, ((size_t)std::max<int64_t>(ctx->m, 1) + 31) / 32 * 4, ctx->stream));
    ctx->ctr_host[0] = RoundCtr{};
    for (int q = 0; q < kBuckets; ++q) ctx->ctr_host[0].n[q] = ctx->n_bins0[q];
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr, ctx->ctr_host, sizeof(RoundCtr), cudaMemcpyHostToDevice,
                                  ctx->stream));
    if (ctx->n > 0) {
        lmx_init_kernel<<<ctx->num_sms * 8, kBlock, 0, ctx->stream>>>((uint32_t)ctx->n, nl, ctx->deg0, ctx->vdeg,
                                                                     ctx->mate_target, ctx->matched);
        LMX_CUDA(ctx, cudaGetLastError());
        ctx->timing.round_launches += 1;
    }
    return LMX_OK;
}

static size_t list_cap(const lmx_ctx *ctx) { return (size_t)std::max<int64_t>(ctx->n_local, 1); }

static int enqueue_round_kernel(lmx_ctx *ctx, int r, uint64_t seed_masked, bool rerandomize) {
    const size_t cap = list_cap(ctx);
    const int mode = r == 0 ? 0 : (r == 1 ? 1 : 2);
    const uint32_t *cur = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
    RoundArgs a;
    a.vbeg = ctx->vbeg;
    a.vdeg = ctx->vdeg;
    a.cand_nbr = reinterpret_cast<uint32_t *>(ctx->cand);
    a.cand_id = a.cand_nbr + cap;
    a.ids0 = ctx->ids0;
    a.wk0 = ctx->wk0;
    a.ids1 = ctx->ids1;
    a.wk1 = ctx->wk1;
    a.matched = ctx->matched;
    for (int q = 0; q < kBuckets; ++q) a.list[q] = cur + (size_t)q * cap;
    a.ctr = ctx->ctr + r;
    a.round = r;
    a.rs = round_seed(seed_masked, (uint64_t)r, rerandomize);
    a.n_distinct = ctx->n_distinct;
    a.tie_rank = ctx->tie_rank;
    a.eid_of_x = ctx->eid_of_x;
    if (mode == 0) launch_round<0>(ctx, a);
    else if (mode == 1) launch_round<1>(ctx, a);
    else launch_round<2>(ctx, a);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

static int enqueue_match_kernel(lmx_ctx *ctx, int r) {
    const size_t cap = list_cap(ctx);
    MatchArgs ma;
    ma.vdeg = ctx->vdeg;
    ma.cand_nbr = reinterpret_cast<const uint32_t *>(ctx->cand);
    ma.cand_id = ma.cand_nbr + cap;
    ma.matched = ctx->matched;
    ma.mate = ctx->mate_target;
    ma.oldid = ctx->relabeled ? ctx->oldid : nullptr;
    ma.list = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
    ma.next = ctx->lists[(r + 1) & 1];
    ma.cap = cap;
    ma.ebits = ctx->ebits;
    ma.eid_of_x = ctx->layout == kDistinct ? ctx->eid_of_x : nullptr;
    ma.lo = (uint32_t)ctx->lo;
    ma.nl = (uint32_t)ctx->n_local;
    ma.remote_ok = ctx->remote_ok;
    ma.mround = ctx->dist_p > 1 ? ctx->mround : nullptr;
    ma.round = r;
    ma.ctr = ctx->ctr + r;
    ma.ctr_next = ctx->ctr + r + 1;
    lmx_match_kernel<<<ctx->match_blocks, kBlock, 0, ctx->stream>>>(ma);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

// The round loop of local_max_seq (matchers.py:87-119) on the device.
// Leaves mate in `mate` (ctx->mate or the caller's device buffer) and the
// matched edge-id bitmap in ctx->ebits.
int lmx_run_rounds(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                   std::vector<lmx_round_stats> &stats, unsigned long long &n_matched) {
    stats.clear();
    n_matched = 0;
    ctx->timing.round_launches = 0;
    ctx->timing.slot_reads = 0;
    ctx->timing.round_kernel_ms = 0;
    ctx->timing.match_kernel_ms = 0;
    ctx->timing.hist_kernel_ms = 0;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    LMX_TRY(begin_match(ctx));
    // optional per-kernel timeline: tl[0] after init, then (after round r, after match r)
    int tl_used = 0;
    auto tl_mark = [&]() -> int {
        if (!ctx->kernel_timing) return LMX_OK;
        if (tl_used >= (int)ctx->tl_events.size()) {
            cudaEvent_t e;
            LMX_CUDA(ctx, cudaEventCreate(&e));
            ctx->tl_events.push_back(e);
        }
        LMX_CUDA(ctx, cudaEventRecord(ctx->tl_events[tl_used++], ctx->stream));
        return LMX_OK;
    };
    LMX_TRY(tl_mark());
    int r = 0;
    int n_rounds = -1;
    int batch = 6;
    while (n_rounds < 0 && ctx->m > 0) {
        LMX_TRY(lmx_ensure_ctr(ctx, r + batch + 1));
        const int r0 = r;
        for (int b = 0; b < batch; ++b, ++r) {
            LMX_TRY(enqueue_round_kernel(ctx, r, seed_masked, rerandomize));
            LMX_TRY(tl_mark());
            LMX_TRY(enqueue_match_kernel(ctx, r));
            LMX_TRY(tl_mark());
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
        // the next batch: as many rounds as the live slots' decay over the last
        // round predicts (+1), 1..4 -- empty rounds past the end cost launches
        batch = 4;
        if (n_rounds < 0 && r >= 2) {
            const double last = (double)ctx->ctr_host[r - 1].live_slots, prev = (double)ctx->ctr_host[r - 2].live_slots;
            if (last > 0 && prev > last) {
                const double q = last / prev;   // per-round survival of live slots
                const double est = std::log(std::max(last, 2.0)) / std::log(1.0 / q) + 1.0;
                batch = std::max(1, std::min(4, (int)std::ceil(est)));
            }
        }
#ifdef LMX_ONLY_BUCKET   // profiling experiments: results are meaningless, stop after one batch
        if (n_rounds < 0) n_rounds = 0;
#endif
    }
    ctx->kernel_ms.clear();
    if (ctx->kernel_timing && tl_used > 1) {
        for (int i = 1; i < tl_used; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->tl_events[i - 1], ctx->tl_events[i]);
            ctx->kernel_ms.push_back(ms);
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

// ---- stepped protocol of the 1D-partitioned engine (bsp.py:101-205) --------
// Per round, driven by the host (paper_1302_4587_b200/dist.py):
//   round kernel -> propose (candidate records for remote partners, exchange A)
//   -> [all-to-all-v] -> accept -> match (local + confirmed remote pairs)
//   -> [all-gather of the owned matched-bitmap words, exchange B]
//   -> [all-reduce of (live slots, matched vertices)].

int lmx_dist_begin_impl(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize) {
    if (ctx->algo == 1) return lmx_scan_dist_begin(ctx, seed_masked, rerandomize);
    ctx->timing.round_launches = 0;
    ctx->dist_round = 0;
    ctx->dist_seed = seed_masked;
    ctx->dist_rr = rerandomize;
    ctx->mate_target = ctx->mate;
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->remote_ok, 0, (size_t)std::max<int64_t>(ctx->n_local, 1) * 4, ctx->stream));
    if (ctx->mround)
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mround, 0xFF, (size_t)std::max<int64_t>(ctx->n, 1) * 4, ctx->stream));
    LMX_TRY(begin_match(ctx));
    LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return LMX_OK;
}

int lmx_dist_round_impl(lmx_ctx *ctx) {
    if (ctx->algo == 1) return lmx_scan_dist_round(ctx);
    LMX_TRY(lmx_ensure_ctr(ctx, ctx->dist_round + 2));
    return enqueue_round_kernel(ctx, ctx->dist_round, ctx->dist_seed, ctx->dist_rr);
}

// Exchange-A records, fully on the device: fill per-destination regions, pack
// them, publish int64 counts.  Returns device pointers; no synchronisation.
int lmx_dist_propose_impl(lmx_ctx *ctx, void **counts_dev, void **packed_dev) {
    if (ctx->algo == 1) return lmx_scan_dist_propose(ctx, counts_dev, packed_dev);
    const int p = ctx->dist_p;
    const int r = ctx->dist_round;
    const size_t cap = list_cap(ctx);
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);
    const size_t need = nl * (size_t)(p + 1);   // p regions + the packed copy
    if (ctx->send_cap < need) {
        lmx_dfree(ctx, ctx->send);
        ctx->send = nullptr;
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->send, need * sizeof(uint2)));
        ctx->send_cap = need;
    }
    // send_cnt block: [64] u32 counts, [64] i64 counts at +256, the p + 1 bounds (u64)
    // at +1024, uploaded once per load
    unsigned long long *bnd = nullptr;
    if (!ctx->send_cnt) {
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->send_cnt, 2048));
        std::vector<unsigned long long> hb(ctx->bounds.begin(), ctx->bounds.end());
        LMX_CUDA(ctx, cudaMemcpyAsync(reinterpret_cast<char *>(ctx->send_cnt) + 1024, hb.data(),
                                      (size_t)(p + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    bnd = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(ctx->send_cnt) + 1024);
    long long *counts64 = reinterpret_cast<long long *>(reinterpret_cast<char *>(ctx->send_cnt) + 256);
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->send_cnt, 0, 64 * sizeof(uint32_t), ctx->stream));
    ProposeArgs pa;
    pa.vdeg = ctx->vdeg;
    pa.cand_nbr = reinterpret_cast<const uint32_t *>(ctx->cand);
    pa.cand_id = pa.cand_nbr + cap;
    pa.list = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
    pa.cap = cap;
    pa.ctr = ctx->ctr + r;
    pa.eid_of_x = ctx->layout == kDistinct ? ctx->eid_of_x : nullptr;
    pa.bounds = bnd;
    pa.p = p;
    pa.lo = (uint32_t)ctx->lo;
    pa.nl = (uint32_t)ctx->n_local;
    pa.cnt = ctx->send_cnt;
    pa.region = ctx->send;
    lmx_propose_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(pa);
    LMX_CUDA(ctx, cudaGetLastError());
    uint2 *packed = ctx->send + nl * (size_t)p;
    lmx_pack_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(ctx->send, ctx->send_cnt, p, (uint32_t)nl,
                                                                 packed, counts64);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 2;
    *counts_dev = counts64;
    *packed_dev = packed;
    return LMX_OK;
}

int lmx_dist_recv_impl(lmx_ctx *ctx, int64_t count, void **ptr) {
    const size_t need = (size_t)std::max<int64_t>(count, 1);
    if (ctx->recv_cap < need) {
        lmx_dfree(ctx, ctx->recv);
        ctx->recv = nullptr;
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->recv, need * sizeof(uint2)));
        ctx->recv_cap = need;
    }
    *ptr = ctx->recv;
    return LMX_OK;
}

int lmx_dist_accept_impl(lmx_ctx *ctx, int64_t count) {
    if (ctx->algo == 1) return lmx_scan_dist_accept(ctx, count);
    if (count <= 0) return LMX_OK;
    const size_t cap = list_cap(ctx);
    lmx_accept_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(
        ctx->recv, (unsigned long long)count, ctx->vdeg, reinterpret_cast<const uint32_t *>(ctx->cand) + cap,
        ctx->layout == kDistinct ? ctx->eid_of_x : nullptr, (uint32_t)ctx->lo, ctx->remote_ok);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

// Enqueue the match kernel; *stats_dev = the round's {live slots, matched
// vertices} (two u64 on the device) for the host's all-reduce.  No sync.
int lmx_dist_match_impl(lmx_ctx *ctx, void **stats_dev) {
    if (ctx->algo == 1) return lmx_scan_dist_match(ctx, stats_dev);
    const int r = ctx->dist_round;
    LMX_TRY(enqueue_match_kernel(ctx, r));
    *stats_dev = &ctx->ctr[r].live_slots;   // live_slots, matched_v are adjacent
    ctx->dist_round = r + 1;
    return LMX_OK;
}

// K5: ascending matched edge ids from the bitmap; mate / ids out.
int lmx_emit_outputs(lmx_ctx *ctx, unsigned long long n_matched, int64_t *mate_out,
                     int64_t *ids_out, int out_where) {
    const size_t n = (size_t)ctx->n;
    const unsigned long long words = ((unsigned long long)std::max<int64_t>(ctx->m, 1) + 31) / 32;
    const int grid = ctx->num_sms * 8;
    if (n_matched > 0 && ids_out) {
        lmx_word_counts<<<grid, kBlock, 0, ctx->stream>>>(ctx->ebits, words, ctx->ebits_off);
        LMX_CUDA(ctx, cudaGetLastError());
        size_t tmp = ctx->sort_tmp_bytes;
        LMX_CUDA(ctx, cub::DeviceScan::ExclusiveSum(ctx->sort_tmp, tmp, ctx->ebits_off, ctx->ebits_off,
                                                    (long long)words, ctx->stream));
        // int64 ids straight into the caller's device buffer, or staged on the
        // device and copied once (a pinned host buffer takes it at link rate)
        lmx_emit_ids<long long><<<grid, kBlock, 0, ctx->stream>>>(
            ctx->ebits, ctx->ebits_off, words, out_where == LMX_DEVICE ? (long long *)ids_out : ctx->mids);
        LMX_CUDA(ctx, cudaGetLastError());
        ctx->timing.round_launches += 2;
    }
    if (out_where == LMX_DEVICE) {
        if (mate_out && n && ctx->mate_target != (long long *)mate_out)
            LMX_CUDA(ctx, cudaMemcpyAsync(mate_out, ctx->mate_target, n * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev2, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    } else {
        if (ctx->mate_early_done && mate_out == ctx->mate_early)   // copied next to the histogram
            LMX_CUDA(ctx, cudaStreamWaitEvent(ctx->stream, ctx->ev_mate, 0));
        else if (mate_out && n)
            LMX_CUDA(ctx, cudaMemcpyAsync(mate_out, ctx->mate_target, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
        ctx->mate_early_done = false;
        ctx->mate_early = nullptr;
        if (ids_out && n_matched)
            LMX_CUDA(ctx, cudaMemcpyAsync(ids_out, ctx->mids, (size_t)n_matched * 8, cudaMemcpyDeviceToHost,
                                          ctx->stream));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev2, ctx->stream));
        LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.rounds_ms = ms;
    cudaEventElapsedTime(&ms, ctx->ev1, ctx->ev2);
    ctx->timing.output_ms = ms;
    return LMX_OK;
}

// Persistent grid sizes: every resident block slot of the device, per instance.
template <int MODE, int L>
static int occ_of(lmx_ctx *ctx) {
    int occ = 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lmx_round_kernel<MODE, L>, kBlock, 0));
    ctx->round_grid[MODE][L] = ctx->num_sms * std::max(occ, 1);
    return LMX_OK;
}

int lmx_configure_grids(lmx_ctx *ctx) {
    LMX_TRY((occ_of<0, kUniform>(ctx)));
    LMX_TRY((occ_of<0, kDistinct>(ctx)));
    LMX_TRY((occ_of<0, kGeneral>(ctx)));
    LMX_TRY((occ_of<1, kUniform>(ctx)));
    LMX_TRY((occ_of<1, kDistinct>(ctx)));
    LMX_TRY((occ_of<1, kGeneral>(ctx)));
    LMX_TRY((occ_of<2, kUniform>(ctx)));
    LMX_TRY((occ_of<2, kDistinct>(ctx)));
    LMX_TRY((occ_of<2, kGeneral>(ctx)));
    int occ = 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, lmx_match_kernel, kBlock, 0));
    ctx->match_blocks = ctx->num_sms * std::max(occ, 1);
    return LMX_OK;
}

#ifdef LMX_PHASE_TIMING
extern "C" int lmx_debug_phase_cycles(unsigned long long *out, int reset) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, lmx::g_phase_cycles, sizeof(unsigned long long) * 64 * 5);
    if (reset) {
        static unsigned long long zero[64 * 5] = {};
        cudaMemcpyToSymbol(lmx::g_phase_cycles, zero, sizeof(zero));
    }
    return 0;
}
#endif
