// lmx_scan.cu -- the weight-ordered round loop ("scan" algorithm) for the
// DISTINCT weight-key layout on one GPU.
//
// Same result as local_max_seq (matchers.py:61-122) and as the compacting
// round loop of lmx_round.cu, with O(m) total slot traffic instead of
// O(sum_r m_r + m):
//
//   * At load time every vertex segment of ids0 is sorted by weight rank,
//     descending (lmx_setup.cu).  With (almost) distinct weights the key order
//     of a vertex's edges is then the same in every round: only the edges of
//     one tied weight need the per-round salt (tiebreak.py:55-80), and those
//     sit next to each other in the segment.
//   * ptr[v] marks the first slot of v not yet known to be dead.  Edges only
//     ever die (matchers.py:111), so v's candidate in round r is the first live
//     slot at or after ptr[v] (or the salt-max of the tied run it starts): one
//     probe for most vertices, and every slot is skipped at most once.
//   * Active lists: A_0 = every vertex with an edge; A_{r+1} = the vertices of
//     A_r that found a candidate and stayed unmatched.  A live edge at round r
//     has both endpoints in A_r, so "no candidate found in round r" is exactly
//     "m_r = 0" (the loop's exit test, matchers.py:87-90).
//   * RoundStats (matchers.py:113-118) without per-round edge counting: an edge
//     dies in round min(mround[u], mround[v]) (the first round one of its ends
//     is matched), so one pass over each edge once (the lower-id adjacency,
//     lowpair) after the loop histograms the death rounds; m_r is the suffix sum.
//
// Kernels: lmx_scan_round_kernel (candidate probe of A_r, thread per vertex),
// lmx_scan_match_kernel (mutual candidates -> bitmap, mate, mround, edge bit;
// appends A_{r+1}), lmx_scan_hist_kernel (death-round histogram).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <vector>

#include "lmx_internal.cuh"

#ifndef LMX_SCAN_MINB
#define LMX_SCAN_MINB 4
#endif
#ifndef LMX_SCAN_VPL
#define LMX_SCAN_VPL 4   // vertices per lane per grab of the probe kernel
#endif
#ifndef LMX_SCAN_MATCH_ITEMS
#define LMX_SCAN_MATCH_ITEMS 4   // vertices per thread per tile of the match kernel
#endif
#ifndef LMX_SCAN_MATCH_MINB
#define LMX_SCAN_MATCH_MINB 8
#endif
#ifndef LMX_HIST_V_GLOBAL
#define LMX_HIST_V_GLOBAL 1
#endif
#ifndef LMX_HIST_PF2
#define LMX_HIST_PF2 1
#endif
#ifndef LMX_HIST_U
#define LMX_HIST_U 2   // uint4 (2 edges) loads per thread per step of the histogram
#endif

namespace lmx {

constexpr int kHistBins = 256;   // death-round bins kept in shared memory (more go global)
constexpr int kVpl = LMX_SCAN_VPL;
#ifndef LMX_SLOW_BALANCE
#define LMX_SLOW_BALANCE 1   // deal a warp's slow-path vertices round-robin to its lanes (0: each lane its own)
#endif
// cache hints for data read once per round (slots skipped past, list
// entries): evict-first, so the candidate words and bitmaps keep L2
#ifndef LMX_STREAM_HINTS
#define LMX_STREAM_HINTS 0
#endif
#if LMX_STREAM_HINTS
#define LMX_LD_STREAM(p) __ldcs(p)
#define LMX_ST_STREAM(p, x) __stcs((p), (x))
#else
#define LMX_LD_STREAM(p) (*(p))
#define LMX_ST_STREAM(p, x) (*(p) = (x))
#endif
#ifndef LMX_SLOW_BATCH
#define LMX_SLOW_BATCH 1     // chunks whose slow vertices are pooled before they are dealt
#endif

constexpr uint32_t kTiedFlag = 0x80000000u;   // candidate word: the weight is tied at v
constexpr uint32_t kNbrMask = 0x7FFFFFFFu;

// Edge id of the current candidate of owned vertex vl (local index; neighbour
// word w != kNone): a tied candidate keeps it in ckey, an untied one sits at
// slot ptr.
__device__ __forceinline__ uint32_t cand_eid(uint32_t vl, uint32_t w, const uint32_t *ckey, const uint32_t *ptr,
                                             const unsigned long long *vbeg, const uint2 *ids) {
    return (w & kTiedFlag) ? ckey[vl] : ids[vbeg[vl] + ptr[vl]].y;
}

// Per-vertex arrays are indexed by the local id v - lo of the owned range
// [lo, lo + nl) (one GPU: lo = 0); lists, neighbours, the matched bitmap and
// the match rounds use device ids.
struct ScanArgs {
    const unsigned long long *vbeg;   // [nl + 1] owned segment offsets
    uint32_t *ptr;              // first possibly-live slot of each vertex (segment offset)
    // each vertex's candidate: the neighbour word (bit 31: the weight is tied)
    // -- the probe's fast path and the match kernel read 4 bytes -- and, for a
    // tied candidate only, its edge id; an untied candidate sits at slot ptr
    // (cand_eid() reads it there when a matched edge needs its id)
    uint32_t *cnbr, *ckey;
    const uint2 *cand0;         // round-0 candidates: the first slot of each segment
    const uint2 *ids;           // ids0 {nbr | tie flags, edge id}, weight-descending per segment
    const uint32_t *matched;    // matched-vertex bitmap
    const uint32_t *alist;      // A_r
    RoundCtr *ctr;              // ctr[r]: pad[0] = |A_r|, pad[1] = grab cursor
    uint64_t rs;                // round seed (tiebreak.py:40-52)
    uint32_t lo, nl;            // owned range
    // stepped multi-GPU protocol (DIST): exchange A's records are appended by
    // the probe itself -- a candidate whose partner is owned elsewhere goes to
    // that owner's region -- so no second pass over A_r is needed
    const unsigned long long *bounds;   // p + 1 cut points (global ids)
    int p;
    uint32_t *cnt;                      // [p] records per destination
    uint2 *region;                      // p regions of capacity nl: {partner, edge id}
};

// Exchange-A record {x, edge id} to the owner of x.
__device__ __forceinline__ void propose_record(const ScanArgs &a, uint32_t x, uint32_t eid) {
    int k = 0;
    while (k + 1 < a.p && x >= a.bounds[k + 1]) ++k;
    const uint32_t pos = atomicAdd(a.cnt + k, 1u);
    a.region[(unsigned long long)k * a.nl + pos] = make_uint2(x, eid);
}

// (Measured and rejected, match kernel: an 8-bit fingerprint array of the
// candidates' neighbours screening the partner gather (-0.08 ms matching,
// +0.06 ms probing); candidates carried in list order next to the lists
// (probe +0.15 ms, matching unchanged).  The partner gather is latency-bound,
// not bandwidth-bound.)
// (Measured and rejected: proposing each candidate to its other end with an
// atomicMax of {round, rank}, so the match kernel reads its own word instead
// of the partner's candidate.  The atomics serialise on the hubs that most
// vertices propose to: probe 2.8 -> 7.0 ms for a 0.26 ms gain in matching.)

__device__ __forceinline__ bool bit_set(const uint32_t *bits, uint32_t u) {
    return (bits[u >> 5] >> (u & 31)) & 1u;
}

__device__ __forceinline__ uint32_t lanemask_lt_u32() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// First live slot at or after p (p is left on it).  False when v has none.
template <bool FIRST>
__device__ __forceinline__ bool advance(const ScanArgs &a, unsigned long long b, uint32_t &p, uint32_t d,
                                        uint2 &out, unsigned long long &reads) {
    while (p < d) {
        const uint32_t cnt = min(4u, d - p);
        uint2 s[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) s[j] = (uint32_t)j < cnt ? LMX_LD_STREAM(a.ids + b + p + j) : make_uint2(kNone, kNone);
        reads += cnt;
        uint32_t live = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if ((uint32_t)j < cnt && (FIRST || !bit_set(a.matched, s[j].x & kSlotNbr))) live |= 1u << j;
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

// `out` (at p, the first live slot at or after ptr) is tied: every live slot
// of the rest of its run of equal weight competes on the edge salt
// (tiebreak.py:55-80); the run ends at an untied slot or the next run start.
template <bool FIRST>
__device__ __forceinline__ void resolve_tie(const ScanArgs &a, unsigned long long b, uint32_t p, uint32_t d,
                                            uint2 &out, unsigned long long &reads) {
    uint64_t best = mix64((uint64_t)out.y ^ a.rs);
    for (uint32_t q = p + 1; q < d; ++q) {
        const uint2 t = a.ids[b + q];
        ++reads;
        if (!(t.x & kSlotTied) || (t.x & kSlotRunStart)) break;
        if (!FIRST && bit_set(a.matched, t.x & kSlotNbr)) continue;
        const uint64_t s = mix64((uint64_t)t.y ^ a.rs);
        if (s > best) {
            best = s;
            out = t;
        }
    }
}

// Round 0: every candidate is the first slot of its segment (cand0, built at
// load), unless that slot's weight is tied.  Round r >= 1: the last round's
// candidate is re-checked first -- it is still the candidate if its
// neighbour is unmatched and its weight unique, so most vertices read 12
// bytes (list, cand) plus one bitmap bit and write nothing.
template <bool FIRST, bool DIST>
__device__ __forceinline__ void probe_body(const ScanArgs &a, unsigned long long (&s_red)[3][kWarps],
                                           uint32_t (*s_slowq)[32 * kVpl * LMX_SLOW_BATCH]) {
    const uint32_t na = a.ctr->pad[0];
    if (na == 0) return;
    const int tid = threadIdx.x, lane = tid & 31;
    unsigned long long found_n = 0, reads = 0, slow_n = 0;
    // thread per vertex, 4 vertices per lane per grab
#ifndef LMX_SCAN_STATIC_PCT
#define LMX_SCAN_STATIC_PCT 0   // rounds >= 1: share of the list split statically (measured: no gain)
#endif
    // The first part of the list is split statically (warp-strided chunks, no
    // atomics); the rest is grabbed chunk by chunk, which balances the slow
    // paths.  Round 0 has no dead slots to skip (only rare tied runs): all
    // static.  (The grab atomics on one address serialise: ~1 per ns.)
    constexpr uint32_t kChunk = 32u * kVpl;
    const uint32_t nchunks = (na + kChunk - 1) / kChunk;
    const uint32_t nstat = FIRST ? nchunks : (uint32_t)((unsigned long long)nchunks * LMX_SCAN_STATIC_PCT / 100);
    uint32_t c = blockIdx.x * (uint32_t)kWarps + (uint32_t)(tid >> 5);
    const uint32_t cstride = gridDim.x * (uint32_t)kWarps;
    // slow path: the candidate died (advance past dead slots) or its weight is tied
    auto slow_one = [&](uint32_t vk, uint32_t ck) {
        const uint32_t vl = vk - a.lo;
        const uint32_t pk = FIRST ? 0u : a.ptr[vl];
        const unsigned long long bk = a.vbeg[vl];
        // the segment end sits next to its start (same sector 3 times in
        // 4): one random gather fewer than reading a degree (2.62 -> 2.52 ms)
        const uint32_t dk = (uint32_t)(a.vbeg[vl + 1] - bk);
        // an untied candidate sits at ptr and is known dead: search past it;
        // a tied one: ptr is the first slot not known dead, live or not
        uint32_t pp = (!FIRST && ck != kNone && !(ck & kTiedFlag)) ? pk + 1 : pk;
        uint2 out = make_uint2(kNone, kNone);
        const bool found = advance<FIRST>(a, bk, pp, dk, out, reads);
        const bool tied = found && (out.x & kSlotTied);
        if (tied) resolve_tie<FIRST>(a, bk, pp, dk, out, reads);
        const uint32_t nbr = out.x & kSlotNbr;
        a.cnbr[vl] = found ? (nbr | (tied ? kTiedFlag : 0u)) : kNone;
        if (tied) a.ckey[vl] = out.y;   // an untied candidate's edge is the slot at ptr
        if (pp != pk) a.ptr[vl] = pp;
        if (DIST && found && nbr - a.lo >= a.nl) propose_record(a, nbr, out.y);
        found_n += found ? 1u : 0u;
        ++slow_n;
    };
#if LMX_SLOW_BALANCE
    // the warp's slow vertices of LMX_SLOW_BATCH chunks, dealt round-robin to
    // its lanes: a lane no longer chains up to kVpl of them while its
    // neighbours idle
    uint32_t qn = 0, nb = 0;
    auto drain = [&]() {
        __syncwarp();
        for (uint32_t q = lane; q < qn; q += 32) {
            const uint32_t e = s_slowq[tid >> 5][q];
            slow_one(e & 0x7FFFFFFFu, (e >> 31) ? 0u : kNone);   // 0: an untied candidate word
        }
        __syncwarp();
        qn = 0;
        nb = 0;
    };
#endif
    for (;;) {
        uint32_t i0 = 0;
        if (c < nstat) {
            i0 = c * kChunk;
            c += cstride;
        } else {
            if (lane == 0) i0 = nstat * kChunk + atomicAdd(&a.ctr->pad[1], kChunk);
            i0 = __shfl_sync(0xffffffffu, i0, 0);
        }
        if (i0 >= na) break;
        uint32_t v[kVpl];
        uint2 c[kVpl];
#pragma unroll
        for (int it = 0; it < kVpl; ++it) {
            const uint32_t i = i0 + it * 32 + lane;
            v[it] = i < na ? LMX_LD_STREAM(a.alist + i) : kNone;
        }
#pragma unroll
        for (int it = 0; it < kVpl; ++it) {
            if (FIRST) {   // the first slot {nbr | tie flags, edge id}
                c[it] = v[it] != kNone ? a.cand0[v[it] - a.lo] : make_uint2(kNone, kNone);
            } else {   // the neighbour word alone: {nbr | tied flag, -}
                const uint32_t w = v[it] != kNone ? a.cnbr[v[it] - a.lo] : kNone;
                c[it] = make_uint2(w, 0u);
            }
        }
        bool keep[kVpl];
#pragma unroll
        for (int it = 0; it < kVpl; ++it)
            keep[it] = c[it].x != kNone && !(c[it].x & kTiedFlag) && (FIRST || !bit_set(a.matched, c[it].x));
        uint32_t slow = 0;
#pragma unroll
        for (int it = 0; it < kVpl; ++it) {
            if (v[it] == kNone) continue;
            if (keep[it]) {
                if (FIRST) a.cnbr[v[it] - a.lo] = c[it].x;   // not tied: no flags; the edge is slot ptr = 0
                ++found_n;
                if (DIST && c[it].x - a.lo >= a.nl)   // untied: round 0 carries the edge id, later it sits at ptr
                    propose_record(a, c[it].x,
                                   FIRST ? c[it].y : a.ids[a.vbeg[v[it] - a.lo] + a.ptr[v[it] - a.lo]].y);
            } else {
                slow |= 1u << it;
            }
        }
#if LMX_SLOW_BALANCE
#pragma unroll
        for (int it = 0; it < kVpl; ++it) {
            const bool sl = (slow >> it) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, sl);
            // the vertex and whether its candidate is untied (then known dead: search past ptr)
            if (sl)
                s_slowq[tid >> 5][qn + __popc(bal & lanemask_lt_u32())] =
                    v[it] | ((c[it].x != kNone && !(c[it].x & kTiedFlag)) ? 0x80000000u : 0u);
            qn += __popc(bal);
        }
        if (++nb == LMX_SLOW_BATCH) drain();
#else
        while (slow) {
            const int k = __ffs(slow) - 1;
            slow &= slow - 1;
            uint32_t vk = 0, ck = kNone;
            // (fetching ptr / degree / offset for all vertices up front, before the
            // liveness test, was measured slower: 2.82 -> 2.91 ms per step)
#pragma unroll
            for (int it = 0; it < kVpl; ++it) {
                if (it == k) {
                    vk = v[it];
                    ck = c[it].x;
                }
            }
            slow_one(vk, ck);
        }
#endif
    }
#if LMX_SLOW_BALANCE
    drain();
#endif
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        found_n += __shfl_xor_sync(0xffffffffu, found_n, off);
        reads += __shfl_xor_sync(0xffffffffu, reads, off);
        slow_n += __shfl_xor_sync(0xffffffffu, slow_n, off);
    }
    const int warp = tid >> 5;
    if (lane == 0) {
        s_red[0][warp] = found_n;
        s_red[1][warp] = reads;
        s_red[2][warp] = slow_n;
    }
    __syncthreads();
    if (tid == 0) {
        unsigned long long t0 = 0, t1 = 0, t2 = 0;
        for (int q = 0; q < kWarps; ++q) {
            t0 += s_red[0][q];
            t1 += s_red[1][q];
            t2 += s_red[2][q];
        }
        if (t0) atomicAdd(&a.ctr->live_slots, t0);   // scan loop: candidates found
        if (t1) atomicAdd(&a.ctr->slot_reads, t1);
        if (t2) atomicAdd(&a.ctr->n[0], (unsigned int)t2);   // scan loop: slow-path vertices
    }
}

template <bool FIRST, bool DIST>
__global__ void __launch_bounds__(kBlock, LMX_SCAN_MINB) lmx_scan_round_kernel(ScanArgs a) {
    __shared__ unsigned long long s_red[3][kWarps];
    __shared__ uint32_t s_slowq[LMX_SLOW_BALANCE ? kWarps : 1][32 * kVpl * LMX_SLOW_BATCH];
    probe_body<FIRST, DIST>(a, s_red, s_slowq);
}

struct ScanMatchArgs {
    bool defer_ebits;             // single GPU: edge bits set after the loop (lmx_scan_edge_bits)
    const uint32_t *cnbr, *ckey;
    const uint32_t *ptr;
    const unsigned long long *vbeg;
    const uint2 *ids;
    uint32_t *matched;
    uint32_t *mround;             // round each vertex was matched in (~0 = never)
    long long *mate;
    const uint32_t *oldid;
    const uint32_t *alist;        // A_r
    uint32_t *anext;              // A_{r+1}
    uint32_t *ebits;
    RoundCtr *ctr;
    RoundCtr *ctr_next;
    int round;
    uint32_t lo, nl;              // owned id range (single GPU: [0, n)); per-vertex arrays are local
    uint32_t *remote_ok;          // [nl] cross-partition matches confirmed by exchange A
};

template <int kItems>
__device__ __forceinline__ void match_body(const ScanMatchArgs &a, uint32_t (&s_cnt)[kWarps], uint32_t &s_base) {
    const uint32_t total = a.ctr->pad[0];
    if (total == 0) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t lt = lanemask_lt_u32();
    unsigned long long matched_v = 0;
    const uint32_t tile = kBlock * kItems;
    for (uint32_t t0 = blockIdx.x * tile; t0 < total; t0 += gridDim.x * tile) {
        uint32_t vv[kItems];
        bool keep[kItems];
        uint32_t wc = 0;
        // staged gathers: list entries, then candidates, then the partners'
        // keys, each stage for all items at once (their latencies overlap)
        uint32_t cc[kItems];
        uint32_t px[kItems];
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t i = t0 + j * kBlock + tid;
            vv[j] = i < total ? LMX_LD_STREAM(a.alist + i) : kNone;
        }
#pragma unroll
        for (int j = 0; j < kItems; ++j) cc[j] = vv[j] != kNone ? a.cnbr[vv[j] - a.lo] : kNone;
        // mutual iff the partner's candidate neighbour is v: both are edges
        // between v and x that are maximal at both ends, hence the same edge
        // (also with parallel edges), so the 4-byte neighbour array suffices
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t x = cc[j] != kNone ? (cc[j] & kNbrMask) : kNone;
            px[j] = (x != kNone && x - a.lo < a.nl) ? (a.cnbr[x - a.lo] & kNbrMask) : kNone;
        }
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t v = vv[j];
            bool k = false;
            if (v != kNone) {
                const uint32_t x = cc[j] != kNone ? (cc[j] & kNbrMask) : kNone;
                if (x != kNone) {
                    bool mutual;
                    if (x - a.lo < a.nl) {
                        mutual = px[j] == v;
                    } else {   // partner on another partition: its owner confirmed the edge (exchange A)
                        mutual = a.remote_ok[v - a.lo] != 0;
                        if (mutual) a.remote_ok[v - a.lo] = 0;
                    }
                    if (mutual) {
                        atomicOr(a.matched + (v >> 5), 1u << (v & 31));
                        a.mround[v] = (uint32_t)a.round;
                        if (a.oldid) a.mate[a.oldid[v]] = (long long)a.oldid[x];
                        else a.mate[v] = (long long)x;
                        ++matched_v;
                        if (!a.defer_ebits && v < x) {   // the lower endpoint records the edge (graph.py:195-203)
                            const uint32_t e = cand_eid(v - a.lo, cc[j], a.ckey, a.ptr, a.vbeg, a.ids);
                            atomicOr(a.ebits + (e >> 5), 1u << (e & 31));
                        }
                    } else {
                        k = true;   // stays active
                    }
                }
            }
            keep[j] = k;
            wc += __popc(__ballot_sync(0xffffffffu, k));
        }
        if (lane == 0) s_cnt[warp] = wc;
        __syncthreads();
        if (tid == 0) {
            uint32_t sum = 0;
            for (int w = 0; w < kWarps; ++w) sum += s_cnt[w];
            s_base = sum ? atomicAdd(&a.ctr_next->pad[0], sum) : 0u;
        }
        __syncthreads();
        uint32_t pos = s_base;
        for (int w = 0; w < warp; ++w) pos += s_cnt[w];
#pragma unroll
        for (int j = 0; j < kItems; ++j) {
            const uint32_t bal = __ballot_sync(0xffffffffu, keep[j]);
            if (keep[j]) LMX_ST_STREAM(a.anext + pos + __popc(bal & lt), vv[j]);
            pos += __popc(bal);
        }
        __syncthreads();
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) matched_v += __shfl_xor_sync(0xffffffffu, matched_v, off);
    if (lane == 0 && matched_v) atomicAdd(&a.ctr->matched_v, matched_v);
}

__global__ void __launch_bounds__(kBlock, LMX_SCAN_MATCH_MINB) lmx_scan_match_kernel(ScanMatchArgs a) {
    __shared__ uint32_t s_cnt[kWarps];
    __shared__ uint32_t s_base;
    match_body<LMX_SCAN_MATCH_ITEMS>(a, s_cnt, s_base);
}

// ---- the whole round loop in one persistent cooperative kernel -------------
// Rounds r0 .. r_end-1 of probe -> grid barrier -> match -> grid barrier,
// ending at the first round that finds no candidate (matchers.py:87-90).
// One launch per matching instead of two per round: no launch gaps, no
// per-kernel tails, no host round trip to learn the round count (the death
// histogram reads it from `result`).  Block 0 stamps %globaltimer after each
// barrier, so the per-round probe / match times come out of the same launch.
#ifndef LMX_LOOP_MINB
#define LMX_LOOP_MINB 4
#endif
#ifndef LMX_LOOP_MATCH_ITEMS
#define LMX_LOOP_MATCH_ITEMS 8
#endif

struct LoopArgs {
    ScanArgs p;               // probe arguments (alist, ctr, rs set per round)
    ScanMatchArgs mt;         // match arguments (lists, ctr, round set per round)
    const uint32_t *bins0;    // A_0
    uint32_t *lists[2];       // A_r ping-pong
    RoundCtr *ctr;
    uint64_t seed_mix;        // mix64(seed), tiebreak.py:40-52
    int rerandomize;
    int r0, r_end;
    uint32_t *result;         // [0]: the round count (r_end if not reached)
    unsigned long long *stamps;   // [2 r_end + 1]: globaltimer at round start / after probe / after match
};

__device__ __forceinline__ unsigned long long globaltimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(kBlock, LMX_LOOP_MINB) lmx_scan_loop_kernel(LoopArgs L) {
    __shared__ unsigned long long s_red[3][kWarps];
    __shared__ uint32_t s_cnt[kWarps];
    __shared__ uint32_t s_base;
    __shared__ uint32_t s_slowq[LMX_SLOW_BALANCE ? kWarps : 1][32 * kVpl * LMX_SLOW_BATCH];
    cooperative_groups::grid_group grid = cooperative_groups::this_grid();
    const bool stamp = L.stamps && blockIdx.x == 0 && threadIdx.x == 0;
    int r = L.r0;
    if (stamp) L.stamps[2 * r] = globaltimer();
    for (; r < L.r_end; ++r) {
        ScanArgs a = L.p;
        a.alist = r == 0 ? L.bins0 : L.lists[r & 1];
        a.ctr = L.ctr + r;
        a.rs = mix64(L.seed_mix ^ (L.rerandomize ? (uint64_t)r : 0ULL));
        if (r == 0) probe_body<true, false>(a, s_red, s_slowq);
        else probe_body<false, false>(a, s_red, s_slowq);
        grid.sync();
        if (stamp) L.stamps[2 * r + 1] = globaltimer();
        if (L.ctr[r].live_slots == 0) break;   // no candidate anywhere: m_r = 0
        ScanMatchArgs ma = L.mt;
        ma.alist = a.alist;
        ma.anext = L.lists[(r + 1) & 1];
        ma.ctr = L.ctr + r;
        ma.ctr_next = L.ctr + r + 1;
        ma.round = r;
        match_body<LMX_LOOP_MATCH_ITEMS>(ma, s_cnt, s_base);
        grid.sync();
        if (stamp) L.stamps[2 * r + 2] = globaltimer();
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *L.result = (uint32_t)r;
}

// Matched-edge bits after the loop (graph.py:195-203: the lower endpoint
// records its edge).  A matched vertex is never probed again, so its
// candidate word and ptr still name its matched edge.  Done here rather than
// in the match kernel, whose tiles would otherwise wait on the key's
// dependent gathers (ptr -> offset -> slot) for their few matched vertices.
#ifndef LMX_EDGE_ITEMS
#define LMX_EDGE_ITEMS 4
#endif
__global__ void lmx_scan_edge_bits(const uint32_t *matched, unsigned long long lo, unsigned long long n,
                                   const uint32_t *cnbr,
                                   const uint32_t *ckey, const uint32_t *ptr, const unsigned long long *vbeg,
                                   const uint2 *ids, uint32_t *ebits) {
    // thread per vertex, LMX_EDGE_ITEMS vertices per thread per step with each
    // stage of the gather chain (word; ptr + offset; slot or key; edge id)
    // issued for all of them at once, so their latencies overlap
    constexpr int K = LMX_EDGE_ITEMS;
    // vertices [lo, n): the owned range (single GPU: all of them)
    const unsigned long long tile = (unsigned long long)blockDim.x * K;
    for (unsigned long long t0 = lo + (unsigned long long)blockIdx.x * tile; t0 < n;
         t0 += (unsigned long long)gridDim.x * tile) {
        uint32_t w[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const unsigned long long v = t0 + (unsigned long long)j * blockDim.x + threadIdx.x;
            w[j] = (v < n && ((matched[v >> 5] >> (v & 31)) & 1u)) ? cnbr[v - lo] : kNone;
        }
        uint32_t eid[K];
#pragma unroll
        for (int j = 0; j < K; ++j) {
            const uint32_t v = (uint32_t)(t0 + (unsigned long long)j * blockDim.x + threadIdx.x);
            eid[j] = kNone;
            if (w[j] != kNone && v < (w[j] & kNbrMask)) eid[j] = cand_eid((uint32_t)(v - lo), w[j], ckey, ptr, vbeg, ids);
        }
#pragma unroll
        for (int j = 0; j < K; ++j)
            if (eid[j] != kNone) atomicOr(ebits + (eid[j] >> 5), 1u << (eid[j] & 31));
    }
}

// Death-round histogram: every edge once; it dies in round min(mround[v],
// mround[u]).  Bins: [0, R) rounds, R = outlived the loop (must stay empty).
// Most edges die in the first rounds: those bins count in registers.

// mround packed for the histogram's random lookups (BITS = 4 or 8: small
// enough to stay in L2; values saturate at the top value)
template <int BITS>
__global__ void lmx_pack_mround(const uint32_t *mround, unsigned long long n, uint32_t *packed) {
    constexpr uint32_t kPer = 32 / BITS, kTop = (1u << BITS) - 1;
    const unsigned long long words = (n + kPer - 1) / kPer;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
        uint32_t x = 0;
#pragma unroll
        for (uint32_t j = 0; j < kPer; ++j) {
            const unsigned long long v = w * kPer + j;
            const uint32_t r = v < n ? min(mround[v], kTop) : kTop;
            x |= r << (j * BITS);
        }
        packed[w] = x;
    }
}

// The packed width is chosen so that every round of this run fits below the
// top value (R < 2^BITS - 1): the top value means "never matched", exactly.
template <int BITS>
__device__ __forceinline__ uint32_t mround_of(const uint32_t *mround, const uint32_t *packed, uint32_t v) {
    if (BITS == 32) return __ldg(mround + v);
    constexpr uint32_t kPer = 32 / BITS, kTop = (1u << BITS) - 1;
    return (__ldg(packed + v / kPer) >> ((v % kPer) * BITS)) & kTop;
}

// Per-thread counters of the first 4 * NACC bins: 16-bit fields in u64
// registers (a thread sees far fewer than 2^16 edges); the rest use atomics.
template <int NACC>
struct HistAcc {
    unsigned long long a[4] = {0, 0, 0, 0};
    __device__ __forceinline__ void add(uint32_t d, uint32_t *s_hist, unsigned long long *hist) {
        const unsigned long long inc = 1ULL << ((d & 3u) * 16u);
        if (d < 4u) a[0] += inc;
        else if (d < 8u) a[1] += inc;
        else if (NACC > 2 && d < 12u) a[2] += inc;
        else if (NACC > 2 && d < 16u) a[3] += inc;
        else if (d < (uint32_t)kHistBins) atomicAdd(&s_hist[d], 1u);
        else atomicAdd(hist + d, 1ULL);
    }
    __device__ __forceinline__ void flush(uint32_t *s_hist) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) {
#pragma unroll
            for (int f = 0; f < 4; ++f) {
                uint32_t x = (uint32_t)((a[k] >> (16 * f)) & 0xFFFFULL);
                for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
                if ((threadIdx.x & 31) == 0 && x) atomicAdd(&s_hist[4 * k + f], x);
            }
        }
    }
};

// lowpair = {v, u} per edge, u < v, grouped by v: the v lookups walk mround
// in order (cache lines reused), the u lookups go to the lower ids -- the
// high-degree end after relabelling.  A flat, coalesced pass, 4 edges per
// thread in flight.
// Used for the u32 rounds (>= 255 rounds); the packed widths use the
// persistent, pipelined lmx_scan_hist_hub_kernel below.  (A low-CSR variant
// -- 4 B per edge, owners rebuilt per tile in shared memory -- moved half the
// bytes but ran 3.1 ms against 2.2: its dependent loads per tile cost more
// than the stream it saved.)
template <int BITS>
__global__ void __launch_bounds__(kBlock) lmx_scan_hist_kernel(const uint2 *lowpair, unsigned long long m,
                                                             const uint32_t *mround, const uint32_t *packed,
                                                             unsigned long long n, uint32_t R,
                                                             unsigned long long *hist) {
    __shared__ uint32_t s_hist[kHistBins];
    const int tid = threadIdx.x;
    for (int i = tid; i < kHistBins; i += kBlock) s_hist[i] = 0;
    __syncthreads();
    HistAcc<BITS == 4 ? 4 : 2> acc;
    const uint4 *q = reinterpret_cast<const uint4 *>(lowpair);
    const uint32_t nq = (uint32_t)(m / 2);   // m < 2^32
    const uint32_t stride = gridDim.x * kBlock;
    constexpr int HU = LMX_HIST_U;   // edge pairs (uint4) per thread per step
    for (uint32_t i = blockIdx.x * kBlock + tid; i < nq; i += HU * stride) {
        uint4 x[HU];
#pragma unroll
        for (int j = 0; j < HU; ++j) x[j] = i + j * stride < nq ? __ldcs(q + i + j * stride) : make_uint4(0, 0, 0, 0);
        uint32_t d[2 * HU];
#pragma unroll
        for (int j = 0; j < HU; ++j) {
            d[2 * j] = min(min(mround_of<BITS>(mround, packed, x[j].x), mround_of<BITS>(mround, packed, x[j].y)), R);
            d[2 * j + 1] =
                min(min(mround_of<BITS>(mround, packed, x[j].z), mround_of<BITS>(mround, packed, x[j].w)), R);
        }
#pragma unroll
        for (int j = 0; j < HU; ++j) {
            if (i + j * stride < nq) {
                acc.add(d[2 * j], s_hist, hist);
                acc.add(d[2 * j + 1], s_hist, hist);
            }
        }
    }
    if ((m & 1ULL) && blockIdx.x == 0 && tid == 0) {
        const uint2 x = lowpair[m - 1];
        acc.add(min(min(mround_of<BITS>(mround, packed, x.x), mround_of<BITS>(mround, packed, x.y)), R), s_hist,
                hist);
    }
    acc.flush(s_hist);
    __syncthreads();
    for (int i = tid; i < kHistBins; i += kBlock)
        if (s_hist[i]) atomicAdd(hist + i, (unsigned long long)s_hist[i]);
}

#ifndef LMX_HIST_HUB_KB
#define LMX_HIST_HUB_KB 80   // packed match rounds of the lowest ids staged in shared memory
#endif
#ifndef LMX_HIST_THREADS
#define LMX_HIST_THREADS 1024
#endif
constexpr int kHistThreads = LMX_HIST_THREADS;

// The same pass, persistent (two 1024-thread blocks per SM) and software-
// pipelined: the next step's edge pairs are loaded before this step's
// lookups, so the stream's DRAM latency overlaps the lookups.  The packed
// rounds of the lowest `hw` words -- the highest-degree vertices after
// relabelling, the target of most u lookups -- are staged once per block in
// shared memory; L1 and L2 serve the rest.
template <int BITS>
__global__ void __launch_bounds__(kHistThreads, 2)
    lmx_scan_hist_hub_kernel(const uint2 *lowpair, unsigned long long m, const uint32_t *packed, uint32_t R,
                             const uint32_t *R_dev, uint32_t hw, unsigned long long *hist) {
    if (R_dev) R = *R_dev;   // speculative batch: the round count is found on the device
    extern __shared__ uint32_t s_dyn[];
    uint32_t *s_hist = s_dyn;
    uint32_t *s_pk = s_dyn + kHistBins;
    constexpr uint32_t kPer = 32 / BITS, kTop = (1u << BITS) - 1;
    const int tid = threadIdx.x;
    for (int i = tid; i < kHistBins; i += kHistThreads) s_hist[i] = 0;
    for (uint32_t i = tid; i < hw; i += kHistThreads) s_pk[i] = __ldg(packed + i);
    __syncthreads();
    auto rnd = [&](uint32_t v) -> uint32_t {
        const uint32_t w = v / kPer;
        const uint32_t x = w < hw ? s_pk[w] : __ldg(packed + w);
        return (x >> ((v % kPer) * BITS)) & kTop;
    };
#if LMX_HIST_V_GLOBAL
    // the higher end v: rarely a hub, and consecutive pairs share its word
    // (lowpair is grouped by v), so L1 serves it without the hub test
    auto rnd_v = [&](uint32_t v) -> uint32_t { return (__ldg(packed + v / kPer) >> ((v % kPer) * BITS)) & kTop; };
#else
    auto rnd_v = rnd;
#endif
    HistAcc<BITS == 4 ? 4 : 2> acc;
    const uint4 *q = reinterpret_cast<const uint4 *>(lowpair);
    const uint32_t nq = (uint32_t)(m / 2);
    const uint32_t stride = gridDim.x * kHistThreads;
    uint32_t i = blockIdx.x * kHistThreads + tid;
    uint4 xn = i < nq ? __ldcs(q + i) : make_uint4(0, 0, 0, 0);
#if LMX_HIST_PF2
    // two steps of the stream in flight
    uint4 xn2 = i + stride < nq ? __ldcs(q + i + stride) : make_uint4(0, 0, 0, 0);
    for (; i < nq; i += stride) {
        const uint4 x = xn;
        xn = xn2;
        if (i + 2 * stride < nq) xn2 = __ldcs(q + i + 2 * stride);
#else
    for (; i < nq; i += stride) {
        const uint4 x = xn;
        if (i + stride < nq) xn = __ldcs(q + i + stride);
#endif
        const uint32_t d0 = min(min(rnd_v(x.x), rnd(x.y)), R);
        const uint32_t d1 = min(min(rnd_v(x.z), rnd(x.w)), R);
        acc.add(d0, s_hist, hist);
        acc.add(d1, s_hist, hist);
    }
    if ((m & 1ULL) && blockIdx.x == 0 && tid == 0) {
        const uint2 x = lowpair[m - 1];
        acc.add(min(min(rnd(x.x), rnd(x.y)), R), s_hist, hist);
    }
    acc.flush(s_hist);
    __syncthreads();
    for (int i2 = tid; i2 < kHistBins; i2 += kHistThreads)
        if (s_hist[i2]) atomicAdd(hist + i2, (unsigned long long)s_hist[i2]);
}

}  // namespace lmx

using namespace lmx;

template <int BITS>
static int hist_hub_launch(lmx_ctx *ctx, unsigned long long mm, uint32_t R, const uint32_t *R_dev) {
    const unsigned long long nn = (unsigned long long)ctx->n;
    constexpr uint32_t kPer = 32 / BITS;
    const unsigned long long words = (nn + kPer - 1) / kPer;
    const uint32_t cap = (uint32_t)(LMX_HIST_HUB_KB * 1024 / 4) - kHistBins;
    const uint32_t hw = (uint32_t)std::min<unsigned long long>(words, cap);
    const size_t smem = (size_t)(kHistBins + hw) * 4;
    LMX_CUDA(ctx, cudaFuncSetAttribute(lmx_scan_hist_hub_kernel<BITS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)(LMX_HIST_HUB_KB * 1024)));
    lmx_scan_hist_hub_kernel<BITS><<<ctx->num_sms * 2, kHistThreads, smem, ctx->stream>>>(ctx->lowpair, mm,
                                                                                          ctx->mpacked, R, R_dev,
                                                                                          hw, ctx->hist);
    return LMX_OK;
}

int lmx_scan_configure_grids(lmx_ctx *ctx) {
    int occ0 = 0, occ1 = 0, occm = 0, occl = 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occl, lmx_scan_loop_kernel, kBlock, 0));
    int coop = 0;
    LMX_CUDA(ctx, cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device));
    ctx->scan_loop_grid = coop ? ctx->num_sms * std::max(occl, 1) : 0;
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ0, lmx_scan_round_kernel<true, false>, kBlock, 0));
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, lmx_scan_round_kernel<false, false>, kBlock, 0));
    LMX_CUDA(ctx, cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occm, lmx_scan_match_kernel, kBlock, 0));
    ctx->scan_grid[0] = ctx->num_sms * std::max(occ0, 1);
    ctx->scan_grid[1] = ctx->num_sms * std::max(occ1, 1);
    ctx->scan_match_grid = ctx->num_sms * std::max(occm, 1);
    return LMX_OK;
}

// Per-match state: counters, outputs, bitmap, match rounds, pointers; round 0's
// list is A_0 = bins0.
static int scan_begin(lmx_ctx *ctx) {
    const size_t n = (size_t)ctx->n;
    cudaStream_t st = ctx->stream;
    LMX_TRY(lmx_ensure_ctr(ctx, 64));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ctr, 0, sizeof(RoundCtr) * (size_t)ctx->ctr_cap, st));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ebits, 0, ((size_t)std::max<int64_t>(ctx->m, 1) + 31) / 32 * 4, st));
    if (n) {
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mate_target, 0xFF, n * 8, st));   // -1
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->matched, 0, (n + 31) / 32 * 4, st));
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mround, 0xFF, n * 4, st));
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->vdeg, 0, (size_t)std::max<int64_t>(ctx->n_local, 1) * 4, st));
    }
    ctx->ctr_host[0] = RoundCtr{};
    ctx->ctr_host[0].pad[0] = ctx->n_bins0[0];
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr, ctx->ctr_host, sizeof(RoundCtr), cudaMemcpyHostToDevice, st));
    return LMX_OK;
}

// Round r's candidate probe over A_r.
// dist: the stepped multi-GPU protocol (records appended to ctx->send;
// lmx_scan_dist_round sets up the buffers and zeroes the counts first).
static int scan_enqueue_probe(lmx_ctx *ctx, int r, uint64_t seed_masked, bool rerandomize, bool dist = false) {
    ScanArgs a = {};
    a.vbeg = ctx->vbeg;
    a.ptr = ctx->vdeg;
    a.cnbr = reinterpret_cast<uint32_t *>(ctx->cand);
    a.ckey = reinterpret_cast<uint32_t *>(ctx->cand) + std::max<int64_t>(ctx->n_local, 1);
    a.cand0 = ctx->cand0;
    a.ids = ctx->ids0;
    a.matched = ctx->matched;
    a.alist = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
    a.ctr = ctx->ctr + r;
    a.rs = round_seed(seed_masked, (uint64_t)r, rerandomize);
    a.lo = (uint32_t)ctx->lo;
    a.nl = (uint32_t)ctx->n_local;
    if (dist) {
        a.bounds = reinterpret_cast<const unsigned long long *>(reinterpret_cast<const char *>(ctx->send_cnt) + 1024);
        a.p = ctx->dist_p;
        a.cnt = ctx->send_cnt;
        a.region = ctx->send;
        if (r == 0) lmx_scan_round_kernel<true, true><<<ctx->scan_grid[0], kBlock, 0, ctx->stream>>>(a);
        else lmx_scan_round_kernel<false, true><<<ctx->scan_grid[1], kBlock, 0, ctx->stream>>>(a);
    } else {
        if (r == 0) lmx_scan_round_kernel<true, false><<<ctx->scan_grid[0], kBlock, 0, ctx->stream>>>(a);
        else lmx_scan_round_kernel<false, false><<<ctx->scan_grid[1], kBlock, 0, ctx->stream>>>(a);
    }
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

// Round r's match kernel over A_r; appends A_{r+1}.
// defer_ebits: the matched-edge bits are set after the loop
// (lmx_scan_edge_bits; the stepped multi-GPU protocol does it in
// lmx_scan_dist_hist) rather than per matched vertex here.
static int scan_enqueue_match(lmx_ctx *ctx, int r, bool defer_ebits) {
    ScanMatchArgs ma;
    ma.cnbr = reinterpret_cast<const uint32_t *>(ctx->cand);
    ma.ckey = reinterpret_cast<const uint32_t *>(ctx->cand) + std::max<int64_t>(ctx->n_local, 1);
    ma.ptr = ctx->vdeg;
    ma.vbeg = ctx->vbeg;
    ma.ids = ctx->ids0;
    ma.defer_ebits = defer_ebits;
    ma.matched = ctx->matched;
    ma.mround = ctx->mround;
    ma.mate = ctx->mate_target;
    ma.oldid = ctx->relabeled ? ctx->oldid : nullptr;
    ma.alist = r == 0 ? ctx->bins0 : ctx->lists[r & 1];
    ma.anext = ctx->lists[(r + 1) & 1];
    ma.ebits = ctx->ebits;
    ma.ctr = ctx->ctr + r;
    ma.ctr_next = ctx->ctr + r + 1;
    ma.round = r;
    ma.lo = (uint32_t)ctx->lo;
    ma.nl = (uint32_t)ctx->n_local;
    ma.remote_ok = ctx->remote_ok;
    lmx_scan_match_kernel<<<ctx->scan_match_grid, kBlock, 0, ctx->stream>>>(ma);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

// The round count of a speculative batch of k rounds, on the device: the
// first round that found no candidate (k if none did).  Stored after the bins.
__global__ void lmx_find_rounds(const RoundCtr *ctr, int k, uint32_t *out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        uint32_t r = (uint32_t)k;
        for (int i = 0; i < k; ++i)
            if (ctr[i].live_slots == 0) {
                r = (uint32_t)i;
                break;
            }
        *out = r;
    }
}

// Death-round histogram of this context's lowpair (all edges; a partition's
// share when p > 1) into ctx->hist, bins [0, n_rounds] (max(., 256) of them).
// spec_k > 0: a speculative batch of spec_k <= 14 rounds whose end is not
// known on the host yet; the count is found on the device (n_rounds unused).
static int scan_hist_launch(lmx_ctx *ctx, int n_rounds, int spec_k = 0) {
    cudaStream_t st = ctx->stream;
    const size_t nbins = std::max<size_t>((size_t)n_rounds + 1, kHistBins);
    if (ctx->hist_cap < nbins) {
        lmx_free(ctx, (void **)&ctx->hist, (ctx->hist_cap + 1) * 8);
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->hist, (nbins + 1) * 8, "death histogram"));
        ctx->hist_cap = nbins;
    }
    if (spec_k > 0) {
        uint32_t *R_dev = reinterpret_cast<uint32_t *>(ctx->hist + ctx->hist_cap);
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->hist, 0, nbins * 8, st));
        lmx_find_rounds<<<1, 32, 0, st>>>(ctx->ctr, spec_k, R_dev);
        if (ctx->lowpair_n == 0) return LMX_OK;
        lmx_pack_mround<4><<<ctx->num_sms * 8, kBlock, 0, st>>>(ctx->mround, (unsigned long long)ctx->n, ctx->mpacked);
        LMX_TRY(hist_hub_launch<4>(ctx, ctx->lowpair_n, 0u, R_dev));
        LMX_CUDA(ctx, cudaGetLastError());
        ctx->timing.round_launches += 3;
        return LMX_OK;
    }
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->hist, 0, nbins * 8, st));
    const int grid = ctx->num_sms * 8;
    const unsigned long long nn = (unsigned long long)ctx->n, mm = ctx->lowpair_n;
    const uint32_t R = (uint32_t)n_rounds;
    if (mm == 0) return LMX_OK;
    if (n_rounds < 15) {
        lmx_pack_mround<4><<<grid, kBlock, 0, st>>>(ctx->mround, nn, ctx->mpacked);
        LMX_TRY(hist_hub_launch<4>(ctx, mm, R, nullptr));
    } else if (n_rounds < 255) {
        lmx_pack_mround<8><<<grid, kBlock, 0, st>>>(ctx->mround, nn, ctx->mpacked);
        LMX_TRY(hist_hub_launch<8>(ctx, mm, R, nullptr));
    } else {
        lmx_scan_hist_kernel<32><<<grid, kBlock, 0, st>>>(ctx->lowpair, mm, ctx->mround, ctx->mpacked, nn, R,
                                                         ctx->hist);
    }
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += n_rounds < 255 ? 2 : 1;
    return LMX_OK;
}

// Matched-edge bits of the vertices [lo, hi) (single GPU: all; a partition:
// its owned range, whose lower endpoints record their edges).
static int scan_edge_bits_launch(lmx_ctx *ctx, unsigned long long lo, unsigned long long hi) {
    if (hi <= lo) return LMX_OK;
    const unsigned long long blocks = std::min<unsigned long long>((hi - lo + kBlock - 1) / kBlock,
                                                                   (unsigned long long)ctx->num_sms * 32);
    lmx_scan_edge_bits<<<(unsigned)blocks, kBlock, 0, ctx->stream>>>(
        ctx->matched, lo, hi, reinterpret_cast<const uint32_t *>(ctx->cand),
        reinterpret_cast<const uint32_t *>(ctx->cand) + std::max<int64_t>(ctx->n_local, 1), ctx->vdeg, ctx->vbeg,
        ctx->ids0, ctx->ebits);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

// Device histogram for a round count held on the device (R_dev): 4-bit
// packed match rounds, which are exact for R < 15 (the caller reruns with the
// right width once it knows R).
static int scan_hist_launch_dev(lmx_ctx *ctx, const uint32_t *R_dev) {
    cudaStream_t st = ctx->stream;
    const size_t nbins = kHistBins;
    if (ctx->hist_cap < nbins) {
        lmx_free(ctx, (void **)&ctx->hist, (ctx->hist_cap + 1) * 8);
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->hist, (nbins + 1) * 8, "death histogram"));
        ctx->hist_cap = nbins;
    }
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->hist, 0, nbins * 8, st));
    if (ctx->lowpair_n == 0) return LMX_OK;
    lmx_pack_mround<4><<<ctx->num_sms * 8, kBlock, 0, st>>>(ctx->mround, (unsigned long long)ctx->n, ctx->mpacked);
    LMX_TRY(hist_hub_launch<4>(ctx, ctx->lowpair_n, 0u, R_dev));
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 2;
    return LMX_OK;
}

// The persistent round loop (lmx_scan_loop_kernel): one cooperative launch
// for all rounds, then the histogram and the matched-edge bits, one
// synchronisation.  Diagnostics (per-round probe / match times) come from the
// kernel's globaltimer stamps.
static int run_rounds_loop(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                           std::vector<lmx_round_stats> &stats, unsigned long long &n_matched) {
    cudaStream_t st = ctx->stream;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    LMX_TRY(scan_begin(ctx));
    int r0 = 0, n_rounds = -1;
    std::vector<unsigned long long> hist;
    uint32_t R = 0;
    while (n_rounds < 0) {
        const int r_end = ctx->ctr_cap - 2;
        uint32_t *result = ctx->loop_aux;   // (reallocated when the counters grow)
        unsigned long long *stamps = reinterpret_cast<unsigned long long *>(ctx->loop_aux + 2);
        LoopArgs L;
        L.p = ScanArgs{};
        L.p.vbeg = ctx->vbeg;
        L.p.ptr = ctx->vdeg;
        L.p.cnbr = reinterpret_cast<uint32_t *>(ctx->cand);
        L.p.ckey = reinterpret_cast<uint32_t *>(ctx->cand) + std::max<int64_t>(ctx->n_local, 1);
        L.p.cand0 = ctx->cand0;
        L.p.ids = ctx->ids0;
        L.p.matched = ctx->matched;
        L.p.lo = (uint32_t)ctx->lo;
        L.p.nl = (uint32_t)ctx->n_local;
        L.mt.defer_ebits = true;
        L.mt.cnbr = L.p.cnbr;
        L.mt.ckey = L.p.ckey;
        L.mt.ptr = ctx->vdeg;
        L.mt.vbeg = ctx->vbeg;
        L.mt.ids = ctx->ids0;
        L.mt.matched = ctx->matched;
        L.mt.mround = ctx->mround;
        L.mt.mate = ctx->mate_target;
        L.mt.oldid = ctx->relabeled ? ctx->oldid : nullptr;
        L.mt.ebits = ctx->ebits;
        L.mt.lo = (uint32_t)ctx->lo;
        L.mt.nl = (uint32_t)ctx->n_local;
        L.mt.remote_ok = ctx->remote_ok;
        L.bins0 = ctx->bins0;
        L.lists[0] = ctx->lists[0];
        L.lists[1] = ctx->lists[1];
        L.ctr = ctx->ctr;
        L.seed_mix = mix64(seed_masked);
        L.rerandomize = rerandomize ? 1 : 0;
        L.r0 = r0;
        L.r_end = r_end;
        L.result = result;
        L.stamps = stamps;
        void *args[] = {&L};
        // The hub end of the candidate words (relabelled: low device ids) is the
        // match phase's most frequent random gather; an L2 access-policy window
        // keeps its first 24 MB resident (RMAT-26: 6.56 -> 6.49 ms per matching;
        // 32 MB and more start to evict the histogram's tables,
        // profiles/r2_l2_persist_rmat26.txt).  LMX_L2_PERSIST_MB=0 turns it off.
        static const long persist_mb = getenv("LMX_L2_PERSIST_MB") ? atol(getenv("LMX_L2_PERSIST_MB")) : 24;
        static int persist_ok = -1;   // the persisting-L2 limit: not yet set / refused / set
        const size_t want = std::min<size_t>((size_t)std::max(persist_mb, 0L) << 20, (size_t)ctx->n_local * 4);
        if (persist_ok == -1 && persist_mb > 0) {
            persist_ok = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_mb << 20) == cudaSuccess;
            cudaGetLastError();
        }
        if (persist_ok == 1 && want > 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(ctx->scan_loop_grid);
            cfg.blockDim = dim3(kBlock);
            cfg.stream = st;
            cudaLaunchAttribute at[2];
            at[0].id = cudaLaunchAttributeCooperative;
            at[0].val.cooperative = 1;
            at[1].id = cudaLaunchAttributeAccessPolicyWindow;
            at[1].val.accessPolicyWindow.base_ptr = ctx->cand;
            at[1].val.accessPolicyWindow.num_bytes = want;
            at[1].val.accessPolicyWindow.hitRatio = 1.0f;
            at[1].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
            at[1].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
            cfg.attrs = at;
            cfg.numAttrs = 2;
            LMX_CUDA(ctx, cudaLaunchKernelEx(&cfg, lmx_scan_loop_kernel, L));
        } else {
            LMX_CUDA(ctx, cudaLaunchCooperativeKernel((const void *)lmx_scan_loop_kernel, dim3(ctx->scan_loop_grid),
                                                      dim3(kBlock), args, 0, st));
        }
        ctx->timing.round_launches += 1;
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev2, st));
        // the matched-edge bits and the death-round histogram are independent:
        // the edge bits run on a side stream next to the histogram
        static const bool serial_tail = getenv("LMX_SERIAL_TAIL") != nullptr;
        if (!serial_tail && !ctx->side_stream) {
            LMX_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->side_stream, cudaStreamNonBlocking));
            LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_side, cudaEventDisableTiming));
            LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_mate, cudaEventDisableTiming));
        }
        if (!serial_tail) {
            LMX_CUDA(ctx, cudaStreamWaitEvent(ctx->side_stream, ctx->ev2, 0));
            cudaStream_t keep = ctx->stream;
            ctx->stream = ctx->side_stream;
            const int rc_eb = scan_edge_bits_launch(ctx, 0, (unsigned long long)ctx->n);
            ctx->stream = keep;
            LMX_TRY(rc_eb);
            LMX_CUDA(ctx, cudaEventRecord(ctx->ev_side, ctx->side_stream));
            if (ctx->mate_early && ctx->mate_target == ctx->mate) {   // final once the loop kernel is done
                LMX_CUDA(ctx, cudaMemcpyAsync(ctx->mate_early, ctx->mate_target, (size_t)ctx->n * 8,
                                              cudaMemcpyDeviceToHost, ctx->side_stream));
                LMX_CUDA(ctx, cudaEventRecord(ctx->ev_mate, ctx->side_stream));
                ctx->mate_early_done = true;
            }
        }
        LMX_TRY(scan_hist_launch_dev(ctx, result));
        if (serial_tail) LMX_TRY(scan_edge_bits_launch(ctx, 0, (unsigned long long)ctx->n));
        else LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_side, 0));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));   // the device loop ends here (an early mate copy may go on)
        hist.assign(kHistBins, 0);
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host, ctx->ctr, sizeof(RoundCtr) * (size_t)ctx->ctr_cap,
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->loop_host, ctx->loop_aux, lmx_loop_aux_bytes(ctx->ctr_cap),
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaMemcpyAsync(hist.data(), ctx->hist, kHistBins * 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        R = ctx->loop_host[0];
        if ((int)R < r_end) {
            n_rounds = (int)R;
        } else {   // more rounds than the counters hold: grow them and continue
            r0 = (int)R;
            if (ctx->mate_early_done) LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_mate, 0));   // (copied again later)
            LMX_TRY(lmx_ensure_ctr(ctx, 2 * ctx->ctr_cap));
        }
    }
    if (n_rounds >= 15) {   // the 4-bit histogram saturated: recount at the right width
        LMX_TRY(scan_hist_launch(ctx, n_rounds));
        const size_t nbins = std::max<size_t>((size_t)n_rounds + 1, kHistBins);
        hist.assign(nbins, 0);
        LMX_CUDA(ctx, cudaMemcpyAsync(hist.data(), ctx->hist, nbins * 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
    }
    ctx->scan_last_rounds = n_rounds;
    ctx->timing.rounds_executed = n_rounds + (n_rounds < ctx->ctr_cap ? 1 : 0);
    // per-round times from the stamps (ns): probe r = [2r, 2r+1], match r = [2r+1, 2r+2]
    ctx->kernel_ms.clear();
    ctx->timing.round_kernel_ms = ctx->timing.match_kernel_ms = 0;
    const unsigned long long *hs = reinterpret_cast<const unsigned long long *>(ctx->loop_host + 2);
    for (int r = r0 == 0 ? 0 : r0; r <= n_rounds && r < ctx->ctr_cap - 2; ++r) {
        const float pm = (float)((double)(hs[2 * r + 1] - hs[2 * r]) * 1e-6);
        const float mm = r < n_rounds ? (float)((double)(hs[2 * r + 2] - hs[2 * r + 1]) * 1e-6) : 0.f;
        ctx->kernel_ms.push_back(pm);
        ctx->kernel_ms.push_back(mm);
        ctx->timing.round_kernel_ms += pm;
        ctx->timing.match_kernel_ms += mm;
    }
    float hms = 0.f;
    cudaEventElapsedTime(&hms, ctx->ev2, ctx->ev1);
    ctx->timing.hist_kernel_ms = hms;
    unsigned long long total = 0;
    for (size_t i = 0; i < hist.size(); ++i) total += hist[i];
    if (total != (unsigned long long)ctx->m) return lmx_fail(ctx, LMX_ECUDA, "internal: death histogram size");
    for (size_t i = (size_t)n_rounds; i < hist.size(); ++i)
        if (hist[i]) return lmx_fail(ctx, LMX_ECUDA, "internal: an edge outlived the round loop");
    long long live = ctx->m;
    unsigned long long total_matched_v = 0;
    ctx->timing.slot_reads = 0;
    for (int i = 0; i < n_rounds; ++i) {
        const RoundCtr &c = ctx->ctr_host[i];
        if (c.matched_v & 1ULL) return lmx_fail(ctx, LMX_ECUDA, "internal: odd matched-vertex count");
        if (live <= 0) return lmx_fail(ctx, LMX_ECUDA, "internal: a round without live edges");
        lmx_round_stats sr;
        sr.edges_before = live;
        sr.edges_matched = (int64_t)(c.matched_v / 2);
        sr.edges_removed = (int64_t)hist[(size_t)i];
        stats.push_back(sr);
        live -= (long long)hist[(size_t)i];
        total_matched_v += c.matched_v;
        ctx->timing.slot_reads += (int64_t)c.slot_reads;
    }
    n_matched = total_matched_v / 2;
    return LMX_OK;
}

int lmx_run_rounds_scan(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                        std::vector<lmx_round_stats> &stats, unsigned long long &n_matched) {
    static const bool stepped = getenv("LMX_SCAN_STEPPED") != nullptr;   // A/B: one launch per kernel
    if (!stepped && ctx->m > 0 && ctx->scan_loop_grid > 0) {
        stats.clear();
        n_matched = 0;
        ctx->timing.round_launches = 0;
        LMX_TRY(lmx_ensure_ctr(ctx, 64));
        return run_rounds_loop(ctx, seed_masked, rerandomize, stats, n_matched);
    }
    stats.clear();
    n_matched = 0;
    ctx->timing.round_launches = 0;
    ctx->timing.slot_reads = 0;
    ctx->timing.round_kernel_ms = 0;
    ctx->timing.match_kernel_ms = 0;
    const size_t n = (size_t)ctx->n;
    cudaStream_t st = ctx->stream;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    LMX_TRY(scan_begin(ctx));

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

    int r = 0, n_rounds = -1, batch = 6;
    const size_t nbins0 = kHistBins;
    std::vector<unsigned long long> hist(nbins0, 0);
    bool have_hist = false;
    // Speculative first batch: the previous matching of this context took R
    // rounds; enqueue R + 2 rounds (those past the end exit at once), the
    // histogram with the round count found on the device, and read back
    // everything with one synchronisation.  A longer run continues below.
    // (Off under per-kernel timing, whose timeline expects one histogram.)
    const int spec = (!ctx->kernel_timing && ctx->scan_last_rounds >= 0 && ctx->scan_last_rounds + 2 <= 14 &&
                      ctx->m > 0) ? ctx->scan_last_rounds + 2 : 0;
    if (spec) {
        LMX_TRY(lmx_ensure_ctr(ctx, spec + 1));
        for (; r < spec; ++r) {
            LMX_TRY(scan_enqueue_probe(ctx, r, seed_masked, rerandomize));
            LMX_TRY(scan_enqueue_match(ctx, r, true));
        }
        LMX_TRY(scan_hist_launch(ctx, 0, spec));
        LMX_TRY(scan_edge_bits_launch(ctx, 0, (unsigned long long)ctx->n));   // (rerun below if the loop goes on: it only sets bits)
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host, ctx->ctr, sizeof(RoundCtr) * (size_t)spec,
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaMemcpyAsync(hist.data(), ctx->hist, nbins0 * 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        for (int i = 0; i < spec; ++i) {
            if (ctx->ctr_host[i].live_slots == 0) {
                n_rounds = i;
                break;
            }
        }
        have_hist = n_rounds >= 0;
        batch = 4;
    }
    while (n_rounds < 0 && ctx->m > 0) {
        LMX_TRY(lmx_ensure_ctr(ctx, r + batch + 1));
        const int r0 = r;
        for (int b = 0; b < batch; ++b, ++r) {
            LMX_TRY(scan_enqueue_probe(ctx, r, seed_masked, rerandomize));
            LMX_TRY(tl_mark());
            LMX_TRY(scan_enqueue_match(ctx, r, true));
            LMX_TRY(tl_mark());
        }
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host + r0, ctx->ctr + r0, sizeof(RoundCtr) * (size_t)batch,
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        for (int i = r0; i < r; ++i) {
            if (ctx->ctr_host[i].live_slots == 0) {   // no candidate anywhere: m_i = 0
                n_rounds = i;
                break;
            }
        }
        batch = 4;
    }
    if (n_rounds < 0) n_rounds = 0;
    ctx->scan_last_rounds = n_rounds;
    // death-round histogram -> RoundStats: bins [0, n_rounds) plus "outlived"
    const size_t nbins = std::max<size_t>((size_t)n_rounds + 1, kHistBins);
    hist.resize(nbins, 0);
    if (ctx->m > 0 && !have_hist) {
        std::fill(hist.begin(), hist.end(), 0ULL);
        LMX_TRY(scan_hist_launch(ctx, n_rounds));
        LMX_TRY(scan_edge_bits_launch(ctx, 0, (unsigned long long)ctx->n));
        LMX_TRY(tl_mark());
        LMX_CUDA(ctx, cudaMemcpyAsync(hist.data(), ctx->hist, nbins * 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
    }
    ctx->kernel_ms.clear();
    ctx->timing.hist_kernel_ms = 0;
    if (ctx->kernel_timing && tl_used > 1) {
        // timeline: init | round, match (per round) | histogram (pack + count)
        const int hist_mark = ctx->m > 0 ? tl_used - 1 : -1;
        for (int i = 1; i < tl_used; ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, ctx->tl_events[i - 1], ctx->tl_events[i]);
            if (i == hist_mark) {
                ctx->timing.hist_kernel_ms = ms;
                continue;
            }
            ctx->kernel_ms.push_back(ms);
            if (i & 1) ctx->timing.round_kernel_ms += ms;
            else ctx->timing.match_kernel_ms += ms;
        }
    }
    ctx->timing.rounds_executed = r;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
    unsigned long long total = 0;
    for (size_t i = 0; i < nbins; ++i) total += hist[i];
    if (total != (unsigned long long)ctx->m) return lmx_fail(ctx, LMX_ECUDA, "internal: death histogram size");
    for (size_t i = (size_t)n_rounds; i < nbins; ++i)
        if (hist[i]) return lmx_fail(ctx, LMX_ECUDA, "internal: an edge outlived the round loop");
    long long live = ctx->m;
    unsigned long long total_matched_v = 0;
    for (int i = 0; i < n_rounds; ++i) {
        const RoundCtr &c = ctx->ctr_host[i];
        if (c.matched_v & 1ULL) return lmx_fail(ctx, LMX_ECUDA, "internal: odd matched-vertex count");
        if (live <= 0) return lmx_fail(ctx, LMX_ECUDA, "internal: a round without live edges");
        lmx_round_stats s;
        s.edges_before = live;
        s.edges_matched = (int64_t)(c.matched_v / 2);
        s.edges_removed = (int64_t)hist[(size_t)i];
        stats.push_back(s);
        live -= (long long)hist[(size_t)i];
        total_matched_v += c.matched_v;
    }
    for (int i = 0; i < r; ++i) ctx->timing.slot_reads += (int64_t)ctx->ctr_host[i].slot_reads;
    n_matched = total_matched_v / 2;
    return LMX_OK;
}

// ---- the stepped multi-GPU protocol on the scan loop (bsp.py:101-205) -------
// Every partition keeps the global weight-ordered segments and global
// per-vertex arrays and works on the vertices it owns: A_0 = owned vertices
// with an edge.  Per round: probe (owned A_r) -> propose (a candidate whose
// partner is owned elsewhere is sent to the partner's owner, exchange A) ->
// accept (the owner confirms iff its own candidate is the same edge) -> match
// -> all-gather of the owned bitmap words (exchange B) -> all-reduce of
// (candidates found, matched vertices): "none found" ends the loop.  After it
// the owned mround slices are all-gathered and each partition histograms the
// death rounds of its own lowpair share; the histograms add up.

namespace lmx {

__global__ void lmx_scan_accept_kernel(const uint2 *rec, unsigned long long k, const uint32_t *cnbr,
                                       const uint32_t *ckey, const uint32_t *ptr, const unsigned long long *vbeg,
                                       const uint2 *ids, uint32_t lo, uint32_t *remote_ok) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint2 r = rec[i];
        if (r.y == kNone) continue;   // the filler of a fixed-capacity exchange (lmx_scan_pad_kernel)
        const uint32_t vl = r.x - lo;
        const uint32_t w = cnbr[vl];
        if (w != kNone && cand_eid(vl, w, ckey, ptr, vbeg, ids) == r.y) remote_ok[vl] = 1u;
    }
}

// Fixed-capacity exchange A (the late rounds, no host round trip): the packed
// records of destination j go to padded[j C, j C + count_j), the rest of its
// C slots is filler {first vertex of j, kNone} that the receiver's accept
// skips.  C bounds every count (no rank proposes more records than it has
// listed vertices); a count above it sets *overflow.
__global__ void lmx_scan_pad_kernel(const uint2 *packed, const long long *counts64, const unsigned long long *bounds,
                                    int p, unsigned long long C, uint2 *padded, unsigned int *overflow) {
    __shared__ unsigned long long s_off[65];
    if (threadIdx.x == 0) {
        unsigned long long o = 0;
        for (int j = 0; j < p; ++j) {
            s_off[j] = o;
            o += (unsigned long long)counts64[j];
        }
    }
    __syncthreads();
    if (blockIdx.x == 0 && threadIdx.x < (unsigned)p && (unsigned long long)counts64[threadIdx.x] > C)
        atomicOr(overflow, 1u);
    const unsigned long long total = (unsigned long long)p * C;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
        const int j = (int)(i / C);
        const unsigned long long t = i - (unsigned long long)j * C;
        padded[i] = t < (unsigned long long)counts64[j] ? packed[s_off[j] + t]
                                                         : make_uint2((uint32_t)bounds[j], kNone);
    }
}

}  // namespace lmx

static int scan_dist_send_buffers(lmx_ctx *ctx);

int lmx_scan_dist_begin(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize) {
    ctx->timing.round_launches = 0;
    ctx->dist_round = 0;
    ctx->dist_seed = seed_masked;
    ctx->dist_rr = rerandomize;
    ctx->mate_target = ctx->mate;
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->remote_ok, 0, (size_t)std::max<int64_t>(ctx->n_local, 1) * 4, ctx->stream));
    LMX_TRY(scan_begin(ctx));
    LMX_TRY(scan_dist_send_buffers(ctx));
    LMX_CUDA(ctx, cudaMemsetAsync(reinterpret_cast<char *>(ctx->send_cnt) + 768, 0, 4, ctx->stream));   // overflow
    LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return LMX_OK;
}

// Exchange-A buffers: p regions of nl records + the packed copy; the counts
// block holds [64] u32 counts, [64] i64 counts at +256, the p + 1 bounds at +1024.
static int scan_dist_send_buffers(lmx_ctx *ctx) {
    const int p = ctx->dist_p;
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);
    const size_t need = nl * (size_t)(p + 1);   // p regions + the packed copy
    if (ctx->send_cap < need) {
        lmx_dfree(ctx, ctx->send);
        ctx->send = nullptr;
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->send, need * sizeof(uint2)));
        ctx->send_cap = need;
    }
    // send_cnt block: [64] u32 counts, [64] i64 counts at +256, the p + 1 bounds at +1024
    if (!ctx->send_cnt) {
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->send_cnt, 2048));
        std::vector<unsigned long long> hb(ctx->bounds.begin(), ctx->bounds.end());
        LMX_CUDA(ctx, cudaMemcpyAsync(reinterpret_cast<char *>(ctx->send_cnt) + 1024, hb.data(),
                                      (size_t)(p + 1) * 8, cudaMemcpyHostToDevice, ctx->stream));
    }
    return LMX_OK;
}

// Round r's probe on the owned lists; it also appends exchange A's records.
int lmx_scan_dist_round(lmx_ctx *ctx) {
    LMX_TRY(lmx_ensure_ctr(ctx, ctx->dist_round + 2));
    LMX_TRY(scan_dist_send_buffers(ctx));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->send_cnt, 0, 64 * sizeof(uint32_t), ctx->stream));
    return scan_enqueue_probe(ctx, ctx->dist_round, ctx->dist_seed, ctx->dist_rr, true);
}

// Exchange A: the probe appended the records; pack them by destination.
int lmx_scan_dist_propose(lmx_ctx *ctx, void **counts_dev, void **packed_dev) {
    const int p = ctx->dist_p;
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);
    if (!ctx->send || !ctx->send_cnt) return lmx_fail(ctx, LMX_ESTATE, "propose before round");
    long long *counts64 = reinterpret_cast<long long *>(reinterpret_cast<char *>(ctx->send_cnt) + 256);
    uint2 *packed = ctx->send + nl * (size_t)p;
    lmx_pack_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(ctx->send, ctx->send_cnt, p, (uint32_t)nl, packed,
                                                                 counts64);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    *counts_dev = counts64;
    *packed_dev = packed;
    return LMX_OK;
}

// The fixed-capacity exchange of the late rounds (after lmx_scan_dist_propose).
int lmx_scan_dist_pad(lmx_ctx *ctx, int64_t C, void **padded_dev, void **overflow_dev) {
    const int p = ctx->dist_p;
    if (!ctx->send || !ctx->send_cnt) return lmx_fail(ctx, LMX_ESTATE, "pad before propose");
    if (C < 1) return lmx_fail(ctx, LMX_EINVAL, "capacity must be >= 1");
    const size_t need = (size_t)C * (size_t)p;
    if (ctx->pad_cap < need) {
        lmx_dfree(ctx, ctx->pad);
        ctx->pad = nullptr;
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ctx->pad, need * sizeof(uint2)));
        ctx->pad_cap = need;
    }
    const size_t nl = (size_t)std::max<int64_t>(ctx->n_local, 1);
    char *cb = reinterpret_cast<char *>(ctx->send_cnt);
    unsigned int *overflow = reinterpret_cast<unsigned int *>(cb + 768);
    lmx_scan_pad_kernel<<<ctx->num_sms * 2, kBlock, 0, ctx->stream>>>(
        ctx->send + nl * (size_t)p, reinterpret_cast<const long long *>(cb + 256),
        reinterpret_cast<const unsigned long long *>(cb + 1024), p, (unsigned long long)C, ctx->pad, overflow);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    *padded_dev = ctx->pad;
    if (overflow_dev) *overflow_dev = overflow;
    return LMX_OK;
}

int lmx_scan_dist_accept(lmx_ctx *ctx, int64_t count) {
    if (count <= 0) return LMX_OK;
    lmx_scan_accept_kernel<<<ctx->num_sms * 4, kBlock, 0, ctx->stream>>>(
        ctx->recv, (unsigned long long)count, reinterpret_cast<const uint32_t *>(ctx->cand),
        reinterpret_cast<const uint32_t *>(ctx->cand) + std::max<int64_t>(ctx->n_local, 1), ctx->vdeg, ctx->vbeg,
        ctx->ids0, (uint32_t)ctx->lo, ctx->remote_ok);
    LMX_CUDA(ctx, cudaGetLastError());
    ctx->timing.round_launches += 1;
    return LMX_OK;
}

int lmx_scan_dist_match(lmx_ctx *ctx, void **stats_dev) {
    const int r = ctx->dist_round;
    LMX_TRY(scan_enqueue_match(ctx, r, true));   // edge bits after the loop (lmx_scan_dist_hist)
    *stats_dev = &ctx->ctr[r].live_slots;   // {candidates found, matched vertices}
    ctx->dist_round = r + 1;
    return LMX_OK;
}

int lmx_scan_dist_hist(lmx_ctx *ctx, int n_rounds, void **hist_dev, int *nbins) {
    if (n_rounds < 0) return lmx_fail(ctx, LMX_EINVAL, "negative round count");
    // the loop is over: the owned range's matched-edge bits (as on one GPU,
    // kept out of the per-round match kernel), then the histogram
    LMX_TRY(scan_edge_bits_launch(ctx, (unsigned long long)ctx->lo, (unsigned long long)ctx->hi));
    LMX_TRY(scan_hist_launch(ctx, n_rounds));
    *hist_dev = ctx->hist;
    *nbins = (int)std::max<size_t>((size_t)n_rounds + 1, kHistBins);
    return LMX_OK;
}
