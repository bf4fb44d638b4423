// lmx_scanload.cu -- K0 for the weight-ordered scan loop (lmx_scan.cu).
//
// The scan loop needs, per owned vertex, its incident edges in descending
// weight order (tiebreak.py:105-113 canonical bits), so that a vertex's
// candidate only ever moves down its segment.  Only the
// order inside a segment matters: a vertex compares its own edges only
// (matchers.py:93-103); edges of equal weight at one vertex form an adjacent
// run that the per-round salt (tiebreak.py:55-59) orders.
//
// lmx_weight_stage (lmx_setup.cu) has sorted the edge ids by weight and
// flagged the weights that occur more than once.  Here:
//   1. owned segment offsets vbeg (local ids v - lo)
//   2. the slot stream in DESCENDING weight order: two records per edge,
//      {neighbour | globally-tied flag, edge id}, keyed by the owner (local id;
//      not owned: the sentinel nl)
//   3. a stable radix sort of the stream by owner: every segment comes out in
//      descending weight order, no per-segment sort
//   4. one pass over the sorted slots: exact tie flags (a globally tied slot
//      is tied at its vertex iff an adjacent slot of the segment has the same
//      weight bits; bit 30 marks a run's first slot), round-0 candidates
//      cand0[v] = the segment's first slot, and the death-round histogram's
//      pairs {v, u < v} (each edge once, grouped by v)
// (Measured and replaced: per-vertex atomic scatter + cub segmented sort:
// 0.77 s at RMAT-26 -- random 8-byte writes and one CTA per long segment.)
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "lmx_internal.cuh"
#include "lmx_sort.cuh"

using namespace lmx;

namespace lmx {

__device__ __forceinline__ unsigned long long canon_bits2(double w) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(w);
    return (b << 1) == 0 ? 0ULL : b;   // -0.0 -> +0.0 (tiebreak.py:112)
}

__global__ void k_owned_deg(const uint32_t *deg0, unsigned long long lo, unsigned long long nl,
                            unsigned long long *vbeg) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i <= nl; i += stride)
        vbeg[i] = i < nl ? deg0[lo + i] : 0ULL;
}

// Endpoints in device ids, packed per edge (one random 8-byte gather in the
// stream instead of two 4-byte ones; the relabel lookups run in edge order).
// 4 edges per thread per step: their new-id gathers are in flight together.
__global__ void k_pack_endpoints(const uint32_t *eu, const uint32_t *ev, const uint32_t *newid,
                                 unsigned long long m, uint2 *euv) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e0 < m;
         e0 += 4 * stride) {
        uint32_t a[4], b[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned long long e = e0 + k * stride;
            a[k] = e < m ? __ldcs(eu + e) : 0u;
            b[k] = e < m ? __ldcs(ev + e) : 0u;
        }
        if (newid) {
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                a[k] = newid[a[k]];
                b[k] = newid[b[k]];
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const unsigned long long e = e0 + k * stride;
            if (e < m) euv[e] = make_uint2(a[k], b[k]);
        }
    }
}

// The slot stream in descending weight order (sorted position j = m-1-i);
// 4 edges per thread per step, the gathers of a step in flight together.
// Stream positions [ib, ib + cnt) of the m edges (a partition streams its
// weight order in chunks), written from okey / sval index 0.
#ifndef LMX_STREAM_ILP
#define LMX_STREAM_ILP 4   // edges per thread per step of the slot stream
#endif
__global__ void k_desc_stream(const uint32_t *eid_sorted, const uint32_t *tied, unsigned long long m,
                              unsigned long long ib, unsigned long long cnt, const uint2 *euv, uint32_t lo,
                              uint32_t nl, uint32_t *okey, uint2 *sval) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    eid_sorted += m - ib - cnt;   // sorted positions j = m-1-(ib+i) for i in [0, cnt)
    tied += m - ib - cnt;
    m = cnt;
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < m;
         i0 += LMX_STREAM_ILP * stride) {
        uint32_t e[LMX_STREAM_ILP], t[LMX_STREAM_ILP];
        uint2 p[LMX_STREAM_ILP];
#pragma unroll
        for (int k = 0; k < LMX_STREAM_ILP; ++k) {
            const unsigned long long i = i0 + k * stride;
            if (i < m) {
                const unsigned long long j = m - 1 - i;
                e[k] = eid_sorted[j];
                t[k] = tied[j] ? kSlotTied : 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < LMX_STREAM_ILP; ++k)
            if (i0 + k * stride < m) p[k] = euv[e[k]];
#pragma unroll
        for (int k = 0; k < LMX_STREAM_ILP; ++k) {
            const unsigned long long i = i0 + k * stride;
            if (i < m) {   // bit 30 marks, until the post pass, the slot of the edge's v end
                const uint32_t oa = p[k].x - lo, ob = p[k].y - lo;
                okey[2 * i] = oa < nl ? oa : nl;
                sval[2 * i] = make_uint2(p[k].y | t[k], e[k]);
                okey[2 * i + 1] = ob < nl ? ob : nl;
                sval[2 * i + 1] = make_uint2(p[k].x | t[k] | kSlotRunStart, e[k]);
            }
        }
    }
}

// Tie flags, cand0 and lowpair over the owner-sorted slots (see header).
__global__ void __launch_bounds__(kBlock) k_scan_post(const uint32_t *owner, uint2 *ids, const double *w,
                                                      unsigned long long S, uint32_t lo, uint2 *cand0,
                                                      uint2 *lowpair, unsigned long long *counts,
                                                      uint32_t *side) {
    __shared__ uint32_t s_cnt[kWarps];
    __shared__ unsigned long long s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    unsigned long long tied_n = 0;
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * kBlock; i0 < S;
         i0 += (unsigned long long)gridDim.x * kBlock) {
        const unsigned long long i = i0 + tid;
        bool emit = false;
        uint32_t vdev = 0, nbr = 0;
        if (i < S) {
            const uint32_t o = owner[i];
            const bool head = i == 0 || owner[i - 1] != o;
            uint2 x = ids[i];
            nbr = x.x & kSlotNbr;
            if (side && (x.x & kSlotRunStart)) atomicOr(side + (i >> 5), 1u << (i & 31));
            uint32_t flags = 0;
            if (x.x & kSlotTied) {   // the weight occurs more than once: compare with the neighbours
                const unsigned long long k = canon_bits2(w[x.y]);
                // (in place: a neighbour may already hold its final flags, but its
                // tied bit only clears when its weight differs from both
                // neighbours', and .y -- the local edge -- is not rewritten here)
                const bool prev = !head && (ids[i - 1].x & kSlotTied) && canon_bits2(w[ids[i - 1].y]) == k;
                const bool next = i + 1 < S && owner[i + 1] == o && (ids[i + 1].x & kSlotTied) &&
                                  canon_bits2(w[ids[i + 1].y]) == k;
                if (prev || next) flags = kSlotTied | (prev ? 0u : kSlotRunStart);
                tied_n += (prev || next) ? 1u : 0u;
            }
            x.x = nbr | flags;
            if (head) cand0[o] = x;
            vdev = o + lo;
            emit = nbr < vdev;
            ids[i].x = x.x;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, emit);
        if (lane == 0) s_cnt[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int q = 0; q < kWarps; ++q) t += s_cnt[q];
            s_base = t ? atomicAdd(counts + 1, (unsigned long long)t) : 0ULL;
        }
        __syncthreads();
        if (emit) {
            unsigned long long p = s_base;
            for (int q = 0; q < warp; ++q) p += s_cnt[q];
            lowpair[p + __popc(bal & lt)] = make_uint2(vdev, nbr);
        }
        __syncthreads();
    }
    for (int off = 16; off > 0; off >>= 1) tied_n += __shfl_xor_sync(0xffffffffu, tied_n, off);
    if (lane == 0 && tied_n) atomicAdd(counts, tied_n);
}

// A partition's slots and round-0 candidates name local edges until here:
// to the global edge ids (salts, exchange records, outputs).
__global__ void k_to_global_eid(uint2 *ids, unsigned long long S, uint2 *cand0, unsigned long long nl,
                                const uint32_t *geid) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < S + nl; i += stride) {
        if (i < S) ids[i].y = geid[ids[i].y];
        else if (cand0[i - S].x != kNone) cand0[i - S].y = geid[cand0[i - S].y];
    }
}

struct OwnedKey {
    uint32_t nl;
    __host__ __device__ __forceinline__ bool operator()(const uint32_t &k) const { return k < nl; }
};

struct OwnedFlag {
    uint32_t nl;
    __host__ __device__ __forceinline__ char operator()(const uint32_t &k) const { return k < nl ? 1 : 0; }
};

}  // namespace lmx

static int lgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    return (int)std::max<unsigned long long>(1, std::min(b, cap));
}

// 4. tie flags, cand0, lowpair over the owner-sorted slots ids0[0, S)
// (owner[i]: local owner of slot i); partitions: slot sides, global edge ids.
static int scan_post(lmx_ctx *ctx, const uint32_t *owner, unsigned long long S, unsigned long long *cnt) {
    cudaStream_t st = ctx->stream;
    const unsigned long long m = (unsigned long long)lmx_edges(ctx), lo = ctx->lo, nl = ctx->hi - ctx->lo;
    const size_t S1 = std::max<unsigned long long>(S, 1);
    cudaError_t e = cudaSuccess;
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->cand0, std::max<unsigned long long>(nl, 1) * 8, "cand0"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->lowpair, std::max<unsigned long long>(std::min(m, S), 1) * 8, "lowpair"));
    e = cudaMemsetAsync(ctx->cand0, 0xFF, std::max<unsigned long long>(nl, 1) * 8, st);
    if (ctx->dist_p > 1 && e == cudaSuccess) {   // which end of its edge each owned slot is (RoundMessages)
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->slot_side, (S1 + 31) / 32 * 4, "slot side"));
        e = cudaMemsetAsync(ctx->slot_side, 0, (S1 + 31) / 32 * 4, st);
    }
    if (e == cudaSuccess && S) {
        k_scan_post<<<lgrid(ctx, S), kBlock, 0, st>>>(owner, ctx->ids0, ctx->w, S, (uint32_t)lo, ctx->cand0,
                                                     ctx->lowpair, cnt, ctx->slot_side);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess && ctx->geid && S + nl) {
        k_to_global_eid<<<lgrid(ctx, S + nl), kBlock, 0, st>>>(ctx->ids0, S, ctx->cand0, nl, ctx->geid);
        e = cudaGetLastError();
    }
    unsigned long long hc[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return lmx_cuda_check(ctx, e, "slot flags");
    trace_mark(ctx, "  scan: flags + lowpair");
    ctx->lowpair_n = hc[1];
    if (ctx->dist_p == 1 && hc[1] != m) return lmx_fail(ctx, LMX_ECUDA, "internal: lowpair count");
    return LMX_OK;
}

// A partition's owned slots (weight order by owner), memory-lean: the
// endpoints are packed (new ids) and the caller-id arrays freed -- a
// partition never reads them again -- then the weight order is streamed in
// chunks, each chunk's owned slots appended (a stable select keeps the
// weight order), and the S owned slots sorted by owner.  Peak: the packed
// endpoints + one chunk of the stream + the owned slots twice, instead of
// the whole two-record-per-edge stream next to everything else.
static int partition_slots(lmx_ctx *ctx, const uint32_t *newid, unsigned long long S, int bits) {
    cudaStream_t st = ctx->stream;
    const unsigned long long m = (unsigned long long)lmx_edges(ctx), lo = ctx->lo, nl = ctx->hi - ctx->lo;
    const size_t S1 = std::max<unsigned long long>(S, 1);
    const unsigned long long C = std::min<unsigned long long>(m, std::max<unsigned long long>(1ULL << 24, (m + 3) / 4));
    uint2 *euv = nullptr, *sval = nullptr, *sorted = nullptr;
    uint32_t *okey_c = nullptr, *okey2 = nullptr, *okey = nullptr;
    unsigned long long *nsel = nullptr, *cnt = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&euv, m * 8, "packed endpoints")) != LMX_OK) break;
        k_pack_endpoints<<<lgrid(ctx, m), kBlock, 0, st>>>(ctx->eu, ctx->ev, newid, m, euv);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        lmx_free(ctx, (void **)&ctx->eu, m * 4);
        lmx_free(ctx, (void **)&ctx->ev, m * 4);
        if ((rc = lmx_alloc(ctx, (void **)&okey2, S1 * 4, "owned keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&okey_c, 2 * C * 4, "stream chunk keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&sval, 2 * C * 8, "stream chunk")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&nsel, 8, "selected")) != LMX_OK) break;
        cub::TransformInputIterator<char, OwnedFlag, const uint32_t *> flags(okey_c, OwnedFlag{(uint32_t)nl});
        size_t t1 = 0, t2 = 0;
        e = cub::DeviceSelect::If(nullptr, t1, okey_c, okey2, nsel, (long long)(2 * C), OwnedKey{(uint32_t)nl}, st);
        if (e == cudaSuccess)
            e = cub::DeviceSelect::Flagged(nullptr, t2, sval, flags, ctx->ids0, nsel, (long long)(2 * C), st);
        if (e != cudaSuccess) break;
        tmp_bytes = std::max(t1, t2);
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "select tmp")) != LMX_OK) break;
        unsigned long long off = 0;
        for (unsigned long long ib = 0; ib < m && e == cudaSuccess; ib += C) {
            const unsigned long long k = std::min(C, m - ib);
            k_desc_stream<<<lgrid(ctx, k), kBlock, 0, st>>>(ctx->ws_eid, ctx->ws_tied, m, ib, k, euv, (uint32_t)lo,
                                                           (uint32_t)nl, okey_c, sval);
            if ((e = cudaGetLastError()) != cudaSuccess) break;
            size_t a1 = t1, a2 = t2;
            e = cub::DeviceSelect::If(tmp, a1, okey_c, okey2 + off, nsel, (long long)(2 * k), OwnedKey{(uint32_t)nl},
                                      st);
            if (e == cudaSuccess)
                e = cub::DeviceSelect::Flagged(tmp, a2, sval, flags, ctx->ids0 + off, nsel, (long long)(2 * k), st);
            unsigned long long got = 0;
            if (e == cudaSuccess) e = cudaMemcpyAsync(&got, nsel, 8, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            off += got;
            if (off > S) { rc = lmx_fail(ctx, LMX_ECUDA, "internal: owned slot count"); break; }
        }
        if (e != cudaSuccess || rc != LMX_OK) break;
        if (off != S) { rc = lmx_fail(ctx, LMX_ECUDA, "internal: owned slot count"); break; }
        lmx_free(ctx, (void **)&euv, m * 8);
        lmx_free(ctx, (void **)&okey_c, 2 * C * 4);
        lmx_free(ctx, (void **)&sval, 2 * C * 8);
        lmx_free(ctx, &tmp, tmp_bytes);
        lmx_free(ctx, (void **)&ctx->ws_eid, m * 4);
        lmx_free(ctx, (void **)&ctx->ws_tied, m * 4);
        trace_mark(ctx, "  scan: chunked stream + owned select");
        // stable sort of the S owned slots by owner: okey2 -> okey, ids0 -> sorted
        if ((rc = lmx_alloc(ctx, (void **)&okey, S1 * 4, "owner keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&sorted, S1 * 8, "sorted slots")) != LMX_OK) break;
        if ((rc = lmx_sort_pairs(ctx, &okey2, &okey, &ctx->ids0, &sorted, (long long)S, 0, bits, st,
                                 "owner sort")) != LMX_OK)
            break;
        lmx_free(ctx, (void **)&ctx->ids0, S1 * 8);
        ctx->ids0 = sorted;
        sorted = nullptr;
        lmx_free(ctx, (void **)&okey2, S1 * 4);
        trace_mark(ctx, "  scan: owner sort");
        if ((rc = lmx_alloc(ctx, (void **)&cnt, 16, "counts")) != LMX_OK) break;
        if ((e = cudaMemsetAsync(cnt, 0, 16, st)) != cudaSuccess) break;
        rc = scan_post(ctx, okey, S, cnt);
    } while (0);
    if (e != cudaSuccess && rc == LMX_OK) rc = lmx_cuda_check(ctx, e, "partition slots");
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&euv, m * 8);
    lmx_free(ctx, (void **)&okey_c, 2 * C * 4);
    lmx_free(ctx, (void **)&sval, 2 * C * 8);
    lmx_free(ctx, (void **)&okey2, S1 * 4);
    lmx_free(ctx, (void **)&okey, S1 * 4);
    lmx_free(ctx, (void **)&sorted, S1 * 8);
    lmx_free(ctx, (void **)&nsel, 8);
    lmx_free(ctx, (void **)&cnt, 16);
    lmx_free(ctx, &tmp, tmp_bytes);
    return rc;
}

// Builds ctx->vbeg (local, n_local + 1), ctx->ids0 (owned slots, flags),
// ctx->cand0, ctx->lowpair / lowpair_n from ctx->eu/ev/w, ctx->deg0 (device
// ids) and the weight stage's ws_eid / ws_tied (descending order from the
// end).  newid: caller id -> device id, or null.
int lmx_scan_build_slots(lmx_ctx *ctx, const uint32_t *newid) {
    cudaStream_t st = ctx->stream;
    // the edges held: all of them, or a partition's local edges (global ids in ctx->geid)
    const unsigned long long m = (unsigned long long)lmx_edges(ctx), lo = ctx->lo, nl = ctx->hi - ctx->lo;
    const unsigned long long slots2 = 2 * m;
    // 1. owned segment offsets
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->vbeg, (nl + 1) * 8, "vbeg"));
    k_owned_deg<<<lgrid(ctx, nl + 1), kBlock, 0, st>>>(ctx->deg0, lo, nl, ctx->vbeg);
    LMX_CUDA(ctx, cudaGetLastError());
    {
        size_t tmp = 0;
        LMX_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st));
        void *t = nullptr;
        LMX_TRY(lmx_alloc(ctx, &t, tmp, "scan tmp"));
        cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st);
        cudaStreamSynchronize(st);
        lmx_free(ctx, &t, tmp);
        LMX_CUDA(ctx, e);
    }
    unsigned long long S = 0;
    LMX_CUDA(ctx, cudaMemcpyAsync(&S, ctx->vbeg + nl, 8, cudaMemcpyDeviceToHost, st));
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    ctx->slots_local = (int64_t)S;
    const size_t S1 = std::max<unsigned long long>(S, 1), M2 = std::max<unsigned long long>(slots2, 1);
    // one GPU: the stream is sorted straight into ids0; a partition first
    // selects its owned slots (weight order kept), then sorts those
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ids0, S1 * 8, "ids0"));
    uint32_t *okey = nullptr, *okey2 = nullptr;
    uint2 *sval = nullptr, *sorted = nullptr;
    const bool part = ctx->dist_p > 1;
    unsigned long long *cnt = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int bits = 1;
    while (bits < 32 && (1ULL << bits) <= nl) ++bits;   // owner keys in [0, nl], nl = not owned
    int rc = LMX_OK;
    if (part && m) return partition_slots(ctx, newid, S, bits);
    do {
        if ((rc = lmx_alloc(ctx, (void **)&okey, M2 * 4, "owner keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&okey2, M2 * 4, "owner keys out")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&sval, M2 * 8, "slot stream")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cnt, 16, "counts")) != LMX_OK) break;
        cudaError_t e = cudaMemsetAsync(cnt, 0, 16, st);
        if (m && e == cudaSuccess) {
            // the packed endpoints borrow the owner-key output buffer (same size)
            uint2 *euv = reinterpret_cast<uint2 *>(okey2);
            k_pack_endpoints<<<lgrid(ctx, m), kBlock, 0, st>>>(ctx->eu, ctx->ev, newid, m, euv);
            trace_mark(ctx, "  scan: packed endpoints");
            k_desc_stream<<<lgrid(ctx, m), kBlock, 0, st>>>(ctx->ws_eid, ctx->ws_tied, m, 0, m, euv, (uint32_t)lo,
                                                           (uint32_t)nl, okey, sval);
            e = cudaGetLastError();
        }
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "slot stream"); break; }
        trace_mark(ctx, "  scan: slot stream");
        if (m && !part) {   // (sval and ids0 have the same size: S = 2m on one GPU)
            if ((rc = lmx_sort_pairs(ctx, &okey, &okey2, &sval, &ctx->ids0, (long long)slots2, 0, bits, st,
                                     "owner sort")) != LMX_OK)
                break;
            trace_mark(ctx, "  scan: owner sort");
        }
        lmx_free(ctx, (void **)&sval, M2 * 8);
        lmx_free(ctx, &tmp, tmp_bytes);
        rc = scan_post(ctx, okey2, S, cnt);   // okey2: the owner of each sorted slot
    } while (0);
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&okey, M2 * 4);
    lmx_free(ctx, (void **)&okey2, M2 * 4);
    lmx_free(ctx, (void **)&sval, M2 * 8);
    lmx_free(ctx, (void **)&sorted, S1 * 8);
    lmx_free(ctx, (void **)&cnt, 16);
    lmx_free(ctx, &tmp, tmp_bytes);
    return rc;
}
