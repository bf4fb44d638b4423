// lmx_scanload.cu -- K0 for the weight-ordered scan loop (lmx_scan.cu).
//
// The scan loop needs, per owned vertex, its incident edges in descending
// weight order (tiebreak.py:105-113 canonical bits), so that a vertex's
// candidate only ever moves down its segment.  Only the
// order INSIDE a segment matters: a vertex compares its own edges only
// (matchers.py:93-103), so no global weight rank is needed -- edges of equal
// weight at one vertex form an adjacent run that the per-round salt
// (tiebreak.py:55-59) orders.
//
//   1. owned degrees and segment offsets (vbeg, local ids v - lo)
//   2. scatter: every edge e with an owned endpoint writes one slot per owned
//      end: key = canonical weight bits, value = {neighbour (device id), e};
//      and, for the death-round histogram, the pair {higher, lower} if this
//      partition owns the higher end (lowpair, edge order on one GPU)
//   3. segmented sort of the slots by key, descending, per owned vertex
//   4. flag pass: ids0[i] = {nbr | tied << 31 | run start << 30, e}, where
//      tied = the weight equals a neighbouring slot's in the same segment;
//      counts the tied slots (the loader falls back to the compacting loop
//      when ties are common: each round would rescan them)
//   5. round-0 candidates cand0[v] = first slot of the segment
//
// Memory: keys + values as cub double buffers, 32 B per owned slot during
// step 3; the value buffer the result lands in becomes ids0 (8 B per slot).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <vector>

#include "lmx_internal.cuh"

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

// Slots of the owned endpoints.  A vertex's slot order is free before the
// segmented sort, so most slots take their place from a per-vertex atomic
// cursor; the slots of the H huge segments (local ids [0, H), the leading
// degree-sorted vertices of a relabelled range) go to a shared region
// [0, vbeg[H]) through one block-aggregated cursor -- per-vertex cursors
// serialise on hubs -- and are sorted by (owner, key) afterwards.
__global__ void __launch_bounds__(kBlock) k_scan_scatter(const uint32_t *eu, const uint32_t *ev, const double *w,
                                                         unsigned long long m, const uint32_t *newid, uint32_t lo,
                                                         uint32_t nl, uint32_t H, const unsigned long long *vbeg,
                                                         uint32_t *fill, unsigned long long *huge_cursor,
                                                         unsigned long long *keys, uint2 *vals, uint32_t *howner) {
    __shared__ uint32_t s_cnt[kWarps];
    __shared__ unsigned long long s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (unsigned long long e0 = (unsigned long long)blockIdx.x * kBlock; e0 < m;
         e0 += (unsigned long long)gridDim.x * kBlock) {
        const unsigned long long e = e0 + tid;
        uint32_t a = kNone, b = kNone;
        unsigned long long kb = 0;
        if (e < m) {
            a = eu[e];
            b = ev[e];
            kb = canon_bits2(w[e]);
            if (newid) {
                a = newid[a];
                b = newid[b];
            }
        }
        const uint32_t al = a - lo, bl = b - lo;   // local ids (>= nl: not owned)
        const bool ha = e < m && al < H, hb = e < m && bl < H;
        // per-vertex cursors for the non-huge owned ends
        if (e < m && al < nl && !ha) {
            const unsigned long long p = vbeg[al] + atomicAdd(fill + al, 1u);
            keys[p] = kb;
            vals[p] = make_uint2(b, (uint32_t)e);
        }
        if (e < m && bl < nl && !hb) {
            const unsigned long long p = vbeg[bl] + atomicAdd(fill + bl, 1u);
            keys[p] = kb;
            vals[p] = make_uint2(a, (uint32_t)e);
        }
        // huge ends: block-aggregated positions in the shared region
        const uint32_t na = __ballot_sync(0xffffffffu, ha), nb = __ballot_sync(0xffffffffu, hb);
        if (lane == 0) s_cnt[warp] = __popc(na) + __popc(nb);
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int q = 0; q < kWarps; ++q) t += s_cnt[q];
            s_base = t ? atomicAdd(huge_cursor, (unsigned long long)t) : 0ULL;
        }
        __syncthreads();
        if (na | nb) {
            unsigned long long p = s_base;
            for (int q = 0; q < warp; ++q) p += s_cnt[q];
            if (ha) {
                const unsigned long long pa = p + __popc(na & lt);
                keys[pa] = kb;
                vals[pa] = make_uint2(b, (uint32_t)e);
                howner[pa] = al;
            }
            if (hb) {
                const unsigned long long pb = p + __popc(na) + __popc(nb & lt);
                keys[pb] = kb;
                vals[pb] = make_uint2(a, (uint32_t)e);
                howner[pb] = bl;
            }
        }
        __syncthreads();
    }
}

__global__ void k_count_huge(const uint32_t *deg0, unsigned long long lo, unsigned long long nl, uint32_t thresh,
                             unsigned long long *count) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long c = 0;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride)
        c += deg0[lo + i] > thresh ? 1u : 0u;
    for (int off = 16; off > 0; off >>= 1) c += __shfl_xor_sync(0xffffffffu, c, off);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// Huge region after the key sort: the owner of each sorted slot (for the
// stable owner sort) and the iota of positions.
__global__ void k_huge_owner_keys(const uint32_t *howner, const uint32_t *idx, unsigned long long k, uint32_t *okey) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
        okey[i] = howner[idx[i]];
}

__global__ void k_iota(uint32_t *x, unsigned long long k) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
        x[i] = (uint32_t)i;
}

// Huge region: gather the records into (owner, key desc) order.
__global__ void k_huge_gather(const uint32_t *idx, unsigned long long k, const unsigned long long *keys,
                              const uint2 *vals, unsigned long long *keys_out, uint2 *vals_out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint32_t j = idx[i];
        keys_out[i] = keys[j];
        vals_out[i] = vals[j];
    }
}

// Owner of every slot (local id), written segment by segment: warp per vertex.
__global__ void k_slot_owner(const unsigned long long *vbeg, unsigned long long nl, uint32_t *sowner) {
    const unsigned long long gw = ((unsigned long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned long long nw = ((unsigned long long)gridDim.x * blockDim.x) >> 5;
    const int lane = threadIdx.x & 31;
    for (unsigned long long v = gw; v < nl; v += nw) {
        const unsigned long long b = vbeg[v], e = vbeg[v + 1];
        for (unsigned long long i = b + lane; i < e; i += 32) sowner[i] = (uint32_t)v;
    }
}

// ids0 flags, round-0 candidates and the death-round histogram's pairs in one
// pass over the sorted slots: tied = the weight equals a neighbouring slot's
// in the same segment; cand0[v] = the segment's first slot; lowpair gets
// {v, u} for every slot of v with neighbour u < v (each edge once, grouped by
// v: block-aggregated appends keep slot order inside a block).
__global__ void __launch_bounds__(kBlock) k_scan_post(const unsigned long long *keys, uint2 *ids,
                                                      const uint32_t *sowner, unsigned long long S, uint32_t lo,
                                                      uint2 *cand0, uint2 *lowpair, unsigned long long *counts) {
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
            const unsigned long long k = keys[i];
            const uint32_t o = sowner[i];
            const bool head = i == 0 || sowner[i - 1] != o;
            const bool prev = !head && keys[i - 1] == k;
            const bool next = i + 1 < S && sowner[i + 1] == o && keys[i + 1] == k;
            const bool tied = prev || next;
            uint2 x = ids[i];
            nbr = x.x;
            x.x |= (tied ? kSlotTied : 0u) | ((tied && !prev) ? kSlotRunStart : 0u);
            ids[i] = x;
            if (head) cand0[o] = x;
            tied_n += tied ? 1u : 0u;
            vdev = o + lo;
            emit = nbr < vdev;
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

// Vertex cut points of the sort chunks: the first vertex whose offset exceeds
// k * chunk (so a chunk holds at most `chunk` slots unless one vertex does).
__global__ void k_chunk_cuts(const unsigned long long *vbeg, unsigned long long v0, unsigned long long nl,
                             unsigned long long chunk, int nc, unsigned long long *cuts) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k > nc) return;
    const unsigned long long target = vbeg[v0] + (unsigned long long)k * chunk;
    unsigned long long a = v0, b = nl;   // first v in [v0, nl] with vbeg[v] > target, minus one
    while (a < b) {
        const unsigned long long mid = (a + b) / 2;
        if (vbeg[mid] <= target) a = mid + 1;
        else b = mid;
    }
    cuts[k] = k == 0 ? v0 : (k == nc ? nl : (a > v0 ? a - 1 : v0));
}

struct SubBase {
    unsigned long long base;
    __host__ __device__ __forceinline__ long long operator()(const unsigned long long &x) const {
        return (long long)(x - base);
    }
};

}  // namespace lmx

static int lgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    return (int)std::max<unsigned long long>(1, std::min(b, cap));
}

#ifndef LMX_HUGE_DEG
#define LMX_HUGE_DEG 4096   // segments longer than this are sorted as one (owner, key) region
#endif

// Builds ctx->vbeg (local, n_local + 1), ctx->ids0 (owned slots, flags),
// ctx->cand0, ctx->lowpair / lowpair_n from ctx->eu/ev/w and ctx->deg0
// (device-id degrees).  newid: caller id -> device id, or null.  Sets
// *tied_slots.  ctx->lo / hi / n_local are set.
int lmx_scan_build_slots(lmx_ctx *ctx, const uint32_t *newid, unsigned long long *tied_slots) {
    cudaStream_t st = ctx->stream;
    const unsigned long long m = (unsigned long long)ctx->m, lo = ctx->lo, nl = ctx->hi - ctx->lo;
    // 1. owned segment offsets
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->vbeg, (nl + 1) * 8, "vbeg"));
    k_owned_deg<<<lgrid(ctx, nl + 1), kBlock, 0, st>>>(ctx->deg0, lo, nl, ctx->vbeg);
    LMX_CUDA(ctx, cudaGetLastError());
    unsigned long long *cnt = nullptr;
    LMX_TRY(lmx_alloc(ctx, (void **)&cnt, 32, "counts"));
    LMX_CUDA(ctx, cudaMemsetAsync(cnt, 0, 32, st));
    {
        size_t tmp = 0;
        LMX_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st));
        void *t = nullptr;
        LMX_TRY(lmx_alloc(ctx, &t, tmp, "scan tmp"));
        cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st);
        // huge segments: the leading vertices of a degree-sorted (relabelled) range
        if (e == cudaSuccess && ctx->relabeled && nl) {
            k_count_huge<<<lgrid(ctx, nl), kBlock, 0, st>>>(ctx->deg0, lo, nl, LMX_HUGE_DEG, cnt + 2);
            e = cudaGetLastError();
        }
        cudaStreamSynchronize(st);
        lmx_free(ctx, &t, tmp);
        LMX_CUDA(ctx, e);
    }
    unsigned long long S = 0, H = 0, Hs = 0;
    LMX_CUDA(ctx, cudaMemcpyAsync(&S, ctx->vbeg + nl, 8, cudaMemcpyDeviceToHost, st));
    LMX_CUDA(ctx, cudaMemcpyAsync(&H, cnt + 2, 8, cudaMemcpyDeviceToHost, st));
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    if (H) {
        LMX_CUDA(ctx, cudaMemcpyAsync(&Hs, ctx->vbeg + H, 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
    }
    ctx->slots_local = (int64_t)S;
    const size_t S1 = std::max<unsigned long long>(S, 1);
    // 2. scatter (ids0 is allocated first so it stays with the graph)
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ids0, S1 * 8, "ids0"));
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    uint2 *vals = nullptr;
    uint32_t *fill = nullptr, *sowner = nullptr, *howner = nullptr, *hidx = nullptr, *hidx2 = nullptr,
             *hok = nullptr, *hok2 = nullptr;
    unsigned long long *hkey2 = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    auto ensure_tmp = [&](size_t need) -> int {
        if (need <= tmp_bytes) return LMX_OK;
        lmx_free(ctx, &tmp, tmp_bytes);
        tmp_bytes = need;
        return lmx_alloc(ctx, &tmp, tmp_bytes, "sort tmp");
    };
    const size_t Hs1 = std::max<unsigned long long>(Hs, 1);
    do {
        if ((rc = lmx_alloc(ctx, (void **)&keys, S1 * 8, "slot keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&keys2, S1 * 8, "slot keys out")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&vals, S1 * 8, "slot values")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&fill, std::max<unsigned long long>(nl, 1) * 4, "slot fill")) != LMX_OK)
            break;
        if ((rc = lmx_alloc(ctx, (void **)&howner, Hs1 * 4, "huge owners")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->lowpair, std::max<unsigned long long>(std::min(m, S), 1) * 8,
                            "lowpair")) != LMX_OK)
            break;
        cudaError_t e = cudaMemsetAsync(fill, 0, std::max<unsigned long long>(nl, 1) * 4, st);
        if (e == cudaSuccess && m) {
            k_scan_scatter<<<lgrid(ctx, m), kBlock, 0, st>>>(ctx->eu, ctx->ev, ctx->w, m, newid, (uint32_t)lo,
                                                            (uint32_t)nl, (uint32_t)H, ctx->vbeg, fill, cnt + 3, keys,
                                                            vals, howner);
            e = cudaGetLastError();
        }
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "slot scatter"); break; }
        trace_mark(ctx, "  scan: scatter");
        lmx_free(ctx, (void **)&fill, std::max<unsigned long long>(nl, 1) * 4);
        // 3a. huge region [0, Hs): sort by key (descending), then stably by owner
        if (Hs) {
            if ((rc = lmx_alloc(ctx, (void **)&hidx, Hs1 * 4, "huge idx")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&hidx2, Hs1 * 4, "huge idx2")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&hkey2, Hs1 * 8, "huge keys2")) != LMX_OK) break;
            k_iota<<<lgrid(ctx, Hs), kBlock, 0, st>>>(hidx, Hs);
            int hb = 1;
            while (hb < 32 && (1ULL << hb) < H) ++hb;
            size_t need = 0, need2 = 0;
            e = cub::DeviceRadixSort::SortPairsDescending(nullptr, need, keys, hkey2, hidx, hidx2, (long long)Hs, 0,
                                                          64, st);
            if (e == cudaSuccess)
                e = cub::DeviceRadixSort::SortPairs(nullptr, need2, hidx, hidx2, hidx, hidx2, (long long)Hs, 0, hb, st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "huge sort sizing"); break; }
            if ((rc = ensure_tmp(std::max(need, need2))) != LMX_OK) break;
            e = cub::DeviceRadixSort::SortPairsDescending(tmp, need, keys, hkey2, hidx, hidx2, (long long)Hs, 0, 64,
                                                          st);
            lmx_free(ctx, (void **)&hkey2, Hs1 * 8);
            // hidx2 = positions in key order; stable sort of their owners
            if ((rc = lmx_alloc(ctx, (void **)&hok, Hs1 * 4, "huge owner keys")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&hok2, Hs1 * 4, "huge owner keys2")) != LMX_OK) break;
            if (e == cudaSuccess) {
                k_huge_owner_keys<<<lgrid(ctx, Hs), kBlock, 0, st>>>(howner, hidx2, Hs, hok);
                e = cub::DeviceRadixSort::SortPairs(tmp, need2, hok, hok2, hidx2, hidx, (long long)Hs, 0, hb, st);
            }
            if (e == cudaSuccess) {
                k_huge_gather<<<lgrid(ctx, Hs), kBlock, 0, st>>>(hidx, Hs, keys, vals, keys2, ctx->ids0);
                e = cudaGetLastError();
            }
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "huge sort"); break; }
            trace_mark(ctx, "  scan: huge segments");
        }
        // 3b. the other segments: segmented sort, descending, in chunks of
        // <= 2^30 slots (cub's item count is an int); keys -> keys2, vals -> ids0
        // as cub double buffers, each chunk's result normalised to (keys2, ids0)
        if (S > Hs) {
            const unsigned long long kChunk = 1ULL << 30;
            const int nc = (int)((S - Hs + kChunk - 1) / kChunk);
            unsigned long long *dcuts = nullptr;
            if ((rc = lmx_alloc(ctx, (void **)&dcuts, (size_t)(nc + 1) * 8, "chunk cuts")) != LMX_OK) break;
            std::vector<unsigned long long> cuts((size_t)nc + 1), hv((size_t)nc + 1);
            k_chunk_cuts<<<1, 64, 0, st>>>(ctx->vbeg, H, nl, kChunk, nc, dcuts);
            e = cudaMemcpyAsync(cuts.data(), dcuts, (size_t)(nc + 1) * 8, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            lmx_free(ctx, (void **)&dcuts, (size_t)(nc + 1) * 8);
            for (int k = 0; k <= nc && e == cudaSuccess; ++k)
                e = cudaMemcpy(&hv[(size_t)k], ctx->vbeg + cuts[(size_t)k], 8, cudaMemcpyDeviceToHost);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "chunk cuts"); break; }
            for (int k = 0; k < nc && rc == LMX_OK; ++k) {
                const unsigned long long v0 = cuts[(size_t)k], v1 = cuts[(size_t)k + 1];
                const unsigned long long base = hv[(size_t)k], items = hv[(size_t)k + 1] - base;
                if (items == 0 || v1 <= v0) continue;
                cub::TransformInputIterator<long long, SubBase, const unsigned long long *> beg(ctx->vbeg + v0,
                                                                                             SubBase{base});
                cub::TransformInputIterator<long long, SubBase, const unsigned long long *> end(ctx->vbeg + v0 + 1,
                                                                                             SubBase{base});
                cub::DoubleBuffer<unsigned long long> dk(keys + base, keys2 + base);
                cub::DoubleBuffer<uint2> dv(vals + base, ctx->ids0 + base);
                size_t need = 0;
                e = cub::DeviceSegmentedSort::SortPairsDescending(nullptr, need, dk, dv, (int)items, (int)(v1 - v0),
                                                                  beg, end, st);
                if (e != cudaSuccess) break;
                if ((rc = ensure_tmp(need)) != LMX_OK) break;
                e = cub::DeviceSegmentedSort::SortPairsDescending(tmp, need, dk, dv, (int)items, (int)(v1 - v0), beg,
                                                                  end, st);
                if (e == cudaSuccess && dk.Current() != keys2 + base)
                    e = cudaMemcpyAsync(keys2 + base, dk.Current(), items * 8, cudaMemcpyDeviceToDevice, st);
                if (e == cudaSuccess && dv.Current() != ctx->ids0 + base)
                    e = cudaMemcpyAsync(ctx->ids0 + base, dv.Current(), items * 8, cudaMemcpyDeviceToDevice, st);
                if (e != cudaSuccess) break;
            }
            if (rc != LMX_OK) break;
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "segmented sort"); break; }
            trace_mark(ctx, "  scan: segmented sort");
        }
        lmx_free(ctx, (void **)&keys, S1 * 8);
        lmx_free(ctx, (void **)&vals, S1 * 8);
        lmx_free(ctx, &tmp, tmp_bytes);
        // 4. owners, tie flags, round-0 candidates, lowpair
        if ((rc = lmx_alloc(ctx, (void **)&ctx->cand0, std::max<unsigned long long>(nl, 1) * 8, "cand0")) != LMX_OK)
            break;
        if ((rc = lmx_alloc(ctx, (void **)&sowner, S1 * 4, "slot owners")) != LMX_OK) break;
        e = cudaMemsetAsync(ctx->cand0, 0xFF, std::max<unsigned long long>(nl, 1) * 8, st);
        if (e == cudaSuccess && nl) {
            k_slot_owner<<<ctx->num_sms * 16, kBlock, 0, st>>>(ctx->vbeg, nl, sowner);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess && S) {
            k_scan_post<<<lgrid(ctx, S), kBlock, 0, st>>>(keys2, ctx->ids0, sowner, S, (uint32_t)lo, ctx->cand0,
                                                         ctx->lowpair, cnt);
            e = cudaGetLastError();
        }
        unsigned long long hc[2] = {0, 0};
        if (e == cudaSuccess) e = cudaMemcpyAsync(hc, cnt, 16, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "slot flags"); break; }
        trace_mark(ctx, "  scan: flags + lowpair");
        *tied_slots = hc[0];
        ctx->lowpair_n = hc[1];
        if (ctx->dist_p == 1 && hc[1] != m) { rc = lmx_fail(ctx, LMX_ECUDA, "internal: lowpair count"); break; }
    } while (0);
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&keys, S1 * 8);
    lmx_free(ctx, (void **)&keys2, S1 * 8);
    lmx_free(ctx, (void **)&vals, S1 * 8);
    lmx_free(ctx, (void **)&fill, std::max<unsigned long long>(nl, 1) * 4);
    lmx_free(ctx, (void **)&sowner, S1 * 4);
    lmx_free(ctx, (void **)&howner, Hs1 * 4);
    lmx_free(ctx, (void **)&hidx, Hs1 * 4);
    lmx_free(ctx, (void **)&hidx2, Hs1 * 4);
    lmx_free(ctx, (void **)&hkey2, Hs1 * 8);
    lmx_free(ctx, (void **)&hok, Hs1 * 4);
    lmx_free(ctx, (void **)&hok2, Hs1 * 4);
    lmx_free(ctx, (void **)&cnt, 32);
    lmx_free(ctx, &tmp, tmp_bytes);
    return rc;
}
