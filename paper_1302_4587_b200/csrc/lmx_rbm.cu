// lmx_rbm.cu -- red-blue matching (rbm, matchers.py:357-410) on the device:
// the paper's GPU competitor, same results as the
// reference (mate, matched ids, RoundStats).
//
// Per round r (rs = round_seed(seed, r, rerandomize=True)):
//   coins    blue(v) = mix64(v ^ rs ^ COIN) & 1 over the caller's vertex ids
//            (tiebreak.py:62-71), one bitmap for the round
//   propose  every live vertex counts its live slots (neighbour unmatched);
//            a blue one picks its max-key live edge to a red neighbour
//            (key = local max's (weight, salt, edge id), tiebreak.py:74-102)
//   accept   a red vertex takes the max-key edge among those proposed to it
//   match    accepted pairs are matched; edges at matched vertices die
// A vertex keeps no state across rounds (prop/acc are rewritten every round,
// matchers.py:395-399).  Slots are read from the pristine ids0 of any layout
// and filtered by the matched bitmap; a vertex whose slots are all dead leaves
// the list.
#include <cub/cub.cuh>

#include <algorithm>
#include <vector>

#include "lmx_internal.cuh"

namespace lmx {

constexpr uint64_t kCoinStream = 0xD6E8FEB86659FD93ULL;   // tiebreak.py:25

struct RbmArgs {
    const unsigned long long *vbeg;
    const uint32_t *deg0;
    const uint2 *ids;          // pristine slots {nbr, id}
    const uint32_t *wk;        // GENERAL layout: weight rank per slot (else null)
    const double *w;           // scan-loop slots: the edge weights (rank = canonical bits)
    int layout;                // kUniform / kDistinct / kGeneral, or kScanSlots
    uint32_t D;
    const uint32_t *tie_rank;
    const uint32_t *eid_of_x;
    const uint32_t *matched;
    const uint32_t *blue;      // coin bitmap of this round
    uint2 *prop;               // blue v: {nbr, id} of its proposal (kNone: none)
    uint2 *acc;                // red v: {nbr, id} of the accepted proposal
    const uint32_t *lin;       // candidate vertices of this round
    uint32_t *lout;            // vertices with live slots this round
    RoundCtr *ctr;             // ctr[r]: pad[0] = |lin|; live_slots; matched_v
    RoundCtr *ctr_next;        // ctr[r+1].pad[0] = |lout|
    uint64_t rs;
};

constexpr int kScanSlots = 3;   // ids0 of the scan loop: {nbr | tie flags, edge id}

struct Key {
    uint64_t rank;
    uint32_t id;
    uint32_t nbr;
    uint64_t salt;
};

__device__ __forceinline__ uint32_t eid_of(const RbmArgs &a, uint32_t id) {
    return a.layout == kDistinct ? a.eid_of_x[id] : id;
}

__device__ __forceinline__ uint64_t rank_of(const RbmArgs &a, uint32_t id, unsigned long long slot) {
    if (a.layout == kDistinct) return id < a.D ? id : a.tie_rank[id - a.D];
    if (a.layout == kGeneral) return a.wk[slot];
    if (a.layout == kScanSlots) {   // canonical weight bits (tiebreak.py:105-113)
        const unsigned long long b = (unsigned long long)__double_as_longlong(a.w[id]);
        return (b << 1) == 0 ? 0ULL : b;
    }
    return 0u;
}

__device__ __forceinline__ uint2 slot_at(const RbmArgs &a, unsigned long long i) {
    uint2 s = a.ids[i];
    if (a.layout == kScanSlots) s.x &= kSlotNbr;
    return s;
}

// lexicographic (rank, salt) max; the edge id never decides (distinct salts)
__device__ __forceinline__ void key_offer(Key &b, uint64_t rank, uint32_t id, uint32_t nbr, const RbmArgs &a) {
    if (b.nbr != kNone && rank < b.rank) return;
    const uint64_t s = mix64((uint64_t)eid_of(a, id) ^ a.rs);
    if (b.nbr == kNone || rank > b.rank || s > b.salt) {
        b.rank = rank;
        b.id = id;
        b.nbr = nbr;
        b.salt = s;
    }
}

__device__ __forceinline__ Key key_warp_max(Key b) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Key o;
        o.rank = __shfl_xor_sync(0xffffffffu, (unsigned long long)b.rank, off);
        o.id = __shfl_xor_sync(0xffffffffu, b.id, off);
        o.nbr = __shfl_xor_sync(0xffffffffu, b.nbr, off);
        o.salt = __shfl_xor_sync(0xffffffffu, (unsigned long long)b.salt, off);
        if (o.nbr != kNone && (b.nbr == kNone || o.rank > b.rank || (o.rank == b.rank && o.salt > b.salt))) b = o;
    }
    return b;
}

__device__ __forceinline__ bool bit(const uint32_t *bits, uint32_t v) { return (bits[v >> 5] >> (v & 31)) & 1u; }

__global__ void k_rbm_coins(unsigned long long n, const uint32_t *oldid, uint64_t rs, uint32_t *blue) {
    const unsigned long long words = (n + 31) / 32;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long w = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; w < words; w += stride) {
        uint32_t x = 0;
        for (uint32_t j = 0; j < 32; ++j) {
            const unsigned long long v = w * 32 + j;
            if (v >= n) break;
            const uint64_t caller = oldid ? (uint64_t)oldid[v] : (uint64_t)v;
            x |= (uint32_t)(mix64(caller ^ rs ^ kCoinStream) & 1ULL) << j;
        }
        blue[w] = x;
    }
}

// warp per vertex of lin: live count, lout, blue proposals
__global__ void __launch_bounds__(kBlock) k_rbm_propose(RbmArgs a) {
    const uint32_t na = a.ctr->pad[0];
    const int lane = threadIdx.x & 31;
    unsigned long long live_sum = 0;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = gw; i < na; i += nw) {
        const uint32_t v = a.lin[i];
        if (bit(a.matched, v)) continue;
        const unsigned long long b = a.vbeg[v];
        const uint32_t d = a.deg0[v];
        const bool vblue = bit(a.blue, v);
        Key best;
        best.nbr = kNone;
        best.rank = 0;
        best.id = kNone;
        best.salt = 0;
        uint32_t live = 0;
        for (uint32_t c = 0; c < d; c += 32) {
            const uint32_t k = c + lane;
            bool alive = false;
            uint2 s = make_uint2(kNone, kNone);
            if (k < d) {
                s = slot_at(a, b + k);
                alive = !bit(a.matched, s.x);
            }
            live += __popc(__ballot_sync(0xffffffffu, alive));
            if (alive && vblue && !bit(a.blue, s.x)) key_offer(best, rank_of(a, s.y, b + k), s.y, s.x, a);
        }
        best = key_warp_max(best);
        if (lane == 0) {
            a.prop[v] = vblue ? make_uint2(best.nbr, best.id) : make_uint2(kNone, kNone);
            if (live) {
                const uint32_t p = atomicAdd(&a.ctr_next->pad[0], 1u);
                a.lout[p] = v;
                live_sum += live;
            }
        }
    }
    if (lane == 0 && live_sum) atomicAdd(&a.ctr->live_slots, live_sum);
}

// warp per red vertex of lout: the max-key proposal it received
__global__ void __launch_bounds__(kBlock) k_rbm_accept(RbmArgs a) {
    const uint32_t na = a.ctr_next->pad[0];
    const int lane = threadIdx.x & 31;
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t i = gw; i < na; i += nw) {
        const uint32_t v = a.lout[i];
        if (bit(a.blue, v)) continue;
        const unsigned long long b = a.vbeg[v];
        const uint32_t d = a.deg0[v];
        Key best;
        best.nbr = kNone;
        best.rank = 0;
        best.id = kNone;
        best.salt = 0;
        for (uint32_t c = 0; c < d; c += 32) {
            const uint32_t k = c + lane;
            if (k < d) {
                const uint2 s = slot_at(a, b + k);
                if (!bit(a.matched, s.x) && bit(a.blue, s.x)) {
                    const uint2 p = a.prop[s.x];
                    if (p.x == v && p.y == s.y) key_offer(best, rank_of(a, s.y, b + k), s.y, s.x, a);
                }
            }
        }
        best = key_warp_max(best);
        if (lane == 0) a.acc[v] = make_uint2(best.nbr, best.id);
    }
}

struct RbmMatchArgs {
    const uint32_t *lout;
    const uint32_t *blue;
    const uint2 *acc;
    uint32_t *matched;
    long long *mate;
    const uint32_t *oldid;
    uint32_t *ebits;
    int layout;
    const uint32_t *eid_of_x;
    RoundCtr *ctr;
    RoundCtr *ctr_next;
};

// thread per red vertex of lout with an accepted proposal: match the pair
__global__ void k_rbm_match(RbmMatchArgs a) {
    const uint32_t na = a.ctr_next->pad[0];
    unsigned long long mv = 0;
    const uint32_t stride = gridDim.x * blockDim.x;
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < na; i += stride) {
        const uint32_t v = a.lout[i];
        if (bit(a.blue, v)) continue;
        const uint2 c = a.acc[v];
        if (c.x == kNone) continue;
        const uint32_t x = c.x;
        atomicOr(a.matched + (v >> 5), 1u << (v & 31));
        atomicOr(a.matched + (x >> 5), 1u << (x & 31));
        const uint32_t cv = a.oldid ? a.oldid[v] : v, cx = a.oldid ? a.oldid[x] : x;
        a.mate[cv] = (long long)cx;
        a.mate[cx] = (long long)cv;
        const uint32_t e = a.layout == kDistinct ? a.eid_of_x[c.y] : c.y;
        atomicOr(a.ebits + (e >> 5), 1u << (e & 31));
        mv += 2;
    }
    for (int off = 16; off > 0; off >>= 1) mv += __shfl_xor_sync(0xffffffffu, mv, off);
    if ((threadIdx.x & 31) == 0 && mv) atomicAdd(&a.ctr->matched_v, mv);
}

struct HasEdgeR {
    const uint32_t *deg;
    __device__ bool operator()(uint32_t v) const { return deg[v] > 0; }
};

}  // namespace lmx

using namespace lmx;

int lmx_rbm_impl(lmx_ctx *ctx, uint64_t seed_masked, int max_rounds, std::vector<lmx_round_stats> &stats,
                 unsigned long long &n_matched) {
    stats.clear();
    n_matched = 0;
    if (ctx->dist_p > 1) return lmx_fail(ctx, LMX_ESTATE, "rbm runs on a whole-graph context (no partition)");
    const unsigned long long n = (unsigned long long)ctx->n, m = (unsigned long long)ctx->m;
    const size_t nn = std::max<size_t>(n, 1);
    cudaStream_t st = ctx->stream;
    ctx->timing.round_launches = 0;
    // per-graph RBM buffers
    if (!ctx->rbm_prop) {
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->rbm_prop, nn * 8, "rbm proposals"));
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->rbm_acc, nn * 8, "rbm accepts"));
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->rbm_blue, (nn + 31) / 32 * 4, "rbm coins"));
        for (int i = 0; i < 2; ++i) LMX_TRY(lmx_alloc(ctx, (void **)&ctx->rbm_list[i], nn * 4, "rbm lists"));
        unsigned long long *cnt = nullptr;
        LMX_TRY(lmx_alloc(ctx, (void **)&cnt, 8, "rbm count"));
        cub::CountingInputIterator<uint32_t> it(0);
        size_t tmp = 0;
        LMX_CUDA(ctx, cub::DeviceSelect::If(nullptr, tmp, it, ctx->rbm_list[0], cnt, (long long)n, HasEdgeR{ctx->deg0},
                                            st));
        void *t = nullptr;
        LMX_TRY(lmx_alloc(ctx, &t, tmp, "select tmp"));
        unsigned long long h = 0;
        cudaError_t e = cub::DeviceSelect::If(t, tmp, it, ctx->rbm_list[0], cnt, (long long)n, HasEdgeR{ctx->deg0}, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        lmx_free(ctx, &t, tmp);
        lmx_free(ctx, (void **)&cnt, 8);
        LMX_CUDA(ctx, e);
        ctx->rbm_n0 = (uint32_t)h;
        // the round-0 list is rbm_list[0]; keep a pristine copy for reruns
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->rbm_list0, nn * 4, "rbm list0"));
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->rbm_list0, ctx->rbm_list[0], (size_t)h * 4, cudaMemcpyDeviceToDevice, st));
    }
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    LMX_TRY(lmx_ensure_ctr(ctx, 64));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ctr, 0, sizeof(RoundCtr) * (size_t)ctx->ctr_cap, st));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->ebits, 0, ((size_t)std::max<unsigned long long>(m, 1) + 31) / 32 * 4, st));
    if (n) {
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->mate_target, 0xFF, n * 8, st));
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->matched, 0, (n + 31) / 32 * 4, st));
    }
    ctx->ctr_host[0] = RoundCtr{};
    ctx->ctr_host[0].pad[0] = ctx->rbm_n0;
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr, ctx->ctr_host, sizeof(RoundCtr), cudaMemcpyHostToDevice, st));
    const int grid = ctx->num_sms * 8;
    int r = 0, n_rounds = -1, batch = 8;
    while (n_rounds < 0 && m > 0) {
        if (r >= max_rounds) return lmx_fail(ctx, LMX_ELIMIT, "rbm: no progress after max_rounds rounds");
        LMX_TRY(lmx_ensure_ctr(ctx, r + batch + 1));
        const int r0 = r;
        for (int b = 0; b < batch; ++b, ++r) {
            RbmArgs a;
            a.vbeg = ctx->vbeg;
            a.deg0 = ctx->deg0;
            a.ids = ctx->ids0;
            a.wk = ctx->wk0;
            a.w = ctx->w;
            a.layout = ctx->algo == 1 ? kScanSlots : ctx->layout;
            a.D = ctx->n_distinct;
            a.tie_rank = ctx->tie_rank;
            a.eid_of_x = ctx->eid_of_x;
            a.matched = ctx->matched;
            a.blue = ctx->rbm_blue;
            a.prop = ctx->rbm_prop;
            a.acc = ctx->rbm_acc;
            a.lin = r == 0 ? ctx->rbm_list0 : ctx->rbm_list[r & 1];
            a.lout = ctx->rbm_list[(r + 1) & 1];
            a.ctr = ctx->ctr + r;
            a.ctr_next = ctx->ctr + r + 1;
            a.rs = round_seed(seed_masked, (uint64_t)r, true);
            k_rbm_coins<<<grid, kBlock, 0, st>>>(n, ctx->relabeled ? ctx->oldid : nullptr, a.rs, ctx->rbm_blue);
            k_rbm_propose<<<grid, kBlock, 0, st>>>(a);
            k_rbm_accept<<<grid, kBlock, 0, st>>>(a);
            RbmMatchArgs ma;
            ma.lout = a.lout;
            ma.blue = ctx->rbm_blue;
            ma.acc = ctx->rbm_acc;
            ma.matched = ctx->matched;
            ma.mate = ctx->mate_target;
            ma.oldid = ctx->relabeled ? ctx->oldid : nullptr;
            ma.ebits = ctx->ebits;
            ma.layout = ctx->algo == 1 ? kScanSlots : ctx->layout;
            ma.eid_of_x = ctx->eid_of_x;
            ma.ctr = ctx->ctr + r;
            ma.ctr_next = ctx->ctr + r + 1;
            k_rbm_match<<<grid, kBlock, 0, st>>>(ma);
            LMX_CUDA(ctx, cudaGetLastError());
            ctx->timing.round_launches += 4;
        }
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->ctr_host + r0, ctx->ctr + r0, sizeof(RoundCtr) * (size_t)batch,
                                      cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        for (int i = r0; i < r; ++i) {
            if (ctx->ctr_host[i].live_slots == 0) {
                n_rounds = i;
                break;
            }
        }
        if (n_rounds < 0 && r >= max_rounds)
            return lmx_fail(ctx, LMX_ELIMIT, "rbm: no progress after max_rounds rounds");
    }
    if (n_rounds < 0) n_rounds = 0;
    if (n_rounds > max_rounds)   // the reference raises once round max_rounds would start
        return lmx_fail(ctx, LMX_ELIMIT, "rbm: no progress after max_rounds rounds");
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
    ctx->timing.rounds_executed = r;
    unsigned long long total_v = 0;
    for (int i = 0; i < n_rounds; ++i) {
        const RoundCtr &c = ctx->ctr_host[i];
        if ((c.live_slots & 1ULL) || (c.matched_v & 1ULL))
            return lmx_fail(ctx, LMX_ECUDA, "internal: odd rbm slot or matched-vertex count");
        lmx_round_stats s;
        s.edges_before = (int64_t)(c.live_slots / 2);
        s.edges_matched = (int64_t)(c.matched_v / 2);
        const unsigned long long nxt = (i + 1 < n_rounds) ? ctx->ctr_host[i + 1].live_slots / 2 : 0;
        s.edges_removed = s.edges_before - (int64_t)nxt;
        stats.push_back(s);
        total_v += c.matched_v;
    }
    n_matched = total_v / 2;
    return LMX_OK;
}
