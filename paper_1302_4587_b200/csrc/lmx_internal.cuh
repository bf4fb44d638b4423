// lmx_internal.cuh -- shared definitions of the B200 local max engine.
//
// Device data layout:
//   vbeg    u64[n+1]   CSR segment starts (graph.py:108-115 offsets, rebuilt on
//                      the device from the edge arrays)
//   ids0    uint2[2m]  pristine slot records {nbr, id} grouped by owner, where
//                      id is the edge id (layouts UNIFORM, GENERAL) or the
//                      edge's weight key (layout DISTINCT, see below); the
//                      scan loop's segments are weight-descending with
//                      {nbr | tie flags, edge id} (lmx_scanload.cu)
//   wk0     u32[2m]    GENERAL layout only: dense rank of the canonical weight
//                      bits (tiebreak.py:105-113 order) of the slot's edge
//   ids1/wk1           working copy: round 1 compacts the survivors of ids0 into
//                      it, rounds >= 2 compact it in place, so ids0 is never
//                      written and lmx_match can rerun on the same graph
//   vdeg    u32[n]     live degree of each vertex (live prefix of its segment)
//   cand    uint2[n]   {nbr, id} of the vertex's candidate (max key) edge
//   matched u32[n/32]  bitmap of matched vertices
//   lists   u32        per round, 5 degree buckets of live vertices (ping-pong)
//
// Weight-key layouts (chosen in K0 from the weight multiset):
//   UNIFORM  every weight equal: the key is the salt alone, id = edge id
//   DISTINCT at most a few tied weights: id = x is itself the weight key:
//            x < D (number of distinct weight values) -> unique weight of
//            dense rank x; x >= D -> tied edge t = x - D with rank
//            tie_rank[t] and edge id eid_of_x[x].  8-byte slots, no salt
//            hashing unless two tied edges meet.  eid_of_x[] maps back.
//   GENERAL  otherwise: id = edge id plus a u32 weight rank per slot (12 B)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/lmx.h"

namespace lmx {

constexpr uint32_t kNone = 0xFFFFFFFFu;
// scan-loop slot records {nbr | flags, edge id} (lmx_scanload.cu): the slot's
// weight equals a neighbouring slot's in its segment / it starts such a run
constexpr uint32_t kSlotTied = 0x80000000u;
constexpr uint32_t kSlotRunStart = 0x40000000u;
constexpr uint32_t kSlotNbr = 0x3FFFFFFFu;   // the scan loop needs n < 2^30
constexpr int kBlock = 256;   // threads per block, every kernel
constexpr int kWarps = kBlock / 32;

// live-degree buckets of the per-round vertex lists and their mappings
//   0: d <= 4            thread per vertex
//   1: 5 <= d <= 32      8-lane group per vertex
//   2: 33 <= d <= 1024   warp per vertex
//   3: 1025 <= d < 32768 block per vertex
//   4: d >= 32768        block per vertex, scheduled first
// compacting loop live-degree buckets: 0: <= 4 a thread per vertex,
// 5: <= 16 a group of 4 lanes, 1: <= 32 a group of 8 lanes, 2: <= 1024 a
// warp, 3: < 32768 a block, 4: hubs, a block each (bucket 5 is numbered last
// so the others keep their indices; 2-lane groups for degree 5..8 measured
// slower: ER-24 unit 4.2 against 3.4 ms)
constexpr int kBuckets = 6;
__host__ __device__ __forceinline__ int bucket_of(uint32_t d) {
    return d <= 4 ? 0 : d <= 16 ? 5 : d <= 32 ? 1 : d <= 1024 ? 2 : d < 32768 ? 3 : 4;
}

enum Layout { kUniform = 0, kDistinct = 1, kGeneral = 2 };

// Per-round device counters.  n[b] sizes round r's bucket lists (written by
// round r-1's match kernel, or set from the round-0 lists).
struct RoundCtr {
    unsigned long long live_slots;   // sum of post-filter live degrees (= 2 m_r)
    unsigned long long matched_v;    // vertices matched this round (= 2 * matched edges)
    unsigned long long slot_reads;   // slots read by the round kernel
    unsigned int n[kBuckets];        // list sizes of this round
    unsigned int cur[kBuckets];      // work cursors of the round kernel
    unsigned int pad[2];
};

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t v) {
    // tiebreak.py:28-37 (SplitMix64 finalizer, wrapping u64)
    uint64_t x = v + 0x9E3779B97F4A7C15ULL;
    x ^= x >> 30;
    x *= 0xBF58476D1CE4E5B9ULL;
    x ^= x >> 27;
    x *= 0x94D049BB133111EBULL;
    x ^= x >> 31;
    return x;
}

inline uint64_t round_seed(uint64_t seed_masked, uint64_t r, bool rerandomize) {
    // tiebreak.py:40-52
    return mix64(mix64(seed_masked) ^ (rerandomize ? r : 0));
}

}  // namespace lmx

struct lmx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    int round_grid[3][3] = {};   // persistent grid of each round-kernel instance [MODE][LAYOUT]
    int match_blocks = 0;
    int scan_grid[3] = {0, 0, 0};   // scan probe grids (round 0, rounds >= 1 one-phase, two-phase)
    int scan_last_rounds = -1;   // rounds of this context's last scan-loop matching (-1: none yet); a
                                 // hint for the first batch only, kept across loads (results never depend on it)
    int scan_match_grid = 0;
    int scan_loop_grid = 0;      // persistent cooperative round loop (0: not available)
    uint32_t *loop_aux = nullptr;        // device: [0] round count, then u64 stamps [2 ctr_cap + 2]
    uint32_t *loop_host = nullptr;       // pinned mirror
    std::string err;

    // graph
    int64_t n = 0, m = 0;
    int layout = lmx::kUniform;
    uint32_t *eu = nullptr, *ev = nullptr;   // edge endpoints (u32)
    double *w = nullptr;                     // edge weights
    unsigned long long *vbeg = nullptr;      // n+1
    uint2 *ids0 = nullptr, *ids1 = nullptr;
    uint32_t *wk0 = nullptr, *wk1 = nullptr; // GENERAL layout
    uint32_t *deg0 = nullptr;                // full degree (u32)
    // DISTINCT layout tables
    uint32_t n_distinct = 0;                 // D
    uint32_t n_tied = 0;
    uint32_t *eid_of_x = nullptr;            // [D + n_tied] -> edge id
    uint32_t *tie_rank = nullptr;            // [n_tied]
    // round-0 bucket lists (built once per graph, ascending vertex id)
    uint32_t *bins0 = nullptr;               // kBuckets regions of capacity n
    unsigned int n_bins0[lmx::kBuckets] = {};

    // match state
    uint32_t *vdeg = nullptr;
    uint2 *cand = nullptr;
    uint32_t *matched = nullptr;
    uint32_t *lists[2] = {nullptr, nullptr}; // ping-pong, kBuckets regions of capacity n
    long long *mids = nullptr;               // matched edge ids, ascending (staging for host outputs)
    uint32_t *ebits = nullptr;               // matched edge-id bitmap, (m + 31) / 32 words
    uint32_t *ebits_off = nullptr;           // per-word exclusive popcount prefix
    lmx::RoundCtr *ctr = nullptr;
    lmx::RoundCtr *ctr_host = nullptr;       // pinned mirror
    int ctr_cap = 0;
    long long *mate = nullptr;               // int64[n]
    long long *mate_target = nullptr;        // where this lmx_match writes mate
    void *sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int64_t dev_bytes = 0;
    int64_t peak_bytes = 0;                  // high-water mark of dev_bytes (LMX_QUERY_PEAK_BYTES)

    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    lmx_timing timing{};
    std::vector<lmx_round_stats> rounds;     // trace of the last lmx_match
    bool kernel_timing = false;
    std::vector<cudaEvent_t> tl_events;      // per-kernel timeline (kernel_timing)
    std::vector<float> kernel_ms;            // its durations: round, match, round, ...
    int force_layout = -1;                   // testing: force a weight-key layout
    int force_relabel = -1;                  // -1 auto (skewed graphs), 0 off, 1 on, 2 once (no scan loop relabel)
    bool relabeled = false;                  // device vertex ids are degree-sorted
    uint32_t *oldid = nullptr;               // device id -> caller's vertex id
    // round-loop algorithm: 0 = compacting rounds (lmx_round.cu),
    // 1 = weight-ordered scan (lmx_scan.cu; DISTINCT layout, single partition)
    int algo = 0;
    int force_algo = -1;                     // -1 auto, 0 compact, 1 scan (if eligible)
    bool scan_rejected = false;              // load time: ties too common for the scan loop
    unsigned long long key32_fallback_m = 0; // the last 32-bit-key weight order fell back at this m
    // rerandomize=False (salts fixed for the run): a load may lay tie-heavy
    // weights out in the total order (weight, salt of round 0) of one seed,
    // which the scan loop then matches with no tie handling
    bool static_order = false;               // option: lay out for static_seed
    uint64_t static_seed = 0;                // masked seed of the next load
    bool static_layout = false;              // the loaded graph is laid out so
    uint64_t static_rs = 0;                  // ... for this round-0 seed
    // partitions (dist_p > 1): after the cut search, eu/ev/w hold only the edges
    // incident to the owned range ("local edges", caller ids), geid their global ids
    bool dist_local = false;
    int64_t m_local = 0;
    uint32_t *geid = nullptr;                // local edge -> global edge id (null: identity)
    int w_uniform = -1;                      // all weights equal (global; decided before the filter)
    uint32_t *slot_side = nullptr;           // partitions: bit per owned slot, 1 = the owner is the edge's v end
    // distributed RMAT build state (lmx_dist_rmat_*; freed by lmx_dist_rmat_finish)
    uint32_t *db_bits = nullptr;             // first-occurrence bitmap over the raw positions
    unsigned long long db_words = 0;
    uint32_t *db_pf = nullptr, *db_pu = nullptr, *db_pv = nullptr;   // this rank's built pairs
    double *db_pw = nullptr;
    unsigned long long db_np = 0, db_cap = 0;
    unsigned long long *db_minmax = nullptr; // weight bits min / max of the rank's pairs
    void *db_send = nullptr, *db_recv = nullptr;
    unsigned long long db_send_n = 0, db_recv_n = 0;
    bool dist_requested = false;             // LMX_OPT_DIST_P was set: stepped protocol
    uint32_t *mround = nullptr;              // scan: round each vertex was matched in (~0 never)
    unsigned long long *lowbeg = nullptr;    // scan (load time only): [n+1] offsets of lowpair
    uint2 *lowpair = nullptr;                // scan: each edge once as {higher id, lower id}, by higher id
    uint32_t *mpacked = nullptr;             // scan: mround packed to 4 / 8 bits (n bytes)
    uint2 *cand0 = nullptr;                  // scan: first slot of each segment (round-0 candidates)
    unsigned long long lowpair_n = 0;        // scan: lowpair entries (m; a partition's share when p > 1)
    // red-blue matching (lmx_rbm.cu), allocated on first use per graph
    uint2 *rbm_prop = nullptr, *rbm_acc = nullptr;
    uint32_t *rbm_blue = nullptr;
    uint32_t *rbm_list[2] = {nullptr, nullptr};
    uint32_t *rbm_list0 = nullptr;
    uint32_t rbm_n0 = 0;
    // weight-key stage results held until the slot build (load time only)
    uint32_t *ws_kofe = nullptr;             // weight key per edge (compacting loop)
    uint32_t *ws_rank = nullptr, *ws_eid = nullptr, *ws_tied = nullptr, *ws_tidx = nullptr;   // by sorted position
    cudaStream_t copy_stream = nullptr;      // pinned-host loads: copy engine stream
    cudaEvent_t ev_copy[3] = {nullptr, nullptr, nullptr};
    // host loads: pinned staging ring of the narrowing workers (kept across loads)
    void *stage_host = nullptr;
    size_t stage_bytes = 0;
    std::vector<cudaEvent_t> stage_ev;       // one per ring slot
    cudaStream_t deg_stream = nullptr;       // per-block degree counts behind the copies
    cudaStream_t load_stream = nullptr;      // lmx_load_graph runs here (ordered with the caller's stream)
    cudaStream_t side_stream = nullptr;      // scan loop: matched-edge bits next to the histogram
    int64_t *mate_early = nullptr;           // page-locked host mate output, copied as soon as it is final
    bool mate_early_done = false;
    cudaEvent_t ev_mate = nullptr;
    cudaEvent_t ev_side = nullptr;
    cudaEvent_t ev_load = nullptr;
    cudaEvent_t ev_deg = nullptr;
    unsigned long long *hist = nullptr;      // scan: death-round histogram
    size_t hist_cap = 0;

    // device block cache (lmx_dmalloc / lmx_dfree)
    std::unordered_map<void *, size_t> live;
    std::multimap<size_t, void *> cache;

    // 1D vertex partition (multi-GPU; single GPU = one range [0, n)).  Per-vertex
    // arrays (vbeg, deg0, vdeg, cand, lists) are indexed by the local id v - lo;
    // slot neighbours, the matched bitmap and mate use global (device) ids.
    int dist_p = 1, dist_rank = 0;           // applied at the next load
    unsigned long long lo = 0, hi = 0;       // owned device-id range
    int64_t n_local = 0, slots_local = 0;
    std::vector<int64_t> bounds;             // p + 1 cut points
    uint32_t *remote_ok = nullptr;           // [n_local] partner owner confirmed the edge
    uint2 *pad = nullptr;                    // fixed-capacity exchange A (late rounds): p * capacity records
    size_t pad_cap = 0;
    uint2 *send = nullptr, *recv = nullptr;  // proposal records {global target, edge id}
    uint32_t *send_cnt = nullptr;            // [p] per destination
    size_t send_cap = 0, recv_cap = 0;
    int dist_round = 0;                      // next round of the stepped protocol
    uint64_t dist_seed = 0;
    bool dist_rr = true;
};

// helpers shared by the translation units
int lmx_fail(lmx_ctx *ctx, int code, const std::string &msg);
int lmx_cuda_check(lmx_ctx *ctx, cudaError_t e, const char *what);
int lmx_alloc(lmx_ctx *ctx, void **p, size_t bytes, const char *what);
cudaError_t lmx_dmalloc(lmx_ctx *ctx, void **p, size_t bytes);   // per-context block cache
void lmx_dfree(lmx_ctx *ctx, void *p);
void lmx_flush_cache(lmx_ctx *ctx);
void lmx_free(lmx_ctx *ctx, void **p, size_t bytes);
void lmx_free_graph(lmx_ctx *ctx);
int lmx_setup_slots(lmx_ctx *ctx);   // builds vbeg/ids0/(wk0)/bins0 from eu/ev/w (+ deg0, weight stage)
int lmx_setup_device_edges(lmx_ctx *ctx);   // deg0 + weight stage + lmx_setup_slots for built eu/ev/w
int lmx_alloc_match_state(lmx_ctx *ctx);
int lmx_weight_stage(lmx_ctx *ctx);
int lmx_partition_bounds(lmx_ctx *ctx, std::vector<int64_t> &bounds);   // bsp.py:60-98 on ctx->deg0
// edges held in ctx->eu / ev / w (all of them, or a partition's local edges)
inline int64_t lmx_edges(const lmx_ctx *ctx) { return ctx->dist_local ? ctx->m_local : ctx->m; }
void trace_mark(lmx_ctx *ctx, const char *what);   // LMX_TRACE_SETUP=1: K0 stage times
// scan loop K0 (lmx_scanload.cu): owned weight-descending segments, cand0, lowpair
int lmx_scan_build_slots(lmx_ctx *ctx, const uint32_t *newid);
int lmx_configure_grids(lmx_ctx *ctx);
int lmx_scan_configure_grids(lmx_ctx *ctx);
int lmx_ensure_ctr(lmx_ctx *ctx, int need);
inline size_t lmx_loop_aux_bytes(int cap) { return 8 + 8 * (2 * (size_t)cap + 4); }
// the stepped multi-GPU protocol on the scan loop (lmx_scan.cu)
int lmx_scan_dist_begin(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize);
int lmx_scan_dist_round(lmx_ctx *ctx);
int lmx_scan_dist_propose(lmx_ctx *ctx, void **counts_dev, void **packed_dev);
int lmx_scan_dist_accept(lmx_ctx *ctx, int64_t count);
int lmx_scan_dist_pad(lmx_ctx *ctx, int64_t C, void **padded_dev, void **overflow_dev);
int lmx_scan_dist_match(lmx_ctx *ctx, void **stats_dev);
int lmx_scan_dist_hist(lmx_ctx *ctx, int n_rounds, void **hist_dev, int *nbins);
namespace lmx {
// exchange-A packing (lmx_round.cu), shared by both round loops
__global__ void lmx_pack_kernel(const uint2 *region, const uint32_t *cnt, int p, uint32_t nl, uint2 *packed,
                                long long *counts64);
}  // namespace lmx
int lmx_rbm_impl(lmx_ctx *ctx, uint64_t seed_masked, int max_rounds, std::vector<lmx_round_stats> &stats,
                 unsigned long long &n_matched);
int lmx_validate_impl(lmx_ctx *ctx, const int64_t *mate, const int64_t *ids, int64_t n_ids, int where,
                      int *valid, int *maximal, double *weight, char *detail, size_t detail_len);
int lmx_run_rounds_scan(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                        std::vector<lmx_round_stats> &stats, unsigned long long &n_matched);
int lmx_load_edges(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                   const double *edge_weight, int where);
int lmx_run_rounds(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                   std::vector<lmx_round_stats> &stats, unsigned long long &n_matched);
int lmx_emit_outputs(lmx_ctx *ctx, unsigned long long n_matched, int64_t *mate_out,
                     int64_t *ids_out, int out_where);
int lmx_dist_begin_impl(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize);
int lmx_dist_round_impl(lmx_ctx *ctx);
int lmx_dist_propose_impl(lmx_ctx *ctx, void **counts_dev, void **packed_dev);
int lmx_dist_recv_impl(lmx_ctx *ctx, int64_t count, void **ptr);
int lmx_dist_accept_impl(lmx_ctx *ctx, int64_t count);
int lmx_dist_match_impl(lmx_ctx *ctx, void **stats_dev);

#define LMX_CUDA(ctx, expr)                                          \
    do {                                                             \
        cudaError_t _e = (expr);                                     \
        if (_e != cudaSuccess) return lmx_cuda_check(ctx, _e, #expr); \
    } while (0)
#define LMX_TRY(expr)                  \
    do {                               \
        int _s = (expr);               \
        if (_s != LMX_OK) return _s;   \
    } while (0)
