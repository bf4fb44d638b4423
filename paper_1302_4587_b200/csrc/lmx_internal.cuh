// lmx_internal.cuh -- shared definitions of the B200 local max engine.
//
// Device data layout:
//   vbeg   u64[n+1]   CSR segment starts (graph.py:108-115 offsets, rebuilt
//                     on the device from the edge arrays)
//   ids0   uint2[2m]  pristine slot records {nbr, eid} sorted by owner
//   wk0    u32[2m]    dense rank of the canonical weight bits of the slot's
//                     edge (tiebreak.py:105-113 order, compressed to 32 bits);
//                     absent when every weight is equal (unit weights)
//   ids1/wk1          working copy of the slots: round 1 compacts the
//                     survivors of ids0 into it, rounds >= 2 compact it in
//                     place, so ids0 is never written and lmx_match can rerun
//   vdeg   u32[n]     live degree of each vertex (prefix of its segment)
//   cand   uint2[n]   {nbr, eid} of the vertex's candidate (max key) edge
//   matched u32[n/32] bitmap of matched vertices
//   L/H    u32[n] x2  live vertex lists (ping-pong), H = hubs (deg > HUB_T)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/lmx.h"

namespace lmx {

constexpr uint32_t kNone = 0xFFFFFFFFu;
constexpr int kBlock = 256;            // threads per block, every kernel
constexpr int kWarps = kBlock / 32;
constexpr uint32_t kThreadMax = 8;     // thread-per-vertex up to this live degree
constexpr uint32_t kHubMin = 4097;     // block-per-vertex from this live degree
constexpr int kLanesItems = 8;         // vertices per lane in a warp chunk
constexpr uint32_t kWarpChunk = 32 * kLanesItems;
constexpr int kMaxRounds = 4096;

// Per-round device counters; round r's work lists are sized by ctr[r].nL/nH
// (written by round r-1's match kernel, or by the init kernel for r = 0).
struct RoundCtr {
    unsigned long long live_slots;   // sum of post-filter live degrees (= 2 m_r)
    unsigned long long matched_v;    // vertices matched this round (= 2 * matched edges)
    unsigned long long slot_reads;   // slots read by the round kernel
    unsigned int nL, nH;             // sizes of this round's lists
    unsigned int cur_hub, cur_L;     // work cursors of the round kernel
    unsigned int cur_match, pad;
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
    int round_blocks = 0;   // persistent grid of the round kernel
    int match_blocks = 0;
    std::string err;

    // graph
    int64_t n = 0, m = 0;
    bool has_wk = false;
    uint32_t *eu = nullptr, *ev = nullptr;   // edge endpoints (u32)
    double *w = nullptr;                     // edge weights
    unsigned long long *vbeg = nullptr;      // n+1
    uint2 *ids0 = nullptr, *ids1 = nullptr;
    uint32_t *wk0 = nullptr, *wk1 = nullptr;
    uint32_t *deg0 = nullptr;                // full degree (u32)
    unsigned int n_hubs0 = 0;

    // match state
    uint32_t *vdeg = nullptr;
    uint2 *cand = nullptr;
    uint32_t *matched = nullptr;
    uint32_t *L[2] = {nullptr, nullptr};
    uint32_t *H[2] = {nullptr, nullptr};
    uint32_t *hubs0 = nullptr;
    uint32_t *mids = nullptr;                // matched edge ids (u32)
    uint32_t *mids_sorted = nullptr;
    unsigned long long *mcount = nullptr;    // total matched edges
    lmx::RoundCtr *ctr = nullptr;            // kMaxRounds + 1
    lmx::RoundCtr *ctr_host = nullptr;       // pinned mirror
    int ctr_cap = 0;
    long long *mate = nullptr;               // int64[n]
    void *sort_tmp = nullptr;
    size_t sort_tmp_bytes = 0;
    int64_t dev_bytes = 0;

    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr;
    lmx_timing timing{};
    std::vector<lmx_round_stats> rounds;   // trace of the last lmx_match
    bool kernel_timing = false;
    std::vector<cudaEvent_t> tl_events;    // per-kernel timeline (kernel_timing)
};

// helpers shared by the translation units
int lmx_fail(lmx_ctx *ctx, int code, const std::string &msg);
int lmx_cuda_check(lmx_ctx *ctx, cudaError_t e, const char *what);
int lmx_alloc(lmx_ctx *ctx, void **p, size_t bytes, const char *what);
void lmx_free(lmx_ctx *ctx, void **p, size_t bytes);
void lmx_free_graph(lmx_ctx *ctx);
int lmx_setup_slots(lmx_ctx *ctx);   // builds vbeg/ids0/wk0 from eu/ev/w
int lmx_alloc_match_state(lmx_ctx *ctx);
int lmx_configure_grids(lmx_ctx *ctx);
int lmx_load_edges(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                   const double *edge_weight, int where);
#include <vector>
int lmx_run_rounds(lmx_ctx *ctx, uint64_t seed_masked, bool rerandomize,
                   std::vector<lmx_round_stats> &stats, unsigned long long &n_matched);
int lmx_emit_outputs(lmx_ctx *ctx, unsigned long long n_matched, int64_t *mate_out,
                     int64_t *ids_out, int out_where);

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
