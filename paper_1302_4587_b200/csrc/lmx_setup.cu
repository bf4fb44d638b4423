// lmx_setup.cu -- K0: device slot records from the reference's edge arrays.
//
// The reference keeps a CSR incidence layout (graph.py:108-115: slots sorted
// by (vertex, edge id), offsets = cumsum of degrees).  local_max_seq itself
// only reads edge_u / edge_v / edge_weight (matchers.py:80-92), so the device
// layout is rebuilt here from those arrays:
//   1. validate + narrow to u32  (graph.py:80-88 domain rules)
//   2. degree histogram, exclusive scan -> vbeg (u64 offsets)
//   3. scatter {nbr, eid} slot records (order inside a segment is free: the
//      key order is total)
//   4. weight order: if all canonical weight bits are equal, no weight key;
//      else dense rank of the canonical bits (tiebreak.py:105-113, -0.0 -> 0)
//      as a u32 key per slot.  The rank preserves the reference's uint64
//      comparison exactly, so argmax results are bit-identical.
#include <cub/cub.cuh>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <thread>

#include "lmx_internal.cuh"
#include "lmx_sort.cuh"

using namespace lmx;

int lmx_fail(lmx_ctx *ctx, int code, const std::string &msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int lmx_cuda_check(lmx_ctx *ctx, cudaError_t e, const char *what) {
    std::string m = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) +
                    ") in " + what;
    if (e == cudaErrorMemoryAllocation) return lmx_fail(ctx, LMX_ENOMEM, m);
    return lmx_fail(ctx, LMX_ECUDA, m);
}

// Single choke point for device allocations, with a per-context block cache:
// freed blocks are kept and handed out again to requests that fit (at most 2x
// oversized), so reloading a graph of similar size does not pay cudaFree /
// cudaMalloc of tens of GB again (measured: seconds of jitter per reload).  The
// stream-ordered pool was also measured: growing it on first use cost seconds.
// All work of a context is ordered on its stream, so reuse is safe.
static size_t round_alloc(size_t bytes) {
    const size_t g = bytes >= (64u << 20) ? (2u << 20) : 256;
    return (std::max<size_t>(bytes, 16) + g - 1) / g * g;
}

void lmx_flush_cache(lmx_ctx *ctx) {
    for (auto &kv : ctx->cache) cudaFree(kv.second);
    ctx->cache.clear();
}

cudaError_t lmx_dmalloc(lmx_ctx *ctx, void **p, size_t bytes) {
    bytes = round_alloc(bytes);
    auto it = ctx->cache.lower_bound(bytes);
    if (it != ctx->cache.end() && it->first <= 2 * bytes) {
        *p = it->second;
        ctx->live[*p] = it->first;
        ctx->cache.erase(it);
        return cudaSuccess;
    }
    cudaError_t e = cudaMalloc(p, bytes);
    if (e == cudaErrorMemoryAllocation && !ctx->cache.empty()) {
        cudaGetLastError();
        cudaStreamSynchronize(ctx->stream);
        lmx_flush_cache(ctx);
        e = cudaMalloc(p, bytes);
    }
    if (e == cudaSuccess) ctx->live[*p] = bytes;
    return e;
}

void lmx_dfree(lmx_ctx *ctx, void *p) {
    if (!p) return;
    auto it = ctx->live.find(p);
    if (it == ctx->live.end()) {   // not ours (should not happen): release directly
        cudaFree(p);
        return;
    }
    ctx->cache.emplace(it->second, p);
    ctx->live.erase(it);
}

int lmx_alloc(lmx_ctx *ctx, void **p, size_t bytes, const char *what) {
    if (*p) return LMX_OK;
    cudaError_t e = lmx_dmalloc(ctx, p, bytes);
    if (e != cudaSuccess) {
        cudaGetLastError();
        *p = nullptr;
        return lmx_fail(ctx, e == cudaErrorMemoryAllocation ? LMX_ENOMEM : LMX_ECUDA,
                        std::string("cudaMalloc(") + std::to_string(bytes) + " B) failed for " + what +
                            ": " + cudaGetErrorString(e));
    }
    ctx->dev_bytes += (int64_t)bytes;
    ctx->peak_bytes = std::max(ctx->peak_bytes, ctx->dev_bytes);
    return LMX_OK;
}

void lmx_free(lmx_ctx *ctx, void **p, size_t bytes) {
    if (*p) {
        lmx_dfree(ctx, *p);
        ctx->dev_bytes -= (int64_t)bytes;
        *p = nullptr;
    }
}

void lmx_free_graph(lmx_ctx *ctx) {
    void **ptrs[] = {(void **)&ctx->eu,       (void **)&ctx->ev,          (void **)&ctx->w,
                     (void **)&ctx->vbeg,     (void **)&ctx->ids0,        (void **)&ctx->ids1,
                     (void **)&ctx->wk0,      (void **)&ctx->wk1,         (void **)&ctx->deg0,
                     (void **)&ctx->vdeg,     (void **)&ctx->cand,        (void **)&ctx->matched,
                     (void **)&ctx->lists[0], (void **)&ctx->lists[1],    (void **)&ctx->bins0,
                     (void **)&ctx->mids,     (void **)&ctx->ebits,       (void **)&ctx->ebits_off,
                     (void **)&ctx->mate,     (void **)&ctx->sort_tmp,    (void **)&ctx->eid_of_x,
                     (void **)&ctx->tie_rank, (void **)&ctx->oldid,
                     (void **)&ctx->remote_ok, (void **)&ctx->send, (void **)&ctx->recv,
                     (void **)&ctx->send_cnt, (void **)&ctx->mround, (void **)&ctx->lowbeg,
                     (void **)&ctx->lowpair, (void **)&ctx->hist, (void **)&ctx->mpacked,
                     (void **)&ctx->cand0,    (void **)&ctx->ws_kofe,     (void **)&ctx->ws_rank,
                     (void **)&ctx->ws_eid,   (void **)&ctx->ws_tied,     (void **)&ctx->ws_tidx,
                     (void **)&ctx->rbm_prop, (void **)&ctx->rbm_acc,     (void **)&ctx->rbm_blue,
                     (void **)&ctx->rbm_list[0], (void **)&ctx->rbm_list[1], (void **)&ctx->rbm_list0,
                     (void **)&ctx->geid,     (void **)&ctx->slot_side,
                     (void **)&ctx->db_bits,  (void **)&ctx->db_pf,       (void **)&ctx->db_pu,
                     (void **)&ctx->db_pv,    (void **)&ctx->db_pw,       (void **)&ctx->db_minmax,
                     (void **)&ctx->db_send,  (void **)&ctx->db_recv,     (void **)&ctx->pad};
    for (void **p : ptrs) {
        lmx_dfree(ctx, *p);
        *p = nullptr;
    }
    ctx->dev_bytes = 0;
    ctx->n = ctx->m = 0;
    ctx->dist_local = false;
    ctx->m_local = 0;
    ctx->w_uniform = -1;
    ctx->db_words = ctx->db_np = ctx->db_cap = ctx->db_send_n = ctx->db_recv_n = 0;
    ctx->pad_cap = 0;
    ctx->layout = kUniform;
    ctx->n_distinct = ctx->n_tied = 0;
    ctx->relabeled = false;
    ctx->algo = 0;
    ctx->static_layout = false;
    ctx->hist_cap = 0;
    ctx->send_cap = ctx->recv_cap = 0;
    ctx->n_local = ctx->slots_local = 0;
    for (int q = 0; q < kBuckets; ++q) ctx->n_bins0[q] = 0;
    ctx->sort_tmp_bytes = 0;
}

namespace lmx {

__device__ __forceinline__ unsigned long long canon_bits(double w) {
    unsigned long long b = (unsigned long long)__double_as_longlong(w);
    return (b << 1) == 0 ? 0ULL : b;   // -0.0 -> +0.0 (tiebreak.py:112)
}

// graph.py:80-88: ids in range, weights finite and >= 0; plus no self loops
// (a built Graph has none, graph.py:89-91).  Records the first bad position
// and counts the degrees of the edges it narrows.
__device__ __forceinline__ bool check_uv(long long a, long long b, long long n) {
    return a >= 0 && b >= 0 && a < n && b < n && a != b;
}
__device__ __forceinline__ bool check_w(double x) { return isfinite(x) && !(x < 0.0); }

// Degree count of one endpoint per lane: lanes of a warp holding the same
// vertex add once (edge lists sorted by their first endpoint, as build_graph
// leaves them, repeat it across neighbouring lanes).
__device__ __forceinline__ void add_degree_grouped(uint32_t *deg, uint32_t a, bool on) {
#ifdef LMX_DEG_PLAIN
    if (on) atomicAdd(deg + a, 1u);
#else
    const uint32_t active = __activemask();
    const uint32_t key = on ? a : 0xFFFFFFFFu;
    const uint32_t peers = __match_any_sync(active, key);
    const int lane = threadIdx.x & 31;
    if (on && (__ffs(peers) - 1) == lane) atomicAdd(deg + a, (uint32_t)__popc(peers));
#endif
}

__global__ void k_convert(const long long *u, const long long *v, const double *w,
                          unsigned long long k, long long n, unsigned long long base, uint32_t *eu,
                          uint32_t *ev, double *wout, uint32_t *deg, unsigned long long *bad) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * blockDim.x; i0 < k; i0 += stride) {
        const unsigned long long i = i0 + threadIdx.x;   // whole warps stay in the loop (match_any)
        const bool in = i < k;
        const long long a = in ? u[i] : 0, b = in ? v[i] : 0;
        const double x = in ? w[i] : 0.0;
        const bool uv = in && check_uv(a, b, n);
        if (in) {
            if (!uv || !check_w(x)) atomicMin(bad, base + i);
            eu[base + i] = (uint32_t)a;
            ev[base + i] = (uint32_t)b;
            wout[base + i] = x;
        }
        if (deg) {
            add_degree_grouped(deg, (uint32_t)a, uv);
            if (uv) atomicAdd(deg + b, 1u);
        }
    }
}

// Pinned-host load: endpoints staged by the copy engine, narrowed here.
__global__ void k_convert_uv(const long long *u, const long long *v, unsigned long long m, long long n,
                             uint32_t *eu, uint32_t *ev, uint32_t *deg, unsigned long long *bad) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const long long a = u[i], b = v[i];
        eu[i] = (uint32_t)a;
        ev[i] = (uint32_t)b;
        if (check_uv(a, b, n)) {
            atomicAdd(deg + a, 1u);
            atomicAdd(deg + b, 1u);
        } else {
            atomicMin(bad, i);
        }
    }
}

__global__ void k_check_w(const double *w, unsigned long long m, unsigned long long *bad) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
        if (!check_w(w[i])) atomicMin(bad, i);
}

__global__ void k_degrees(const uint32_t *eu, const uint32_t *ev, unsigned long long m, uint32_t *deg) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e0 = (unsigned long long)blockIdx.x * blockDim.x; e0 < m; e0 += stride) {
        const unsigned long long e = e0 + threadIdx.x;
        const bool in = e < m;
        add_degree_grouped(deg, in ? eu[e] : 0u, in);
        if (in) atomicAdd(deg + ev[e], 1u);
    }
}

// Degrees of the vertices [lo, hi) only: the slice's counters stay in L2
// (random atomics over a 256 MB array otherwise go to DRAM one sector each).
__global__ void k_degrees_slice(const uint32_t *eu, const uint32_t *ev, unsigned long long m, uint32_t lo,
                                uint32_t hi, uint32_t *deg) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const uint2 ab = make_uint2(__ldcs(eu + e), __ldcs(ev + e));
        if (ab.x - lo < hi - lo) atomicAdd(deg + ab.x, 1u);
        if (ab.y - lo < hi - lo) atomicAdd(deg + ab.y, 1u);
    }
}

__global__ void k_widen_deg(const uint32_t *deg, unsigned long long *out, unsigned long long n) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i <= n;
         i += stride)
        out[i] = i < n ? deg[i] : 0ULL;
}

// Slot records of the owned vertices [lo, hi): owner-local offsets, global nbr ids.
// The slot id is the edge id, or its weight key x (DISTINCT); GENERAL also
// writes the weight rank per slot.  kofe = weight key of each edge (or null).
__global__ void k_scatter(const uint32_t *eu, const uint32_t *ev, unsigned long long m,
                          const unsigned long long *vbeg, const uint32_t *newid, unsigned long long lo,
                          unsigned long long hi, uint32_t *fill, uint2 *ids, const uint32_t *kofe, bool distinct,
                          uint32_t *wk, const uint32_t *geid, uint32_t *side) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += stride) {
        uint32_t a = eu[e], b = ev[e];
        if (newid) {
            a = newid[a];
            b = newid[b];
        }
        const uint32_t key = kofe ? kofe[e] : 0u;
        const uint32_t id = distinct ? key : (geid ? geid[e] : (uint32_t)e);   // global edge id
        if (a >= lo && a < hi) {
            const unsigned long long pa = vbeg[a - lo] + atomicAdd(fill + (a - lo), 1u);
            ids[pa] = make_uint2(b, id);
            if (wk) wk[pa] = key;
        }
        if (b >= lo && b < hi) {
            const unsigned long long pb = vbeg[b - lo] + atomicAdd(fill + (b - lo), 1u);
            ids[pb] = make_uint2(a, id);
            if (wk) wk[pb] = key;
            if (side) atomicOr(side + (pb >> 5), 1u << (pb & 31));   // this owner is the edge's v end
        }
    }
}

// partition_graph's cut search (bsp.py:73-74): cut k = the first index whose
// degree-prefix offset reaches k * 2m / p (numpy compares the int64 offsets
// with the float64 targets as float64, side="left").
__global__ void k_cuts(const unsigned long long *off, unsigned long long n, int p, unsigned long long *cuts) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double two_m = (double)off[n];
    cuts[0] = 0;
    for (int k = 1; k < p; ++k) {
        const double target = ((double)k * two_m) / (double)p;
        unsigned long long lo = 0, hi = n + 1;   // lower_bound over off[0..n]
        while (lo < hi) {
            const unsigned long long mid = (lo + hi) / 2;
            if ((double)off[mid] < target) lo = mid + 1;
            else hi = mid;
        }
        cuts[k] = lo;
    }
    cuts[p] = n;
}

// Owned degrees (device ids [lo, lo + nl)) -> to be scanned into local offsets.
__global__ void k_slice_local(const uint32_t *deg, unsigned long long lo, unsigned long long nl,
                              unsigned long long *vl) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i <= nl; i += stride)
        vl[i] = i < nl ? deg[lo + i] : 0ULL;
}

// relabelling helpers: sort key = (partition of v) << 32 | ~degree, stable ->
// inside each partition's range: descending degree, ascending id
__global__ void k_relabel_keys(const uint32_t *deg, unsigned long long n, const unsigned long long *bounds, int p,
                               unsigned long long *key, uint32_t *val) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long part = 0;
        while ((int)part + 1 < p && i >= bounds[part + 1]) ++part;
        key[i] = (part << 32) | (unsigned long long)(~deg[i]);
        val[i] = (uint32_t)i;
    }
}

__global__ void k_relabel_apply(const uint32_t *oldid, const uint32_t *deg_old, unsigned long long n,
                                uint32_t *newid, uint32_t *deg_new) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t o = oldid[i];
        newid[o] = (uint32_t)i;
        deg_new[i] = deg_old[o];
    }
}

__global__ void k_minmax_bits(const double *w, unsigned long long m, unsigned long long *mm) {
    unsigned long long lo = ~0ULL, hi = 0;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += stride) {
        const unsigned long long b = canon_bits(w[e]);
        lo = b < lo ? b : lo;
        hi = b > hi ? b : hi;
    }
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, off);
        const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, off);
        lo = l2 < lo ? l2 : lo;
        hi = h2 > hi ? h2 : hi;
    }
    if ((threadIdx.x & 31) == 0) {
        atomicMin(mm, lo);
        atomicMax(mm + 1, hi);
    }
}

__global__ void k_keys(const double *w, unsigned long long m, unsigned long long *keys, uint32_t *vals) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m;
         e += stride) {
        keys[e] = canon_bits(w[e]);
        vals[e] = (uint32_t)e;
    }
}

// static order: the round-0 salt of every edge (tiebreak.py:54-58), then the
// canonical weight bits in salt order (for the stable weight pass)
__global__ void k_salt_keys(unsigned long long m, uint64_t rs, unsigned long long *keys, uint32_t *vals) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        keys[e] = mix64((uint64_t)e ^ rs);
        vals[e] = (uint32_t)e;
    }
}

__global__ void k_weight_keys_of(const double *w, const uint32_t *eid, unsigned long long m,
                                 unsigned long long *keys) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
        keys[i] = canon_bits(w[eid[i]]);
}

// Weight order through 32-bit keys (the 64-bit sort's 8 passes -> 4): key32 =
// floor((w - wmin) * scale), a monotone map of the value, so different
// key32 mean different weights and the sort by key32 leaves only the runs of
// equal key32 to order by the exact (canonical bits, edge id) -- most of
// them singletons for spread-out weights.  A run longer than kRunCap sets
// `fallback` (the exact 64-bit sort then runs instead).
constexpr uint32_t kRunCap = 64;

__global__ void k_keys32(const double *w, unsigned long long m, double wmin, double scale, uint32_t *keys,
                         uint32_t *vals) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const double t = floor((w[e] - wmin) * scale);
        keys[e] = t >= 4294967295.0 ? 0xFFFFFFFFu : (t > 0.0 ? (uint32_t)t : 0u);
        vals[e] = (uint32_t)e;
    }
}

// Per run of equal key32 (its first position's thread): exact order by
// (canonical weight bits, edge id), dense-rank heads (i > 0 and the weight
// differs from position i - 1) and tie flags, as k_heads / k_tied give them
// on the exactly sorted keys.
__global__ void k_key32_runs(const uint32_t *sk, uint32_t *se, const double *w, unsigned long long m,
                             uint32_t *head, uint32_t *tied, unsigned int *fallback) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const uint32_t k = sk[i];
        if (i > 0 && sk[i - 1] == k) continue;   // not a run start
        uint32_t L = 1;
        while (i + L < m && sk[i + L] == k && L <= kRunCap) ++L;
        if (L == 1) {
            head[i] = i > 0 ? 1u : 0u;
            tied[i] = 0u;
            continue;
        }
        if (L > kRunCap) {
            atomicOr(fallback, 1u);
            continue;
        }
        if (L <= 4) {   // the common short runs, in registers (odd-even transposition sort)
            uint32_t e4[4];
            unsigned long long f4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                e4[j] = (uint32_t)j < L ? se[i + j] : 0xFFFFFFFFu;
                f4[j] = (uint32_t)j < L ? canon_bits(w[e4[j]]) : ~0ULL;
            }
#pragma unroll
            for (int pass = 0; pass < 4; ++pass) {
#pragma unroll
                for (int j = pass & 1; j + 1 < 4; j += 2) {
                    const bool sw = f4[j] > f4[j + 1] || (f4[j] == f4[j + 1] && e4[j] > e4[j + 1]);
                    if (sw) {
                        const unsigned long long tf = f4[j];
                        f4[j] = f4[j + 1];
                        f4[j + 1] = tf;
                        const uint32_t te = e4[j];
                        e4[j] = e4[j + 1];
                        e4[j + 1] = te;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((uint32_t)j >= L) break;
                se[i + j] = e4[j];
                head[i + j] = (i + j > 0 && (j == 0 || f4[j] != f4[j - 1])) ? 1u : 0u;
                tied[i + j] = ((j > 0 && f4[j] == f4[j - 1]) || ((uint32_t)j + 1 < L && f4[j] == f4[j + 1])) ? 1u : 0u;
            }
            continue;
        }
        uint32_t e[kRunCap];
        unsigned long long f[kRunCap];
        for (uint32_t j = 0; j < L; ++j) {
            e[j] = se[i + j];
            f[j] = canon_bits(w[e[j]]);
        }
        for (uint32_t j = 1; j < L; ++j) {   // insertion sort by (weight bits, edge id)
            const uint32_t ej = e[j];
            const unsigned long long fj = f[j];
            uint32_t q = j;
            while (q > 0 && (f[q - 1] > fj || (f[q - 1] == fj && e[q - 1] > ej))) {
                f[q] = f[q - 1];
                e[q] = e[q - 1];
                --q;
            }
            f[q] = fj;
            e[q] = ej;
        }
        for (uint32_t j = 0; j < L; ++j) {
            se[i + j] = e[j];
            head[i + j] = (i + j > 0 && (j == 0 || f[j] != f[j - 1])) ? 1u : 0u;
            tied[i + j] = ((j > 0 && f[j] == f[j - 1]) || (j + 1 < L && f[j] == f[j + 1])) ? 1u : 0u;
        }
    }
}

__global__ void k_heads(const unsigned long long *sorted, unsigned long long m, uint32_t *flag) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += stride)
        flag[i] = (i > 0 && sorted[i] != sorted[i - 1]) ? 1u : 0u;
}

// tied[i]: the sorted weight at i occurs more than once
__global__ void k_tied(const unsigned long long *sorted, unsigned long long m, uint32_t *tied) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += stride)
        tied[i] = ((i > 0 && sorted[i] == sorted[i - 1]) || (i + 1 < m && sorted[i] == sorted[i + 1])) ? 1u : 0u;
}

// GENERAL: rank per edge.  DISTINCT: weight key x per edge plus the maps back.
__global__ void k_keys_out(const uint32_t *rank, const uint32_t *tie_idx, const uint32_t *tied,
                           const uint32_t *eid, unsigned long long m, int distinct, uint32_t D,
                           uint32_t *key_of_eid, uint32_t *eid_of_x, uint32_t *tie_rank, const uint32_t *geid) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += stride) {
        const uint32_t e = eid[i];
        if (!distinct) {
            key_of_eid[e] = rank[i];
            continue;
        }
        uint32_t x;
        if (tied[i]) {
            x = D + tie_idx[i];
            tie_rank[tie_idx[i]] = rank[i];
        } else {
            x = rank[i];
        }
        key_of_eid[e] = x;
        eid_of_x[x] = geid ? geid[e] : e;   // the global edge id (salts, outputs)
    }
}

__global__ void k_slot_key(uint2 *ids, unsigned long long slots, const uint32_t *key_of_eid, uint32_t *wk) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < slots;
         i += stride) {
        if (wk) wk[i] = key_of_eid[ids[i].y];
        else ids[i].y = key_of_eid[ids[i].y];
    }
}

struct InBucket {
    const uint32_t *deg;
    int q;
    __device__ bool operator()(uint32_t v) const { return deg[v] > 0 && bucket_of(deg[v]) == q; }
};

struct HasEdge {
    const uint32_t *deg;
    __device__ bool operator()(uint32_t v) const { return deg[v] > 0; }
};

}  // namespace lmx

static int grid_for(lmx_ctx *ctx, unsigned long long work);

static int grid_for(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

// All degrees from device edge arrays (ids already validated): in vertex
// slices of LMX_DEG_SLICE_MB of counters, one pass over the edges each.
static int count_degrees(lmx_ctx *ctx, const uint32_t *eu, const uint32_t *ev, unsigned long long m,
                         unsigned long long n, uint32_t *deg) {
    static const long slice_mb = getenv("LMX_DEG_SLICE_MB") ? atol(getenv("LMX_DEG_SLICE_MB")) : 48;
    if (m == 0) return LMX_OK;
    if (slice_mb <= 0) {
        k_degrees<<<grid_for(ctx, m), kBlock, 0, ctx->stream>>>(eu, ev, m, deg);
        LMX_CUDA(ctx, cudaGetLastError());
        return LMX_OK;
    }
    const unsigned long long per = std::max<unsigned long long>(1, ((unsigned long long)slice_mb << 20) / 4);
    for (unsigned long long lo = 0; lo < n; lo += per) {
        const unsigned long long hi = std::min(n, lo + per);
        k_degrees_slice<<<grid_for(ctx, m), kBlock, 0, ctx->stream>>>(eu, ev, m, (uint32_t)lo, (uint32_t)hi, deg);
        LMX_CUDA(ctx, cudaGetLastError());
    }
    return LMX_OK;
}

// Build vbeg / ids0 / wk0 / deg0 / hubs0 from ctx->eu, ev, w (K0).
// LMX_TRACE_SETUP=1: synchronise and print the wall time of each K0 stage.
void trace_mark(lmx_ctx *ctx, const char *what) {
    static const bool on = getenv("LMX_TRACE_SETUP") != nullptr;
    static std::chrono::steady_clock::time_point last = std::chrono::steady_clock::now();
    if (!on) return;
    cudaStreamSynchronize(ctx->stream);
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[lmx setup] %-24s %9.3f ms  (live %.2f GB, peak %.2f GB)\n", what,
            std::chrono::duration<double, std::milli>(now - last).count(), ctx->dev_bytes / 1e9,
            ctx->peak_bytes / 1e9);
    last = now;
}

// Static order (LMX_OPT_STATIC_ORDER, rerandomize=False): eids sorted by the
// strict total order (weight, round-0 salt) -- salts are a bijection of the
// edge id, so there are no ties -- for the scan loop's weight-ordered
// segments (ws_eid, ascending; ws_tied all zero).  Uniform weights: the salt
// alone.  Otherwise a stable weight pass over the salt order.
static int static_order_stage(lmx_ctx *ctx, bool uniform) {
    const unsigned long long m = (unsigned long long)ctx->m;
    cudaStream_t st = ctx->stream;
    const uint64_t rs = round_seed(ctx->static_seed, 0, false);
    unsigned long long *keys = nullptr, *keys2 = nullptr;
    uint32_t *vals = nullptr, *vals2 = nullptr, *tied = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&keys, m * 8, "static keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&keys2, m * 8, "static keys2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&vals, m * 4, "static vals")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&vals2, m * 4, "static vals2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&tied, m * 4, "static tied")) != LMX_OK) break;
        k_salt_keys<<<grid_for(ctx, m), kBlock, 0, st>>>(m, rs, keys, vals);
        if ((rc = lmx_sort_pairs(ctx, &keys, &keys2, &vals, &vals2, (long long)m, 0, 64, st, "static salt sort")) !=
            LMX_OK)
            break;
        if (!uniform) {   // stable: equal weights keep the salt order
            k_weight_keys_of<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, vals2, m, keys);
            if ((rc = lmx_sort_pairs(ctx, &keys, &keys2, &vals2, &vals, (long long)m, 0, 64, st,
                                     "static weight sort")) != LMX_OK)
                break;
            std::swap(vals, vals2);
        }
        e = cudaMemsetAsync(tied, 0, m * 4, st);
        if (e != cudaSuccess) break;
        ctx->ws_eid = vals2;
        ctx->ws_tied = tied;
        vals2 = tied = nullptr;
    } while (0);
    if (e != cudaSuccess && rc == LMX_OK) rc = lmx_cuda_check(ctx, e, "static order sort");
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&keys, m * 8);
    lmx_free(ctx, (void **)&keys2, m * 8);
    lmx_free(ctx, (void **)&vals, m * 4);
    lmx_free(ctx, (void **)&vals2, m * 4);
    lmx_free(ctx, (void **)&tied, m * 4);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) return rc;
    ctx->algo = 1;
    ctx->layout = kDistinct;
    ctx->n_distinct = (uint32_t)m;
    ctx->n_tied = 0;
    ctx->static_layout = true;
    ctx->static_rs = rs;
    trace_mark(ctx, "  static order sort");
    return LMX_OK;
}

// The 32-bit-key weight order (see k_keys32).  *exact = true when it does not
// apply (spread too narrow, or a run of equal 32-bit keys longer than
// kRunCap): the caller then sorts the 64-bit weight bits.
static int weight_order_key32(lmx_ctx *ctx, unsigned long long m, const unsigned long long *wbits, uint32_t *head,
                              uint32_t *eids, uint32_t *tied, bool *exact) {
    *exact = true;
    if (getenv("LMX_EXACT_WEIGHT_SORT") || m < (1ULL << 16)) return LMX_OK;
    // a graph no larger than one whose 32-bit keys left a long run (heavily
    // tied weights, e.g. the levels of a coarsening) goes to the exact sort
    // directly: the attempt would only add to its cost
    if (ctx->key32_fallback_m && m <= ctx->key32_fallback_m) return LMX_OK;
    cudaStream_t st = ctx->stream;
    unsigned long long *mm = nullptr;
    uint32_t *k1 = nullptr, *k2 = nullptr, *v1 = nullptr;
    unsigned int *fb = nullptr;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    do {
        unsigned long long got[2] = {0, 0};
        if (wbits) {   // the layout check's min / max
            got[0] = wbits[0];
            got[1] = wbits[1];
        } else {
            if ((rc = lmx_alloc(ctx, (void **)&mm, 16, "minmax")) != LMX_OK) break;
            unsigned long long init[2] = {~0ULL, 0ULL};
            if ((e = cudaMemcpyAsync(mm, init, 16, cudaMemcpyHostToDevice, st)) != cudaSuccess) break;
            k_minmax_bits<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, mm);
            if ((e = cudaMemcpyAsync(got, mm, 16, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
            if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        }
        double wmin, wmax;   // canonical bits of non-negative doubles: the value's bits
        memcpy(&wmin, &got[0], 8);
        memcpy(&wmax, &got[1], 8);
        const double spread = wmax - wmin;
        const double scale = 4294967295.0 / spread;
        if (!(spread > 1e-280) || !std::isfinite(scale)) break;   // exact sort
        if ((rc = lmx_alloc(ctx, (void **)&k1, m * 4, "key32")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&k2, m * 4, "key32 sorted")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&v1, m * 4, "key32 vals")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&fb, 4, "run fallback")) != LMX_OK) break;
        if ((e = cudaMemsetAsync(fb, 0, 4, st)) != cudaSuccess) break;
        k_keys32<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, wmin, scale, k1, v1);
        uint32_t *vo = eids;
        if ((rc = lmx_sort_pairs(ctx, &k1, &k2, &v1, &vo, (long long)m, 0, 32, st, "key32 sort")) != LMX_OK) break;
        if (vo != eids) {   // the sorted ids ended in the scratch buffer
            if ((e = cudaMemcpyAsync(eids, vo, m * 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) break;
            v1 = vo;
        }
        trace_mark(ctx, "    key32 sort");
        k_key32_runs<<<grid_for(ctx, m), kBlock, 0, st>>>(k2, eids, ctx->w, m, head, tied, fb);
        unsigned int hfb = 1;
        if ((e = cudaMemcpyAsync(&hfb, fb, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        *exact = hfb != 0;
        ctx->key32_fallback_m = *exact ? m : 0;
    } while (0);
    if (e != cudaSuccess && rc == LMX_OK) rc = lmx_cuda_check(ctx, e, "32-bit weight order");
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&mm, 16);
    lmx_free(ctx, (void **)&k1, m * 4);
    lmx_free(ctx, (void **)&k2, m * 4);
    lmx_free(ctx, (void **)&v1, m * 4);
    lmx_free(ctx, (void **)&fb, 4);
    return rc;
}

// Weight keys (tiebreak.py:105-113 order) from ctx->w alone, so a pinned-host
// load can run it while the endpoint arrays are still in flight: layout
// choice, dense ranks and tie indices, and the round-loop algorithm.  Leaves
// ctx->ws_kofe (weight key per edge; compacting loop) or ctx->ws_{rank, eid,
// tied, tidx} (sorted-position arrays; scan loop) for lmx_setup_slots.
int lmx_weight_stage(lmx_ctx *ctx) {
    const unsigned long long m = (unsigned long long)lmx_edges(ctx);
    cudaStream_t st = ctx->stream;
    uint32_t *kofe = nullptr;
    // weight key layout
    bool uniform = true, have_wbits = false;
    unsigned long long wbits[2] = {0, 0};   // min / max canonical weight bits
    if (ctx->dist_local) {
        uniform = ctx->w_uniform != 0;   // decided on ALL edges: every partition takes the same loop
    } else if (m) {
        unsigned long long *mm = nullptr;
        LMX_TRY(lmx_alloc(ctx, (void **)&mm, 16, "minmax"));
        unsigned long long init[2] = {~0ULL, 0ULL};
        LMX_CUDA(ctx, cudaMemcpyAsync(mm, init, 16, cudaMemcpyHostToDevice, st));
        k_minmax_bits<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, mm);
        LMX_CUDA(ctx, cudaGetLastError());
        LMX_CUDA(ctx, cudaMemcpyAsync(wbits, mm, 16, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        lmx_free(ctx, (void **)&mm, 16);
        uniform = wbits[0] == wbits[1];
        have_wbits = true;
    }
    if (ctx->dist_p > 1 && !ctx->dist_local) {
        // a partition sorts its local edges only: lmx_setup_slots comes back
        // after the cut search and the filter
        ctx->w_uniform = uniform ? 1 : 0;
        return LMX_OK;
    }
    ctx->layout = kUniform;
    const bool want_static = ctx->static_order && !ctx->dist_local && ctx->dist_p <= 1 && m &&
                             ctx->force_algo != 0 && ctx->n < (1LL << 30) && ctx->force_layout == -1;
    if (want_static && uniform) return static_order_stage(ctx, true);
    if (ctx->dist_local && m == 0 && !uniform && ctx->force_algo != 0 && ctx->n < (1LL << 30)) {
        ctx->algo = 1;   // a partition without local edges still runs the loop its peers run
        ctx->layout = kDistinct;
        return LMX_OK;
    }
    if (m && (!uniform || (ctx->force_layout != -1 && ctx->force_layout != kUniform))) {
        unsigned long long *keys = nullptr, *keys2 = nullptr;
        uint32_t *vals = nullptr, *vals2 = nullptr, *tied = nullptr, *tidx = nullptr;
        void *tmp = nullptr;
        size_t tmp_bytes = 0;
        int rc = LMX_OK;
        bool static_pending = false;
        do {
            if ((rc = lmx_alloc(ctx, (void **)&vals, m * 4, "sort vals")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&vals2, m * 4, "sort vals2")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&tied, m * 4, "tied")) != LMX_OK) break;
            // vals <- dense-rank heads, vals2 <- edge ids by weight, tied <- tie flags
            bool exact = true;
            if ((rc = weight_order_key32(ctx, m, have_wbits ? wbits : nullptr, vals, vals2, tied, &exact)) != LMX_OK)
                break;
            if (exact) {   // spread too narrow for 32-bit keys: the 64-bit sort of the weight bits
                if ((rc = lmx_alloc(ctx, (void **)&keys, m * 8, "sort keys")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&keys2, m * 8, "sort keys2")) != LMX_OK) break;
                k_keys<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, keys, vals);
                if ((rc = lmx_sort_pairs(ctx, &keys, &keys2, &vals, &vals2, (long long)m, 0, 64, st, "key sort")) !=
                    LMX_OK)
                    break;
                lmx_free(ctx, (void **)&keys, m * 8);   // the sort's scratch half
                k_heads<<<grid_for(ctx, m), kBlock, 0, st>>>(keys2, m, vals);
                k_tied<<<grid_for(ctx, m), kBlock, 0, st>>>(keys2, m, tied);
                lmx_free(ctx, (void **)&keys2, m * 8);
            }
            trace_mark(ctx, "  weight sort");
            if ((rc = lmx_alloc(ctx, (void **)&tidx, m * 4, "tie idx")) != LMX_OK) break;
            size_t t2 = 0;
            cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, t2, vals, vals, (long long)m, st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "scan sizing"); break; }
            tmp_bytes = t2;
            if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "scan tmp")) != LMX_OK) break;
            // dense rank of the weight value (the heads in vals)
            e = cub::DeviceScan::InclusiveSum(tmp, t2, vals, vals, (long long)m, st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "rank scan"); break; }
            // tie indices
            e = cub::DeviceScan::ExclusiveSum(tmp, t2, tied, tidx, (long long)m, st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "tie scan"); break; }
            uint32_t last_rank = 0, last_tidx = 0, last_tied = 0;
            e = cudaMemcpyAsync(&last_rank, vals + m - 1, 4, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&last_tidx, tidx + m - 1, 4, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&last_tied, tied + m - 1, 4, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "rank readback"); break; }
            const unsigned long long D = (unsigned long long)last_rank + 1;
            const unsigned long long T = (unsigned long long)last_tidx + last_tied;
            // partitions: the choice must agree across them, and T is local -> distinct
            bool distinct = (T <= m / 16 || ctx->dist_p > 1) && (D + T < 0xFFFFFFFFULL);
            if (ctx->force_layout == kDistinct) distinct = D + T < 0xFFFFFFFFULL;
            if (ctx->force_layout == kGeneral) distinct = false;
            if (want_static && !distinct) {   // tie-heavy: the static order instead (after the frees)
                static_pending = true;
                break;
            }
            ctx->layout = distinct ? kDistinct : kGeneral;
            ctx->n_distinct = (uint32_t)D;
            ctx->n_tied = (uint32_t)T;
            // round-loop algorithm: the weight-ordered scan loop needs (almost)
            // distinct weights -- a tied run is rescanned every round -- and
            // n < 2^30 (slot flag bits); it keeps the descending order itself
            // (eid by sorted position + global tie flags) for lmx_scan_build_slots
            if (distinct && ctx->force_algo != 0 && !ctx->scan_rejected && ctx->n < (1LL << 30)) {
                ctx->algo = 1;
                ctx->ws_eid = vals2;
                ctx->ws_tied = tied;
                vals2 = tied = nullptr;
                break;
            }
            if ((rc = lmx_alloc(ctx, (void **)&kofe, m * 4, "key of edge")) != LMX_OK) break;
            uint32_t *key_of_eid = kofe;
            if (distinct) {
                if ((rc = lmx_alloc(ctx, (void **)&ctx->eid_of_x, (D + T) * 4, "eid_of_x")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&ctx->tie_rank, std::max<unsigned long long>(T, 1) * 4,
                                    "tie_rank")) != LMX_OK)
                    break;
            }
            k_keys_out<<<grid_for(ctx, m), kBlock, 0, st>>>(vals, tidx, tied, vals2, m, distinct ? 1 : 0,
                                                           (uint32_t)D, key_of_eid, ctx->eid_of_x, ctx->tie_rank,
                                                           ctx->geid);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "weight keys"); break; }
        } while (0);
        cudaStreamSynchronize(st);
        lmx_free(ctx, (void **)&keys, m * 8);
        lmx_free(ctx, (void **)&keys2, m * 8);
        lmx_free(ctx, (void **)&vals, m * 4);
        lmx_free(ctx, (void **)&vals2, m * 4);
        lmx_free(ctx, (void **)&tied, m * 4);
        lmx_free(ctx, (void **)&tidx, m * 4);
        lmx_free(ctx, &tmp, tmp_bytes);
        if (rc != LMX_OK) {
            lmx_free(ctx, (void **)&kofe, m * 4);
            return rc;
        }
        if (static_pending) return static_order_stage(ctx, false);
        if (ctx->algo == 1) lmx_free(ctx, (void **)&kofe, m * 4);
    }
    ctx->ws_kofe = kofe;
    return LMX_OK;
}

// Edge arrays already on the device (lmx_build.cu): degrees, weight stage, slots.
int lmx_setup_device_edges(lmx_ctx *ctx) {
    const unsigned long long n = (unsigned long long)ctx->n, m = (unsigned long long)ctx->m;
    cudaStream_t st = ctx->stream;
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->deg0, std::max<size_t>(n, 1) * 4, "deg0"));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->deg0, 0, std::max<size_t>(n, 1) * 4, st));
    if (m) {
        LMX_TRY(count_degrees(ctx, ctx->eu, ctx->ev, m, n, ctx->deg0));
    }
    LMX_TRY(lmx_weight_stage(ctx));
    return lmx_setup_slots(ctx);
}

void lmx_free_weight_stage(lmx_ctx *ctx) {
    const size_t m4 = (size_t)std::max<int64_t>(lmx_edges(ctx), 1) * 4;   // a partition: its local edges
    lmx_free(ctx, (void **)&ctx->ws_kofe, m4);
    lmx_free(ctx, (void **)&ctx->ws_rank, m4);
    lmx_free(ctx, (void **)&ctx->ws_eid, m4);
    lmx_free(ctx, (void **)&ctx->ws_tied, m4);
    lmx_free(ctx, (void **)&ctx->ws_tidx, m4);
}

// Partition cut points of bsp.py:60-98 (partition_graph) on the caller-id
// degree prefix: cut k = searchsorted(offsets, k * 2m / p, side="left") as
// numpy compares int64 offsets with float64 targets; the host then forces
// them strictly increasing and leaves each later worker a vertex (:78-81).
int lmx_partition_bounds(lmx_ctx *ctx, std::vector<int64_t> &bounds) {
    const int p = ctx->dist_p;
    const unsigned long long n = (unsigned long long)ctx->n;
    bounds.assign(2, 0);
    bounds[1] = (int64_t)n;
    if (p <= 1) return LMX_OK;
    if ((unsigned long long)p > n) return lmx_fail(ctx, LMX_EINVAL, "p exceeds the vertex count");
    cudaStream_t st = ctx->stream;
    unsigned long long *off = nullptr, *cuts = nullptr;
    LMX_TRY(lmx_alloc(ctx, (void **)&off, (n + 1) * 8, "partition offsets"));
    LMX_TRY(lmx_alloc(ctx, (void **)&cuts, (size_t)(p + 1) * 8, "cuts"));
    k_widen_deg<<<grid_for(ctx, n + 1), kBlock, 0, st>>>(ctx->deg0, off, n);
    size_t tmp = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, tmp, off, off, (long long)(n + 1), st);
    void *t = nullptr;
    if (e == cudaSuccess) {
        int rc = lmx_alloc(ctx, &t, tmp, "scan tmp");
        if (rc != LMX_OK) return rc;
        e = cub::DeviceScan::ExclusiveSum(t, tmp, off, off, (long long)(n + 1), st);
    }
    std::vector<unsigned long long> hc((size_t)p + 1, 0);
    if (e == cudaSuccess) {
        k_cuts<<<1, 64, 0, st>>>(off, n, p, cuts);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaMemcpyAsync(hc.data(), cuts, (size_t)(p + 1) * 8, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    lmx_free(ctx, &t, tmp);
    lmx_free(ctx, (void **)&off, (n + 1) * 8);
    lmx_free(ctx, (void **)&cuts, (size_t)(p + 1) * 8);
    LMX_CUDA(ctx, e);
    // bsp.py:78-81: cuts = max.accumulate(cuts - steps) + steps; clip to [steps, n - p + steps]
    std::vector<long long> c((size_t)p - 1);
    long long run = LLONG_MIN;
    for (int k = 1; k < p; ++k) {
        const long long step = k;
        run = std::max(run, (long long)hc[(size_t)k] - step);
        long long x = run + step;
        x = std::min(std::max(x, step), (long long)n - p + step);
        c[(size_t)k - 1] = x;
    }
    bounds.assign((size_t)p + 1, 0);
    for (int k = 1; k < p; ++k) bounds[(size_t)k] = c[(size_t)k - 1];
    bounds[(size_t)p] = (int64_t)n;
    return LMX_OK;
}

__global__ void k_local_flags(const uint32_t *eu, const uint32_t *ev, unsigned long long m, uint32_t lo, uint32_t nl,
                              uint32_t *flag) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        flag[e] = (eu[e] - lo < nl || ev[e] - lo < nl) ? 1u : 0u;
}

__global__ void k_gather_local(const uint32_t *geid, unsigned long long k, const uint32_t *eu, const uint32_t *ev,
                               const double *w, uint32_t *eu2, uint32_t *ev2, double *w2) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const uint32_t e = geid[i];
        eu2[i] = eu[e];
        ev2[i] = ev[e];
        w2[i] = w[e];
    }
}

// A partition keeps the edges incident to its range (bsp.py:86-90
// local_edges), in edge order, with their global ids: everything after this
// (weight sort, slot stream, owner sort) is sized by the local edges.
static int filter_local_edges(lmx_ctx *ctx) {
    cudaStream_t st = ctx->stream;
    const unsigned long long m = (unsigned long long)ctx->m;
    const uint32_t lo = (uint32_t)ctx->lo, nl = (uint32_t)(ctx->hi - ctx->lo);
    const size_t m1 = std::max<unsigned long long>(m, 1);
    uint32_t *flag = nullptr, *geid = nullptr, *eu2 = nullptr, *ev2 = nullptr;
    double *w2 = nullptr;
    unsigned long long *cnt = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    unsigned long long k = 0;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&flag, m1 * 4, "local flags")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&geid, m1 * 4, "local edge ids")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cnt, 8, "local count")) != LMX_OK) break;
        k_local_flags<<<grid_for(ctx, m1), kBlock, 0, st>>>(ctx->eu, ctx->ev, m, lo, nl, flag);
        cub::CountingInputIterator<uint32_t> it(0u);
        cudaError_t e = cub::DeviceSelect::Flagged(nullptr, tmp_bytes, it, flag, geid, cnt, (long long)m, st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "filter sizing"); break; }
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "filter tmp")) != LMX_OK) break;
        e = cub::DeviceSelect::Flagged(tmp, tmp_bytes, it, flag, geid, cnt, (long long)m, st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&k, cnt, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "filter"); break; }
        const size_t k1 = std::max<unsigned long long>(k, 1);
        if ((rc = lmx_alloc(ctx, (void **)&eu2, k1 * 4, "local edge_u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ev2, k1 * 4, "local edge_v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&w2, k1 * 8, "local edge_weight")) != LMX_OK) break;
        if (k) k_gather_local<<<grid_for(ctx, k), kBlock, 0, st>>>(geid, k, ctx->eu, ctx->ev, ctx->w, eu2, ev2, w2);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "local gather"); break; }
    } while (0);
    lmx_free(ctx, (void **)&flag, m1 * 4);
    lmx_free(ctx, (void **)&cnt, 8);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) {
        lmx_free(ctx, (void **)&geid, m1 * 4);
        lmx_free(ctx, (void **)&eu2, m1 * 4);
        lmx_free(ctx, (void **)&ev2, m1 * 4);
        lmx_free(ctx, (void **)&w2, m1 * 8);
        return rc;
    }
    lmx_free(ctx, (void **)&ctx->eu, m1 * 4);
    lmx_free(ctx, (void **)&ctx->ev, m1 * 4);
    lmx_free(ctx, (void **)&ctx->w, m1 * 8);
    ctx->eu = eu2;
    ctx->ev = ev2;
    ctx->w = w2;
    ctx->geid = geid;
    ctx->m_local = (int64_t)k;
    ctx->dist_local = true;
    lmx_flush_cache(ctx);   // the global arrays' blocks are not reused
    return LMX_OK;
}

// vbeg / ids0 / deg0 (device ids) / bins0 / match state from ctx->eu, ev, w
// (caller ids; deg0 counted by the conversion).  DESIGN.md §3.
int lmx_setup_slots(lmx_ctx *ctx) {
    trace_mark(ctx, "edges on device");
    const unsigned long long n = (unsigned long long)ctx->n, m = (unsigned long long)ctx->m;
    cudaStream_t st = ctx->stream;
    // 1D vertex partition (bsp.py:60-98), caller ids; single GPU: [0, n)
    LMX_TRY(lmx_partition_bounds(ctx, ctx->bounds));
    ctx->lo = (unsigned long long)ctx->bounds[(size_t)ctx->dist_rank];
    ctx->hi = (unsigned long long)ctx->bounds[(size_t)ctx->dist_rank + 1];
    const unsigned long long lo = ctx->lo, nl = ctx->hi - ctx->lo;
    ctx->n_local = (int64_t)nl;
    if (ctx->dist_p > 1 && !ctx->dist_local) {   // keep the local edges, then their weight stage
        LMX_TRY(filter_local_edges(ctx));
        LMX_TRY(lmx_weight_stage(ctx));
        trace_mark(ctx, "local edges + weight stage");
    }
    const unsigned long long me = (unsigned long long)lmx_edges(ctx);   // edges held
    // Degree-descending relabelling of skewed graphs, inside
    // each partition's range (the ranges stay the reference's): hubs get the
    // low ids of their range, so the matched bitmap and candidate lookups
    // that follow the skew hit a small, cache-resident id range.
    uint32_t *newid = nullptr;
    ctx->relabeled = false;
    if (n > 1 && m) {
        bool relabel = ctx->force_relabel == 1;
        // "once": one matching per load -- the scan loop's relabelling costs
        // its load more than it saves one matching (RMAT-26: +23 / -3.7 ms)
        if (ctx->force_relabel == -1 || (ctx->force_relabel == 2 && ctx->algo != 1)) {
            uint32_t *mx = nullptr;
            size_t tmp = 0;
            LMX_TRY(lmx_alloc(ctx, (void **)&mx, 4, "max degree"));
            LMX_CUDA(ctx, cub::DeviceReduce::Max(nullptr, tmp, ctx->deg0, mx, (long long)n, st));
            void *t = nullptr;
            LMX_TRY(lmx_alloc(ctx, &t, tmp, "reduce tmp"));
            uint32_t maxdeg = 0;
            cudaError_t e = cub::DeviceReduce::Max(t, tmp, ctx->deg0, mx, (long long)n, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(&maxdeg, mx, 4, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            lmx_free(ctx, &t, tmp);
            lmx_free(ctx, (void **)&mx, 4);
            LMX_CUDA(ctx, e);
            const double avg = 2.0 * (double)m / (double)n;
            relabel = (double)maxdeg > 64.0 * std::max(avg, 1.0);
        }
        if (relabel) {
            unsigned long long *key = nullptr, *key2 = nullptr;
            uint32_t *val = nullptr, *dnew = nullptr, *bdev = nullptr;
            void *t = nullptr;
            size_t tmp = 0;
            const int p = ctx->dist_p;
            int rc = LMX_OK;
            do {
                if ((rc = lmx_alloc(ctx, (void **)&ctx->oldid, n * 4, "oldid")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&newid, n * 4, "newid")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&key, n * 8, "relabel key")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&key2, n * 8, "relabel key2")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&val, n * 4, "relabel val")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&dnew, n * 4, "deg new")) != LMX_OK) break;
                if ((rc = lmx_alloc(ctx, (void **)&bdev, (size_t)(p + 1) * 8, "bounds")) != LMX_OK) break;
                std::vector<unsigned long long> hb(ctx->bounds.begin(), ctx->bounds.end());
                cudaError_t e = cudaMemcpyAsync(bdev, hb.data(), (size_t)(p + 1) * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) {
                    k_relabel_keys<<<grid_for(ctx, n), kBlock, 0, st>>>(ctx->deg0, n,
                                                                       reinterpret_cast<unsigned long long *>(bdev),
                                                                       p, key, val);
                    e = cudaGetLastError();
                }
                int bits = 32;
                while (p > 1 && (1 << (bits - 32)) < p) ++bits;
                if (e == cudaSuccess)
                    e = cub::DeviceRadixSort::SortPairs(nullptr, tmp, key, key2, val, ctx->oldid, (long long)n, 0,
                                                        bits, st);
                if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "relabel sort size"); break; }
                if ((rc = lmx_alloc(ctx, &t, tmp, "relabel tmp")) != LMX_OK) break;
                e = cub::DeviceRadixSort::SortPairs(t, tmp, key, key2, val, ctx->oldid, (long long)n, 0, bits, st);
                if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "relabel sort"); break; }
                k_relabel_apply<<<grid_for(ctx, n), kBlock, 0, st>>>(ctx->oldid, ctx->deg0, n, newid, dnew);
                e = cudaMemcpyAsync(ctx->deg0, dnew, n * 4, cudaMemcpyDeviceToDevice, st);
                if (e == cudaSuccess) e = cudaStreamSynchronize(st);
                if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "relabel"); break; }
            } while (0);
            cudaStreamSynchronize(st);
            lmx_free(ctx, (void **)&key, n * 8);
            lmx_free(ctx, (void **)&key2, n * 8);
            lmx_free(ctx, (void **)&val, n * 4);
            lmx_free(ctx, (void **)&dnew, n * 4);
            lmx_free(ctx, (void **)&bdev, (size_t)(ctx->dist_p + 1) * 8);
            lmx_free(ctx, &t, tmp);
            if (rc != LMX_OK) {
                lmx_free(ctx, (void **)&newid, n * 4);
                return rc;
            }
            ctx->relabeled = true;
        }
    }
    trace_mark(ctx, "partition + relabel");
    if (ctx->algo == 1) {
        int rc = lmx_scan_build_slots(ctx, newid);
        if (rc != LMX_OK) {
            lmx_free(ctx, (void **)&newid, n * 4);
            return rc;
        }
        trace_mark(ctx, "ordered slots");
    }
    unsigned long long slots = (unsigned long long)ctx->slots_local;
    if (ctx->algo == 0) {
        // compacting loop: segments of the owned range, local offsets
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->vbeg, (nl + 1) * 8, "vbeg"));
        k_slice_local<<<grid_for(ctx, nl + 1), kBlock, 0, st>>>(ctx->deg0, lo, nl, ctx->vbeg);
        LMX_CUDA(ctx, cudaGetLastError());
        size_t tmp = 0;
        LMX_CUDA(ctx, cub::DeviceScan::ExclusiveSum(nullptr, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st));
        void *t = nullptr;
        LMX_TRY(lmx_alloc(ctx, &t, tmp, "scan tmp"));
        cudaError_t e = cub::DeviceScan::ExclusiveSum(t, tmp, ctx->vbeg, ctx->vbeg, (long long)(nl + 1), st);
        cudaStreamSynchronize(st);
        lmx_free(ctx, &t, tmp);
        LMX_CUDA(ctx, e);
        LMX_CUDA(ctx, cudaMemcpyAsync(&slots, ctx->vbeg + nl, 8, cudaMemcpyDeviceToHost, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        ctx->slots_local = (int64_t)slots;
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ids0, std::max<size_t>(slots, 1) * 8, "ids0"));
    }
    // the compacting loop's per-vertex degrees are local; the scan loop keeps deg0 by device id
    if (ctx->algo == 0 && ctx->dist_p > 1) {
        uint32_t *dl = nullptr;
        LMX_TRY(lmx_alloc(ctx, (void **)&dl, std::max<size_t>(nl, 1) * 4, "deg0 local"));
        if (nl) LMX_CUDA(ctx, cudaMemcpyAsync(dl, ctx->deg0 + lo, nl * 4, cudaMemcpyDeviceToDevice, st));
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        lmx_free(ctx, (void **)&ctx->deg0, std::max<size_t>(n, 1) * 4);
        ctx->deg0 = dl;
    }
    LMX_TRY(lmx_alloc_match_state(ctx));
    trace_mark(ctx, "offsets + allocation");
    if (ctx->algo == 0 && ctx->dist_p > 1) {   // which end of its edge each owned slot is (RoundMessages)
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->slot_side, (std::max<size_t>(slots, 1) + 31) / 32 * 4, "slot side"));
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->slot_side, 0, (std::max<size_t>(slots, 1) + 31) / 32 * 4, st));
    }
    if (me && ctx->algo == 0) {
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ids1, std::max<size_t>(slots, 1) * 8, "ids1"));
        if (ctx->layout == kGeneral) {
            LMX_TRY(lmx_alloc(ctx, (void **)&ctx->wk0, slots * 4, "wk0"));
            LMX_TRY(lmx_alloc(ctx, (void **)&ctx->wk1, slots * 4, "wk1"));
        }
        // fill counters reuse vdeg (local)
        LMX_CUDA(ctx, cudaMemsetAsync(ctx->vdeg, 0, std::max<size_t>(nl, 1) * 4, st));
        k_scatter<<<grid_for(ctx, me), kBlock, 0, st>>>(ctx->eu, ctx->ev, me, ctx->vbeg, newid, lo, ctx->hi,
                                                       ctx->vdeg, ctx->ids0, ctx->ws_kofe,
                                                       ctx->layout == kDistinct, ctx->wk0, ctx->geid, ctx->slot_side);
        LMX_CUDA(ctx, cudaGetLastError());
        trace_mark(ctx, "slot scatter");
    }
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    lmx_free(ctx, (void **)&newid, n * 4);
    lmx_free_weight_stage(ctx);
    if (ctx->algo == 1 || ctx->dist_p > 1)   // match rounds: scan-loop RoundStats, message accounting
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mround, std::max<size_t>(n, 1) * 4, "mround"));
    if (ctx->algo == 1)
        LMX_TRY(lmx_alloc(ctx, (void **)&ctx->mpacked, (std::max<size_t>(n, 1) + 3) / 4 * 4, "mround packed"));
    // round-0 bucket lists of the owned vertices (compacting loop: local
    // indices per live-degree bucket; scan loop: device ids with an edge)
    const size_t cap = std::max<size_t>(nl, 1);
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->bins0, cap * 4 * (ctx->algo == 1 ? 1 : kBuckets), "bins0"));
    {
        unsigned long long *cnt = nullptr;
        LMX_TRY(lmx_alloc(ctx, (void **)&cnt, 8 * kBuckets, "bucket counts"));
        cub::CountingInputIterator<uint32_t> it(ctx->algo == 1 ? (uint32_t)lo : 0u);
        // deg0 is indexed by device id (scan) or locally (compacting, p > 1),
        // matching the counting iterator's base
        size_t tmp = 0;
        LMX_CUDA(ctx, cub::DeviceSelect::If(nullptr, tmp, it, ctx->bins0, cnt, (long long)nl,
                                            InBucket{ctx->deg0, 0}, st));
        void *t = nullptr;
        LMX_TRY(lmx_alloc(ctx, &t, tmp, "select tmp"));
        cudaError_t e = cudaSuccess;
        if (ctx->algo == 1) {   // scan: one list of every vertex with an edge
            LMX_CUDA(ctx, cudaMemsetAsync(cnt, 0, 8 * kBuckets, st));
            size_t tb = tmp;
            e = cub::DeviceSelect::If(t, tb, it, ctx->bins0, cnt, (long long)nl, HasEdge{ctx->deg0}, st);
        }
        for (int q = 0; q < kBuckets && e == cudaSuccess && ctx->algo == 0; ++q) {
            size_t tb = tmp;
            e = cub::DeviceSelect::If(t, tb, it, ctx->bins0 + (size_t)q * cap, cnt + q, (long long)nl,
                                      InBucket{ctx->deg0, q}, st);
        }
        unsigned long long h[kBuckets] = {};
        if (e == cudaSuccess) e = cudaMemcpyAsync(h, cnt, 8 * kBuckets, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        lmx_free(ctx, &t, tmp);
        lmx_free(ctx, (void **)&cnt, 8 * kBuckets);
        LMX_CUDA(ctx, e);
        for (int q = 0; q < kBuckets; ++q) ctx->n_bins0[q] = (unsigned int)h[q];
    }
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    trace_mark(ctx, "bucket lists");
    return LMX_OK;
}

// Host-memory loads.  The int64 endpoint arrays are narrowed to u32 (and
// range-checked) by a pool of host threads into a pinned staging ring and the
// copy engine moves the narrowed blocks: 8 instead of 16 bytes per edge cross
// the host link, which is what bounds the load from host memory.  The weights
// go first (directly when they are page-locked) so the weight-key stage runs
// on the device while the endpoint blocks are still arriving; each block's
// degree counts run on a third stream right behind its copy.
bool lmx_narrow_block(const int64_t *u, const int64_t *v, size_t k, uint64_t n, uint32_t *ou, uint32_t *ov,
                      bool streaming);

namespace {

int load_threads() {
    const char *env = getenv("LMX_LOAD_THREADS");
    int t = env ? atoi(env) : (int)std::thread::hardware_concurrency();
    return std::max(1, std::min(t, 64));
}

}  // namespace

// Fills ctx->eu/ev/w/deg0 from host arrays; *host_bad = the first edge whose
// endpoints fail check_uv (or ~0); device-side weight checks go to `bad`.
// *weights_done: the weight-key stage already ran (page-locked weights).
static int load_host_narrowed(lmx_ctx *ctx, const int64_t *edge_u, const int64_t *edge_v, const double *edge_weight,
                              unsigned long long *bad, unsigned long long *host_bad, bool *weights_done) {
    const unsigned long long m = (unsigned long long)ctx->m;
    const uint64_t n = (uint64_t)ctx->n;
    cudaStream_t st = ctx->stream;
    bool w_pinned = !getenv("LMX_NO_ZEROCOPY");
    if (w_pinned) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, edge_weight) != cudaSuccess || at.type != cudaMemoryTypeHost) {
            cudaGetLastError();
            w_pinned = false;
        }
    }
    const auto t_start = std::chrono::steady_clock::now();
    const int T = load_threads();
    const int R = getenv("LMX_LOAD_RING") ? std::max(2, atoi(getenv("LMX_LOAD_RING"))) : 4;
    const unsigned long long bmax = getenv("LMX_LOAD_BLOCK") ? std::max(1ULL << 12, strtoull(getenv("LMX_LOAD_BLOCK"), 0, 10))
                                                             : (1ULL << 19);
    unsigned long long B = std::max<unsigned long long>(1ULL << 12, (m + 4ULL * T - 1) / (4ULL * T));
    B = (std::min<unsigned long long>(B, bmax) + 7) & ~7ULL;   // 32-byte aligned slot halves
    const size_t slot_bytes = (size_t)B * (w_pinned ? 8 : 16);
    const bool streaming = getenv("LMX_LOAD_NT") ? atoi(getenv("LMX_LOAD_NT")) != 0 : true;
    const size_t ring = slot_bytes * T * R;
    if (ctx->stage_bytes < ring) {
        if (ctx->stage_host) cudaFreeHost(ctx->stage_host);
        ctx->stage_host = nullptr;
        ctx->stage_bytes = 0;
        LMX_CUDA(ctx, cudaHostAlloc(&ctx->stage_host, ring, cudaHostAllocPortable));
        ctx->stage_bytes = ring;
    }
    while (ctx->stage_ev.size() < (size_t)T * R) {
        cudaEvent_t e;
        LMX_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ctx->stage_ev.push_back(e);
    }
    if (!ctx->copy_stream) {
        LMX_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (cudaEvent_t &e : ctx->ev_copy) LMX_CUDA(ctx, cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    if (!ctx->deg_stream) {
        LMX_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->deg_stream, cudaStreamNonBlocking));
        LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_deg, cudaEventDisableTiming));
    }
    cudaStream_t cs = ctx->copy_stream, ds = ctx->deg_stream;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[0], st));   // allocations / memsets before the copies
    LMX_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_copy[0], 0));
    LMX_CUDA(ctx, cudaStreamWaitEvent(ds, ctx->ev_copy[0], 0));
    if (w_pinned) {
        LMX_CUDA(ctx, cudaMemcpyAsync(ctx->w, edge_weight, (size_t)m * 8, cudaMemcpyHostToDevice, cs));
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[1], cs));
        LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_copy[1], 0));
        k_check_w<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, bad);
        LMX_CUDA(ctx, cudaGetLastError());
    }
    const unsigned long long nblocks = (m + B - 1) / B;
    std::atomic<unsigned long long> first_bad{~0ULL}, next_block{0};
    std::mutex err_mu;
    cudaError_t werr = cudaSuccess;
    auto worker = [&](int t) {
        cudaError_t e = cudaSetDevice(ctx->device);
        char *mine = (char *)ctx->stage_host + (size_t)t * R * slot_bytes;
        for (unsigned long long it = 0; e == cudaSuccess; ++it) {
            const unsigned long long b = next_block.fetch_add(1);
            if (b >= nblocks) break;
            const int j = (int)(it % R);
            cudaEvent_t ev = ctx->stage_ev[(size_t)t * R + j];
            if (it >= (unsigned long long)R && (e = cudaEventSynchronize(ev)) != cudaSuccess) break;
            const unsigned long long off = b * B, k = std::min<unsigned long long>(B, m - off);
            uint32_t *su = (uint32_t *)(mine + (size_t)j * slot_bytes), *sv = su + B;
            const bool block_bad = lmx_narrow_block(edge_u + off, edge_v + off, k, n, su, sv, streaming);
            if (block_bad) {
                for (unsigned long long i = 0; i < k; ++i) {
                    const uint64_t a = (uint64_t)edge_u[off + i], c = (uint64_t)edge_v[off + i];
                    if (a >= n || c >= n || a == c) {
                        unsigned long long cur = first_bad.load();
                        while (off + i < cur && !first_bad.compare_exchange_weak(cur, off + i)) {
                        }
                        break;
                    }
                }
            }
            e = cudaMemcpyAsync(ctx->eu + off, su, k * 4, cudaMemcpyHostToDevice, cs);
            if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->ev + off, sv, k * 4, cudaMemcpyHostToDevice, cs);
            if (e == cudaSuccess && !w_pinned) {
                double *sw = (double *)(sv + B);
                memcpy(sw, edge_weight + off, k * 8);
                e = cudaMemcpyAsync(ctx->w + off, sw, k * 8, cudaMemcpyHostToDevice, cs);
            }
            if (e == cudaSuccess) e = cudaEventRecord(ev, cs);
            if (e == cudaSuccess) e = cudaStreamWaitEvent(ds, ev, 0);
            if (e == cudaSuccess && !block_bad) {   // (a failing load never reads the degrees)
                k_degrees<<<grid_for(ctx, k), kBlock, 0, ds>>>(ctx->eu + off, ctx->ev + off, k, ctx->deg0);
                e = cudaGetLastError();
            }
        }
        if (e != cudaSuccess) {
            std::lock_guard<std::mutex> g(err_mu);
            if (werr == cudaSuccess) werr = e;
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < T; ++t) pool.emplace_back(worker, t);
    int rc = LMX_OK;
    if (w_pinned) {   // the weight-key stage overlaps the endpoint copies
        rc = lmx_weight_stage(ctx);
        *weights_done = true;
    }
    for (std::thread &th : pool) th.join();
    const auto t_join = std::chrono::steady_clock::now();
    if (rc != LMX_OK || werr != cudaSuccess) {   // no copy may still read the ring
        cudaStreamSynchronize(cs);
        cudaStreamSynchronize(ds);
    }
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, werr);
    if (!w_pinned) {
        LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[1], cs));
        LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_copy[1], 0));
        k_check_w<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, m, bad);
        LMX_CUDA(ctx, cudaGetLastError());
    }
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev_deg, ds));
    LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_deg, 0));
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[2], cs));
    LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_copy[2], 0));
    *host_bad = first_bad.load();
    if (getenv("LMX_TRACE_SETUP")) {
        LMX_CUDA(ctx, cudaStreamSynchronize(st));
        const auto t_end = std::chrono::steady_clock::now();
        fprintf(stderr, "[lmx setup] host load: %d threads, blocks of %llu edges, weights %s; workers done %.1f ms, "
                "copies + degrees done %.1f ms\n", T, B, w_pinned ? "page-locked" : "staged",
                std::chrono::duration<double, std::milli>(t_join - t_start).count(),
                std::chrono::duration<double, std::milli>(t_end - t_start).count());
        trace_mark(ctx, "host narrow + copies");
    }
    return LMX_OK;
}

// lmx_load_graph: validate + narrow the edge arrays, then K0.
int lmx_load_edges(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                   const double *edge_weight, int where) {
    if (n < 0 || m < 0) return lmx_fail(ctx, LMX_EINVAL, "negative n or m");
    if (n >= (int64_t)0xFFFFFFFFLL) return lmx_fail(ctx, LMX_ELIMIT, "n exceeds the 32-bit vertex id range");
    if (m >= (int64_t)0xFFFFFFFFLL) return lmx_fail(ctx, LMX_ELIMIT, "m exceeds the 32-bit edge id range");
    if (m > 0 && (!edge_u || !edge_v || !edge_weight))
        return lmx_fail(ctx, LMX_EINVAL, "null edge array");
    lmx_free_graph(ctx);
    ctx->n = n;
    ctx->m = m;
    cudaStream_t st = ctx->stream;
    const size_t mm = std::max<int64_t>(m, 1);
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->eu, mm * 4, "edge_u"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->ev, mm * 4, "edge_v"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->w, mm * 8, "edge_weight"));
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->deg0, std::max<size_t>(n, 1) * 4, "deg0"));
    LMX_CUDA(ctx, cudaMemsetAsync(ctx->deg0, 0, std::max<size_t>(n, 1) * 4, st));
    unsigned long long *bad = nullptr;
    LMX_TRY(lmx_alloc(ctx, (void **)&bad, 8, "bad"));
    LMX_CUDA(ctx, cudaMemsetAsync(bad, 0xFF, 8, st));
    // Pinned (page-locked) host arrays: the copy engine brings the weights
    // first and the weight-key stage (sorts) runs on the device while the
    // endpoint arrays are still crossing the host link.
    bool pinned = false;
    if (m > 0 && where == LMX_HOST && !getenv("LMX_NO_ZEROCOPY")) {
        pinned = true;
        const void *hp[3] = {edge_u, edge_v, edge_weight};
        for (int i = 0; i < 3; ++i) {
            cudaPointerAttributes at;
            if (cudaPointerGetAttributes(&at, hp[i]) != cudaSuccess || at.type != cudaMemoryTypeHost) {
                cudaGetLastError();
                pinned = false;
                break;
            }
        }
    }
    bool weights_done = false, device_degrees = false;
    unsigned long long host_bad = ~0ULL;
    if (m > 0 && where == LMX_HOST && !getenv("LMX_LOAD_LEGACY")) {
        LMX_TRY(load_host_narrowed(ctx, edge_u, edge_v, edge_weight, bad, &host_bad, &weights_done));
    } else if (m > 0) {
        if (pinned) {
            if (!ctx->copy_stream) {
                LMX_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
                LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_copy[0], cudaEventDisableTiming));
                LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_copy[1], cudaEventDisableTiming));
                LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_copy[2], cudaEventDisableTiming));
            }
            cudaStream_t cs = ctx->copy_stream;
            long long *su = nullptr, *sv = nullptr;
            LMX_TRY(lmx_alloc(ctx, (void **)&su, mm * 8, "stage u"));
            LMX_TRY(lmx_alloc(ctx, (void **)&sv, mm * 8, "stage v"));
            LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[0], st));   // blocks reused from the cache are idle
            LMX_CUDA(ctx, cudaStreamWaitEvent(cs, ctx->ev_copy[0], 0));
            LMX_CUDA(ctx, cudaMemcpyAsync(ctx->w, edge_weight, (size_t)m * 8, cudaMemcpyHostToDevice, cs));
            LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[1], cs));
            LMX_CUDA(ctx, cudaMemcpyAsync(su, edge_u, (size_t)m * 8, cudaMemcpyHostToDevice, cs));
            LMX_CUDA(ctx, cudaMemcpyAsync(sv, edge_v, (size_t)m * 8, cudaMemcpyHostToDevice, cs));
            LMX_CUDA(ctx, cudaEventRecord(ctx->ev_copy[2], cs));
            LMX_CUDA(ctx, cudaStreamWaitEvent(st, ctx->ev_copy[1], 0));
            k_check_w<<<grid_for(ctx, m), kBlock, 0, st>>>(ctx->w, (unsigned long long)m, bad);
            LMX_CUDA(ctx, cudaGetLastError());
            int rc = lmx_weight_stage(ctx);   // overlaps the endpoint copies
            cudaError_t e = cudaStreamWaitEvent(st, ctx->ev_copy[2], 0);
            if (e == cudaSuccess) {
                k_convert_uv<<<grid_for(ctx, m), kBlock, 0, st>>>(su, sv, (unsigned long long)m, n, ctx->eu,
                                                                 ctx->ev, ctx->deg0, bad);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            lmx_free(ctx, (void **)&su, mm * 8);
            lmx_free(ctx, (void **)&sv, mm * 8);
            if (rc != LMX_OK) return rc;
            LMX_CUDA(ctx, e);
            weights_done = true;
        } else if (where == LMX_DEVICE) {
            k_convert<<<grid_for(ctx, m), kBlock, 0, st>>>((const long long *)edge_u, (const long long *)edge_v,
                                                          edge_weight, (unsigned long long)m, n, 0, ctx->eu,
                                                          ctx->ev, ctx->w, nullptr, bad);
            LMX_CUDA(ctx, cudaGetLastError());
            device_degrees = true;   // counted once the ids are known valid
        } else {
            // chunked H2D through two staging buffers of int64 ids
            const unsigned long long chunk = 1ULL << 24;
            long long *su = nullptr, *sv = nullptr;
            double *sw = nullptr;
            const size_t cb = std::min<unsigned long long>(chunk, (unsigned long long)m);
            LMX_TRY(lmx_alloc(ctx, (void **)&su, cb * 8, "stage u"));
            LMX_TRY(lmx_alloc(ctx, (void **)&sv, cb * 8, "stage v"));
            LMX_TRY(lmx_alloc(ctx, (void **)&sw, cb * 8, "stage w"));
            cudaError_t e = cudaSuccess;
            for (unsigned long long off = 0; off < (unsigned long long)m && e == cudaSuccess; off += chunk) {
                const unsigned long long k = std::min<unsigned long long>(chunk, (unsigned long long)m - off);
                e = cudaMemcpyAsync(su, edge_u + off, k * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaMemcpyAsync(sv, edge_v + off, k * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaMemcpyAsync(sw, edge_weight + off, k * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) {
                    k_convert<<<grid_for(ctx, k), kBlock, 0, st>>>(su, sv, sw, k, n, off, ctx->eu, ctx->ev,
                                                                  ctx->w, ctx->deg0, bad);
                    e = cudaGetLastError();
                }
            }
            cudaStreamSynchronize(st);
            lmx_free(ctx, (void **)&su, cb * 8);
            lmx_free(ctx, (void **)&sv, cb * 8);
            lmx_free(ctx, (void **)&sw, cb * 8);
            LMX_CUDA(ctx, e);
        }
    }
    trace_mark(ctx, "convert + degrees");
    unsigned long long badpos = 0;
    LMX_CUDA(ctx, cudaMemcpyAsync(&badpos, bad, 8, cudaMemcpyDeviceToHost, st));
    LMX_CUDA(ctx, cudaStreamSynchronize(st));
    lmx_free(ctx, (void **)&bad, 8);
    badpos = std::min(badpos, host_bad);
    if (badpos != ~0ULL) {
        int64_t u = 0, v = 0;
        double w = 0;
        if (where == LMX_HOST) {
            u = edge_u[badpos];
            v = edge_v[badpos];
            w = edge_weight[badpos];
        } else {
            cudaMemcpy(&u, edge_u + badpos, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&v, edge_v + badpos, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&w, edge_weight + badpos, 8, cudaMemcpyDeviceToHost);
        }
        lmx_free_graph(ctx);
        char buf[256];
        if (u < 0 || v < 0 || u >= n || v >= n)
            snprintf(buf, sizeof buf, "edge %llu: vertex id out of range for n=%lld: (%lld, %lld)",
                     (unsigned long long)badpos, (long long)n, (long long)u, (long long)v);
        else if (u == v)
            snprintf(buf, sizeof buf, "edge %llu: self-loop (%lld, %lld) in a built graph",
                     (unsigned long long)badpos, (long long)u, (long long)v);
        else
            snprintf(buf, sizeof buf, "edge %llu: weight must be finite and >= 0, got %.17g",
                     (unsigned long long)badpos, w);
        return lmx_fail(ctx, LMX_EINVAL, buf);
    }
    if (device_degrees) {
        LMX_TRY(count_degrees(ctx, ctx->eu, ctx->ev, (unsigned long long)m, (unsigned long long)n, ctx->deg0));
        trace_mark(ctx, "degrees (sliced)");
    }
    if (!weights_done) LMX_TRY(lmx_weight_stage(ctx));
    trace_mark(ctx, "weight stage");
    return lmx_setup_slots(ctx);
}
