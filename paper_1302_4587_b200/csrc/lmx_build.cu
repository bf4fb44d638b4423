// lmx_build.cu -- device graph builders.
//
// lmx_build_graph: the build_graph numbering contract (graph.py:59-119) for
// raw triple lists too large for the reference's Python dict loop:
//   * reject negative / out-of-range ids and NaN / inf / negative weights,
//     naming the first bad input position (graph.py:80-88);
//   * drop self-loops (graph.py:89-91);
//   * collapse parallel pairs: keep the first occurrence of the maximum
//     weight (strict '>' double comparison, graph.py:99-100) with that
//     occurrence's orientation and weight bits;
//   * edge ids follow the first occurrence of each pair (graph.py:94-98);
//   * n = num_vertices, or max id over non-loop triples + 1 (graph.py:103).
// Implementation: stable LSD radix sort of (pair key, position), one thread
// per equal-key run, a prefix sum over first-occurrence flags for the ids.
//
// lmx_gen_rmat: RMAT (Chakrabarti et al.; Graph500 a,b,c,d) raw triples from a
// counter-based hash, so the CPU oracle (oracle/oracle.py:rmat_raw) generates
// the identical list:
//   s_q  = mix64(seed ^ 0x524D4154...)            (stream keys, q = 0, 1, 2)
//   level bits: h = mix64(s_0 ^ (i * 16 + l / 4)), x = (h >> 16 * (l % 4)) & 0xFFFF
//     quadrant (0,0) if x < A, (0,1) if x < A+B, (1,0) if x < A+B+C, else (1,1)
//     with A = round(a * 65536) etc.; bit (scale-1-l) of u / v
//   weight: (mix64(s_1 ^ i) >> 11) * 2^-53  in [0, 1)
//   permute: x -> bijection on scale bits (odd multiplies mod 2^scale, xor
//     shifts, xor with s_2), applied to both endpoints.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "lmx_internal.cuh"
#include "lmx_sort.cuh"

using namespace lmx;

namespace lmx {

constexpr uint64_t kRmatTag0 = 0x524D41545F4C5654ULL;   // "RMAT_LVT"
constexpr uint64_t kRmatTag1 = 0x524D41545F574754ULL;   // "RMAT_WGT"
constexpr uint64_t kRmatTag2 = 0x524D41545F504552ULL;   // "RMAT_PER"

struct RmatParams {
    int scale;
    uint32_t A, AB, ABC;   // cumulative 16-bit thresholds
    uint64_t s0, s1, s2;
    int permute;
};

__host__ __device__ __forceinline__ uint32_t rmat_perm(uint32_t x, const RmatParams &p) {
    const uint64_t mask = (p.scale >= 64) ? ~0ULL : ((1ULL << p.scale) - 1);
    const int h = p.scale / 2 + 1;
    uint64_t y = x;
    y = (y * 0x9E3779B97F4A7C15ULL) & mask;
    y ^= y >> h;
    y = (y * 0xBF58476D1CE4E5B9ULL) & mask;
    y ^= y >> (p.scale - h > 0 ? p.scale - h : 1);
    y ^= p.s2 & mask;
    return (uint32_t)y;
}

// Raw triple i of the stream (see the file header).
__device__ __forceinline__ void rmat_one(const RmatParams &p, unsigned long long i, uint32_t &u, uint32_t &v,
                                         double &w) {
    uint32_t a = 0, b = 0;
    uint64_t h = 0;
    for (int l = 0; l < p.scale; ++l) {
        if ((l & 3) == 0) h = mix64(p.s0 ^ (i * 16ULL + (unsigned long long)(l >> 2)));
        const uint32_t x = (uint32_t)((h >> (16 * (l & 3))) & 0xFFFFu);
        const uint32_t bit = 1u << (p.scale - 1 - l);
        if (x < p.A) {
        } else if (x < p.AB) {
            b |= bit;
        } else if (x < p.ABC) {
            a |= bit;
        } else {
            a |= bit;
            b |= bit;
        }
    }
    if (p.permute) {
        a = rmat_perm(a, p);
        b = rmat_perm(b, p);
    }
    u = a;
    v = b;
    w = (double)(mix64(p.s1 ^ i) >> 11) * (1.0 / 9007199254740992.0);
}

__global__ void k_rmat_raw(RmatParams p, unsigned long long k, uint32_t *u, uint32_t *v, double *w) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride)
        rmat_one(p, i, u[i], v[i], w[i]);
}

// ---- distributed build (a partition generates the whole raw stream and keeps
// the triples whose LOWER endpoint falls in its build range) -------------------
// Pass 0 counts, pass 1 appends {u, v, w, raw position} (block-aggregated).
template <bool WRITE>
__global__ void __launch_bounds__(kBlock) k_rmat_keep(RmatParams p, unsigned long long k, uint32_t nparts,
                                                      uint32_t part, unsigned long long *cursor, uint32_t *ku,
                                                      uint32_t *kv, double *kw, uint32_t *kpos) {
    __shared__ uint32_t s_cnt[kWarps];
    __shared__ unsigned long long s_base;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t lt;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(lt));
    for (unsigned long long i0 = (unsigned long long)blockIdx.x * kBlock; i0 < k;
         i0 += (unsigned long long)gridDim.x * kBlock) {
        const unsigned long long i = i0 + tid;
        uint32_t a = 0, b = 0;
        double w = 0;
        bool keep = false;
        if (i < k) {
            rmat_one(p, i, a, b, w);
            const uint32_t lo = a < b ? a : b;
            const uint32_t hi = a < b ? b : a;
            // the pair's build rank: a hash of the unordered pair, so every
            // occurrence of a pair meets on one rank and the ranks get even
            // shares whatever the id distribution (self-loops dropped, graph.py:89-91)
            keep = a != b && (uint32_t)(mix64(((uint64_t)lo << 32) | hi) % nparts) == part;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) s_cnt[warp] = __popc(bal);
        __syncthreads();
        if (tid == 0) {
            uint32_t t = 0;
            for (int q = 0; q < kWarps; ++q) t += s_cnt[q];
            s_base = t ? atomicAdd(cursor, (unsigned long long)t) : 0ULL;
        }
        __syncthreads();
        if (WRITE && keep) {
            unsigned long long pos = s_base;
            for (int q = 0; q < warp; ++q) pos += s_cnt[q];
            pos += __popc(bal & lt);
            ku[pos] = a;
            kv[pos] = b;
            kw[pos] = w;
            kpos[pos] = (uint32_t)i;
        }
        __syncthreads();
    }
}

__global__ void k_pair_keys_local(const uint32_t *u, const uint32_t *v, unsigned long long k, int bits,
                                  unsigned long long *key, uint32_t *idx) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const unsigned long long a = u[i], b = v[i];
        key[i] = ((a < b ? a : b) << bits) | (a < b ? b : a);
        idx[i] = (uint32_t)i;
    }
}

// One thread per run of equal pairs: the first occurrence (smallest raw
// position) numbers the pair; the kept occurrence is the heaviest, the
// earliest of equal weights (graph.py:94-100) -- kept order is arbitrary here,
// so positions decide explicitly.  Sets the first-occurrence bit (global raw
// position) and counts the pair into both endpoints' degrees.
__global__ void k_runs_dist(const unsigned long long *key, const uint32_t *idx, unsigned long long k,
                            const uint32_t *u, const uint32_t *v, const double *w, const uint32_t *pos,
                            uint32_t *first_bits, uint32_t *deg, uint32_t *pf, uint32_t *pu, uint32_t *pv,
                            double *pw, unsigned long long *npairs) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const unsigned long long kk = key[i];
        if (i > 0 && key[i - 1] == kk) continue;
        uint32_t best = idx[i], first = pos[idx[i]];
        double bw = w[best];
        uint32_t bp = first;
        for (unsigned long long j = i + 1; j < k && key[j] == kk; ++j) {
            const uint32_t c = idx[j];
            const uint32_t cp = pos[c];
            const double cw = w[c];
            first = cp < first ? cp : first;
            if (cw > bw || (cw == bw && cp < bp)) {
                bw = cw;
                best = c;
                bp = cp;
            }
        }
        atomicOr(first_bits + (first >> 5), 1u << (first & 31));
        atomicAdd(deg + u[best], 1u);
        atomicAdd(deg + v[best], 1u);
        const unsigned long long q = atomicAdd(npairs, 1ULL);
        pf[q] = first;
        pu[q] = u[best];
        pv[q] = v[best];
        pw[q] = bw;
    }
}

__global__ void k_word_popc(const uint32_t *bits, unsigned long long words, unsigned long long *cnt) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i <= words; i += stride)
        cnt[i] = i < words ? (unsigned long long)__popc(bits[i]) : 0ULL;
}

// Records {eid, u, v, w} to the owners of u and v (once if the same):
// pass 0 counts per destination, pass 1 writes into its region.
struct DistRec {
    uint32_t eid, u, v, pad;
    double w;
};

template <bool WRITE>
__global__ void k_route(const uint32_t *pf, const uint32_t *pu, const uint32_t *pv, const double *pw,
                        unsigned long long np, const uint32_t *first_bits, const unsigned long long *word_prefix,
                        const unsigned long long *bounds, int p, unsigned long long *cnt,
                        const unsigned long long *region, DistRec *out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += stride) {
        const uint32_t f = pf[i];
        const uint32_t below = first_bits[f >> 5] & ((1u << (f & 31)) - 1u);
        const uint32_t eid = (uint32_t)(word_prefix[f >> 5] + (unsigned long long)__popc(below));
        int ou = 0, ov = 0;
        while (ou + 1 < p && pu[i] >= bounds[ou + 1]) ++ou;
        while (ov + 1 < p && pv[i] >= bounds[ov + 1]) ++ov;
        for (int t = 0; t < (ou == ov ? 1 : 2); ++t) {
            const int d = t == 0 ? ou : ov;
            const unsigned long long q = atomicAdd(cnt + d, 1ULL);
            if (WRITE) {
                DistRec r;
                r.eid = eid;
                r.u = pu[i];
                r.v = pv[i];
                r.pad = 0;
                r.w = pw[i];
                out[region[d] + q] = r;
            }
        }
    }
}

__global__ void k_rec_unpack(const DistRec *rec, const uint32_t *idx, unsigned long long k, uint32_t *eu,
                             uint32_t *ev, double *w, uint32_t *geid) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const DistRec r = rec[idx ? idx[i] : i];
        eu[i] = r.u;
        ev[i] = r.v;
        w[i] = r.w;
        geid[i] = r.eid;
    }
}

// Validation of raw int64 triples (graph.py:80-88); narrows ids to u32.
__global__ void k_raw_convert(const long long *u, const long long *v, const double *w, unsigned long long k,
                              long long nlimit, unsigned long long base, uint32_t *uo, uint32_t *vo,
                              double *wo, unsigned long long *bad, unsigned long long *maxid) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long mx = 0;
    bool any = false;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride) {
        const long long a = u[i], b = v[i];
        const double x = w[i];
        bool ok = a >= 0 && b >= 0 && a < 0xFFFFFFFFLL && b < 0xFFFFFFFFLL && isfinite(x) && !(x < 0.0);
        if (nlimit >= 0) ok = ok && a < nlimit && b < nlimit;
        if (!ok) atomicMin(bad, base + i);
        uo[base + i] = (uint32_t)a;
        vo[base + i] = (uint32_t)b;
        wo[base + i] = x;
        if (ok && a != b) {
            const unsigned long long t = (unsigned long long)(a > b ? a : b);
            mx = t > mx ? t : mx;
            any = true;
        }
    }
    if (any) atomicMax(maxid, mx + 1);
}

__global__ void k_max_id(const uint32_t *u, const uint32_t *v, unsigned long long k, unsigned long long *maxid) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    unsigned long long mx = 0;
    bool any = false;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride) {
        if (u[i] != v[i]) {
            const unsigned long long t = u[i] > v[i] ? u[i] : v[i];
            mx = t > mx ? t : mx;
            any = true;
        }
    }
    if (any) atomicMax(maxid, mx + 1);
}

__global__ void k_pair_keys(const uint32_t *u, const uint32_t *v, unsigned long long k, int bits,
                            unsigned long long *key, uint32_t *idx) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    const unsigned long long all = (bits >= 32) ? 0xFFFFFFFFULL : ((1ULL << bits) - 1);
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride) {
        const unsigned long long a = u[i], b = v[i];
        const unsigned long long lo = a < b ? a : b, hi = a < b ? b : a;
        key[i] = (a == b) ? ((all << bits) | all) : ((lo << bits) | hi);   // loops -> one sentinel run
        idx[i] = (uint32_t)i;
    }
}

// One thread per run head: keep the first occurrence of the max weight.
__global__ void k_runs(const unsigned long long *key, const uint32_t *idx, unsigned long long k,
                       unsigned long long sentinel, const uint32_t *u, const uint32_t *v, const double *w,
                       uint32_t *first_flag, uint32_t *kept) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride) {
        const unsigned long long kk = key[i];
        if (kk == sentinel) continue;
        if (i > 0 && key[i - 1] == kk) continue;
        uint32_t best = idx[i];
        double bw = w[best];
        for (unsigned long long j = i + 1; j < k && key[j] == kk; ++j) {
            const uint32_t c = idx[j];
            const double cw = w[c];
            if (cw > bw) {   // graph.py:99 strict '>' keeps the earliest of equal weights
                bw = cw;
                best = c;
            }
        }
        first_flag[idx[i]] = 1u;   // idx ascending inside a run: idx[i] is the first occurrence
        kept[i] = best;
    }
}

__global__ void k_emit(const unsigned long long *key, const uint32_t *idx, unsigned long long k,
                       unsigned long long sentinel, const uint32_t *kept, const uint32_t *eid_of_pos,
                       const uint32_t *u, const uint32_t *v, const double *w, uint32_t *eu, uint32_t *ev,
                       double *ew) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k;
         i += stride) {
        const unsigned long long kk = key[i];
        if (kk == sentinel) continue;
        if (i > 0 && key[i - 1] == kk) continue;
        const uint32_t e = eid_of_pos[idx[i]];
        const uint32_t c = kept[i];
        eu[e] = u[c];
        ev[e] = v[c];
        ew[e] = w[c];
    }
}

__global__ void k_fill_ones(double *w, unsigned long long k) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride)
        w[i] = 1.0;
}

__global__ void k_export(const uint32_t *eu, const uint32_t *ev, unsigned long long m, long long *u,
                         long long *v) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < m;
         i += stride) {
        u[i] = eu[i];
        v[i] = ev[i];
    }
}

}  // namespace lmx

static int bgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    return (int)std::max<unsigned long long>(1, std::min(b, cap));
}

static int bits_for(unsigned long long n) {
    int b = 1;
    while (b < 32 && (1ULL << b) < n) ++b;
    return b;
}

// Dedupe/number raw triples ru/rv/rw (device, k entries) into ctx->eu/ev/w; frees the raw arrays.
static int build_from_raw(lmx_ctx *ctx, uint32_t *ru, uint32_t *rv, double *rw, unsigned long long k,
                          long long n) {
    cudaStream_t st = ctx->stream;
    const int bits = bits_for((unsigned long long)std::max<long long>(n, 2));
    const unsigned long long all = (bits >= 32) ? 0xFFFFFFFFULL : ((1ULL << bits) - 1);
    const unsigned long long sentinel = (all << bits) | all;
    unsigned long long *key = nullptr, *key2 = nullptr;
    uint32_t *idx = nullptr, *idx2 = nullptr, *flag = nullptr, *kept = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    const size_t kk = std::max<unsigned long long>(k, 1);
    int rc = LMX_OK;
    unsigned long long m = 0;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&key, kk * 8, "build keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&key2, kk * 8, "build keys2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&idx, kk * 4, "build idx")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&idx2, kk * 4, "build idx2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&flag, (kk + 1) * 4, "build flags")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&kept, kk * 4, "build kept")) != LMX_OK) break;
        k_pair_keys<<<bgrid(ctx, k), kBlock, 0, st>>>(ru, rv, k, bits, key, idx);
        if ((rc = lmx_sort_pairs(ctx, &key, &key2, &idx, &idx2, (long long)k, 0, 2 * bits, st, "build sort")) !=
            LMX_OK)
            break;
        size_t t2 = 0;
        cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, t2, flag, flag, (long long)(k + 1), st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "build sizing"); break; }
        tmp_bytes = t2;
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "build tmp")) != LMX_OK) break;
        e = cudaMemsetAsync(flag, 0, (kk + 1) * 4, st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "build sort"); break; }
        k_runs<<<bgrid(ctx, k), kBlock, 0, st>>>(key2, idx2, k, sentinel, ru, rv, rw, flag, kept);
        e = cub::DeviceScan::ExclusiveSum(tmp, t2, flag, flag, (long long)(k + 1), st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&m, flag + k, 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "build runs"); break; }
        m &= 0xFFFFFFFFULL;
        lmx_free_graph(ctx);
        ctx->n = n;
        ctx->m = (int64_t)m;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->eu, std::max<size_t>(m, 1) * 4, "edge_u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->ev, std::max<size_t>(m, 1) * 4, "edge_v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->w, std::max<size_t>(m, 1) * 8, "edge_weight")) != LMX_OK) break;
        k_emit<<<bgrid(ctx, k), kBlock, 0, st>>>(key2, idx2, k, sentinel, kept, flag, ru, rv, rw, ctx->eu,
                                                ctx->ev, ctx->w);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "build emit"); break; }
    } while (0);
    cudaStreamSynchronize(st);
    // dev_bytes accounting of these temporaries is not tracked after lmx_free_graph; just free
    lmx_dfree(ctx, key);
    lmx_dfree(ctx, key2);
    lmx_dfree(ctx, idx);
    lmx_dfree(ctx, idx2);
    lmx_dfree(ctx, flag);
    lmx_dfree(ctx, kept);
    lmx_dfree(ctx, tmp);
    lmx_dfree(ctx, ru);
    lmx_dfree(ctx, rv);
    lmx_dfree(ctx, rw);
    if (rc != LMX_OK) return rc;
    return lmx_setup_device_edges(ctx);
}

static RmatParams rmat_params(int scale, double a, double b, double c, uint64_t seed, int permute) {
    RmatParams p;
    p.scale = scale;
    const double A = std::nearbyint(a * 65536.0), B = std::nearbyint(b * 65536.0), C = std::nearbyint(c * 65536.0);
    p.A = (uint32_t)A;
    p.AB = (uint32_t)(A + B);
    p.ABC = (uint32_t)(A + B + C);
    p.s0 = mix64(seed ^ kRmatTag0);
    p.s1 = mix64(seed ^ kRmatTag1);
    p.s2 = mix64(seed ^ kRmatTag2);
    p.permute = permute;
    return p;
}

static int rmat_check(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c) {
    if (scale < 1 || scale > 31) return lmx_fail(ctx, LMX_EINVAL, "scale must be in [1, 31]");
    if (edge_factor < 1) return lmx_fail(ctx, LMX_EINVAL, "edge_factor must be >= 1");
    if (!(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0))
        return lmx_fail(ctx, LMX_EINVAL, "RMAT probabilities must be >= 0 with a+b+c <= 1");
    const unsigned long long k = (unsigned long long)edge_factor << scale;
    if (k >= 0xFFFFFFFFULL) return lmx_fail(ctx, LMX_ELIMIT, "raw edge count exceeds 32-bit positions");
    return LMX_OK;
}

extern "C" {

int lmx_gen_rmat_raw(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                     int permute, int64_t *u_out, int64_t *v_out, double *w_out, int out_where) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    LMX_TRY(rmat_check(ctx, scale, edge_factor, a, b, c));
    const unsigned long long k = (unsigned long long)edge_factor << scale;
    const RmatParams p = rmat_params(scale, a, b, c, seed, permute);
    uint32_t *ru = nullptr, *rv = nullptr;
    double *rw = nullptr;
    long long *lu = nullptr, *lv = nullptr;
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ru, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rv, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rw, k * 8));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&lu, k * 8));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&lv, k * 8));
    k_rmat_raw<<<bgrid(ctx, k), kBlock, 0, ctx->stream>>>(p, k, ru, rv, rw);
    k_export<<<bgrid(ctx, k), kBlock, 0, ctx->stream>>>(ru, rv, k, lu, lv);
    const cudaMemcpyKind kind = out_where == LMX_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    cudaError_t e = cudaMemcpyAsync(u_out, lu, k * 8, kind, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(v_out, lv, k * 8, kind, ctx->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(w_out, rw, k * 8, kind, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    lmx_dfree(ctx, ru);
    lmx_dfree(ctx, rv);
    lmx_dfree(ctx, rw);
    lmx_dfree(ctx, lu);
    lmx_dfree(ctx, lv);
    LMX_CUDA(ctx, e);
    return LMX_OK;
}

int lmx_gen_rmat(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                 int permute) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    LMX_TRY(rmat_check(ctx, scale, edge_factor, a, b, c));
    const unsigned long long k = (unsigned long long)edge_factor << scale;
    const RmatParams p = rmat_params(scale, a, b, c, seed, permute);
    lmx_free_graph(ctx);
    uint32_t *ru = nullptr, *rv = nullptr;
    double *rw = nullptr;
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ru, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rv, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rw, k * 8));
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    k_rmat_raw<<<bgrid(ctx, k), kBlock, 0, ctx->stream>>>(p, k, ru, rv, rw);
    LMX_CUDA(ctx, cudaGetLastError());
    LMX_TRY(build_from_raw(ctx, ru, rv, rw, k, 1LL << scale));
    lmx_flush_cache(ctx);   // the raw-build temporaries will not be reused
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    LMX_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.setup_ms = ms;
    return LMX_OK;
}

// G(n, m)-style random graph (the C1 family, generate.py:48-89, scaled up):
// k = edge_factor * 2^scale uniform raw pairs from the RMAT generator with
// a = b = c = d = 1/4, weights 1.0 (unit) or the generator's U[0,1), then
// build_graph semantics (self-loops dropped, duplicates collapsed).
int lmx_gen_er(lmx_ctx *ctx, int scale, int edge_factor, uint64_t seed, int unit_weights) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    LMX_TRY(rmat_check(ctx, scale, edge_factor, 0.25, 0.25, 0.25));
    const unsigned long long k = (unsigned long long)edge_factor << scale;
    const RmatParams p = rmat_params(scale, 0.25, 0.25, 0.25, seed, 0);
    lmx_free_graph(ctx);
    uint32_t *ru = nullptr, *rv = nullptr;
    double *rw = nullptr;
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ru, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rv, k * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rw, k * 8));
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    k_rmat_raw<<<bgrid(ctx, k), kBlock, 0, ctx->stream>>>(p, k, ru, rv, rw);
    if (unit_weights) k_fill_ones<<<bgrid(ctx, k), kBlock, 0, ctx->stream>>>(rw, k);
    LMX_CUDA(ctx, cudaGetLastError());
    LMX_TRY(build_from_raw(ctx, ru, rv, rw, k, 1LL << scale));
    lmx_flush_cache(ctx);
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    LMX_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.setup_ms = ms;
    return LMX_OK;
}

int lmx_build_graph(lmx_ctx *ctx, int64_t k, const int64_t *u, const int64_t *v, const double *w,
                    int64_t num_vertices, int where) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (k < 0) return lmx_fail(ctx, LMX_EINVAL, "negative triple count");
    if (k >= (int64_t)0xFFFFFFFFLL) return lmx_fail(ctx, LMX_ELIMIT, "triple count exceeds 32-bit positions");
    if (num_vertices >= (int64_t)0xFFFFFFFFLL) return lmx_fail(ctx, LMX_ELIMIT, "n exceeds 32-bit ids");
    lmx_free_graph(ctx);
    cudaStream_t st = ctx->stream;
    const unsigned long long kk = (unsigned long long)k;
    uint32_t *ru = nullptr, *rv = nullptr;
    double *rw = nullptr;
    unsigned long long *flags = nullptr;   // [0] first bad, [1] max id + 1
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&ru, std::max<size_t>(kk, 1) * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rv, std::max<size_t>(kk, 1) * 4));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&rw, std::max<size_t>(kk, 1) * 8));
    LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&flags, 16));
    unsigned long long init[2] = {~0ULL, 0ULL};
    LMX_CUDA(ctx, cudaMemcpyAsync(flags, init, 16, cudaMemcpyHostToDevice, st));
    cudaError_t e = cudaSuccess;
    if (kk > 0) {
        if (where == LMX_DEVICE) {
            k_raw_convert<<<bgrid(ctx, kk), kBlock, 0, st>>>((const long long *)u, (const long long *)v, w, kk,
                                                             num_vertices, 0, ru, rv, rw, flags, flags + 1);
            e = cudaGetLastError();
        } else {
            const unsigned long long chunk = 1ULL << 24;
            const size_t cb = std::min<unsigned long long>(chunk, kk);
            long long *su = nullptr, *sv = nullptr;
            double *sw = nullptr;
            LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&su, cb * 8));
            LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&sv, cb * 8));
            LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&sw, cb * 8));
            for (unsigned long long off = 0; off < kk && e == cudaSuccess; off += chunk) {
                const unsigned long long c = std::min(chunk, kk - off);
                e = cudaMemcpyAsync(su, u + off, c * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaMemcpyAsync(sv, v + off, c * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) e = cudaMemcpyAsync(sw, w + off, c * 8, cudaMemcpyHostToDevice, st);
                if (e == cudaSuccess) {
                    k_raw_convert<<<bgrid(ctx, c), kBlock, 0, st>>>(su, sv, sw, c, num_vertices, off, ru, rv, rw,
                                                                   flags, flags + 1);
                    e = cudaGetLastError();
                }
            }
            cudaStreamSynchronize(st);
            lmx_dfree(ctx, su);
            lmx_dfree(ctx, sv);
            lmx_dfree(ctx, sw);
        }
    }
    unsigned long long got[2] = {0, 0};
    if (e == cudaSuccess) e = cudaMemcpyAsync(got, flags, 16, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    lmx_dfree(ctx, flags);
    if (e != cudaSuccess) {
        lmx_dfree(ctx, ru);
        lmx_dfree(ctx, rv);
        lmx_dfree(ctx, rw);
        return lmx_cuda_check(ctx, e, "build_graph input");
    }
    if (got[0] != ~0ULL) {
        lmx_dfree(ctx, ru);
        lmx_dfree(ctx, rv);
        lmx_dfree(ctx, rw);
        const unsigned long long pos = got[0];
        int64_t a = 0, b = 0;
        double x = 0;
        if (where == LMX_HOST) {
            a = u[pos];
            b = v[pos];
            x = w[pos];
        } else {
            cudaMemcpy(&a, u + pos, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&b, v + pos, 8, cudaMemcpyDeviceToHost);
            cudaMemcpy(&x, w + pos, 8, cudaMemcpyDeviceToHost);
        }
        char buf[256];
        if (a < 0 || b < 0)
            snprintf(buf, sizeof buf, "edge %llu: negative vertex id (%lld, %lld)", pos, (long long)a, (long long)b);
        else if (num_vertices >= 0 && (a >= num_vertices || b >= num_vertices))
            snprintf(buf, sizeof buf, "edge %llu: vertex id out of range for n=%lld: (%lld, %lld)", pos,
                     (long long)num_vertices, (long long)a, (long long)b);
        else if (std::isnan(x) || std::isinf(x) || x < 0)
            snprintf(buf, sizeof buf, "edge %llu: weight must be finite and >= 0, got %.17g", pos, x);
        else
            snprintf(buf, sizeof buf, "edge %llu: vertex id exceeds 32-bit range", pos);
        return lmx_fail(ctx, LMX_EINVAL, buf);
    }
    const long long n = num_vertices >= 0 ? num_vertices : (long long)got[1];
    const int rc = build_from_raw(ctx, ru, rv, rw, kk, n);
    lmx_flush_cache(ctx);   // the raw-build temporaries will not be reused
    return rc;
}

int lmx_graph_export(lmx_ctx *ctx, int64_t *edge_u, int64_t *edge_v, double *edge_weight, int out_where) {
    if (!ctx) return LMX_EINVAL;
    if (ctx->dist_local) return lmx_fail(ctx, LMX_ESTATE, "a partition holds only its local edges");
    cudaSetDevice(ctx->device);
    const unsigned long long m = (unsigned long long)ctx->m;
    if (m == 0) return LMX_OK;
    long long *lu = nullptr, *lv = nullptr;
    if (out_where == LMX_DEVICE) {
        lu = (long long *)edge_u;
        lv = (long long *)edge_v;
    } else {
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&lu, m * 8));
        LMX_CUDA(ctx, lmx_dmalloc(ctx, (void **)&lv, m * 8));
    }
    k_export<<<bgrid(ctx, m), kBlock, 0, ctx->stream>>>(ctx->eu, ctx->ev, m, lu, lv);
    cudaError_t e = cudaGetLastError();
    const cudaMemcpyKind kind = out_where == LMX_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost;
    if (e == cudaSuccess && out_where != LMX_DEVICE) {
        e = cudaMemcpyAsync(edge_u, lu, m * 8, kind, ctx->stream);
        if (e == cudaSuccess) e = cudaMemcpyAsync(edge_v, lv, m * 8, kind, ctx->stream);
    }
    if (e == cudaSuccess && edge_weight) e = cudaMemcpyAsync(edge_weight, ctx->w, m * 8, kind, ctx->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (out_where != LMX_DEVICE) {
        lmx_dfree(ctx, lu);
        lmx_dfree(ctx, lv);
    }
    LMX_CUDA(ctx, e);
    return LMX_OK;
}

}  // extern "C"

// ---- distributed RMAT build (C ABI, see include/lmx.h) ---------------------

namespace lmx {
__global__ void k_pair_minmax(const double *w, unsigned long long k, unsigned long long *mm) {
    unsigned long long lo = ~0ULL, hi = 0;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        unsigned long long b = (unsigned long long)__double_as_longlong(w[i]);
        b = (b << 1) == 0 ? 0ULL : b;
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
}  // namespace lmx

extern "C" {

// Phase 1: generate the whole raw stream, keep the triples whose unordered
// pair hashes to this rank, collapse parallel pairs (graph.py:94-100) and
// record each pair's first raw position.
int lmx_dist_rmat_build(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                        int permute, void **bits_dev, int64_t *words_out, void **deg_dev, void **minmax_dev) {
    if (!ctx || !bits_dev || !words_out || !deg_dev || !minmax_dev) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (ctx->dist_p < 2) return lmx_fail(ctx, LMX_ESTATE, "set LMX_OPT_DIST_P > 1 first");
    LMX_TRY(rmat_check(ctx, scale, edge_factor, a, b, c));
    const unsigned long long n = 1ULL << scale, k = (unsigned long long)edge_factor << scale;
    const RmatParams P = rmat_params(scale, a, b, c, seed, permute);
    const int p = ctx->dist_p, rank = ctx->dist_rank;
    lmx_free_graph(ctx);
    ctx->n = (int64_t)n;
    cudaStream_t st = ctx->stream;
    unsigned long long *cursor = nullptr, *key = nullptr, *key2 = nullptr;
    uint32_t *ku = nullptr, *kv = nullptr, *kpos = nullptr, *idx = nullptr, *idx2 = nullptr;
    double *kw = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    unsigned long long K = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    do {
        if ((rc = lmx_alloc(ctx, (void **)&cursor, 16, "keep cursor")) != LMX_OK) break;
        e = cudaMemsetAsync(cursor, 0, 16, st);
        if (e != cudaSuccess) break;
        k_rmat_keep<false><<<bgrid(ctx, k), kBlock, 0, st>>>(P, k, (uint32_t)p, (uint32_t)rank, cursor, nullptr,
                                                            nullptr, nullptr, nullptr);
        e = cudaMemcpyAsync(&K, cursor, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        const size_t K1 = std::max<unsigned long long>(K, 1);
        if ((rc = lmx_alloc(ctx, (void **)&ku, K1 * 4, "kept u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&kv, K1 * 4, "kept v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&kw, K1 * 8, "kept w")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&kpos, K1 * 4, "kept pos")) != LMX_OK) break;
        e = cudaMemsetAsync(cursor, 0, 16, st);
        if (e != cudaSuccess) break;
        k_rmat_keep<true><<<bgrid(ctx, k), kBlock, 0, st>>>(P, k, (uint32_t)p, (uint32_t)rank, cursor, ku, kv, kw,
                                                           kpos);
        // group the kept triples by pair
        const int bits = bits_for(n);
        if ((rc = lmx_alloc(ctx, (void **)&key, K1 * 8, "pair keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&key2, K1 * 8, "pair keys2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&idx, K1 * 4, "pair idx")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&idx2, K1 * 4, "pair idx2")) != LMX_OK) break;
        k_pair_keys_local<<<bgrid(ctx, K1), kBlock, 0, st>>>(ku, kv, K, bits, key, idx);
        if ((rc = lmx_sort_pairs(ctx, &key, &key2, &idx, &idx2, (long long)K, 0, 2 * bits, st, "pair sort")) !=
            LMX_OK)
            break;
        lmx_free(ctx, (void **)&key, K1 * 8);
        lmx_free(ctx, (void **)&idx, K1 * 4);
        // pairs, first-occurrence bits, degree contributions
        ctx->db_words = (k + 31) / 32;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_bits, ctx->db_words * 4, "first-occurrence bits")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->deg0, n * 4, "deg0")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_pf, K1 * 4, "pairs first")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_pu, K1 * 4, "pairs u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_pv, K1 * 4, "pairs v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_pw, K1 * 8, "pairs w")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->db_minmax, 16, "pair minmax")) != LMX_OK) break;
        ctx->db_cap = K1;
        e = cudaMemsetAsync(ctx->db_bits, 0, ctx->db_words * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(ctx->deg0, 0, n * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(cursor, 0, 16, st);
        unsigned long long mm0[2] = {~0ULL, 0ULL};
        if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->db_minmax, mm0, 16, cudaMemcpyHostToDevice, st);
        if (e != cudaSuccess) break;
        if (K)
            k_runs_dist<<<bgrid(ctx, K), kBlock, 0, st>>>(key2, idx2, K, ku, kv, kw, kpos, ctx->db_bits, ctx->deg0,
                                                         ctx->db_pf, ctx->db_pu, ctx->db_pv, ctx->db_pw, cursor);
        e = cudaMemcpyAsync(&ctx->db_np, cursor, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        if (ctx->db_np)
            k_pair_minmax<<<bgrid(ctx, ctx->db_np), kBlock, 0, st>>>(ctx->db_pw, ctx->db_np, ctx->db_minmax);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    } while (0);
    const size_t K1 = std::max<unsigned long long>(K, 1);
    lmx_free(ctx, (void **)&cursor, 16);
    lmx_free(ctx, (void **)&key, K1 * 8);
    lmx_free(ctx, (void **)&key2, K1 * 8);
    lmx_free(ctx, (void **)&idx, K1 * 4);
    lmx_free(ctx, (void **)&idx2, K1 * 4);
    lmx_free(ctx, (void **)&ku, K1 * 4);
    lmx_free(ctx, (void **)&kv, K1 * 4);
    lmx_free(ctx, (void **)&kw, K1 * 8);
    lmx_free(ctx, (void **)&kpos, K1 * 4);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, e);
    *bits_dev = ctx->db_bits;
    *words_out = (int64_t)ctx->db_words;
    *deg_dev = ctx->deg0;
    *minmax_dev = ctx->db_minmax;
    return LMX_OK;
}

// Phase 2 (after the bitmap and the degrees are summed over the ranks): the
// global edge ids (first occurrences numbered in raw order, graph.py:94-98),
// partition_graph's cuts on the global degrees, and the records of this
// rank's pairs packed by destination (the owners of both ends).
int lmx_dist_rmat_route(lmx_ctx *ctx, void **send_dev, int64_t *counts_out, int64_t *m_out) {
    if (!ctx || !send_dev || !counts_out || !m_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (!ctx->db_bits) return lmx_fail(ctx, LMX_ESTATE, "lmx_dist_rmat_build first");
    cudaStream_t st = ctx->stream;
    const int p = ctx->dist_p;
    const unsigned long long W = ctx->db_words, np = ctx->db_np;
    unsigned long long *prefix = nullptr, *cnt = nullptr, *region = nullptr, *bdev = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    unsigned long long m = 0;
    std::vector<unsigned long long> hc((size_t)p, 0), hr((size_t)p + 1, 0);
    do {
        if ((rc = lmx_alloc(ctx, (void **)&prefix, (W + 1) * 8, "word prefix")) != LMX_OK) break;
        k_word_popc<<<bgrid(ctx, W + 1), kBlock, 0, st>>>(ctx->db_bits, W, prefix);
        e = cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, prefix, prefix, (long long)(W + 1), st);
        if (e != cudaSuccess) break;
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "prefix tmp")) != LMX_OK) break;
        e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, prefix, prefix, (long long)(W + 1), st);
        if (e == cudaSuccess) e = cudaMemcpyAsync(&m, prefix + W, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        if (m >= 0xFFFFFFFFULL) { rc = lmx_fail(ctx, LMX_ELIMIT, "m exceeds the 32-bit edge id range"); break; }
        ctx->m = (int64_t)m;
        if ((rc = lmx_partition_bounds(ctx, ctx->bounds)) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&bdev, (size_t)(p + 1) * 8, "bounds")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cnt, (size_t)p * 8, "route counts")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&region, (size_t)(p + 1) * 8, "route regions")) != LMX_OK) break;
        std::vector<unsigned long long> hb(ctx->bounds.begin(), ctx->bounds.end());
        e = cudaMemcpyAsync(bdev, hb.data(), (size_t)(p + 1) * 8, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (size_t)p * 8, st);
        if (e != cudaSuccess) break;
        if (np)
            k_route<false><<<bgrid(ctx, np), kBlock, 0, st>>>(ctx->db_pf, ctx->db_pu, ctx->db_pv, ctx->db_pw, np,
                                                             ctx->db_bits, prefix, bdev, p, cnt, nullptr, nullptr);
        e = cudaMemcpyAsync(hc.data(), cnt, (size_t)p * 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        for (int q = 0; q < p; ++q) hr[(size_t)q + 1] = hr[(size_t)q] + hc[(size_t)q];
        ctx->db_send_n = hr[(size_t)p];
        if ((rc = lmx_alloc(ctx, &ctx->db_send, std::max<unsigned long long>(ctx->db_send_n, 1) * sizeof(DistRec),
                            "route records")) != LMX_OK)
            break;
        e = cudaMemcpyAsync(region, hr.data(), (size_t)(p + 1) * 8, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(cnt, 0, (size_t)p * 8, st);
        if (e != cudaSuccess) break;
        if (np)
            k_route<true><<<bgrid(ctx, np), kBlock, 0, st>>>(ctx->db_pf, ctx->db_pu, ctx->db_pv, ctx->db_pw, np,
                                                            ctx->db_bits, prefix, bdev, p, cnt, region,
                                                            reinterpret_cast<DistRec *>(ctx->db_send));
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    } while (0);
    lmx_free(ctx, (void **)&prefix, (W + 1) * 8);
    lmx_free(ctx, (void **)&cnt, (size_t)p * 8);
    lmx_free(ctx, (void **)&region, (size_t)(p + 1) * 8);
    lmx_free(ctx, (void **)&bdev, (size_t)(p + 1) * 8);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, e);
    // the build's pair arrays and bitmap are no longer needed
    lmx_free(ctx, (void **)&ctx->db_bits, W * 4);
    lmx_free(ctx, (void **)&ctx->db_pf, ctx->db_cap * 4);
    lmx_free(ctx, (void **)&ctx->db_pu, ctx->db_cap * 4);
    lmx_free(ctx, (void **)&ctx->db_pv, ctx->db_cap * 4);
    lmx_free(ctx, (void **)&ctx->db_pw, ctx->db_cap * 8);
    for (int q = 0; q < p; ++q) counts_out[q] = (int64_t)hc[(size_t)q];
    *send_dev = ctx->db_send;
    *m_out = (int64_t)m;
    return LMX_OK;
}

int lmx_dist_rmat_recv_buffer(lmx_ctx *ctx, int64_t count, void **recv_dev) {
    if (!ctx || !recv_dev || count < 0) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    lmx_free(ctx, &ctx->db_recv, std::max<unsigned long long>(ctx->db_recv_n, 1) * sizeof(DistRec));
    ctx->db_recv_n = (unsigned long long)count;
    LMX_TRY(lmx_alloc(ctx, &ctx->db_recv, std::max<unsigned long long>(ctx->db_recv_n, 1) * sizeof(DistRec),
                      "received records"));
    *recv_dev = ctx->db_recv;
    return LMX_OK;
}

int lmx_dist_load_local(lmx_ctx *ctx, int64_t n, int64_t m, const uint32_t *deg, int64_t k, const void *records,
                        int w_uniform) {
    if (!ctx || n < 1 || m < 0 || k < 0 || k > m || !deg || (k && !records)) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (ctx->dist_p < 2) return lmx_fail(ctx, LMX_ESTATE, "set LMX_OPT_DIST_P > 1 first");
    if (n > (int64_t)0xFFFFFFFEu || m > (int64_t)0xFFFFFFFEu)
        return lmx_fail(ctx, LMX_ELIMIT, "more than 2^32 - 2 vertices or edges");
    lmx_free_graph(ctx);
    ctx->n = n;
    ctx->m = m;
    cudaStream_t st = ctx->stream;
    LMX_TRY(lmx_alloc(ctx, (void **)&ctx->deg0, (size_t)n * 4, "global degrees"));
    LMX_CUDA(ctx, cudaMemcpyAsync(ctx->deg0, deg, (size_t)n * 4, cudaMemcpyHostToDevice, st));
    void *dst = nullptr;
    LMX_TRY(lmx_dist_rmat_recv_buffer(ctx, k, &dst));
    if (k) LMX_CUDA(ctx, cudaMemcpyAsync(dst, records, (size_t)k * sizeof(DistRec), cudaMemcpyHostToDevice, st));
    return lmx_dist_rmat_finish(ctx, w_uniform);
}

// Phase 3: the received records are this rank's local edges (bsp.py:86-90),
// in arrival order (slots carry the global edge ids, so the local order is
// free); then the partition's K0.
int lmx_dist_rmat_finish(lmx_ctx *ctx, int w_uniform) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (!ctx->db_recv) return lmx_fail(ctx, LMX_ESTATE, "lmx_dist_rmat_recv_buffer first");
    cudaStream_t st = ctx->stream;
    const unsigned long long k = ctx->db_recv_n;
    const size_t k1 = std::max<unsigned long long>(k, 1);
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    lmx_free(ctx, &ctx->db_send, std::max<unsigned long long>(ctx->db_send_n, 1) * sizeof(DistRec));
    do {
        if ((rc = lmx_alloc(ctx, (void **)&ctx->eu, k1 * 4, "local edge_u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->ev, k1 * 4, "local edge_v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->w, k1 * 8, "local edge_weight")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->geid, k1 * 4, "local edge ids")) != LMX_OK) break;
        if (k) {
            k_rec_unpack<<<bgrid(ctx, k), kBlock, 0, st>>>(reinterpret_cast<const DistRec *>(ctx->db_recv), nullptr,
                                                          k, ctx->eu, ctx->ev, ctx->w, ctx->geid);
            e = cudaGetLastError();
        }
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    } while (0);
    lmx_free(ctx, &ctx->db_recv, k1 * sizeof(DistRec));
    lmx_free(ctx, (void **)&ctx->db_minmax, 16);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, e);
    ctx->m_local = (int64_t)k;
    ctx->dist_local = true;
    ctx->w_uniform = w_uniform ? 1 : 0;
    LMX_TRY(lmx_weight_stage(ctx));   // on the local edges
    LMX_TRY(lmx_setup_slots(ctx));
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
    LMX_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.setup_ms = ms;
    return LMX_OK;
}

}  // extern "C"
