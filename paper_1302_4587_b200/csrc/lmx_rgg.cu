// lmx_rgg.cu -- the reference's random geometric graph generator on the device
// (gen_rgg, generate.py:113-143 with radius_edges_grid :146-197 and
// _morton_order :97-110), emitting the identical edge list, so BASELINE
// config C2 (x = 22) is built in milliseconds instead of minutes of Python.
//
//   points   numpy's default_rng(seed).random((n, 2)): PCG64 (XSL-RR 128/64,
//            step then output) from the initial state the caller takes from
//            numpy's SeedSequence; each thread jumps ahead to its chunk
//            (LCG advance in O(log k)); double = (u64 >> 11) * 2^-53
//   order    stable sort by the Morton key of (clip(uint32(p * 65536), 65535))
//   cells    side = floor(1 / r) cells per axis, c = min(int(x / (1 / side)),
//            side - 1); points ordered by (cell, index)
//   edges    per cell ascending, per own point in that order, candidates of
//            the 3 x 3 neighbourhood (dx outer, dy inner, each cell in index
//            order): own < cand and d2 < r2 with d2 = dx*dx + dy*dy rounded
//            per operation (numpy's einsum: no fused multiply-add);
//            weight sqrt(d2) ("euclidean") or the next rng.random(m) draws
//            ("random").  Pairs are distinct with u < v, so build_graph's
//            numbering is the emission order.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>

#include "lmx_internal.cuh"

using namespace lmx;

namespace lmx {

typedef unsigned __int128 u128;

__host__ __device__ __forceinline__ u128 pcg_mult() {
    return ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
}

// state after `delta` steps (PCG's LCG jump-ahead)
__device__ __forceinline__ u128 pcg_advance(u128 state, u128 inc, unsigned long long delta) {
    u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
    while (delta) {
        if (delta & 1ULL) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

__device__ __forceinline__ double pcg_double(u128 &state, u128 inc) {
    state = state * pcg_mult() + inc;
    const unsigned long long hi = (unsigned long long)(state >> 64), lo = (unsigned long long)state;
    const unsigned long long x = hi ^ lo;
    const unsigned rot = (unsigned)(hi >> 58);
    const unsigned long long o = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(o >> 11) * (1.0 / 9007199254740992.0);
}

// out[j] = the (first + j)-th random() draw, j < k; chunks of `chunk` per thread
__global__ void k_pcg_doubles(unsigned long long s_hi, unsigned long long s_lo, unsigned long long i_hi,
                              unsigned long long i_lo, unsigned long long first, unsigned long long k,
                              unsigned long long chunk, double *out) {
    const unsigned long long t = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned long long j0 = t * chunk;
    if (j0 >= k) return;
    const u128 inc = ((u128)i_hi << 64) | (u128)i_lo;
    u128 st = pcg_advance(((u128)s_hi << 64) | (u128)s_lo, inc, first + j0);
    const unsigned long long j1 = min(k, j0 + chunk);
    for (unsigned long long j = j0; j < j1; ++j) out[j] = pcg_double(st, inc);
}

__device__ __forceinline__ unsigned long long spread16(unsigned long long b) {
    b = (b | (b << 16)) & 0x0000FFFF0000FFFFULL;
    b = (b | (b << 8)) & 0x00FF00FF00FF00FFULL;
    b = (b | (b << 4)) & 0x0F0F0F0F0F0F0F0FULL;
    b = (b | (b << 2)) & 0x3333333333333333ULL;
    b = (b | (b << 1)) & 0x5555555555555555ULL;
    return b;
}

__device__ __forceinline__ unsigned long long quant16(double v) {
    // np.clip((p * 65536.0).astype(np.uint32), 0, 65535); p in [0, 1)
    const double s = __dmul_rn(v, 65536.0);
    unsigned long long q = (unsigned long long)s;
    return q > 65535ULL ? 65535ULL : q;
}

__global__ void k_morton_keys(const double *xy, unsigned long long n, unsigned long long *key, uint32_t *idx) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        key[i] = spread16(quant16(xy[2 * i])) | (spread16(quant16(xy[2 * i + 1])) << 1);
        idx[i] = (uint32_t)i;
    }
}

// points in Morton order + their cells
__global__ void k_cells(const double *xy, const uint32_t *perm, unsigned long long n, double inv_side, long long side,
                        double2 *P, uint32_t *cell, uint32_t *idx) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t j = perm[i];
        const double x = xy[2 * j], y = xy[2 * j + 1];
        P[i] = make_double2(x, y);
        long long cx = (long long)__ddiv_rn(x, inv_side), cy = (long long)__ddiv_rn(y, inv_side);
        cx = cx < side - 1 ? cx : side - 1;
        cy = cy < side - 1 ? cy : side - 1;
        cell[i] = (uint32_t)(cx * side + cy);
        idx[i] = (uint32_t)i;
    }
}

__global__ void k_cell_bounds(const uint32_t *sorted_cell, unsigned long long n, uint32_t *cbeg, uint32_t *cend) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        const uint32_t c = sorted_cell[i];
        if (i == 0 || sorted_cell[i - 1] != c) cbeg[c] = (uint32_t)i;
        if (i + 1 == n || sorted_cell[i + 1] != c) cend[c] = (uint32_t)i + 1;
    }
}

// Pass 0: count the edges of each own point (position p of the (cell, index)
// order); pass 1: write them at off[p].
template <bool WRITE>
__global__ void k_rgg_edges(const double2 *P, const uint32_t *order, const uint32_t *sorted_cell, const uint32_t *cbeg,
                            const uint32_t *cend, unsigned long long n, long long side, double r2,
                            unsigned long long *cnt, uint32_t *eu, uint32_t *ev, double *dist) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long p = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += stride) {
        const uint32_t own = order[p];
        const uint32_t c = sorted_cell[p];
        const long long px = c / side, py = c % side;
        const double2 a = P[own];
        unsigned long long k = WRITE ? cnt[p] : 0ULL;
        for (int dx = -1; dx <= 1; ++dx) {
            const long long qx = px + dx;
            if (qx < 0 || qx >= side) continue;
            for (int dy = -1; dy <= 1; ++dy) {
                const long long qy = py + dy;
                if (qy < 0 || qy >= side) continue;
                const uint32_t q = (uint32_t)(qx * side + qy);
                const uint32_t b = cbeg[q], e = cend[q];
                for (uint32_t s = b; s < e; ++s) {
                    const uint32_t cand = order[s];
                    if (own >= cand) continue;
                    const double2 bq = P[cand];
                    const double d0 = __dsub_rn(a.x, bq.x), d1 = __dsub_rn(a.y, bq.y);
                    const double d2 = __dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1));
                    if (d2 < r2) {
                        if (WRITE) {
                            eu[k] = own;
                            ev[k] = cand;
                            dist[k] = __dsqrt_rn(d2);
                        }
                        ++k;
                    }
                }
            }
        }
        if (!WRITE) cnt[p] = k;
    }
}

}  // namespace lmx

static int rgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    const unsigned long long cap = (unsigned long long)ctx->num_sms * 16;
    return (int)std::max<unsigned long long>(1, std::min(b, cap));
}

extern "C" int lmx_gen_rgg(lmx_ctx *ctx, int x, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi,
                           uint64_t inc_lo, double radius, int weight_random) {
    if (!ctx) return LMX_EINVAL;
    if (x < 2 || x > 30) return lmx_fail(ctx, LMX_EINVAL, "x must be in [2, 30]");
    if (!(radius > 0.0)) return lmx_fail(ctx, LMX_EINVAL, "radius must be > 0");
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    lmx_free_graph(ctx);
    cudaStream_t st = ctx->stream;
    const unsigned long long n = 1ULL << x;
    const long long side = std::max(1LL, (long long)std::floor(1.0 / radius));
    const double inv_side = 1.0 / (double)side;
    const double r2 = radius * radius;
    double *xy = nullptr;
    double2 *P = nullptr;
    unsigned long long *key = nullptr, *key2 = nullptr, *cnt = nullptr;
    uint32_t *idx = nullptr, *perm = nullptr, *cell = nullptr, *cell2 = nullptr, *order = nullptr, *cbeg = nullptr,
             *cend = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    const unsigned long long ncell = (unsigned long long)side * (unsigned long long)side;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, st));
    do {
        if ((rc = lmx_alloc(ctx, (void **)&xy, 2 * n * 8, "rgg points")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&key, n * 8, "morton keys")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&key2, n * 8, "morton keys2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&idx, n * 4, "idx")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&perm, n * 4, "perm")) != LMX_OK) break;
        const unsigned long long chunk = 64, k = 2 * n;
        k_pcg_doubles<<<(unsigned)((k / chunk + kBlock) / kBlock), kBlock, 0, st>>>(state_hi, state_lo, inc_hi, inc_lo,
                                                                                  0, k, chunk, xy);
        k_morton_keys<<<rgrid(ctx, n), kBlock, 0, st>>>(xy, n, key, idx);
        e = cub::DeviceRadixSort::SortPairs(nullptr, tmp_bytes, key, key2, idx, perm, (long long)n, 0, 32, st);
        if (e != cudaSuccess) break;
        if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "rgg sort tmp")) != LMX_OK) break;
        e = cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, key, key2, idx, perm, (long long)n, 0, 32, st);
        if (e != cudaSuccess) break;
        lmx_free(ctx, (void **)&key, n * 8);
        lmx_free(ctx, (void **)&key2, n * 8);
        if ((rc = lmx_alloc(ctx, (void **)&P, n * 16, "rgg morton points")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cell, n * 4, "cells")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cell2, n * 4, "cells2")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&order, n * 4, "cell order")) != LMX_OK) break;
        k_cells<<<rgrid(ctx, n), kBlock, 0, st>>>(xy, perm, n, inv_side, side, P, cell, idx);
        int cb = 1;
        while (cb < 32 && (1ULL << cb) < ncell) ++cb;
        size_t need = 0;
        e = cub::DeviceRadixSort::SortPairs(nullptr, need, cell, cell2, idx, order, (long long)n, 0, cb, st);
        if (e != cudaSuccess) break;
        if (need > tmp_bytes) {
            lmx_free(ctx, &tmp, tmp_bytes);
            tmp_bytes = need;
            if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "rgg sort tmp")) != LMX_OK) break;
        }
        e = cub::DeviceRadixSort::SortPairs(tmp, need, cell, cell2, idx, order, (long long)n, 0, cb, st);
        if (e != cudaSuccess) break;
        if ((rc = lmx_alloc(ctx, (void **)&cbeg, ncell * 4, "cell begin")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&cend, ncell * 4, "cell end")) != LMX_OK) break;
        e = cudaMemsetAsync(cbeg, 0, ncell * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(cend, 0, ncell * 4, st);
        if (e != cudaSuccess) break;
        k_cell_bounds<<<rgrid(ctx, n), kBlock, 0, st>>>(cell2, n, cbeg, cend);
        if ((rc = lmx_alloc(ctx, (void **)&cnt, (n + 1) * 8, "edge counts")) != LMX_OK) break;
        k_rgg_edges<false><<<rgrid(ctx, n), kBlock, 0, st>>>(P, order, cell2, cbeg, cend, n, side, r2, cnt, nullptr,
                                                            nullptr, nullptr);
        e = cudaMemsetAsync(cnt + n, 0, 8, st);
        size_t need2 = 0;
        if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, need2, cnt, cnt, (long long)(n + 1), st);
        if (e != cudaSuccess) break;
        if (need2 > tmp_bytes) {
            lmx_free(ctx, &tmp, tmp_bytes);
            tmp_bytes = need2;
            if ((rc = lmx_alloc(ctx, &tmp, tmp_bytes, "rgg scan tmp")) != LMX_OK) break;
        }
        e = cub::DeviceScan::ExclusiveSum(tmp, need2, cnt, cnt, (long long)(n + 1), st);
        unsigned long long m = 0;
        if (e == cudaSuccess) e = cudaMemcpyAsync(&m, cnt + n, 8, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) break;
        if (m >= 0xFFFFFFFFULL) { rc = lmx_fail(ctx, LMX_ELIMIT, "m exceeds the 32-bit edge id range"); break; }
        ctx->n = (int64_t)n;
        ctx->m = (int64_t)m;
        const size_t mm = std::max<unsigned long long>(m, 1);
        if ((rc = lmx_alloc(ctx, (void **)&ctx->eu, mm * 4, "edge_u")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->ev, mm * 4, "edge_v")) != LMX_OK) break;
        if ((rc = lmx_alloc(ctx, (void **)&ctx->w, mm * 8, "edge_weight")) != LMX_OK) break;
        k_rgg_edges<true><<<rgrid(ctx, n), kBlock, 0, st>>>(P, order, cell2, cbeg, cend, n, side, r2, cnt, ctx->eu,
                                                           ctx->ev, ctx->w);
        if (weight_random && m) {   // rng.random(m): the draws after the 2n coordinates
            k_pcg_doubles<<<(unsigned)((m / chunk + kBlock) / kBlock), kBlock, 0, st>>>(state_hi, state_lo, inc_hi,
                                                                                      inc_lo, 2 * n, m, chunk, ctx->w);
        }
        e = cudaGetLastError();
    } while (0);
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&xy, 2 * n * 8);
    lmx_free(ctx, (void **)&key, n * 8);
    lmx_free(ctx, (void **)&key2, n * 8);
    lmx_free(ctx, (void **)&idx, n * 4);
    lmx_free(ctx, (void **)&perm, n * 4);
    lmx_free(ctx, (void **)&P, n * 16);
    lmx_free(ctx, (void **)&cell, n * 4);
    lmx_free(ctx, (void **)&cell2, n * 4);
    lmx_free(ctx, (void **)&order, n * 4);
    lmx_free(ctx, (void **)&cbeg, ncell * 4);
    lmx_free(ctx, (void **)&cend, ncell * 4);
    lmx_free(ctx, (void **)&cnt, (n + 1) * 8);
    lmx_free(ctx, &tmp, tmp_bytes);
    if (rc != LMX_OK) {
        lmx_free_graph(ctx);
        return rc;
    }
    if (e != cudaSuccess) {
        lmx_free_graph(ctx);
        return lmx_cuda_check(ctx, e, "rgg generator");
    }
    rc = lmx_setup_device_edges(ctx);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, st));
    LMX_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.setup_ms = ms;
    return LMX_OK;
}
