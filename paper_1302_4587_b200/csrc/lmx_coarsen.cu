// lmx_coarsen.cu -- graph-partitioning coarsening on the device (config C4,
// SURVEY.md §8f rank 2; the paper's motivating use).
//
// One level = local max matching (lmx_match) on edge ratings, then contraction:
//   ratings  r(e) = w(e)^2 / (c(u) c(v))   (w = edge weight, c = node weight)
//   coarse ids: every matched pair and every unmatched vertex becomes one coarse
//     vertex, numbered by the smaller member in ascending order (prefix sum
//     over "representative" flags: v unmatched or v < mate[v])
//   coarse node weight = sum of the members' c
//   coarse edges: fine edges between different coarse vertices, parallel edges
//     merged by summing w; listed in ascending (min, max) coarse-pair order,
//     oriented (min, max), edge id = position
// The reference has no contraction; oracle/oracle.py:contract
// restates these rules in numpy for the parity tests.  Weights in the mesh
// pipeline are integer-valued sums (unit level-0 weights), so every f64 sum is
// exact and independent of summation order.
//
// Mesh: side x side jittered-grid triangulation ("Delaunay-style"): vertex
// i*side + j, edges right, down and one diagonal per cell whose direction is a
// counter-based hash of (seed, cell), enumerated cell by cell in row-major
// order (right, down, diagonal).
#include <cub/cub.cuh>

#include <algorithm>

#include "lmx_internal.cuh"

using namespace lmx;

namespace lmx {

constexpr uint64_t kMeshTag = 0x4D4553485F444941ULL;   // "MESH_DIA"

// Edges of vertex (i, j), in this order: right (i, j+1), down (i+1, j), the
// diagonal of cell (i, j).  Rows 0..side-2 emit 3*side - 2 edges each (the last
// column only 'down'), the last row side - 1 'right' edges, so vertex (i, j)'s
// first edge is i*(3*side - 2) + j*(i < side-1 ? 3 : 1).
__global__ void k_mesh(unsigned long long side, unsigned long long seed_mix, long long *eu, long long *ev,
                       double *w) {
    const unsigned long long n = side * side;
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const unsigned long long i = v / side, j = v % side;
        const unsigned long long has_down = (i + 1 < side) ? 1 : 0;
        unsigned long long e = i * (3 * side - 2) + j * (has_down ? 3 : 1);
        if (j + 1 < side) {
            eu[e] = (long long)v;
            ev[e] = (long long)(v + 1);
            w[e] = 1.0;
            ++e;
        }
        if (has_down) {
            eu[e] = (long long)v;
            ev[e] = (long long)(v + side);
            w[e] = 1.0;
            ++e;
            if (j + 1 < side) {
                const bool main = (mix64(seed_mix ^ v) & 1ULL) != 0;
                eu[e] = (long long)(main ? v : v + 1);
                ev[e] = (long long)(main ? v + side + 1 : v + side);
                w[e] = 1.0;
            }
        }
    }
}

__global__ void k_ratings(unsigned long long m, const long long *eu, const long long *ev, const double *w,
                          const double *c, double *r) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const double we = w[e];
        r[e] = (we * we) / (c[eu[e]] * c[ev[e]]);
    }
}

__global__ void k_rep_flags(unsigned long long n, const long long *mate, unsigned long long *flag) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += stride) {
        if (v == n) {
            flag[v] = 0;
            continue;
        }
        const long long mv = mate[v];
        flag[v] = (mv < 0 || (long long)v < mv) ? 1ULL : 0ULL;
    }
}

__global__ void k_cid(unsigned long long n, const long long *mate, const unsigned long long *scan, long long *cid,
                      const double *c, double *cc) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const long long mv = mate[v];
        const unsigned long long rep = (mv < 0 || (long long)v < mv) ? v : (unsigned long long)mv;
        const long long id = (long long)scan[rep];
        cid[v] = id;
        atomicAdd(cc + id, c[v]);   // integer-valued sums: exact in any order
    }
}

__global__ void k_coarse_keys(unsigned long long m, const long long *eu, const long long *ev, const long long *cid,
                              unsigned long long *key, unsigned long long sentinel) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
        const unsigned long long a = (unsigned long long)cid[eu[e]], b = (unsigned long long)cid[ev[e]];
        key[e] = (a == b) ? sentinel : ((a < b ? a : b) << 32 | (a < b ? b : a));
    }
}

__global__ void k_split_keys(unsigned long long k, const unsigned long long *key, long long *eu, long long *ev) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        eu[i] = (long long)(key[i] >> 32);
        ev[i] = (long long)(key[i] & 0xFFFFFFFFULL);
    }
}

}  // namespace lmx

static int cgrid(lmx_ctx *ctx, unsigned long long work) {
    unsigned long long b = (work + kBlock - 1) / kBlock;
    return (int)std::max<unsigned long long>(1, std::min<unsigned long long>(b, (unsigned long long)ctx->num_sms * 16));
}

extern "C" {

int lmx_mesh_edges(lmx_ctx *ctx, int64_t side, uint64_t seed, int64_t *eu, int64_t *ev, double *w,
                   int64_t *m_out) {
    if (!ctx || side < 2 || side > 65535) return lmx_fail(ctx, LMX_EINVAL, "mesh side must be in [2, 65535]");
    cudaSetDevice(ctx->device);
    const unsigned long long s = (unsigned long long)side;
    const unsigned long long m = (s - 1) * (3 * s - 1);
    k_mesh<<<cgrid(ctx, s * s), kBlock, 0, ctx->stream>>>(s, mix64(seed ^ kMeshTag), (long long *)eu,
                                                         (long long *)ev, w);
    LMX_CUDA(ctx, cudaGetLastError());
    LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    *m_out = (int64_t)m;
    return LMX_OK;
}

int lmx_ratings(lmx_ctx *ctx, int64_t m, const int64_t *eu, const int64_t *ev, const double *w, const double *c,
                double *r) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (m > 0)
        k_ratings<<<cgrid(ctx, (unsigned long long)m), kBlock, 0, ctx->stream>>>(
            (unsigned long long)m, (const long long *)eu, (const long long *)ev, w, c, r);
    LMX_CUDA(ctx, cudaGetLastError());
    LMX_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
    return LMX_OK;
}

int lmx_contract(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *eu, const int64_t *ev, const double *w,
                 const double *c, const int64_t *mate, int64_t *cid, int64_t *n_out, int64_t *m_out, int64_t *ceu,
                 int64_t *cev, double *cw, double *cc) {
    if (!ctx || n < 0 || m < 0) return LMX_EINVAL;
    if (n >= (int64_t)0xFFFFFFFFLL) return lmx_fail(ctx, LMX_ELIMIT, "n exceeds 32-bit ids");
    cudaSetDevice(ctx->device);
    cudaStream_t st = ctx->stream;
    const unsigned long long N = (unsigned long long)n, M = (unsigned long long)m;
    unsigned long long *flag = nullptr, *key = nullptr, *key2 = nullptr, *ukey = nullptr, *nu = nullptr;
    double *w2 = nullptr;
    void *tmp = nullptr;
    size_t tmp_bytes = 0;
    int rc = LMX_OK;
    cudaError_t e = cudaSuccess;
    do {
        if ((e = lmx_dmalloc(ctx, (void **)&flag, (N + 1) * 8)) != cudaSuccess) break;
        if ((e = lmx_dmalloc(ctx, (void **)&key, std::max<unsigned long long>(M, 1) * 8)) != cudaSuccess) break;
        if ((e = lmx_dmalloc(ctx, (void **)&key2, std::max<unsigned long long>(M, 1) * 8)) != cudaSuccess) break;
        if ((e = lmx_dmalloc(ctx, (void **)&ukey, std::max<unsigned long long>(M, 1) * 8)) != cudaSuccess) break;
        if ((e = lmx_dmalloc(ctx, (void **)&w2, std::max<unsigned long long>(M, 1) * 8)) != cudaSuccess) break;
        if ((e = lmx_dmalloc(ctx, (void **)&nu, 8)) != cudaSuccess) break;
        // coarse ids
        k_rep_flags<<<cgrid(ctx, N + 1), kBlock, 0, st>>>(N, (const long long *)mate, flag);
        size_t t1 = 0, t2 = 0, t3 = 0;
        e = cub::DeviceScan::ExclusiveSum(nullptr, t1, flag, flag, (long long)(N + 1), st);
        if (e == cudaSuccess)
            e = cub::DeviceRadixSort::SortPairs(nullptr, t2, key, key2, w, w2, (long long)M, 0, 64, st);
        if (e == cudaSuccess)
            e = cub::DeviceReduce::ReduceByKey(nullptr, t3, key2, ukey, w2, cw, nu, cuda::std::plus<double>(),
                                               (long long)M, st);
        if (e != cudaSuccess) break;
        tmp_bytes = std::max(t1, std::max(t2, t3));
        if ((e = lmx_dmalloc(ctx, (void **)&tmp, tmp_bytes)) != cudaSuccess) break;
        e = cub::DeviceScan::ExclusiveSum(tmp, t1, flag, flag, (long long)(N + 1), st);
        if (e != cudaSuccess) break;
        unsigned long long nc = 0;
        if ((e = cudaMemcpyAsync(&nc, flag + N, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaMemsetAsync(cc, 0, std::max<unsigned long long>(N, 1) * 8, st)) != cudaSuccess) break;
        k_cid<<<cgrid(ctx, N), kBlock, 0, st>>>(N, (const long long *)mate, flag, (long long *)cid, c, cc);
        // coarse edges: sort pair keys (self loops -> sentinel, sorted last), sum runs
        const unsigned long long sentinel = ~0ULL;
        k_coarse_keys<<<cgrid(ctx, M), kBlock, 0, st>>>(M, (const long long *)eu, (const long long *)ev,
                                                       (const long long *)cid, key, sentinel);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        size_t tb = tmp_bytes;
        e = cub::DeviceRadixSort::SortPairs(tmp, tb, key, key2, w, w2, (long long)M, 0, 64, st);
        if (e != cudaSuccess) break;
        tb = tmp_bytes;
        e = cub::DeviceReduce::ReduceByKey(tmp, tb, key2, ukey, w2, cw, nu, cuda::std::plus<double>(),
                                           (long long)M, st);
        if (e != cudaSuccess) break;
        unsigned long long nk = 0;
        if ((e = cudaMemcpyAsync(&nk, nu, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        // drop the sentinel run (self loops) if present
        unsigned long long last = 0;
        if (nk > 0) {
            if ((e = cudaMemcpy(&last, ukey + nk - 1, 8, cudaMemcpyDeviceToHost)) != cudaSuccess) break;
            if (last == sentinel) --nk;
        }
        k_split_keys<<<cgrid(ctx, nk), kBlock, 0, st>>>(nk, ukey, (long long *)ceu, (long long *)cev);
        if ((e = cudaGetLastError()) != cudaSuccess) break;
        if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
        *n_out = (int64_t)nc;
        *m_out = (int64_t)nk;
    } while (0);
    lmx_dfree(ctx, flag);
    lmx_dfree(ctx, key);
    lmx_dfree(ctx, key2);
    lmx_dfree(ctx, ukey);
    lmx_dfree(ctx, w2);
    lmx_dfree(ctx, nu);
    lmx_dfree(ctx, tmp);
    if (e != cudaSuccess) rc = lmx_cuda_check(ctx, e, "lmx_contract");
    return rc;
}

}  // extern "C"
