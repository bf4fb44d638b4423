// lmx_validate.cu -- validate_matching (graph.py:212-237) and Matching.weight
// (graph.py:54-56, 191-192) on the device, against the loaded graph.
//
// Validation: one pass over the matched edges (range, vertex reuse through a
// per-vertex count, mate consistency), one over the vertices (a mate entry
// without a matched edge), one over all edges (an edge with both ends free:
// not maximal).  The first offence of each kind is recorded by the smallest
// id, so the verdict and the detail are deterministic (the reference's detail
// follows frozenset iteration order).
//
// Weight: edge_weight[sorted ids].sum() in numpy is a pairwise summation with
// a fixed shape (numpy's pairwise_sum: runs < 8 summed in order, blocks of
// <= 128 with 8 interleaved accumulators, longer runs split at n/2 rounded
// down to a multiple of 8).  The leaves are summed on the device exactly as
// numpy does, and the host combines them in the same recursion, so the weight
// is bit-identical to the reference's.
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <vector>

#include "lmx_internal.cuh"

namespace lmx {

struct Offence {            // smallest offending id per kind (~0 = none)
    unsigned long long range_edge;
    unsigned long long shared_vertex;
    unsigned long long mate_edge;
    unsigned long long stray_vertex;
    unsigned long long free_edge;
};

__global__ void k_val_edges(const long long *ids, unsigned long long k, unsigned long long m, const uint32_t *eu,
                            const uint32_t *ev, const long long *mate, uint32_t *cnt, Offence *off) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
        const long long e = ids[i];
        if (e < 0 || (unsigned long long)e >= m) {
            atomicMin(&off->range_edge, (unsigned long long)i);   // position: the id itself may be negative
            continue;
        }
        const uint32_t u = eu[e], v = ev[e];
        atomicAdd(cnt + u, 1u);
        atomicAdd(cnt + v, 1u);
        if (mate[u] != (long long)v || mate[v] != (long long)u) atomicMin(&off->mate_edge, (unsigned long long)e);
    }
}

__global__ void k_val_vertices(const uint32_t *cnt, const long long *mate, unsigned long long n, Offence *off) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long v = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
        const uint32_t c = cnt[v];
        if (c > 1) atomicMin(&off->shared_vertex, v);
        if (c == 0 && mate[v] != -1) atomicMin(&off->stray_vertex, v);
    }
}

__global__ void k_val_maximal(const uint32_t *eu, const uint32_t *ev, unsigned long long m, const long long *mate,
                              Offence *off) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long e = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride)
        if (mate[eu[e]] == -1 && mate[ev[e]] == -1) atomicMin(&off->free_edge, e);
}

// numpy pairwise_sum leaf (n <= 128) over w[ids[lo .. lo + n)]
__global__ void k_weight_leaves(const long long *ids, const double *w, const unsigned long long *leaf_lo,
                                const uint32_t *leaf_n, unsigned long long nleaves, double *out) {
    const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
    for (unsigned long long L = (unsigned long long)blockIdx.x * blockDim.x + threadIdx.x; L < nleaves;
         L += stride) {
        const unsigned long long lo = leaf_lo[L];
        const uint32_t n = leaf_n[L];
        double res;
        if (n < 8) {
            res = 0.0;
            for (uint32_t i = 0; i < n; ++i) res += w[ids[lo + i]];
        } else {
            double r[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) r[j] = w[ids[lo + j]];
            uint32_t i = 8;
            for (; i < n - (n % 8); i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] += w[ids[lo + i + j]];
            }
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
            for (; i < n; ++i) res += w[ids[lo + i]];
        }
        out[L] = res;
    }
}

}  // namespace lmx

using namespace lmx;

// numpy's pairwise_sum recursion: leaves in order, then the same combination
static void pw_leaves(unsigned long long lo, unsigned long long n, std::vector<unsigned long long> &los,
                      std::vector<uint32_t> &ns) {
    if (n <= 128) {
        los.push_back(lo);
        ns.push_back((uint32_t)n);
        return;
    }
    unsigned long long n2 = n / 2;
    n2 -= n2 % 8;
    pw_leaves(lo, n2, los, ns);
    pw_leaves(lo + n2, n - n2, los, ns);
}

static double pw_combine(unsigned long long n, const std::vector<double> &leaf, size_t &next) {
    if (n <= 128) return leaf[next++];
    unsigned long long n2 = n / 2;
    n2 -= n2 % 8;
    const double a = pw_combine(n2, leaf, next);
    const double b = pw_combine(n - n2, leaf, next);
    return a + b;
}

int lmx_validate_impl(lmx_ctx *ctx, const int64_t *mate, const int64_t *ids, int64_t n_ids, int where,
                      int *valid, int *maximal, double *weight, char *detail, size_t detail_len) {
    const unsigned long long n = (unsigned long long)ctx->n, m = (unsigned long long)ctx->m;
    const unsigned long long k = (unsigned long long)std::max<int64_t>(n_ids, 0);
    cudaStream_t st = ctx->stream;
    const int grid = ctx->num_sms * 8;
    const long long *dmate = (const long long *)mate, *dids = (const long long *)ids;
    long long *tmate = nullptr, *tids = nullptr;
    uint32_t *cnt = nullptr;
    Offence *off = nullptr;
    unsigned long long *leaf_lo = nullptr;
    uint32_t *leaf_n = nullptr;
    double *leaf_sum = nullptr;
    std::vector<unsigned long long> los;
    std::vector<uint32_t> ns;
    if (k) pw_leaves(0, k, los, ns);
    const size_t nl = los.size();
    int rc = LMX_OK;
    Offence h;
    std::vector<double> sums(nl);
    do {
        if (where == LMX_HOST) {
            if ((rc = lmx_alloc(ctx, (void **)&tmate, std::max<unsigned long long>(n, 1) * 8, "mate copy")) != LMX_OK)
                break;
            if ((rc = lmx_alloc(ctx, (void **)&tids, std::max<unsigned long long>(k, 1) * 8, "ids copy")) != LMX_OK)
                break;
            cudaError_t e = n ? cudaMemcpyAsync(tmate, mate, n * 8, cudaMemcpyHostToDevice, st) : cudaSuccess;
            if (e == cudaSuccess && k) e = cudaMemcpyAsync(tids, ids, k * 8, cudaMemcpyHostToDevice, st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "validate inputs"); break; }
            dmate = tmate;
            dids = tids;
        }
        if ((rc = lmx_alloc(ctx, (void **)&cnt, std::max<unsigned long long>(n, 1) * 4, "vertex counts")) != LMX_OK)
            break;
        if ((rc = lmx_alloc(ctx, (void **)&off, sizeof(Offence), "offences")) != LMX_OK) break;
        cudaError_t e = cudaMemsetAsync(cnt, 0, std::max<unsigned long long>(n, 1) * 4, st);
        if (e == cudaSuccess) e = cudaMemsetAsync(off, 0xFF, sizeof(Offence), st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "validate init"); break; }
        if (k) k_val_edges<<<grid, kBlock, 0, st>>>(dids, k, m, ctx->eu, ctx->ev, dmate, cnt, off);
        if (n) k_val_vertices<<<grid, kBlock, 0, st>>>(cnt, dmate, n, off);
        if (m) k_val_maximal<<<grid, kBlock, 0, st>>>(ctx->eu, ctx->ev, m, dmate, off);
        e = cudaGetLastError();
        if (e == cudaSuccess) e = cudaMemcpyAsync(&h, off, sizeof(Offence), cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "validate"); break; }
        // weight (only meaningful when every id is in range)
        if (nl && h.range_edge == ~0ULL) {
            if ((rc = lmx_alloc(ctx, (void **)&leaf_lo, nl * 8, "weight leaves")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&leaf_n, nl * 4, "weight leaves")) != LMX_OK) break;
            if ((rc = lmx_alloc(ctx, (void **)&leaf_sum, nl * 8, "weight leaves")) != LMX_OK) break;
            e = cudaMemcpyAsync(leaf_lo, los.data(), nl * 8, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) e = cudaMemcpyAsync(leaf_n, ns.data(), nl * 4, cudaMemcpyHostToDevice, st);
            if (e == cudaSuccess) {
                k_weight_leaves<<<grid, kBlock, 0, st>>>(dids, ctx->w, leaf_lo, leaf_n, nl, leaf_sum);
                e = cudaGetLastError();
            }
            if (e == cudaSuccess) e = cudaMemcpyAsync(sums.data(), leaf_sum, nl * 8, cudaMemcpyDeviceToHost, st);
            if (e == cudaSuccess) e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "weight"); break; }
        }
    } while (0);
    cudaStreamSynchronize(st);
    lmx_free(ctx, (void **)&tmate, std::max<unsigned long long>(n, 1) * 8);
    lmx_free(ctx, (void **)&tids, std::max<unsigned long long>(k, 1) * 8);
    lmx_free(ctx, (void **)&cnt, std::max<unsigned long long>(n, 1) * 4);
    lmx_free(ctx, (void **)&off, sizeof(Offence));
    lmx_free(ctx, (void **)&leaf_lo, nl * 8);
    lmx_free(ctx, (void **)&leaf_n, nl * 4);
    lmx_free(ctx, (void **)&leaf_sum, nl * 8);
    if (rc != LMX_OK) return rc;

    char buf[160] = "";
    bool ok = true;
    if (h.range_edge != ~0ULL) {
        snprintf(buf, sizeof buf, "edge id at position %llu out of range", h.range_edge);
        ok = false;
    } else if (h.shared_vertex != ~0ULL) {
        snprintf(buf, sizeof buf, "vertex shared by two matched edges (vertex %llu)", h.shared_vertex);
        ok = false;
    } else if (h.mate_edge != ~0ULL) {
        snprintf(buf, sizeof buf, "mate table disagrees with matched edge %llu", h.mate_edge);
        ok = false;
    } else if (h.stray_vertex != ~0ULL) {
        snprintf(buf, sizeof buf, "mate entry set for an unmatched vertex");
        ok = false;
    }
    if (valid) *valid = ok ? 1 : 0;
    if (maximal) *maximal = (ok && h.free_edge == ~0ULL) ? 1 : 0;
    if (weight) {
        size_t next = 0;
        *weight = (k && h.range_edge == ~0ULL) ? pw_combine(k, sums, next) : 0.0;
    }
    if (detail && detail_len) {
        strncpy(detail, buf, detail_len - 1);
        detail[detail_len - 1] = '\0';
    }
    return LMX_OK;
}
