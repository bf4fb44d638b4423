// lmx_capi.cu -- the extern "C" boundary declared in include/lmx.h.
#include <cstdio>
#include <cstring>
#include <vector>

#include "lmx_internal.cuh"

namespace {
thread_local std::string g_create_err;
}  // namespace

extern "C" {

int lmx_abi_version(void) { return LMX_ABI_VERSION; }

int lmx_create(int device, lmx_ctx **out) {
    if (!out) return LMX_EINVAL;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        g_create_err = std::string("no CUDA device available: ") + cudaGetErrorString(e);
        cudaGetLastError();
        return LMX_ECUDA;
    }
    if (device < 0 || device >= count) {
        g_create_err = "device index out of range";
        return LMX_EINVAL;
    }
    lmx_ctx *ctx = new lmx_ctx();
    ctx->device = device;
    int rc = LMX_OK;
    do {
        if ((e = cudaSetDevice(device)) != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "cudaSetDevice"); break; }
        cudaDeviceProp prop;
        if ((e = cudaGetDeviceProperties(&prop, device)) != cudaSuccess) { rc = lmx_cuda_check(ctx, e, "props"); break; }
        if (prop.major != 10) {
            rc = lmx_fail(ctx, LMX_ECUDA, std::string("liblmx is built for sm_100a (B200); device is ") + prop.name);
            break;
        }
        ctx->num_sms = prop.multiProcessorCount;
        if ((e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking)) != cudaSuccess) {
            rc = lmx_cuda_check(ctx, e, "stream");
            break;
        }
        ctx->own_stream = true;
        if ((e = cudaEventCreate(&ctx->ev0)) != cudaSuccess || (e = cudaEventCreate(&ctx->ev1)) != cudaSuccess ||
            (e = cudaEventCreate(&ctx->ev2)) != cudaSuccess) {
            rc = lmx_cuda_check(ctx, e, "events");
            break;
        }
        rc = lmx_configure_grids(ctx);
        if (rc == LMX_OK) rc = lmx_scan_configure_grids(ctx);
    } while (0);
    if (rc != LMX_OK) {
        g_create_err = ctx->err;
        lmx_destroy(ctx);
        return rc;
    }
    *out = ctx;
    return LMX_OK;
}

void lmx_destroy(lmx_ctx *ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    lmx_free_graph(ctx);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    lmx_flush_cache(ctx);
    for (auto &kv : ctx->live) cudaFree(kv.first);   // anything still outstanding
    ctx->live.clear();
    if (ctx->ctr) cudaFree(ctx->ctr);
    if (ctx->ctr_host) cudaFreeHost(ctx->ctr_host);
    if (ctx->loop_aux) cudaFree(ctx->loop_aux);
    if (ctx->loop_host) cudaFreeHost(ctx->loop_host);
    if (ctx->ev0) cudaEventDestroy(ctx->ev0);
    if (ctx->ev1) cudaEventDestroy(ctx->ev1);
    if (ctx->ev2) cudaEventDestroy(ctx->ev2);
    for (cudaEvent_t e : ctx->tl_events) cudaEventDestroy(e);
    for (cudaEvent_t e : ctx->ev_copy)
        if (e) cudaEventDestroy(e);
    if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
    for (cudaEvent_t e : ctx->stage_ev) cudaEventDestroy(e);
    if (ctx->ev_deg) cudaEventDestroy(ctx->ev_deg);
    if (ctx->deg_stream) cudaStreamDestroy(ctx->deg_stream);
    if (ctx->ev_load) cudaEventDestroy(ctx->ev_load);
    if (ctx->ev_side) cudaEventDestroy(ctx->ev_side);
    if (ctx->ev_mate) cudaEventDestroy(ctx->ev_mate);
    if (ctx->side_stream) cudaStreamDestroy(ctx->side_stream);
    if (ctx->load_stream) cudaStreamDestroy(ctx->load_stream);
    if (ctx->stage_host) cudaFreeHost(ctx->stage_host);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
}

const char *lmx_last_error(const lmx_ctx *ctx) {
    if (!ctx) return g_create_err.c_str();
    return ctx->err.c_str();
}

int lmx_set_stream(lmx_ctx *ctx, void *cuda_stream) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (ctx->stream) cudaStreamSynchronize(ctx->stream);
    if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
    if (cuda_stream) {
        ctx->stream = (cudaStream_t)cuda_stream;
        ctx->own_stream = false;
    } else {
        cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
        if (e != cudaSuccess) return lmx_cuda_check(ctx, e, "stream");
        ctx->own_stream = true;
    }
    return LMX_OK;
}

int lmx_load_graph(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                   const double *edge_weight, int where) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev0, ctx->stream));
    // The load runs on the engine's own non-blocking stream, ordered after the
    // caller's prior work and before its later work: a caller stream that is
    // the legacy default stream would otherwise serialise against the copy
    // and degree streams of a host load.
    if (!ctx->load_stream) {
        LMX_CUDA(ctx, cudaStreamCreateWithFlags(&ctx->load_stream, cudaStreamNonBlocking));
        LMX_CUDA(ctx, cudaEventCreateWithFlags(&ctx->ev_load, cudaEventDisableTiming));
    }
    cudaStream_t user = ctx->stream;
    LMX_CUDA(ctx, cudaStreamWaitEvent(ctx->load_stream, ctx->ev0, 0));
    ctx->stream = ctx->load_stream;
    int rc = lmx_load_edges(ctx, n, m, edge_u, edge_v, edge_weight, where);
    cudaError_t e = cudaEventRecord(ctx->ev_load, ctx->load_stream);
    ctx->stream = user;
    if (e == cudaSuccess) e = cudaStreamWaitEvent(user, ctx->ev_load, 0);
    if (rc != LMX_OK) return rc;
    LMX_CUDA(ctx, e);
    LMX_CUDA(ctx, cudaEventRecord(ctx->ev1, ctx->stream));
    LMX_CUDA(ctx, cudaEventSynchronize(ctx->ev1));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    ctx->timing.setup_ms = ms;
    return LMX_OK;
}

int lmx_match(lmx_ctx *ctx, uint64_t seed_masked, int rerandomize, int64_t *mate_out,
              int64_t *matched_ids_out, int64_t *n_matched_out, lmx_round_stats *rounds_out,
              int max_rounds, int *n_rounds_out, int out_where) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (!ctx->vbeg) return lmx_fail(ctx, LMX_ESTATE, "no graph loaded (call lmx_load_graph first)");
    std::vector<lmx_round_stats> &stats = ctx->rounds;
    unsigned long long nm = 0;
    if (ctx->static_layout && (rerandomize || lmx::round_seed(seed_masked, 0, false) != ctx->static_rs)) {
        return lmx_fail(ctx, LMX_ESTATE, "the loaded graph is laid out for the fixed salt order of one seed "
                                         "(LMX_OPT_STATIC_ORDER): it matches only that seed with rerandomize=0; "
                                         "reload for this call");
    }
    ctx->mate_target = (out_where == LMX_DEVICE && mate_out) ? (long long *)mate_out : ctx->mate;
    // a page-locked host mate buffer can take the mate array while the
    // histogram and the id emission still run (scan loop)
    ctx->mate_early = nullptr;
    ctx->mate_early_done = false;
    if (out_where == LMX_HOST && mate_out && ctx->n > 0) {
        cudaPointerAttributes at;
        if (cudaPointerGetAttributes(&at, mate_out) == cudaSuccess && at.type == cudaMemoryTypeHost)
            ctx->mate_early = mate_out;
        cudaGetLastError();
    }
    if (ctx->algo == 1) LMX_TRY(lmx_run_rounds_scan(ctx, seed_masked, rerandomize != 0, stats, nm));
    else LMX_TRY(lmx_run_rounds(ctx, seed_masked, rerandomize != 0, stats, nm));
    LMX_TRY(lmx_emit_outputs(ctx, nm, mate_out, matched_ids_out, out_where));
    if (n_matched_out) *n_matched_out = (int64_t)nm;
    if (n_rounds_out) *n_rounds_out = (int)stats.size();
    if (rounds_out)
        for (int i = 0; i < (int)stats.size() && i < max_rounds; ++i) rounds_out[i] = stats[i];
    if (rounds_out && (int)stats.size() > max_rounds) {
        // mate / ids / counts are complete; *n_rounds_out holds the size needed
        char buf[200];
        snprintf(buf, sizeof buf,
                 "rounds_out holds %d of %d rounds (outputs complete); fetch the trace with lmx_last_rounds "
                 "or call again with max_rounds >= %d",
                 max_rounds, (int)stats.size(), (int)stats.size());
        return lmx_fail(ctx, LMX_ELIMIT, buf);
    }
    return LMX_OK;
}

int lmx_last_rounds(lmx_ctx *ctx, lmx_round_stats *out, int cap) {
    if (!ctx) return -1;
    std::vector<lmx_round_stats> &stats = ctx->rounds;
    for (int i = 0; i < (int)stats.size() && i < cap; ++i) out[i] = stats[i];
    return (int)stats.size();
}

int lmx_set_option(lmx_ctx *ctx, int option, int64_t value) {
    if (!ctx) return LMX_EINVAL;
    if (option == LMX_OPT_KERNEL_TIMING) {
        ctx->kernel_timing = value != 0;
        return LMX_OK;
    }
    if (option == LMX_OPT_LAYOUT) {
        if (value < -1 || value > 2) return lmx_fail(ctx, LMX_EINVAL, "layout must be -1, 0, 1 or 2");
        ctx->force_layout = (int)value;
        return LMX_OK;
    }
    if (option == LMX_OPT_RELABEL) {
        if (value < -1 || value > 2) return lmx_fail(ctx, LMX_EINVAL, "relabel must be -1, 0, 1 or 2");
        ctx->force_relabel = (int)value;
        return LMX_OK;
    }
    if (option == LMX_OPT_DIST_P) {
        if (value < 1 || value > 64) return lmx_fail(ctx, LMX_EINVAL, "dist p must be in [1, 64]");
        ctx->dist_p = (int)value;
        ctx->dist_requested = true;
        return LMX_OK;
    }
    if (option == LMX_OPT_ALGO) {
        if (value < -1 || value > 1) return lmx_fail(ctx, LMX_EINVAL, "algo must be -1, 0 or 1");
        ctx->force_algo = (int)value;
        return LMX_OK;
    }
    if (option == LMX_OPT_DIST_RANK) {
        if (value < 0 || value >= ctx->dist_p) return lmx_fail(ctx, LMX_EINVAL, "dist rank out of range");
        ctx->dist_rank = (int)value;
        return LMX_OK;
    }
    if (option == LMX_OPT_STATIC_ORDER) {
        if (value < 0 || value > 1) return lmx_fail(ctx, LMX_EINVAL, "static order must be 0 or 1");
        ctx->static_order = value != 0;
        return LMX_OK;
    }
    if (option == LMX_OPT_STATIC_SEED) {
        ctx->static_seed = (uint64_t)value;
        return LMX_OK;
    }
    if (option == LMX_QUERY_STATIC) return ctx->static_layout ? 1 : 0;
    if (option == LMX_QUERY_LAYOUT) return ctx->layout;
    if (option == LMX_QUERY_RELABELED) return ctx->relabeled ? 1 : 0;
    if (option == LMX_QUERY_ALGO) return ctx->algo;
    if (option == LMX_QUERY_PEAK_BYTES) {   // in MiB (the return is an int); value != 0 resets the mark
        const int r = (int)(ctx->peak_bytes >> 20);
        if (value) ctx->peak_bytes = ctx->dev_bytes;
        return r;
    }
    return lmx_fail(ctx, LMX_EINVAL, "unknown option");
}

int lmx_last_timing(const lmx_ctx *ctx, lmx_timing *out) {
    if (!ctx || !out) return LMX_EINVAL;
    *out = ctx->timing;
    return LMX_OK;
}

int lmx_last_kernel_times(const lmx_ctx *ctx, float *out, int cap) {
    if (!ctx) return -1;
    const int k = (int)ctx->kernel_ms.size();
    for (int i = 0; i < k && i < cap && out; ++i) out[i] = ctx->kernel_ms[i];
    return k;
}

int lmx_last_round_counters(const lmx_ctx *ctx, int64_t *out, int cap_rounds) {
    if (!ctx) return -1;
    const int k = (int)ctx->timing.rounds_executed;
    for (int i = 0; i < k && i < cap_rounds && out && ctx->ctr_host; ++i) {
        const lmx::RoundCtr &c = ctx->ctr_host[i];
        int64_t *o = out + 8 * i;
        o[0] = (int64_t)c.slot_reads;
        o[1] = (int64_t)c.live_slots;
        o[2] = (int64_t)c.matched_v;
        // scan loop: |A_r| (vertices probed), slow-path probes; compact: bucket sizes 0..4
        // (live degree <= 4, 17..32 + 5..16 (buckets 1 and 5 together), 33..1024, block, hub)
        if (ctx->algo == 1) {
            o[3] = c.pad[0];
            o[4] = c.n[0];
            o[5] = o[6] = o[7] = 0;
        } else {
            for (int q = 0; q < 5; ++q) o[3 + q] = c.n[q];
            o[4] += c.n[5];
        }
    }
    return k;
}

int lmx_local_max(int device, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                  const double *edge_weight, uint64_t seed_masked, int rerandomize, int64_t *mate_out,
                  int64_t *matched_ids_out, int64_t *n_matched_out, lmx_round_stats *rounds_out,
                  int max_rounds, int *n_rounds_out, char *err, size_t errlen) {
    lmx_ctx *ctx = nullptr;
    int rc = lmx_create(device, &ctx);
    if (rc == LMX_OK && !rerandomize) {   // one seed, fixed salts: the static order serves tied weights
        ctx->static_order = true;
        ctx->static_seed = seed_masked;
    }
    if (rc == LMX_OK) ctx->force_relabel = 2;   // one matching per load (LMX_OPT_RELABEL)
    if (rc == LMX_OK) rc = lmx_load_graph(ctx, n, m, edge_u, edge_v, edge_weight, LMX_HOST);
    if (rc == LMX_OK)
        rc = lmx_match(ctx, seed_masked, rerandomize, mate_out, matched_ids_out, n_matched_out, rounds_out,
                       max_rounds, n_rounds_out, LMX_HOST);
    if (rc != LMX_OK && err && errlen) {
        const char *msg = lmx_last_error(ctx);
        std::strncpy(err, msg, errlen - 1);
        err[errlen - 1] = 0;
    }
    lmx_destroy(ctx);
    return rc;
}

// ---- 1D-partitioned (multi-GPU) stepped protocol ---------------------------

int lmx_dist_bounds(const lmx_ctx *ctx, int64_t *bounds_out) {
    if (!ctx || !bounds_out) return LMX_EINVAL;
    for (size_t i = 0; i < ctx->bounds.size(); ++i) bounds_out[i] = ctx->bounds[i];
    return LMX_OK;
}

int lmx_dist_begin(lmx_ctx *ctx, uint64_t seed_masked, int rerandomize) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (!ctx->vbeg) return lmx_fail(ctx, LMX_ESTATE, "no graph loaded");
    return lmx_dist_begin_impl(ctx, seed_masked, rerandomize != 0);
}

int lmx_dist_mround(lmx_ctx *ctx, void **mround_dev) {
    if (!ctx || !mround_dev) return LMX_EINVAL;
    if (!ctx->mround) return lmx_fail(ctx, LMX_ESTATE, "no match rounds (load with LMX_OPT_DIST_P)");
    *mround_dev = ctx->mround;
    return LMX_OK;
}

int lmx_dist_hist(lmx_ctx *ctx, int n_rounds, void **hist_dev, int *nbins) {
    if (!ctx || !hist_dev || !nbins) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (ctx->algo != 1) return lmx_fail(ctx, LMX_ESTATE, "the compacting round loop counts edges per round");
    return lmx_scan_dist_hist(ctx, n_rounds, hist_dev, nbins);
}

int lmx_dist_round(lmx_ctx *ctx) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    return lmx_dist_round_impl(ctx);
}

int lmx_dist_propose(lmx_ctx *ctx, void **counts_dev_out, void **send_dev_out) {
    if (!ctx || !counts_dev_out || !send_dev_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    return lmx_dist_propose_impl(ctx, counts_dev_out, send_dev_out);
}

int lmx_dist_recv_buffer(lmx_ctx *ctx, int64_t count, void **recv_out) {
    if (!ctx || !recv_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    return lmx_dist_recv_impl(ctx, count, recv_out);
}

int lmx_dist_accept(lmx_ctx *ctx, int64_t count) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    return lmx_dist_accept_impl(ctx, count);
}

int lmx_dist_pad(lmx_ctx *ctx, int64_t capacity, void **padded_dev_out, void **overflow_dev_out) {
    if (!ctx || !padded_dev_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    if (ctx->algo != 1) return lmx_fail(ctx, LMX_ESTATE, "fixed-capacity exchange: scan loop partitions only");
    return lmx_scan_dist_pad(ctx, capacity, padded_dev_out, overflow_dev_out);
}

int lmx_dist_list_size(lmx_ctx *ctx, void **size_dev_out) {
    if (!ctx || !size_dev_out) return LMX_EINVAL;
    if (ctx->algo != 1) return lmx_fail(ctx, LMX_ESTATE, "list size: scan loop partitions only");
    if (!ctx->ctr) return lmx_fail(ctx, LMX_ESTATE, "lmx_dist_begin first");
    *size_dev_out = &ctx->ctr[ctx->dist_round].pad[0];
    return LMX_OK;
}

int lmx_dist_match(lmx_ctx *ctx, void **stats_dev_out) {
    if (!ctx || !stats_dev_out) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    return lmx_dist_match_impl(ctx, stats_dev_out);
}

int lmx_dist_state(lmx_ctx *ctx, void **matched_bitmap, void **mate, void **edge_bits, void **stream) {
    if (!ctx) return LMX_EINVAL;
    if (matched_bitmap) *matched_bitmap = ctx->matched;
    if (mate) *mate = ctx->mate;
    if (edge_bits) *edge_bits = ctx->ebits;
    if (stream) *stream = ctx->stream;
    return LMX_OK;
}

int lmx_graph_size(const lmx_ctx *ctx, int64_t *n_out, int64_t *m_out) {
    if (!ctx) return LMX_EINVAL;
    if (n_out) *n_out = ctx->n;
    if (m_out) *m_out = ctx->m;
    return LMX_OK;
}

int64_t lmx_device_bytes(const lmx_ctx *ctx) { return ctx ? ctx->dev_bytes : 0; }

int lmx_rbm(lmx_ctx *ctx, uint64_t seed_masked, int64_t *mate_out, int64_t *matched_ids_out,
            int64_t *n_matched_out, lmx_round_stats *rounds_out, int max_rounds, int *n_rounds_out, int out_where) {
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (!ctx->vbeg) return lmx_fail(ctx, LMX_ESTATE, "no graph loaded (call lmx_load_graph first)");
    std::vector<lmx_round_stats> &stats = ctx->rounds;
    unsigned long long nm = 0;
    ctx->mate_target = (out_where == LMX_DEVICE && mate_out) ? (long long *)mate_out : ctx->mate;
    LMX_TRY(lmx_rbm_impl(ctx, seed_masked, max_rounds > 0 ? max_rounds : 10000, stats, nm));
    LMX_TRY(lmx_emit_outputs(ctx, nm, mate_out, matched_ids_out, out_where));
    if (n_matched_out) *n_matched_out = (int64_t)nm;
    if (n_rounds_out) *n_rounds_out = (int)stats.size();
    if (rounds_out)
        for (int i = 0; i < (int)stats.size() && i < max_rounds; ++i) rounds_out[i] = stats[i];
    return LMX_OK;
}

int lmx_validate(lmx_ctx *ctx, const int64_t *mate, const int64_t *ids, int64_t n_ids, int where,
                 int *valid, int *maximal, double *weight, char *detail, size_t detail_len) {
    if (ctx && ctx->dist_local) return lmx_fail(ctx, LMX_ESTATE, "validate needs the whole graph (not a partition)");
    if (!ctx) return LMX_EINVAL;
    cudaSetDevice(ctx->device);
    ctx->err.clear();
    if (!ctx->eu && ctx->m > 0) return lmx_fail(ctx, LMX_ESTATE, "no graph loaded");
    if (n_ids < 0 || (n_ids > 0 && !ids) || (ctx->n > 0 && !mate))
        return lmx_fail(ctx, LMX_EINVAL, "null or negative validate inputs");
    return lmx_validate_impl(ctx, mate, ids, n_ids, where, valid, maximal, weight, detail, detail_len);
}

}  // extern "C"

