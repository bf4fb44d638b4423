/*
 * lmx.h -- C ABI of the B200-native local max matching engine (liblmx.so).
 *
 * This is the drop-in boundary for the reference's matching entry point.
 * The reference is pure Python with no FFI, so each entry
 * point below names the reference function whose contract it takes over;
 * INTEGRATION.md shows the ctypes binding the reference would add.
 *
 *   lmx_local_max      <- locmax.matchers.local_max_seq(g, seed, rerandomize)
 *                         (/root/reference/pkg/src/locmax/matchers.py:61-122),
 *                         one-shot: host Graph arrays in, host Matching + trace out
 *   lmx_load_graph     <- the read-only Graph arrays local_max_seq consumes
 *                         (graph.py:20-34; only num_vertices, edge_u, edge_v,
 *                         edge_weight are read, matchers.py:80-92)
 *   lmx_match          <- local_max_seq's round loop (matchers.py:87-119) plus
 *                         matching_from_edge_ids (graph.py:195-203) and the
 *                         RoundStats trace (matchers.py:21-25,117)
 *   lmx_build_graph    <- locmax.graph.build_graph (graph.py:59-119) numbering
 *                         contract, on the device, for inputs too large for the
 *                         reference's Python dict loop
 *   lmx_gen_rmat       <- (new generator, SURVEY.md §8d C3/N★/C5; the reference
 *                         has none)
 *
 * Conventions: plain pointers and sizes; int status return (LMX_OK = 0);
 * the message of the last failure is available from lmx_last_error(ctx) or,
 * for the one-shot call, in the caller's err buffer.  Inputs are never
 * mutated (graph.py:117-118 ownership rule); outputs are caller-allocated.
 * Device pointers are CUDA device addresses valid in the ctx's device.
 */
#ifndef LMX_H
#define LMX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LMX_ABI_VERSION 1

/* status codes */
#define LMX_OK 0
#define LMX_EINVAL 1   /* domain error (bad ids, NaN/inf/negative weight): ValueError */
#define LMX_ECUDA 2    /* CUDA runtime / launch failure: RuntimeError */
#define LMX_ENOMEM 3   /* device allocation failed: MemoryError */
#define LMX_ELIMIT 4   /* instance exceeds the 32-bit vertex / edge id range */
#define LMX_ESTATE 5   /* call out of order (no graph loaded, ...) */

/* where a pointer lives */
#define LMX_HOST 0
#define LMX_DEVICE 1

typedef struct lmx_ctx lmx_ctx;

/* matchers.py:21-25 RoundStats */
typedef struct {
    int64_t edges_before;
    int64_t edges_matched;
    int64_t edges_removed;
} lmx_round_stats;

/* Per-call timing of the last lmx_match / lmx_load_graph (CUDA events). */
typedef struct {
    double setup_ms;        /* lmx_load_graph: H2D + slot-record build (K0) */
    double rounds_ms;       /* lmx_match: first round kernel .. last match kernel */
    double output_ms;       /* lmx_match: matched-id sort + output copies */
    int64_t round_launches; /* kernels launched by the round loop */
    int64_t slot_reads;     /* slots read by the round kernels (for roofline) */
    double round_kernel_ms; /* sum of round-kernel durations (LMX_OPT_KERNEL_TIMING) */
    double match_kernel_ms; /* sum of match-kernel durations (LMX_OPT_KERNEL_TIMING) */
    int64_t rounds_executed;/* rounds enqueued, incl. empty speculative ones */
    double hist_kernel_ms;  /* scan loop: death-round histogram (LMX_OPT_KERNEL_TIMING) */
} lmx_timing;

/* options for lmx_set_option */
#define LMX_OPT_KERNEL_TIMING 1 /* record a CUDA event after every round/match kernel */
#define LMX_OPT_LAYOUT 2        /* weight-key layout of the next load: -1 auto, 0 uniform
                                   (only valid if all weights are equal), 1 distinct, 2 general */
#define LMX_OPT_RELABEL 3       /* degree-descending vertex relabelling of the next load:
                                   -1 auto (skewed degree distributions), 0 off, 1 on,
                                   2 once: auto, except for the scan loop, for a load that
                                   serves ONE matching (relabelling costs the scan loop's
                                   load more than it saves one matching; lmx_local_max's
                                   choice) */
#define LMX_OPT_DIST_P 4        /* number of 1D vertex partitions of the next load (1 = single GPU) */
#define LMX_OPT_DIST_RANK 5     /* which partition this context owns (set after LMX_OPT_DIST_P) */
#define LMX_OPT_ALGO 6          /* round loop of the next load: -1 auto, 0 compacting rounds,
                                   1 weight-ordered scan (taken only for the distinct layout on a
                                   context without LMX_OPT_DIST_P; results are identical) */
#define LMX_OPT_STATIC_ORDER 7  /* rerandomize=False: 1 = the next load lays graphs with tied weights
                                   out in the fixed total order (weight, salt) of the seed given by
                                   LMX_OPT_STATIC_SEED (tiebreak.py:40-59: with rerandomize off every
                                   round's salts are round 0's), so the weight-ordered scan loop
                                   serves them; such a graph then only matches with that seed and
                                   rerandomize=0 (LMX_ESTATE otherwise).  0 = off (default) */
#define LMX_OPT_STATIC_SEED 8   /* the masked seed (uint64 bits as int64) for LMX_OPT_STATIC_ORDER */
#define LMX_QUERY_LAYOUT 100    /* lmx_set_option returns the loaded graph's layout */
#define LMX_QUERY_RELABELED 101 /* lmx_set_option returns 1 if the loaded graph is relabelled */
#define LMX_QUERY_ALGO 102      /* lmx_set_option returns the loaded graph's round loop (0 / 1) */
#define LMX_QUERY_STATIC 104    /* lmx_set_option returns 1 if the loaded graph has the static order */
#define LMX_QUERY_PEAK_BYTES 103 /* lmx_set_option returns the context's device-memory high-water mark
                                    in MiB (allocations through the context); value != 0 resets it */

int lmx_abi_version(void);

/* Create / destroy an engine bound to one CUDA device. */
int lmx_create(int device, lmx_ctx **out);
void lmx_destroy(lmx_ctx *ctx);
const char *lmx_last_error(const lmx_ctx *ctx);

/* Run all work on this stream (a cudaStream_t passed as void*); NULL = the
 * context's own non-blocking stream.  The legacy default stream (what
 * PyTorch's torch.cuda.default_stream().cuda_stream == 0 denotes) is passed as
 * cudaStreamLegacy, (void*)1. */
int lmx_set_stream(lmx_ctx *ctx, void *cuda_stream);

/*
 * Load (replace) the graph: n vertices, m edges in the reference's edge-array
 * form (edge ids are positions 0..m-1).  Validation follows graph.py:80-88:
 * ids in [0, n), no self loops, weights finite and >= 0 (-0.0 allowed).
 * Builds the per-vertex slot records on the device (K0).
 */
int lmx_load_graph(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u,
                   const int64_t *edge_v, const double *edge_weight, int where);

/*
 * Local max maximal matching of the loaded graph (matchers.py:61-122).
 * seed_masked = the Python seed & (2^64-1) (tiebreak.py:49).
 * mate_out: int64[n] (-1 = unmatched); matched_ids_out: int64[>= n/2],
 * ascending original edge ids; rounds_out: lmx_round_stats[max_rounds].
 * Outputs live where `out_where` says.  The loaded graph stays intact, so
 * lmx_match may be called repeatedly (e.g. different seeds).
 */
int lmx_match(lmx_ctx *ctx, uint64_t seed_masked, int rerandomize, int64_t *mate_out,
              int64_t *matched_ids_out, int64_t *n_matched_out, lmx_round_stats *rounds_out,
              int max_rounds, int *n_rounds_out, int out_where);

int lmx_last_timing(const lmx_ctx *ctx, lmx_timing *out);
int lmx_set_option(lmx_ctx *ctx, int option, int64_t value);

/* Copy the RoundStats trace of the last lmx_match (up to cap entries);
 * returns the number of rounds, or -1 on a bad ctx. */
int lmx_last_rounds(lmx_ctx *ctx, lmx_round_stats *out, int cap);

/* Diagnostics (LMX_OPT_KERNEL_TIMING on): per executed round of the last
 * lmx_match, the round-kernel and match-kernel durations in ms, interleaved
 * (out[2r], out[2r+1]); returns the number of floats available. */
int lmx_last_kernel_times(const lmx_ctx *ctx, float *out, int cap);

/* Diagnostics: per executed round of the last lmx_match, 8 counters
 * {slot reads, removal/live count, matched vertices, list sizes[5]}
 * (engine-specific meaning); returns the number of rounds. */
int lmx_last_round_counters(const lmx_ctx *ctx, int64_t *out, int cap_rounds);

/* One-shot host-buffer entry point: the local_max_seq drop-in for an FFI
 * binding.  err may be NULL.  If the matching takes more than max_rounds
 * rounds, mate / ids / n_matched are still complete, *n_rounds_out is the
 * round count and LMX_ELIMIT is returned: call again with a larger rounds_out
 * (INTEGRATION.md §2 does). */
int lmx_local_max(int device, int64_t n, int64_t m, const int64_t *edge_u,
                  const int64_t *edge_v, const double *edge_weight, uint64_t seed_masked,
                  int rerandomize, int64_t *mate_out, int64_t *matched_ids_out,
                  int64_t *n_matched_out, lmx_round_stats *rounds_out, int max_rounds,
                  int *n_rounds_out, char *err, size_t errlen);

/*
 * build_graph (graph.py:59-119) on the device.  Raw triples (u, v, w),
 * count k, already validated for range/weight domain by the caller or by
 * this call (returns LMX_EINVAL naming the first bad position).  Drops
 * self-loops; collapses parallel pairs to the heaviest occurrence (earliest on
 * ties) keeping that occurrence's orientation; numbers edges by first
 * occurrence of the pair.  num_vertices < 0 => max id + 1 over non-loop
 * edges.  The result becomes the context's loaded graph; lmx_graph_size and
 * lmx_graph_export read it back.
 */
int lmx_build_graph(lmx_ctx *ctx, int64_t k, const int64_t *u, const int64_t *v,
                    const double *w, int64_t num_vertices, int where);

/* Synthetic RMAT (Graph500 a,b,c; d = 1-a-b-c) with edge_factor * 2^scale raw
 * edges, U[0,1) weights from a counter-based hash of (seed, raw index), optional
 * bijective vertex relabelling, then build_graph semantics.  Loads the result. */
int lmx_gen_rmat(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c,
                 uint64_t seed, int permute);

/* G(n, m)-style random graph, the C1 family at scale (generate.py:48-89 idea;
 * BASELINE config C1 is n = 2^16, m = 4n, unit weights): edge_factor * 2^scale
 * uniform raw pairs (the RMAT generator with a = b = c = d = 1/4, no
 * relabelling), weights 1.0 if unit_weights else U[0,1), then build_graph
 * semantics.  Loads the result. */
int lmx_gen_er(lmx_ctx *ctx, int scale, int edge_factor, uint64_t seed, int unit_weights);

/* gen_rgg(x, seed, weight_mode) (generate.py:113-143, radius_edges_grid
 * :146-197, _morton_order :97-110) on the device, the identical edge list:
 * 2^x points from numpy's PCG64 whose initial 128-bit state and increment
 * (default_rng(seed).bit_generator.state) the caller passes in halves;
 * radius = rgg_threshold(n) (generate.py:92-94, computed by the caller);
 * weight_random 0: Euclidean distances, 1: the next rng.random(m) draws.
 * Loads the result. */
int lmx_gen_rgg(lmx_ctx *ctx, int x, uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                double radius, int weight_random);

/* Raw RMAT triples only (no build), for oracle parity of the generator. */
int lmx_gen_rmat_raw(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c,
                     uint64_t seed, int permute, int64_t *u_out, int64_t *v_out,
                     double *w_out, int out_where);

int lmx_graph_size(const lmx_ctx *ctx, int64_t *n_out, int64_t *m_out);

/* Copy the loaded graph's edge arrays out (graph.py Graph.edge_u/v/weight). */
int lmx_graph_export(lmx_ctx *ctx, int64_t *edge_u, int64_t *edge_v, double *edge_weight,
                     int out_where);

/*
 * 1D-partitioned local max (bsp_local_max, bsp.py:101-205).
 * With LMX_OPT_DIST_P = p and LMX_OPT_DIST_RANK = k set before the load, the
 * context owns the k-th of p contiguous vertex ranges with equal degree sums
 * (bsp.py:60-98, cuts rounded to 32 so ranks own whole bitmap words) and the
 * slots of all edges incident to it.  The host drives each round:
 *   lmx_dist_round      candidates of the owned vertices
 *   lmx_dist_propose    records {partner, edge id} for partners owned elsewhere,
 *                       grouped by destination rank (exchange A, barrier 1);
 *                       on the scan loop the round kernel already appended
 *                       them, and this call only packs them (call it after
 *                       lmx_dist_round of the same round)
 *   lmx_dist_recv_buffer / lmx_dist_accept   received records
 *   lmx_dist_match      local + confirmed cross-rank matches; returns the
 *                       owned live-slot and matched-vertex counts
 * then all-gathers the owned words of the matched bitmap (exchange B,
 * barrier 2) and all-reduces the counts (RoundStats, termination; on the
 * scan loop dist.py sends them with the next round's record counts).
 * Scan loop: after the loop, lmx_dist_hist also sets the owned range's
 * matched-edge bits.  The
 * matching equals the single-GPU one for every p (bsp.py:113-115).
 */
int lmx_dist_bounds(const lmx_ctx *ctx, int64_t *bounds_out);   /* p + 1 device-id cut points */
int lmx_dist_begin(lmx_ctx *ctx, uint64_t seed_masked, int rerandomize);
int lmx_dist_round(lmx_ctx *ctx);
/* Device outputs, no synchronisation: int64[p] record counts per destination
 * and the records {partner, edge id} (uint32 pairs) packed in destination order. */
int lmx_dist_propose(lmx_ctx *ctx, void **counts_dev_out, void **send_dev_out);
int lmx_dist_recv_buffer(lmx_ctx *ctx, int64_t count, void **recv_out);
int lmx_dist_accept(lmx_ctx *ctx, int64_t count);
/* The late rounds' exchange A without a host round trip (scan loop
 * partitions): after lmx_dist_propose, lay the records out in p slots of
 * `capacity` records each (destination j's records first, the rest filler
 * the receiver's lmx_dist_accept skips), so the all-to-all has equal, host-
 * known splits and lmx_dist_accept takes p * capacity.  capacity must bound
 * every rank's count: the largest list size of any rank at or before this
 * round (lists only shrink); *overflow_dev_out (u32, may be NULL) becomes
 * nonzero if it did not.  lmx_dist_list_size: the device u32 holding this
 * rank's list size for the next round (valid after lmx_dist_match). */
int lmx_dist_pad(lmx_ctx *ctx, int64_t capacity, void **padded_dev_out, void **overflow_dev_out);
int lmx_dist_list_size(lmx_ctx *ctx, void **size_dev_out);
/* Enqueues the match step; *stats_dev_out = device {live slots, matched
 * vertices} (two uint64) of the round, for the all-reduce.  No synchronisation. */
int lmx_dist_match(lmx_ctx *ctx, void **stats_dev_out);
/* Device pointers: matched bitmap (n bits, global device ids), mate (int64[n],
 * caller ids, only owned vertices set), matched-edge bitmap (m bits, edges
 * recorded by this rank), and the context's cudaStream_t. */
int lmx_dist_state(lmx_ctx *ctx, void **matched_bitmap, void **mate, void **edge_bits, void **stream);
/*
 * Contexts whose load chose the weight-ordered scan loop (LMX_QUERY_ALGO == 1)
 * run the same protocol, with {candidates found, matched vertices} as the
 * round's counts ("none found" ends the loop).  RoundStats then come from the
 * death rounds of the edges: the host all-gathers the owned slices of the
 * match-round array (lmx_dist_mround: uint32[n], global device ids) and sums
 * the partitions' histograms (lmx_dist_hist: uint64[*nbins] on the device,
 * bins [0, n_rounds), bin n_rounds = outlived).
 */
int lmx_dist_mround(lmx_ctx *ctx, void **mround_dev);
/*
 * The reference's boundary accounting (bsp.py:29-41 RoundMessages,
 * :148-170), for either round loop, after lmx_dist_mround's slices are
 * all-gathered: *hist_dev = device uint64[2 (n_rounds + 1)]: [0, n_rounds]
 * candidate records by the last round they are sent in (one per owned
 * vertex and receiving partition), then cut edges by death round (each once,
 * from its lower end).  Summed over partitions, the suffix sums are
 * RoundMessages.candidate_records and .cut_edges_surviving.
 */
int lmx_dist_messages(lmx_ctx *ctx, int n_rounds, void **hist_dev);

/*
 * Distributed RMAT build: no rank ever holds the whole graph (config C5).
 * With LMX_OPT_DIST_P = p > 1 and LMX_OPT_DIST_RANK set:
 *   lmx_dist_rmat_build   every rank generates the raw stream (lmx_gen_rmat's
 *                         recipe) and keeps the triples whose lower end lies in
 *                         [rank n / p, (rank + 1) n / p); parallel pairs are
 *                         collapsed as graph.py:94-100 does; out: the bitmap of
 *                         first-occurrence raw positions (*words u32 words), the
 *                         degree contributions (u32[n], caller ids) and the
 *                         weight-bit min / max (u64[2]), all on the device
 *   (host: sum the bitmaps -- the bit sets are disjoint -- and the degrees
 *    over the ranks, in place; min / max of the weight bits)
 *   lmx_dist_rmat_route   global edge ids (graph.py's first-occurrence order),
 *                         partition_graph's cuts on the summed degrees, and this
 *                         rank's pairs packed by destination: 24-byte records
 *                         {edge id, u, v, pad, weight} to the owners of u and v;
 *                         counts_out: int64[p]; m_out: the global edge count
 *   (host: all-to-all-v of the records)
 *   lmx_dist_rmat_recv_buffer / lmx_dist_rmat_finish   the received records are
 *                         the rank's local edges (bsp.py:86-90); ordered by edge
 *                         id, then the partition's K0.  w_uniform: all weights
 *                         equal over the whole graph.
 * The resulting partition equals the one lmx_gen_rmat + LMX_OPT_DIST_P loads.
 */
int lmx_dist_rmat_build(lmx_ctx *ctx, int scale, int edge_factor, double a, double b, double c, uint64_t seed,
                        int permute, void **bits_dev, int64_t *words_out, void **deg_dev, void **minmax_dev);
int lmx_dist_rmat_route(lmx_ctx *ctx, void **send_dev, int64_t *counts_out, int64_t *m_out);
int lmx_dist_rmat_recv_buffer(lmx_ctx *ctx, int64_t count, void **recv_dev);
int lmx_dist_rmat_finish(lmx_ctx *ctx, int w_uniform);

/* Load one partition from its local edges in HOST memory (a multi-GPU job
 * whose ranks already hold their shares, and the multi-GPU end-to-end leg of
 * bench.py): records = the rank's k local edges (bsp.py:86-90) as the 24-byte
 * records lmx_dist_rmat_route produces ({edge id, u, v, pad, weight}: global
 * edge ids and caller vertex ids); deg = the global degrees u32[n] (caller
 * ids), from which partition_graph's cuts follow (bsp.py:60-98); m = the
 * global edge count.  Both are copied to the device on the context's stream
 * (page-locked memory copies at link rate), then the partition's K0 runs as
 * in lmx_dist_rmat_finish.  Replaces the worker state setup of
 * bsp_local_max (bsp.py:117-135) for one worker. */
int lmx_dist_load_local(lmx_ctx *ctx, int64_t n, int64_t m, const uint32_t *deg, int64_t k, const void *records,
                        int w_uniform);
int lmx_dist_hist(lmx_ctx *ctx, int n_rounds, void **hist_dev, int *nbins);

/*
 * Coarsening (config C4; the paper's graph-partitioning use, PAPER.md:32-35,
 * 407-411; absent from the reference).  All pointers are device
 * pointers; the caller sizes the outputs (m_coarse <= m, n_coarse <= n).
 *   lmx_mesh_edges  side x side jittered-grid triangulation: (side-1)(3 side-1)
 *                   unit-weight edges, vertex i*side+j (capacity of eu/ev/w)
 *   lmx_ratings     r(e) = w(e)^2 / (c(u) c(v))
 *   lmx_contract    matched pairs / unmatched vertices -> coarse vertices
 *                   (ascending smallest member), node weights summed, parallel
 *                   edges merged by summed weight in ascending (min, max) order
 */
int lmx_mesh_edges(lmx_ctx *ctx, int64_t side, uint64_t seed, int64_t *edge_u, int64_t *edge_v,
                   double *edge_weight, int64_t *m_out);
int lmx_ratings(lmx_ctx *ctx, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                const double *edge_weight, const double *node_weight, double *rating_out);
int lmx_contract(lmx_ctx *ctx, int64_t n, int64_t m, const int64_t *edge_u, const int64_t *edge_v,
                 const double *edge_weight, const double *node_weight, const int64_t *mate,
                 int64_t *coarse_id_out, int64_t *n_out, int64_t *m_out, int64_t *coarse_u,
                 int64_t *coarse_v, double *coarse_w, double *coarse_c);

/* Device memory in use by the context (bytes). */
int64_t lmx_device_bytes(const lmx_ctx *ctx);

/*
 * validate_matching(g, m) (graph.py:212-237) and Matching.weight(g)
 * (graph.py:54-56,191-192) against the loaded graph (caller's vertex and edge
 * ids).  mate: int64[n]; ids: the matched edge ids, ascending (as
 * Matching.sorted_edge_ids()), n_ids of them; both where `where` says.
 * valid / maximal: the MatchingCheck flags; weight: edge_weight[ids].sum()
 * with numpy's pairwise summation order, bit-identical; detail: the first
 * offence by smallest id ("" when valid).  Any out may be NULL.
 */
int lmx_validate(lmx_ctx *ctx, const int64_t *mate, const int64_t *ids, int64_t n_ids, int where,
                 int *valid, int *maximal, double *weight, char *detail, size_t detail_len);

/*
 * The PRAM restatement's incidence layout and cross pointers
 * (pram.py:54-124 PramState, :127-166 compute_cross_pointers; Lemma 2,
 * PAPER.md:233-257) for the loaded graph: slots sorted by (vertex, edge id)
 * (graph.py:108-115), cross[i] = the other slot of slot i's edge, computed by
 * the reference's two write/read step pairs through a per-edge scratch cell,
 * each step's writes counted and checked for exclusivity (pram.py:28-51
 * WriteLog.record), then PramState.check_consistent's involution checks.
 * cross_out: int64[2m] or NULL (where `out_where` says).  log_out: int64[4] =
 * {steps, writes, conflicts, first slot failing the consistency check or -1}.
 */
int lmx_pram_cross(lmx_ctx *ctx, int64_t *cross_out, int64_t *log_out, int out_where);

/*
 * rbm(g, seed) (matchers.py:357-410): red-blue matching on the loaded graph,
 * the paper's GPU competitor.  Outputs as lmx_match (mate, ascending matched
 * ids, RoundStats).  max_rounds (the reference uses 10 000; <= 0 means that):
 * LMX_ELIMIT when the loop has not finished by then (RbmDidNotConverge).
 * rounds_out (may be NULL) receives up to max_rounds entries; the full trace
 * is in lmx_last_rounds.
 */
int lmx_rbm(lmx_ctx *ctx, uint64_t seed_masked, int64_t *mate_out, int64_t *matched_ids_out,
            int64_t *n_matched_out, lmx_round_stats *rounds_out, int max_rounds, int *n_rounds_out,
            int out_where);

#ifdef __cplusplus
}
#endif
#endif /* LMX_H */
