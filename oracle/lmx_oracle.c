/*
 * lmx_oracle.c -- CPU restatement of the reference local max matching path.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity checker for the CUDA
 * engine in paper_1302_4587_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  The
 * product path never links or calls it.
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * the npz files in tests/golden, which tests/golden/make_golden.py produced by running the
 * unmodified reference package (/root/reference/pkg/src/locmax) in the build
 * container.
 *
 * Restated reference functions (file:line relative to /root/reference/pkg/src/locmax):
 *   lmxo_mix64          tiebreak.py:28-37   (SplitMix64 finalizer, constants :20-22)
 *   lmxo_round_seed     tiebreak.py:40-52
 *   lmxo_edge_salt      tiebreak.py:55-59
 *   lmxo_weight_bits    tiebreak.py:105-113 (+0.0 canonicalises -0.0)
 *   lmxo_local_max      matchers.py:61-122  (local_max_seq) + graph.py:195-203
 *                        (matching_from_edge_ids)
 *
 * Build: oracle/Makefile -> oracle/_build/liblmx_oracle.so (plain gcc -O2).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define LMXO_GOLDEN 0x9E3779B97F4A7C15ULL
#define LMXO_MIX_A 0xBF58476D1CE4E5B9ULL
#define LMXO_MIX_B 0x94D049BB133111EBULL

/* tiebreak.py:28-37 */
uint64_t lmxo_mix64(uint64_t v) {
    uint64_t x = v + LMXO_GOLDEN;
    x ^= x >> 30;
    x *= LMXO_MIX_A;
    x ^= x >> 27;
    x *= LMXO_MIX_B;
    x ^= x >> 31;
    return x;
}

/* tiebreak.py:40-52; the caller masks the Python seed to 64 bits (:49). */
uint64_t lmxo_round_seed(uint64_t seed_masked, uint64_t round_index, int rerandomize) {
    uint64_t r = rerandomize ? round_index : 0;
    return lmxo_mix64(lmxo_mix64(seed_masked) ^ r);
}

/* tiebreak.py:55-59 */
uint64_t lmxo_edge_salt(uint64_t round_seed_value, uint64_t edge_id) {
    return lmxo_mix64(edge_id ^ round_seed_value);
}

/* tiebreak.py:105-113: (w + 0.0) viewed as uint64. */
uint64_t lmxo_weight_bits(double w) {
    double c = w + 0.0;
    uint64_t b;
    memcpy(&b, &c, sizeof b);
    return b;
}

/*
 * matchers.py:61-122.  Pass 1 (:93-103) takes the lexicographic maximum of
 * (weight bits, salt, edge id) per endpoint; the reference does it in three
 * scatter-max stages, each restricted to the ties of the previous stage,
 * which is exactly a lexicographic max, restated here as one scan.
 * Pass 2 (:104-109): an edge wins iff it is the candidate at both ends.
 * Pass 3 (:110-118): edges with a matched endpoint die; survivors' endpoints
 * get the dummy candidate back.
 *
 * Outputs: mate[n] (-1 unmatched), matched_ids (ascending, <= n/2 entries),
 * rounds_out[3*r] = (edges_before, edges_matched, edges_removed).
 * Returns the number of rounds, or -1 on allocation failure, -2 if
 * max_rounds is too small.
 */
int lmxo_local_max(int64_t n, int64_t m, const int64_t *eu, const int64_t *ev,
                   const double *w, uint64_t seed_masked, int rerandomize,
                   int64_t *mate, int64_t *matched_ids, int64_t *n_matched,
                   int64_t *rounds_out, int max_rounds) {
    /* Lean state (RMAT-26 runs in ~32 GB with the graph): the weight bits and
     * salts are recomputed where the reference keeps them in arrays
     * (matchers.py:88-92); the live list is u32 while m < 2^32. */
    const int narrow = m < (int64_t)0xFFFFFFFFLL;
    uint64_t *cand_w = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
    uint64_t *cand_s = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
    int64_t *cand_id = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    unsigned char *vm = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
    void *live = malloc((size_t)(m > 0 ? m : 1) * (narrow ? sizeof(uint32_t) : sizeof(int64_t)));
    unsigned char *edge_won = (unsigned char *)calloc((size_t)(m > 0 ? m : 1), 1);
    if (!cand_w || !cand_s || !cand_id || !vm || !live || !edge_won) {
        free(cand_w); free(cand_s); free(cand_id); free(vm); free(live); free(edge_won);
        return -1;
    }
    uint32_t *live32 = (uint32_t *)live;
    int64_t *live64 = (int64_t *)live;
#define LIVE(i) (narrow ? (int64_t)live32[i] : live64[i])
#define SET_LIVE(i, e) do { if (narrow) live32[i] = (uint32_t)(e); else live64[i] = (e); } while (0)
    for (int64_t v = 0; v < n; ++v) cand_id[v] = -1;
    for (int64_t e = 0; e < m; ++e) SET_LIVE(e, e);
    int64_t nlive = m;
    int round_index = 0;
    int status = 0;
    while (nlive > 0) {
        if (round_index >= max_rounds) { status = -2; break; }
        uint64_t rs = lmxo_round_seed(seed_masked, (uint64_t)round_index, rerandomize);
        /* pass 1 */
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = LIVE(i);
            uint64_t kw = lmxo_weight_bits(w[e]);
            uint64_t ks = lmxo_edge_salt(rs, (uint64_t)e);
            int64_t ends[2] = {eu[e], ev[e]};
            for (int k = 0; k < 2; ++k) {
                int64_t x = ends[k];
                int better = 0;
                if (cand_id[x] < 0) better = 1;
                else if (kw != cand_w[x]) better = kw > cand_w[x];
                else if (ks != cand_s[x]) better = ks > cand_s[x];
                else better = e > cand_id[x];
                if (better) { cand_w[x] = kw; cand_s[x] = ks; cand_id[x] = e; }
            }
        }
        /* pass 2 */
        int64_t won = 0;
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = LIVE(i);
            if (cand_id[eu[e]] == e && cand_id[ev[e]] == e) {
                edge_won[e] = 1;
                ++won;
            }
        }
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = LIVE(i);
            if (edge_won[e]) { vm[eu[e]] = 1; vm[ev[e]] = 1; }
        }
        /* pass 3 */
        int64_t k = 0;
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = LIVE(i);
            if (!(vm[eu[e]] || vm[ev[e]])) {
                SET_LIVE(k, e);
                ++k;
                cand_w[eu[e]] = cand_w[ev[e]] = 0;
                cand_s[eu[e]] = cand_s[ev[e]] = 0;
                cand_id[eu[e]] = cand_id[ev[e]] = -1;
            }
        }
        rounds_out[3 * round_index + 0] = nlive;
        rounds_out[3 * round_index + 1] = won;
        rounds_out[3 * round_index + 2] = nlive - k;
        nlive = k;
        ++round_index;
    }
#undef LIVE
#undef SET_LIVE
    /* graph.py:195-203 */
    for (int64_t v = 0; v < n; ++v) mate[v] = -1;
    int64_t cnt = 0;
    for (int64_t e = 0; e < m; ++e) {
        if (edge_won[e]) {
            mate[eu[e]] = ev[e];
            mate[ev[e]] = eu[e];
            matched_ids[cnt++] = e;
        }
    }
    *n_matched = cnt;
    free(cand_w); free(cand_s); free(cand_id); free(vm); free(live); free(edge_won);
    return status < 0 ? status : round_index;
}

/* Salts of many edge ids under one round seed (tiebreak.py:55-59), for tests. */
void lmxo_edge_salts(uint64_t round_seed_value, const uint64_t *ids, int64_t k, uint64_t *out) {
    for (int64_t i = 0; i < k; ++i) out[i] = lmxo_edge_salt(round_seed_value, ids[i]);
}

/* ------------------------------------------------------------------------
 * Input restatements for the scale fixtures (tests/golden/make_golden_scale.py).
 *
 * lmxo_rmat_raw: the RMAT generator of csrc/lmx_build.cu (header comment),
 * restated from its published recipe, identical to oracle.py:rmat_raw (the
 * two are cross-checked in tests/test_oracle_golden.py).  Raw triple i:
 *   h = mix64(s0 ^ (i*16 + l/4)) every 4 levels, x = 16-bit field l%4 of h;
 *   quadrant thresholds A, A+B, A+B+C (16-bit fixed point);
 *   w = (mix64(s1 ^ i) >> 11) * 2^-53; optional bijective relabelling.
 * Pure function of i, so the loop is split over threads (OpenMP).
 */

/* Split [0, total) over the host's threads (pure per-index work only). */
typedef void (*lmxo_range_fn)(void *arg, int64_t begin, int64_t end);
typedef struct { lmxo_range_fn fn; void *arg; int64_t b, e; } lmxo_job;
static void *lmxo_job_run(void *p) { lmxo_job *j = (lmxo_job *)p; j->fn(j->arg, j->b, j->e); return NULL; }
static void lmxo_parallel(int64_t total, lmxo_range_fn fn, void *arg, int chunks) {
    long nt = sysconf(_SC_NPROCESSORS_ONLN);
    if (nt < 1) nt = 1;
    if (nt > 64) nt = 64;
    if (chunks < (int)nt) chunks = (int)nt;
    if (chunks > 4096) chunks = 4096;
    /* chunks are handed out round-robin to nt workers: chunk c -> worker c % nt */
    pthread_t th[64];
    lmxo_job jobs[4096];
    for (int c = 0; c < chunks; ++c) {
        jobs[c].fn = fn; jobs[c].arg = arg;
        jobs[c].b = total * c / chunks; jobs[c].e = total * (c + 1) / chunks;
    }
    for (int c0 = 0; c0 < chunks; c0 += (int)nt) {
        int started = 0;
        for (int t = 0; t < nt && c0 + t < chunks; ++t, ++started)
            pthread_create(&th[t], NULL, lmxo_job_run, &jobs[c0 + t]);
        for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    }
}

#define LMXO_RMAT_TAG0 0x524D41545F4C5654ULL
#define LMXO_RMAT_TAG1 0x524D41545F574754ULL
#define LMXO_RMAT_TAG2 0x524D41545F504552ULL

static uint64_t lmxo_rmat_perm(uint64_t x, int scale, uint64_t s2) {
    const uint64_t mask = (scale >= 64) ? ~0ULL : ((1ULL << scale) - 1);
    const int h = scale / 2 + 1;
    const int h2 = scale - h > 0 ? scale - h : 1;
    uint64_t y = x;
    y = (y * 0x9E3779B97F4A7C15ULL) & mask;
    y ^= y >> h;
    y = (y * 0xBF58476D1CE4E5B9ULL) & mask;
    y ^= y >> h2;
    y ^= s2 & mask;
    return y;
}

typedef struct {
    int scale, permute;
    uint32_t A, AB, ABC;
    uint64_t s0, s1, s2;
    uint32_t *u, *v;
    double *w;
} lmxo_rmat_job;

static void lmxo_rmat_range(void *arg, int64_t begin, int64_t end) {
    const lmxo_rmat_job *p = (const lmxo_rmat_job *)arg;
    for (int64_t i = begin; i < end; ++i) {
        uint64_t a = 0, b = 0, h = 0;
        for (int l = 0; l < p->scale; ++l) {
            if ((l & 3) == 0) h = lmxo_mix64(p->s0 ^ ((uint64_t)i * 16ULL + (uint64_t)(l >> 2)));
            const uint32_t x = (uint32_t)((h >> (16 * (l & 3))) & 0xFFFFu);
            const uint64_t bit = 1ULL << (p->scale - 1 - l);
            if (x >= p->AB) a |= bit;                                /* quadrants (1,0), (1,1) */
            if ((x >= p->A && x < p->AB) || x >= p->ABC) b |= bit;   /* quadrants (0,1), (1,1) */
        }
        if (p->permute) {
            a = lmxo_rmat_perm(a, p->scale, p->s2);
            b = lmxo_rmat_perm(b, p->scale, p->s2);
        }
        p->u[i] = (uint32_t)a;
        p->v[i] = (uint32_t)b;
        p->w[i] = (double)(lmxo_mix64(p->s1 ^ (uint64_t)i) >> 11) * (1.0 / 9007199254740992.0);
    }
}

void lmxo_rmat_raw(int scale, int64_t k, uint32_t A, uint32_t AB, uint32_t ABC, uint64_t seed_masked,
                   int permute, uint32_t *u, uint32_t *v, double *w) {
    lmxo_rmat_job job;
    job.scale = scale; job.permute = permute;
    job.A = A; job.AB = AB; job.ABC = ABC;
    job.s0 = lmxo_mix64(seed_masked ^ LMXO_RMAT_TAG0);
    job.s1 = lmxo_mix64(seed_masked ^ LMXO_RMAT_TAG1);
    job.s2 = lmxo_mix64(seed_masked ^ LMXO_RMAT_TAG2);
    job.u = u; job.v = v; job.w = w;
    lmxo_parallel(k, lmxo_rmat_range, &job, 64);
}

/*
 * lmxo_build_graph: graph.py:59-119 numbering contract on raw triples with
 * 32-bit ids (validated by the caller), in O(k) memory beyond the inputs:
 *   * self-loops dropped (:89-91);
 *   * pairs grouped by their lower endpoint (a counting sort, positions stay
 *     ascending), then by the higher one (a stable sort per bucket);
 *   * per pair: the first occurrence of the maximum weight (strict '>', :99)
 *     is kept with its orientation and weight bits (:100);
 *   * edge ids follow each pair's first occurrence (:94-98).
 * rep (caller scratch, u32[k]) maps a first-occurrence position to the kept
 * position.  Outputs (capacity k): int64 eu/ev, f64 ew.  Returns m, or -1 on
 * allocation failure.  num_vertices sizes the buckets (ids < num_vertices).
 */
typedef struct { uint32_t hi, pos; } lmxo_hp;

static int lmxo_hp_cmp(const void *a, const void *b) {
    const lmxo_hp *x = (const lmxo_hp *)a, *y = (const lmxo_hp *)b;
    if (x->hi != y->hi) return x->hi < y->hi ? -1 : 1;
    return x->pos < y->pos ? -1 : (x->pos > y->pos ? 1 : 0);
}

typedef struct {
    lmxo_hp *bk;
    const uint64_t *off;
    const double *w;
    uint32_t *rep;
} lmxo_bucket_job;

static void lmxo_bucket_range(void *arg, int64_t begin, int64_t end) {
    const lmxo_bucket_job *p = (const lmxo_bucket_job *)arg;
    for (int64_t x = begin; x < end; ++x) {
        lmxo_hp *seg = p->bk + p->off[x];
        const uint64_t len = p->off[x + 1] - p->off[x];
        if (len > 1) qsort(seg, (size_t)len, sizeof(lmxo_hp), lmxo_hp_cmp);
        for (uint64_t j = 0; j < len;) {
            uint64_t t = j;
            uint32_t best = seg[j].pos;
            while (t + 1 < len && seg[t + 1].hi == seg[j].hi) {
                ++t;
                if (p->w[seg[t].pos] > p->w[best]) best = seg[t].pos;   /* strict '>' keeps the earliest */
            }
            p->rep[seg[j].pos] = best;   /* seg[j].pos is the pair's first occurrence */
            j = t + 1;
        }
    }
}

int64_t lmxo_build_graph(int64_t k, const uint32_t *u, const uint32_t *v, const double *w,
                         int64_t num_vertices, uint32_t *rep, int64_t *eu, int64_t *ev, double *ew) {
    const int64_t n = num_vertices;
    uint64_t *off = (uint64_t *)calloc((size_t)n + 2, sizeof(uint64_t));
    if (!off) return -1;
    for (int64_t i = 0; i < k; ++i)
        if (u[i] != v[i]) ++off[(u[i] < v[i] ? u[i] : v[i]) + 1];
    for (int64_t x = 0; x < n; ++x) off[x + 1] += off[x];
    const uint64_t total = off[n];
    lmxo_hp *bk = (lmxo_hp *)malloc((size_t)(total ? total : 1) * sizeof(lmxo_hp));
    uint64_t *cur = (uint64_t *)malloc((size_t)(n ? n : 1) * sizeof(uint64_t));
    if (!bk || !cur) { free(off); free(bk); free(cur); return -1; }
    memcpy(cur, off, (size_t)n * sizeof(uint64_t));
    for (int64_t i = 0; i < k; ++i) {
        if (u[i] == v[i]) continue;
        const uint32_t lo = u[i] < v[i] ? u[i] : v[i], hi = u[i] < v[i] ? v[i] : u[i];
        lmxo_hp r = {hi, (uint32_t)i};
        bk[cur[lo]++] = r;
    }
    free(cur);
    for (int64_t i = 0; i < k; ++i) rep[i] = 0xFFFFFFFFu;
    lmxo_bucket_job job = {bk, off, w, rep};
    lmxo_parallel(n, lmxo_bucket_range, &job, 4096);
    free(bk);
    free(off);
    int64_t m = 0;
    for (int64_t i = 0; i < k; ++i) {
        const uint32_t c = rep[i];
        if (c == 0xFFFFFFFFu) continue;
        eu[m] = u[c];
        ev[m] = v[c];
        ew[m] = w[c];
        ++m;
    }
    return m;
}
