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
    uint64_t *cand_w = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
    uint64_t *cand_s = (uint64_t *)calloc((size_t)(n > 0 ? n : 1), sizeof(uint64_t));
    int64_t *cand_id = (int64_t *)malloc((size_t)(n > 0 ? n : 1) * sizeof(int64_t));
    unsigned char *vm = (unsigned char *)calloc((size_t)(n > 0 ? n : 1), 1);
    int64_t *live = (int64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(int64_t));
    unsigned char *edge_won = (unsigned char *)calloc((size_t)(m > 0 ? m : 1), 1);
    uint64_t *wb = (uint64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    uint64_t *salt = (uint64_t *)malloc((size_t)(m > 0 ? m : 1) * sizeof(uint64_t));
    if (!cand_w || !cand_s || !cand_id || !vm || !live || !edge_won || !wb || !salt) {
        free(cand_w); free(cand_s); free(cand_id); free(vm); free(live);
        free(edge_won); free(wb); free(salt);
        return -1;
    }
    for (int64_t v = 0; v < n; ++v) cand_id[v] = -1;
    for (int64_t e = 0; e < m; ++e) { live[e] = e; wb[e] = lmxo_weight_bits(w[e]); }
    int64_t nlive = m;
    int round_index = 0;
    int status = 0;
    while (nlive > 0) {
        if (round_index >= max_rounds) { status = -2; break; }
        uint64_t rs = lmxo_round_seed(seed_masked, (uint64_t)round_index, rerandomize);
        /* pass 1 */
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = live[i];
            uint64_t kw = wb[e];
            uint64_t ks = lmxo_edge_salt(rs, (uint64_t)e);
            salt[e] = ks;
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
            int64_t e = live[i];
            if (cand_id[eu[e]] == e && cand_id[ev[e]] == e) {
                edge_won[e] = 1;
                ++won;
            }
        }
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = live[i];
            if (edge_won[e]) { vm[eu[e]] = 1; vm[ev[e]] = 1; }
        }
        /* pass 3 */
        int64_t k = 0;
        for (int64_t i = 0; i < nlive; ++i) {
            int64_t e = live[i];
            if (!(vm[eu[e]] || vm[ev[e]])) {
                live[k++] = e;
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
    free(cand_w); free(cand_s); free(cand_id); free(vm); free(live);
    free(edge_won); free(wb); free(salt);
    return status < 0 ? status : round_index;
}

/* Salts of many edge ids under one round seed (tiebreak.py:55-59), for tests. */
void lmxo_edge_salts(uint64_t round_seed_value, const uint64_t *ids, int64_t k, uint64_t *out) {
    for (int64_t i = 0; i < k; ++i) out[i] = lmxo_edge_salt(round_seed_value, ids[i]);
}
