/* oracle/pms8_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference PMS8 per-S1-l-mer search
 * (/root/reference/proj), used by tests/ as the parity checker and by
 * bench.py's cpu_baseline leg only when oracle/_ref is missing. Never linked
 * into, or called by, the product (paper_1307_0571_b200/).
 *
 * Parity status: PINNED — tests/test_oracle.py checks this restatement against
 * golden vectors produced by the reference itself (oracle/_ref, built from the
 * reference sources by oracle/Makefile; generator script tests/golden/make_golden.py).
 *
 * Codes are uint8 in [0, sigma); sequences are n x m row-major. Motifs are
 * returned as l codes each, sorted lexicographically and deduplicated
 * (canonical_motif_set, src/solver.cpp:16-21).
 */
#ifndef PMS8_ORACLE_H
#define PMS8_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* generate_planted_instance, src/instance.cpp:22-73 (mt19937_64 + bounded_draw).
 * codes_out: n*m, motif_out: l codes, positions_out: n. exact=1: exactly_d. */
int pms8o_generate(int n, int m, int l, int d, int sigma, uint64_t seed, int exact, uint8_t* codes_out,
                   uint8_t* motif_out, int32_t* positions_out);

/* neighborhood_size, src/instance.cpp:75-87; decimal string into buf. */
int pms8o_neighborhood_size(int l, int d, int sigma, char* buf, int buflen);

/* estimate_threshold, src/solver.cpp:75-117. */
int pms8o_estimate_threshold(int n, int m, int l, int d, int sigma);

/* Theorem 1, src/pruning.cpp:65-75 (strings as codes). */
int pms8o_triple_ok(const uint8_t* a, const uint8_t* b, const uint8_t* c, int l, int d1, int d2, int d3);

/* consensus_total_distance, src/pruning.cpp:27-43. tuple: k rows of l codes. */
int pms8o_consensus_distance(const uint8_t* tuple, int k, int l);

/* NeighborhoodEnumerator prepare/descend/prune, src/neighborhood.cpp:164-270,
 * include/pms8/neighborhood.hpp:52-88. Visits in code order; writes up to cap
 * neighbours (l codes each) and returns the total count. level: 0 none,
 * 1 pairs, 2 full. */
int64_t pms8o_common_neighborhood(const uint8_t* tuple, int k, int l, int sigma, int d, int level, uint8_t* out,
                                  int64_t cap);

/* MotifSearch::run_anchored over the given S1 offsets (all offsets when
 * anchors == NULL), src/solver.cpp:227-432 + src/parallel.cpp:35-90.
 * t <= 0 uses estimate_threshold. Output sorted+unique; returns count (may
 * exceed cap; only cap written). counters (may be NULL): [pushes, tuples,
 * leaves, emitted, filter_slots, verify_compares]. */
int64_t pms8o_solve(const uint8_t* codes, int n, int m, int l, int d, int sigma, int t, const int32_t* anchors,
                    int nanchors, uint8_t* out, int64_t cap, int64_t* counters);

/* naive_is_motif, src/oracle.cpp:16-37. */
int pms8o_is_motif(const uint8_t* codes, int n, int m, int l, int d, const uint8_t* motif);

/* brute_force_solve, src/oracle.cpp:65-75 (sigma^l scan; caller bounds it). */
int64_t pms8o_brute_force(const uint8_t* codes, int n, int m, int l, int d, int sigma, uint8_t* out, int64_t cap);

#ifdef __cplusplus
}
#endif
#endif
