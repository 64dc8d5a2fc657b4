/* oracle.h — CPU oracle for the MapSQ join path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load this library.
 * It shares no code, header, table or helper with the CUDA path (paper_1702_03484_b200/).
 *
 * What it computes (PAPER.md, arXiv 1702.03484):
 *   - partial matching of one triple pattern: standard SPARQL triple-pattern
 *     matching over a set of dictionary-encoded triples;
 *   - the join of two partial-match tables Tp1, Tp2 (Alg. 1 Require/Ensure): the
 *     natural join on ALL shared variables, as a bag of solution mappings;
 *   - the chained joins of a basic graph pattern and the final projection.
 * Tier 0 (nested loop, the "plain join algorithm" of P:113) is the definition written out.
 * Tier 1 (sort-merge) is the same definition grouped by key with a library sort; it is pinned
 * to tier 0 and to brute force in tests/test_oracle_pins.py.
 * Readings of ambiguous passages (R1-R16) are listed in DESIGN.md §2.
 *
 * Tables are row-major: rows[r * ncols + c] is the value of variable var[c] in row r.
 */
#ifndef MAPSQ_ORACLE_H
#define MAPSQ_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORACLE_MAX_COLS 16

typedef struct {
  uint64_t nrows;
  uint32_t ncols;
  int32_t var[ORACLE_MAX_COLS];
  uint32_t *rows; /* malloc'd, nrows*ncols, freed with oracle_free */
} oracle_table;

enum { ORACLE_OK = 0, ORACLE_E_INVALID = 1, ORACLE_E_NO_SHARED = 2, ORACLE_E_NOMEM = 3 };

/* var[j] >= 0: variable id at position j (s, p, o); var[j] == -1: constant id[j]. */
int oracle_scan(uint64_t n, const uint32_t *s, const uint32_t *p, const uint32_t *o,
                const int32_t var[3], const uint32_t id[3], oracle_table *out);
int oracle_join_nested(const oracle_table *a, const oracle_table *b, oracle_table *out);
int oracle_join_sortmerge(const oracle_table *a, const oracle_table *b, oracle_table *out);
/* Left-deep fold of the patterns in the given order, then projection onto proj[0..nproj)
 * (nproj == 0: all variables in first-appearance order).  Bag semantics. */
int oracle_query(uint64_t n, const uint32_t *s, const uint32_t *p, const uint32_t *o,
                 const int32_t *pat_var, const uint32_t *pat_id, int npats, const int32_t *proj,
                 int nproj, oracle_table *out);
/* Sort rows lexicographically (ascending u32 tuples) in place. */
void oracle_canonical_sort(oracle_table *t);
void oracle_free(oracle_table *t);
/* Multiset fingerprint of a table's rows, ACCUMULATED into acc = {count, sum mod 2^64, xor} of
 * the per-row hash h = fold(h := splitmix64_step(h ^ v)) over the row's values in column order
 * (SURVEY §8(c) step 6).  Order-independent; call repeatedly over chunks of one table. */
void oracle_fingerprint(const oracle_table *t, uint64_t acc[3]);
/* The same over SoA columns cols[0..ncols), each nrows long (device results copied to host). */
void oracle_fingerprint_cols(uint64_t nrows, uint32_t ncols, const uint32_t *const *cols,
                             uint64_t acc[3]);

#ifdef __cplusplus
}
#endif
#endif
