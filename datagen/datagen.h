/* datagen.h — seeded synthetic workload generators for the MapSQ hot path.
 *
 * INPUT INFRASTRUCTURE ONLY.  This module is shared by the CPU oracle's tests and by the GPU
 * path's tests/bench; it produces dictionary-encoded triples and (key, value) tables and holds
 * NONE of the join method's arithmetic (no map / sort / reduce / join).  Every random draw is a
 * counter-based splitmix64 hash of (seed, entity coordinates), so any university range or row
 * range can be generated independently and the data are identical for any sharding.
 *
 * Workload shapes follow the paper's benchmark description: "LUBM is an ontology for university
 * domain and generates arbitrary scale dataset", and BASELINE.json configs C1-C5.
 * The recipe (ranges, ID layout, emission order) is written down in DESIGN.md §3.
 */
#ifndef MAPSQ_DATAGEN_H
#define MAPSQ_DATAGEN_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* ---- LUBM-shaped vocabulary (fixed IDs 0..63) ---- */
enum {
  LUBM_P_TYPE = 0, LUBM_P_NAME = 1, LUBM_P_EMAIL = 2, LUBM_P_TELEPHONE = 3,
  LUBM_P_SUBORGANIZATIONOF = 4, LUBM_P_WORKSFOR = 5, LUBM_P_HEADOF = 6, LUBM_P_MEMBEROF = 7,
  LUBM_P_UGDEGREEFROM = 8, LUBM_P_MSDEGREEFROM = 9, LUBM_P_PHDDEGREEFROM = 10,
  LUBM_P_RESEARCHINTEREST = 11, LUBM_P_TEACHEROF = 12, LUBM_P_TAKESCOURSE = 13,
  LUBM_P_ADVISOR = 14, LUBM_P_TAOF = 15, LUBM_P_PUBAUTHOR = 16,
  LUBM_N_PRED = 17,
  LUBM_C_UNIVERSITY = 32, LUBM_C_DEPARTMENT = 33, LUBM_C_RESEARCHGROUP = 34,
  LUBM_C_FULLPROF = 35, LUBM_C_ASSOCPROF = 36, LUBM_C_ASSISTPROF = 37, LUBM_C_LECTURER = 38,
  LUBM_C_UGSTUDENT = 39, LUBM_C_GRADSTUDENT = 40, LUBM_C_COURSE = 41, LUBM_C_GRADCOURSE = 42,
  LUBM_C_PUBLICATION = 43
};
#define LUBM_FIRST_UNIV_ID 64u
#define LUBM_N_RESEARCH 100u

/* Bookkeeping computed while generating (independent of oracle and GPU path): exact result
 * cardinalities of the BASELINE.json config queries, derived from the generator's own draws. */
typedef struct {
  uint64_t n_triples;
  uint64_t pred_count[32];
  uint64_t n_dept, n_faculty, n_ug, n_grad;
  uint64_t c1_rs;    /* ?x worksFor ?d . ?d subOrganizationOf ?u             = #worksFor */
  uint64_t c2_j1;    /* ?X memberOf ?Z . ?Z subOrganizationOf ?Y              = #memberOf */
  uint64_t c2_j2;    /* ... . ?X undergraduateDegreeFrom ?Y   = #grads whose ug univ is home */
  uint64_t c3_j1, c3_j2, c3_j3; /* star on dept ?x: #dept, sum F_d, sum F_d*S_d */
  uint64_t c5_j1;    /* ?x advisor ?y . ?y teacherOf ?z                      = sum_p A_p*T_p */
  uint64_t c5_j2;    /* ... . ?x takesCourse ?z      = #(x,z): x takes z, advisor(x) teaches z */
} lubm_stats;

/* Pool of university IDs referenced by degreeFrom: max(n_univ_total, 1000). */
uint32_t lubm_pool_size(uint32_t n_univ_total);
/* First ID of university u's block (requires summing the blocks of universities [0,u)). */
uint64_t lubm_univ_base(uint64_t seed, uint32_t n_univ_total, uint32_t u);
/* Dictionary size (1 + max ID) of the full dataset / of universities [0,u_hi). */
uint64_t lubm_id_end(uint64_t seed, uint32_t n_univ_total, uint32_t u_hi);
/* Count the triples of universities [u_lo,u_hi) and fill bookkeeping (stats may be NULL). */
uint64_t lubm_count(uint64_t seed, uint32_t n_univ_total, uint32_t u_lo, uint32_t u_hi,
                    lubm_stats *stats);
/* Emit the triples of universities [u_lo,u_hi) into s/p/o (capacity from lubm_count), SoA,
 * in generation order (per university, per department).  Returns the number written. */
uint64_t lubm_generate(uint64_t seed, uint32_t n_univ_total, uint32_t u_lo, uint32_t u_hi,
                       uint32_t *s, uint32_t *p, uint32_t *o, lubm_stats *stats);

/* ---- C4: Zipf(s) join keys (SURVEY §8.c R15 reading) ----
 * rank r ~ Zipf(s) on [1, 2^kbits] by rejection-inversion (Hörmann & Derflinger 1996);
 * key = (A_side*(r-1) + B_side) mod 2^kbits with A_side odd (a bijection per side);
 * value = splitmix64-derived 32-bit payload.  Rows [i_lo, i_hi) of side `side`. */
void zipf_table(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i_lo, uint64_t i_hi,
                uint32_t *key, uint32_t *val);
/* One rank draw for row i (exposed for distribution tests). */
uint64_t zipf_rank(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i);

/* Uniform random (key, value) table for tests: key in [0,key_domain), value in [0,val_domain). */
void uniform_table(uint64_t seed, uint64_t n, uint32_t key_domain, uint32_t val_domain,
                   uint32_t *key, uint32_t *val);

int datagen_num_threads(void);

#ifdef __cplusplus
}
#endif
#endif
