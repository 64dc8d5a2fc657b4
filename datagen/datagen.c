/* datagen.c — seeded synthetic workload generators (input infrastructure; see datagen.h).
 *
 * LUBM-shaped university graph: the paper benchmarks on LUBM ("an ontology for
 * university domain [that] generates arbitrary scale dataset"); the UBA generator itself is an
 * external tool, so this is a structural analogue with UBA-like ranges (recipe in
 * DESIGN.md §3).  Every draw is splitmix64 of (seed, university, department, attribute, index),
 * so universities are independent and any range can be generated on any rank.
 */
#include "datagen.h"
#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static inline uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
static inline uint64_t h4(uint64_t seed, uint64_t a, uint64_t b, uint64_t c, uint64_t d) {
  uint64_t h = splitmix64(seed ^ 0x5851F42D4C957F2DULL);
  h = splitmix64(h ^ a);
  h = splitmix64(h ^ b);
  h = splitmix64(h ^ c);
  return splitmix64(h ^ d);
}
static inline uint32_t uni(uint64_t r, uint32_t lo, uint32_t hi) {
  return lo + (uint32_t)(r % (uint64_t)(hi - lo + 1));
}

/* attribute tags of the hash coordinates */
enum {
  T_NDEPT = 1, T_NFULL, T_NASSOC, T_NASSIST, T_NLECT, T_NGROUP, T_NUG, T_NGRAD, T_NC, T_NG, T_NPUB,
  T_FUG, T_FMS, T_FPHD, T_RI, T_UG_NTAKE, T_UG_TAKE, T_UG_HASADV, T_UG_ADV, T_GR_UGDEG,
  T_GR_NTAKE, T_GR_TAKE, T_GR_ADV, T_GR_HASTA, T_GR_TA
};
#define TAG(t, i) ((((uint64_t)(t)) << 32) | (uint64_t)(i))
#define DEPT_NONE 0xFFFFFFFFull
#define MAXF 64

typedef struct {
  uint32_t nrank[4], F, nprof, ngroups, nug, ngrad;
  uint32_t nc[MAXF], ng[MAXF], npub[MAXF];
  uint32_t cb[MAXF], gb[MAXF], pb[MAXF];
  uint32_t ncourse, ngcourse, npubs;
  uint32_t off_group, off_fac, off_ug, off_grad, off_course, off_gcourse, off_pub, E, Pn;
  uint64_t nids;
} dept_layout;

uint32_t lubm_pool_size(uint32_t n_univ_total) { return n_univ_total > 1000 ? n_univ_total : 1000; }

static uint32_t univ_ndept(uint64_t seed, uint32_t u) {
  return uni(h4(seed, u, DEPT_NONE, TAG(T_NDEPT, 0), 0), 15, 25);
}

static void layout(uint64_t seed, uint32_t u, uint32_t d, dept_layout *L) {
  static const uint32_t lo[4] = {7, 10, 8, 5}, hi[4] = {10, 14, 11, 7};
  static const uint32_t plo[4] = {15, 10, 5, 0}, phi[4] = {20, 18, 10, 5};
  L->F = 0;
  for (int r = 0; r < 4; r++) {
    L->nrank[r] = uni(h4(seed, u, d, TAG(T_NFULL + r, 0), 0), lo[r], hi[r]);
    L->F += L->nrank[r];
  }
  L->nprof = L->nrank[0] + L->nrank[1] + L->nrank[2];
  L->ngroups = uni(h4(seed, u, d, TAG(T_NGROUP, 0), 0), 10, 20);
  L->nug = L->F * uni(h4(seed, u, d, TAG(T_NUG, 0), 0), 8, 14);
  L->ngrad = L->F * uni(h4(seed, u, d, TAG(T_NGRAD, 0), 0), 3, 4);
  uint32_t c = 0, g = 0, p = 0, fi = 0;
  for (int r = 0; r < 4; r++)
    for (uint32_t j = 0; j < L->nrank[r]; j++, fi++) {
      L->nc[fi] = uni(h4(seed, u, d, TAG(T_NC, fi), 0), 1, 2);
      L->ng[fi] = uni(h4(seed, u, d, TAG(T_NG, fi), 0), 1, 2);
      L->npub[fi] = uni(h4(seed, u, d, TAG(T_NPUB, fi), 0), plo[r], phi[r]);
      L->cb[fi] = c; c += L->nc[fi];
      L->gb[fi] = g; g += L->ng[fi];
      L->pb[fi] = p; p += L->npub[fi];
    }
  L->ncourse = c; L->ngcourse = g; L->npubs = p;
  L->off_group = 0;
  L->off_fac = L->ngroups;
  L->off_ug = L->off_fac + L->F;
  L->off_grad = L->off_ug + L->nug;
  L->off_course = L->off_grad + L->ngrad;
  L->off_gcourse = L->off_course + L->ncourse;
  L->off_pub = L->off_gcourse + L->ngcourse;
  L->E = L->off_pub + L->npubs;
  L->Pn = L->F + L->nug + L->ngrad;
  /* entities, their name literals, the department's name literal, email + telephone literals */
  L->nids = 2ull * L->E + 1 + 2ull * L->Pn;
}

static uint64_t univ_ids(uint64_t seed, uint32_t u) {
  uint32_t nd = univ_ndept(seed, u);
  uint64_t n = nd + 1; /* department entities + university name literal */
  for (uint32_t d = 0; d < nd; d++) {
    dept_layout L;
    layout(seed, u, d, &L);
    n += L.nids;
  }
  return n;
}

static inline uint64_t id_base0(uint32_t P) { return LUBM_FIRST_UNIV_ID + (uint64_t)P + LUBM_N_RESEARCH; }

/* k distinct values in [0, range), in draw order */
static void pick_distinct(uint64_t seed, uint32_t u, uint32_t d, uint64_t tag, uint32_t k,
                          uint32_t range, uint32_t *out) {
  for (uint32_t j = 0; j < k; j++) {
    for (uint32_t t = 0;; t++) {
      uint32_t c = (uint32_t)(h4(seed, u, d, tag, ((uint64_t)j << 16) | t) % range);
      int dup = 0;
      for (uint32_t q = 0; q < j; q++) dup |= (out[q] == c);
      if (!dup) { out[j] = c; break; }
    }
  }
}

#define EMIT(S_, P_, O_)                                                   \
  do {                                                                     \
    if (os) { os[k] = (uint32_t)(S_); op[k] = (uint32_t)(P_); oo[k] = (uint32_t)(O_); } \
    k++;                                                                   \
    st->pred_count[(P_)]++;                                                \
  } while (0)

/* Emit (or only count, when os == NULL) all triples of university u whose ID block starts at
 * `base`.  Bookkeeping counters accumulate into *st. */
static uint64_t emit_univ(uint64_t seed, uint32_t P, uint32_t u, uint64_t base, uint32_t *os,
                          uint32_t *op, uint32_t *oo, lubm_stats *st) {
  uint64_t k = 0;
  const uint32_t nd = univ_ndept(seed, u);
  const uint64_t uid = LUBM_FIRST_UNIV_ID + u;
  const uint64_t ri0 = LUBM_FIRST_UNIV_ID + (uint64_t)P;
  EMIT(uid, LUBM_P_TYPE, LUBM_C_UNIVERSITY);
  EMIT(uid, LUBM_P_NAME, base + nd);
  uint64_t b = base + nd + 1;
  for (uint32_t d = 0; d < nd; d++) {
    dept_layout L;
    layout(seed, u, d, &L);
    const uint64_t did = base + d, E = L.E, Pn = L.Pn;
    uint32_t adv_count[MAXF];
    memset(adv_count, 0, sizeof adv_count);
    EMIT(did, LUBM_P_TYPE, LUBM_C_DEPARTMENT);
    EMIT(did, LUBM_P_NAME, b + 2 * E);
    EMIT(did, LUBM_P_SUBORGANIZATIONOF, uid);
    for (uint32_t g = 0; g < L.ngroups; g++) {
      uint64_t e = L.off_group + g;
      EMIT(b + e, LUBM_P_TYPE, LUBM_C_RESEARCHGROUP);
      EMIT(b + e, LUBM_P_NAME, b + E + e);
      EMIT(b + e, LUBM_P_SUBORGANIZATIONOF, did);
    }
    uint32_t fi = 0;
    for (int r = 0; r < 4; r++)
      for (uint32_t j = 0; j < L.nrank[r]; j++, fi++) {
        uint64_t e = L.off_fac + fi, id = b + e, pers = fi;
        EMIT(id, LUBM_P_TYPE, LUBM_C_FULLPROF + r);
        EMIT(id, LUBM_P_NAME, b + E + e);
        EMIT(id, LUBM_P_EMAIL, b + 2 * E + 1 + pers);
        EMIT(id, LUBM_P_TELEPHONE, b + 2 * E + 1 + Pn + pers);
        EMIT(id, LUBM_P_WORKSFOR, did);
        EMIT(id, LUBM_P_UGDEGREEFROM, LUBM_FIRST_UNIV_ID + h4(seed, u, d, TAG(T_FUG, fi), 0) % P);
        EMIT(id, LUBM_P_MSDEGREEFROM, LUBM_FIRST_UNIV_ID + h4(seed, u, d, TAG(T_FMS, fi), 0) % P);
        EMIT(id, LUBM_P_PHDDEGREEFROM, LUBM_FIRST_UNIV_ID + h4(seed, u, d, TAG(T_FPHD, fi), 0) % P);
        if (r < 3) EMIT(id, LUBM_P_RESEARCHINTEREST, ri0 + h4(seed, u, d, TAG(T_RI, fi), 0) % LUBM_N_RESEARCH);
        if (fi == 0) EMIT(id, LUBM_P_HEADOF, did);
        for (uint32_t c = 0; c < L.nc[fi]; c++) EMIT(id, LUBM_P_TEACHEROF, b + L.off_course + L.cb[fi] + c);
        for (uint32_t c = 0; c < L.ng[fi]; c++) EMIT(id, LUBM_P_TEACHEROF, b + L.off_gcourse + L.gb[fi] + c);
      }
    for (uint32_t c = 0; c < L.ncourse; c++) {
      uint64_t e = L.off_course + c;
      EMIT(b + e, LUBM_P_TYPE, LUBM_C_COURSE);
      EMIT(b + e, LUBM_P_NAME, b + E + e);
    }
    for (uint32_t c = 0; c < L.ngcourse; c++) {
      uint64_t e = L.off_gcourse + c;
      EMIT(b + e, LUBM_P_TYPE, LUBM_C_GRADCOURSE);
      EMIT(b + e, LUBM_P_NAME, b + E + e);
    }
    for (uint32_t f = 0; f < L.F; f++)
      for (uint32_t j = 0; j < L.npub[f]; j++) {
        uint64_t e = L.off_pub + L.pb[f] + j;
        EMIT(b + e, LUBM_P_TYPE, LUBM_C_PUBLICATION);
        EMIT(b + e, LUBM_P_NAME, b + E + e);
        EMIT(b + e, LUBM_P_PUBAUTHOR, b + L.off_fac + f);
      }
    for (uint32_t i = 0; i < L.nug; i++) {
      uint64_t e = L.off_ug + i, id = b + e, pers = L.F + i;
      EMIT(id, LUBM_P_TYPE, LUBM_C_UGSTUDENT);
      EMIT(id, LUBM_P_NAME, b + E + e);
      EMIT(id, LUBM_P_EMAIL, b + 2 * E + 1 + pers);
      EMIT(id, LUBM_P_TELEPHONE, b + 2 * E + 1 + Pn + pers);
      EMIT(id, LUBM_P_MEMBEROF, did);
      uint32_t nt = uni(h4(seed, u, d, TAG(T_UG_NTAKE, i), 0), 2, 4), take[4];
      pick_distinct(seed, u, d, TAG(T_UG_TAKE, i), nt, L.ncourse, take);
      for (uint32_t t = 0; t < nt; t++) EMIT(id, LUBM_P_TAKESCOURSE, b + L.off_course + take[t]);
      if (h4(seed, u, d, TAG(T_UG_HASADV, i), 0) % 5 == 0) {
        uint32_t a = uni(h4(seed, u, d, TAG(T_UG_ADV, i), 0), 0, L.nprof - 1);
        EMIT(id, LUBM_P_ADVISOR, b + L.off_fac + a);
        adv_count[a]++;
        for (uint32_t t = 0; t < nt; t++)
          st->c5_j2 += (take[t] >= L.cb[a] && take[t] < L.cb[a] + L.nc[a]);
      }
    }
    for (uint32_t i = 0; i < L.ngrad; i++) {
      uint64_t e = L.off_grad + i, id = b + e, pers = L.F + L.nug + i;
      EMIT(id, LUBM_P_TYPE, LUBM_C_GRADSTUDENT);
      EMIT(id, LUBM_P_NAME, b + E + e);
      EMIT(id, LUBM_P_EMAIL, b + 2 * E + 1 + pers);
      EMIT(id, LUBM_P_TELEPHONE, b + 2 * E + 1 + Pn + pers);
      EMIT(id, LUBM_P_MEMBEROF, did);
      uint32_t ug = (uint32_t)(h4(seed, u, d, TAG(T_GR_UGDEG, i), 0) % P);
      EMIT(id, LUBM_P_UGDEGREEFROM, LUBM_FIRST_UNIV_ID + ug);
      st->c2_j2 += (ug == u);
      uint32_t nt = uni(h4(seed, u, d, TAG(T_GR_NTAKE, i), 0), 1, 3), take[4];
      pick_distinct(seed, u, d, TAG(T_GR_TAKE, i), nt, L.ngcourse, take);
      for (uint32_t t = 0; t < nt; t++) EMIT(id, LUBM_P_TAKESCOURSE, b + L.off_gcourse + take[t]);
      uint32_t a = uni(h4(seed, u, d, TAG(T_GR_ADV, i), 0), 0, L.nprof - 1);
      EMIT(id, LUBM_P_ADVISOR, b + L.off_fac + a);
      adv_count[a]++;
      for (uint32_t t = 0; t < nt; t++)
        st->c5_j2 += (take[t] >= L.gb[a] && take[t] < L.gb[a] + L.ng[a]);
      if (h4(seed, u, d, TAG(T_GR_HASTA, i), 0) % 4 == 0)
        EMIT(id, LUBM_P_TAOF, b + L.off_course + uni(h4(seed, u, d, TAG(T_GR_TA, i), 0), 0, L.ncourse - 1));
    }
    st->n_dept += 1;
    st->n_faculty += L.F;
    st->n_ug += L.nug;
    st->n_grad += L.ngrad;
    st->c1_rs += L.F;
    st->c2_j1 += (uint64_t)L.nug + L.ngrad;
    st->c3_j1 += 1;
    st->c3_j2 += L.F;
    st->c3_j3 += (uint64_t)L.F * ((uint64_t)L.nug + L.ngrad);
    for (uint32_t a = 0; a < L.F; a++) st->c5_j1 += (uint64_t)adv_count[a] * (L.nc[a] + L.ng[a]);
    b += L.nids;
  }
  st->n_triples += k;
  return k;
}

static void stats_add(lubm_stats *a, const lubm_stats *b) {
  uint64_t *x = (uint64_t *)a;
  const uint64_t *y = (const uint64_t *)b;
  for (size_t i = 0; i < sizeof(lubm_stats) / sizeof(uint64_t); i++) x[i] += y[i];
}

uint64_t lubm_univ_base(uint64_t seed, uint32_t n_univ_total, uint32_t u) {
  uint64_t base = id_base0(lubm_pool_size(n_univ_total));
  long long n = (long long)u;
#pragma omp parallel for reduction(+ : base) schedule(static)
  for (long long v = 0; v < n; v++) base += univ_ids(seed, (uint32_t)v);
  return base;
}

uint64_t lubm_id_end(uint64_t seed, uint32_t n_univ_total, uint32_t u_hi) {
  return lubm_univ_base(seed, n_univ_total, u_hi);
}

uint64_t lubm_count(uint64_t seed, uint32_t n_univ_total, uint32_t u_lo, uint32_t u_hi,
                    lubm_stats *stats) {
  const uint32_t P = lubm_pool_size(n_univ_total);
  lubm_stats tot;
  memset(&tot, 0, sizeof tot);
#pragma omp parallel
  {
    lubm_stats loc;
    memset(&loc, 0, sizeof loc);
#pragma omp for schedule(dynamic, 4)
    for (long long u = u_lo; u < (long long)u_hi; u++)
      emit_univ(seed, P, (uint32_t)u, 0, NULL, NULL, NULL, &loc);
#pragma omp critical
    stats_add(&tot, &loc);
  }
  if (stats) *stats = tot;
  return tot.n_triples;
}

uint64_t lubm_generate(uint64_t seed, uint32_t n_univ_total, uint32_t u_lo, uint32_t u_hi,
                       uint32_t *s, uint32_t *p, uint32_t *o, lubm_stats *stats) {
  const uint32_t P = lubm_pool_size(n_univ_total);
  const uint32_t nu = u_hi - u_lo;
  uint64_t *tcount = (uint64_t *)calloc((size_t)nu + 1, sizeof(uint64_t));
  uint64_t *ibase = (uint64_t *)calloc((size_t)nu + 1, sizeof(uint64_t));
  lubm_stats tot;
  memset(&tot, 0, sizeof tot);
  const uint64_t base_lo = lubm_univ_base(seed, n_univ_total, u_lo);
#pragma omp parallel
  {
    lubm_stats scratch;
    memset(&scratch, 0, sizeof scratch);
#pragma omp for schedule(dynamic, 4)
    for (long long i = 0; i < (long long)nu; i++) {
      tcount[i] = emit_univ(seed, P, u_lo + (uint32_t)i, 0, NULL, NULL, NULL, &scratch);
      ibase[i] = univ_ids(seed, u_lo + (uint32_t)i);
    }
  }
  /* exclusive prefix sums: triple offsets and ID bases per university */
  uint64_t t = 0, b = base_lo;
  for (uint32_t i = 0; i < nu; i++) {
    uint64_t tc = tcount[i], ic = ibase[i];
    tcount[i] = t; ibase[i] = b;
    t += tc; b += ic;
  }
  tcount[nu] = t;
#pragma omp parallel
  {
    lubm_stats loc;
    memset(&loc, 0, sizeof loc);
#pragma omp for schedule(dynamic, 4)
    for (long long i = 0; i < (long long)nu; i++) {
      uint64_t off = tcount[i];
      emit_univ(seed, P, u_lo + (uint32_t)i, ibase[i], s + off, p + off, o + off, &loc);
    }
#pragma omp critical
    stats_add(&tot, &loc);
  }
  free(tcount);
  free(ibase);
  if (stats) *stats = tot;
  return t;
}

/* ---------------- Zipf(s) by rejection-inversion (Hörmann & Derflinger 1996) ----------------
 * W. Hörmann, G. Derflinger, "Rejection-inversion to generate variates from monotone discrete
 * distributions", ACM TOMACS 6(3), 1996.  The formulation below (the helper1/helper2 series for
 * log1p(x)/x and expm1(x)/x near 0, H/H^-1 over [1.5, N + 0.5], the squeeze constant
 * s = 2 - H^-1(H(2.5) - h(2)) and the acceptance test) follows the structure of Apache Commons
 * Math's RejectionInversionZipfSampler (Apache License 2.0), re-implemented here in C with a
 * counter-based uniform per row so any row range is generated independently. */
static double zh(double x, double s) { return exp(-s * log(x)); }
static double zhelper1(double x) { return fabs(x) > 1e-8 ? log1p(x) / x : 1.0 - x * (0.5 - x * (1.0 / 3.0 - 0.25 * x)); }
static double zhelper2(double x) { return fabs(x) > 1e-8 ? expm1(x) / x : 1.0 + x * 0.5 * (1.0 + x * (1.0 / 3.0) * (1.0 + 0.25 * x)); }
static double zH(double x, double s) { double lx = log(x); return zhelper2((1.0 - s) * lx) * lx; }
static double zHinv(double x, double s) {
  double t = x * (1.0 - s);
  if (t < -1.0) t = -1.0;
  return exp(zhelper1(t) * x);
}

typedef struct { double s, N, hx1, hN, sp; } zipf_consts;
static zipf_consts zipf_init(double s, uint32_t kbits) {
  zipf_consts z;
  z.s = s;
  z.N = ldexp(1.0, (int)kbits);
  z.hx1 = zH(1.5, s) - 1.0;
  z.hN = zH(z.N + 0.5, s);
  z.sp = 2.0 - zHinv(zH(2.5, s) - zh(2.0, s), s);
  return z;
}
static uint64_t zipf_draw(const zipf_consts *z, uint64_t seed, int side, uint64_t i) {
  for (uint64_t t = 0;; t++) {
    double u01 = (double)(h4(seed, 0xC4C4u + (uint64_t)side, i, t, 0x21) >> 11) * 0x1.0p-53;
    double ux = z->hN + u01 * (z->hx1 - z->hN);
    double x = zHinv(ux, z->s);
    double kd = floor(x + 0.5);
    if (kd < 1.0) kd = 1.0;
    if (kd > z->N) kd = z->N;
    if (kd - x <= z->sp || ux >= zH(kd + 0.5, z->s) - zh(kd, z->s)) return (uint64_t)kd;
  }
}

uint64_t zipf_rank(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i) {
  zipf_consts z = zipf_init(s, kbits);
  return zipf_draw(&z, seed, side, i);
}

void zipf_table(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i_lo, uint64_t i_hi,
                uint32_t *key, uint32_t *val) {
  const uint64_t mask = (kbits >= 64) ? ~0ull : ((1ull << kbits) - 1);
  const uint64_t A = (h4(seed, 0xA0A0u + (uint64_t)side, 0, 0, 0) | 1ull) & mask;
  const uint64_t B = h4(seed, 0xB0B0u + (uint64_t)side, 0, 0, 0) & mask;
  const zipf_consts z = zipf_init(s, kbits);
  const long long n = (long long)(i_hi - i_lo);
#pragma omp parallel for schedule(static, 65536)
  for (long long j = 0; j < n; j++) {
    uint64_t i = i_lo + (uint64_t)j;
    uint64_t r = zipf_draw(&z, seed, side, i);
    if (key) key[j] = (uint32_t)((A * (r - 1) + B) & mask);
    if (val) val[j] = (uint32_t)(h4(seed, 0x7A7Au + (uint64_t)side, i, 0, 0x56) >> 32);
  }
}

void uniform_table(uint64_t seed, uint64_t n, uint32_t key_domain, uint32_t val_domain,
                   uint32_t *key, uint32_t *val) {
#pragma omp parallel for schedule(static, 65536)
  for (long long j = 0; j < (long long)n; j++) {
    if (key) key[j] = (uint32_t)(h4(seed, 0x0E0Eu, (uint64_t)j, 0, 1) % key_domain);
    if (val) val[j] = (uint32_t)(h4(seed, 0x0E0Eu, (uint64_t)j, 0, 2) % val_domain);
  }
}

int datagen_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
