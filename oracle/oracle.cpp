// oracle.cpp — plain, slow, single-threaded CPU oracle.  TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// Every function cites the passage it follows.  Nothing here is blocked, fused or reordered
// beyond the definition: scan is a linear filter, tier 0 is the nested loop, tier 1 groups rows
// by key with std::sort and emits each key's product.
#include "oracle.h"

#include <algorithm>
#include <array>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

namespace {

int alloc_rows(oracle_table *t, uint64_t nrows) {
  t->nrows = nrows;
  size_t bytes = (size_t)nrows * t->ncols * sizeof(uint32_t);
  t->rows = (uint32_t *)std::malloc(bytes ? bytes : 4);
  return t->rows ? ORACLE_OK : ORACLE_E_NOMEM;
}

// Join spec ("The key of them is their shared variable, and the value is other
// variables"; P:137-138 join only when patterns share variables; reading R5/R6 in DESIGN.md):
// shared = vars(A) ∩ vars(B) ascending by id; output = shared ++ A's rest ++ B's rest.
struct Spec {
  std::vector<int> a_key, b_key;     // column positions of the shared vars in A / B
  std::vector<int> a_rest, b_rest;   // non-shared column positions, in table order
};

int make_spec(const oracle_table *a, const oracle_table *b, oracle_table *out, Spec *sp) {
  if (a->ncols == 0 || b->ncols == 0 || a->ncols > ORACLE_MAX_COLS || b->ncols > ORACLE_MAX_COLS)
    return ORACLE_E_INVALID;
  std::vector<int> shared;
  for (uint32_t i = 0; i < a->ncols; i++)
    for (uint32_t j = 0; j < b->ncols; j++)
      if (a->var[i] == b->var[j]) shared.push_back(a->var[i]);
  if (shared.empty()) return ORACLE_E_NO_SHARED;
  std::sort(shared.begin(), shared.end());
  auto pos = [](const oracle_table *t, int v) {
    for (uint32_t c = 0; c < t->ncols; c++)
      if (t->var[c] == v) return (int)c;
    return -1;
  };
  for (int v : shared) {
    sp->a_key.push_back(pos(a, v));
    sp->b_key.push_back(pos(b, v));
  }
  for (uint32_t c = 0; c < a->ncols; c++)
    if (!std::binary_search(shared.begin(), shared.end(), a->var[c])) sp->a_rest.push_back((int)c);
  for (uint32_t c = 0; c < b->ncols; c++)
    if (!std::binary_search(shared.begin(), shared.end(), b->var[c])) sp->b_rest.push_back((int)c);
  uint32_t w = (uint32_t)(shared.size() + sp->a_rest.size() + sp->b_rest.size());
  if (w > ORACLE_MAX_COLS) return ORACLE_E_INVALID;
  out->ncols = w;
  int k = 0;
  for (int v : shared) out->var[k++] = v;
  for (int c : sp->a_rest) out->var[k++] = a->var[c];
  for (int c : sp->b_rest) out->var[k++] = b->var[c];
  return ORACLE_OK;
}

// One output row: μ1 ∪ μ2 written as key ++ A rest ++ B rest (RS = Key | value1, value2).
inline void emit(std::vector<uint32_t> &buf, const Spec &sp, const uint32_t *ra, const uint32_t *rb) {
  for (int c : sp.a_key) buf.push_back(ra[c]);
  for (int c : sp.a_rest) buf.push_back(ra[c]);
  for (int c : sp.b_rest) buf.push_back(rb[c]);
}

int finish(std::vector<uint32_t> &buf, oracle_table *out) {
  uint64_t nrows = out->ncols ? buf.size() / out->ncols : 0;
  if (alloc_rows(out, nrows) != ORACLE_OK) return ORACLE_E_NOMEM;
  if (!buf.empty()) std::memcpy(out->rows, buf.data(), buf.size() * sizeof(uint32_t));
  return ORACLE_OK;
}

// Tier 1: group both sides by the shared-variable key with std::sort (ties by row index),
// then for every key present on both sides emit the full |A_k| x |B_k| product in
// (A row, B row) order — the natural join grouped by key (reading R2 in DESIGN.md).
template <int C>
int sortmerge_fixed(const oracle_table *a, const oracle_table *b, const Spec &sp,
                    std::vector<uint32_t> &buf) {
  using Key = std::array<uint32_t, C>;
  auto keyed = [](const oracle_table *t, const std::vector<int> &kc) {
    std::vector<std::pair<Key, uint64_t>> v(t->nrows);
    for (uint64_t r = 0; r < t->nrows; r++) {
      for (int i = 0; i < C; i++) v[r].first[i] = t->rows[r * t->ncols + kc[i]];
      v[r].second = r;
    }
    std::sort(v.begin(), v.end());
    return v;
  };
  auto A = keyed(a, sp.a_key);
  auto B = keyed(b, sp.b_key);
  size_t i = 0, j = 0;
  while (i < A.size() && j < B.size()) {
    if (A[i].first < B[j].first) { i++; continue; }
    if (B[j].first < A[i].first) { j++; continue; }
    size_t i1 = i, j1 = j;
    while (i1 < A.size() && A[i1].first == A[i].first) i1++;
    while (j1 < B.size() && B[j1].first == B[j].first) j1++;
    for (size_t x = i; x < i1; x++)
      for (size_t y = j; y < j1; y++)
        emit(buf, sp, a->rows + A[x].second * a->ncols, b->rows + B[y].second * b->ncols);
    i = i1;
    j = j1;
  }
  return ORACLE_OK;
}

// Generic key width: sort row indices by the key columns (lexicographic), ties by index.
int sortmerge_generic(const oracle_table *a, const oracle_table *b, const Spec &sp,
                      std::vector<uint32_t> &buf) {
  auto order = [](const oracle_table *t, const std::vector<int> &kc) {
    std::vector<uint64_t> idx(t->nrows);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](uint64_t x, uint64_t y) {
      for (int c : kc) {
        uint32_t vx = t->rows[x * t->ncols + c], vy = t->rows[y * t->ncols + c];
        if (vx != vy) return vx < vy;
      }
      return x < y;
    });
    return idx;
  };
  auto cmp = [&](uint64_t ra, uint64_t rb) {  // -1, 0, 1 comparing A row key with B row key
    for (size_t i = 0; i < sp.a_key.size(); i++) {
      uint32_t va = a->rows[ra * a->ncols + sp.a_key[i]], vb = b->rows[rb * b->ncols + sp.b_key[i]];
      if (va != vb) return va < vb ? -1 : 1;
    }
    return 0;
  };
  auto A = order(a, sp.a_key);
  auto B = order(b, sp.b_key);
  size_t i = 0, j = 0;
  while (i < A.size() && j < B.size()) {
    int c = cmp(A[i], B[j]);
    if (c < 0) { i++; continue; }
    if (c > 0) { j++; continue; }
    size_t i1 = i, j1 = j;
    while (i1 < A.size() && cmp(A[i1], B[j]) == 0) i1++;
    while (j1 < B.size() && cmp(A[i], B[j1]) == 0) j1++;
    for (size_t x = i; x < i1; x++)
      for (size_t y = j; y < j1; y++)
        emit(buf, sp, a->rows + A[x] * a->ncols, b->rows + B[y] * b->ncols);
    i = i1;
    j = j1;
  }
  return ORACLE_OK;
}

}  // namespace

extern "C" {

// Partial matching of one triple pattern (SPEC S:162 semantics): a linear
// filter over all triples.  A constant position must equal the triple's term; a repeated
// variable must bind equal terms; the schema is the pattern's distinct variables in (s,p,o)
// order and rows keep triple order.  An absent constant simply matches nothing (reading R10).
int oracle_scan(uint64_t n, const uint32_t *s, const uint32_t *p, const uint32_t *o,
                const int32_t var[3], const uint32_t id[3], oracle_table *out) {
  std::memset(out, 0, sizeof *out);
  int pos_of_col[3];
  for (int j = 0; j < 3; j++) {
    if (var[j] < -1) return ORACLE_E_INVALID;
    if (var[j] < 0) continue;
    int found = -1;
    for (uint32_t c = 0; c < out->ncols; c++)
      if (out->var[c] == var[j]) found = (int)c;
    if (found < 0) {
      pos_of_col[out->ncols] = j;
      out->var[out->ncols++] = var[j];
    }
  }
  if (out->ncols == 0) return ORACLE_E_INVALID;
  std::vector<uint32_t> buf;
  for (uint64_t i = 0; i < n; i++) {
    const uint32_t t[3] = {s[i], p[i], o[i]};
    bool ok = true;
    for (int j = 0; j < 3 && ok; j++) {
      if (var[j] < 0) {
        ok = (t[j] == id[j]);
      } else {
        for (int q = 0; q < j; q++)
          if (var[q] == var[j] && t[q] != t[j]) ok = false;
      }
    }
    if (!ok) continue;
    for (uint32_t c = 0; c < out->ncols; c++) buf.push_back(t[pos_of_col[c]]);
  }
  return finish(buf, out);
}

// Tier 0: the nested-loop join, "plain join algorithms, such as nested-loop join":
// for every pair (a, b) that agrees on every shared variable, emit a ∪ b once (bag semantics).
int oracle_join_nested(const oracle_table *a, const oracle_table *b, oracle_table *out) {
  std::memset(out, 0, sizeof *out);
  Spec sp;
  int rc = make_spec(a, b, out, &sp);
  if (rc) return rc;
  std::vector<uint32_t> buf;
  for (uint64_t x = 0; x < a->nrows; x++) {
    const uint32_t *ra = a->rows + x * a->ncols;
    for (uint64_t y = 0; y < b->nrows; y++) {
      const uint32_t *rb = b->rows + y * b->ncols;
      bool eq = true;
      for (size_t k = 0; k < sp.a_key.size(); k++) eq = eq && (ra[sp.a_key[k]] == rb[sp.b_key[k]]);
      if (eq) emit(buf, sp, ra, rb);
    }
  }
  return finish(buf, out);
}

int oracle_join_sortmerge(const oracle_table *a, const oracle_table *b, oracle_table *out) {
  std::memset(out, 0, sizeof *out);
  Spec sp;
  int rc = make_spec(a, b, out, &sp);
  if (rc) return rc;
  std::vector<uint32_t> buf;
  switch (sp.a_key.size()) {
    case 1: rc = sortmerge_fixed<1>(a, b, sp, buf); break;
    case 2: rc = sortmerge_fixed<2>(a, b, sp, buf); break;
    case 3: rc = sortmerge_fixed<3>(a, b, sp, buf); break;
    default: rc = sortmerge_generic(a, b, sp, buf); break;
  }
  if (rc) return rc;
  return finish(buf, out);
}

// Query = "partial matching and MapReduce-based join": scan every pattern, fold the
// joins left-deep in the given order (each pattern must share a variable with the accumulated
// result, P:137-138 / reading R8-R9), then project (no dedup, reading R3).
int oracle_query(uint64_t n, const uint32_t *s, const uint32_t *p, const uint32_t *o,
                 const int32_t *pat_var, const uint32_t *pat_id, int npats, const int32_t *proj,
                 int nproj, oracle_table *out) {
  std::memset(out, 0, sizeof *out);
  if (npats <= 0) return ORACLE_E_INVALID;
  std::vector<int32_t> order;  // first-appearance order of the variables
  for (int i = 0; i < npats; i++)
    for (int j = 0; j < 3; j++) {
      int32_t v = pat_var[3 * i + j];
      if (v >= 0 && std::find(order.begin(), order.end(), v) == order.end()) order.push_back(v);
    }
  std::vector<int32_t> want(proj, proj + nproj);
  if (nproj == 0) want = order;
  for (int32_t v : want)
    if (std::find(order.begin(), order.end(), v) == order.end()) return ORACLE_E_INVALID;
  if (want.size() > ORACLE_MAX_COLS) return ORACLE_E_INVALID;

  oracle_table acc;
  int rc = oracle_scan(n, s, p, o, pat_var, pat_id, &acc);
  if (rc) return rc;
  for (int i = 1; i < npats; i++) {
    oracle_table t, r;
    rc = oracle_scan(n, s, p, o, pat_var + 3 * i, pat_id + 3 * i, &t);
    if (rc) { oracle_free(&acc); return rc; }
    rc = oracle_join_sortmerge(&acc, &t, &r);
    oracle_free(&t);
    oracle_free(&acc);
    if (rc) return rc;
    acc = r;
  }
  out->ncols = (uint32_t)want.size();
  std::vector<int> src;
  for (uint32_t c = 0; c < out->ncols; c++) {
    out->var[c] = want[c];
    for (uint32_t k = 0; k < acc.ncols; k++)
      if (acc.var[k] == want[c]) src.push_back((int)k);
  }
  if (alloc_rows(out, acc.nrows)) { oracle_free(&acc); return ORACLE_E_NOMEM; }
  for (uint64_t r = 0; r < acc.nrows; r++)
    for (uint32_t c = 0; c < out->ncols; c++)
      out->rows[r * out->ncols + c] = acc.rows[r * acc.ncols + src[c]];
  oracle_free(&acc);
  return ORACLE_OK;
}

void oracle_canonical_sort(oracle_table *t) {
  const uint32_t w = t->ncols;
  if (t->nrows < 2 || w == 0) return;
  std::vector<uint64_t> idx(t->nrows);
  std::iota(idx.begin(), idx.end(), 0);
  const uint32_t *rows = t->rows;
  std::sort(idx.begin(), idx.end(), [&](uint64_t x, uint64_t y) {
    return std::lexicographical_compare(rows + x * w, rows + x * w + w, rows + y * w, rows + y * w + w);
  });
  std::vector<uint32_t> tmp((size_t)t->nrows * w);
  for (uint64_t r = 0; r < t->nrows; r++)
    std::memcpy(tmp.data() + r * w, rows + idx[r] * w, w * sizeof(uint32_t));
  std::memcpy(t->rows, tmp.data(), tmp.size() * sizeof(uint32_t));
}

// Whole-output multiset fingerprint: parity of outputs too large to sort
// and compare on the host is judged on (row count, sum mod 2^64, xor) of a per-row hash.  Both
// reductions are order-independent, so the fingerprint is a function of the multiset of rows.
// Row hash: h = 0; for each column value v in order: h = splitmix64_step(h ^ v), where
// splitmix64_step(x) is one output of Steele et al.'s splitmix64 generator from state x
// (add the golden gamma 0x9E3779B97F4A7C15, then the 30/27/31 xor-shift-multiply finaliser).
// This is test infrastructure: it hashes rows, it computes nothing of the join.
static inline uint64_t fp_step(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

void oracle_fingerprint(const oracle_table *t, uint64_t acc[3]) {
  for (uint64_t r = 0; r < t->nrows; r++) {
    uint64_t h = 0;
    for (uint32_t c = 0; c < t->ncols; c++) h = fp_step(h ^ t->rows[r * t->ncols + c]);
    acc[0] += 1;
    acc[1] += h;
    acc[2] ^= h;
  }
}

void oracle_fingerprint_cols(uint64_t nrows, uint32_t ncols, const uint32_t *const *cols,
                             uint64_t acc[3]) {
  for (uint64_t r = 0; r < nrows; r++) {
    uint64_t h = 0;
    for (uint32_t c = 0; c < ncols; c++) h = fp_step(h ^ cols[c][r]);
    acc[0] += 1;
    acc[1] += h;
    acc[2] ^= h;
  }
}

void oracle_free(oracle_table *t) {
  std::free(t->rows);
  t->rows = nullptr;
  t->nrows = 0;
}

}  // extern "C"
