// api.cu — host orchestration and the C ABI of libmapsq (include/mapsq.h).
//
// The host side plays the paper's CPU role, "CPU is used to assigns subqueries and GPU is used
// to compute the join of subqueries": it validates the plan, derives each join's
// spec (shared variables, key packing), sizes buffers after the single blocking count read of
// each operator, and folds the joins left-deep.  All data-path work runs in
// the kernels of scan.cu / radix.cu / reduce.cu / partition.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <set>
#include <utility>

#include "internal.cuh"

#include <memory>

using namespace mapsq;

namespace mapsq {

mapsq_status set_error(mapsq_ctx *ctx, mapsq_status st, const std::string &msg) {
  if (ctx) ctx->err = msg;
  return st;
}

mapsq_status cuda_check(mapsq_ctx *ctx, cudaError_t e, const char *what) {
  if (e == cudaSuccess) return MAPSQ_OK;
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    return set_error(ctx, MAPSQ_E_NOMEM, std::string(what) + ": " + cudaGetErrorString(e));
  }
  if (ctx) ctx->cuda_broken = true;
  return set_error(ctx, MAPSQ_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

void *dalloc(mapsq_ctx *ctx, size_t bytes, cudaStream_t s) {
  if (bytes == 0) bytes = 16;
  bytes = (bytes + 255) & ~size_t(255);
  if (ctx->custom_alloc) return ctx->alloc.alloc(ctx->alloc.ctx, bytes, (void *)s);
  void *p = nullptr;
  if (cudaMallocAsync(&p, bytes, s) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return p;
}

void dfree(mapsq_ctx *ctx, void *p, cudaStream_t s) {
  if (!p) return;
  if (ctx->custom_alloc)
    ctx->alloc.free(ctx->alloc.ctx, p, (void *)s);
  else
    cudaFreeAsync(p, s);
}

void set_smem_limit(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::set<std::pair<int, const void *>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({dev, kernel}).second)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

Scratch::Scratch(mapsq_ctx *c, cudaStream_t st) : ctx(c), s(st), mark(c->arena_used) {
  if (ctx->arena_depth++ == 0) {
    ctx->arena_demand = 0;
    if (ctx->arena && ctx->arena_stream != s && ctx->arena_ev)
      cudaStreamWaitEvent(s, ctx->arena_ev, 0);  // previous user of the arena on another stream
    if (!ctx->custom_alloc && ctx->arena_hw > ctx->arena_cap) {
      if (ctx->arena) cudaFreeAsync(ctx->arena, s);
      ctx->arena = nullptr;
      ctx->arena_cap = 0;
      const size_t want = (ctx->arena_hw + ctx->arena_hw / 8 + 4095) & ~size_t(4095);
      void *p = nullptr;
      if (cudaMallocAsync(&p, want, s) == cudaSuccess) {
        ctx->arena = static_cast<char *>(p);
        ctx->arena_cap = want;
      } else {
        cudaGetLastError();
      }
    }
    ctx->arena_used = 0;
    mark = 0;
  }
}

Scratch::~Scratch() {
  for (void *p : ptrs) dfree(ctx, p, s);
  ctx->arena_used = mark;
  if (--ctx->arena_depth == 0) {
    ctx->arena_hw = std::max(ctx->arena_hw, ctx->arena_demand);
    if (!ctx->arena_ev) cudaEventCreateWithFlags(&ctx->arena_ev, cudaEventDisableTiming);
    cudaEventRecord(ctx->arena_ev, s);
    ctx->arena_stream = s;
  }
}

void *Scratch::raw(size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  ctx->arena_demand += bytes;
  if (ctx->arena && ctx->arena_used + bytes <= ctx->arena_cap) {
    void *p = ctx->arena + ctx->arena_used;
    ctx->arena_used += bytes;
    return p;
  }
  void *p = dalloc(ctx, bytes, s);
  if (p) ptrs.push_back(p);
  return p;
}

KTimer::KTimer(mapsq_ctx *c, cudaStream_t st, const char *name, uint64_t bytes, int nlaunch)
    : ctx(c), s(st), on(c->profiling) {
  ctx->counters.launches += nlaunch;
  if (!on) return;
  t.name = name;
  t.bytes = bytes;
  for (cudaEvent_t *e : {&t.ev0, &t.ev1}) {
    if (!ctx->free_events.empty()) {
      *e = ctx->free_events.back();
      ctx->free_events.pop_back();
    } else {
      cudaEventCreate(e);
    }
  }
  cudaEventRecord(t.ev0, s);
}

KTimer::~KTimer() {
  if (!on) return;
  cudaEventRecord(t.ev1, s);
  ctx->pending.push_back(t);
}

}  // namespace mapsq

namespace {

#define TRY(x)                                  \
  do {                                          \
    mapsq_status _st = (x);                     \
    if (_st != MAPSQ_OK) return _st;            \
  } while (0)
#define CK(call)                                \
  do {                                          \
    cudaError_t _e = (call);                    \
    if (_e != cudaSuccess) return cuda_check(ctx, _e, #call); \
  } while (0)
#define CKL(what) CK(cudaGetLastError())
#define NEED(ptr)                                                                  \
  do {                                                                             \
    if (!(ptr)) return set_error(ctx, MAPSQ_E_NOMEM, "device allocation failed"); \
  } while (0)

inline cudaStream_t S(void *stream) { return (cudaStream_t)stream; }

mapsq_status enter(mapsq_ctx *ctx) {
  if (!ctx) return MAPSQ_E_INVALID;
  if (ctx->cuda_broken) return MAPSQ_E_CUDA;
  int cur = -1;
  cudaGetDevice(&cur);
  if (cur != ctx->device) CK(cudaSetDevice(ctx->device));
  return MAPSQ_OK;
}

mapsq_status ensure_pinned(mapsq_ctx *ctx, size_t words) {
  if (ctx->pinned_words >= words) return MAPSQ_OK;
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  ctx->pinned = nullptr;
  size_t w = std::max<size_t>(words, 256);
  CK(cudaMallocHost((void **)&ctx->pinned, w * sizeof(uint64_t)));
  ctx->pinned_words = w;
  return MAPSQ_OK;
}

void clear_table(mapsq_table *t) {
  std::memset(t, 0, sizeof *t);
}

mapsq_status check_table(mapsq_ctx *ctx, const mapsq_table *t, const char *name) {
  if (!t) return set_error(ctx, MAPSQ_E_INVALID, std::string(name) + " is NULL");
  if (t->ncols == 0 || t->ncols > MAPSQ_MAX_COLS)
    return set_error(ctx, MAPSQ_E_INVALID, std::string(name) + ": ncols out of range");
  for (uint32_t i = 0; i < t->ncols; i++) {
    if (t->var[i] < 0) return set_error(ctx, MAPSQ_E_INVALID, std::string(name) + ": negative var id");
    if (t->nrows && !t->col[i]) return set_error(ctx, MAPSQ_E_INVALID, std::string(name) + ": NULL column");
    for (uint32_t j = 0; j < i; j++)
      if (t->var[i] == t->var[j])
        return set_error(ctx, MAPSQ_E_INVALID, std::string(name) + ": duplicate variable");
  }
  return MAPSQ_OK;
}

// Allocate a table of `rows` x `ncols` as one allocation with 16 B aligned column strides.
mapsq_status alloc_table(mapsq_ctx *ctx, mapsq_table *t, uint64_t rows, uint32_t ncols,
                         cudaStream_t s) {
  t->nrows = rows;
  t->ncols = ncols;
  t->owner = nullptr;
  if (rows == 0) {
    for (uint32_t c = 0; c < ncols; c++) t->col[c] = nullptr;
    return MAPSQ_OK;
  }
  const uint64_t stride = (rows + 3) & ~3ull;
  void *p = dalloc(ctx, stride * ncols * sizeof(uint32_t), s);
  if (!p) return set_error(ctx, MAPSQ_E_NOMEM, "output allocation failed");
  t->owner = p;
  for (uint32_t c = 0; c < ncols; c++) t->col[c] = static_cast<uint32_t *>(p) + c * stride;
  return MAPSQ_OK;
}

// ------------------------------------------------------------------------------ join plan
mapsq_status plan_join(mapsq_ctx *ctx, const mapsq_table *a, const mapsq_table *b,
                       mapsq_join_plan *pl, int wide_mode = MAPSQ_WIDE_KEY_HASH) {
  std::memset(pl, 0, sizeof *pl);
  TRY(check_table(ctx, a, "tp1"));
  TRY(check_table(ctx, b, "tp2"));
  if (!(a->flags & MAPSQ_TABLE_BOUNDS) || !(b->flags & MAPSQ_TABLE_BOUNDS))
    return set_error(ctx, MAPSQ_E_INVALID, "plan_join needs column bounds on both tables");
  pl->n1 = a->nrows;
  pl->n2 = b->nrows;
  if (a->nrows + b->nrows >= (1ull << 32))
    return set_error(ctx, MAPSQ_E_INVALID, "n1 + n2 must be < 2^32 per join per GPU");
  // shared variables, ascending id (reading R5/R6)
  int32_t sh[MAPSQ_MAX_COLS];
  uint32_t ns = 0;
  for (uint32_t i = 0; i < a->ncols; i++)
    for (uint32_t j = 0; j < b->ncols; j++)
      if (a->var[i] == b->var[j]) sh[ns++] = a->var[i];
  if (ns == 0) return set_error(ctx, MAPSQ_E_NO_SHARED, "join inputs share no variable");
  std::sort(sh, sh + ns);
  pl->nshared = ns;
  auto colof = [](const mapsq_table *t, int32_t v) {
    for (uint32_t c = 0; c < t->ncols; c++)
      if (t->var[c] == v) return (int32_t)c;
    return (int32_t)-1;
  };
  auto is_shared = [&](int32_t v) { return std::binary_search(sh, sh + ns, v); };
  for (uint32_t c = 0; c < a->ncols; c++)
    if (!is_shared(a->var[c])) pl->rest_col1[pl->nrest1++] = (int32_t)c;
  for (uint32_t c = 0; c < b->ncols; c++)
    if (!is_shared(b->var[c])) pl->rest_col2[pl->nrest2++] = (int32_t)c;
  pl->out_ncols = ns + pl->nrest1 + pl->nrest2;
  if (pl->out_ncols > MAPSQ_MAX_COLS)
    return set_error(ctx, MAPSQ_E_INVALID, "join output wider than MAPSQ_MAX_COLS");
  uint32_t k = 0;
  for (uint32_t c = 0; c < ns; c++) pl->out_var[k++] = sh[c];
  for (uint32_t c = 0; c < pl->nrest1; c++) pl->out_var[k++] = a->var[pl->rest_col1[c]];
  for (uint32_t c = 0; c < pl->nrest2; c++) pl->out_var[k++] = b->var[pl->rest_col2[c]];
  // key packing over the UNION of both sides' bounds (every row stays representable); the
  // output's key bounds are the intersection
  uint32_t kb_all = 0;
  for (uint32_t c = 0; c < ns; c++) {
    pl->shared[c] = sh[c];
    const int32_t ca = colof(a, sh[c]), cb = colof(b, sh[c]);
    pl->key_col1[c] = ca;
    pl->key_col2[c] = cb;
    const uint32_t ulo = std::min(a->lo[ca], b->lo[cb]), uhi = std::max(a->hi[ca], b->hi[cb]);
    pl->key_lo[c] = ulo;
    pl->key_hi[c] = uhi;
    pl->key_bits[c] = bits_for((uint64_t)uhi - ulo);
    kb_all += pl->key_bits[c];
    if (std::max(a->lo[ca], b->lo[cb]) > std::min(a->hi[ca], b->hi[cb])) pl->disjoint = 1;
  }
  const uint64_t n = a->nrows + b->nrows;
  pl->ib = n > 1 ? bits_for(n - 1) : 1;
  uint32_t packed = (ns >= 32) ? ~0u : ((1u << ns) - 1u);
  if (wide_mode == MAPSQ_WIDE_KEY_HASH && (kb_all + pl->ib > 64 || kb_all > 32)) {
    // HASH: key' = the top min(32, 64 - ib) bits of a 64-bit mix of every shared column (at most
    // 4 digit passes however wide the key); ReduceDuplicate verifies each pair's columns
    pl->path = MAPSQ_PATH_HASH;
    pl->packed_mask = 0;
    pl->kb = std::min<uint32_t>(32, 64 - pl->ib);
    pl->passes = (pl->kb + MAPSQ_RADIX_BITS - 1) / MAPSQ_RADIX_BITS;
    for (uint32_t c = 0; c < ns; c++) pl->key_shift[c] = 0;
    return MAPSQ_OK;
  }
  if (kb_all + pl->ib <= 64) {
    pl->path = MAPSQ_PATH_P64;
  } else if (wide_mode == MAPSQ_WIDE_KEY_KV) {
    if (kb_all > 64) return set_error(ctx, MAPSQ_E_UNSUPPORTED, "packed join key wider than 64 bits");
    pl->path = MAPSQ_PATH_KV;
  } else {
    // RESIDUAL: pack the widest shared columns that fit 64 - ib bits (ties: lower var id first);
    // the rest are compared exactly inside each packed-key group
    uint32_t order[MAPSQ_MAX_COLS];
    for (uint32_t c = 0; c < ns; c++) order[c] = c;
    std::stable_sort(order, order + ns,
                     [&](uint32_t x, uint32_t y) { return pl->key_bits[x] > pl->key_bits[y]; });
    packed = 0;
    uint32_t used = 0;
    for (uint32_t q = 0; q < ns; q++) {
      const uint32_t c = order[q];
      if (used + pl->key_bits[c] + pl->ib <= 64) {
        packed |= 1u << c;
        used += pl->key_bits[c];
      }
    }
    pl->path = MAPSQ_PATH_RESIDUAL;
  }
  pl->packed_mask = packed;
  uint32_t kb = 0, sft = 0;
  for (int c = (int)ns - 1; c >= 0; c--) {  // first packed shared variable most significant
    if (!(packed >> c & 1u)) {
      pl->key_shift[c] = 0;
      continue;
    }
    pl->key_shift[c] = sft;
    sft += pl->key_bits[c];
    kb += pl->key_bits[c];
  }
  pl->kb = kb;
  pl->passes = (kb + MAPSQ_RADIX_BITS - 1) / MAPSQ_RADIX_BITS;
  return MAPSQ_OK;
}

mapsq_status bounds_of(mapsq_ctx *ctx, mapsq_table *t, cudaStream_t s) {
  if (t->flags & MAPSQ_TABLE_BOUNDS) return MAPSQ_OK;
  if (t->nrows == 0) {
    for (uint32_t c = 0; c < t->ncols; c++) t->lo[c] = t->hi[c] = 0;
    t->flags |= MAPSQ_TABLE_BOUNDS;
    return MAPSQ_OK;
  }
  Scratch sc(ctx, s);
  uint32_t *b = sc.get<uint32_t>(2 * t->ncols);
  NEED(b);
  for (uint32_t c = 0; c < t->ncols; c++) {
    CK(cudaMemsetAsync(b + 2 * c, 0xff, 4, s));
    CK(cudaMemsetAsync(b + 2 * c + 1, 0, 4, s));
  }
  {
    KTimer kt(ctx, s, "minmax", t->nrows * 4ull * t->ncols, (int)t->ncols);
    launch_minmax(t->col, t->ncols, t->nrows, b, s);
    CKL("minmax");
  }
  TRY(ensure_pinned(ctx, t->ncols));
  CK(cudaMemcpyAsync(ctx->pinned, b, 8 * t->ncols, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint32_t *h = reinterpret_cast<const uint32_t *>(ctx->pinned);
  for (uint32_t c = 0; c < t->ncols; c++) {
    t->lo[c] = h[2 * c];
    t->hi[c] = h[2 * c + 1];
  }
  t->flags |= MAPSQ_TABLE_BOUNDS;
  return MAPSQ_OK;
}

// ------------------------------------------------------------------------------ sort driver
// Stable LSD sort of keys (and optional vals) by `passes` 8-bit digits starting at bit_lo, the
// digit histograms `hist` (passes x 256, exclusive-scanned) already built.  a/b are ping-pong
// buffers; returns in *which the buffer (0 = a, 1 = b) holding the result.  (n0, gap): the input
// in ka is two segments — key i >= n0 sits at ka[i + gap] (the semi-join filter's output); the
// first pass reads both and writes one contiguous array.
mapsq_status radix_sort(mapsq_ctx *ctx, uint64_t *ka, uint64_t *kb_, uint32_t *va, uint32_t *vb,
                        uint64_t n, uint32_t bit_lo, uint32_t nbits, uint32_t *hist, Scratch &sc,
                        cudaStream_t s, int *which, uint64_t n0 = ~0ull, uint64_t gap = 0) {
  *which = 0;
  const uint32_t passes = (nbits + 7) / 8;
  if (gap && n0 < n && (passes == 0 || va))
    return set_error(ctx, MAPSQ_E_INVALID, "internal: a two-segment sort input needs a P64 pass");
  if (passes == 0 || n == 0) return MAPSQ_OK;
  const uint64_t ntiles = ceil_div(n, kSortTile);
  uint64_t *status = sc.get<uint64_t>(ntiles * kRadix);
  uint32_t *counters = sc.get<uint32_t>(kMaxPasses);
  NEED(status);
  NEED(counters);
  CK(cudaMemsetAsync(counters, 0, kMaxPasses * sizeof(uint32_t), s));
  const uint64_t bytes = n * (va ? 24ull : 16ull);
  for (uint32_t p = 0; p < passes; p++) {
    const uint32_t shift = bit_lo + 8 * p;
    const uint32_t bits = std::min<uint32_t>(8, nbits - 8 * p);
    CK(cudaMemsetAsync(status, 0, ntiles * kRadix * sizeof(uint64_t), s));
    uint64_t *kin = (*which == 0) ? ka : kb_, *kout = (*which == 0) ? kb_ : ka;
    uint32_t *vin = va ? ((*which == 0) ? va : vb) : nullptr;
    uint32_t *vout = va ? ((*which == 0) ? vb : va) : nullptr;
    {
      KTimer kt(ctx, s, va ? "radix_pass_kv" : "radix_pass", bytes);
      const bool more = p + 1 < passes;
      const uint32_t nbits_next = more ? std::min<uint32_t>(8, nbits - 8 * (p + 1)) : 0;
      launch_radix_pass(kin, kout, vin, vout, n, shift, bits, hist + p * kRadix, status,
                        counters + p, more ? hist + (p + 1) * kRadix : nullptr, shift + 8,
                        nbits_next, s, p == 0 ? n0 : ~0ull, p == 0 ? gap : 0);
      CKL("radix_pass");
    }
    *which ^= 1;
  }
  return MAPSQ_OK;
}

void fill_empty_join(const mapsq_join_plan &pl, const mapsq_table *a, const mapsq_table *b,
                     mapsq_table *rs);

// Output bounds: key columns get the intersection, the rest inherit their source's bounds.
void set_join_bounds(const mapsq_join_plan &pl, const mapsq_table *a, const mapsq_table *b,
                     mapsq_table *rs) {
  rs->flags = MAPSQ_TABLE_BOUNDS;
  uint32_t k = 0;
  for (uint32_t c = 0; c < pl.nshared; c++, k++) {
    rs->lo[k] = std::max(a->lo[pl.key_col1[c]], b->lo[pl.key_col2[c]]);
    rs->hi[k] = std::min(a->hi[pl.key_col1[c]], b->hi[pl.key_col2[c]]);
    if (rs->lo[k] > rs->hi[k]) rs->lo[k] = rs->hi[k] = 0;
  }
  for (uint32_t c = 0; c < pl.nrest1; c++, k++) {
    rs->lo[k] = a->lo[pl.rest_col1[c]];
    rs->hi[k] = a->hi[pl.rest_col1[c]];
  }
  for (uint32_t c = 0; c < pl.nrest2; c++, k++) {
    rs->lo[k] = b->lo[pl.rest_col2[c]];
    rs->hi[k] = b->hi[pl.rest_col2[c]];
  }
}

void fill_empty_join(const mapsq_join_plan &pl, const mapsq_table *a, const mapsq_table *b,
                     mapsq_table *rs) {
  clear_table(rs);
  rs->ncols = pl.out_ncols;
  for (uint32_t c = 0; c < pl.out_ncols; c++) rs->var[c] = pl.out_var[c];
  set_join_bounds(pl, a, b, rs);
}

PackArgs pack_args(const mapsq_join_plan &pl, const mapsq_table *a, const mapsq_table *b) {
  PackArgs pa;
  std::memset(&pa, 0, sizeof pa);
  const bool hash = pl.path == MAPSQ_PATH_HASH;
  for (uint32_t c = 0; c < pl.nshared; c++) {
    if (!hash && !(pl.packed_mask >> c & 1u)) continue;
    pa.key1[pa.nkey] = a->col[pl.key_col1[c]];
    pa.key2[pa.nkey] = b->col[pl.key_col2[c]];
    pa.lo[pa.nkey] = pl.key_lo[c];
    pa.shift[pa.nkey] = pl.key_shift[c];
    pa.nkey++;
  }
  pa.n1 = pl.n1;
  pa.n2 = pl.n2;
  pa.ib = pl.ib;
  pa.kb = pl.kb;
  pa.hash = hash;
  pa.kv = pl.path == MAPSQ_PATH_KV;
  pa.bit_lo = pa.kv ? 0 : pl.ib;
  // the Map kernel counts only the first digit; each digit pass counts the next one (measured
  // on C4: Map 2.5 ms vs 3.2 ms with every digit counted up front, digit passes unchanged)
  pa.passes = pl.passes ? 1 : 0;
  pa.last_mask = pl.passes == 1 ? ((1u << pl.kb) - 1u) : 0xffu;
  return pa;
}

// filter rounds with hashed bitmaps: ~8 bits per key of the smaller side (at most 2^29 bits, so
// one bitmap stays L2-resident) and a fresh seed per round
// MAPSQ_DEBUG=1 in the environment: per-join diagnostics on stderr (filter rounds)
bool debug_on() {
  static const bool on = [] {
    const char *e = std::getenv("MAPSQ_DEBUG");
    return e && *e && *e != '0';
  }();
  return on;
}

// developer knobs for ablations (read once): MAPSQ_SJ_COLBITS caps the hashed column round's bitmaps
uint32_t env_u32(const char *name, uint32_t dflt) {
  const char *e = std::getenv(name);
  return (e && *e) ? (uint32_t)std::strtoul(e, nullptr, 10) : dflt;
}

// Tp2 streaming in (ctx->stream_b, mapsq_query_host_indexed): s waits until rows [0, rows) of it
// are in place (the chunk holding row rows - 1; the copy stream lands chunks in order)
mapsq_status wait_stream_b(mapsq_ctx *ctx, uint64_t rows, cudaStream_t s) {
  const StreamIn *sb = ctx->stream_b;
  if (!sb || sb->ev.empty() || rows == 0) return MAPSQ_OK;
  const uint64_t k = std::min<uint64_t>((rows - 1) / sb->chunk_rows, sb->ev.size() - 1);
  return cuda_check(ctx, cudaStreamWaitEvent(s, sb->ev[k], 0), "stream wait");
}

uint32_t word_round_bits(uint64_t small) {
  const uint32_t b = bits_for(8 * std::max<uint64_t>(small, 1));
  return std::max<uint32_t>(16, std::min<uint32_t>(kSemijoinBits, b));
}
uint64_t word_round_seed(int round) { return 0x632BE59BD9B4E019ull * (uint64_t)(round + 1); }

// Semi-join filter in front of the Map (row f2's reducer, reading R18).  Leaves the
// surviving words key' << ib | rowid in cur as two segments — side A's at cur[0, *nA), side B's
// at cur[*offB, *offB + *nB) — each in row order, with their first radix digit counted into hist;
// alt is free for the sort.  cur/alt may be replaced.  A round: probe the larger side L against
// the smaller side's bitmap (survivors staged per 512-row slice in the stage buffer), scan its
// slice counts and gather its survivors into their segment, set bm_L from those words, then the
// same for the smaller side against bm_L; one blocking read of the two survivor counts.
// carry[side] (n, src set by the caller): columns to carry through the column round (SjCarry);
// on return carry[side].n is 0 unless they were carried (out[] then holds the side's survivors'
// values, allocated from sc, and the words' row ids index them).
// Value-carrying words (carry[side].pv): the column round's gathers write them from the staged
// row-id words (both sides), every other Map writes them directly.
mapsq_status filter_map(mapsq_ctx *ctx, mapsq_join_plan &pl, const mapsq_table *a,
                        const mapsq_table *b, Scratch &sc, cudaStream_t s, uint64_t *&cur,
                        uint64_t *&alt, uint32_t *hist, uint64_t *nA_out, uint64_t *offB_out,
                        uint64_t *nB_out, SjCarry carry[2], uint32_t ib_row) {
  const uint64_t n1 = pl.n1, n2 = pl.n2, n = n1 + n2;
  bool pv = carry[0].pv;
  PackArgs pa = pack_args(pl, a, b);
  // value-carrying words come only from the column round's gathers: a filter that Maps every
  // row (composite packed keys, or a skipped filter) uses row-id words (measured: the Map that
  // loads the values too ran 0.27-0.33 vs 0.17 ms on C5 J1, more than the expansion saves)
  auto pv_off = [&] {
    if (!pv) return;
    pv = false;
    pl.ib = ib_row;
    pa = pack_args(pl, a, b);
  };
  const uint64_t bmw = std::max<uint64_t>(
      1, (1ull << std::max(kSemijoinBits, env_u32("MAPSQ_SJ_COLBITS", kSemijoinBits))) / 32);
  const uint64_t nsl_max = sj_slices(n1) + sj_slices(n2) + 2;
  uint32_t *bm = sc.get<uint32_t>(2 * bmw);
  uint32_t *cnt = sc.get<uint32_t>(nsl_max);
  uint64_t *off = sc.get<uint64_t>(nsl_max);
  uint64_t *ftmp = sc.get<uint64_t>(scan_tmp_words(nsl_max));
  uint64_t *fsc = sc.get<uint64_t>(4);  // [0] / [1] survivors of side A / B, [2..3] sample
  NEED(bm); NEED(cnt); NEED(off); NEED(ftmp); NEED(fsc);
  unsigned long long *sample = reinterpret_cast<unsigned long long *>(fsc + 2);
  uint64_t *stage = alt;       // survivors staged per slice (free again when the filter ends)
  uint64_t *spare = nullptr;   // the word rounds' output buffer (allocated on first use)
  const uint32_t dmask = pa.last_mask;
  uint64_t nA = n1, offB = n1, nB = n2, nw = n;  // the current segments (in cur)
  bool exact = false;    // the last round's bitmaps were exact (no false positives)
  bool skipped = false;  // the sampled probe said the filter would drop < 10%
  // after building the smaller side's bitmap, a sample of the larger side (every 16th 512-row
  // slice, at most ~4 M rows) is probed; if >= 90% of it survives the filter cannot pay (C5 J1
  // drops 6%) and the join goes unfiltered
  auto sample_says_skip = [&](bool *skip) -> mapsq_status {
    TRY(ensure_pinned(ctx, 2));
    CK(cudaMemcpyAsync(ctx->pinned, sample, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t surv = ctx->pinned[0], rows = ctx->pinned[1];
    *skip = ctx->semijoin == MAPSQ_SEMIJOIN_AUTO && rows > 0 && surv * 10 >= rows * 9;
    return MAPSQ_OK;
  };
  auto pending_pos = [&]() -> size_t { return ctx->profiling ? ctx->pending.size() - 1 : ~size_t(0); };
  auto add_bytes = [&](size_t pos, uint64_t bytes) {
    if (pos < ctx->pending.size()) ctx->pending[pos].bytes += bytes;
  };
  // scan one side's slice counts (slices [sl0, sl0 + nsl)) and gather its staged survivors to
  // out; fsc[side] receives their number
  std::vector<size_t> gpos;
  const SjCarry none{};
  const SjCarry use[2] = {carry[0], carry[1]};  // (n cleared below unless the column round carries)
  carry[0].n = carry[1].n = 0;
  auto scan_gather = [&](int side, uint64_t sl0, uint64_t nsl, uint64_t *out,
                         const SjCarry &cr = SjCarry{}) -> mapsq_status {
    {
      KTimer kt(ctx, s, "filter_scan", 12ull * nsl);
      launch_exclusive_scan_u32(cnt + sl0, off + sl0, nsl, ftmp, fsc + side, s);
      CKL("filter_scan");
    }
    {
      KTimer kt(ctx, s, "filter_gather", 12ull * nsl);
      launch_sj_gather(stage + sl0 * kSjSlice, cnt + sl0, off + sl0, nsl, out,
                       pl.passes ? hist : nullptr, pl.ib, dmask, cr, pl.ib, side ? n1 : 0, s);
      CKL("filter_gather");
    }
    gpos.push_back(pending_pos());
    return MAPSQ_OK;
  };
  // the round's one blocking read: both sides' survivors; the staged / gathered bytes go to the
  // probe and gather timers
  // (ncL / ncS: columns carried by L / S — 4 B read + 4 B written per survivor in the gather)
  auto read_counts = [&](size_t posL, size_t posS, size_t posSet, int sideL, uint32_t ncL = 0,
                         uint32_t ncS = 0) -> mapsq_status {
    TRY(ensure_pinned(ctx, 2));
    CK(cudaMemcpyAsync(ctx->pinned, fsc, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    const uint64_t before = nw, sa = ctx->pinned[0], sb = ctx->pinned[1];
    const uint64_t survL = sideL ? sb : sa, survS = sideL ? sa : sb;
    add_bytes(posL, 8ull * survL);
    add_bytes(posS, 8ull * survS);
    add_bytes(posSet, 8ull * survL);
    if (gpos.size() == 2) {
      add_bytes(gpos[0], (16ull + 8ull * ncL) * survL);
      add_bytes(gpos[1], (16ull + 8ull * ncS) * survS);
    }
    gpos.clear();
    if (debug_on())
      std::fprintf(stderr, "[mapsq] filter round: %llu -> %llu words (A %llu, B %llu)\n",
                   (unsigned long long)before, (unsigned long long)(sa + sb),
                   (unsigned long long)sa, (unsigned long long)sb);
    return MAPSQ_OK;
  };
  CK(cudaMemsetAsync(fsc, 0, 2 * sizeof(uint64_t), s));
  // round 0 reads the key columns directly — a single packed column (exact or hashed bitmap),
  // or a hashed composite key (blocked Bloom bitmaps, key_hash computed from the columns); other
  // packed composite keys are Mapped first and filtered as words
  const bool colhash = pa.hash;
  const bool colpath = (pa.nkey == 1 && pl.kb <= 32 && !pa.hash) || colhash;
  if (!colpath) pv_off();
  if (colpath) {
    const bool s_is_b = n2 <= n1;  // S = the smaller side (ties: B)
    const uint64_t nS = s_is_b ? n2 : n1, nL = s_is_b ? n1 : n2;
    const uint32_t colbits = env_u32("MAPSQ_SJ_COLBITS", kSemijoinBits);
    const uint32_t bbits = colhash ? std::min(std::max<uint32_t>(16, bits_for(8 * std::max<uint64_t>(nS, 1))), colbits)
                                   : std::min<uint32_t>(pl.kb, kSemijoinBits);
    const uint32_t hashed = colhash || pl.kb > bbits;
    const uint64_t bw = std::max<uint64_t>(2, (1ull << bbits) / 32);
    uint32_t *bmS = bm, *bmL = bm + bw;
    const uint64_t kbytes = 4ull * pa.nkey;
    CK(cudaMemsetAsync(bm, 0, 2 * bw * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(sample, 0, 2 * sizeof(uint64_t), s));
    // Tp2 streaming in: as S it is waited for whole before the build; as L the build runs while
    // it arrives, the sample reads its first chunk only and the probe runs chunk by chunk
    const StreamIn *sb = ctx->stream_b;
    if (s_is_b) TRY(wait_stream_b(ctx, n2, s));
    const uint64_t l_rows = (sb && !s_is_b) ? sb->chunk_rows : ~0ull;
    {
      KTimer kt(ctx, s, "filter_build", kbytes * (nS + sj_sample_rows(std::min(nL, l_rows))), 2);
      mapsq_status wst = MAPSQ_OK;
      launch_sj_build_sample_cols(pa, s_is_b, bmS, bbits, hashed, sample, s, l_rows,
                                  [&] { if (!s_is_b) wst = wait_stream_b(ctx, std::min(n2, l_rows), s); });
      TRY(wst);
      CKL("filter_build");
      ctx->counters.filter_accesses += nS + sj_sample_rows(std::min(nL, l_rows));
    }
    TRY(sample_says_skip(&skipped));
    if (skipped) pv_off();
    if (!skipped) {
      const uint64_t slA = sj_slices(n1), slB = sj_slices(n2);
      const uint64_t seedL = word_round_seed(0);
      // carried columns (MAPSQ_SJ_CARRY: 0 off, 1 on, 2 = auto: exact bitmaps — this round is the
      // last, its survivors are exactly the rows ReduceDuplicate reads — and the sampled probe
      // kept at most half of the larger side; after a hashed round the word rounds still drop
      // most survivors (C5 J2: 49.5 M -> 9.5 M), so carrying for all of them does not pay)
      const uint64_t ssurv = ctx->pinned[0], srows = ctx->pinned[1];
      const uint32_t cmode = env_u32("MAPSQ_SJ_CARRY", 2);
      const bool do_carry = cmode == 1 || (cmode == 2 && !hashed && !colhash && srows > 0 &&
                                           2 * ssurv <= srows);
      SjCarry cr[2] = {none, none};
      if (pv) {  // (no carried columns: the values ride in the words)
        cr[0] = use[0];
        cr[1] = use[1];
      } else if (do_carry) {
        for (int sd = 0; sd < 2; sd++) {
          for (uint32_t c = 0; c < use[sd].n; c++) {
            cr[sd].src[c] = use[sd].src[c];
            cr[sd].out[c] = sc.get<uint32_t>(sd ? n2 : n1);
            NEED(cr[sd].out[c]);
          }
          cr[sd].n = use[sd].n;
          carry[sd] = cr[sd];
        }
      }
      // plain bitmaps: L's survivors set bm_L while probed (bit = key'); hashed composite keys:
      // bm_L (a wblock of the survivors' key') is set from L's gathered survivor words
      const bool set_in_probe = !colhash;
      const int sideL = s_is_b ? 0 : 1, sideS = 1 - sideL;
      uint64_t *outL = cur + (sideL ? n1 : 0), *outS = cur + (sideS ? n1 : 0);
      size_t posL, posS, posSet = ~size_t(0);
      CK(cudaMemsetAsync(hist, 0, kRadix * sizeof(uint32_t), s));
      {
        KTimer kt(ctx, s, "filter_probe", kbytes * nL);
        if (sb && sideL == 1) {  // chunk by chunk as Tp2's copies land
          for (uint64_t lo = 0; lo < n2; lo += sb->chunk_rows) {
            const uint64_t hi = std::min(n2, lo + sb->chunk_rows);
            TRY(wait_stream_b(ctx, hi, s));
            launch_sj_probe_cols(pa, true, colhash ? 1 : 0, bmS, bbits, hashed, 0,
                                 set_in_probe ? bmL : nullptr, stage, cnt, s, lo, hi);
          }
        } else {
          launch_sj_probe_cols(pa, sideL == 1, colhash ? 1 : 0, bmS, bbits, hashed, 0,
                               set_in_probe ? bmL : nullptr, stage, cnt, s);
        }
        CKL("filter_probe");
      }
      TRY(wait_stream_b(ctx, n2, s));  // (all of Tp2 from here on)
      posL = pending_pos();
      TRY(scan_gather(sideL, sideL ? slA : 0, sideL ? slB : slA, outL, cr[sideL]));
      if (!set_in_probe) {
        KTimer kt(ctx, s, "filter_set", 0);
        launch_sj_set_words(outL, fsc + sideL, nL, 2, bmL, pl.ib, bbits, 0, seedL, s);
        CKL("filter_set");
        posSet = pending_pos();
      }
      {
        KTimer kt(ctx, s, "filter_probe", kbytes * nS);
        launch_sj_probe_cols(pa, sideS == 1, colhash ? 2 : 0, bmL, bbits, hashed, seedL, nullptr,
                             stage, cnt, s);
        CKL("filter_probe");
      }
      posS = pending_pos();
      TRY(scan_gather(sideS, sideS ? slA : 0, sideS ? slB : slA, outS, cr[sideS]));
      ctx->counters.filter_accesses += nL + nS;
      TRY(read_counts(posL, posS, posSet, sideL, pv ? 0 : cr[sideL].n, pv ? 0 : cr[sideS].n));
      nA = ctx->pinned[0];
      nB = ctx->pinned[1];
      offB = n1;
      nw = nA + nB;
      // exact bitmaps leave no false positive; a hashed round that dropped < 10% of the rows
      // says the keys mostly match, so refinement rounds would not pay
      exact = (!hashed && !colhash) || nw * 10 > n * 9;
    }
  } else {
    // composite packed keys: Map every row, then filter the words
    TRY(wait_stream_b(ctx, n2, s));
    pa.passes = 0;  // (the histogram is counted by the last round's gathers)
    KTimer kt(ctx, s, "pack_hist", 4ull * pl.nshared * n + 8ull * n);
    launch_pack_hist(pa, cur, nullptr, hist, s);
    CKL("pack_hist");
  }
  // word rounds: the first one for non-column keys (sampled first), then refinements while a
  // hashed round still drops >= 10% of its input (each round sizes its bitmaps to ~8 bits per
  // key of the smaller side, with a fresh hash seed).  Input segments in cur, output in spare.
  // (at most two rounds in all: C5's third round removed 19% of 7.1M words for ~0.15 ms, more
  // than those words cost the sort and the verification)
  for (int round = colpath ? 1 : 0;
       !skipped && round < 2 && !exact && (round == 0 || nw >= kSemijoinMinRows) && nA && nB;
       round++) {
    const SjSeg A{cur, nA}, B{cur + offB, nB};
    const uint64_t slA = sj_slices(nA), slB = sj_slices(nB);
    const bool s_is_b = nB <= nA;
    const int sideL = s_is_b ? 0 : 1, sideS = 1 - sideL;
    const SjSeg S = s_is_b ? B : A, L = s_is_b ? A : B;
    const uint64_t sl0S = s_is_b ? slA : 0, sl0L = s_is_b ? 0 : slA;
    const uint32_t bbits = word_round_bits(S.rows);
    const uint64_t bw = (1ull << bbits) / 32;
    uint32_t *bmS = bm, *bmL = bm + bw;
    const uint64_t seed = word_round_seed(round);
    CK(cudaMemsetAsync(bm, 0, 2 * bw * sizeof(uint32_t), s));
    if (round == 0) CK(cudaMemsetAsync(sample, 0, 2 * sizeof(uint64_t), s));
    {
      KTimer kt(ctx, s, "filter_build", 8ull * (S.rows + (round == 0 ? sj_sample_rows(L.rows) : 0)),
                round == 0 ? 2 : 1);
      launch_sj_build_words(S, pl.ib, seed, bbits, bmS, s);
      if (round == 0) launch_sj_sample_words(L, pl.ib, seed, bbits, bmS, sample, s);
      CKL("filter_build");
      ctx->counters.filter_accesses += S.rows + (round == 0 ? sj_sample_rows(L.rows) : 0);
    }
    if (round == 0) {
      TRY(sample_says_skip(&skipped));
      if (skipped) break;
    }
    if (!spare) {
      spare = sc.get<uint64_t>(nw + 2 * kSjSlice);
      NEED(spare);
    }
    uint64_t *outL = spare + (sideL ? nA : 0), *outS = spare + (sideS ? nA : 0);
    CK(cudaMemsetAsync(hist, 0, kRadix * sizeof(uint32_t), s));
    {
      KTimer kt(ctx, s, "filter_probe", 8ull * L.rows);
      launch_sj_probe_words(L, sl0L, pl.ib, bmS, bbits, seed, stage, cnt, s);
      CKL("filter_probe");
    }
    const size_t posL = pending_pos();
    TRY(scan_gather(sideL, sl0L, sideL ? slB : slA, outL));
    {
      KTimer kt(ctx, s, "filter_set", 0);
      launch_sj_set_words(outL, fsc + sideL, L.rows, 2, bmL, pl.ib, bbits, 0, seed, s);
      CKL("filter_set");
    }
    const size_t posSet = pending_pos();
    {
      KTimer kt(ctx, s, "filter_probe", 8ull * S.rows);
      launch_sj_probe_words(S, sl0S, pl.ib, bmL, bbits, seed, stage, cnt, s);
      CKL("filter_probe");
    }
    const size_t posS = pending_pos();
    TRY(scan_gather(sideS, sl0S, sideS ? slB : slA, outS));
    ctx->counters.filter_accesses += L.rows + S.rows;
    const uint64_t before = nw;
    TRY(read_counts(posL, posS, posSet, sideL));
    offB = nA;
    nA = ctx->pinned[0];
    nB = ctx->pinned[1];
    nw = nA + nB;
    std::swap(cur, spare);  // the output segments become the input; the old input is free
    if (nw * 10 > before * 9) break;  // < 10% dropped: further rounds would not pay
  }
  if (skipped) {  // unfiltered: every row's word, the first digit's histogram
    TRY(wait_stream_b(ctx, n2, s));
    nw = n;
    nA = n1;
    offB = n1;
    nB = n2;
    CK(cudaMemsetAsync(hist, 0, kRadix * sizeof(uint32_t), s));
    if (colpath) {
      const PackArgs pm = pack_args(pl, a, b);
      KTimer kt(ctx, s, "pack_hist", 4ull * pl.nshared * n + 8ull * n);
      launch_pack_hist(pm, cur, nullptr, hist, s);
      CKL("pack_hist");
    } else {
      KTimer kt(ctx, s, "key_hist", 8ull * n);
      launch_key_hist(cur, n, pl.ib, 1, pl.passes == 1 ? pl.kb : 8, hist, s);
      CKL("key_hist");
    }
  }
  *nA_out = nA;
  *offB_out = offB;
  *nB_out = nB;
  carry[0].pv = carry[1].pv = pv;
  return MAPSQ_OK;
}

// One launch for a tiny P64 join (small.cu): the output is allocated for min(n1 * n2, 2^16) rows;
// one blocking read of |RS|.  *done = false (nothing allocated) when |RS| exceeds that.
mapsq_status small_join(mapsq_ctx *ctx, const mapsq_join_plan &pl, const mapsq_table *a,
                        const mapsq_table *b, mapsq_table *rs, cudaStream_t s, bool *done) {
  *done = false;
  const uint64_t cap = std::min<uint64_t>(pl.n1 * pl.n2, 1ull << 16);
  Scratch sc(ctx, s);
  unsigned long long *mdev = sc.get<unsigned long long>(1);
  NEED(mdev);
  fill_empty_join(pl, a, b, rs);
  TRY(alloc_table(ctx, rs, cap, pl.out_ncols, s));
  const PackArgs pa = pack_args(pl, a, b);
  ExpandArgs ea;
  std::memset(&ea, 0, sizeof ea);
  ea.n1 = pl.n1;
  ea.ib = pl.ib;
  ea.nkey = pl.nshared;
  for (uint32_t c = 0; c < pl.nshared; c++) {
    ea.key_lo[c] = pl.key_lo[c];
    ea.key_shift[c] = pl.key_shift[c];
    ea.key_mask[c] = (uint32_t)((1ull << pl.key_bits[c]) - 1);
  }
  ea.nrest1 = pl.nrest1;
  ea.nrest2 = pl.nrest2;
  for (uint32_t c = 0; c < pl.nrest1; c++) ea.rest1[c] = a->col[pl.rest_col1[c]];
  for (uint32_t c = 0; c < pl.nrest2; c++) ea.rest2[c] = b->col[pl.rest_col2[c]];
  for (uint32_t c = 0; c < pl.out_ncols; c++) ea.out[c] = rs->col[c];
  {
    KTimer kt(ctx, s, "small_join", 4ull * (pl.n1 * (pl.nshared + pl.nrest1) + pl.n2 * (pl.nshared + pl.nrest2)));
    launch_small_join(pa, ea, cap, mdev, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      dfree(ctx, rs->owner, s);
      clear_table(rs);
      return cuda_check(ctx, e, "small_join");
    }
  }
  TRY(ensure_pinned(ctx, 1));
  CK(cudaMemcpyAsync(ctx->pinned, mdev, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));  // the one blocking read: |RS|
  const uint64_t m = ctx->pinned[0];
  if (m > cap) {  // does not fit the allocation: the regular path
    dfree(ctx, rs->owner, s);
    clear_table(rs);
    return MAPSQ_OK;
  }
  rs->nrows = m;
  if (m == 0) {
    dfree(ctx, rs->owner, s);
    rs->owner = nullptr;
    for (uint32_t c = 0; c < pl.out_ncols; c++) rs->col[c] = nullptr;
  }
  ctx->counters.join_out_rows += m;
  *done = true;
  return MAPSQ_OK;
}

// ------------------------------------------------------------------------------ join
mapsq_status join_impl(mapsq_ctx *ctx, const mapsq_table *tp1_in, const mapsq_table *tp2_in,
                       mapsq_table *rs, cudaStream_t s) {
  clear_table(rs);
  TRY(check_table(ctx, tp1_in, "tp1"));
  TRY(check_table(ctx, tp2_in, "tp2"));
  mapsq_table a = *tp1_in, b = *tp2_in;
  TRY(bounds_of(ctx, &a, s));
  if (!(b.flags & MAPSQ_TABLE_BOUNDS)) TRY(wait_stream_b(ctx, b.nrows, s));
  TRY(bounds_of(ctx, &b, s));
  mapsq_join_plan pl;
  TRY(plan_join(ctx, &a, &b, &pl, ctx->wide_key_mode));
  const uint64_t n1 = pl.n1, n2 = pl.n2, n = n1 + n2;
  ctx->counters.joins++;
  ctx->counters.join_in_rows += n;
  ctx->counters.last_kb = pl.kb;
  ctx->counters.last_ib = pl.ib;
  ctx->counters.last_passes = pl.passes;
  ctx->counters.last_path = pl.path;
  ctx->counters.last_groups = 0;
  ctx->counters.last_filtered = 0;
  if (n1 == 0 || n2 == 0 || pl.disjoint) {
    fill_empty_join(pl, &a, &b, rs);
    return MAPSQ_OK;
  }
  if (pl.path == MAPSQ_PATH_P64 && n <= kSmallMaxRows && ctx->small_joins) {
    TRY(wait_stream_b(ctx, n2, s));
    bool done = false;
    TRY(small_join(ctx, pl, &a, &b, rs, s, &done));
    if (done) return MAPSQ_OK;
  }
  // value-carrying words (kPvIb): P64 joins with at most one non-key column per side whose key
  // fits 31 bits (MAPSQ_PV=0 in the environment: row-id words, for ablations).  The plan's ib
  // becomes 33 for the words; n1 (the label boundary ReduceDuplicate compares with) 2^32.
  // (candidates here; the semi-join filter's column round makes them, see filter_map)
  bool pv = pl.path == MAPSQ_PATH_P64 && pl.nrest1 <= 1 && pl.nrest2 <= 1 &&
            pl.kb + kPvIb <= 64 && n1 < (1ull << 32) && n2 < (1ull << 32) &&
            env_u32("MAPSQ_PV", 1) != 0;
  const uint32_t ib_row = pl.ib;
  Scratch sc(ctx, s);
  const bool kv = pl.path == MAPSQ_PATH_KV;
  // (+2 slices: the semi-join filter stages each side's survivors at slice-aligned offsets)
  uint64_t *wa = sc.get<uint64_t>(n + 2 * kSjSlice), *wb = sc.get<uint64_t>(n + 2 * kSjSlice);
  uint32_t *va = kv ? sc.get<uint32_t>(n) : nullptr, *vb = kv ? sc.get<uint32_t>(n) : nullptr;
  uint32_t *hist = sc.get<uint32_t>(kMaxPasses * kRadix);
  NEED(wa);
  NEED(wb);
  NEED(hist);
  if (kv) {
    NEED(va);
    NEED(vb);
  }
  // ---- Map (row a3) + first-digit histogram; optionally behind the semi-join filter
  CK(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
  uint64_t *cur = wa, *alt = wb;  // the words entering the sort are in cur
  uint64_t nw = n, seg_n0 = n, seg_gap = 0;
  const bool filt = !kv && pl.kb > 0 &&
                    (ctx->semijoin == MAPSQ_SEMIJOIN_ON ||
                     (ctx->semijoin == MAPSQ_SEMIJOIN_AUTO && n >= kSemijoinMinRows));
  pv = pv && filt;
  if (pv) pl.ib = kPvIb;
  if (filt && pl.path == MAPSQ_PATH_HASH && pl.kb < 64 - pl.ib &&
      env_u32("MAPSQ_HASH_WIDEN", 0)) {
    // (ablation knob) widen key' beyond 32 bits: after the filter only ~|L'|·|S'| / 2^32
    // colliding pairs remain (C5 J2: 3.5e6 x 3.5e6 / 2^32 ~ 3e3), so the default keeps 32 bits and
    // saves a digit pass
    pl.kb = std::min<uint32_t>(64 - pl.ib, 40);
    pl.passes = (pl.kb + MAPSQ_RADIX_BITS - 1) / MAPSQ_RADIX_BITS;
    ctx->counters.last_kb = pl.kb;
    ctx->counters.last_passes = pl.passes;
  }
  const bool residual = pl.path == MAPSQ_PATH_RESIDUAL || pl.path == MAPSQ_PATH_HASH;
  uint64_t rowsA = n1, rowsB = n2;  // rows of the columns ReduceDuplicate gathers from
  if (filt) {
    // the columns ReduceDuplicate reads by row id, offered to the filter to carry: every column
    // (verification reads the shared ones too) or the non-key columns (expand decodes the key);
    // with value-carrying words the side's one non-key column goes into the words instead
    SjCarry carry[2];
    uint32_t ccol[2][MAPSQ_MAX_COLS];
    for (int sd = 0; sd < 2; sd++) {
      const mapsq_table &t = sd ? b : a;
      carry[sd].n = 0;
      carry[sd].pv = pv;
      if (pv) {
        const uint32_t nr = sd ? pl.nrest2 : pl.nrest1;
        if (nr) carry[sd].src[carry[sd].n++] = t.col[sd ? pl.rest_col2[0] : pl.rest_col1[0]];
        continue;
      }
      const uint32_t nr = sd ? pl.nrest2 : pl.nrest1;
      for (uint32_t c = 0; c < (residual ? t.ncols : nr); c++) {
        const uint32_t j = residual ? c : (sd ? pl.rest_col2[c] : pl.rest_col1[c]);
        ccol[sd][carry[sd].n] = j;
        carry[sd].src[carry[sd].n++] = t.col[j];
      }
    }
    uint64_t nA = 0, offB = 0, nB = 0;
    TRY(filter_map(ctx, pl, &a, &b, sc, s, cur, alt, hist, &nA, &offB, &nB, carry, ib_row));
    pv = carry[0].pv;
    TRY(wait_stream_b(ctx, n2, s));  // (filter_map waited; anything later reads all of Tp2)
    nw = nA + nB;
    seg_n0 = nA;
    seg_gap = offB - nA;
    ctx->counters.last_filtered = n - nw;
    if (nA == 0 || nB == 0) {  // a side without survivors: no key on both sides
      fill_empty_join(pl, &a, &b, rs);
      return MAPSQ_OK;
    }
    // carried: the words' row ids now index the survivors' dense columns (side B's from n1 on)
    for (int sd = 0; sd < 2 && !pv; sd++) {
      mapsq_table &t = sd ? b : a;
      for (uint32_t c = 0; c < carry[sd].n; c++) t.col[ccol[sd][c]] = carry[sd].out[c];
      if (carry[sd].n) (sd ? rowsB : rowsA) = sd ? nB : nA;
    }
  } else {
    TRY(wait_stream_b(ctx, n2, s));
    const PackArgs pa = pack_args(pl, &a, &b);
    KTimer kt(ctx, s, "pack_hist", 4ull * (pl.nshared + (pv ? 1 : 0)) * n + (kv ? 12ull : 8ull) * n);
    launch_pack_hist(pa, cur, va, hist, s);
    CKL("pack_hist");
  }
  const uint64_t lab = pv ? (1ull << 32) : n1;  // the words' label boundary
  ctx->counters.last_ib = pl.ib;
  // ---- Sort (row a4)
  int which = 0;
  TRY(radix_sort(ctx, cur, alt, va, vb, nw, kv ? 0 : pl.ib, pl.kb, hist, sc, s, &which, seg_n0,
                 seg_gap));
  uint64_t *words = which ? alt : cur;
  uint32_t *vals = kv ? (which ? vb : va) : nullptr;
  sc.release(which ? cur : alt);
  if (kv) sc.release(which ? va : vb);
  // ---- ReduceDuplicate 1 (row a5): groups + counts + exclusive scan
  const uint64_t cap = std::min(n1, n2);
  uint32_t *gs = sc.get<uint32_t>(cap), *gp = sc.get<uint32_t>(cap), *ge = sc.get<uint32_t>(cap);
  uint64_t *gc = sc.get<uint64_t>(cap), *go = sc.get<uint64_t>(cap);
  const uint64_t gtiles = find_groups_tiles(nw);
  uint64_t *gstatus = sc.get<uint64_t>(gtiles);
  uint64_t *scal = sc.get<uint64_t>(4);  // [0] ngroups, [1] |RS|, [2] tile counter
  uint64_t *tmp = sc.get<uint64_t>(scan_tmp_words(cap));
  NEED(gs); NEED(gp); NEED(ge); NEED(gc); NEED(go); NEED(gstatus); NEED(scal); NEED(tmp);
  CK(cudaMemsetAsync(gstatus, 0, gtiles * sizeof(uint64_t), s));
  CK(cudaMemsetAsync(scal, 0, 4 * sizeof(uint64_t), s));
  {
    KTimer kt(ctx, s, "find_groups", nw * 8ull);
    GroupOut g{gs, gp, ge, gc};
    launch_find_groups(kv ? nullptr : words, kv ? words : nullptr, vals, nw, lab, pl.ib, g,
                       gstatus, reinterpret_cast<uint32_t *>(scal + 2), scal, s);
    CKL("find_groups");
  }
  // RESIDUAL and HASH: the nL * nR pairs of a key' group are candidates, verified on the shared
  // columns not (exactly) in key'
  {
    KTimer kt(ctx, s, "scan_counts", cap * 16ull);
    launch_exclusive_scan_u64_dev(gc, go, scal, cap, tmp, scal + 1, s);
    CKL("scan_counts");
  }
  TRY(ensure_pinned(ctx, 2));
  CK(cudaMemcpyAsync(ctx->pinned, scal, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));  // the one blocking read: |RS| (candidates) sizes the output
  const uint64_t ngroups = ctx->pinned[0], m = ctx->pinned[1];
  ctx->counters.last_groups = ngroups;
  if (residual) {
    const uint64_t C = m;  // candidate pairs: an upper bound of |RS|
    ResidualArgs ra;
    std::memset(&ra, 0, sizeof ra);
    ra.words = words;
    ra.n1 = n1;
    ra.ib = pl.ib;
    ra.gstart = gs;
    ra.gsplit = gp;
    ra.gend = ge;
    for (uint32_t c = 0; c < pl.nshared; c++)
      if (!(pl.packed_mask >> c & 1u)) {
        ra.res1[ra.nres] = a.col[pl.key_col1[c]];
        ra.res2[ra.nres] = b.col[pl.key_col2[c]];
        ra.nres++;
      }
    uint32_t k = 0;
    for (uint32_t c = 0; c < pl.nshared; c++, k++) {
      ra.src_side[k] = 0;
      ra.src[k] = a.col[pl.key_col1[c]];
    }
    for (uint32_t c = 0; c < pl.nrest1; c++, k++) {
      ra.src_side[k] = 0;
      ra.src[k] = a.col[pl.rest_col1[c]];
    }
    for (uint32_t c = 0; c < pl.nrest2; c++, k++) {
      ra.src_side[k] = 1;
      ra.src[k] = b.col[pl.rest_col2[c]];
    }
    ra.nout = k;
    fill_empty_join(pl, &a, &b, rs);
    if (C == 0) {
      ctx->counters.join_out_rows += 0;
      return MAPSQ_OK;
    }
    const uint64_t vt = verify_tiles(C);
    uint64_t *vstatus = sc.get<uint64_t>(vt + 1), *tile_g0 = sc.get<uint64_t>(vt + 1);
    uint32_t *vctr = sc.get<uint32_t>(2);
    unsigned long long *vtot = sc.get<unsigned long long>(2);
    NEED(vstatus); NEED(tile_g0); NEED(vctr); NEED(vtot);
    // the output is sized by the candidate count when that is a tight bound (hashed keys: the
    // candidates are the matches plus the rare key' collisions); otherwise the matches are
    // counted first (a second candidate-parallel pass without writes)
    uint64_t cap_rows = C;
    if (C > 2 * (n1 + n2) + (1ull << 20)) {
      CK(cudaMemsetAsync(vtot, 0, 2 * sizeof(uint64_t), s));
      {
        KTimer kt(ctx, s, "verify_count", 8ull * nw);
        launch_verify_emit(ra, go, tile_g0, ngroups, C, false, vstatus, vctr, vtot, s);
        CKL("verify_count");
      }
      CK(cudaMemcpyAsync(ctx->pinned, vtot, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      cap_rows = ctx->pinned[0];
      if (cap_rows == 0) return MAPSQ_OK;
    }
    TRY(alloc_table(ctx, rs, cap_rows, pl.out_ncols, s));
    for (uint32_t c = 0; c < k; c++) ra.out[c] = rs->col[c];
    CK(cudaMemsetAsync(vstatus, 0, (vt + 1) * sizeof(uint64_t), s));
    CK(cudaMemsetAsync(vctr, 0, 2 * sizeof(uint32_t), s));
    CK(cudaMemsetAsync(vtot, 0, 2 * sizeof(uint64_t), s));
    size_t pos = ~size_t(0);
    {
      KTimer kt(ctx, s, "verify_emit", 8ull * nw, 2);
      launch_verify_emit(ra, go, tile_g0, ngroups, C, true, vstatus, vctr, vtot, s);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) {
        dfree(ctx, rs->owner, s);
        clear_table(rs);
        return cuda_check(ctx, e, "verify_emit");
      }
    }
    if (ctx->profiling) pos = ctx->pending.size() - 1;
    CK(cudaMemcpyAsync(ctx->pinned, vtot, sizeof(uint64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));  // |RS|: the matched candidates
    const uint64_t mm = ctx->pinned[0];
    rs->nrows = mm;
    if (mm == 0) {  // nothing matched: release the allocation, keep the schema
      dfree(ctx, rs->owner, s);
      rs->owner = nullptr;
      for (uint32_t c = 0; c < pl.out_ncols; c++) rs->col[c] = nullptr;
    }
    if (pos < ctx->pending.size()) ctx->pending[pos].bytes += 4ull * mm * pl.out_ncols;
    ctx->counters.join_out_rows += mm;
    return MAPSQ_OK;
  }
  // ---- ReduceDuplicate 2 (row a6): expand into RS
  fill_empty_join(pl, &a, &b, rs);
  TRY(alloc_table(ctx, rs, m, pl.out_ncols, s));
  if (m) {
    ExpandArgs ea;
    std::memset(&ea, 0, sizeof ea);
    ea.words = kv ? nullptr : words;
    ea.keys = kv ? words : nullptr;
    ea.vals = vals;
    ea.n1 = lab;
    ea.ib = pl.ib;
    ea.gstart = gs;
    ea.gsplit = gp;
    ea.gend = ge;
    ea.goff = go;
    ea.ngroups = ngroups;
    ea.m = m;
    ea.nkey = pl.nshared;
    for (uint32_t c = 0; c < pl.nshared; c++) {
      ea.key_lo[c] = pl.key_lo[c];
      ea.key_shift[c] = pl.key_shift[c];
      ea.key_mask[c] = (uint32_t)((1ull << pl.key_bits[c]) - 1);
    }
    ea.nrest1 = pl.nrest1;
    ea.nrest2 = pl.nrest2;
    // (value-carrying words: no source columns, the values come from the words)
    for (uint32_t c = 0; c < pl.nrest1; c++) ea.rest1[c] = pv ? nullptr : a.col[pl.rest_col1[c]];
    for (uint32_t c = 0; c < pl.nrest2; c++) ea.rest2[c] = pv ? nullptr : b.col[pl.rest_col2[c]];
    for (uint32_t c = 0; c < pl.out_ncols; c++) ea.out[c] = rs->col[c];
    ea.tile_g0 = sc.get<uint64_t>(expand_tiles(m) + 1);
    NEED(ea.tile_g0);
    const uint64_t bytes = 4ull * m * pl.out_ncols + 8ull * nw +
                           (pv ? 0ull : 4ull * (rowsA * pl.nrest1 + rowsB * pl.nrest2));
    KTimer kt(ctx, s, "expand", bytes, 2);
    launch_expand(ea, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      dfree(ctx, rs->owner, s);
      clear_table(rs);
      return cuda_check(ctx, e, "expand");
    }
  }
  ctx->counters.join_out_rows += m;
  return MAPSQ_OK;
}

// ------------------------------------------------------------------------------ scan
mapsq_status build_scan_args(mapsq_ctx *ctx, const mapsq_pattern *pats, int k, ScanArgs *a,
                             int32_t vars[][3]) {
  std::memset(a, 0, sizeof *a);
  if (!pats || k < 1 || k > MAPSQ_MAX_PATTERNS)
    return set_error(ctx, MAPSQ_E_INVALID, "pattern count out of range");
  a->k = k;
  for (int j = 0; j < k; j++) {
    ScanPat &p = a->pat[j];
    for (int q = 0; q < 3; q++) {
      const int32_t v = pats[j].var[q];
      if (v < -1) return set_error(ctx, MAPSQ_E_INVALID, "bad pattern variable");
      if (v == -1) {
        p.const_mask |= 1u << q;
        p.id[q] = pats[j].id[q];
        p.c[q] = pats[j].id[q];
        p.m[q] = ~0u;
        a->need_count |= 1u << q;
        continue;
      }
      bool seen = false;
      for (int r = 0; r < q; r++)
        if (pats[j].var[r] == v) {
          seen = true;
          p.eq_mask |= (r == 0 && q == 1) ? 1u : (r == 0 && q == 2) ? 2u : 4u;
          a->need_count |= (1u << q) | (1u << r);
        }
      if (!seen) {
        vars[j][p.ncols] = v;
        p.src[p.ncols++] = q;
        a->need_write |= 1u << q;
      }
    }
    if (p.ncols == 0) return set_error(ctx, MAPSQ_E_INVALID, "pattern without variables");
  }
  return MAPSQ_OK;
}

mapsq_status scan_impl(mapsq_ctx *ctx, const mapsq_triples *T, const mapsq_pattern *pats, int k,
                       mapsq_table *out, cudaStream_t s) {
  if (!out) return set_error(ctx, MAPSQ_E_INVALID, "out is NULL");
  for (int j = 0; j < k && j < MAPSQ_MAX_PATTERNS; j++) clear_table(&out[j]);
  if (!T) return set_error(ctx, MAPSQ_E_INVALID, "triples is NULL");
  if (T->n && (!T->s || !T->p || !T->o)) return set_error(ctx, MAPSQ_E_INVALID, "NULL triple column");
  ScanArgs a;
  int32_t vars[MAPSQ_MAX_PATTERNS][3];
  TRY(build_scan_args(ctx, pats, k, &a, vars));
  for (int j = 0; j < k; j++) {
    out[j].ncols = a.pat[j].ncols;
    for (uint32_t c = 0; c < a.pat[j].ncols; c++) out[j].var[c] = vars[j][c];
    out[j].flags = MAPSQ_TABLE_BOUNDS;
  }
  ctx->counters.scans += k;
  ctx->counters.scanned_triples += T->n;
  const uint64_t n = T->n;
  if (n == 0) return MAPSQ_OK;
  Scratch sc(ctx, s);
  const uint64_t ntiles = ceil_div(n, kScanTile);
  const uint64_t mask_words = ceil_div(n, 32);
  uint32_t *masks = sc.get<uint32_t>(k * mask_words);
  uint32_t *tcnt = sc.get<uint32_t>(k * ntiles);
  uint64_t *toff = sc.get<uint64_t>(k * ntiles + 1);
  uint64_t *tmp = sc.get<uint64_t>(scan_tmp_words(k * ntiles));
  uint32_t *bnd = sc.get<uint32_t>(2 * MAPSQ_MAX_PATTERNS * 3);
  NEED(masks); NEED(tcnt); NEED(toff); NEED(tmp); NEED(bnd);
  const int npos_count = __builtin_popcount(a.need_count);
  {
    KTimer kt(ctx, s, "scan_count", 4ull * npos_count * n + 4ull * k * mask_words);
    launch_scan_count(*T, a, masks, mask_words, tcnt, ntiles, s);
    CKL("scan_count");
  }
  {
    KTimer kt(ctx, s, "scan_tiles", 12ull * k * ntiles);
    launch_exclusive_scan_u32(tcnt, toff, k * ntiles, tmp, toff + k * ntiles, s);
    CKL("scan_tiles");
  }
  TRY(ensure_pinned(ctx, k + 1));
  for (int j = 0; j <= k; j++)
    CK(cudaMemcpyAsync(ctx->pinned + j, toff + (uint64_t)j * ntiles, sizeof(uint64_t),
                       cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));  // blocking read of the k match counts
  uint64_t rows[MAPSQ_MAX_PATTERNS], total = 0;
  for (int j = 0; j < k; j++) {
    rows[j] = ctx->pinned[j + 1] - ctx->pinned[j];
    total += rows[j];
  }
  ScanOut so;
  std::memset(&so, 0, sizeof so);
  for (int j = 0; j < k; j++) {
    mapsq_status st = alloc_table(ctx, &out[j], rows[j], a.pat[j].ncols, s);
    if (st != MAPSQ_OK) {
      for (int q = 0; q < j; q++) {
        dfree(ctx, out[q].owner, s);
        clear_table(&out[q]);
      }
      return st;
    }
    for (uint32_t c = 0; c < a.pat[j].ncols; c++) so.col[j * 3 + c] = out[j].col[c];
  }
  if (total == 0) return MAPSQ_OK;
  uint32_t *bmin = bnd, *bmax = bnd + MAPSQ_MAX_PATTERNS * 3;
  CK(cudaMemsetAsync(bmin, 0xff, MAPSQ_MAX_PATTERNS * 3 * sizeof(uint32_t), s));
  CK(cudaMemsetAsync(bmax, 0, MAPSQ_MAX_PATTERNS * 3 * sizeof(uint32_t), s));
  {
    uint64_t outb = 0;
    for (int j = 0; j < k; j++) outb += 4ull * rows[j] * a.pat[j].ncols;
    const int npos_write = __builtin_popcount(a.need_write);
    KTimer kt(ctx, s, "scan_write",
              4ull * k * mask_words + 4ull * npos_write * total + outb);
    launch_scan_write(*T, a, masks, mask_words, toff, ntiles, so, bmin, bmax, s);
    CKL("scan_write");
  }
  CK(cudaMemcpyAsync(ctx->pinned, bnd, 2 * MAPSQ_MAX_PATTERNS * 3 * sizeof(uint32_t),
                     cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint32_t *h = reinterpret_cast<const uint32_t *>(ctx->pinned);
  for (int j = 0; j < k; j++)
    for (uint32_t c = 0; c < a.pat[j].ncols; c++) {
      out[j].lo[c] = rows[j] ? h[j * 3 + c] : 0;
      out[j].hi[c] = rows[j] ? h[MAPSQ_MAX_PATTERNS * 3 + j * 3 + c] : 0;
    }
  return MAPSQ_OK;
}

}  // namespace

struct mapsq_index {
  uint64_t n = 0;
  void *owner = nullptr;  // s | p | o, one allocation (16 B aligned column strides)
  uint32_t *s = nullptr, *p = nullptr, *o = nullptr;
  std::vector<uint32_t> pred;   // distinct predicates, ascending
  std::vector<uint64_t> start;  // pred[i] occupies rows [start[i], start[i + 1])
  std::vector<uint32_t> slo, shi, olo, ohi;
};

namespace {

// ------------------------------------------------------------------------------ index (f1)
mapsq_status index_build_impl(mapsq_ctx *ctx, const mapsq_triples *T, mapsq_index **out,
                              cudaStream_t s) {
  if (!out) return set_error(ctx, MAPSQ_E_INVALID, "out is NULL");
  *out = nullptr;
  if (!T) return set_error(ctx, MAPSQ_E_INVALID, "triples is NULL");
  if (T->n && (!T->s || !T->p || !T->o)) return set_error(ctx, MAPSQ_E_INVALID, "NULL triple column");
  const uint64_t n = T->n;
  std::unique_ptr<mapsq_index> idx(new (std::nothrow) mapsq_index());
  if (!idx) return set_error(ctx, MAPSQ_E_NOMEM, "index allocation failed");
  idx->n = n;
  idx->start.push_back(0);
  if (n == 0) {
    *out = idx.release();
    return MAPSQ_OK;
  }
  const uint32_t ib = n > 1 ? bits_for(n - 1) : 1;
  Scratch sc(ctx, s);
  uint32_t *pb = sc.get<uint32_t>(2);
  NEED(pb);
  CK(cudaMemsetAsync(pb, 0xff, 4, s));
  CK(cudaMemsetAsync(pb + 1, 0, 4, s));
  {
    const uint32_t *cols[1] = {T->p};
    KTimer kt(ctx, s, "minmax", 4ull * n);
    launch_minmax(cols, 1, n, pb, s);
    CKL("minmax");
  }
  TRY(ensure_pinned(ctx, 1));
  CK(cudaMemcpyAsync(ctx->pinned, pb, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint32_t p_lo = reinterpret_cast<const uint32_t *>(ctx->pinned)[0];
  const uint32_t p_hi = reinterpret_cast<const uint32_t *>(ctx->pinned)[1];
  const uint32_t pbits = p_hi > p_lo ? bits_for((uint64_t)p_hi - p_lo) : 0;
  if (pbits + ib > 64)
    return set_error(ctx, MAPSQ_E_UNSUPPORTED, "predicate bits + row bits exceed 64");
  // Map + stable sort on the predicate bits only (the row id below keeps the triple order)
  // (+2 slices: the semi-join filter stages each side's survivors at slice-aligned offsets)
  uint64_t *wa = sc.get<uint64_t>(n + 2 * kSjSlice), *wb = sc.get<uint64_t>(n + 2 * kSjSlice);
  uint32_t *hist = sc.get<uint32_t>(kMaxPasses * kRadix);
  NEED(wa); NEED(wb); NEED(hist);
  CK(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
  {
    PackArgs pa;
    std::memset(&pa, 0, sizeof pa);
    pa.nkey = pbits ? 1 : 0;
    pa.key1[0] = T->p;
    pa.key2[0] = T->p + n;  // (no RIGHT rows: n2 == 0)
    pa.lo[0] = p_lo;
    pa.shift[0] = 0;
    pa.n1 = n;
    pa.n2 = 0;
    pa.ib = ib;
    pa.bit_lo = ib;
    const uint32_t passes = (pbits + 7) / 8;
    pa.passes = passes ? 1 : 0;
    pa.last_mask = passes == 1 ? ((1u << pbits) - 1u) : 0xffu;
    KTimer kt(ctx, s, "pack_hist", 4ull * n + 8ull * n);
    launch_pack_hist(pa, wa, nullptr, hist, s);
    CKL("pack_hist");
  }
  int which = 0;
  TRY(radix_sort(ctx, wa, wb, nullptr, nullptr, n, ib, pbits, hist, sc, s, &which));
  const uint64_t *words = which ? wb : wa;
  const uint64_t stride = (n + 3) & ~3ull;
  idx->owner = dalloc(ctx, 3 * stride * sizeof(uint32_t), s);
  if (!idx->owner) return set_error(ctx, MAPSQ_E_NOMEM, "index allocation failed");
  idx->s = static_cast<uint32_t *>(idx->owner);
  idx->p = idx->s + stride;
  idx->o = idx->p + stride;
  struct OwnerGuard {
    mapsq_ctx *ctx; mapsq_index *idx; cudaStream_t s; bool keep = false;
    ~OwnerGuard() { if (!keep) dfree(ctx, idx->owner, s); }
  } guard{ctx, idx.get(), s};
  const uint32_t cap = (uint32_t)std::min<uint64_t>(n, 1u << 20);
  uint32_t *head_p = sc.get<uint32_t>(cap);
  uint64_t *head_start = sc.get<uint64_t>(cap);
  uint32_t *nheads = sc.get<uint32_t>(1);
  NEED(head_p); NEED(head_start); NEED(nheads);
  CK(cudaMemsetAsync(nheads, 0, 4, s));
  {
    KTimer kt(ctx, s, "index_gather", 8ull * n + 8ull * n + 12ull * n);
    launch_index_gather(words, n, ib, p_lo, T->s, T->o, idx->s, idx->p, idx->o, head_p,
                        head_start, nheads, cap, s);
    CKL("index_gather");
  }
  CK(cudaMemcpyAsync(ctx->pinned, nheads, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  const uint32_t R = reinterpret_cast<const uint32_t *>(ctx->pinned)[0];
  if (R > cap) return set_error(ctx, MAPSQ_E_UNSUPPORTED, "more than 2^20 distinct predicates");
  std::vector<uint32_t> hp(R);
  std::vector<uint64_t> hs(R);
  CK(cudaMemcpyAsync(hp.data(), head_p, 4ull * R, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hs.data(), head_start, 8ull * R, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<uint32_t> ord(R);
  for (uint32_t i = 0; i < R; i++) ord[i] = i;
  std::sort(ord.begin(), ord.end(), [&](uint32_t a, uint32_t b) { return hs[a] < hs[b]; });
  idx->pred.resize(R);
  idx->start.assign(R + 1, n);
  for (uint32_t i = 0; i < R; i++) {
    idx->pred[i] = hp[ord[i]];
    idx->start[i] = hs[ord[i]];
  }
  uint64_t *starts = sc.get<uint64_t>(R + 1);
  uint32_t *bnd = sc.get<uint32_t>(4ull * R);
  NEED(starts); NEED(bnd);
  CK(cudaMemcpyAsync(starts, idx->start.data(), 8ull * (R + 1), cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(bnd, 0xff, 8ull * R, s));
  CK(cudaMemsetAsync(bnd + 2ull * R, 0, 8ull * R, s));
  {
    KTimer kt(ctx, s, "index_bounds", 8ull * n);
    launch_index_bounds(idx->s, idx->o, n, starts, R, bnd, s);
    CKL("index_bounds");
  }
  std::vector<uint32_t> hb(4ull * R);
  CK(cudaMemcpyAsync(hb.data(), bnd, 16ull * R, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  idx->slo.assign(hb.begin(), hb.begin() + R);
  idx->olo.assign(hb.begin() + R, hb.begin() + 2 * R);
  idx->shi.assign(hb.begin() + 2 * R, hb.begin() + 3 * R);
  idx->ohi.assign(hb.begin() + 3 * R, hb.end());
  guard.keep = true;
  *out = idx.release();
  return MAPSQ_OK;
}

// position of predicate p in idx->pred, or -1
int64_t index_find(const mapsq_index *idx, uint32_t p) {
  auto it = std::lower_bound(idx->pred.begin(), idx->pred.end(), p);
  if (it == idx->pred.end() || *it != p) return -1;
  return it - idx->pred.begin();
}

mapsq_status scan_indexed_impl(mapsq_ctx *ctx, const mapsq_index *idx, const mapsq_pattern *pats,
                               int k, mapsq_table *out, cudaStream_t s) {
  if (!out) return set_error(ctx, MAPSQ_E_INVALID, "out is NULL");
  for (int j = 0; j < k && j < MAPSQ_MAX_PATTERNS; j++) clear_table(&out[j]);
  if (!idx) return set_error(ctx, MAPSQ_E_INVALID, "index is NULL");
  {
    ScanArgs a;  // validation + schemas, exactly as the unindexed scan
    int32_t vars[MAPSQ_MAX_PATTERNS][3];
    TRY(build_scan_args(ctx, pats, k, &a, vars));
  }
  // groups: patterns scanned over one row range of the permuted table
  struct Group { uint64_t b, e; std::vector<int> pats; };
  std::vector<Group> groups;
  for (int j = 0; j < k; j++) {
    const mapsq_pattern &P = pats[j];
    uint64_t b = 0, e = idx->n;
    int64_t r = -2;
    if (P.var[1] < 0) {
      r = index_find(idx, P.id[1]);
      b = r >= 0 ? idx->start[r] : 0;
      e = r >= 0 ? idx->start[r + 1] : 0;
    }
    const bool view = P.var[1] < 0 && P.var[0] >= 0 && P.var[2] >= 0 && P.var[0] != P.var[2];
    if (view || r == -1) {
      // zero-copy view of the predicate's s/o range (or an empty table: p absent)
      mapsq_table &t = out[j];
      clear_table(&t);
      const bool pure = view;
      uint32_t nc = 0;
      const uint32_t *srcs[3] = {idx->s + b, idx->p + b, idx->o + b};
      for (int q = 0; q < 3; q++) {
        const int32_t v = P.var[q];
        if (v < 0) continue;
        bool dup = false;
        for (uint32_t c = 0; c < nc; c++) dup |= t.var[c] == v;
        if (dup) continue;
        t.var[nc] = v;
        t.col[nc] = (r >= 0 && pure) ? const_cast<uint32_t *>(srcs[q]) : nullptr;
        if (r >= 0 && pure) {
          t.lo[nc] = q == 0 ? idx->slo[r] : idx->olo[r];
          t.hi[nc] = q == 0 ? idx->shi[r] : idx->ohi[r];
        }
        nc++;
      }
      t.ncols = nc;
      t.nrows = r >= 0 ? e - b : 0;
      t.flags = MAPSQ_TABLE_BOUNDS;
      t.owner = nullptr;
      continue;
    }
    bool placed = false;
    for (auto &g : groups)
      if (g.b == b && g.e == e) {
        g.pats.push_back(j);
        placed = true;
      }
    if (!placed) groups.push_back(Group{b, e, {j}});
  }
  ctx->counters.scans += k;
  for (size_t gi = 0; gi < groups.size(); gi++) {
    const Group &g = groups[gi];
    mapsq_triples V{g.e - g.b, idx->s + g.b, idx->p + g.b, idx->o + g.b};
    mapsq_pattern gp[MAPSQ_MAX_PATTERNS];
    mapsq_table gt[MAPSQ_MAX_PATTERNS];
    for (size_t q = 0; q < g.pats.size(); q++) gp[q] = pats[g.pats[q]];
    ctx->counters.scans -= g.pats.size();  // (scan_impl counts them again)
    mapsq_status st = scan_impl(ctx, &V, gp, (int)g.pats.size(), gt, s);
    if (st != MAPSQ_OK) {
      for (int j = 0; j < k; j++) {
        dfree(ctx, out[j].owner, s);
        clear_table(&out[j]);
      }
      return st;
    }
    for (size_t q = 0; q < g.pats.size(); q++) out[g.pats[q]] = gt[q];
  }
  return MAPSQ_OK;
}

// ------------------------------------------------------------------------------ query
mapsq_status query_impl(mapsq_ctx *ctx, const mapsq_triples *T, const mapsq_pattern *pats,
                        int npats, const int32_t *proj, int nproj, mapsq_table *rs,
                        cudaStream_t s, const mapsq_index *idx = nullptr,
                        const JoinStep *step = nullptr) {
  if (!rs) return set_error(ctx, MAPSQ_E_INVALID, "rs is NULL");
  clear_table(rs);
  if (!pats || npats < 1 || npats > MAPSQ_MAX_PATTERNS)
    return set_error(ctx, MAPSQ_E_INVALID, "pattern count out of range");
  if (nproj < 0 || nproj > MAPSQ_MAX_COLS || (nproj > 0 && !proj))
    return set_error(ctx, MAPSQ_E_INVALID, "bad projection");
  // first-appearance variable order and connectivity
  std::vector<int32_t> order;
  for (int i = 0; i < npats; i++) {
    bool shares = (i == 0);
    for (int q = 0; q < 3; q++) {
      const int32_t v = pats[i].var[q];
      if (v < 0) continue;
      if (std::find(order.begin(), order.end(), v) != order.end()) {
        // shared with an EARLIER pattern?
        for (int j = 0; j < i && !shares; j++)
          for (int r = 0; r < 3; r++)
            if (pats[j].var[r] == v) shares = true;
      }
    }
    for (int q = 0; q < 3; q++) {
      const int32_t v = pats[i].var[q];
      if (v >= 0 && std::find(order.begin(), order.end(), v) == order.end()) order.push_back(v);
    }
    if (!shares)
      return set_error(ctx, MAPSQ_E_NO_SHARED, "pattern " + std::to_string(i) +
                                                   " shares no variable with the patterns before it");
  }
  std::vector<int32_t> want(proj, proj + nproj);
  if (nproj == 0) want = order;
  if (want.size() > MAPSQ_MAX_COLS) return set_error(ctx, MAPSQ_E_INVALID, "projection too wide");
  for (int32_t v : want)
    if (std::find(order.begin(), order.end(), v) == order.end())
      return set_error(ctx, MAPSQ_E_INVALID, "projected variable not in the query");

  mapsq_table tabs[MAPSQ_MAX_PATTERNS];
  if (idx)
    TRY(scan_indexed_impl(ctx, idx, pats, npats, tabs, s));
  else
    TRY(scan_impl(ctx, T, pats, npats, tabs, s));
  mapsq_table acc = tabs[0];
  for (int i = 1; i < npats; i++) {
    mapsq_table r;
    mapsq_status st = step ? (*step)(&acc, &tabs[i], &r, s) : join_impl(ctx, &acc, &tabs[i], &r, s);
    dfree(ctx, acc.owner, s);
    dfree(ctx, tabs[i].owner, s);
    if (st != MAPSQ_OK) {
      for (int j = i + 1; j < npats; j++) dfree(ctx, tabs[j].owner, s);
      return st;
    }
    acc = r;
  }
  // projection: zero-copy column selection (bag semantics)
  mapsq_table out;
  clear_table(&out);
  out.nrows = acc.nrows;
  out.ncols = (uint32_t)want.size();
  out.owner = acc.owner;
  out.flags = acc.flags;
  for (uint32_t c = 0; c < out.ncols; c++) {
    for (uint32_t k = 0; k < acc.ncols; k++)
      if (acc.var[k] == want[c]) {
        out.var[c] = want[c];
        out.col[c] = acc.col[k];
        out.lo[c] = acc.lo[k];
        out.hi[c] = acc.hi[k];
      }
  }
  *rs = out;
  return MAPSQ_OK;
}

}  // namespace

// entry points for dist.cu (the distributed join and query reuse the single-GPU operators)
namespace mapsq {
mapsq_status api_enter(mapsq_ctx *ctx) { return enter(ctx); }
mapsq_status api_check_table(mapsq_ctx *ctx, const mapsq_table *t, const char *name) {
  return check_table(ctx, t, name);
}
mapsq_status api_ensure_pinned(mapsq_ctx *ctx, size_t words) { return ensure_pinned(ctx, words); }
mapsq_status join_tables(mapsq_ctx *ctx, const mapsq_table *a, const mapsq_table *b,
                         mapsq_table *rs, cudaStream_t s) {
  return join_impl(ctx, a, b, rs, s);
}
mapsq_status query_fold(mapsq_ctx *ctx, const mapsq_triples *T, const mapsq_index *idx,
                        const mapsq_pattern *pats, int npats, const int32_t *proj, int nproj,
                        mapsq_table *rs, cudaStream_t s, const JoinStep *step) {
  return query_impl(ctx, T, pats, npats, proj, nproj, rs, s, idx, step);
}
}  // namespace mapsq

// ================================================================================ C ABI
MAPSQ_API const char *mapsq_version(void) { return "mapsq-b200 0.1 (sm_100a)"; }

MAPSQ_API mapsq_status mapsq_create(mapsq_ctx **out, int device, const mapsq_allocator *al) {
  if (!out) return MAPSQ_E_INVALID;
  *out = nullptr;
  mapsq_ctx *ctx = new (std::nothrow) mapsq_ctx();
  if (!ctx) return MAPSQ_E_NOMEM;
  ctx->device = device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    delete ctx;
    return MAPSQ_E_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    delete ctx;
    return MAPSQ_E_CUDA;
  }
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  int l2 = 0;
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, device);
  ctx->l2_bytes = (size_t)l2;
  if (al && al->alloc && al->free) {
    ctx->alloc = *al;
    ctx->custom_alloc = true;
  } else {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  *out = ctx;
  return MAPSQ_OK;
}

MAPSQ_API void mapsq_destroy(mapsq_ctx *ctx) {
  if (!ctx) return;
  for (auto &p : ctx->pending) {
    cudaEventDestroy(p.ev0);
    cudaEventDestroy(p.ev1);
  }
  for (auto e : ctx->free_events) cudaEventDestroy(e);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  if (ctx->host_arena) cudaFreeHost(ctx->host_arena);
  if (ctx->arena) cudaFree(ctx->arena);
  if (ctx->arena_ev) cudaEventDestroy(ctx->arena_ev);
  dist_free(ctx);
  if (ctx->copy_stream) cudaStreamDestroy(ctx->copy_stream);
  if (ctx->unpack_stream) cudaStreamDestroy(ctx->unpack_stream);
  delete ctx;
}

MAPSQ_API const char *mapsq_last_error(const mapsq_ctx *ctx) {
  return ctx ? ctx->err.c_str() : "no context";
}

MAPSQ_API void mapsq_table_release(mapsq_ctx *ctx, mapsq_table *t, void *stream) {
  if (!ctx || !t) return;
  if (t->owner) dfree(ctx, t->owner, S(stream));
  clear_table(t);
}

MAPSQ_API mapsq_status mapsq_scan_patterns(mapsq_ctx *ctx, const mapsq_triples *T,
                                           const mapsq_pattern *pats, int k, mapsq_table *out,
                                           void *stream) {
  TRY(enter(ctx));
  return scan_impl(ctx, T, pats, k, out, S(stream));
}

MAPSQ_API mapsq_status mapsq_scan_pattern(mapsq_ctx *ctx, const mapsq_triples *T,
                                          const mapsq_pattern *pat, mapsq_table *out,
                                          void *stream) {
  TRY(enter(ctx));
  return scan_impl(ctx, T, pat, 1, out, S(stream));
}

MAPSQ_API mapsq_status mapsq_index_build(mapsq_ctx *ctx, const mapsq_triples *T,
                                         mapsq_index **out, void *stream) {
  TRY(enter(ctx));
  return index_build_impl(ctx, T, out, S(stream));
}

MAPSQ_API void mapsq_index_destroy(mapsq_ctx *ctx, mapsq_index *idx) {
  if (!idx) return;
  if (idx->owner && ctx) {
    cudaSetDevice(ctx->device);
    cudaDeviceSynchronize();  // no enqueued work may still read the index
    dfree(ctx, idx->owner, nullptr);
    cudaStreamSynchronize(nullptr);
  }
  delete idx;
}

MAPSQ_API mapsq_status mapsq_index_triples(const mapsq_index *idx, mapsq_triples *out,
                                           uint32_t *npreds) {
  if (!idx || !out) return MAPSQ_E_INVALID;
  *out = mapsq_triples{idx->n, idx->s, idx->p, idx->o};
  if (npreds) *npreds = (uint32_t)idx->pred.size();
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_index_range(const mapsq_index *idx, uint32_t p, uint64_t *begin,
                                         uint64_t *end) {
  if (!idx || !begin || !end) return MAPSQ_E_INVALID;
  const int64_t r = index_find(idx, p);
  *begin = r >= 0 ? idx->start[r] : 0;
  *end = r >= 0 ? idx->start[r + 1] : 0;
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_scan_patterns_indexed(mapsq_ctx *ctx, const mapsq_index *idx,
                                                   const mapsq_pattern *pats, int k,
                                                   mapsq_table *out, void *stream) {
  TRY(enter(ctx));
  return scan_indexed_impl(ctx, idx, pats, k, out, S(stream));
}

MAPSQ_API mapsq_status mapsq_query_indexed(mapsq_ctx *ctx, const mapsq_index *idx,
                                           const mapsq_pattern *pats, int npats,
                                           const int32_t *proj, int nproj, mapsq_table *rs,
                                           void *stream) {
  TRY(enter(ctx));
  if (!idx) return set_error(ctx, MAPSQ_E_INVALID, "index is NULL");
  return query_impl(ctx, nullptr, pats, npats, proj, nproj, rs, S(stream), idx);
}

MAPSQ_API mapsq_status mapsq_plan_join(const mapsq_table *tp1, const mapsq_table *tp2,
                                       mapsq_join_plan *plan) {
  if (!plan) return MAPSQ_E_INVALID;
  return plan_join(nullptr, tp1, tp2, plan);
}

MAPSQ_API mapsq_status mapsq_plan_join_mode(const mapsq_table *tp1, const mapsq_table *tp2,
                                            int wide_mode, mapsq_join_plan *plan) {
  if (!plan || wide_mode < MAPSQ_WIDE_KEY_RESIDUAL || wide_mode > MAPSQ_WIDE_KEY_HASH)
    return MAPSQ_E_INVALID;
  return plan_join(nullptr, tp1, tp2, plan, wide_mode);
}

MAPSQ_API mapsq_status mapsq_join(mapsq_ctx *ctx, const mapsq_table *tp1, const mapsq_table *tp2,
                                  mapsq_table *rs, void *stream) {
  TRY(enter(ctx));
  if (!rs) return set_error(ctx, MAPSQ_E_INVALID, "rs is NULL");
  return join_impl(ctx, tp1, tp2, rs, S(stream));
}

MAPSQ_API mapsq_status mapsq_query(mapsq_ctx *ctx, const mapsq_triples *T,
                                   const mapsq_pattern *pats, int npats, const int32_t *proj,
                                   int nproj, mapsq_table *rs, void *stream) {
  TRY(enter(ctx));
  return query_impl(ctx, T, pats, npats, proj, nproj, rs, S(stream));
}

// Copy a result table into the context's pinned result arena (grown on demand) and release it;
// synchronous.  Shared by the host-buffer entry points.
static mapsq_status result_to_host(mapsq_ctx *ctx, mapsq_table *rs, cudaStream_t s,
                                   uint64_t *host_rows, uint32_t *out_ncols, int32_t *out_var,
                                   uint32_t **host_cols) {
  const uint64_t m = rs->nrows;
  const uint32_t w = rs->ncols;
  const size_t need = std::max<size_t>(16, (size_t)m * w * sizeof(uint32_t));
  if (need > ctx->host_arena_bytes) {
    if (ctx->host_arena) cudaFreeHost(ctx->host_arena);
    ctx->host_arena = nullptr;
    ctx->host_arena_bytes = 0;
    cudaError_t e = cudaMallocHost(&ctx->host_arena, need);
    if (e != cudaSuccess) {
      ctx->host_arena = nullptr;
      mapsq_table_release(ctx, rs, s);
      return cuda_check(ctx, e, "cudaMallocHost(result arena)");
    }
    ctx->host_arena_bytes = need;
  }
  uint32_t *arena = static_cast<uint32_t *>(ctx->host_arena);
  mapsq_status st = MAPSQ_OK;
  for (uint32_t c = 0; c < w; c++) {
    out_var[c] = rs->var[c];
    host_cols[c] = arena + (size_t)c * m;
    if (m && st == MAPSQ_OK) {
      cudaError_t e = cudaMemcpyAsync(host_cols[c], rs->col[c], m * 4, cudaMemcpyDeviceToHost, s);
      if (e != cudaSuccess) st = cuda_check(ctx, e, "D2H result");
    }
  }
  cudaError_t e = cudaStreamSynchronize(s);
  mapsq_table_release(ctx, rs, s);
  if (st == MAPSQ_OK && e != cudaSuccess) st = cuda_check(ctx, e, "sync");
  if (st != MAPSQ_OK) return st;
  *out_ncols = w;
  *host_rows = m;
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_query_host(mapsq_ctx *ctx, uint64_t n, const uint32_t *s_host,
                                        const uint32_t *p_host, const uint32_t *o_host,
                                        const mapsq_pattern *pats, int npats,
                                        const int32_t *proj, int nproj, uint64_t *host_rows,
                                        uint32_t *out_ncols, int32_t *out_var,
                                        uint32_t **host_cols, void *stream) {
  TRY(enter(ctx));
  if (!host_rows || !out_ncols || !out_var || !host_cols || (n && (!s_host || !p_host || !o_host)))
    return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  *host_rows = 0;
  *out_ncols = 0;
  cudaStream_t s = S(stream);
  mapsq_table rs;
  {
    Scratch sc(ctx, s);
    uint32_t *d = sc.get<uint32_t>(3 * n + 12);
    NEED(d);
    uint32_t *ds = d, *dp = d + n, *dob = d + 2 * n;
    // H2D in chunks (one copy engine stream); the scan starts once the table is resident
    const uint64_t chunk = 1ull << 26;
    for (uint64_t off = 0; off < n; off += chunk) {
      const uint64_t c = std::min(chunk, n - off);
      CK(cudaMemcpyAsync(ds + off, s_host + off, c * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dp + off, p_host + off, c * 4, cudaMemcpyHostToDevice, s));
      CK(cudaMemcpyAsync(dob + off, o_host + off, c * 4, cudaMemcpyHostToDevice, s));
    }
    mapsq_triples T{n, ds, dp, dob};
    TRY(query_impl(ctx, &T, pats, npats, proj, nproj, &rs, s));
  }
  return result_to_host(ctx, &rs, s, host_rows, out_ncols, out_var, host_cols);
}

// ------------------------------------------------------------------ host-resident index (e2e)
struct mapsq_host_index {
  uint64_t n = 0;
  uint32_t *s = nullptr, *p = nullptr, *o = nullptr;  // pinned, one allocation at s (plain)
  // compressed mirror (hoststore.cu): one frame-of-reference segment per (range, column s/p/o)
  uint32_t *blob = nullptr;                            // pinned
  std::vector<uint64_t> seg_off[3], seg_words[3];      // per range, in 32-bit words
  std::vector<uint32_t> pred;
  std::vector<uint64_t> start;
  std::vector<uint32_t> slo, shi, olo, ohi;
};

MAPSQ_API void mapsq_host_index_destroy(mapsq_host_index *h) {
  if (!h) return;
  if (h->s) cudaFreeHost(h->s);
  if (h->blob) cudaFreeHost(h->blob);
  delete h;
}

namespace mapsq {
// Compressed mirror: per predicate range and column, frame-of-reference blocks of 1024 values
// (hoststore.cu) — stats kernel, host layout of the segments, pack kernel, one D2H per segment.
static mapsq_status compress_index(mapsq_ctx *ctx, const mapsq_index *idx, mapsq_host_index *h,
                                   cudaStream_t s) {
  const size_t np = idx->pred.size();
  const uint32_t *cols[3] = {idx->s, idx->p, idx->o};
  // per segment: values, blocks, block offset in the concatenated stats arrays
  std::vector<uint64_t> nv(3 * np), nb(3 * np), b0(3 * np + 1, 0);
  for (size_t r = 0; r < np; r++)
    for (int c = 0; c < 3; c++) {
      const size_t g = 3 * r + c;
      nv[g] = idx->start[r + 1] - idx->start[r];
      nb[g] = for_blocks(nv[g]);
      b0[g + 1] = b0[g] + nb[g];
    }
  const uint64_t NB = b0[3 * np];
  Scratch sc(ctx, s);
  uint32_t *dbase = sc.get<uint32_t>(NB + 1), *dbits = sc.get<uint32_t>(NB + 1);
  uint32_t *ddmin = sc.get<uint32_t>(NB + 1);
  uint32_t *dwoff = sc.get<uint32_t>(NB + 3 * np + 1);
  NEED(dbase); NEED(dbits); NEED(ddmin); NEED(dwoff);
  for (size_t r = 0; r < np; r++)
    for (int c = 0; c < 3; c++) {
      const size_t g = 3 * r + c;
      launch_for_stats(cols[c] + idx->start[r], nv[g], dbase + b0[g], dbits + b0[g],
                       ddmin + b0[g], s);
    }
  CK(cudaGetLastError());
  std::vector<uint32_t> hbase(NB), hbits(NB), hdmin(NB);
  CK(cudaMemcpyAsync(hbase.data(), dbase, 4 * NB, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hbits.data(), dbits, 4 * NB, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(hdmin.data(), ddmin, 4 * NB, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  // segment layout: base[nb] | mode_bits[nb] | dmin[nb] | woff[nb + 1] | payload
  std::vector<uint64_t> soff(3 * np + 1, 0), pay(3 * np);
  std::vector<uint32_t> hwoff(NB + 3 * np);
  for (size_t g = 0; g < 3 * np; g++) {
    uint64_t w = 0;
    for (uint64_t b = 0; b < nb[g]; b++) {
      hwoff[b0[g] + g + b] = (uint32_t)w;
      w += for_block_words(hbits[b0[g] + b]);
    }
    hwoff[b0[g] + g + nb[g]] = (uint32_t)w;
    if (w >> 32) return set_error(ctx, MAPSQ_E_UNSUPPORTED, "compressed segment over 16 GB");
    pay[g] = w;
    soff[g + 1] = soff[g] + 4 * nb[g] + 1 + w;
  }
  const uint64_t total = soff[3 * np];
  void *blob = nullptr;
  CK(cudaMallocHost(&blob, 4 * std::max<uint64_t>(total, 1)));
  h->blob = static_cast<uint32_t *>(blob);
  for (int c = 0; c < 3; c++) {
    h->seg_off[c].resize(np);
    h->seg_words[c].resize(np);
  }
  for (size_t r = 0; r < np; r++)
    for (int c = 0; c < 3; c++) {
      const size_t g = 3 * r + c;
      uint32_t *seg = h->blob + soff[g];
      std::memcpy(seg, hbase.data() + b0[g], 4 * nb[g]);
      std::memcpy(seg + nb[g], hbits.data() + b0[g], 4 * nb[g]);
      std::memcpy(seg + 2 * nb[g], hdmin.data() + b0[g], 4 * nb[g]);
      std::memcpy(seg + 3 * nb[g], hwoff.data() + b0[g] + g, 4 * (nb[g] + 1));
      h->seg_off[c][r] = soff[g];
      h->seg_words[c][r] = soff[g + 1] - soff[g];
    }
  // pack every segment's payload on the device, then copy it into the pinned blob
  uint64_t maxpay = 0;
  for (uint64_t w : pay) maxpay = std::max(maxpay, w);
  uint32_t *dpay = sc.get<uint32_t>(maxpay + 1);
  NEED(dpay);
  CK(cudaMemcpyAsync(dwoff, hwoff.data(), 4 * (NB + 3 * np), cudaMemcpyHostToDevice, s));
  for (size_t r = 0; r < np; r++)
    for (int c = 0; c < 3; c++) {
      const size_t g = 3 * r + c;
      if (!pay[g]) continue;
      launch_for_pack(cols[c] + idx->start[r], nv[g], dbase + b0[g], dbits + b0[g],
                      ddmin + b0[g], dwoff + b0[g] + g, dpay, s);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h->blob + soff[g] + 4 * nb[g] + 1, dpay, 4 * pay[g],
                         cudaMemcpyDeviceToHost, s));
    }
  CK(cudaStreamSynchronize(s));
  return MAPSQ_OK;
}
}  // namespace mapsq

MAPSQ_API mapsq_status mapsq_index_to_host(mapsq_ctx *ctx, const mapsq_index *idx,
                                           mapsq_host_index **out, void *stream) {
  TRY(enter(ctx));
  if (!idx || !out) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  *out = nullptr;
  std::unique_ptr<mapsq_host_index> h(new (std::nothrow) mapsq_host_index());
  if (!h) return set_error(ctx, MAPSQ_E_NOMEM, "host allocation failed");
  h->n = idx->n;
  h->pred = idx->pred;
  h->start = idx->start;
  h->slo = idx->slo;
  h->shi = idx->shi;
  h->olo = idx->olo;
  h->ohi = idx->ohi;
  if (idx->n && ctx->host_compress) {
    TRY(compress_index(ctx, idx, h.get(), S(stream)));
  } else if (idx->n) {
    void *p = nullptr;
    CK(cudaMallocHost(&p, 12 * idx->n));
    h->s = static_cast<uint32_t *>(p);
    h->p = h->s + idx->n;
    h->o = h->p + idx->n;
    cudaStream_t s = S(stream);
    CK(cudaMemcpyAsync(h->s, idx->s, 4 * idx->n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h->p, idx->p, 4 * idx->n, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(h->o, idx->o, 4 * idx->n, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  *out = h.release();
  return MAPSQ_OK;
}

namespace mapsq {
mapsq_status query_host_indexed_impl(mapsq_ctx *ctx, const mapsq_host_index *h,
                                     const mapsq_pattern *pats, int npats, const int32_t *proj,
                                     int nproj, uint64_t *host_rows, uint32_t *out_ncols,
                                     int32_t *out_var, uint32_t **host_cols, uint64_t *h2d_bytes,
                                     void *stream, const JoinStep *step) {
  TRY(enter(ctx));
  if (!h || !host_rows || !out_ncols || !out_var || !host_cols || !pats || npats < 1 ||
      npats > MAPSQ_MAX_PATTERNS)
    return set_error(ctx, MAPSQ_E_INVALID, "bad argument");
  *host_rows = 0;
  *out_ncols = 0;
  if (h2d_bytes) *h2d_bytes = 0;
  cudaStream_t s = S(stream);
  // the predicate ranges the query touches (every row if a pattern has a variable predicate) and
  // whether a pattern scans the range (then its p column is needed; views read only s and o)
  const size_t np = h->pred.size();
  bool all = false;
  std::vector<int> need(np, 0);  // 0 no, 1 s/o, 2 s/p/o
  for (int j = 0; j < npats; j++) {
    const mapsq_pattern &P = pats[j];
    if (P.var[1] >= 0) {
      all = true;
      continue;
    }
    auto it = std::lower_bound(h->pred.begin(), h->pred.end(), P.id[1]);
    if (it == h->pred.end() || *it != P.id[1]) continue;  // absent: matches nothing
    const bool view = P.var[0] >= 0 && P.var[2] >= 0 && P.var[0] != P.var[2];
    int &nd = need[it - h->pred.begin()];
    nd = std::max(nd, view ? 1 : 2);
  }
  // pattern -> predicate range (-1: absent predicate, or the whole table when `all`)
  std::vector<int> prange(npats, -1);
  for (int j = 0; j < npats; j++)
    if (!all && pats[j].var[1] < 0) {
      auto it = std::lower_bound(h->pred.begin(), h->pred.end(), pats[j].id[1]);
      if (it != h->pred.end() && *it == pats[j].id[1]) prange[j] = (int)(it - h->pred.begin());
    }
  if (!ctx->copy_stream) CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
  if (!ctx->unpack_stream)
    CK(cudaStreamCreateWithFlags(&ctx->unpack_stream, cudaStreamNonBlocking));
  cudaStream_t cs = ctx->copy_stream, us = ctx->unpack_stream;
  mapsq_index D;  // device-side index over the copied ranges (columns owned by the scratch)
  mapsq_table rs;
  uint64_t bytes = 0;
  {
    Scratch sc(ctx, s);
    // the H2D copies run on the copy stream in the order the query first uses the ranges; the
    // compute stream waits for a range only where it first reads it (scans: up front; views: at
    // the join that consumes them), so later ranges stream in while the first joins run
    // (compressed chunks are expanded on a second stream, so that the copy engine never waits
    // for an expansion kernel)
    struct Copies {
      cudaStream_t cs, us;
      std::vector<cudaEvent_t> ev;
      ~Copies() {
        cudaStreamSynchronize(cs);  // no copy may outlive the scratch it writes
        cudaStreamSynchronize(us);
        for (cudaEvent_t e : ev)
          if (e) cudaEventDestroy(e);
      }
    } cp{cs, us, std::vector<cudaEvent_t>(np + 1, nullptr)};
    // rows per streamed chunk, a multiple of 512 (MAPSQ_STREAM_CHUNK: override, for tests)
    const uint64_t kStreamChunk =
        std::max<uint64_t>(512, (uint64_t)env_u32("MAPSQ_STREAM_CHUNK", 32u << 20) & ~511ull);
    uint64_t rows = 0, cwords = 0;
    for (size_t r = 0; r < np; r++)
      if (all || need[r]) {
        rows += h->start[r + 1] - h->start[r];
        if (h->blob)
          cwords += h->seg_words[0][r] + h->seg_words[2][r] +
                    ((all || need[r] == 2) ? h->seg_words[1][r] : 0);
      }
    const uint64_t stride = (rows + 3) & ~3ull;
    uint32_t *d = sc.get<uint32_t>(3 * stride + 12);
    NEED(d);
    // compressed mirror: the touched segments land here and are expanded into D's columns
    uint32_t *cstage = h->blob ? sc.get<uint32_t>(cwords + 4) : nullptr;
    if (h->blob) NEED(cstage);
    uint64_t cpos = 0;
    D.n = rows;
    D.s = d;
    D.p = d + stride;
    D.o = d + 2 * stride;
    D.start.push_back(0);
    std::vector<uint64_t> at(np, 0);
    for (size_t r = 0; r < np; r++) {
      if (!all && !need[r]) continue;
      at[r] = D.start.back();
      D.pred.push_back(h->pred[r]);
      D.start.push_back(at[r] + h->start[r + 1] - h->start[r]);
      D.slo.push_back(h->slo[r]);
      D.shi.push_back(h->shi[r]);
      D.olo.push_back(h->olo[r]);
      D.ohi.push_back(h->ohi[r]);
    }
    // MAPSQ_DEBUG: the copy stream's range completion times and the joins' / readback's end,
    // relative to the query's start (timing events; stderr)
    struct DbgEvents {  // (destroyed on every exit path)
      std::vector<cudaEvent_t> v;
      ~DbgEvents() {
        for (cudaEvent_t e : v) cudaEventDestroy(e);
      }
    } dbgev;
    std::vector<cudaEvent_t> &dbg = dbgev.v;
    auto dbg_mark = [&](cudaStream_t st) {
      if (!debug_on()) return;
      cudaEvent_t e;
      cudaEventCreate(&e);
      cudaEventRecord(e, st);
      dbg.push_back(e);
    };
    dbg_mark(s);
    // the scratch may still be read by earlier work on s: the copies start after it
    CK(cudaEventCreateWithFlags(&cp.ev[np], cudaEventDisableTiming));
    CK(cudaEventRecord(cp.ev[np], s));
    CK(cudaStreamWaitEvent(cs, cp.ev[np], 0));
    // A range is copied in chunks of kStreamChunk rows (one event each) so that a join whose
    // Tp2 it is can start on the first chunks (JoinStep below, ctx->stream_b).
    // MAPSQ_DEBUG_COPY_DELAY=<us>: before each chunk the copy stream poisons the chunk's rows and
    // sleeps — a read that does not wait for its chunk then sees the poison (tests).
    const uint32_t delay_us = env_u32("MAPSQ_DEBUG_COPY_DELAY", 0);
    std::vector<StreamIn> streams(np);
    auto copy_range = [&](size_t r) -> mapsq_status {
      const uint64_t b = h->start[r], c = h->start[r + 1] - b;
      const bool with_p = all || need[r] == 2;
      StreamIn &si = streams[r];
      si.rows = c;
      si.chunk_rows = c > 2 * kStreamChunk ? kStreamChunk : std::max<uint64_t>(c, 1);
      // compressed segments: every column's segment is staged whole in cstage (headers, then
      // each chunk's payload words), and a chunk's blocks are expanded once they have landed
      uint64_t cw[3] = {0, 0, 0};
      const uint64_t nb = for_blocks(c);
      if (h->blob)
        for (int col : {0, 2, 1}) {
          if (col == 1 && !with_p) continue;
          cw[col] = cpos;
          const uint32_t *seg = h->blob + h->seg_off[col][r];
          CK(cudaMemcpyAsync(cstage + cpos, seg, 4 * (4 * nb + 1), cudaMemcpyHostToDevice, cs));
          cpos += h->seg_words[col][r];
          bytes += 4 * h->seg_words[col][r];
        }
      for (uint64_t lo = 0; lo < c || (c == 0 && lo == 0); lo += si.chunk_rows) {
        const uint64_t hi = std::min(c, lo + si.chunk_rows);
        for (int col : {0, 2, 1}) {
          if (col == 1 && !with_p) continue;
          uint32_t *dst = (col == 0 ? D.s : (col == 1 ? D.p : D.o)) + at[r];
          if (delay_us && hi > lo) CK(cudaMemsetAsync(dst + lo, 0xff, 4 * (hi - lo), cs));
        }
        if (delay_us) launch_delay_us(delay_us, cs);
        const uint64_t b0 = lo / 128, b1 = std::min(nb, (hi + 127) / 128);
        for (int col : {0, 2, 1}) {
          if (col == 1 && !with_p) continue;
          uint32_t *dst = (col == 0 ? D.s : (col == 1 ? D.p : D.o)) + at[r];
          if (hi <= lo) continue;
          if (h->blob) {
            const uint32_t *seg = h->blob + h->seg_off[col][r];
            const uint32_t *woff = seg + 3 * nb;  // (host copy of the segment's word offsets)
            const uint64_t p0 = 4 * nb + 1 + woff[b0], p1 = 4 * nb + 1 + woff[b1];
            if (p1 > p0)
              CK(cudaMemcpyAsync(cstage + cw[col] + p0, seg + p0, 4 * (p1 - p0),
                                 cudaMemcpyHostToDevice, cs));
          } else {
            const uint32_t *src = (col == 0 ? h->s : (col == 1 ? h->p : h->o)) + b;
            CK(cudaMemcpyAsync(dst + lo, src + lo, 4 * (hi - lo), cudaMemcpyHostToDevice, cs));
            bytes += 4 * (hi - lo);
          }
        }
        cudaEvent_t e;
        CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        CK(cudaEventRecord(e, cs));
        if (h->blob && hi > lo) {  // expand the chunk's blocks on the second stream
          CK(cudaStreamWaitEvent(us, e, 0));
          for (int col : {0, 2, 1}) {
            if (col == 1 && !with_p) continue;
            uint32_t *dst = (col == 0 ? D.s : (col == 1 ? D.p : D.o)) + at[r];
            launch_for_unpack_blocks(cstage + cw[col], c, b0, b1, dst, us);
            CK(cudaGetLastError());
          }
          cp.ev.push_back(e);  // (the copy event; the chunk's event is the expansion's)
          CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          CK(cudaEventRecord(e, us));
        }
        si.ev.push_back(e);
        if (c == 0) break;
      }
      // (destroyed with the copies: the last chunk's event stands for the whole range)
      cp.ev[r] = si.ev.back();
      cp.ev.insert(cp.ev.end(), si.ev.begin(), si.ev.end() - 1);
      dbg_mark(h->blob ? us : cs);
      if (debug_on()) std::fprintf(stderr, "[mapsq] e2e range %zu: %llu rows, %llu B so far\n", r,
                                   (unsigned long long)c, (unsigned long long)bytes);
      return MAPSQ_OK;
    };
    std::vector<char> copied(np, 0);
    for (int j = 0; j < npats; j++)  // first-use order
      if (prange[j] >= 0 && !copied[prange[j]]) {
        TRY(copy_range(prange[j]));
        copied[prange[j]] = 1;
      }
    for (size_t r = 0; r < np; r++)  // everything else the query reads (variable predicates)
      if ((all || need[r]) && !copied[r]) TRY(copy_range(r));
    auto wait_range = [&](int r) -> mapsq_status {
      if (r >= 0 && cp.ev[r]) CK(cudaStreamWaitEvent(s, cp.ev[r], 0));
      return MAPSQ_OK;
    };
    // scans read their ranges before the first join; so does a variable-predicate pattern
    for (int j = 0; j < npats; j++) {
      const mapsq_pattern &P = pats[j];
      const bool view = P.var[1] < 0 && P.var[0] >= 0 && P.var[2] >= 0 && P.var[0] != P.var[2];
      if (!view || all)
        for (size_t r = 0; r < np; r++)
          if (all ? true : (int)r == prange[j]) TRY(wait_range((int)r));
    }
    const JoinStep inner = step ? *step : JoinStep([ctx](const mapsq_table *a, const mapsq_table *t,
                                                         mapsq_table *out, cudaStream_t st) {
      return join_tables(ctx, a, t, out, st);
    });
    // a join waits for the copies of exactly the ranges its inputs' columns live in (zero-copy
    // views of the copied predicate ranges), whatever order the fold takes them in
    auto wait_table = [&](const mapsq_table *t) -> mapsq_status {
      for (uint32_t c = 0; c < t->ncols; c++) {
        const uint32_t *q = t->col[c];
        if (!q) continue;
        for (size_t r = 0; r < np; r++) {
          if (!cp.ev[r]) continue;
          const uint64_t len = h->start[r + 1] - h->start[r];
          for (const uint32_t *base : {D.s, D.o, D.p})
            if (q >= base + at[r] && q < base + at[r] + len) TRY(wait_range((int)r));
        }
      }
      return MAPSQ_OK;
    };
    // ... except a Tp2 that is one predicate range: the join waits for its chunks as it reads
    // them (ctx->stream_b)
    auto stream_of = [&](const mapsq_table *t) -> const StreamIn * {
      int rr = -1;
      for (uint32_t c = 0; c < t->ncols; c++) {
        const uint32_t *q = t->col[c];
        if (!q) continue;
        int hit = -1;
        for (size_t r = 0; r < np; r++) {
          if (!cp.ev[r]) continue;
          const uint64_t len = h->start[r + 1] - h->start[r];
          for (const uint32_t *base : {D.s, D.o, D.p})
            if (q == base + at[r] && t->nrows == len) hit = (int)r;
        }
        if (hit < 0 || (rr >= 0 && hit != rr)) return nullptr;
        rr = hit;
      }
      return rr >= 0 && !step ? &streams[rr] : nullptr;  // (distributed joins: whole ranges)
    };
    const JoinStep waited = [&](const mapsq_table *a, const mapsq_table *t, mapsq_table *out,
                                cudaStream_t st) -> mapsq_status {
      TRY(wait_table(a));
      const StreamIn *sb = stream_of(t);
      if (!sb) TRY(wait_table(t));
      ctx->stream_b = sb;
      const mapsq_status rc = inner(a, t, out, st);
      ctx->stream_b = nullptr;
      return rc;
    };
    TRY(query_impl(ctx, nullptr, pats, npats, proj, nproj, &rs, s, &D, &waited));
    for (size_t r = 0; r < np; r++) TRY(wait_range((int)r));  // (a one-pattern view result)
    dbg_mark(s);
    // the result may be a zero-copy view of the copied ranges: read it back inside this scope
    TRY(result_to_host(ctx, &rs, s, host_rows, out_ncols, out_var, host_cols));
    dbg_mark(s);
    if (!dbg.empty()) {
      cudaStreamSynchronize(s);
      cudaStreamSynchronize(cs);
      std::string line = "[mapsq] e2e ms from start: ranges";
      for (size_t i = 1; i < dbg.size(); i++) {
        float ms = 0;
        cudaEventElapsedTime(&ms, dbg[0], dbg[i]);
        line += (i + 2 == dbg.size() ? " | joins " : (i + 1 == dbg.size() ? " | readback " : " ")) +
                std::to_string(ms);
      }
      std::fprintf(stderr, "%s\n", line.c_str());
    }
  }
  if (h2d_bytes) *h2d_bytes = bytes;
  return MAPSQ_OK;
}
}  // namespace mapsq

MAPSQ_API mapsq_status mapsq_query_host_indexed(mapsq_ctx *ctx, const mapsq_host_index *h,
                                                const mapsq_pattern *pats, int npats,
                                                const int32_t *proj, int nproj,
                                                uint64_t *host_rows, uint32_t *out_ncols,
                                                int32_t *out_var, uint32_t **host_cols,
                                                uint64_t *h2d_bytes, void *stream) {
  return query_host_indexed_impl(ctx, h, pats, npats, proj, nproj, host_rows, out_ncols, out_var,
                                 host_cols, h2d_bytes, stream, nullptr);
}

MAPSQ_API mapsq_status mapsq_table_bounds(mapsq_ctx *ctx, mapsq_table *t, void *stream) {
  TRY(enter(ctx));
  TRY(check_table(ctx, t, "table"));
  t->flags &= ~MAPSQ_TABLE_BOUNDS;
  return bounds_of(ctx, t, S(stream));
}

MAPSQ_API mapsq_status mapsq_map_words(mapsq_ctx *ctx, const mapsq_table *tp1,
                                       const mapsq_table *tp2, const mapsq_join_plan *plan,
                                       uint64_t *words, void *stream) {
  TRY(enter(ctx));
  if (!plan || !words || !tp1 || !tp2) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  if (plan->path == MAPSQ_PATH_KV) return set_error(ctx, MAPSQ_E_INVALID, "map_words needs a P64 or RESIDUAL plan");
  if (plan->n1 + plan->n2 == 0) return MAPSQ_OK;
  cudaStream_t s = S(stream);
  Scratch sc(ctx, s);
  uint32_t *hist = sc.get<uint32_t>(kMaxPasses * kRadix);
  NEED(hist);
  CK(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
  const PackArgs pa = pack_args(*plan, tp1, tp2);
  KTimer kt(ctx, s, "pack_hist", 4ull * plan->nshared * (plan->n1 + plan->n2) + 8ull * (plan->n1 + plan->n2));
  launch_pack_hist(pa, words, nullptr, hist, s);
  CKL("pack_hist");
  return MAPSQ_OK;
}

static mapsq_status sort_entry(mapsq_ctx *ctx, uint64_t *keys, uint32_t *vals, uint64_t n,
                               uint32_t bit_lo, uint32_t bit_hi, cudaStream_t s) {
  if (!keys || bit_hi > 64 || bit_lo > bit_hi) return set_error(ctx, MAPSQ_E_INVALID, "bad sort arguments");
  const uint32_t nbits = bit_hi - bit_lo;
  if (n < 2 || nbits == 0) return MAPSQ_OK;
  if (n >= (1ull << 32)) return set_error(ctx, MAPSQ_E_INVALID, "n must be < 2^32");
  Scratch sc(ctx, s);
  uint64_t *kb_ = sc.get<uint64_t>(n);
  uint32_t *vb = vals ? sc.get<uint32_t>(n) : nullptr;
  uint32_t *hist = sc.get<uint32_t>(kMaxPasses * kRadix);
  NEED(kb_);
  NEED(hist);
  if (vals) NEED(vb);
  const uint32_t passes = (nbits + 7) / 8;
  CK(cudaMemsetAsync(hist, 0, kMaxPasses * kRadix * sizeof(uint32_t), s));
  {
    KTimer kt(ctx, s, "key_hist", 8ull * n);
    launch_key_hist(keys, n, bit_lo, 1, passes == 1 ? nbits : 8, hist, s);  // first digit only
    CKL("key_hist");
  }
  int which = 0;
  TRY(radix_sort(ctx, keys, kb_, vals, vb, n, bit_lo, nbits, hist, sc, s, &which));
  if (which) {
    CK(cudaMemcpyAsync(keys, kb_, n * 8, cudaMemcpyDeviceToDevice, s));
    if (vals) CK(cudaMemcpyAsync(vals, vb, n * 4, cudaMemcpyDeviceToDevice, s));
  }
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_sort_words(mapsq_ctx *ctx, uint64_t *words, uint64_t n,
                                        uint32_t bit_lo, uint32_t bit_hi, void *stream) {
  TRY(enter(ctx));
  return sort_entry(ctx, words, nullptr, n, bit_lo, bit_hi, S(stream));
}

MAPSQ_API mapsq_status mapsq_sort_pairs(mapsq_ctx *ctx, uint64_t *keys, uint32_t *vals,
                                        uint64_t n, uint32_t bit_lo, uint32_t bit_hi,
                                        void *stream) {
  TRY(enter(ctx));
  if (!vals) return set_error(ctx, MAPSQ_E_INVALID, "vals is NULL");
  return sort_entry(ctx, keys, vals, n, bit_lo, bit_hi, S(stream));
}

MAPSQ_API mapsq_status mapsq_reduce_groups(mapsq_ctx *ctx, const uint64_t *words, uint64_t n1,
                                           uint64_t n2, uint32_t ib, uint32_t *group_start,
                                           uint32_t *group_split, uint32_t *group_end,
                                           uint64_t *group_off, uint64_t *ngroups,
                                           uint64_t *total, void *stream) {
  TRY(enter(ctx));
  if (!ngroups || !total) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  *ngroups = *total = 0;
  const uint64_t n = n1 + n2, cap = std::min(n1, n2);
  if (n == 0 || cap == 0) return MAPSQ_OK;
  if (!words || !group_start || !group_split || !group_end || !group_off || ib > 32)
    return set_error(ctx, MAPSQ_E_INVALID, "bad reduce arguments");
  cudaStream_t s = S(stream);
  Scratch sc(ctx, s);
  uint64_t *gc = sc.get<uint64_t>(cap);
  const uint64_t gtiles = find_groups_tiles(n);
  uint64_t *gstatus = sc.get<uint64_t>(gtiles);
  uint64_t *scal = sc.get<uint64_t>(4);
  uint64_t *tmp = sc.get<uint64_t>(scan_tmp_words(cap));
  NEED(gc); NEED(gstatus); NEED(scal); NEED(tmp);
  CK(cudaMemsetAsync(gstatus, 0, gtiles * sizeof(uint64_t), s));
  CK(cudaMemsetAsync(scal, 0, 4 * sizeof(uint64_t), s));
  {
    KTimer kt(ctx, s, "find_groups", n * 8ull);
    GroupOut g{group_start, group_split, group_end, gc};
    launch_find_groups(words, nullptr, nullptr, n, n1, ib, g, gstatus,
                       reinterpret_cast<uint32_t *>(scal + 2), scal, s);
    CKL("find_groups");
  }
  {
    KTimer kt(ctx, s, "scan_counts", cap * 16ull);
    launch_exclusive_scan_u64_dev(gc, group_off, scal, cap, tmp, scal + 1, s);
    CKL("scan_counts");
  }
  TRY(ensure_pinned(ctx, 2));
  CK(cudaMemcpyAsync(ctx->pinned, scal, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  *ngroups = ctx->pinned[0];
  *total = ctx->pinned[1];
  return MAPSQ_OK;
}

// ------------------------------------------------------------------ partition (row e, K8)
struct mapsq_partition_state {
  PartArgs pa;
  uint64_t ntiles;
  uint64_t *tile_off;   // dest-major exclusive offsets of the per-tile counts (+ total)
  uint64_t *tables;     // device: dst_row[nparts] then dst_cols[nparts * ncols]
  uint64_t counts[kMaxParts];
};

MAPSQ_API void mapsq_partition_state_free(mapsq_ctx *ctx, mapsq_partition_state *st) {
  if (!ctx || !st) return;
  cudaStream_t s = nullptr;
  if (st->tile_off) dfree(ctx, st->tile_off, s);
  if (st->tables) dfree(ctx, st->tables, s);
  delete st;
}

MAPSQ_API mapsq_status mapsq_partition_plan(mapsq_ctx *ctx, const mapsq_table *in,
                                            const int32_t *key_vars, int nkey, int nparts,
                                            uint64_t *counts_host, mapsq_partition_state **state,
                                            void *stream) {
  return mapsq_partition_plan_masked(ctx, in, key_vars, nkey, nparts, nullptr, counts_host, state,
                                     stream);
}

MAPSQ_API mapsq_status mapsq_partition_plan_masked(mapsq_ctx *ctx, const mapsq_table *in,
                                                   const int32_t *key_vars, int nkey, int nparts,
                                                   const uint32_t *row_mask, uint64_t *counts_host,
                                                   mapsq_partition_state **state, void *stream) {
  return mapsq::partition_plan_impl(ctx, in, key_vars, nkey, nparts, row_mask, nullptr, 0, 0,
                                    counts_host, state, stream);
}

namespace mapsq {
// K8 plan; rows whose key equals one of the nheavy keys heavy[h * kMaxHeavyCols ..] (skew
// handling, dist.cu; nkey <= kMaxHeavyCols) go to destination `self` instead of their hash.
mapsq_status partition_plan_impl(mapsq_ctx *ctx, const mapsq_table *in, const int32_t *key_vars,
                                 int nkey, int nparts, const uint32_t *row_mask,
                                 const uint32_t *heavy, int nheavy, int self,
                                 uint64_t *counts_host, mapsq_partition_state **state,
                                 void *stream) {
  TRY(enter(ctx));
  if (!state || !counts_host || !key_vars) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  *state = nullptr;
  TRY(check_table(ctx, in, "in"));
  if (nparts < 1 || nparts > kMaxParts || nkey < 1 || nkey > (int)in->ncols)
    return set_error(ctx, MAPSQ_E_INVALID, "bad partition arguments");
  cudaStream_t s = S(stream);
  auto *st = new (std::nothrow) mapsq_partition_state();
  if (!st) return set_error(ctx, MAPSQ_E_NOMEM, "host allocation failed");
  PartArgs &pa = st->pa;
  std::memset(&pa, 0, sizeof pa);
  pa.nkey = (uint32_t)nkey;
  for (int q = 0; q < nkey; q++) {
    int c = -1;
    for (uint32_t j = 0; j < in->ncols; j++)
      if (in->var[j] == key_vars[q]) c = (int)j;
    if (c < 0) {
      delete st;
      return set_error(ctx, MAPSQ_E_INVALID, "partition key variable not in table");
    }
    pa.key[q] = in->col[c];
  }
  pa.ncols = in->ncols;
  pa.n = in->nrows;
  pa.nparts = (uint32_t)nparts;
  pa.mask = row_mask;
  if (nheavy > 0) {
    if (nheavy > kMaxHeavy || nkey > kMaxHeavyCols || self < 0 || self >= nparts) {
      delete st;
      return set_error(ctx, MAPSQ_E_INVALID, "bad heavy-key arguments");
    }
    pa.nheavy = (uint32_t)nheavy;
    pa.self = (uint32_t)self;
    std::memcpy(pa.heavy, heavy, sizeof(uint32_t) * kMaxHeavyCols * nheavy);
  }
  for (uint32_t c = 0; c < in->ncols; c++) pa.in[c] = in->col[c];
  for (int d = 0; d < nparts; d++) counts_host[d] = st->counts[d] = 0;
  if (in->nrows == 0) {
    *state = st;
    return MAPSQ_OK;
  }
  st->ntiles = ceil_div(in->nrows, kPartTile);
  st->tile_off = static_cast<uint64_t *>(dalloc(ctx, (st->ntiles * nparts + 1) * 8, s));
  st->tables = static_cast<uint64_t *>(dalloc(ctx, (size_t)nparts * (1 + in->ncols) * 8, s));
  if (!st->tile_off || !st->tables) {
    mapsq_partition_state_free(ctx, st);
    return set_error(ctx, MAPSQ_E_NOMEM, "device allocation failed");
  }
  Scratch sc(ctx, s);
  uint32_t *th = sc.get<uint32_t>(st->ntiles * nparts);
  uint64_t *tmp = sc.get<uint64_t>(scan_tmp_words(st->ntiles * nparts));
  if (!th || !tmp) {
    mapsq_partition_state_free(ctx, st);
    return set_error(ctx, MAPSQ_E_NOMEM, "device allocation failed");
  }
  mapsq_status rc = MAPSQ_OK;
  {
    KTimer kt(ctx, s, "partition_hist", 4ull * nkey * in->nrows);
    launch_partition_hist(pa, th, st->ntiles, s);
  }
  {
    KTimer kt(ctx, s, "scan_tiles", 12ull * st->ntiles * nparts);
    launch_exclusive_scan_u32(th, st->tile_off, st->ntiles * nparts, tmp,
                              st->tile_off + st->ntiles * nparts, s);
  }
  rc = cuda_check(ctx, cudaGetLastError(), "partition_plan");
  if (rc == MAPSQ_OK) rc = ensure_pinned(ctx, nparts + 1);
  for (int d = 0; d <= nparts && rc == MAPSQ_OK; d++)
    rc = cuda_check(ctx, cudaMemcpyAsync(ctx->pinned + d, st->tile_off + (uint64_t)d * st->ntiles, 8,
                                         cudaMemcpyDeviceToHost, s), "counts D2H");
  if (rc == MAPSQ_OK) rc = cuda_check(ctx, cudaStreamSynchronize(s), "counts sync");
  if (rc != MAPSQ_OK) {
    mapsq_partition_state_free(ctx, st);
    return rc;
  }
  for (int d = 0; d < nparts; d++) counts_host[d] = st->counts[d] = ctx->pinned[d + 1] - ctx->pinned[d];
  *state = st;
  return MAPSQ_OK;
}

// The rows of `in` selected by `mask` (bit per row), in row order, into a new table (one-destination
// K8 plan + scatter).  Caller releases *out.
mapsq_status compact_rows(mapsq_ctx *ctx, const mapsq_table *in, const uint32_t *mask,
                          mapsq_table *out, cudaStream_t s) {
  clear_table(out);
  uint64_t cnt = 0;
  mapsq_partition_state *st = nullptr;
  TRY(partition_plan_impl(ctx, in, in->var, 1, 1, mask, nullptr, 0, 0, &cnt, &st, s));
  mapsq_status rc = alloc_table(ctx, out, cnt, in->ncols, s);
  if (rc == MAPSQ_OK) {
    out->flags = in->flags;
    for (uint32_t c = 0; c < in->ncols; c++) {
      out->var[c] = in->var[c];
      out->lo[c] = in->lo[c];
      out->hi[c] = in->hi[c];
    }
    if (cnt) {
      const uint64_t row0 = 0;
      rc = mapsq_partition_scatter(ctx, st, &row0, out->col, s);
    }
  }
  mapsq_partition_state_free(ctx, st);
  if (rc != MAPSQ_OK) {
    dfree(ctx, out->owner, s);
    clear_table(out);
  }
  return rc;
}
}  // namespace mapsq

MAPSQ_API mapsq_status mapsq_partition_scatter(mapsq_ctx *ctx, mapsq_partition_state *st,
                                               const uint64_t *dest_row,
                                               uint32_t *const *dest_cols, void *stream) {
  TRY(enter(ctx));
  if (!st || !dest_row || !dest_cols) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  if (st->pa.n == 0) return MAPSQ_OK;
  cudaStream_t s = S(stream);
  const uint32_t np = st->pa.nparts, nc = st->pa.ncols;
  TRY(ensure_pinned(ctx, (size_t)np * (1 + nc)));
  for (uint32_t d = 0; d < np; d++) {
    ctx->pinned[d] = dest_row[d];
    for (uint32_t c = 0; c < nc; c++) {
      const uint32_t *p = dest_cols[d * nc + c];
      if (!p && st->counts[d]) return set_error(ctx, MAPSQ_E_INVALID, "NULL destination column");
      ctx->pinned[np + d * nc + c] = (uint64_t)(uintptr_t)p;
    }
  }
  CK(cudaMemcpyAsync(st->tables, ctx->pinned, (size_t)np * (1 + nc) * 8, cudaMemcpyHostToDevice, s));
  {
    KTimer kt(ctx, s, "partition_scatter", 8ull * nc * st->pa.n);
    launch_partition_scatter(st->pa, st->tile_off, st->ntiles, st->tables, st->tables + np, s);
    CKL("partition_scatter");
  }
  // the pinned staging buffer is reused by the next call: make sure the copy has been consumed
  CK(cudaStreamSynchronize(s));
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_partition(mapsq_ctx *ctx, const mapsq_table *in,
                                       const int32_t *key_vars, int nkey, int nparts,
                                       mapsq_table *out, uint64_t *counts_host, void *stream) {
  TRY(enter(ctx));
  if (!out || !counts_host) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  clear_table(out);
  mapsq_partition_state *st = nullptr;
  TRY(mapsq_partition_plan(ctx, in, key_vars, nkey, nparts, counts_host, &st, stream));
  cudaStream_t s = S(stream);
  *out = *in;
  out->owner = nullptr;
  mapsq_status rc = alloc_table(ctx, out, in->nrows, in->ncols, s);
  if (rc == MAPSQ_OK && in->nrows) {
    // local destination: every destination's block lives in `out`, destination-major
    uint64_t rows[kMaxParts];
    uint32_t *cols[kMaxParts * MAPSQ_MAX_COLS];
    uint64_t run = 0;
    for (int d = 0; d < nparts; d++) {
      rows[d] = run;
      run += counts_host[d];
      for (uint32_t c = 0; c < in->ncols; c++) cols[d * in->ncols + c] = out->col[c];
    }
    rc = mapsq_partition_scatter(ctx, st, rows, cols, stream);
  }
  mapsq_partition_state_free(ctx, st);
  if (rc != MAPSQ_OK) {
    dfree(ctx, out->owner, s);
    clear_table(out);
  }
  return rc;
}

// ------------------------------------------------------------------ CUDA IPC (peer arenas)
MAPSQ_API mapsq_status mapsq_ipc_alloc(mapsq_ctx *ctx, size_t bytes, void **dev_ptr) {
  TRY(enter(ctx));
  if (!dev_ptr) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  *dev_ptr = nullptr;
  CK(cudaMalloc(dev_ptr, bytes ? bytes : 256));
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_ipc_free(mapsq_ctx *ctx, void *dev_ptr) {
  TRY(enter(ctx));
  if (dev_ptr) CK(cudaFree(dev_ptr));
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_ipc_export(mapsq_ctx *ctx, void *dev_ptr, void *handle64) {
  TRY(enter(ctx));
  if (!dev_ptr || !handle64) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  cudaIpcMemHandle_t h;
  CK(cudaIpcGetMemHandle(&h, dev_ptr));
  std::memcpy(handle64, &h, 64);
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_ipc_open(mapsq_ctx *ctx, const void *handle64, void **dev_ptr) {
  TRY(enter(ctx));
  if (!dev_ptr || !handle64) return set_error(ctx, MAPSQ_E_INVALID, "NULL argument");
  cudaIpcMemHandle_t h;
  std::memcpy(&h, handle64, 64);
  CK(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess));
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_ipc_close(mapsq_ctx *ctx, void *dev_ptr) {
  TRY(enter(ctx));
  CK(cudaIpcCloseMemHandle(dev_ptr));
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_set_option(mapsq_ctx *ctx, int option, int64_t value) {
  if (!ctx) return MAPSQ_E_INVALID;
  if (option == MAPSQ_OPT_WIDE_KEY && value >= MAPSQ_WIDE_KEY_RESIDUAL && value <= MAPSQ_WIDE_KEY_HASH) {
    ctx->wide_key_mode = (int)value;
    return MAPSQ_OK;
  }
  if (option == MAPSQ_OPT_SEMIJOIN && value >= MAPSQ_SEMIJOIN_OFF && value <= MAPSQ_SEMIJOIN_ON) {
    ctx->semijoin = (int)value;
    return MAPSQ_OK;
  }
  if (option == MAPSQ_OPT_SMALL_JOIN && (value == 0 || value == 1)) {
    ctx->small_joins = value != 0;
    return MAPSQ_OK;
  }
  if (option == MAPSQ_OPT_SKEW && (value == 0 || value == 1)) {
    ctx->skew = value != 0;
    return MAPSQ_OK;
  }
  if (option == MAPSQ_OPT_HOST_COMPRESS && (value == 0 || value == 1)) {
    ctx->host_compress = value != 0;
    return MAPSQ_OK;
  }
  return set_error(ctx, MAPSQ_E_INVALID, "unknown option or value");
}

MAPSQ_API mapsq_status mapsq_set_profiling(mapsq_ctx *ctx, int on) {
  if (!ctx) return MAPSQ_E_INVALID;
  ctx->profiling = on != 0;
  return MAPSQ_OK;
}

static void resolve_pending(mapsq_ctx *ctx) {
  for (auto &p : ctx->pending) {
    float ms = 0;
    cudaEventSynchronize(p.ev1);
    cudaEventElapsedTime(&ms, p.ev0, p.ev1);
    auto it = ctx->kagg.find(p.name);
    if (it == ctx->kagg.end()) {
      ctx->korder.push_back(p.name);
      it = ctx->kagg.emplace(p.name, KAgg{}).first;
    }
    it->second.launches++;
    it->second.ms += ms;
    it->second.bytes += p.bytes;
    ctx->free_events.push_back(p.ev0);
    ctx->free_events.push_back(p.ev1);
  }
  ctx->pending.clear();
}

MAPSQ_API mapsq_status mapsq_stats_reset(mapsq_ctx *ctx) {
  if (!ctx) return MAPSQ_E_INVALID;
  resolve_pending(ctx);
  ctx->kagg.clear();
  ctx->korder.clear();
  std::memset(&ctx->counters, 0, sizeof ctx->counters);
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_get_stats(mapsq_ctx *ctx, mapsq_stats *st) {
  if (!ctx || !st) return MAPSQ_E_INVALID;
  resolve_pending(ctx);
  *st = ctx->counters;
  st->nkernels = 0;
  for (const auto &name : ctx->korder) {
    if (st->nkernels >= MAPSQ_MAX_KSTATS) break;
    mapsq_kernel_stat &k = st->kernel[st->nkernels++];
    std::memset(&k, 0, sizeof k);
    std::strncpy(k.name, name.c_str(), sizeof k.name - 1);
    const KAgg &a = ctx->kagg[name];
    k.launches = a.launches;
    k.total_ms = a.ms;
    k.algo_bytes = a.bytes;
  }
  return MAPSQ_OK;
}
