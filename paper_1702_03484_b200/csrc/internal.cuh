// internal.cuh — shared internals of libmapsq: context, device helpers, kernel launchers.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <functional>
#include <map>
#include <string>
#include <vector>

#include "mapsq.h"

#define MAPSQ_API extern "C" __attribute__((visibility("default")))

namespace mapsq {

constexpr int kRadix = 256;          // 8-bit digits (MAPSQ_RADIX_BITS)
constexpr int kSortThreads = 256;    // one thread per digit in the look-back
constexpr int kSortItems = 16;       // keys per thread per tile
constexpr int kSortTile = kSortThreads * kSortItems;
constexpr int kMaxPasses = 8;        // 64 key bits / 8

// Look-back status words: [63:62] flag, [61:0] count.
constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagInc = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 62) - 1;

// ---------------------------------------------------------------- context
struct PendingTiming {
  std::string name;
  cudaEvent_t ev0, ev1;
  uint64_t bytes;
};
struct KAgg {
  uint64_t launches = 0;
  double ms = 0;
  uint64_t bytes = 0;
};
struct DistState;

}  // namespace mapsq

namespace mapsq {
// A join input whose rows arrive in chunks (mapsq_query_host_indexed: a predicate range copied
// host -> device chunk by chunk): chunk k = rows [k * chunk_rows, min(rows, (k + 1) * chunk_rows))
// is in place once ev[k] (recorded on the copy stream, in chunk order) has completed.
struct StreamIn {
  uint64_t rows = 0, chunk_rows = 0;
  std::vector<cudaEvent_t> ev;
};
}  // namespace mapsq

struct mapsq_ctx {
  int device = 0;
  int num_sms = 148;
  size_t l2_bytes = 0;
  mapsq_allocator alloc{};
  bool custom_alloc = false;
  std::string err;
  bool cuda_broken = false;
  bool profiling = false;
  int wide_key_mode = MAPSQ_WIDE_KEY_HASH;
  int semijoin = MAPSQ_SEMIJOIN_AUTO;
  bool small_joins = true;  // MAPSQ_OPT_SMALL_JOIN: one-CTA path for joins of <= 4096 rows
  bool skew = true;         // MAPSQ_OPT_SKEW: heavy keys split / broadcast in distributed joins
  bool host_compress = true;  // MAPSQ_OPT_HOST_COMPRESS: mapsq_index_to_host compresses the mirror
  std::vector<mapsq::PendingTiming> pending;
  std::vector<cudaEvent_t> free_events;
  std::map<std::string, mapsq::KAgg> kagg;
  std::vector<std::string> korder;
  mapsq_stats counters{};
  uint64_t *pinned = nullptr;  // small pinned host buffer for the blocking size reads
  size_t pinned_words = 0;
  void *host_arena = nullptr;  // pinned result arena of mapsq_query_host (reused across calls)
  size_t host_arena_bytes = 0;
  // device scratch arena: grow-only bump allocator reused by every operation (stream ordered)
  char *arena = nullptr;
  size_t arena_cap = 0, arena_used = 0, arena_demand = 0, arena_hw = 0;
  int arena_depth = 0;
  cudaStream_t arena_stream = nullptr;
  cudaEvent_t arena_ev = nullptr;
  mapsq::DistState *dist = nullptr;  // communicator + exchange arenas (dist.cu), or NULL
  cudaStream_t copy_stream = nullptr;  // H2D copies of mapsq_query_host_indexed (lazily created)
  cudaStream_t unpack_stream = nullptr;  // expansion of the compressed copies (lazily created)
  // set by mapsq_query_host_indexed around one join: its Tp2 input streams in (the join waits
  // chunk by chunk where it can — the semi-join filter's probe of the larger side — and for all
  // of it before anything else reads it)
  const mapsq::StreamIn *stream_b = nullptr;
};

namespace mapsq {

// ---------------------------------------------------------------- host helpers
mapsq_status set_error(mapsq_ctx *ctx, mapsq_status st, const std::string &msg);
// operators shared with dist.cu (api.cu)
using JoinStep = std::function<mapsq_status(const mapsq_table *acc, const mapsq_table *t,
                                            mapsq_table *out, cudaStream_t s)>;
mapsq_status api_enter(mapsq_ctx *ctx);
mapsq_status api_check_table(mapsq_ctx *ctx, const mapsq_table *t, const char *name);
mapsq_status api_ensure_pinned(mapsq_ctx *ctx, size_t words);
mapsq_status join_tables(mapsq_ctx *ctx, const mapsq_table *a, const mapsq_table *b,
                         mapsq_table *rs, cudaStream_t s);
mapsq_status query_fold(mapsq_ctx *ctx, const mapsq_triples *T, const mapsq_index *idx,
                        const mapsq_pattern *pats, int npats, const int32_t *proj, int nproj,
                        mapsq_table *rs, cudaStream_t s, const JoinStep *step);
void dist_free(mapsq_ctx *ctx);  // dist.cu: communicator, arenas, peer mappings
mapsq_status query_host_indexed_impl(mapsq_ctx *ctx, const mapsq_host_index *h,
                                     const mapsq_pattern *pats, int npats, const int32_t *proj,
                                     int nproj, uint64_t *host_rows, uint32_t *out_ncols,
                                     int32_t *out_var, uint32_t **host_cols, uint64_t *h2d_bytes,
                                     void *stream, const JoinStep *step);
mapsq_status cuda_check(mapsq_ctx *ctx, cudaError_t e, const char *what);
void *dalloc(mapsq_ctx *ctx, size_t bytes, cudaStream_t s);
void dfree(mapsq_ctx *ctx, void *p, cudaStream_t s);

// Scratch allocations of one operation.  They come from the context's grow-only arena (bump
// pointer, reset when the guard leaves scope); what does not fit is taken from the allocator and
// freed (stream ordered) on exit, and the arena grows to the observed high-water mark before the
// next operation, so steady-state operations never touch the allocator for scratch.
struct Scratch {
  mapsq_ctx *ctx;
  cudaStream_t s;
  size_t mark;
  std::vector<void *> ptrs;
  Scratch(mapsq_ctx *c, cudaStream_t st);
  ~Scratch();
  void *raw(size_t bytes);
  template <typename T>
  T *get(size_t count) {
    return static_cast<T *>(raw(count * sizeof(T) + 16));
  }
  void release(void *p) {  // only allocator-backed blocks are returned early
    for (auto &q : ptrs)
      if (q == p) {
        dfree(ctx, q, s);
        q = nullptr;
      }
  }
};

// Launch bracket: counts the launch and, while profiling, records events around it.
struct KTimer {
  mapsq_ctx *ctx;
  cudaStream_t s;
  PendingTiming t;
  bool on;
  KTimer(mapsq_ctx *c, cudaStream_t st, const char *name, uint64_t bytes, int nlaunch = 1);
  ~KTimer();
};

// Raise a kernel's dynamic shared-memory limit once per (device, kernel) (the attribute is per
// device context; a process-wide flag would skip the second device).
void set_smem_limit(const void *kernel, size_t bytes);

inline uint32_t bits_for(uint64_t range_max) {  // bits needed to represent 0..range_max
  uint32_t b = 0;
  while (b < 64 && (range_max >> b) != 0) b++;
  return b;
}
__host__ __device__ inline uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t *p, uint64_t v) {
  asm volatile("st.relaxed.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
__device__ __forceinline__ uint32_t lt_or_eq_mask(uint32_t lane) {  // lanes 0..lane
  return lane >= 31 ? 0xffffffffu : ((2u << lane) - 1u);
}
__device__ __forceinline__ void st_cs_u32(uint32_t *p, uint32_t v) {
  asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_cs_v4(uint32_t *p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

// ---- 1D bulk copies (TMA engine) into shared memory, completion tracked by an mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// bytes must be a multiple of 16 and both addresses 16 B aligned
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
  asm volatile(
      "{\n .reg .pred p;\n MBAR_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra MBAR_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Decoupled look-back over one count per tile, run by ALL 32 lanes of one warp: lane l inspects
// tile (t0 - l), so 32 predecessors are examined per round trip instead of one.  Publishes
// AGG(agg) then INC(excl + agg) for `tile` and returns the exclusive prefix (all lanes).
// Counts are < 2^32 (n < 2^32 per join), so 32-bit warp reductions suffice.
__device__ __forceinline__ uint64_t warp_lookback(uint64_t *status, uint64_t tile, uint32_t agg) {
  const uint32_t lane = threadIdx.x & 31;
  if (tile == 0) {
    if (lane == 0) st_relaxed_u64(status, kFlagInc | agg);
    return 0;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagAgg | agg);
  uint64_t excl = 0;
  int64_t t0 = (int64_t)tile - 1;
  while (true) {
    const int64_t t = t0 - (int64_t)lane;
    const uint64_t v = t >= 0 ? ld_relaxed_u64(status + t) : kFlagInc;  // virtual INC(0)
    const uint64_t flag = v & ~kValMask;
    const uint32_t inc = __ballot_sync(0xffffffffu, flag == kFlagInc);
    const uint32_t zero = __ballot_sync(0xffffffffu, flag == 0);
    const int first_inc = inc ? __ffs(inc) - 1 : 32;
    const uint32_t need = first_inc >= 31 ? 0xffffffffu : ((2u << first_inc) - 1u);
    if (zero & need) {
      __nanosleep(32);
      continue;
    }
    const uint32_t val = ((int)lane <= first_inc) ? (uint32_t)(v & kValMask) : 0u;
    excl += __reduce_add_sync(0xffffffffu, val);
    if (first_inc < 32) break;
    t0 -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | (excl + agg));
  return excl;
}

// ---------------------------------------------------------------- launchers (kernels/*.cu)
struct ScanPat {
  uint32_t const_mask;   // bit j: position j is a constant
  uint32_t id[3];
  uint32_t eq_mask;      // bit 0: s==p, bit 1: s==o, bit 2: p==o required
  uint32_t ncols;
  uint32_t src[3];       // output column c takes position src[c]
  // the constant tests as masked XORs: match <=> ((s^c[0])&m[0] | (p^c[1])&m[1] | (o^c[2])&m[2]) == 0
  uint32_t c[3], m[3];
};
struct ScanArgs {
  int k;
  ScanPat pat[MAPSQ_MAX_PATTERNS];
  uint32_t need_count;   // positions (bit j) the predicate pass must read
  uint32_t need_write;   // positions the gather pass must read
};
constexpr int kScanThreads = 256;
constexpr int kScanWordsPerWarp = 32;                     // 32 mask words of 32 triples
constexpr uint64_t kScanTile = 8ull * kScanWordsPerWarp * 32;  // 8192 triples per CTA tile

void launch_scan_count(const mapsq_triples &T, const ScanArgs &a, uint32_t *masks,
                       uint64_t mask_words, uint32_t *tile_counts, uint64_t ntiles,
                       cudaStream_t s);
struct ScanOut {
  uint32_t *col[MAPSQ_MAX_PATTERNS * 3];  // pattern j, column c -> col[j * 3 + c]
};
void launch_scan_write(const mapsq_triples &T, const ScanArgs &a, const uint32_t *masks,
                       uint64_t mask_words, const uint64_t *tile_off, uint64_t ntiles,
                       const ScanOut &out, uint32_t *bmin, uint32_t *bmax, cudaStream_t s);

// exclusive scan of u32 / u64 counts into u64 offsets (one single-pass look-back kernel);
// writes the total to *total_dev.  `tmp` needs scan_tmp_words(n) u64.
uint64_t scan_tmp_words(uint64_t n);
int launch_exclusive_scan_u32(const uint32_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s);
int launch_exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s);
int launch_exclusive_scan_u64_dev(const uint64_t *in, uint64_t *out, const uint64_t *n_dev,
                                  uint64_t cap, uint64_t *tmp, uint64_t *total_dev,
                                  cudaStream_t s);

struct PackArgs {
  uint32_t nkey;
  const uint32_t *key1[MAPSQ_MAX_COLS];
  const uint32_t *key2[MAPSQ_MAX_COLS];
  uint32_t lo[MAPSQ_MAX_COLS];
  uint32_t shift[MAPSQ_MAX_COLS];
  uint64_t n1, n2;
  uint32_t ib;
  uint32_t bit_lo;   // first sorted bit (ib for P64, 0 for KV)
  uint32_t passes;
  uint32_t last_mask;  // digit mask of the last pass ((1 << bits) - 1)
  uint32_t kv;       // 1: write keys[] = key', vals[] = rowid; 0: words = key' << ib | rowid
  uint32_t kb;       // packed key bits
  uint32_t hash;     // 1 (PATH_HASH): key' = key_hash over the raw values of all nkey columns
};
// Value-carrying words (filtered P64 joins with at most one non-key column per side and kb <= 31):
// the low 33 bits hold (label, value) instead of the row id, so ReduceDuplicate reads the non-key
// values from the sorted words themselves (no gathers).  The sort's stability keeps the rows'
// order.  The semi-join filter's column round writes them in its gathers (SjCarry::pv).
constexpr uint32_t kPvIb = 33;

// PATH_HASH key': a 64-bit mix of the shared columns' raw values, top kb bits.  Equal keys get
// equal key'; ReduceDuplicate verifies every pair's columns, so collisions cost time only.
__host__ __device__ __forceinline__ uint64_t key_hash_step(uint64_t h, uint32_t v) {
  h ^= v;
  h *= 0xbf58476d1ce4e5b9ull;
  return h ^ (h >> 29);
}
__host__ __device__ __forceinline__ uint64_t key_hash_final(uint64_t h, uint32_t kb) {
  h ^= h >> 32;
  h *= 0x94d049bb133111ebull;
  h ^= h >> 29;
  return h >> (64 - kb);
}
constexpr uint64_t kKeyHashSeed = 0x9E3779B97F4A7C15ull;
// Map (K2): pack words (or KV pairs) and build the digit histograms of every pass.
void launch_pack_hist(const PackArgs &a, uint64_t *words, uint32_t *vals, uint32_t *hist,
                      cudaStream_t s);
// Histograms of existing keys (for mapsq_sort_words on caller data).
void launch_key_hist(const uint64_t *keys, uint64_t n, uint32_t bit_lo, uint32_t passes,
                     uint32_t last_bits, uint32_t *hist, cudaStream_t s);
// One onesweep digit pass (K3).
// hist_pass: this pass's RAW digit counts (the kernel scans them); hist_next (may be NULL):
// zeroed counts the pass fills with the next digit (bits [next_shift, next_shift + next_bits)).
void launch_radix_pass(const uint64_t *kin, uint64_t *kout, const uint32_t *vin, uint32_t *vout,
                       uint64_t n, uint32_t shift, uint32_t bits, const uint32_t *hist_pass,
                       uint64_t *status, uint32_t *tile_counter, uint32_t *hist_next,
                       uint32_t next_shift, uint32_t next_bits, cudaStream_t s,
                       uint64_t n0 = ~0ull, uint64_t gap = 0);
// (n0, gap): two-segment input — key i >= n0 is read at kin[i + gap] (P64 words only: the
// semi-join filter leaves side A's and side B's survivors as two segments)

// ReduceDuplicate (K4): groups present on both sides, in key order.
struct GroupOut {
  uint32_t *start, *split, *end;
  uint64_t *cnt;
};
void launch_find_groups(const uint64_t *words, const uint64_t *keys, const uint32_t *vals,
                        uint64_t n, uint64_t n1, uint32_t ib, GroupOut g, uint64_t *status,
                        uint32_t *tile_counter, uint64_t *ngroups_dev, cudaStream_t s);

struct ExpandArgs {
  const uint64_t *words;   // P64 sorted words (or nullptr)
  const uint64_t *keys;    // KV sorted key' (or nullptr)
  const uint32_t *vals;    // KV sorted rowids
  uint64_t n1;
  uint32_t ib;
  const uint32_t *gstart, *gsplit, *gend;
  const uint64_t *goff;
  uint64_t ngroups;
  uint64_t m;
  uint32_t nkey;
  uint32_t key_lo[MAPSQ_MAX_COLS], key_shift[MAPSQ_MAX_COLS], key_mask[MAPSQ_MAX_COLS];
  uint32_t nrest1, nrest2;
  const uint32_t *rest1[MAPSQ_MAX_COLS];
  const uint32_t *rest2[MAPSQ_MAX_COLS];
  uint32_t *out[MAPSQ_MAX_COLS];  // nkey + nrest1 + nrest2 columns
  const uint64_t *tile_g0;        // scratch of expand_tiles(m) words: first group of each tile
};
// One-CTA Algorithm 1 (small.cu) for joins of at most kSmallMaxRows rows on the P64 path: writes
// |RS| to *m_out and, when |RS| <= cap, the rows into ea.out (capacity cap rows).
constexpr uint64_t kSmallMaxRows = 4096;
size_t small_join_smem(uint64_t n);
void launch_small_join(const PackArgs &pa, const ExpandArgs &ea, uint64_t cap,
                       unsigned long long *m_out, cudaStream_t s);
// launches the tile -> first-group kernel, then the expansion (2 launches)
void launch_expand(const ExpandArgs &a, cudaStream_t s);
uint64_t expand_tiles(uint64_t m);

// RESIDUAL / HASH paths (wide keys): groups are equal on key' (packed columns or a hash); the
// residual shared columns are compared exactly for every (LEFT, RIGHT) candidate pair.
struct ResidualArgs {
  const uint64_t *words;  // sorted P64 words over key'
  uint64_t n1;
  uint32_t ib;
  const uint32_t *gstart, *gsplit, *gend;
  uint32_t nres;
  const uint32_t *res1[MAPSQ_MAX_COLS];  // residual columns of tp1 / tp2, same variable order
  const uint32_t *res2[MAPSQ_MAX_COLS];
  // output column c comes from side src_side[c] (0 = tp1, 1 = tp2), column src[c]
  uint32_t nout;
  uint32_t src_side[MAPSQ_MAX_COLS];
  const uint32_t *src[MAPSQ_MAX_COLS];
  uint32_t *out[MAPSQ_MAX_COLS];
};
// Candidate-parallel verification over the C candidate pairs (coff = exclusive scan of nL * nR
// per group): write = true stores the matched pairs in (key', tp1 row, tp2 row) order at out[0 ..)
// (capacity C) and their number in *total; write = false only adds the number of matches to
// *total.  status: verify_tiles(C) zeroed words, tile_ctr zeroed, tile_g0 verify_tiles(C) + 1.
uint64_t verify_tiles(uint64_t candidates);
void launch_verify_emit(const ResidualArgs &a, const uint64_t *coff, uint64_t *tile_g0,
                        uint64_t ngroups, uint64_t C, bool write, uint64_t *status,
                        uint32_t *tile_ctr, unsigned long long *total, cudaStream_t s);
uint64_t find_groups_tiles(uint64_t n);

void launch_minmax(const uint32_t *const *cols, uint32_t ncols, uint64_t n, uint32_t *bounds,
                   cudaStream_t s);

// Semi-join filter (filter.cu, reading R18): key-presence bitmaps of 2^bbits bits; per side a
// probe that stages its survivors' words (key' << ib | rowid) compacted per 512-row slice, then a
// scan of the slice counts and a gather of the survivors into one contiguous array (A then B).
constexpr uint64_t kSemijoinMinRows = 1ull << 22;  // AUTO: joins of at least this many rows
constexpr uint32_t kSemijoinBits = 29;             // 2 x 64 MB bitmaps at most (L2-sized)
constexpr uint64_t kSjSlice = 512;                 // rows per warp slice
struct SjSeg {                                     // one side's packed words (ascending row ids)
  const uint64_t *w;
  uint64_t rows;
};
uint64_t sj_slices(uint64_t rows);  // ceil(rows / 512)
// rows the sampled probe reads of a side of `rows` rows (every 16th 512-row slice, at most ~4 M)
uint64_t sj_sample_rows(uint64_t rows);
// Stage layout: side A's slices first (slice s at stage[s * 512 ..], count cnt[s]), then side
// B's from slice sj_slices(n1) on; stage needs (sj_slices(n1) + sj_slices(n2)) * 512 words.
// Column round, phase 0: build bmS from the smaller side's key columns (side B if s_is_b) and
// probe a 1/16 sample of the larger side against it: sample[0] += survivors, sample[1] += rows.
// Single packed column: plain bitmap (bit_index); PATH_HASH: blocked Bloom (cblock of the
// key_hash chain).
void launch_sj_build_sample_cols(const PackArgs &a, bool s_is_b, void *bmS, uint32_t bbits,
                                 uint32_t hashed, unsigned long long *sample, cudaStream_t s,
                                 uint64_t l_rows = ~0ull,
                                 const std::function<void()> &before_sample = nullptr);
// (l_rows: sample only the larger side's first l_rows rows; before_sample runs between the two
// launches — the streamed path waits there for those rows)
// Columns carried through the column round: the gather also moves the survivors'
// values of these columns of the side (loaded by the staged words' row ids) into dense columns
// (survivor i of the side at out[c][i]) and replaces each word's row id by the survivor's
// position (+ n1 on side B): ReduceDuplicate then reads the dense survivor columns instead of
// gathering from the side's full columns.  n = 0: nothing carried.
struct SjCarry {
  uint32_t n;
  const uint32_t *src[MAPSQ_MAX_COLS];
  uint32_t *out[MAPSQ_MAX_COLS];
  // pv = 1 (value-carrying words): the gather instead rewrites each word's low 33 bits to
  // (label, src[0][row]) — label 1 on side B (id0 > 0), value 0 when n = 0; out[] is unused
  uint32_t pv;
};
// Probe one side's key columns (side B if side_b) against bm (bm_kind 0 plain / 1 cblock of the
// chain / 2 wblock of key' with seed) and stage its survivors; bm_set (plain, single-column keys
// only): survivors also set their bit there.
void launch_sj_probe_cols(const PackArgs &a, bool side_b, int bm_kind, const void *bm,
                          uint32_t bbits, uint32_t hashed, uint64_t seed, uint32_t *bm_set,
                          uint64_t *stage, uint32_t *cnt, cudaStream_t s, uint64_t row_lo = 0,
                          uint64_t row_hi = ~0ull);  // rows [row_lo, row_hi) (row_lo % 512 == 0)
// Word rounds: probe packed words (their slices start at slice0) against a wblock bitmap.
void launch_sj_probe_words(const SjSeg &in, uint64_t slice0, uint32_t ib, const void *bm,
                           uint32_t bbits, uint64_t seed, uint64_t *stage, uint32_t *cnt,
                           cudaStream_t s);
// Set the bits of w[0 .. *count) (count on the device, <= max_rows): kind 0 plain bit_index of
// key' = w >> ib, kind 2 wblock of key' with seed.
void launch_sj_set_words(const uint64_t *w, const uint64_t *count, uint64_t max_rows, int kind,
                         void *bm, uint32_t ib, uint32_t bbits, uint32_t hashed, uint64_t seed,
                         cudaStream_t s);
// out[off[s] ..] = the staged survivors of slice s (off = exclusive scan of cnt); hist += digit 0.
// With carried columns (cr.n > 0) their survivors' values move too (read at the staged word's row
// id - id0) and a word's row id becomes its position + id0.
void launch_sj_gather(const uint64_t *stage, const uint32_t *cnt, const uint64_t *off,
                      uint64_t nslices, uint64_t *out, uint32_t *hist, uint32_t bit_lo,
                      uint32_t dmask, const SjCarry &cr, uint32_t ib, uint64_t id0,
                      cudaStream_t s);
// Distributed pre-filter (dist.cu, f2): blocked Bloom bitmaps (cblock) of the key_hash chain of
// the RAW key values — the same on every rank — built / probed on one side's key columns.
// build: bm |= the side's keys.  probe: mask bit per row (row r -> bit r & 31 of mask[r >> 5]) =
// key present in bm; with bm_set the survivors also set their bits there.  sample: 1/16 of the
// side's rows probed, sample[0] += survivors, sample[1] += rows.
void launch_sj_chain_build(const PackArgs &a, bool side_b, void *bm, uint32_t bbits, cudaStream_t s);
void launch_sj_chain_probe(const PackArgs &a, bool side_b, const void *bm, uint32_t bbits,
                           void *bm_set, uint32_t *mask, cudaStream_t s);
void launch_sj_chain_sample(const PackArgs &a, bool side_b, const void *bm, uint32_t bbits,
                            unsigned long long *sample, cudaStream_t s);
// OR-reduce `words` 64-bit words of every rank's bitmap over the peer mappings: this rank reduces
// the slice [rank, rank + 1) * words / world of all peers and stores the result into all of them
// (reduce-scatter and all-gather fused in one NVLink kernel).  peers: device array of world
// pointers (this rank's own included).
void launch_peer_or(unsigned long long *const *peers, int world, int rank, uint64_t words,
                    cudaStream_t s);
void launch_sj_build_words(const SjSeg &S, uint32_t ib, uint64_t seed, uint32_t bbits, void *bm,
                           cudaStream_t s);
void launch_sj_sample_words(const SjSeg &L, uint32_t ib, uint64_t seed, uint32_t bbits,
                            const void *bm, unsigned long long *sample, cudaStream_t s);

// Compressed host store (hoststore.cu): frame-of-reference / delta blocks of 128 values.
uint64_t for_blocks(uint64_t n);
uint64_t for_block_words(uint32_t bits);
void launch_for_stats(const uint32_t *col, uint64_t n, uint32_t *base, uint32_t *bits,
                      uint32_t *dmin, cudaStream_t s);
// expand blocks [b0, b1) of a segment of n values (launch_for_unpack: all of them)
void launch_for_unpack_blocks(const uint32_t *seg, uint64_t n, uint64_t b0, uint64_t b1,
                              uint32_t *out, cudaStream_t s);
void launch_delay_us(uint32_t us, cudaStream_t s);
void launch_for_pack(const uint32_t *col, uint64_t n, const uint32_t *base, const uint32_t *bits,
                     const uint32_t *dmin, const uint32_t *woff, uint32_t *payload,
                     cudaStream_t s);
void launch_for_unpack(const uint32_t *seg, uint64_t n, uint32_t *out, cudaStream_t s);

// Predicate index (index.cu): permute s/p/o by the sorted words, record predicate run heads
// (unordered, atomic slots < cap); per-run bounds [slo | olo | shi | ohi].
void launch_index_gather(const uint64_t *words, uint64_t n, uint32_t ib, uint32_t p_lo,
                         const uint32_t *s, const uint32_t *o, uint32_t *s2, uint32_t *p2,
                         uint32_t *o2, uint32_t *head_p, uint64_t *head_start, uint32_t *nheads,
                         uint32_t cap, cudaStream_t st);
void launch_index_bounds(const uint32_t *s2, const uint32_t *o2, uint64_t n,
                         const uint64_t *starts, uint32_t nruns, uint32_t *bounds,
                         cudaStream_t st);

struct PartArgs {
  uint32_t nkey;
  const uint32_t *key[MAPSQ_MAX_COLS];
  uint32_t ncols;
  const uint32_t *in[MAPSQ_MAX_COLS];
  uint64_t n;
  uint32_t nparts;
  const uint32_t *mask;  // NULL, or bit r & 31 of mask[r >> 5]: row r is partitioned (else dropped)
  // skew (dist.cu): rows whose key (nkey <= kMaxHeavyCols values) equals one of the nheavy keys
  // heavy[h * kMaxHeavyCols ..] stay on this rank (dest = self) instead of their hash destination
  uint32_t nheavy, self;
  uint32_t heavy[8 * 4];
};
constexpr int kMaxHeavy = 8;
constexpr int kMaxHeavyCols = 4;
// keep[r] = in[r] && key(r) not heavy; bcast[r] = in[r] && key(r) heavy (a.heavy / a.nheavy;
// in = a.mask, NULL = all rows).  Both ceil(n / 32) words.
void launch_heavy_mask(const PartArgs &a, uint32_t *keep, uint32_t *bcast, cudaStream_t s);
mapsq_status partition_plan_impl(mapsq_ctx *ctx, const mapsq_table *in, const int32_t *key_vars,
                                 int nkey, int nparts, const uint32_t *row_mask,
                                 const uint32_t *heavy, int nheavy, int self,
                                 uint64_t *counts_host, mapsq_partition_state **state,
                                 void *stream);
mapsq_status compact_rows(mapsq_ctx *ctx, const mapsq_table *in, const uint32_t *mask,
                          mapsq_table *out, cudaStream_t s);
void launch_partition_hist(const PartArgs &a, uint32_t *tile_hist, uint64_t ntiles,
                           cudaStream_t s);
// dst_row[d]: first row of this rank's block in destination d's arena; dst_cols[d * ncols + c]:
// column c of d's arena (a device or an NVLink peer pointer)
void launch_partition_scatter(const PartArgs &a, const uint64_t *tile_off, uint64_t ntiles,
                              const uint64_t *dst_row, const uint64_t *dst_cols, cudaStream_t s);
constexpr int kPartThreads = 256;
constexpr int kPartItems = 16;
constexpr uint64_t kPartTile = kPartThreads * kPartItems;
constexpr int kMaxParts = 64;

}  // namespace mapsq
