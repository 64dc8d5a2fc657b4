/* mapsq.h — C ABI of libmapsq.so, the B200 (sm_100a) implementation of MapSQ's join path.
 *
 * Paper: "MapSQ: A MapReduce-based Framework for SPARQL Queries on GPU", arXiv 1702.03484
 * (PAPER.md).  The library answers a SPARQL basic graph pattern in the paper's two steps,
 * "partial matching and MapReduce-based join":
 *   1. mapsq_scan_pattern / mapsq_scan_patterns — partial matches of each triple pattern
 *      (gStore's black box replaced by a GPU scan over the triple table);
 *   2. mapsq_join — Algorithm 1: Map (label rows LEFT/RIGHT, :122-125),
 *      Sort (:126), ReduceDuplicate (emit every LEFT x RIGHT pair of each key, :127-133);
 *   3. mapsq_query — the left-deep chain of joins over the patterns (:137-138, :165) and the
 *      SELECT projection (:52).
 *
 * Conventions (all functions):
 *   - Every device buffer is a plain CUDA device pointer; every call is enqueued on `stream`
 *     (a cudaStream_t passed as void*, NULL = legacy default stream) and returns when the work
 *     is enqueued, except for the documented blocking reads of output sizes.
 *   - Inputs are borrowed and never modified.  Output tables are allocated by the library
 *     (through the context's allocator) and owned by the caller, who frees them with
 *     mapsq_table_release.  Scratch memory is freed, in stream order, before the call returns.
 *   - Each function returns a mapsq_status; no C++ exception crosses the ABI.  On error every
 *     output table is {nrows = 0, col[] = NULL, owner = NULL} with nothing allocated, and
 *     mapsq_last_error(ctx) describes the failure.  A CUDA error is sticky for the context.
 *   - Term IDs are uint32 (dictionary-encoded RDF terms); row counts and offsets are uint64.
 *   - Semantics are SPARQL solution mappings with bag semantics (readings R1-R16):
 *     a join on ALL shared variables, no deduplication, output schema
 *     shared (ascending variable id) ++ tp1 non-shared ++ tp2 non-shared.
 */
#ifndef MAPSQ_H
#define MAPSQ_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MAPSQ_OK = 0,
  MAPSQ_E_INVALID = 1,     /* NULL pointer, ncols == 0 or > MAPSQ_MAX_COLS, duplicate variable in a
                              schema, pattern without variables, n1 + n2 >= 2^32, bad argument */
  MAPSQ_E_NO_SHARED = 2,   /* join inputs share no variable; query pattern not connected to the
                              patterns before it */
  MAPSQ_E_NOMEM = 3,       /* the allocator returned NULL; nothing is partially written */
  MAPSQ_E_CUDA = 4,        /* CUDA error (text in mapsq_last_error); sticky for the context,
                              except a "CUDA IPC" failure of the fused exchange (see below) */
  MAPSQ_E_NCCL = 5,        /* NCCL missing or a control-plane collective failed (text in
                              mapsq_last_error); distributed entry points only */
  MAPSQ_E_UNSUPPORTED = 6  /* packed key wider than 64 bits after range compression (KV mode), too
                              many predicates for the index */
} mapsq_status;

#define MAPSQ_MAX_COLS 16
#define MAPSQ_MAX_PATTERNS 16
#define MAPSQ_TABLE_BOUNDS 1u /* flags bit: lo[]/hi[] hold valid inclusive column bounds */

/* A partial-match table, "Tp1 and Tp2 are the partial matches of each triple pattern"
 * (Alg. 1 Require).  Structure of arrays: col[c][r] is the ID bound to
 * variable var[c] in row r.  lo/hi are optional inclusive bounds of each column (valid iff
 * flags & MAPSQ_TABLE_BOUNDS); the library fills them on every table it produces and uses
 * them to range-compress join keys.  `owner` is the allocation behind col[] for tables the
 * library produced (NULL for caller-built tables, which the library never frees). */
typedef struct {
  uint64_t nrows;
  uint32_t ncols;
  uint32_t flags;
  int32_t var[MAPSQ_MAX_COLS];
  uint32_t lo[MAPSQ_MAX_COLS];
  uint32_t hi[MAPSQ_MAX_COLS];
  uint32_t *col[MAPSQ_MAX_COLS];
  void *owner;
} mapsq_table;

/* Dictionary-encoded triple table, structure of arrays of n (s, p, o) IDs (a set: no
 * duplicate triples; duplicates would be matched as many times as they occur). */
typedef struct {
  uint64_t n;
  const uint32_t *s, *p, *o;
} mapsq_triples;

/* Triple pattern P(s, p, o): var[j] >= 0 is a variable id at position j (0 = subject,
 * 1 = predicate, 2 = object); var[j] == -1 is the constant id[j].  A repeated variable
 * requires equal IDs; a constant absent from the data matches nothing (empty result, not an
 * error).  The partial-match schema is the pattern's distinct variables in (s, p, o) order. */
typedef struct {
  int32_t var[3];
  uint32_t id[3];
} mapsq_pattern;

/* Device-memory allocator (stream ordered).  NULL in mapsq_create selects cudaMallocAsync on
 * the device's default memory pool with an unbounded release threshold. */
typedef struct {
  void *(*alloc)(void *ctx, size_t bytes, void *stream);
  void (*free)(void *ctx, void *ptr, void *stream);
  void *ctx;
} mapsq_allocator;

typedef struct mapsq_ctx mapsq_ctx;

/* Host-side join spec.  Derived from the two schemas and column bounds:
 *   shared = vars(tp1) ∩ vars(tp2) ascending by id ("the key of them is their shared
 *   variable"; generalised to >= 1 shared variables, reading R5);
 *   key' = concatenation of (value - lo) of each PACKED shared column, first one most
 *   significant, each in key_bits[c] = bits(hi - lo) bits; kb = sum over packed columns;
 *   ib = bits(n1 + n2 - 1) index bits.
 *   path P64 when every shared column fits (kb + ib <= 64): one word key' << ib | rowid per row,
 *   rowid >= n1 meaning RIGHT.  When the full key does not fit, path RESIDUAL packs the
 *   widest shared columns that fit (packed_mask bit c set for shared[c]) and the remaining
 *   "residual" shared columns are compared exactly inside each packed-key group during
 *   ReduceDuplicate; path KV (u64 key' + u32 rowid pairs, every shared column packed) is the
 *   alternative selected with MAPSQ_OPT_WIDE_KEY = MAPSQ_WIDE_KEY_KV.
 *   path HASH (the default for keys wider than 32 bits or than 64 - ib bits):
 *   key' = the top kb = min(32, 64 - ib) bits of a 64-bit mix of the raw values of EVERY shared
 *   column (packed_mask = 0); equal keys share key', and ReduceDuplicate compares all shared
 *   columns of every (LEFT, RIGHT) pair of a key' group, so hash collisions never produce a
 *   wrong row.  Output rows are grouped by key' (not in key order). */
typedef struct {
  uint64_t n1, n2;
  uint32_t nshared;
  int32_t shared[MAPSQ_MAX_COLS];
  int32_t key_col1[MAPSQ_MAX_COLS], key_col2[MAPSQ_MAX_COLS]; /* column of shared[c] in tp1/tp2 */
  uint32_t key_lo[MAPSQ_MAX_COLS], key_hi[MAPSQ_MAX_COLS];    /* intersected bounds per shared var */
  uint32_t key_bits[MAPSQ_MAX_COLS], key_shift[MAPSQ_MAX_COLS];
  uint32_t nrest1, nrest2;
  int32_t rest_col1[MAPSQ_MAX_COLS], rest_col2[MAPSQ_MAX_COLS];
  uint32_t out_ncols;
  int32_t out_var[MAPSQ_MAX_COLS];
  uint32_t kb, ib;
  uint32_t path;    /* MAPSQ_PATH_* */
  uint32_t passes;  /* radix digit passes over the kb key bits */
  uint32_t disjoint;/* 1 when the key bounds do not overlap: the join is empty */
  uint32_t packed_mask; /* bit c: shared[c] is packed into key' (all bits set unless RESIDUAL) */
} mapsq_join_plan;
#define MAPSQ_PATH_P64 0u
#define MAPSQ_PATH_KV 1u
#define MAPSQ_PATH_RESIDUAL 2u
#define MAPSQ_PATH_HASH 3u
#define MAPSQ_RADIX_BITS 8u

/* Per-kernel timing (recorded with CUDA events on the launching stream while profiling is on)
 * and counters accumulated since the last mapsq_stats_reset. */
#define MAPSQ_MAX_KSTATS 32
typedef struct {
  char name[32];
  uint64_t launches;
  double total_ms;         /* sum of event-timed durations of those launches */
  uint64_t algo_bytes;     /* algorithmic bytes of those launches (DESIGN.md §5 byte model) */
} mapsq_kernel_stat;
typedef struct {
  uint64_t launches;       /* kernels launched by the library (profiling on or off) */
  uint64_t join_in_rows;   /* sum over joins of n1 + n2 */
  uint64_t join_out_rows;  /* sum over joins of |RS| */
  uint64_t scanned_triples;
  uint64_t joins, scans;
  uint64_t last_kb, last_ib, last_passes, last_path;
  uint64_t last_groups;    /* groups (keys on both sides) of the last join */
  uint64_t last_filtered;  /* rows the semi-join filter dropped in the last join */
  uint64_t filter_accesses;/* random bitmap accesses of the filter since the reset: builds and
                              probes (survivors setting the larger side's bits not counted) */
  uint64_t exchanges;      /* hash exchanges run by mapsq_join_dist / mapsq_query_dist */
  uint64_t exchange_rows;  /* rows this rank stored into OTHER ranks' arenas */
  uint64_t exchange_bytes; /* bytes of those rows (4 B per column) */
  uint64_t exchange_recv_rows;  /* rows OTHER ranks stored into this rank's arenas */
  uint64_t exchange_recv_bytes; /* bytes of those rows */
  uint64_t skew_keys;      /* heavy keys split / broadcast by the distributed joins */
  uint32_t nkernels;       /* per-kernel (per-phase) device times and algorithmic bytes: */
  mapsq_kernel_stat kernel[MAPSQ_MAX_KSTATS];
} mapsq_stats;

/* ---- context ---- */
mapsq_status mapsq_create(mapsq_ctx **out, int device, const mapsq_allocator *allocator);
void mapsq_destroy(mapsq_ctx *ctx);
const char *mapsq_last_error(const mapsq_ctx *ctx);
const char *mapsq_version(void);
/* Free an output table (stream ordered); a table with owner == NULL is only cleared. */
void mapsq_table_release(mapsq_ctx *ctx, mapsq_table *t, void *stream);

/* ---- partial matching (row a1) ----
 * Scan the triple table once per call and produce the partial matches of each of the k
 * patterns (k <= MAPSQ_MAX_PATTERNS): rows in triple order, schema as in mapsq_pattern.
 * One pass evaluates every pattern's predicate (reading only the constant positions) and
 * records a match bitmap; after ONE blocking read of the k row counts, a second pass gathers
 * the bound positions of matching triples only.  out[i] receives pattern i's table with
 * exact column bounds. */
mapsq_status mapsq_scan_patterns(mapsq_ctx *ctx, const mapsq_triples *triples,
                                 const mapsq_pattern *pats, int k, mapsq_table *out,
                                 void *stream);
mapsq_status mapsq_scan_pattern(mapsq_ctx *ctx, const mapsq_triples *triples,
                                const mapsq_pattern *pat, mapsq_table *out, void *stream);

/* ---- join (rows a2-a6): Algorithm 1, PAPER.md:116-135 ----
 * rs = tp1 ⋈ tp2 on all shared variables (bag semantics).  Map packs each row's key and its
 * LEFT (tp1) / RIGHT (tp2) label with the row id; an LSD radix sort orders the words by key
 * (stable, so LEFT rows precede RIGHT rows and row ids ascend within a key); ReduceDuplicate
 * finds each key's LEFT/RIGHT split, counts nL * nR, scans the counts and writes every pair.
 * Output rows are ordered (key', tp1 row, tp2 row) and are deterministic on one GPU.
 * Blocks once, to read |RS| for the output allocation.  Tables without bounds get them from a
 * min/max pass (one more blocking read). */
mapsq_status mapsq_join(mapsq_ctx *ctx, const mapsq_table *tp1, const mapsq_table *tp2,
                        mapsq_table *rs, void *stream);
/* Host-only: the join spec for two tables that carry bounds (no device work), for the default
 * wide-key mode (mapsq_plan_join) or a given MAPSQ_WIDE_KEY_* mode. */
mapsq_status mapsq_plan_join(const mapsq_table *tp1, const mapsq_table *tp2,
                             mapsq_join_plan *plan);
mapsq_status mapsq_plan_join_mode(const mapsq_table *tp1, const mapsq_table *tp2, int wide_mode,
                                  mapsq_join_plan *plan);

/* ---- query (row a7) ----
 * Scan all patterns in one fused pass (mapsq_scan_patterns), fold the joins left-deep in the
 * given order (pattern i must share a variable with patterns 0..i-1, else MAPSQ_E_NO_SHARED),
 * then project onto proj[0..nproj) (nproj == 0: all variables in first-appearance order).
 * Projection is zero-copy column selection with bag semantics (no DISTINCT). */
mapsq_status mapsq_query(mapsq_ctx *ctx, const mapsq_triples *triples,
                         const mapsq_pattern *pats, int npats, const int32_t *proj, int nproj,
                         mapsq_table *rs, void *stream);
/* End-to-end variant over HOST buffers: s/p/o are host pointers (pinned memory recommended)
 * holding n triples.  The triples are copied to the device, the query runs as mapsq_query, and
 * the result columns are copied back into a pinned result arena owned by the context.  On
 * return (synchronous) *host_rows is the row count, *out_ncols the width, out_var[c] the
 * variable of column c and host_cols[c] a pointer to that column's *host_rows IDs inside the
 * arena.  The arena (and every host_cols pointer) stays valid until the next
 * mapsq_query_host on this context or mapsq_destroy; the caller never frees it. */
mapsq_status mapsq_query_host(mapsq_ctx *ctx, uint64_t n, const uint32_t *s_host,
                              const uint32_t *p_host, const uint32_t *o_host,
                              const mapsq_pattern *pats, int npats, const int32_t *proj,
                              int nproj, uint64_t *host_rows, uint32_t *out_ncols,
                              int32_t *out_var, uint32_t **host_cols, void *stream);

/* ---- predicate-range index ----
 * The store-side access path of partial matching (PAPER.md:154, :164 leave matching to the
 * store; SPEC S:169-177 picks an index per pattern).  mapsq_index_build copies the triple table
 * into index-owned device memory, stably partitioned by predicate (within one predicate the
 * original triple order is kept), and records each predicate's row range and the exact bounds
 * of its subjects and objects.  Blocking (a few size reads); runs once per loaded dataset.
 * Memory: 12 B per triple for the permuted columns + per-predicate metadata; scratch during the
 * build 16 B per triple.  Fails with MAPSQ_E_UNSUPPORTED if there are more than 2^20 distinct
 * predicates or bits(p_hi - p_lo) + bits(n - 1) > 64.
 *
 * mapsq_scan_patterns_indexed: the same tables as mapsq_scan_patterns over the original
 * triples (same rows, and for a constant-predicate pattern the same row order):
 *   - P(?a, p, ?b) with a != b: a zero-copy view of the predicate's s/o range (owner == NULL,
 *     valid until mapsq_index_destroy; no kernel runs);
 *   - any other pattern with a constant predicate: the fused scan over that predicate's range;
 *   - a pattern with a variable predicate: the fused scan over the whole (permuted) table, rows
 *     in index order (predicate-major).
 * mapsq_query_indexed: mapsq_query with the scans above. */
typedef struct mapsq_index mapsq_index;
mapsq_status mapsq_index_build(mapsq_ctx *ctx, const mapsq_triples *triples, mapsq_index **out,
                               void *stream);
void mapsq_index_destroy(mapsq_ctx *ctx, mapsq_index *idx);
/* The permuted table (device pointers owned by the index) and its predicate count. */
mapsq_status mapsq_index_triples(const mapsq_index *idx, mapsq_triples *out, uint32_t *npreds);
/* Row range [*begin, *end) of predicate p in the permuted table (empty if p is absent). */
mapsq_status mapsq_index_range(const mapsq_index *idx, uint32_t p, uint64_t *begin,
                               uint64_t *end);
mapsq_status mapsq_scan_patterns_indexed(mapsq_ctx *ctx, const mapsq_index *idx,
                                         const mapsq_pattern *pats, int k, mapsq_table *out,
                                         void *stream);
mapsq_status mapsq_query_indexed(mapsq_ctx *ctx, const mapsq_index *idx,
                                 const mapsq_pattern *pats, int npats, const int32_t *proj,
                                 int nproj, mapsq_table *rs, void *stream);

/* ---- host-resident store (end-to-end path over host memory) ----
 * The paper's division of labour: the store answers partial matching on the host and the GPU
 * joins the partial matches.  mapsq_index_to_host mirrors an index into
 * pinned host memory (blocking, once per dataset): by default compressed (MAPSQ_OPT_HOST_COMPRESS:
 * frame-of-reference or delta blocks of 128 values per range and column, expanded on the GPU after the
 * copy — lossless), else 12 B per triple + metadata.
 * mapsq_query_host_indexed answers a query from that mirror: it copies to the device ONLY the
 * predicate ranges the query's patterns touch (s and o of every constant-predicate range; p too
 * when a pattern scans the range instead of viewing it; the whole table if a pattern has a
 * variable predicate), runs mapsq_query_indexed's path on them, and reads the result back into the
 * context's pinned result arena exactly as mapsq_query_host does (same output contract, same
 * result rows as mapsq_query_indexed over the device index).  *h2d_bytes (optional) receives the
 * bytes copied host -> device.  The copies run on a context-owned copy stream in the order the
 * query first uses the ranges, in chunks of 32 M rows (compressed chunks are expanded on a second
 * context-owned stream), and `stream` waits for each range only where it first reads it (later
 * ranges stream in while the first joins run); a join whose Tp2 is one range waits chunk by chunk
 * where it reads it in row order (the semi-join filter's probe of the larger side) and for the
 * whole range before anything else reads it.  Synchronous. */
typedef struct mapsq_host_index mapsq_host_index;
mapsq_status mapsq_index_to_host(mapsq_ctx *ctx, const mapsq_index *idx, mapsq_host_index **out,
                                 void *stream);
void mapsq_host_index_destroy(mapsq_host_index *h);
mapsq_status mapsq_query_host_indexed(mapsq_ctx *ctx, const mapsq_host_index *h,
                                      const mapsq_pattern *pats, int npats, const int32_t *proj,
                                      int nproj, uint64_t *host_rows, uint32_t *out_ncols,
                                      int32_t *out_var, uint32_t **host_cols, uint64_t *h2d_bytes,
                                      void *stream);

/* ---- phase entry points (for phase-level parity tests; the same kernels mapsq_join runs) ----
 * Map (K2, row a3): words[r] = key'(tp1 row r) << ib | r and words[n1 + r] = key'(tp2 row r)
 * << ib | (n1 + r) for a P64 plan (a RESIDUAL plan packs only its packed_mask columns; a KV
 * plan is rejected).  `words` is a caller-owned device array of n1 + n2. */
mapsq_status mapsq_map_words(mapsq_ctx *ctx, const mapsq_table *tp1, const mapsq_table *tp2,
                             const mapsq_join_plan *plan, uint64_t *words, void *stream);
/* Sort (K3, row a4): stable LSD radix sort of n words by bits [bit_lo, bit_hi), in place
 * (device array; the library allocates the ping-pong buffer). */
mapsq_status mapsq_sort_words(mapsq_ctx *ctx, uint64_t *words, uint64_t n, uint32_t bit_lo,
                              uint32_t bit_hi, void *stream);
/* Stable LSD radix sort of (key, value) pairs by key bits [bit_lo, bit_hi), in place. */
mapsq_status mapsq_sort_pairs(mapsq_ctx *ctx, uint64_t *keys, uint32_t *vals, uint64_t n,
                              uint32_t bit_lo, uint32_t bit_hi, void *stream);
/* ReduceDuplicate part 1 (K4+K5, row a5) on sorted P64 words: for every key present on both
 * sides, in key order, group_start/group_split/group_end (device arrays of capacity
 * min(n1, n2)) receive the run [start, end) and its first RIGHT position, and group_off the
 * exclusive prefix of nL * nR.  *ngroups and *total (host) receive the group count and |RS|
 * (blocking). */
mapsq_status mapsq_reduce_groups(mapsq_ctx *ctx, const uint64_t *words, uint64_t n1, uint64_t n2,
                                 uint32_t ib, uint32_t *group_start, uint32_t *group_split,
                                 uint32_t *group_end, uint64_t *group_off, uint64_t *ngroups,
                                 uint64_t *total, void *stream);

/* ---- multi-GPU exchange (SURVEY §8 row e) ----
 * Hash partition on the join key, fused with the all-to-all: every rank sends each row to rank
 * dest = (fmix32(h) * nparts) >> 32 (multiply-shift range reduction), h the FNV-1a-style fold (h = (h ^ v) * 16777619 from 2166136261)
 * of the row's values of key_vars[0..nkey) in that order.
 *
 * mapsq_partition_plan: per-tile destination histogram + scan; counts_host[d] receives the number
 * of rows for destination d (blocking read).  *state keeps the plan for the scatter (free it with
 * mapsq_partition_state_free; `in` must stay valid until then).
 * mapsq_partition_scatter: ONE kernel writes every row straight into its destination: column c of
 * destination d starts at dest_cols[d * ncols + c] — a local device pointer or a peer rank's
 * arena opened with mapsq_ipc_open (NVLink stores) — and this rank's rows for d occupy rows
 * [dest_row[d], dest_row[d] + counts[d]) of it, stable within the destination.  Returns when
 * the kernel has completed (the caller then synchronises the ranks before reading). */
typedef struct mapsq_partition_state mapsq_partition_state;
mapsq_status mapsq_partition_plan(mapsq_ctx *ctx, const mapsq_table *in, const int32_t *key_vars,
                                  int nkey, int nparts, uint64_t *counts_host,
                                  mapsq_partition_state **state, void *stream);
/* The same with a row mask (device, ceil(nrows / 32) words): row r takes part iff bit (r & 31) of
 * row_mask[r >> 5] is set; dropped rows are neither counted nor scattered (the distributed
 * semi-join pre-filter exchanges only rows whose key may occur on the other side).  NULL = all. */
mapsq_status mapsq_partition_plan_masked(mapsq_ctx *ctx, const mapsq_table *in,
                                         const int32_t *key_vars, int nkey, int nparts,
                                         const uint32_t *row_mask, uint64_t *counts_host,
                                         mapsq_partition_state **state, void *stream);
mapsq_status mapsq_partition_scatter(mapsq_ctx *ctx, mapsq_partition_state *state,
                                     const uint64_t *dest_row, uint32_t *const *dest_cols,
                                     void *stream);
void mapsq_partition_state_free(mapsq_ctx *ctx, mapsq_partition_state *state);
/* Local convenience: `out` receives a table with the same schema whose rows are grouped by
 * destination (destination-major, stable within a destination); counts_host[d] as above. */
mapsq_status mapsq_partition(mapsq_ctx *ctx, const mapsq_table *in, const int32_t *key_vars,
                             int nkey, int nparts, mapsq_table *out, uint64_t *counts_host,
                             void *stream);
/* CUDA IPC of a device allocation (64-byte handle) so peer ranks can store into it.  Export only
 * pointers returned by mapsq_ipc_alloc (a whole cudaMalloc allocation: the handle maps its base). */
mapsq_status mapsq_ipc_alloc(mapsq_ctx *ctx, size_t bytes, void **dev_ptr);
mapsq_status mapsq_ipc_free(mapsq_ctx *ctx, void *dev_ptr);
mapsq_status mapsq_ipc_export(mapsq_ctx *ctx, void *dev_ptr, void *handle64);
mapsq_status mapsq_ipc_open(mapsq_ctx *ctx, const void *handle64, void **dev_ptr);
mapsq_status mapsq_ipc_close(mapsq_ctx *ctx, void *dev_ptr);
/* Host-only layout of one exchange (no device work): from the world x world count matrix
 * (count_matrix[s * world + d] = rows rank s sends to rank d), dest_row[d] = this rank's first row
 * in rank d's receive block (sources s < rank come first, so a received table is grouped by
 * source rank), recv[d] = rows rank d receives, and need_bytes[d] = bytes of rank d's receive
 * block: ncols columns of stride_rows(recv[d]) = recv[d] rounded up to a multiple of 4 rows
 * (16 B aligned columns). */
mapsq_status mapsq_exchange_layout(int world, int rank, int ncols, const uint64_t *count_matrix,
                                   uint64_t *dest_row, uint64_t *recv, uint64_t *need_bytes);

/* ---- distributed join and query (SURVEY §8 rows b and e) ----
 * One process per GPU, one context per process.  The equi-join decomposes over disjoint key
 * sets (PAPER.md:126-133 join each key's group independently), so each join is one hash
 * exchange of both inputs on ALL shared variables (mapsq_partition_plan's destination function)
 * followed by the local Algorithm-1 join; RS stays sharded (the union over ranks is RS).
 * The exchange is the fused kernel above: every rank owns two receive arenas (one per join side,
 * grow-only cudaMalloc allocations exported with CUDA IPC and opened by every peer), the ranks
 * all-gather the count matrix with NCCL, and mapsq_partition_scatter stores each row straight
 * into its destination's arena over NVLink / NVSwitch.  NCCL (libnccl.so.2, loaded at
 * mapsq_dist_init) carries only the count matrix, the arena handles, the column bounds (min/max
 * all-reduce, so the local join range-compresses keys without a min/max pass) and the two
 * barriers around each scatter.  Every call is collective: all ranks call it in the same order.
 * Errors: argument errors are detected before the first collective on every rank alike (same
 * tables' schemas).  Growing the receive arenas is collective in outcome: if any rank cannot
 * allocate, export or open an arena, EVERY rank returns MAPSQ_E_CUDA with "CUDA IPC" in the
 * message after the same collectives (the context stays usable; the fused exchange is disabled
 * for the communicator and the caller may fall back to another exchange).  A rank that fails
 * later (allocation, CUDA, NCCL) returns its status while its peers may stay blocked in the next
 * collective — the caller aborts the job (queries are stateless and are simply re-run).
 *
 * mapsq_dist_unique_id: a fresh 128-byte NCCL unique id (one rank creates it; the caller
 *   broadcasts it, e.g. with torch.distributed).
 * mapsq_dist_init: join the communicator (blocking, collective).  Returns MAPSQ_E_NCCL if NCCL
 *   cannot be loaded or the init fails; MAPSQ_E_INVALID if already initialised.  The state is
 *   freed by mapsq_destroy.
 * mapsq_join_dist: rs_shard = this rank's part of tp1 ⋈ tp2 (tp1_shard, tp2_shard are this
 *   rank's rows of each input, any distribution).  Blocking.  Output owned by the caller.
 * mapsq_query_dist / mapsq_query_dist_indexed: every rank scans its shard of the triple table
 *   (rows of the triple table distributed in any way: a pattern matches each triple where it
 *   lives, no exchange), then folds the joins left-deep with one exchange per join; an input
 *   already partitioned on the join's key (the previous join's result, when the key is unchanged)
 *   is not exchanged again.  Projection as mapsq_query. */
/* mapsq_query_dist_host_indexed: the end-to-end form over this rank's host-resident store
 *   (mapsq_query_host_indexed's contract: only the touched predicate ranges go host -> device;
 *   this rank's result shard lands in the context's pinned result arena). */
#define MAPSQ_DIST_ID_BYTES 128
mapsq_status mapsq_dist_unique_id(void *id128);
mapsq_status mapsq_dist_init(mapsq_ctx *ctx, const void *id128, int rank, int world);
/* The same distributed state with the control plane (count matrix all-gather, bounds max-reduce,
 * arena-handle all-gather, barriers) carried by caller-supplied blocking collectives over HOST
 * buffers instead of NCCL — e.g. torch.distributed's gloo backend.  The data plane is unchanged
 * (the fused scatter kernel stores rows into the peers' CUDA-IPC arenas), and no kernel ever
 * waits on another rank: every cross-rank dependency is a host-side collective after a stream
 * synchronisation.  This is also how several rank processes can share one GPU (each rank maps
 * the others' arenas through CUDA IPC), which NCCL refuses.  Each callback returns 0 on success:
 *   allgather(user, send, recv, bytes): recv[r * bytes ..] = rank r's `send` (bytes each);
 *   allreduce_max_u32(user, buf, n): buf[i] = max over ranks of buf[i], in place;
 *   barrier(user). */
typedef struct {
  int (*allgather)(void *user, const void *send, void *recv, size_t bytes);
  int (*allreduce_max_u32)(void *user, uint32_t *buf, size_t n);
  int (*barrier)(void *user);
  void *user;
} mapsq_collectives;
mapsq_status mapsq_dist_init_host(mapsq_ctx *ctx, const mapsq_collectives *coll, int rank,
                                  int world);
mapsq_status mapsq_join_dist(mapsq_ctx *ctx, const mapsq_table *tp1_shard,
                             const mapsq_table *tp2_shard, mapsq_table *rs_shard, void *stream);
mapsq_status mapsq_query_dist(mapsq_ctx *ctx, const mapsq_triples *shard,
                              const mapsq_pattern *pats, int npats, const int32_t *proj, int nproj,
                              mapsq_table *rs_shard, void *stream);
mapsq_status mapsq_query_dist_indexed(mapsq_ctx *ctx, const mapsq_index *shard,
                                      const mapsq_pattern *pats, int npats, const int32_t *proj,
                                      int nproj, mapsq_table *rs_shard, void *stream);
mapsq_status mapsq_query_dist_host_indexed(mapsq_ctx *ctx, const mapsq_host_index *shard,
                                           const mapsq_pattern *pats, int npats,
                                           const int32_t *proj, int nproj, uint64_t *host_rows,
                                           uint32_t *out_ncols, int32_t *out_var,
                                           uint32_t **host_cols, uint64_t *h2d_bytes,
                                           void *stream);

/* Compute exact inclusive bounds lo[]/hi[] of every column of a (caller-built) table and set
 * MAPSQ_TABLE_BOUNDS (one min/max pass, blocking).  An empty table gets lo = hi = 0. */
mapsq_status mapsq_table_bounds(mapsq_ctx *ctx, mapsq_table *t, void *stream);

/* ---- options ---- */
#define MAPSQ_OPT_WIDE_KEY 1      /* how a join whose full key does not fit 64 - ib bits runs: */
#define MAPSQ_WIDE_KEY_RESIDUAL 0 /*   packed widest columns + residual check */
#define MAPSQ_WIDE_KEY_KV 1       /*   (u64 key, u32 rowid) pair sort over every key bit */
#define MAPSQ_WIDE_KEY_HASH 2     /*   hashed composite key + exact pair check (default) */
/* Semi-join filter in front of the Map (SURVEY §8 row f2's reducer): rows whose packed key is
 * absent from the other side produce nothing in ReduceDuplicate and
 * are dropped before the sort; RS and its row order are unchanged.  Costs extra reads of the key
 * columns, two key-presence bitmaps (<= 64 MB each) and a few more blocking reads per join. */
#define MAPSQ_OPT_SEMIJOIN 2
#define MAPSQ_SEMIJOIN_OFF 0
#define MAPSQ_SEMIJOIN_AUTO 1     /*   default: joins with n1 + n2 >= 2^22 rows, unless a 1/16
                                       sample says >= 90% of the rows would survive */
#define MAPSQ_SEMIJOIN_ON 2       /*   every P64 / RESIDUAL / HASH join */
/* Joins of at most 4096 input rows on the P64 path run Algorithm 1 in ONE kernel launch (one CTA:
 * Map, sort and ReduceDuplicate in shared memory; same rows in the same order) with one blocking
 * read of |RS|; 0 disables it (every join takes the multi-kernel path). */
#define MAPSQ_OPT_SMALL_JOIN 3    /*   1 (default) / 0 */
/* Distributed joins: heavy keys (estimated from a sample to exceed max(1024, N / (4 world)) rows)
 * keep one side's rows on their rank and broadcast the other side's rows to every rank. */
#define MAPSQ_OPT_SKEW 4          /*   1 (default) / 0 */
/* mapsq_index_to_host keeps every column of every predicate range as blocks of 128 values, each in
 * the narrower of two codings (a block's minimum + offsets, or its first value + deltas, in the
 * fewest bits that hold them); the host-indexed
 * query copies the touched blocks and expands them on the GPU (lossless).  0: plain 32-bit
 * columns (12 B per triple).  Read when the mirror is made. */
#define MAPSQ_OPT_HOST_COMPRESS 5 /*   1 (default) / 0 */
mapsq_status mapsq_set_option(mapsq_ctx *ctx, int option, int64_t value);

/* ---- statistics ---- */
mapsq_status mapsq_set_profiling(mapsq_ctx *ctx, int on);
mapsq_status mapsq_stats_reset(mapsq_ctx *ctx);
/* Blocks until the recorded events complete, then fills *st. */
mapsq_status mapsq_get_stats(mapsq_ctx *ctx, mapsq_stats *st);

#ifdef __cplusplus
}
#endif
#endif /* MAPSQ_H */
