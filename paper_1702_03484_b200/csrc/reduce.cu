// reduce.cu — ReduceDuplicate (Alg. 1 l.6-11), SURVEY §8 rows a5-a6.
//
// K4 find_groups: in the sorted words, a key present on BOTH sides has exactly one position
// where a LEFT word is followed by a RIGHT word of the same key (the "split"; LEFT precedes
// RIGHT inside a key because the label is the high part of the rowid field).  Every such split
// is one output group — the flag "contributes to reduce unnecessary computation": keys
// with one label only produce nothing and are never visited again.  The splits are compacted in
// key order with a single-pass decoupled look-back; the thread owning a split gallops outwards
// to the run's ends and stores (start, split, end) and nL * nR.
// RESIDUAL / HASH verify-emit: candidate-parallel check of the residual shared columns of every
// (LEFT, RIGHT) pair of a key' group, writing the matches in order (see below).
// K6 expand: "GPU's SIMD architectures contribute to accelerate cartesian product in parallel"
// (P:149).  Output-row parallel, so skewed keys are load balanced: every thread owns 4
// consecutive output rows, finds its group by a binary search bracketed per CTA, and writes
// (key columns decoded from the word, Tp1 non-shared, Tp2 non-shared) in (key, left rowid,
// right rowid) order with 16 B streaming stores.
#include <cstdlib>

#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kGThreads = 256;
#ifndef MAPSQ_G_ITEMS
#define MAPSQ_G_ITEMS 32
#endif
constexpr int kGItems = MAPSQ_G_ITEMS;  // words per lane per warp slice
constexpr uint64_t kGTile = kGThreads * kGItems;
constexpr int kGWarps = kGThreads / 32;
constexpr int kGSlice = 32 * kGItems;       // elements per warp slice
constexpr int kGMaxRec = kGSlice / 2;       // at most one split per two elements

struct WordView {
  const uint64_t *words, *keys;
  const uint32_t *vals;
  uint64_t n1;
  uint32_t ib;
  uint64_t idx_mask;
  __device__ __forceinline__ uint64_t key(uint64_t i) const {
    return words ? (words[i] >> ib) : keys[i];
  }
};

// first index of the run of key k that contains position `from` (key(from) == k), by galloping
__device__ uint64_t run_start(const WordView &W, uint64_t from, uint64_t k) {
  int64_t lo = (int64_t)from, step = 1;
  while (true) {
    const int64_t c = lo - step;
    if (c < 0 || W.key((uint64_t)c) != k) break;
    lo = c;
    step <<= 1;
  }
  int64_t L = (lo - step > -1) ? lo - step : -1, R = lo;  // key(L) != k (or -1), key(R) == k
  while (R - L > 1) {
    const int64_t m = (L + R) >> 1;
    if (W.key((uint64_t)m) == k) R = m; else L = m;
  }
  return (uint64_t)R;
}
// one past the last index of the run of key k that contains position `from`
__device__ uint64_t run_end(const WordView &W, uint64_t from, uint64_t k, uint64_t n) {
  int64_t hi = (int64_t)from, step = 1;
  while (true) {
    const int64_t c = hi + step;
    if (c >= (int64_t)n || W.key((uint64_t)c) != k) break;
    hi = c;
    step <<= 1;
  }
  int64_t L = hi, R = (hi + step < (int64_t)n) ? hi + step : (int64_t)n;
  while (R - L > 1) {
    const int64_t m = (L + R) >> 1;
    if (W.key((uint64_t)m) == k) L = m; else R = m;
  }
  return (uint64_t)R;
}

// K4.  Warp w sweeps its contiguous slice of the tile item by item (32 consecutive words per
// item).  Ballots give the run heads (key differs from the previous word) and the splits
// (LEFT word followed by a RIGHT word of the same key); a split's run starts at the last head
// at or before it and ends at the next head after it, both tracked across items in registers
// ("pending" end).  Only a run crossing the slice boundary needs a gallop (at most one start and
// one end per slice).  Records go to shared memory, the tile's split count is resolved with a
// warp-parallel decoupled look-back, and records are stored in key order.  Positions are 32-bit
// (n < 2^32); for P64 words "same key" is ((w ^ w_prev) >> ib) == 0 and the label is the low
// word's rowid compared with n1.
template <bool KV>
__global__ void __launch_bounds__(kGThreads)
find_groups_kernel(const WordView W, uint64_t n64, GroupOut g, uint64_t *__restrict__ status,
                   uint32_t *__restrict__ tile_counter, uint64_t *__restrict__ ngroups_dev) {
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_nrec[kGWarps];
  __shared__ uint64_t s_base;
  // per-warp record buffers (dynamic shared memory: kGWarps x kGMaxRec each)
  extern __shared__ __align__(16) unsigned char g_smem[];
  auto s_start = reinterpret_cast<uint32_t (*)[kGMaxRec]>(g_smem);
  auto s_end = reinterpret_cast<uint32_t (*)[kGMaxRec]>(g_smem + sizeof(uint32_t) * kGWarps * kGMaxRec);
  auto s_split = reinterpret_cast<uint16_t (*)[kGMaxRec]>(g_smem + 2 * sizeof(uint32_t) * kGWarps * kGMaxRec);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
  __syncthreads();
  const uint32_t n = (uint32_t)n64;
  const uint64_t tile = s_tile;
  const uint64_t sbeg64 = tile * kGTile + (uint64_t)warp * kGSlice;
  const uint32_t sbeg = sbeg64 < n64 ? (uint32_t)sbeg64 : n;  // slice [sbeg, send)
  const uint32_t send = (n - sbeg) > (uint32_t)kGSlice ? sbeg + kGSlice : n;
  const uint32_t le = lt_or_eq_mask(lane), lt = lanemask_lt();
  const uint32_t imask = (uint32_t)W.idx_mask, n1 = (uint32_t)W.n1, ib = W.ib;
  uint32_t nrec = 0;
  int32_t pending = -1;             // record whose run has not ended yet
  uint32_t last_head = 0xffffffffu; // last head seen in this slice (none yet)
  int32_t first_unknown = -1;       // first record whose run started before the slice
  // previous element: (key, label) as one comparable pair
  uint64_t carry_w = 0, carry_k = ~0ull;
  uint32_t carry_v = 0;
  if (sbeg < send && sbeg > 0) {
    if (KV) { carry_k = W.keys[sbeg - 1]; carry_v = W.vals[sbeg - 1]; }
    else carry_w = W.words[sbeg - 1];
  }
  constexpr int kB = 8;
#pragma unroll 1
  for (uint32_t it0 = 0; it0 < (uint32_t)kGItems; it0 += kB) {
    uint64_t ww[kB];
    uint32_t vv[KV ? kB : 1];
#pragma unroll
    for (int u = 0; u < kB; u++) {
      const uint32_t i = sbeg + (it0 + u) * 32 + lane;
      if (KV) {
        ww[u] = i < send ? __ldcs(W.keys + i) : 0ull;
        vv[KV ? u : 0] = i < send ? __ldcs(W.vals + i) : 0u;
      } else {
        ww[u] = i < send ? __ldcs(W.words + i) : 0ull;
      }
    }
#pragma unroll
    for (int u = 0; u < kB; u++) {
      const uint32_t ibase = sbeg + (it0 + u) * 32;
      if (ibase >= send) break;  // warp-uniform
      const uint32_t i = ibase + lane;
      const bool in = i < send;
      const uint64_t w = ww[u];
      uint64_t wp = __shfl_up_sync(0xffffffffu, w, 1);
      bool same, r, rp;
      if (KV) {
        const uint32_t v = vv[KV ? u : 0];
        uint32_t vp = __shfl_up_sync(0xffffffffu, v, 1);
        if (lane == 0) { wp = carry_k; vp = carry_v; }
        same = w == wp;
        r = v >= n1;
        rp = vp >= n1;
      } else {
        if (lane == 0) wp = carry_w;
        same = ((w ^ wp) >> ib) == 0;
        // (value-carrying words, ib = kPvIb: the label is bit 32)
        r = ib > 32 ? (uint32_t)(w >> 32) & 1u : ((uint32_t)w & imask) >= n1;
        rp = ib > 32 ? (uint32_t)(wp >> 32) & 1u : ((uint32_t)wp & imask) >= n1;
      }
      const bool head = in && (i == 0 || !same || (lane == 0 && sbeg == 0 && i == 0));
      const bool split = in && i > 0 && r && !rp && same;
      const uint32_t hm = __ballot_sync(0xffffffffu, head);
      const uint32_t sm = __ballot_sync(0xffffffffu, split);
      if (pending >= 0 && hm) {  // the pending run ends at this item's first head
        if (lane == 0) s_end[warp][pending] = ibase + __ffs(hm) - 1;
        pending = -1;
      }
      if (sm) {  // warp-uniform: rare relative to elements
        if (split) {
          const uint32_t idx = nrec + __popc(sm & lt);
          const uint32_t hb = hm & le;  // heads at or before this lane
          const uint32_t ha = hm & ~le;  // heads after this lane
          s_start[warp][idx] = hb ? ibase + 31 - __clz(hb) : last_head;
          s_split[warp][idx] = (uint16_t)(i - sbeg);
          if (ha) s_end[warp][idx] = ibase + __ffs(ha) - 1;  // else: pending
        }
        const int hi_lane = 31 - __clz(sm);
        if (!(hm & ~lt_or_eq_mask(hi_lane))) pending = (int32_t)(nrec + __popc(sm) - 1);
        if (first_unknown < 0 && last_head == 0xffffffffu && !(hm & lt_or_eq_mask(__ffs(sm) - 1)))
          first_unknown = (int32_t)nrec;
        nrec += __popc(sm);
      }
      if (hm) last_head = ibase + 31 - __clz(hm);
      if (KV) {
        carry_k = __shfl_sync(0xffffffffu, w, 31);
        carry_v = __shfl_sync(0xffffffffu, vv[KV ? u : 0], 31);
      } else {
        carry_w = __shfl_sync(0xffffffffu, w, 31);
      }
    }
  }
  __syncwarp();
  // runs crossing the slice boundary: gallop (at most one start and one end per slice)
  if (lane == 0) {
    if (first_unknown >= 0) {
      const uint64_t sp = sbeg + s_split[warp][first_unknown];
      s_start[warp][first_unknown] = (uint32_t)run_start(W, sp, W.key(sp));
    }
    if (pending >= 0) {
      const uint64_t sp = sbeg + s_split[warp][pending];
      s_end[warp][pending] = (uint32_t)run_end(W, sp, W.key(sp), n64);
    }
    s_nrec[warp] = nrec;
  }
  __syncthreads();
  if (warp == 0) {
    const uint32_t c = lane < kGWarps ? s_nrec[lane] : 0u;
    uint32_t x = c;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, x, 31);
    if (lane < kGWarps) s_nrec[lane] = x - c;  // exclusive prefix over warps
    const uint64_t excl = warp_lookback(status, tile, total);
    if (lane == 0) {
      s_base = excl;
      if (tile == gridDim.x - 1) *ngroups_dev = excl + total;
    }
  }
  __syncthreads();
  const uint64_t out0 = s_base + s_nrec[warp];
  for (uint32_t q = lane; q < nrec; q += 32) {
    const uint64_t st = s_start[warp][q], sp = sbeg + s_split[warp][q], en = s_end[warp][q];
    g.start[out0 + q] = (uint32_t)st;
    g.split[out0 + q] = (uint32_t)sp;
    g.end[out0 + q] = (uint32_t)en;
    g.cnt[out0 + q] = (sp - st) * (en - sp);
  }
}

// Random 4 B column gathers (verification): MAPSQ_GATHER_HINT 1 = ld.global.nc.L2::64B (the
// L2 fetches 64 B on a miss instead of 128: C5 J2's verification 2.81 -> 1.52 GB of DRAM reads,
// 0.57 -> 0.54 ms — it is bound by the gathers' latency more than by their bytes), 2 = also no
// L1 allocation, 0 = plain read-only loads (ablation knob)
#ifndef MAPSQ_GATHER_HINT
#define MAPSQ_GATHER_HINT 1
#endif
__device__ __forceinline__ uint32_t ld_rnd(const uint32_t *p) {
#if MAPSQ_GATHER_HINT == 1
  uint32_t v;
  asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#elif MAPSQ_GATHER_HINT == 2
  uint32_t v;
  asm("ld.global.nc.L1::no_allocate.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// ------------------------------------------------------------------------------ expand (K6)
constexpr int kEThreads = 256;
constexpr int kERowsPerThread = 8;           // rows per thread = chunks x rows per chunk
constexpr uint64_t kETile = (uint64_t)kEThreads * kERowsPerThread;
constexpr int kEGroups = 1024;               // groups staged in shared memory per tile

// K5b: tile t of the expansion (rows [t * tile_rows, ...)) starts inside group tile_g0[t], the
// last group whose offset is <= t * tile_rows: one thread per tile, a binary search over the
// offsets (a hot group spanning many tiles costs nothing extra).
__global__ void __launch_bounds__(256)
tile_groups_kernel(const uint64_t *__restrict__ goff, uint64_t ngroups, uint64_t ntiles,
                   uint64_t *__restrict__ tile_g0, uint64_t tile_rows) {
  for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < ntiles;
       t += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t r = t * tile_rows;
    uint64_t lo = 0, hi = ngroups - 1;  // goff[0] == 0 <= r
    while (lo < hi) {
      const uint64_t mid = (lo + hi + 1) >> 1;
      if (__ldg(goff + mid) <= r) lo = mid; else hi = mid - 1;
    }
    tile_g0[t] = lo;
  }
}

__device__ __forceinline__ uint64_t group_of(const uint64_t *off, uint64_t lo, uint64_t hi,
                                             uint64_t r) {
  // largest g in [lo, hi] with off[g] <= r  (off strictly increasing, off[lo] <= r)
  while (lo < hi) {
    const uint64_t m = (lo + hi + 1) >> 1;
    if (off[m] <= r) lo = m; else hi = m - 1;
  }
  return lo;
}

// K6.  A CTA owns kETile consecutive output rows; two threads bracket its group range [g0, g1]
// with binary searches and, when it has at most kEGroups groups (always, except for tiles full of
// 1-row groups), the groups' (offset, start, split, end) are staged in shared memory.  Each
// thread owns kEChunks chunks of kERows consecutive rows (chunk c of thread t starts at row
// t0 + (c * kEThreads + t) * kERows, so a warp's chunks are contiguous): it locates its group in
// shared memory, then computes the 8 (LEFT, RIGHT) positions, issues all word loads, then all
// column gathers, then 16 B streaming stores — so the latencies of one thread's rows overlap.
// FULL: every row of the tile exists (all tiles but the last; launched separately), so the
// per-row bounds checks and partial-chunk paths compile away.
template <int kERows, int kEChunks, bool FULL>
__global__ void __launch_bounds__(kEThreads, 5)
expand_kernel(const ExpandArgs a, uint64_t tile0, uint64_t ntiles) {
  static_assert(kERows * kEChunks == kERowsPerThread && kERows % 4 == 0, "tile shape");
  __shared__ const uint32_t *s_src[MAPSQ_MAX_COLS];
  __shared__ uint32_t *s_dst[MAPSQ_MAX_COLS];
  __shared__ uint64_t s_g[2];
  __shared__ uint64_t s_off[kEGroups + 1];
  __shared__ uint32_t s_start[kEGroups], s_split[kEGroups], s_end[kEGroups];
  const int tid = threadIdx.x;
  const uint32_t nout = a.nkey + a.nrest1 + a.nrest2;
  if (tid < MAPSQ_MAX_COLS) {
    s_dst[tid] = a.out[tid];
    const uint32_t c = tid;
    s_src[tid] = c < a.nkey ? nullptr
               : (c < a.nkey + a.nrest1 ? a.rest1[c - a.nkey] : a.rest2[c - a.nkey - a.nrest1]);
  }
  const uint64_t tile = tile0 + blockIdx.x;
  const uint64_t t0 = tile * kETile;
  // the tile's group range from the precomputed first group of every tile (tile_groups_kernel):
  // the groups of rows [t0, t0 + kETile) lie in [first(t), first(t + 1)]
  if (tid == 0) {
    s_g[0] = a.tile_g0[tile];
    s_g[1] = tile + 1 < ntiles ? a.tile_g0[tile + 1] : a.ngroups - 1;
  }
  __syncthreads();
  const uint64_t g0 = s_g[0], g1 = s_g[1];
  const bool staged = g1 - g0 + 1 <= (uint64_t)kEGroups;
  if (staged) {
    for (uint64_t q = tid; q <= g1 - g0; q += kEThreads) {
      const uint64_t g = g0 + q;
      s_off[q] = a.goff[g];
      s_start[q] = a.gstart[g];
      s_split[q] = a.gsplit[g];
      s_end[q] = a.gend[g];
    }
    if (tid == 0) s_off[g1 - g0 + 1] = (g1 + 1 < a.ngroups) ? a.goff[g1 + 1] : a.m;
  }
  __syncthreads();
  const uint64_t idx_mask = (a.ib >= 64) ? ~0ull : ((1ull << a.ib) - 1);
  constexpr int R = kERows * kEChunks;
  // (positions and in-group counters are 32-bit — n < 2^32 — and the group end is tracked as a
  // count-down of the rows left in it: the walk is 32-bit arithmetic except at group changes)
  uint32_t lpos[R], rpos[R];
  int nrow[kEChunks];
#pragma unroll
  for (int c = 0; c < kEChunks; c++) {
    const uint64_t r0 = t0 + ((uint64_t)c * kEThreads + tid) * kERows;
    nrow[c] = 0;
    if (!FULL && r0 >= a.m) continue;
    // locate r0's group
    uint64_t gl, gend;
    uint32_t start, split, end;
    uint64_t gbeg;
    if (staged) {
      uint32_t lo = 0, hi = (uint32_t)(g1 - g0);
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_off[mid] <= r0) lo = mid; else hi = mid - 1;
      }
      gl = lo;
      gbeg = s_off[gl];
      gend = s_off[gl + 1];
      start = s_start[gl]; split = s_split[gl]; end = s_end[gl];
    } else {
      gl = group_of(a.goff, g0, g1, r0);
      gbeg = a.goff[gl];
      gend = (gl + 1 < a.ngroups) ? a.goff[gl + 1] : a.m;
      start = a.gstart[gl]; split = a.gsplit[gl]; end = a.gend[gl];
    }
    uint32_t nR = end - split;
    const uint64_t local = r0 - gbeg;
    uint32_t li, ri;
    if ((local >> 32) == 0) {
      li = (uint32_t)local / nR;
      ri = (uint32_t)local - li * nR;
    } else {
      li = (uint32_t)(local / nR);
      ri = (uint32_t)(local - (uint64_t)li * nR);
    }
    uint32_t left = (uint32_t)min(gend - r0, (uint64_t)0xffffffffu);  // rows left in the group
    const uint32_t nv = FULL ? kERows : (uint32_t)min(a.m - r0, (uint64_t)kERows);
#pragma unroll
    for (int j = 0; j < kERows; j++) {
      if (!FULL && (uint32_t)j >= nv) break;
      if (left == 0) {  // next group (groups are never empty)
        gl++;
        const uint64_t gb = gend;
        if (staged) {
          gend = s_off[gl + 1];
          start = s_start[gl]; split = s_split[gl]; end = s_end[gl];
        } else {
          gend = (gl + 1 < a.ngroups) ? a.goff[gl + 1] : a.m;
          start = a.gstart[gl]; split = a.gsplit[gl]; end = a.gend[gl];
        }
        left = (uint32_t)min(gend - gb, (uint64_t)0xffffffffu);
        nR = end - split;
        li = 0;
        ri = 0;
      }
      lpos[c * kERows + j] = start + li;
      rpos[c * kERows + j] = split + ri;
      nrow[c]++;
      left--;
      if (++ri == nR) {
        ri = 0;
        li++;
      }
    }
  }
  // all word loads of the thread's rows, then decode
  uint64_t lkey[R];
  uint32_t lidx[R], ridx[R];
#pragma unroll
  for (int q = 0; q < R; q++) {
    const bool v = FULL || (q % kERows) < nrow[q / kERows];
    if (a.words) {
      const uint64_t lw = v ? __ldg(a.words + lpos[q]) : 0ull;
      const uint64_t rw = v ? __ldg(a.words + rpos[q]) : 0ull;
      lkey[q] = lw >> a.ib;
      lidx[q] = (uint32_t)(lw & idx_mask);
      ridx[q] = (uint32_t)((rw & idx_mask) - a.n1);
    } else {
      lkey[q] = v ? __ldg(a.keys + lpos[q]) : 0ull;
      lidx[q] = v ? __ldg(a.vals + lpos[q]) : 0u;
      ridx[q] = v ? __ldg(a.vals + rpos[q]) - (uint32_t)a.n1 : 0u;
    }
  }
  for (uint32_t col = 0; col < nout; col++) {
    uint32_t val[R];
    if (col < a.nkey) {
      const uint32_t sh = a.key_shift[col], mk = a.key_mask[col], lo = a.key_lo[col];
#pragma unroll
      for (int q = 0; q < R; q++) val[q] = (uint32_t)(lkey[q] >> sh & mk) + lo;
    } else {
      const uint32_t *src = s_src[col];
      const bool left = col < a.nkey + a.nrest1;
      if (src == nullptr) {  // value-carrying words: the "row id" is the value itself
#pragma unroll
        for (int q = 0; q < R; q++) val[q] = left ? lidx[q] : ridx[q];
      } else {
#pragma unroll
        for (int q = 0; q < R; q++) {
          const bool v = FULL || (q % kERows) < nrow[q / kERows];
          val[q] = v ? __ldg(src + (left ? lidx[q] : ridx[q])) : 0u;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < kEChunks; c++) {
      if (!FULL && nrow[c] == 0) continue;
      const uint64_t r0 = t0 + ((uint64_t)c * kEThreads + tid) * kERows;
      uint32_t *dst = s_dst[col] + r0;
      if (FULL || nrow[c] == kERows) {
#pragma unroll
        for (int v4 = 0; v4 < kERows; v4 += 4)
          st_cs_v4(dst + v4, make_uint4(val[c * kERows + v4], val[c * kERows + v4 + 1],
                                        val[c * kERows + v4 + 2], val[c * kERows + v4 + 3]));
      } else {
#pragma unroll
        for (int j = 0; j < kERows; j++)  // (static indices: no local-memory copy of val[])
          if (j < nrow[c]) st_cs_u32(dst + j, val[c * kERows + j]);
      }
    }
  }
}

// ------------------------------------------------------------------ RESIDUAL / HASH paths
// The sorted words group rows by key' (a packed subset of the shared columns, or a hash of all of
// them), so a key' group's (LEFT, RIGHT) pairs are CANDIDATES: a pair belongs to RS iff the rows
// also agree on every residual shared column (reading R19).  "GPU's SIMD architectures contribute
// to accelerate cartesian product in parallel": the verification is candidate-parallel
// like the expansion — a CTA owns 1024 consecutive candidates (offsets = exclusive scan of
// nL * nR), each thread 4 consecutive ones (C5 J2: 0.52 ms vs 0.57 with 8, 0.56 with 16), so a hot key' group is spread over many CTAs.  Each
// thread compares its candidates' residual columns, the CTA counts the matches, and (WRITE)
// tiles claimed in order resolve their output offset by decoupled look-back and write the matched
// pairs in (key', Tp1 row, Tp2 row) order — one pass, the output gathered only for matches.
// WRITE = false only counts the matches (for joins whose candidate count is too large to size
// the output by).
constexpr int kVThreads = 256;
#ifndef MAPSQ_V_PER
#define MAPSQ_V_PER 4
#endif
constexpr int kVPer = MAPSQ_V_PER;  // (ablation knob -DMAPSQ_V_PER)
constexpr uint64_t kVTile = (uint64_t)kVThreads * kVPer;

template <bool WRITE>
__global__ void __launch_bounds__(kVThreads)
verify_emit_kernel(const ResidualArgs a, const uint64_t *__restrict__ coff,
                   const uint64_t *__restrict__ tile_g0, uint64_t ngroups, uint64_t C,
                   uint64_t *__restrict__ status, uint32_t *__restrict__ tile_ctr,
                   unsigned long long *__restrict__ total) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_g[2], s_base;
  __shared__ uint64_t s_off[kEGroups + 1];
  __shared__ uint32_t s_start[kEGroups], s_split[kEGroups], s_end[kEGroups];
  __shared__ uint32_t s_wsum[kVThreads / 32];
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    const uint32_t t = WRITE ? atomicAdd(tile_ctr, 1u) : blockIdx.x;  // in order (look-back)
    s_tile = t;
    s_g[0] = tile_g0[t];
    s_g[1] = t + 1 < gridDim.x ? tile_g0[t + 1] : ngroups - 1;
  }
  __syncthreads();
  const uint64_t tile = s_tile, t0 = tile * kVTile;
  const uint64_t g0 = s_g[0], g1 = s_g[1];
  const bool staged = g1 - g0 + 1 <= (uint64_t)kEGroups;
  if (staged) {
    for (uint64_t q = tid; q <= g1 - g0; q += kVThreads) {
      const uint64_t g = g0 + q;
      s_off[q] = coff[g];
      s_start[q] = a.gstart[g];
      s_split[q] = a.gsplit[g];
      s_end[q] = a.gend[g];
    }
    if (tid == 0) s_off[g1 - g0 + 1] = (g1 + 1 < ngroups) ? coff[g1 + 1] : C;
  }
  __syncthreads();
  const uint64_t mask = (1ull << a.ib) - 1;
  const uint64_t r0 = t0 + (uint64_t)tid * kVPer;
  uint32_t lidx[kVPer], ridx[kVPer], match = 0;
  if (r0 < C) {
    uint64_t gl, gend;
    uint32_t start, split, end;
    if (staged) {
      uint32_t lo = 0, hi = (uint32_t)(g1 - g0);
      while (lo < hi) {
        const uint32_t mid = (lo + hi + 1) >> 1;
        if (s_off[mid] <= r0) lo = mid; else hi = mid - 1;
      }
      gl = lo;
      gend = s_off[gl + 1];
      start = s_start[gl]; split = s_split[gl]; end = s_end[gl];
      gl += g0;
    } else {
      gl = group_of(coff, g0, g1, r0);
      gend = (gl + 1 < ngroups) ? coff[gl + 1] : C;
      start = a.gstart[gl]; split = a.gsplit[gl]; end = a.gend[gl];
    }
    uint64_t nR = end - split, local = r0 - coff[gl];
    uint64_t li = local / nR, ri = local - li * nR;
    uint32_t valid = 0;
#pragma unroll
    for (int j = 0; j < kVPer; j++) {  // candidate positions, then all word loads together
      const uint64_t r = r0 + j;
      if (r >= C) break;
      if (r >= gend) {  // next group (groups are never empty)
        gl++;
        gend = (gl + 1 < ngroups) ? coff[gl + 1] : C;
        start = a.gstart[gl]; split = a.gsplit[gl]; end = a.gend[gl];
        nR = end - split;
        li = ri = 0;
      }
      lidx[j] = (uint32_t)(start + li);
      ridx[j] = (uint32_t)(split + ri);
      valid |= 1u << j;
      if (++ri == nR) { ri = 0; li++; }
    }
#pragma unroll
    for (int j = 0; j < kVPer; j++) {
      if (!(valid >> j & 1u)) continue;
      lidx[j] = (uint32_t)(__ldg(a.words + lidx[j]) & mask);
      ridx[j] = (uint32_t)((__ldg(a.words + ridx[j]) & mask) - a.n1);
    }
    match = valid;
    for (uint32_t c = 0; c < a.nres; c++) {  // every candidate's loads of a column together
      uint32_t x[kVPer], y[kVPer];
#pragma unroll
      for (int j = 0; j < kVPer; j++) {
        x[j] = (match >> j & 1u) ? ld_rnd(a.res1[c] + lidx[j]) : 0u;
        y[j] = (match >> j & 1u) ? ld_rnd(a.res2[c] + ridx[j]) : 0u;
      }
#pragma unroll
      for (int j = 0; j < kVPer; j++)
        if (x[j] != y[j]) match &= ~(1u << j);
    }
  }
  // block scan of the per-thread match counts
  const uint32_t cnt = __popc(match);
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t wpre = 0, agg = 0;
#pragma unroll
  for (int w = 0; w < kVThreads / 32; w++) {
    const uint32_t v = s_wsum[w];
    if ((uint32_t)w < warp) wpre += v;
    agg += v;
  }
  if (!WRITE) {
    if (tid == 0 && agg) atomicAdd(total, (unsigned long long)agg);
    return;
  }
  if (warp == 0) {
    const uint64_t excl = warp_lookback(status, tile, agg);
    if (lane == 0) {
      s_base = excl;
      if (tile + 1 == gridDim.x) *total = excl + agg;
    }
  }
  __syncthreads();
  if (!match) return;
  const uint64_t pos0 = s_base + wpre + x - cnt;
  for (uint32_t c = 0; c < a.nout; c++) {  // a column's gathers in flight together, then stores
    const uint32_t *src = a.src[c];
    const bool right = a.src_side[c];
    uint32_t v[kVPer];
#pragma unroll
    for (int j = 0; j < kVPer; j++)
      v[j] = (match >> j & 1u) ? ld_rnd(src + (right ? ridx[j] : lidx[j])) : 0u;
    uint32_t *dst = a.out[c] + pos0;
    uint32_t q = 0;
#pragma unroll
    for (int j = 0; j < kVPer; j++)
      if (match >> j & 1u) dst[q++] = v[j];
  }
}

}  // namespace

void launch_find_groups(const uint64_t *words, const uint64_t *keys, const uint32_t *vals,
                        uint64_t n, uint64_t n1, uint32_t ib, GroupOut g, uint64_t *status,
                        uint32_t *tile_counter, uint64_t *ngroups_dev, cudaStream_t s) {
  WordView W;
  W.words = words;
  W.keys = keys;
  W.vals = vals;
  W.n1 = n1;
  W.ib = ib;
  W.idx_mask = (ib >= 64) ? ~0ull : ((1ull << ib) - 1);
  const uint64_t ntiles = ceil_div(n, kGTile);
  constexpr size_t smem = (2 * sizeof(uint32_t) + sizeof(uint16_t)) * kGWarps * kGMaxRec;
  set_smem_limit((const void *)find_groups_kernel<false>, smem);
  set_smem_limit((const void *)find_groups_kernel<true>, smem);
  if (words)
    find_groups_kernel<false><<<(unsigned)ntiles, kGThreads, smem, s>>>(W, n, g, status, tile_counter,
                                                                   ngroups_dev);
  else
    find_groups_kernel<true><<<(unsigned)ntiles, kGThreads, smem, s>>>(W, n, g, status, tile_counter,
                                                                  ngroups_dev);
}

uint64_t find_groups_tiles(uint64_t n) { return ceil_div(n, kGTile); }

uint64_t verify_tiles(uint64_t candidates) { return ceil_div(candidates, kVTile); }

void launch_verify_emit(const ResidualArgs &a, const uint64_t *coff, uint64_t *tile_g0,
                        uint64_t ngroups, uint64_t C, bool write, uint64_t *status,
                        uint32_t *tile_ctr, unsigned long long *total, cudaStream_t s) {
  if (C == 0 || ngroups == 0) return;
  const uint64_t ntiles = verify_tiles(C);
  const unsigned gg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(ntiles, 256), 148 * 16));
  tile_groups_kernel<<<gg, 256, 0, s>>>(coff, ngroups, ntiles, tile_g0, kVTile);
  if (write)
    verify_emit_kernel<true><<<(unsigned)ntiles, kVThreads, 0, s>>>(a, coff, tile_g0, ngroups, C,
                                                                   status, tile_ctr, total);
  else
    verify_emit_kernel<false><<<(unsigned)ntiles, kVThreads, 0, s>>>(a, coff, tile_g0, ngroups, C,
                                                                    status, tile_ctr, total);
}

uint64_t expand_tiles(uint64_t m) { return ceil_div(m, kETile); }

void launch_expand(const ExpandArgs &a, cudaStream_t s) {
  if (a.m == 0) return;
  const uint64_t nblocks = ceil_div(a.m, kETile);
  const unsigned gg = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(nblocks, 256), 148 * 16));
  tile_groups_kernel<<<gg, 256, 0, s>>>(a.goff, a.ngroups, nblocks,
                                        const_cast<uint64_t *>(a.tile_g0), kETile);
  // long runs of one group (C3's star: ~2e4 rows per group) favour 2 chunks of 4 rows per
  // thread; short groups (C5's first join: ~20 rows) one chunk of 8 rows (C3 2.50 vs 2.72 ms,
  // C5 J1 0.88 vs 0.81 ms)
  const uint64_t nfull = a.m / kETile;  // tiles with every row (the last one may be partial)
  static const uint32_t shape = [] {  // (ablation knob MAPSQ_EXPAND_SHAPE: 1 = 8x1, 2 = 4x2)
    const char *e = std::getenv("MAPSQ_EXPAND_SHAPE");
    return (e && *e) ? (uint32_t)std::strtoul(e, nullptr, 10) : 0u;
  }();
  // (no gathers — value-carrying words — also favour 4-row chunks: C4 0.80 -> 0.72 ms)
  bool gathers = false;
  for (uint32_t c = 0; c < a.nrest1; c++) gathers |= a.rest1[c] != nullptr;
  for (uint32_t c = 0; c < a.nrest2; c++) gathers |= a.rest2[c] != nullptr;
  if (shape == 2 || (shape == 0 && (a.m >= 256 * a.ngroups || !gathers))) {
    if (nfull) expand_kernel<4, 2, true><<<(unsigned)nfull, kEThreads, 0, s>>>(a, 0, nblocks);
    if (nblocks > nfull) expand_kernel<4, 2, false><<<1, kEThreads, 0, s>>>(a, nfull, nblocks);
  } else {
    if (nfull) expand_kernel<8, 1, true><<<(unsigned)nfull, kEThreads, 0, s>>>(a, 0, nblocks);
    if (nblocks > nfull) expand_kernel<8, 1, false><<<1, kEThreads, 0, s>>>(a, nfull, nblocks);
  }
}

}  // namespace mapsq
