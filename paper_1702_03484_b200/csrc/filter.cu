// filter.cu — semi-join key-presence filter in front of the Map (SURVEY §8 row f2's semi-join
// reducer, applied on one GPU as well).
//
// ReduceDuplicate emits nothing for a key that occurs on one side only (Alg. 1 l.6-11,
// PAPER.md:127-133; the LEFT/RIGHT flag exists "to reduce unnecessary computation"), so
// such rows can be dropped before the sort without changing RS (reading R18).  One round:
//   1. build:  bm_S = key-presence bitmap of the smaller side S (exact bit = key' when it fits,
//      else a hash of key' — false positives only let rows through, they never drop a match);
//   2. probe L (the larger side) against bm_S: every warp stages its 512-row slice's survivors'
//      words key' << ib | rowid, compacted in row order, plus the slice's count;
//   3. bm_L = bits of L's survivors — set during the probe (exact bitmaps) or from the staged
//      words (8 B per survivor instead of re-reading L's key columns);
//   4. probe S against bm_L, staging its survivors the same way;
//   5. scan the slice counts (side A's slices first) and gather the staged survivors into one
//      contiguous array.
// Within a side the compaction is stable, so the words keep the (key', label, rowid) order of the
// unfiltered join after the stable sort — RS and its row order are unchanged.  Hashed rounds are
// refined by further rounds on the surviving words with fresh seeds (blocked Bloom bitmaps).
#include <cstring>
#include <map>
#include <type_traits>

#include "internal.cuh"

namespace mapsq {
namespace {

#ifndef MAPSQ_G_ROWS
#define MAPSQ_G_ROWS 8
#endif
constexpr int kFThreads = 256;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFItems = 16;                    // rows per lane per slice
constexpr int kFWarpRows = 32 * kFItems;       // 512-row warp slice
constexpr int kFCopies = 4;                    // private digit-histogram copies
constexpr int kSampleStride = 16;              // the sampled probe reads every 16th slice,
constexpr uint64_t kSampleSlices = 8192;       // and at most ~8192 slices (4 M rows)
#ifndef MAPSQ_PROBE_MINB
#define MAPSQ_PROBE_MINB 3  // CTAs per SM of the 64-bit-key probe (ablation knob)
#endif
#ifndef MAPSQ_G_SLICES
#define MAPSQ_G_SLICES 8
#endif
constexpr int kGSlices = MAPSQ_G_SLICES;       // slices per warp iteration of the gather
constexpr int kGRows = MAPSQ_G_ROWS;           // rows per lane in flight in the gather

// MODE 0: one packed key column and kb <= 32 (key' = v - lo in 32-bit arithmetic); 1: generic
// packed composite key; 2: PATH_HASH key over exactly 2 columns; 3: PATH_HASH over nkey columns.
template <int MODE>
using KeyT = typename std::conditional<MODE == 0, uint32_t, uint64_t>::type;
template <int MODE>
__device__ __forceinline__ uint32_t mode_nkey(const PackArgs &a) {
  return MODE == 0 ? 1u : (MODE == 2 ? 2u : a.nkey);
}

__device__ __forceinline__ uint32_t bit_index(uint64_t key, uint32_t bbits, uint32_t hashed) {
  return hashed ? (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - bbits)) : (uint32_t)key;
}

// One side of the join as the filter kernels see it: rows j in [0, rows), key column c at
// col[c][j], row id (in the word) j + id0, slices starting at slice0.
struct Side {
  const uint32_t *col[MAPSQ_MAX_COLS];
  uint64_t rows, id0, slice0;
};

// key' of rows base + it * 32 + lane (it < kFItems), column-outer loads (all of a column's
// loads in flight together); rows >= rows get key' 0 (callers mask them)
// FINAL = false (hash modes, filter-only uses): the key_hash chain without its final mix — the
// filter's bitmap index mixes again, and only the words need the exact key'.
template <int MODE, bool FINAL = true, int N = kFItems>
__device__ __forceinline__ void load_keys(const PackArgs &a, const Side &sd, uint64_t base,
                                          uint32_t lane, KeyT<MODE> key[N],
                                          uint32_t keep = 0xffffu) {
  constexpr bool hash = MODE >= 2;
#pragma unroll
  for (int it = 0; it < N; it++) key[it] = hash ? kKeyHashSeed : 0;
  const uint32_t nk = mode_nkey<MODE>(a);
  for (uint32_t c = 0; c < nk; c++) {
    const uint32_t *p = sd.col[c];
    const uint32_t lo = a.lo[c], sh = a.shift[c];
    uint32_t v[N];
#pragma unroll
    for (int it = 0; it < N; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      v[it] = (j < sd.rows && (keep >> it & 1u)) ? __ldcs(p + j) : lo;
    }
#pragma unroll
    for (int it = 0; it < N; it++)
      key[it] = MODE == 0 ? (KeyT<MODE>)(v[it] - lo)
                     : (KeyT<MODE>)(hash ? key_hash_step(key[it], v[it])
                                         : (key[it] | (uint64_t)(v[it] - lo) << sh));
  }
  if (hash && FINAL) {
#pragma unroll
    for (int it = 0; it < N; it++) key[it] = (KeyT<MODE>)key_hash_final(key[it], a.kb);
  }
}

// Bitmap accesses of the filter kernels carry an L2 evict_last policy: the bitmap (up to
// 64 MB) should survive the key columns streaming past it (those are loaded evict-first, __ldcs).
#ifndef MAPSQ_L2_HINT
#define MAPSQ_L2_HINT 1
#endif
__device__ __forceinline__ uint64_t bm_policy() {
  uint64_t p = 0;
#if MAPSQ_L2_HINT
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
// Bitmap reads ask the L2 for 64-byte fills on a miss (.L2::64B) instead of the default 128: the
// probes touch 8 bytes per key (C5's composite-key probe: 4.49 -> 4.29 GB DRAM, C4's 4.33 ->
// 4.04 GB; builds -3%).  MAPSQ_BM_64B=0: the default fill (ablation).
#ifndef MAPSQ_BM_64B
#define MAPSQ_BM_64B 1
#endif
__device__ __forceinline__ uint64_t ld_bm(const unsigned long long *p, uint64_t pol) {
#if MAPSQ_L2_HINT && MAPSQ_BM_64B
  uint64_t v;
  asm("ld.global.nc.L2::cache_hint.L2::64B.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
#elif MAPSQ_L2_HINT
  uint64_t v;
  asm("ld.global.nc.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(v) : "l"(p), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(p);
#endif
}
__device__ __forceinline__ void red_or_bm(unsigned long long *p, uint64_t m, uint64_t pol) {
#if MAPSQ_L2_HINT
  asm volatile("red.global.or.L2::cache_hint.b64 [%0], %1, %2;" ::"l"(p), "l"(m), "l"(pol) : "memory");
#else
  (void)pol;
  atomicOr(p, (unsigned long long)m);
#endif
}

__device__ __forceinline__ uint32_t ld_bm32(const uint32_t *p, uint64_t pol) {
#if MAPSQ_L2_HINT && MAPSQ_BM_64B
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.L2::64B.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#elif MAPSQ_L2_HINT
  uint32_t v;
  asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
  return v;
#else
  (void)pol;
  return __ldg(p);
#endif
}
__device__ __forceinline__ void red_or_bm32(uint32_t *p, uint32_t m, uint64_t pol) {
#if MAPSQ_L2_HINT
  asm volatile("red.global.or.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(p), "r"(m), "l"(pol) : "memory");
#else
  (void)pol;
  atomicOr(p, m);
#endif
}

// Set bit(key') in bm for the rows whose `keep` bit is set.  Test before set (a plain atomicOr
// per row serialises on hot keys: 40 ms vs 5.9 ms for 5e8 Zipf rows, tools/bitmap_bench.cu), and
// runs of equal keys in consecutive rows (clustered data) set their bit once: a lane whose left
// neighbour holds the same bit skips.
// TEST = false (keys mostly distinct, e.g. hashed composite keys): fire-and-forget RED.OR only
// (208 vs 75 G rows/s for distinct keys, tools/bitmap_bench.cu).
// HINT = false: no L2 policy (the probe's SET bitmap: with the probed one also hot, two 64 MB
// evict_last bitmaps overflow L2 — C4's column probe 2.28 -> 2.57 ms with both hinted).
template <bool TEST = true, bool HINT = true, int N = kFItems>
__device__ __forceinline__ void set_bits(uint32_t *bm, const uint32_t bidx[N],
                                         uint32_t keep, uint32_t lane) {
  const uint64_t pol = HINT ? bm_policy() : 0;
  uint32_t word[N];
#pragma unroll
  for (int it = 0; it < N; it++)  // (read-only path: a stale word costs one more atomic)
    word[it] = (TEST && (keep >> it & 1u)) ? (HINT ? ld_bm32(bm + (bidx[it] >> 5), pol) : __ldg(bm + (bidx[it] >> 5))) : 0u;
#pragma unroll
  for (int it = 0; it < N; it++) {
    const uint32_t b = bidx[it];
    const uint32_t k = keep >> it & 1u;
    const uint32_t bp = __shfl_up_sync(0xffffffffu, b, 1);
    const uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    const bool dup = lane > 0 && kp && bp == b;
    if (k && !dup && !(word[it] >> (b & 31) & 1u)) {
      if (HINT)
        red_or_bm32(bm + (b >> 5), 1u << (b & 31), pol);
      else
        atomicOr(bm + (b >> 5), 1u << (b & 31));
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
filter_build_kernel(const PackArgs a, const Side sd, uint32_t *__restrict__ bm, uint32_t bbits,
                    uint32_t hashed) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE>(a, sd, base, lane, key);
    uint32_t bidx[kFItems], keep = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      bidx[it] = bit_index(key[it], bbits, hashed);
      keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < sd.rows) << it;
    }
    set_bits(bm, bidx, keep, lane);
  }
}

// Sampled probe: every `stride`-th warp slice of the side is probed against bm; sample[0] +=
// survivors, sample[1] += rows probed.  Lets the host skip a filter that would drop little.
template <int MODE>
__global__ void __launch_bounds__(kFThreads)
filter_sample_kernel(const PackArgs a, const Side sd, const uint32_t *__restrict__ bm,
                     uint32_t bbits, uint32_t hashed, uint32_t stride,
                     unsigned long long *__restrict__ sample) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  uint32_t c = 0, rows = 0;
  for (uint64_t ws = ((uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5)) * stride;
       ws * kFWarpRows < sd.rows; ws += nwarps * stride) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE>(a, sd, base, lane, key);
    uint32_t word[kFItems], bidx[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {  // all probes in flight together
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      bidx[it] = bit_index(key[it], bbits, hashed);
      word[it] = j < sd.rows ? ld_bm32(bm + (bidx[it] >> 5), pol) : 0u;
    }
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      rows += base + (uint64_t)it * 32 + lane < sd.rows;
      c += word[it] >> (bidx[it] & 31) & 1u;
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  rows = __reduce_add_sync(0xffffffffu, rows);
  if (lane == 0 && rows) {
    atomicAdd(sample, (unsigned long long)c);
    atomicAdd(sample + 1, (unsigned long long)rows);
  }
}

// ---- blocked Bloom bitmaps (hashed keys): a key sets/tests TWO bits of one 64-bit word (one
// memory access, like a plain bitmap, but ~2/3 of its false positives at C5's load factor).
// wblock: chosen by a mix of key' with a per-round seed (rounds on packed words and the larger
// side's bitmap of the column round), so a later round's false positives are independent of an
// earlier one's.
__device__ __forceinline__ void wblock_key(uint64_t key, uint64_t seed, uint32_t bbits,
                                           uint32_t &idx, uint64_t &m) {
  const uint64_t h = (key ^ seed) * 0x9E3779B97F4A7C15ull;
  idx = (uint32_t)(h >> (70 - bbits));  // 2^(bbits - 6) 64-bit words
  const uint64_t g = h * 0xD6E8FEB86659FD93ull;
  m = (1ull << (g >> 58)) | (1ull << ((g >> 52) & 63));
}
// cblock: the column round's smaller-side bitmap, indexed straight from the 64-bit key_hash
// chain value of the shared columns (already mixed: no further multiply; being wider than the
// words' key' it also removes most key' collisions)
__device__ __forceinline__ void cblock(uint64_t h, uint32_t bbits, uint32_t &idx, uint64_t &m) {
  idx = (uint32_t)(h >> (70 - bbits));
  m = (1ull << (h & 63)) | (1ull << ((h >> 6) & 63));
}

// set (idx, m) for the rows whose keep bit is set (fire-and-forget RED.OR: keys mostly distinct);
// a lane whose left neighbour sets the same block bits skips.  TEST: read the word first and skip
// bits already set (skewed keys: a hot key's word would otherwise serialise its atomics).
template <bool TEST = false, int N = kFItems>
__device__ __forceinline__ void set_blocks(unsigned long long *bm, const uint32_t idx[N],
                                           const uint64_t m[N], uint32_t keep,
                                           uint32_t lane) {
  const uint64_t pol = bm_policy();
  uint64_t cur[TEST ? N : 1];
  if (TEST) {
#pragma unroll
    for (int it = 0; it < N; it++)
      cur[TEST ? it : 0] = (keep >> it & 1u) ? ld_bm(bm + idx[it], pol) : 0ull;
  }
#pragma unroll
  for (int it = 0; it < N; it++) {
    const uint32_t k = keep >> it & 1u;
    const uint32_t ip = __shfl_up_sync(0xffffffffu, idx[it], 1);
    const uint64_t mp = __shfl_up_sync(0xffffffffu, m[it], 1);
    const uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    const bool dup = lane > 0 && kp && ip == idx[it] && mp == m[it];
    const bool have = TEST && (cur[TEST ? it : 0] & m[it]) == m[it];
    if (k && !dup && !have) red_or_bm(bm + idx[it], m[it], pol);
  }
}

// Word segment of one side (packed words key' << ib | row id of that side's rows, ascending).
template <int N = kFItems>
__device__ __forceinline__ void load_words(const SjSeg &sd, uint64_t base, uint32_t lane,
                                           uint64_t w[N]) {
#pragma unroll
  for (int it = 0; it < N; it++) {
    const uint64_t j = base + (uint64_t)it * 32 + lane;
    w[it] = j < sd.rows ? __ldcs(sd.w + j) : 0ull;
  }
}

__global__ void __launch_bounds__(kFThreads, 4)
wfilter_build_kernel(const SjSeg sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                     unsigned long long *__restrict__ bm) {
  constexpr int NB = kFItems / 2;  // batches of 8 rows per lane: four CTAs per SM
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
#pragma unroll
    for (int half = 0; half < 2; half++) {
      const uint64_t base = ws * kFWarpRows + (uint64_t)half * NB * 32;
      uint32_t idx[NB], keep = 0;
      uint64_t w[NB], m[NB];
      load_words<NB>(sd, base, lane, w);
#pragma unroll
      for (int it = 0; it < NB; it++) {
        wblock_key(w[it] >> ib, seed, bbits, idx[it], m[it]);
        keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < sd.rows) << it;
      }
      set_blocks<false, NB>(bm, idx, m, keep, lane);
    }
  }
}

__global__ void __launch_bounds__(kFThreads)
wfilter_sample_kernel(const SjSeg sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                      const unsigned long long *__restrict__ bm, uint32_t stride,
                      unsigned long long *__restrict__ sample) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  uint32_t c = 0, rows = 0;
  for (uint64_t ws = ((uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5)) * stride;
       ws * kFWarpRows < sd.rows; ws += nwarps * stride) {
    const uint64_t base = ws * kFWarpRows;
    uint64_t w[kFItems], v[kFItems], m[kFItems];
    load_words(sd, base, lane, w);
#pragma unroll
    for (int it = 0; it < kFItems; it++) {  // all probes in flight together
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      uint32_t idx;
      wblock_key(w[it] >> ib, seed, bbits, idx, m[it]);
      v[it] = j < sd.rows ? ld_bm(bm + idx, pol) : 0ull;
    }
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const bool in = base + (uint64_t)it * 32 + lane < sd.rows;
      rows += in;
      c += in && (v[it] & m[it]) == m[it];
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  rows = __reduce_add_sync(0xffffffffu, rows);
  if (lane == 0 && rows) {
    atomicAdd(sample, (unsigned long long)c);
    atomicAdd(sample + 1, (unsigned long long)rows);
  }
}

// ---- hashed composite keys (PATH_HASH), first round on the key columns: the smaller side's
// blocked Bloom bitmap from the key_hash chain of its shared columns (load_keys<MODE, false>)
template <int MODE, bool TEST = false>
__global__ void __launch_bounds__(kFThreads, TEST ? 3 : 4)
cfilter_build_kernel(const PackArgs a, const Side sd, uint32_t bbits,
                     unsigned long long *__restrict__ bm) {
  // batches of 8 rows per lane (two per 512-row slice): ~60 registers, four CTAs per SM
  constexpr int NB = kFItems / 2;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
#pragma unroll
    for (int half = 0; half < 2; half++) {
      const uint64_t base = ws * kFWarpRows + (uint64_t)half * NB * 32;
      KeyT<MODE> key[NB];
      load_keys<MODE, false, NB>(a, sd, base, lane, key);
      uint32_t idx[NB], keep = 0;
      uint64_t m[NB];
#pragma unroll
      for (int it = 0; it < NB; it++) {
        cblock(key[it], bbits, idx[it], m[it]);
        keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < sd.rows) << it;
      }
      set_blocks<TEST, NB>(bm, idx, m, keep, lane);
    }
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
cfilter_sample_kernel(const PackArgs a, const Side sd, uint32_t bbits,
                      const unsigned long long *__restrict__ bm, uint32_t stride,
                      unsigned long long *__restrict__ sample) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  uint32_t c = 0, rows = 0;
  for (uint64_t ws = ((uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5)) * stride;
       ws * kFWarpRows < sd.rows; ws += nwarps * stride) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE, false>(a, sd, base, lane, key);
    uint64_t v[kFItems], m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      uint32_t idx;
      cblock(key[it], bbits, idx, m[it]);
      v[it] = j < sd.rows ? ld_bm(bm + idx, pol) : 0ull;
    }
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const bool in = base + (uint64_t)it * 32 + lane < sd.rows;
      rows += in;
      c += in && (v[it] & m[it]) == m[it];
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  rows = __reduce_add_sync(0xffffffffu, rows);
  if (lane == 0 && rows) {
    atomicAdd(sample, (unsigned long long)c);
    atomicAdd(sample + 1, (unsigned long long)rows);
  }
}

// ---- probe + slice-local compaction: ONE pass over a side's keys ------------------------------
// Each warp owns 512-row slices (grid-stride, no CTA barrier, every load of a column in flight
// together): it probes the bitmap and writes its slice's survivors' words key' << ib | row id,
// compacted in row order, to stage[slice * 512 ..] plus the slice's survivor count.  No key column
// is read twice and no survivor mask is stored; a scan of the slice counts and sj_gather then move
// only the survivors (8 B each) to their final, contiguous positions.  With SET the survivors
// also set their bit in a second (plain) bitmap.
//   KM (key mode): 0 one packed column (plain bitmap), 2 / 3 PATH_HASH over 2 / nkey columns,
//                  4 packed words of a previous round;
//   BM (probed bitmap): 0 plain bit (bit_index of key'), 1 cblock of the key_hash chain,
//                  2 wblock of key' with `seed`.
__device__ __forceinline__ uint64_t opaque(uint64_t x) {
  asm volatile("mov.b64 %0, %0;" : "+l"(x));
  return x;
}

// bitmap slot of key' (or the chain, BM 1): idx and the bit mask tested / set there
template <int BM>
__device__ __forceinline__ void probe_slot(uint64_t key, uint32_t bbits, uint32_t hashed,
                                           uint64_t seed, uint32_t &idx, uint64_t &m) {
  if (BM == 0) {
    const uint32_t b = bit_index(key, bbits, hashed);
    idx = b >> 5;
    m = 1ull << (b & 31);
  } else if (BM == 1) {
    cblock(key, bbits, idx, m);
  } else {
    wblock_key(key, seed, bbits, idx, m);
  }
}

template <int KM, int BM, bool SET>
__global__ void __launch_bounds__(kFThreads, MAPSQ_PROBE_MINB)
sj_probe_stage_kernel(const PackArgs a, const Side sd, const SjSeg ws, const void *__restrict__ bm,
                      uint32_t bbits, uint32_t hashed, uint64_t seed,
                      uint32_t *__restrict__ bm_set, uint64_t *__restrict__ stage,
                      uint32_t *__restrict__ cnt) {
  // registers: the keys and the probed bitmap words only (slots and masks are recomputed from
  // the key, a few ALU ops) — 32-bit for a single packed column against a plain bitmap.  64-bit
  // keys are processed in batches of 8 rows per lane (two per 512-row slice) so three CTAs fit
  // an SM (the same loads in flight per SM, more warps to hide the random-access latency).
  using KT = typename std::conditional<KM == 0, uint32_t, uint64_t>::type;
  using VT = typename std::conditional<BM == 0, uint32_t, uint64_t>::type;
  constexpr int NB = kFItems / 2;
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  const uint64_t rows = KM == 4 ? ws.rows : sd.rows;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  const uint64_t pol = bm_policy();
  constexpr int CM = KM == 4 ? 1 : KM;  // column mode for load_keys (unused for words)
  for (uint64_t wsl = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5); wsl * kFWarpRows < rows;
       wsl += nwarps) {
    uint32_t r = 0;  // the slice's survivors so far
#pragma unroll
    for (int half = 0; half < kFItems / NB; half++) {
      const uint64_t base = wsl * kFWarpRows + (uint64_t)half * NB * 32;
      // key' (the words themselves for KM 4; the key_hash chain for BM 1) of every item
      KT key[NB];
      if (KM == 4) {
        uint64_t w[NB];
        load_words<NB>(ws, base, lane, w);
#pragma unroll
        for (int it = 0; it < NB; it++) key[it] = (KT)w[it];
      } else {
        KeyT<CM> k[NB];
        load_keys<CM, BM != 1, NB>(a, sd, base, lane, k);
#pragma unroll
        for (int it = 0; it < NB; it++) key[it] = (KT)k[it];
      }
      const uint32_t lim = base < rows ? (uint32_t)std::min<uint64_t>(rows - base, NB * 32) : 0u;
      VT v[NB];
#pragma unroll
      for (int it = 0; it < NB; it++) {  // all probes of the batch in flight together
        const bool in = (uint32_t)it * 32 + lane < lim;
        uint32_t idx;
        uint64_t m;
        probe_slot<BM>(KM == 4 ? (uint64_t)key[it] >> a.ib : (uint64_t)key[it], bbits, hashed, seed,
                       idx, m);
        if (BM == 0)
          v[it] = in ? (VT)ld_bm32(reinterpret_cast<const uint32_t *>(bm) + idx, pol) : (VT)0;
        else
          v[it] = in ? (VT)ld_bm(reinterpret_cast<const unsigned long long *>(bm) + idx, pol) : (VT)0;
      }
      uint32_t keep = 0;
#pragma unroll
      for (int it = 0; it < NB; it++) {
        uint32_t idx;
        uint64_t m;
        // (an opaque copy: the slot is recomputed here instead of being kept live across the probes)
        const uint64_t kq = opaque((uint64_t)key[it]);
        probe_slot<BM>(KM == 4 ? kq >> a.ib : kq, bbits, hashed, seed, idx, m);
        const bool k = ((uint64_t)v[it] & m) == m && (uint32_t)it * 32 + lane < lim;
        keep |= (uint32_t)k << it;
        const uint32_t bal = __ballot_sync(0xffffffffu, k);
        if (k) {
          uint64_t w;
          if (KM == 4) {
            w = key[it];
          } else {
            const uint64_t kp = (BM == 1) ? key_hash_final(key[it], a.kb) : (uint64_t)key[it];
            w = (kp << a.ib) | (base + (uint64_t)it * 32 + lane + sd.id0);
          }
          __stcs(stage + wsl * kFWarpRows + r + __popc(bal & lt), w);
        }
        r += __popc(bal);
      }
      if (SET) {
        uint32_t bidx[NB];
#pragma unroll
        for (int it = 0; it < NB; it++) bidx[it] = bit_index((uint64_t)key[it], bbits, hashed);
        set_bits<true, false, NB>(bm_set, bidx, keep, lane);
      }
    }
    if (lane == 0) cnt[sd.slice0 + wsl] = r;
  }
}

// The single packed column against a plain bitmap (KM 0, BM 0): 32-bit keys, 16 rows per lane in
// one batch, four CTAs per SM.
template <int KM, int BM, bool SET>
__global__ void __launch_bounds__(kFThreads, 4)
sj_probe_stage16_kernel(const PackArgs a, const Side sd, const SjSeg ws, const void *__restrict__ bm,
                      uint32_t bbits, uint32_t hashed, uint64_t seed,
                      uint32_t *__restrict__ bm_set, uint64_t *__restrict__ stage,
                      uint32_t *__restrict__ cnt) {
  // registers: the keys and the probed bitmap words only (slots and masks are recomputed from
  // the key, a few ALU ops) — 32-bit for a single packed column against a plain bitmap
  using KT = typename std::conditional<KM == 0, uint32_t, uint64_t>::type;
  using VT = typename std::conditional<BM == 0, uint32_t, uint64_t>::type;
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  const uint64_t rows = KM == 4 ? ws.rows : sd.rows;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  const uint64_t pol = bm_policy();
  constexpr int CM = KM == 4 ? 1 : KM;  // column mode for load_keys (unused for words)
  for (uint64_t wsl = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5); wsl * kFWarpRows < rows;
       wsl += nwarps) {
    const uint64_t base = wsl * kFWarpRows;
    // key' (the words themselves for KM 4; the key_hash chain for BM 1) of every item
    KT key[kFItems];
    if (KM == 4) {
      uint64_t w[kFItems];
      load_words(ws, base, lane, w);
#pragma unroll
      for (int it = 0; it < kFItems; it++) key[it] = (KT)w[it];
    } else {
      KeyT<CM> k[kFItems];
      load_keys<CM, BM != 1>(a, sd, base, lane, k);
#pragma unroll
      for (int it = 0; it < kFItems; it++) key[it] = (KT)k[it];
    }
    const uint32_t lim = (uint32_t)std::min<uint64_t>(rows - base, kFWarpRows);
    VT v[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {  // all probes in flight together
      const bool in = (uint32_t)it * 32 + lane < lim;
      uint32_t idx;
      uint64_t m;
      probe_slot<BM>(KM == 4 ? (uint64_t)key[it] >> a.ib : (uint64_t)key[it], bbits, hashed, seed,
                     idx, m);
      if (BM == 0)
        v[it] = in ? (VT)ld_bm32(reinterpret_cast<const uint32_t *>(bm) + idx, pol) : (VT)0;
      else
        v[it] = in ? (VT)ld_bm(reinterpret_cast<const unsigned long long *>(bm) + idx, pol) : (VT)0;
    }
    uint32_t keep = 0, r = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      uint32_t idx;
      uint64_t m;
      // (an opaque copy: the slot is recomputed here instead of being kept live across the probes)
      const uint64_t kq = opaque((uint64_t)key[it]);
      probe_slot<BM>(KM == 4 ? kq >> a.ib : kq, bbits, hashed, seed, idx, m);
      const bool k = ((uint64_t)v[it] & m) == m && (uint32_t)it * 32 + lane < lim;
      keep |= (uint32_t)k << it;
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      if (k) {
        uint64_t w;
        if (KM == 4) {
          w = key[it];
        } else {
          const uint64_t kp = (BM == 1) ? key_hash_final(key[it], a.kb) : (uint64_t)key[it];
          w = (kp << a.ib) | (base + (uint64_t)it * 32 + lane + sd.id0);
        }
        __stcs(stage + base + r + __popc(bal & lt), w);
      }
      r += __popc(bal);
    }
    if (lane == 0) cnt[sd.slice0 + wsl] = r;
    if (SET) {
      uint32_t bidx[kFItems];
#pragma unroll
      for (int it = 0; it < kFItems; it++) bidx[it] = bit_index((uint64_t)key[it], bbits, hashed);
      set_bits<true, false>(bm_set, bidx, keep, lane);
    }
  }
}

// a survivor's value of a carried column, with 64-byte L2 fills (C4: ~2 survivors per 128-byte
// line; the gathers' DRAM reads 1.80 -> 1.30 GB, 0.69 -> 0.59 ms; MAPSQ_VAL_64B=0: default fills)
#ifndef MAPSQ_VAL_64B
#define MAPSQ_VAL_64B 1
#endif
__device__ __forceinline__ uint32_t ld_val(const uint32_t *p) {
#if MAPSQ_VAL_64B
  uint32_t v;
  asm("ld.global.nc.L2::64B.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
#else
  return __ldg(p);
#endif
}

// Gather: slice s's staged survivors (cnt[s] words at stage[s * 512 ..]) go to out[off[s] ..]
// (the exclusive scan of the counts over side A's slices then side B's: the output is
// contiguous, side A first, row order kept); digit 0 of the words is counted into hist.
// With CARRY the survivors' values of the carried columns are gathered too (by the staged word's
// row id: ascending within a slice, so a warp's loads share lines) into out[c][position], and each
// word's row id becomes its position + id0 (side B's offset by n1).
template <bool CARRY>
__global__ void __launch_bounds__(kFThreads)
sj_gather_kernel(const uint64_t *__restrict__ stage, const uint32_t *__restrict__ cnt,
                 const uint64_t *__restrict__ off, uint64_t nslices, uint64_t *__restrict__ out,
                 uint32_t *__restrict__ hist, uint32_t bit_lo, uint32_t dmask, const SjCarry cr,
                 uint32_t ib, uint64_t id0) {
  __shared__ uint32_t s_h[kFCopies][kRadix];
  if (hist)
    for (uint32_t i = threadIdx.x; i < kFCopies * kRadix; i += kFThreads) (&s_h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31;
  uint32_t *h = s_h[(threadIdx.x >> 5) % kFCopies];
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  const uint64_t imask = (1ull << ib) - 1;
  // a warp moves the survivors of kGSlices consecutive slices per iteration as ONE flat list (a
  // slice keeps ~36 of its 512 rows on C4: per-slice loops left the loads of a warp nearly
  // serial); their output positions are contiguous: off[s0] + flat index
  const uint64_t ngrp = (nslices + kGSlices - 1) / kGSlices;
  for (uint64_t g = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5); g < ngrp; g += nwarps) {
    const uint64_t s0 = g * kGSlices;
    uint32_t c = 0;
    uint64_t p = 0;
    if (lane < kGSlices && s0 + lane < nslices) {
      c = __ldg(cnt + s0 + lane);
      p = __ldg(off + s0 + lane);
    }
    uint32_t e = c;  // inclusive scan of the counts over lanes 0 .. kGSlices - 1
#pragma unroll
    for (int o = 1; o < kGSlices; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, e, o);
      if (lane >= (uint32_t)o) e += y;
    }
    const uint32_t total = __shfl_sync(0xffffffffu, e, kGSlices - 1);
    if (total == 0) continue;  // warp-uniform
    const uint64_t pos = __shfl_sync(0xffffffffu, p, 0);
    uint32_t ends[kGSlices];
#pragma unroll
    for (int i = 0; i < kGSlices; i++) ends[i] = __shfl_sync(0xffffffffu, e, i);
    const uint32_t excl = e - c;
    for (uint32_t f0 = 0; f0 < total; f0 += kGRows * 32) {  // kGRows rows per lane in flight
      uint64_t w[kGRows];
#pragma unroll
      for (int q = 0; q < kGRows; q++) {
        const uint32_t f = f0 + q * 32 + lane;
        uint32_t j = 0;
#pragma unroll
        for (int i = 0; i < kGSlices - 1; i++) j += f >= ends[i];
        const uint32_t st = __shfl_sync(0xffffffffu, excl, j);
        w[q] = f < total ? __ldcs(stage + (s0 + j) * kFWarpRows + (f - st)) : 0ull;
      }
      uint32_t pvv[kGRows];  // value-carrying words: the side's value of each survivor's row
#pragma unroll
      for (int q = 0; q < kGRows; q++) {
        const uint32_t f = f0 + q * 32 + lane;
        pvv[q] = (CARRY && cr.pv && cr.n && f < total)
                     ? ld_val(cr.src[0] + ((w[q] & imask) - id0)) : 0u;
      }
#pragma unroll
      for (int q = 0; q < kGRows; q++) {
        const uint32_t f = f0 + q * 32 + lane;
        if (f < total) {
          const uint64_t x = !CARRY ? w[q]
                             : cr.pv ? ((w[q] >> ib) << ib) | (id0 ? 1ull << 32 : 0ull) | pvv[q]
                                     : ((w[q] >> ib) << ib) | (pos + f + id0);
          __stcs(out + pos + f, x);
          if (hist) atomicAdd(h + ((uint32_t)(x >> bit_lo) & dmask), 1u);
        }
      }
      if (CARRY && !cr.pv) {
        for (uint32_t k = 0; k < cr.n; k++) {
          uint32_t v[kGRows];
#pragma unroll
          for (int q = 0; q < kGRows; q++) {
            const uint32_t f = f0 + q * 32 + lane;
            v[q] = f < total ? ld_val(cr.src[k] + ((w[q] & imask) - id0)) : 0u;
          }
#pragma unroll
          for (int q = 0; q < kGRows; q++) {
            const uint32_t f = f0 + q * 32 + lane;
            if (f < total) __stcs(cr.out[k] + pos + f, v[q]);
          }
        }
      }
    }
  }
  if (hist) {
    __syncthreads();
    for (uint32_t d = threadIdx.x; d < kRadix; d += kFThreads) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < kFCopies; q++) c += s_h[q][d];
      if (c) atomicAdd(hist + d, c);
    }
  }
}

// Set the bits of the words w[0 .. *count) (a side's survivors, gathered) in bm: KIND 0 = plain
// bit of key' (test before set), 2 = wblock of key' with `seed`.  Reads 8 B per survivor
// instead of the side's key columns.
template <int KIND>
__global__ void __launch_bounds__(kFThreads, 4)
sj_set_words_kernel(const uint64_t *__restrict__ w, const uint64_t *__restrict__ count,
                    uint32_t ib, uint32_t bbits, uint32_t hashed, uint64_t seed, void *bm) {
  constexpr int NB = kFItems / 2;  // batches of 8 rows per lane: four CTAs per SM
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t rows = *count;
  const SjSeg sd{w, rows};
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < rows; ws += nwarps) {
#pragma unroll
    for (int half = 0; half < 2; half++) {
      const uint64_t base = ws * kFWarpRows + (uint64_t)half * NB * 32;
      uint64_t wv[NB];
      load_words<NB>(sd, base, lane, wv);
      uint32_t idx[NB], keep = 0;
      uint64_t m[NB];
#pragma unroll
      for (int it = 0; it < NB; it++) {
        keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < rows) << it;
        if (KIND == 0)
          idx[it] = bit_index(wv[it] >> ib, bbits, hashed);
        else
          wblock_key(wv[it] >> ib, seed, bbits, idx[it], m[it]);
      }
      if (KIND == 0)
        set_bits<true, true, NB>(reinterpret_cast<uint32_t *>(bm), idx, keep, lane);
      else
        set_blocks<false, NB>(reinterpret_cast<unsigned long long *>(bm), idx, m, keep, lane);
    }
  }
}

// ---- distributed pre-filter: mask-producing probe over the key_hash chain (cblock bitmaps)
template <int MODE, bool SET>
__global__ void __launch_bounds__(kFThreads)
sj_chain_probe_kernel(const PackArgs a, const Side sd, uint32_t bbits,
                      const unsigned long long *__restrict__ bm,
                      unsigned long long *__restrict__ bm_set, uint32_t *__restrict__ mask) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE, false>(a, sd, base, lane, key);
    uint64_t v[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      uint32_t idx;
      uint64_t m;
      cblock(key[it], bbits, idx, m);
      v[it] = base + (uint64_t)it * 32 + lane < sd.rows ? ld_bm(bm + idx, pol) : 0ull;
    }
    uint32_t keep = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      uint32_t idx;
      uint64_t m;
      cblock(opaque(key[it]), bbits, idx, m);
      const bool k = (v[it] & m) == m && base + (uint64_t)it * 32 + lane < sd.rows;
      keep |= (uint32_t)k << it;
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      if (lane == 0 && base + (uint64_t)it * 32 < sd.rows) mask[(base >> 5) + it] = bal;
    }
    if (SET) {
      uint32_t idx[kFItems];
      uint64_t m[kFItems];
#pragma unroll
      for (int it = 0; it < kFItems; it++) cblock(key[it], bbits, idx[it], m[it]);
      set_blocks<true>(bm_set, idx, m, keep, lane);
    }
  }
}

// Every rank reduces its slice of the bitmap words over all peers and writes the OR back to all
// of them: 16 B vector loads / stores over the NVLink peer mappings.
__global__ void __launch_bounds__(256)
peer_or_kernel(unsigned long long *const *__restrict__ peers, int world, uint64_t lo, uint64_t hi) {
  for (uint64_t w = lo + 2 * ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x); w < hi;
       w += 2ull * gridDim.x * blockDim.x) {
    ulonglong2 v = make_ulonglong2(0, 0);
    if (w + 1 < hi) {
      for (int q = 0; q < world; q++) {
        const ulonglong2 x = __ldcg(reinterpret_cast<const ulonglong2 *>(peers[q] + w));
        v.x |= x.x;
        v.y |= x.y;
      }
      for (int q = 0; q < world; q++) *reinterpret_cast<ulonglong2 *>(peers[q] + w) = v;
    } else {
      unsigned long long x = 0;
      for (int q = 0; q < world; q++) x |= __ldcg(peers[q] + w);
      for (int q = 0; q < world; q++) peers[q][w] = x;
    }
  }
}

Side side_of(const PackArgs &a, bool b) {
  Side sd;
  for (uint32_t c = 0; c < MAPSQ_MAX_COLS; c++)
    sd.col[c] = c < a.nkey ? (b ? a.key2[c] : a.key1[c]) : nullptr;
  sd.rows = b ? a.n2 : a.n1;
  sd.id0 = b ? a.n1 : 0;
  sd.slice0 = b ? ceil_div(a.n1, kFWarpRows) : 0;
  return sd;
}

uint32_t sample_stride(uint64_t rows) {  // slices between sampled slices
  return (uint32_t)std::max<uint64_t>(kSampleStride, ceil_div(ceil_div(rows, kFWarpRows), kSampleSlices));
}

int sample_grid(uint64_t rows) {  // one warp per sampled slice (up to 148 x 8 CTAs)
  const uint64_t sampled = ceil_div(ceil_div(rows, kFWarpRows), sample_stride(rows));
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(sampled, kFWarps), 148 * 8));
}

int grid_for_rows(uint64_t rows) {
  const uint64_t blocks = ceil_div(ceil_div(rows, kFWarpRows), kFWarps);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(blocks, 148 * 8));
}

int filter_mode(const PackArgs &a) {
  if (a.hash) return a.nkey == 2 ? 2 : 3;
  return (a.nkey == 1 && a.kb <= 32) ? 0 : 1;
}

template <int KM, int BM, bool SET>
void probe_launch(const PackArgs &a, const Side &sd, const SjSeg &ws, const void *bm,
                  uint32_t bbits, uint32_t hashed, uint64_t seed, uint32_t *bm_set,
                  uint64_t *stage, uint32_t *cnt, cudaStream_t s) {
  const uint64_t rows = KM == 4 ? ws.rows : sd.rows;
  if (rows == 0) return;
  if constexpr (KM == 0)
    sj_probe_stage16_kernel<KM, BM, SET><<<grid_for_rows(rows), kFThreads, 0, s>>>(
        a, sd, ws, bm, bbits, hashed, seed, bm_set, stage, cnt);
  else
    sj_probe_stage_kernel<KM, BM, SET><<<grid_for_rows(rows), kFThreads, 0, s>>>(
        a, sd, ws, bm, bbits, hashed, seed, bm_set, stage, cnt);
}

}  // namespace

uint64_t sj_slices(uint64_t rows) { return ceil_div(rows, kFWarpRows); }
uint64_t sj_sample_rows(uint64_t rows) {
  return std::min(rows, ceil_div(ceil_div(rows, kFWarpRows), sample_stride(rows)) * kFWarpRows);
}

void launch_sj_build_sample_cols(const PackArgs &a, bool s_is_b, void *bmS, uint32_t bbits,
                                 uint32_t hashed, unsigned long long *sample, cudaStream_t s,
                                 uint64_t l_rows, const std::function<void()> &before_sample) {
  const Side S = side_of(a, s_is_b);
  Side L = side_of(a, !s_is_b);
  L.rows = std::min(L.rows, l_rows);
  const int gs = grid_for_rows(S.rows);
  const int mode = filter_mode(a);
  if (mode == 0) {
    filter_build_kernel<0><<<gs, kFThreads, 0, s>>>(a, S, (uint32_t *)bmS, bbits, hashed);
    if (before_sample) before_sample();
    if (L.rows)
      filter_sample_kernel<0><<<sample_grid(L.rows), kFThreads, 0, s>>>(
          a, L, (const uint32_t *)bmS, bbits, hashed, sample_stride(L.rows), sample);
  } else if (mode == 2) {
    cfilter_build_kernel<2><<<gs, kFThreads, 0, s>>>(a, S, bbits, (unsigned long long *)bmS);
    if (before_sample) before_sample();
    if (L.rows)
      cfilter_sample_kernel<2><<<sample_grid(L.rows), kFThreads, 0, s>>>(
          a, L, bbits, (const unsigned long long *)bmS, sample_stride(L.rows), sample);
  } else {
    cfilter_build_kernel<3><<<gs, kFThreads, 0, s>>>(a, S, bbits, (unsigned long long *)bmS);
    if (before_sample) before_sample();
    if (L.rows)
      cfilter_sample_kernel<3><<<sample_grid(L.rows), kFThreads, 0, s>>>(
          a, L, bbits, (const unsigned long long *)bmS, sample_stride(L.rows), sample);
  }
}

void launch_sj_probe_cols(const PackArgs &a, bool side_b, int bm_kind, const void *bm,
                          uint32_t bbits, uint32_t hashed, uint64_t seed, uint32_t *bm_set,
                          uint64_t *stage, uint32_t *cnt, cudaStream_t s, uint64_t row_lo,
                          uint64_t row_hi) {
  Side sd = side_of(a, side_b);
  const SjSeg none{nullptr, 0};
  // rows [row_lo, row_hi) of the side: its slices from row_lo / 512 on
  row_hi = std::min(row_hi, sd.rows);
  if (row_lo >= row_hi) return;
  for (uint32_t c = 0; c < a.nkey; c++) sd.col[c] += row_lo;
  sd.rows = row_hi - row_lo;
  sd.id0 += row_lo;
  sd.slice0 += row_lo / kFWarpRows;
  // the side's slices: stage[slice * 512 ..] and cnt[slice], side B after side A's slices
  stage += sd.slice0 * kFWarpRows;
  const int mode = filter_mode(a);
  if (mode == 0) {
    if (bm_set)
      probe_launch<0, 0, true>(a, sd, none, bm, bbits, hashed, seed, bm_set, stage, cnt, s);
    else
      probe_launch<0, 0, false>(a, sd, none, bm, bbits, hashed, seed, nullptr, stage, cnt, s);
  } else if (mode == 2) {
    if (bm_kind == 1)
      probe_launch<2, 1, false>(a, sd, none, bm, bbits, hashed, seed, nullptr, stage, cnt, s);
    else
      probe_launch<2, 2, false>(a, sd, none, bm, bbits, hashed, seed, nullptr, stage, cnt, s);
  } else {
    if (bm_kind == 1)
      probe_launch<3, 1, false>(a, sd, none, bm, bbits, hashed, seed, nullptr, stage, cnt, s);
    else
      probe_launch<3, 2, false>(a, sd, none, bm, bbits, hashed, seed, nullptr, stage, cnt, s);
  }
}

void launch_sj_probe_words(const SjSeg &in, uint64_t slice0, uint32_t ib, const void *bm,
                           uint32_t bbits, uint64_t seed, uint64_t *stage, uint32_t *cnt,
                           cudaStream_t s) {
  PackArgs a;
  std::memset(&a, 0, sizeof a);
  a.ib = ib;
  Side sd;
  std::memset(&sd, 0, sizeof sd);
  sd.slice0 = slice0;
  probe_launch<4, 2, false>(a, sd, in, bm, bbits, 0, seed, nullptr, stage + slice0 * kFWarpRows,
                            cnt, s);
}

void launch_sj_set_words(const uint64_t *w, const uint64_t *count, uint64_t max_rows, int kind,
                         void *bm, uint32_t ib, uint32_t bbits, uint32_t hashed, uint64_t seed,
                         cudaStream_t s) {
  if (max_rows == 0) return;
  const int g = grid_for_rows(max_rows);
  if (kind == 0)
    sj_set_words_kernel<0><<<g, kFThreads, 0, s>>>(w, count, ib, bbits, hashed, seed, bm);
  else
    sj_set_words_kernel<2><<<g, kFThreads, 0, s>>>(w, count, ib, bbits, hashed, seed, bm);
}

void launch_sj_gather(const uint64_t *stage, const uint32_t *cnt, const uint64_t *off,
                      uint64_t nslices, uint64_t *out, uint32_t *hist, uint32_t bit_lo,
                      uint32_t dmask, const SjCarry &cr, uint32_t ib, uint64_t id0,
                      cudaStream_t s) {
  if (nslices == 0) return;
  const int g = grid_for_rows(nslices * kFWarpRows);
  if (cr.n || cr.pv)
    sj_gather_kernel<true><<<g, kFThreads, 0, s>>>(stage, cnt, off, nslices, out, hist, bit_lo,
                                                   dmask, cr, ib, id0);
  else
    sj_gather_kernel<false><<<g, kFThreads, 0, s>>>(stage, cnt, off, nslices, out, hist, bit_lo,
                                                    dmask, cr, ib, id0);
}

void launch_sj_chain_build(const PackArgs &a, bool side_b, void *bm, uint32_t bbits, cudaStream_t s) {
  const Side sd = side_of(a, side_b);
  if (sd.rows == 0) return;
  auto *b = reinterpret_cast<unsigned long long *>(bm);
  // (test before set: the distributed filter also serves skewed single-column keys)
  if (a.nkey == 2)
    cfilter_build_kernel<2, true><<<grid_for_rows(sd.rows), kFThreads, 0, s>>>(a, sd, bbits, b);
  else
    cfilter_build_kernel<3, true><<<grid_for_rows(sd.rows), kFThreads, 0, s>>>(a, sd, bbits, b);
}

void launch_sj_chain_probe(const PackArgs &a, bool side_b, const void *bm, uint32_t bbits,
                           void *bm_set, uint32_t *mask, cudaStream_t s) {
  const Side sd = side_of(a, side_b);
  if (sd.rows == 0) return;
  const auto *b = reinterpret_cast<const unsigned long long *>(bm);
  auto *bs = reinterpret_cast<unsigned long long *>(bm_set);
  const int g = grid_for_rows(sd.rows);
  if (a.nkey == 2) {
    if (bs) sj_chain_probe_kernel<2, true><<<g, kFThreads, 0, s>>>(a, sd, bbits, b, bs, mask);
    else sj_chain_probe_kernel<2, false><<<g, kFThreads, 0, s>>>(a, sd, bbits, b, bs, mask);
  } else {
    if (bs) sj_chain_probe_kernel<3, true><<<g, kFThreads, 0, s>>>(a, sd, bbits, b, bs, mask);
    else sj_chain_probe_kernel<3, false><<<g, kFThreads, 0, s>>>(a, sd, bbits, b, bs, mask);
  }
}

void launch_sj_chain_sample(const PackArgs &a, bool side_b, const void *bm, uint32_t bbits,
                            unsigned long long *sample, cudaStream_t s) {
  const Side sd = side_of(a, side_b);
  if (sd.rows == 0) return;
  const auto *b = reinterpret_cast<const unsigned long long *>(bm);
  if (a.nkey == 2)
    cfilter_sample_kernel<2><<<sample_grid(sd.rows), kFThreads, 0, s>>>(a, sd, bbits, b, sample_stride(sd.rows), sample);
  else
    cfilter_sample_kernel<3><<<sample_grid(sd.rows), kFThreads, 0, s>>>(a, sd, bbits, b, sample_stride(sd.rows), sample);
}

void launch_peer_or(unsigned long long *const *peers, int world, int rank, uint64_t words,
                    cudaStream_t s) {
  const uint64_t lo = words * rank / world & ~1ull, hi = rank + 1 == world ? words : (words * (rank + 1) / world & ~1ull);
  if (hi <= lo) return;
  const uint64_t n2 = (hi - lo + 1) / 2;
  const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n2, 256), 148 * 8));
  peer_or_kernel<<<g, 256, 0, s>>>(peers, world, lo, hi);
}

void launch_sj_build_words(const SjSeg &S, uint32_t ib, uint64_t seed, uint32_t bbits, void *bm,
                           cudaStream_t s) {
  if (S.rows == 0) return;
  wfilter_build_kernel<<<grid_for_rows(S.rows), kFThreads, 0, s>>>(
      S, ib, seed, bbits, reinterpret_cast<unsigned long long *>(bm));
}

void launch_sj_sample_words(const SjSeg &L, uint32_t ib, uint64_t seed, uint32_t bbits,
                            const void *bm, unsigned long long *sample, cudaStream_t s) {
  if (L.rows == 0) return;
  wfilter_sample_kernel<<<sample_grid(L.rows), kFThreads, 0, s>>>(
      L, ib, seed, bbits, reinterpret_cast<const unsigned long long *>(bm), sample_stride(L.rows), sample);
}

}  // namespace mapsq
