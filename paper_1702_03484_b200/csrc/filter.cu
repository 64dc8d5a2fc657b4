// filter.cu — semi-join key-presence filter in front of the Map (SURVEY §8 row f2's semi-join
// reducer, applied on one GPU as well).
//
// ReduceDuplicate emits nothing for a key that occurs on one side only (Alg. 1 l.6-11,
// PAPER.md:127-133; the LEFT/RIGHT flag exists "to reduce unnecessary computation"), so
// such rows can be dropped before the sort without changing RS.  Key-presence bitmaps over the
// packed key key' (exact when kb <= bbits, else indexed by a multiplicative hash of key' —
// false positives only let rows through, they never drop a match) are built in three passes:
//   1. build:  bm_S = keys of the smaller side S;
//   2. probe L (the larger side) against bm_S; every surviving L row also sets its bit in bm_L
//      (so bm_L holds exactly the keys of L that occur in S);
//   3. probe S against bm_L.
// Each probe records one survivor bit per row and a count per 512-row warp slice (side A's rows
// fill slices [0, nslA), side B's the slices after), the counts are scanned, and an emit pass
// writes each slice's survivors at its offset in row order.  The compaction is stable, so the
// surviving words keep ascending row ids and the sort's (key', label, rowid) order — and
// therefore RS and its row order — are exactly those of the unfiltered join.
#include <type_traits>

#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kFThreads = 256;
constexpr int kFWarps = kFThreads / 32;
constexpr int kFItems = 16;                    // rows per lane per slice
constexpr int kFWarpRows = 32 * kFItems;       // 512-row warp slice
constexpr int kFCopies = 4;                    // private digit-histogram copies
constexpr uint32_t kDenseSlice = 160;          // survivors above which the emit walks items
constexpr int kSampleStride = 16;              // the sampled probe reads every 16th slice

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
template <int MODE, bool FINAL = true>
__device__ __forceinline__ void load_keys(const PackArgs &a, const Side &sd, uint64_t base,
                                          uint32_t lane, KeyT<MODE> key[kFItems],
                                          uint32_t keep = 0xffffu) {
  constexpr bool hash = MODE >= 2;
#pragma unroll
  for (int it = 0; it < kFItems; it++) key[it] = hash ? kKeyHashSeed : 0;
  const uint32_t nk = mode_nkey<MODE>(a);
  for (uint32_t c = 0; c < nk; c++) {
    const uint32_t *p = sd.col[c];
    const uint32_t lo = a.lo[c], sh = a.shift[c];
    uint32_t v[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      v[it] = (j < sd.rows && (keep >> it & 1u)) ? __ldcs(p + j) : lo;
    }
#pragma unroll
    for (int it = 0; it < kFItems; it++)
      key[it] = MODE == 0 ? (KeyT<MODE>)(v[it] - lo)
                     : (KeyT<MODE>)(hash ? key_hash_step(key[it], v[it])
                                         : (key[it] | (uint64_t)(v[it] - lo) << sh));
  }
  if (hash && FINAL) {
#pragma unroll
    for (int it = 0; it < kFItems; it++) key[it] = (KeyT<MODE>)key_hash_final(key[it], a.kb);
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
__device__ __forceinline__ uint64_t ld_bm(const unsigned long long *p, uint64_t pol) {
#if MAPSQ_L2_HINT
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
#if MAPSQ_L2_HINT
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
template <bool TEST = true, bool HINT = true>
__device__ __forceinline__ void set_bits(uint32_t *bm, const uint32_t bidx[kFItems],
                                         uint32_t keep, uint32_t lane) {
  const uint64_t pol = HINT ? bm_policy() : 0;
  uint32_t word[kFItems];
#pragma unroll
  for (int it = 0; it < kFItems; it++)  // (read-only path: a stale word costs one more atomic)
    word[it] = (TEST && (keep >> it & 1u)) ? (HINT ? ld_bm32(bm + (bidx[it] >> 5), pol) : __ldg(bm + (bidx[it] >> 5))) : 0u;
#pragma unroll
  for (int it = 0; it < kFItems; it++) {
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

// Probe the side's rows against bm_probe: survivor bits -> mask[(slice0 + ws) * 16 ..], counts
// -> cnt[slice0 + ws]; with SET the survivors also set their bit in bm_set.
template <int MODE, bool SET>
__global__ void __launch_bounds__(kFThreads)
filter_probe_kernel(const PackArgs a, const Side sd, const uint32_t *__restrict__ bm_probe,
                    uint32_t *__restrict__ bm_set, uint32_t bbits, uint32_t hashed,
                    uint32_t *__restrict__ mask, uint32_t *__restrict__ cnt) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE>(a, sd, base, lane, key);
    uint32_t word[kFItems], bidx[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      bidx[it] = bit_index(key[it], bbits, hashed);
      word[it] = j < sd.rows ? ld_bm32(bm_probe + (bidx[it] >> 5), pol) : 0u;
    }
    uint32_t my = 0, c = 0, keep = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const bool k = word[it] >> (bidx[it] & 31) & 1u;
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      keep |= (uint32_t)k << it;
      if (lane == (uint32_t)it) my = bal;
      c += __popc(bal);
    }
    if (lane < (uint32_t)kFItems) mask[(sd.slice0 + ws) * kFItems + lane] = my;
    if (lane == 0) cnt[sd.slice0 + ws] = c;
    if (SET && c) set_bits<true, false>(bm_set, bidx, keep, lane);
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

// Warp-cooperative survivor addressing: lanes 0..15 hold the slice's 16 survivor-bit words
// (`my`, bit l of word it = row it * 32 + l survives).  slice_prefix returns each lane's
// exclusive prefix of the popcounts; survivor_row maps survivor r (< count) to its row in the
// slice, so a warp emits 32 survivors per step with consecutive (coalesced) stores.
__device__ __forceinline__ uint32_t slice_prefix(uint32_t my, uint32_t lane) {
  const uint32_t c = __popc(my);
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 16; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  return x - c;
}
__device__ __forceinline__ uint32_t survivor_row(uint32_t my, uint32_t pre, uint32_t r) {
  uint32_t it = 0;  // the item holding survivor r: the last q with pre_q <= r
#pragma unroll
  for (int q = 1; q < kFItems; q++) it += __shfl_sync(0xffffffffu, pre, q) <= r;
  uint32_t m = __shfl_sync(0xffffffffu, my, it);
  uint32_t k = r - __shfl_sync(0xffffffffu, pre, it), pos = 0;
#pragma unroll
  for (int sh = 16; sh > 0; sh >>= 1) {  // k-th set bit of m
    const uint32_t low = __popc(m & ((1u << sh) - 1u));
    if (k >= low) {
      k -= low;
      m >>= sh;
      pos += sh;
    }
  }
  return it * 32 + pos;
}

// Emit: the survivors of slice s go to words[off[s] ..] in row order (stable), as
// key' << ib | row id; digit 0 of the survivors is counted into hist.
template <int MODE>
__global__ void __launch_bounds__(kFThreads)
filter_emit_kernel(const PackArgs a, const Side sa, const Side sb,
                   const uint32_t *__restrict__ mask, const uint32_t *__restrict__ cnt,
                   const uint64_t *__restrict__ off, uint64_t *__restrict__ words,
                   uint32_t *__restrict__ hist) {
  __shared__ uint32_t s_h[kFCopies][kRadix];
  for (uint32_t i = threadIdx.x; i < kFCopies * kRadix; i += kFThreads) (&s_h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  uint32_t *h = s_h[(threadIdx.x >> 5) % kFCopies];
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  const uint64_t nslices = sb.slice0 + ceil_div(sb.rows, kFWarpRows);
  const uint32_t nk = mode_nkey<MODE>(a);
  for (uint64_t s = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5); s < nslices;
       s += nwarps) {
    if (__ldg(cnt + s) == 0) continue;  // warp-uniform
    const bool is_b = s >= sb.slice0;
    const Side &sd = is_b ? sb : sa;
    const uint64_t base = (s - sd.slice0) * kFWarpRows;
    const uint32_t my = lane < (uint32_t)kFItems ? __ldg(mask + s * kFItems + lane) : 0u;
    const uint32_t pre = slice_prefix(my, lane);
    const uint32_t c = __shfl_sync(0xffffffffu, pre + __popc(my), kFItems - 1);
    const uint64_t pos = __ldg(off + s);
    if (c > kDenseSlice) {  // dense slice: walk the 16 items (lanes = rows of the item)
      uint64_t p = pos;
#pragma unroll 4
      for (int it = 0; it < kFItems; it++) {
        const uint32_t bal = __shfl_sync(0xffffffffu, my, it);
        if (bal >> lane & 1u) {
          const uint64_t j = base + (uint64_t)it * 32 + lane;
          constexpr bool hash = MODE >= 2;
          uint64_t key = hash ? kKeyHashSeed : 0;
          for (uint32_t q = 0; q < nk; q++) {
            const uint32_t raw = __ldg(sd.col[q] + j), v = raw - a.lo[q];
            key = hash ? key_hash_step(key, raw) : (key | (MODE == 0 ? (uint64_t)v : (uint64_t)v << a.shift[q]));
          }
          if (hash) key = key_hash_final(key, a.kb);
          const uint64_t w = (key << a.ib) | (j + sd.id0);
          __stcs(words + p + __popc(bal & lt), w);
          if (a.passes) atomicAdd(h + ((uint32_t)(w >> a.bit_lo) & a.last_mask), 1u);
        }
        p += __popc(bal);
      }
      continue;
    }
    for (uint32_t r0 = 0; r0 < c; r0 += 32) {  // sparse slice: 32 survivors per step
      const uint32_t r = r0 + lane;
      const uint32_t row = survivor_row(my, pre, r < c ? r : 0);
      if (r < c) {
        const uint64_t j = base + row;
        constexpr bool hash = MODE >= 2;
        uint64_t key = hash ? kKeyHashSeed : 0;
        for (uint32_t q = 0; q < nk; q++) {
          const uint32_t raw = __ldg(sd.col[q] + j), v = raw - a.lo[q];
          key = hash ? key_hash_step(key, raw) : (key | (MODE == 0 ? (uint64_t)v : (uint64_t)v << a.shift[q]));
        }
        if (hash) key = key_hash_final(key, a.kb);
        const uint64_t w = (key << a.ib) | (j + sd.id0);
        __stcs(words + pos + r, w);
        if (a.passes) atomicAdd(h + ((uint32_t)(w >> a.bit_lo) & a.last_mask), 1u);
      }
    }
  }
  __syncthreads();
  if (a.passes)
    for (uint32_t d = threadIdx.x; d < kRadix; d += kFThreads) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < kFCopies; q++) c += s_h[q][d];
      if (c) atomicAdd(hist + d, c);
    }
}

// ---- refinement rounds on packed words (key' = w >> ib): words [0, split) are side A's,
// [split, n) side B's (the emit keeps the sides contiguous).  The bitmaps are blocked Bloom
// filters: a key sets/tests TWO bits of one 64-bit word (one memory access, like a plain bitmap,
// but ~2/3 of its false positives at C5's load factor), chosen by a mix of key' with a
// per-round seed, so a second round's false positives are independent of the first's.
struct WSide {
  const uint64_t *w;
  uint64_t rows, slice0;
};

__device__ __forceinline__ void wblock(uint64_t w, uint32_t ib, uint64_t seed, uint32_t bbits,
                                       uint32_t &idx, uint64_t &m) {
  const uint64_t h = ((w >> ib) ^ seed) * 0x9E3779B97F4A7C15ull;
  idx = (uint32_t)(h >> (70 - bbits));  // 2^(bbits - 6) 64-bit words
  const uint64_t g = h * 0xD6E8FEB86659FD93ull;
  m = (1ull << (g >> 58)) | (1ull << ((g >> 52) & 63));
}

// set (idx, m) for the rows whose keep bit is set (fire-and-forget RED.OR: keys mostly distinct);
// a lane whose left neighbour sets the same block bits skips
__device__ __forceinline__ void set_blocks(unsigned long long *bm, const uint32_t idx[kFItems],
                                           const uint64_t m[kFItems], uint32_t keep,
                                           uint32_t lane) {
  const uint64_t pol = bm_policy();
#pragma unroll
  for (int it = 0; it < kFItems; it++) {
    const uint32_t k = keep >> it & 1u;
    const uint32_t ip = __shfl_up_sync(0xffffffffu, idx[it], 1);
    const uint64_t mp = __shfl_up_sync(0xffffffffu, m[it], 1);
    const uint32_t kp = __shfl_up_sync(0xffffffffu, k, 1);
    const bool dup = lane > 0 && kp && ip == idx[it] && mp == m[it];
    if (k && !dup) red_or_bm(bm + idx[it], m[it], pol);
  }
}

__global__ void __launch_bounds__(kFThreads)
wfilter_build_kernel(const WSide sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                     unsigned long long *__restrict__ bm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    uint32_t idx[kFItems], keep = 0;
    uint64_t w[kFItems], m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      w[it] = j < sd.rows ? __ldcs(sd.w + j) : 0ull;
    }
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      wblock(w[it], ib, seed, bbits, idx[it], m[it]);
      keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < sd.rows) << it;
    }
    set_blocks(bm, idx, m, keep, lane);
  }
}

__global__ void __launch_bounds__(kFThreads)
wfilter_probe_kernel(const WSide sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                     const unsigned long long *__restrict__ bm_probe,
                     uint32_t *__restrict__ mask, uint32_t *__restrict__ cnt) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    uint64_t w[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      w[it] = j < sd.rows ? __ldcs(sd.w + j) : 0ull;
    }
    uint64_t v[kFItems], m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      uint32_t idx;
      wblock(w[it], ib, seed, bbits, idx, m[it]);
      v[it] = j < sd.rows ? ld_bm(bm_probe + idx, pol) : 0ull;
    }
    uint32_t my = 0, c = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const bool k = (v[it] & m[it]) == m[it] && base + (uint64_t)it * 32 + lane < sd.rows;
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      if (lane == (uint32_t)it) my = bal;
      c += __popc(bal);
    }
    if (lane < (uint32_t)kFItems) mask[(sd.slice0 + ws) * kFItems + lane] = my;
    if (lane == 0) cnt[sd.slice0 + ws] = c;
  }
}

// Set the survivors' block bits in bm (recorded in mask) — a separate pass after the probe, so
// only one bitmap is hot in L2 at a time (two 64 MB bitmaps overflow it): C5's (?x, ?z) join
// 5.7 -> 4.7 ms over its three rounds.
__global__ void __launch_bounds__(kFThreads)
wfilter_setmask_kernel(const WSide sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                       const uint32_t *__restrict__ mask, const uint32_t *__restrict__ cnt,
                       unsigned long long *__restrict__ bm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    if (__ldg(cnt + sd.slice0 + ws) == 0) continue;  // warp-uniform
    const uint32_t my = lane < (uint32_t)kFItems ? __ldg(mask + (sd.slice0 + ws) * kFItems + lane) : 0u;
    uint32_t keep = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) keep |= (__shfl_sync(0xffffffffu, my, it) >> lane & 1u) << it;
    const uint64_t base = ws * kFWarpRows;
    uint32_t idx[kFItems];
    uint64_t m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t w = (keep >> it & 1u) ? __ldcs(sd.w + base + (uint64_t)it * 32 + lane) : 0ull;
      wblock(w, ib, seed, bbits, idx[it], m[it]);
    }
    set_blocks(bm, idx, m, keep, lane);
  }
}

__global__ void __launch_bounds__(kFThreads)
wfilter_sample_kernel(const WSide sd, uint32_t ib, uint64_t seed, uint32_t bbits,
                      const unsigned long long *__restrict__ bm, uint32_t stride,
                      unsigned long long *__restrict__ sample) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  uint32_t c = 0, rows = 0;
  for (uint64_t ws = ((uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5)) * stride;
       ws * kFWarpRows < sd.rows; ws += nwarps * stride) {
    const uint64_t base = ws * kFWarpRows;
    uint64_t w[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      w[it] = j < sd.rows ? __ldcs(sd.w + j) : 0ull;
    }
    uint64_t v[kFItems], m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {  // all probes in flight together
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      uint32_t idx;
      wblock(w[it], ib, seed, bbits, idx, m[it]);
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

// ---- hashed composite keys, first round on the key columns (no word is written for a dropped
// row): the word rounds' blocked Bloom bitmaps and pass structure, with key' = key_hash of the
// row's shared columns computed from the columns (load_keys<MODE>, MODE 2/3).
// the column round's block index and bit pair straight from the 64-bit key_hash chain value
// (already mixed: no further multiply)
__device__ __forceinline__ void cblock(uint64_t h, uint32_t bbits, uint32_t &idx, uint64_t &m) {
  idx = (uint32_t)(h >> (70 - bbits));
  m = (1ull << (h & 63)) | (1ull << ((h >> 6) & 63));
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
cfilter_build_kernel(const PackArgs a, const Side sd, uint64_t seed, uint32_t bbits,
                     unsigned long long *__restrict__ bm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE, false>(a, sd, base, lane, key);
    uint32_t idx[kFItems], keep = 0;
    uint64_t m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      cblock(key[it], bbits, idx[it], m[it]);
      keep |= (uint32_t)(base + (uint64_t)it * 32 + lane < sd.rows) << it;
    }
    set_blocks(bm, idx, m, keep, lane);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
cfilter_probe_kernel(const PackArgs a, const Side sd, uint64_t seed, uint32_t bbits,
                     const unsigned long long *__restrict__ bm_probe,
                     uint32_t *__restrict__ mask, uint32_t *__restrict__ cnt) {
  const uint64_t pol = bm_policy();
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE, false>(a, sd, base, lane, key);
    uint64_t v[kFItems], m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const uint64_t j = base + (uint64_t)it * 32 + lane;
      uint32_t idx;
      cblock(key[it], bbits, idx, m[it]);
      v[it] = j < sd.rows ? ld_bm(bm_probe + idx, pol) : 0ull;
    }
    uint32_t my = 0, c = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) {
      const bool k = (v[it] & m[it]) == m[it] && base + (uint64_t)it * 32 + lane < sd.rows;
      const uint32_t bal = __ballot_sync(0xffffffffu, k);
      if (lane == (uint32_t)it) my = bal;
      c += __popc(bal);
    }
    if (lane < (uint32_t)kFItems) mask[(sd.slice0 + ws) * kFItems + lane] = my;
    if (lane == 0) cnt[sd.slice0 + ws] = c;
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
cfilter_setmask_kernel(const PackArgs a, const Side sd, uint64_t seed, uint32_t bbits,
                       const uint32_t *__restrict__ mask, const uint32_t *__restrict__ cnt,
                       unsigned long long *__restrict__ bm) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  for (uint64_t ws = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5);
       ws * kFWarpRows < sd.rows; ws += nwarps) {
    if (__ldg(cnt + sd.slice0 + ws) == 0) continue;  // warp-uniform
    const uint32_t my = lane < (uint32_t)kFItems ? __ldg(mask + (sd.slice0 + ws) * kFItems + lane) : 0u;
    uint32_t keep = 0;
#pragma unroll
    for (int it = 0; it < kFItems; it++) keep |= (__shfl_sync(0xffffffffu, my, it) >> lane & 1u) << it;
    const uint64_t base = ws * kFWarpRows;
    KeyT<MODE> key[kFItems];
    load_keys<MODE, false>(a, sd, base, lane, key, keep);
    uint32_t idx[kFItems];
    uint64_t m[kFItems];
#pragma unroll
    for (int it = 0; it < kFItems; it++) cblock(key[it], bbits, idx[it], m[it]);
    set_blocks(bm, idx, m, keep, lane);
  }
}

template <int MODE>
__global__ void __launch_bounds__(kFThreads)
cfilter_sample_kernel(const PackArgs a, const Side sd, uint64_t seed, uint32_t bbits,
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

template <int MODE>
void cfilter_passes(const PackArgs &a, const Side &S, const Side &L, unsigned long long *bmS,
                    unsigned long long *bmL, uint32_t bbits, uint64_t seed, uint32_t *mask,
                    uint32_t *cnt, int phase, unsigned long long *sample, cudaStream_t s);

__global__ void __launch_bounds__(kFThreads)
wfilter_emit_kernel(const WSide sa, const WSide sb, const uint32_t *__restrict__ mask,
                    const uint32_t *__restrict__ cnt, const uint64_t *__restrict__ off,
                    uint64_t *__restrict__ out, uint32_t *__restrict__ hist, uint32_t bit_lo,
                    uint32_t dmask) {
  __shared__ uint32_t s_h[kFCopies][kRadix];
  for (uint32_t i = threadIdx.x; i < kFCopies * kRadix; i += kFThreads) (&s_h[0][0])[i] = 0;
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31, lt = lanemask_lt();
  uint32_t *h = s_h[(threadIdx.x >> 5) % kFCopies];
  const uint64_t nwarps = (uint64_t)gridDim.x * kFWarps;
  const uint64_t nslices = sb.slice0 + ceil_div(sb.rows, kFWarpRows);
  for (uint64_t s = (uint64_t)blockIdx.x * kFWarps + (threadIdx.x >> 5); s < nslices;
       s += nwarps) {
    if (__ldg(cnt + s) == 0) continue;  // warp-uniform
    const WSide &sd = s >= sb.slice0 ? sb : sa;
    const uint64_t base = (s - sd.slice0) * kFWarpRows;
    const uint32_t my = lane < (uint32_t)kFItems ? __ldg(mask + s * kFItems + lane) : 0u;
    const uint32_t pre = slice_prefix(my, lane);
    const uint32_t c = __shfl_sync(0xffffffffu, pre + __popc(my), kFItems - 1);
    const uint64_t pos = __ldg(off + s);
    if (c > kDenseSlice) {  // dense slice: walk the 16 items (lanes = rows of the item)
      uint64_t p = pos;
#pragma unroll 4
      for (int it = 0; it < kFItems; it++) {
        const uint32_t bal = __shfl_sync(0xffffffffu, my, it);
        if (bal >> lane & 1u) {
          const uint64_t w = __ldg(sd.w + base + (uint64_t)it * 32 + lane);
          __stcs(out + p + __popc(bal & lt), w);
          if (hist) atomicAdd(h + ((uint32_t)(w >> bit_lo) & dmask), 1u);
        }
        p += __popc(bal);
      }
      continue;
    }
    for (uint32_t r0 = 0; r0 < c; r0 += 32) {  // sparse slice: 32 survivors per step
      const uint32_t r = r0 + lane;
      const uint32_t row = survivor_row(my, pre, r < c ? r : 0);
      if (r < c) {
        const uint64_t w = __ldg(sd.w + base + row);
        __stcs(out + pos + r, w);
        if (hist) atomicAdd(h + ((uint32_t)(w >> bit_lo) & dmask), 1u);
      }
    }
  }
  __syncthreads();
  if (hist)
    for (uint32_t d = threadIdx.x; d < kRadix; d += kFThreads) {
      uint32_t c = 0;
#pragma unroll
      for (int q = 0; q < kFCopies; q++) c += s_h[q][d];
      if (c) atomicAdd(hist + d, c);
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

int sample_grid(uint64_t rows) {  // one warp per sampled slice (up to 148 x 8 CTAs)
  const uint64_t sampled = ceil_div(ceil_div(rows, kFWarpRows), kSampleStride);
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

template <int MODE>
void filter_passes(const PackArgs &a, const Side &S, const Side &L, uint32_t *bmS, uint32_t *bmL,
                   uint32_t bbits, uint32_t hashed, uint32_t *mask, uint32_t *cnt, int phase,
                   unsigned long long *sample, cudaStream_t s) {
  const int gs = grid_for_rows(S.rows), gl = grid_for_rows(L.rows);
  if (phase == 0) {  // build S, sample L
    filter_build_kernel<MODE><<<gs, kFThreads, 0, s>>>(a, S, bmS, bbits, hashed);
    filter_sample_kernel<MODE><<<sample_grid(L.rows), kFThreads, 0, s>>>(
        a, L, bmS, bbits, hashed, kSampleStride, sample);
    return;
  }
  filter_probe_kernel<MODE, true><<<gl, kFThreads, 0, s>>>(a, L, bmS, bmL, bbits, hashed, mask,
                                                           cnt);
  filter_probe_kernel<MODE, false><<<gs, kFThreads, 0, s>>>(a, S, bmL, nullptr, bbits, hashed,
                                                            mask, cnt);
}

template <int MODE>
void cfilter_passes(const PackArgs &a, const Side &S, const Side &L, unsigned long long *bmS,
                    unsigned long long *bmL, uint32_t bbits, uint64_t seed, uint32_t *mask,
                    uint32_t *cnt, int phase, unsigned long long *sample, cudaStream_t s) {
  const int gs = grid_for_rows(S.rows), gl = grid_for_rows(L.rows);
  if (phase == 0) {  // build S, sample L
    cfilter_build_kernel<MODE><<<gs, kFThreads, 0, s>>>(a, S, seed, bbits, bmS);
    cfilter_sample_kernel<MODE><<<sample_grid(L.rows), kFThreads, 0, s>>>(
        a, L, seed, bbits, bmS, kSampleStride, sample);
    return;
  }
  cfilter_probe_kernel<MODE><<<gl, kFThreads, 0, s>>>(a, L, seed, bbits, bmS, mask, cnt);
  cfilter_setmask_kernel<MODE><<<gl, kFThreads, 0, s>>>(a, L, seed, bbits, mask, cnt, bmL);
  cfilter_probe_kernel<MODE><<<gs, kFThreads, 0, s>>>(a, S, seed, bbits, bmL, mask, cnt);
}

}  // namespace

uint64_t filter_slices(uint64_t n1, uint64_t n2) {
  return ceil_div(n1, kFWarpRows) + ceil_div(n2, kFWarpRows);
}
uint64_t filter_mask_words(uint64_t n1, uint64_t n2) { return filter_slices(n1, n2) * kFItems; }

void launch_filter(const PackArgs &a, uint32_t *bmS, uint32_t *bmL, uint32_t bbits,
                   uint32_t hashed, uint32_t *mask, uint32_t *cnt, int phase,
                   unsigned long long *sample, cudaStream_t s) {
  const bool b_small = a.n2 < a.n1;
  const Side S = side_of(a, b_small), L = side_of(a, !b_small);
  switch (filter_mode(a)) {
    case 0: filter_passes<0>(a, S, L, bmS, bmL, bbits, hashed, mask, cnt, phase, sample, s); break;
    case 1: filter_passes<1>(a, S, L, bmS, bmL, bbits, hashed, mask, cnt, phase, sample, s); break;
    case 2: filter_passes<2>(a, S, L, bmS, bmL, bbits, hashed, mask, cnt, phase, sample, s); break;
    default: filter_passes<3>(a, S, L, bmS, bmL, bbits, hashed, mask, cnt, phase, sample, s); break;
  }
}

void launch_cfilter(const PackArgs &a, uint32_t *bmS32, uint32_t *bmL32, uint32_t bbits,
                    uint64_t seed, uint32_t *mask, uint32_t *cnt, int phase,
                    unsigned long long *sample, cudaStream_t s) {
  unsigned long long *bmS = reinterpret_cast<unsigned long long *>(bmS32);
  unsigned long long *bmL = reinterpret_cast<unsigned long long *>(bmL32);
  const bool b_small = a.n2 < a.n1;
  const Side S = side_of(a, b_small), L = side_of(a, !b_small);
  if (a.nkey == 2)
    cfilter_passes<2>(a, S, L, bmS, bmL, bbits, seed, mask, cnt, phase, sample, s);
  else
    cfilter_passes<3>(a, S, L, bmS, bmL, bbits, seed, mask, cnt, phase, sample, s);
}

void launch_wfilter(const uint64_t *words, uint64_t n, uint64_t split, uint32_t ib,
                    uint64_t seed, uint32_t bbits, uint32_t *bmS32, uint32_t *bmL32,
                    uint32_t *mask, uint32_t *cnt, int phase, unsigned long long *sample,
                    cudaStream_t s) {
  unsigned long long *bmS = reinterpret_cast<unsigned long long *>(bmS32);
  unsigned long long *bmL = reinterpret_cast<unsigned long long *>(bmL32);
  const WSide A{words, split, 0}, B{words + split, n - split, ceil_div(split, kFWarpRows)};
  const bool b_small = B.rows < A.rows;
  const WSide S = b_small ? B : A, L = b_small ? A : B;
  const int gs = grid_for_rows(S.rows), gl = grid_for_rows(L.rows);
  if (phase != 1) {  // build S (and, phase 0, sample L)
    if (S.rows) wfilter_build_kernel<<<gs, kFThreads, 0, s>>>(S, ib, seed, bbits, bmS);
    if (phase == 0) {
      if (L.rows)
        wfilter_sample_kernel<<<sample_grid(L.rows), kFThreads, 0, s>>>(
            L, ib, seed, bbits, bmS, kSampleStride, sample);
      return;
    }
  }
  if (L.rows) {
    wfilter_probe_kernel<<<gl, kFThreads, 0, s>>>(L, ib, seed, bbits, bmS, mask, cnt);
    wfilter_setmask_kernel<<<gl, kFThreads, 0, s>>>(L, ib, seed, bbits, mask, cnt, bmL);
  }
  if (S.rows) wfilter_probe_kernel<<<gs, kFThreads, 0, s>>>(S, ib, seed, bbits, bmL, mask, cnt);
}

void launch_wfilter_emit(const uint64_t *words, uint64_t n, uint64_t split, const uint32_t *mask,
                         const uint32_t *cnt, const uint64_t *off, uint64_t *out, uint32_t *hist,
                         uint32_t bit_lo, uint32_t dmask, cudaStream_t s) {
  const WSide A{words, split, 0}, B{words + split, n - split, ceil_div(split, kFWarpRows)};
  wfilter_emit_kernel<<<grid_for_rows(n), kFThreads, 0, s>>>(A, B, mask, cnt, off, out, hist,
                                                            bit_lo, dmask);
}

void launch_filter_emit(const PackArgs &a, const uint32_t *mask, const uint32_t *cnt,
                        const uint64_t *off, uint64_t *words, uint32_t *hist, cudaStream_t s) {
  const Side A = side_of(a, false), B = side_of(a, true);
  const int g = grid_for_rows(a.n1 + a.n2);
  switch (filter_mode(a)) {
    case 0: filter_emit_kernel<0><<<g, kFThreads, 0, s>>>(a, A, B, mask, cnt, off, words, hist); break;
    case 1: filter_emit_kernel<1><<<g, kFThreads, 0, s>>>(a, A, B, mask, cnt, off, words, hist); break;
    case 2: filter_emit_kernel<2><<<g, kFThreads, 0, s>>>(a, A, B, mask, cnt, off, words, hist); break;
    default: filter_emit_kernel<3><<<g, kFThreads, 0, s>>>(a, A, B, mask, cnt, off, words, hist); break;
  }
}

}  // namespace mapsq
