// radix.cu — K2 (Map: key-label packing + upfront digit histograms) and K3 (Sort: one-sweep
// LSD radix digit pass with decoupled look-back), SURVEY §8 rows a3-a4.
//
// Map (Alg. 1 l.1-4, "split and emit intermediate"): each row of Tp1 becomes
// the word key'<<ib | r (label LEFT) and each row of Tp2 the word key'<<ib | (n1 + r) (label
// RIGHT): the label is the bit "rowid >= n1" (reading R1: LEFT = Tp1).
// Sort (Alg. 1 l.5, "sort intermediates"): a stable LSD radix sort over only the kb
// key bits.  Because the low ib bits already hold (label, rowid) in ascending order, stability
// yields the total order (key', LEFT before RIGHT, rowid) — the sorted array is unique.
//
// The digit pass is a one-sweep design: tiles are claimed in order through an atomic counter,
// ranked by a warp multisplit (peer lanes from shared-memory atomicOr masks), and their global
// digit offsets are resolved by decoupled look-back over per-(tile, digit) status words; each
// pass's global digit counts come from the previous kernel (the Map kernel counts digit 0,
// every pass counts the next digit).
#include <type_traits>

#include "internal.cuh"

namespace mapsq {
namespace {

#ifndef MAPSQ_RADIX_ITEMS
#define MAPSQ_RADIX_ITEMS 24
#endif
#ifndef MAPSQ_RADIX_MINB
#define MAPSQ_RADIX_MINB 3
#endif
#ifndef MAPSQ_RADIX_WIN
#define MAPSQ_RADIX_WIN 4  // look-back window of the P64 digit pass (predecessors read at once)
#endif
constexpr int kWarps = kSortThreads / 32;
constexpr int kLookWin = 8;
constexpr int kHistThreads = 256;
constexpr int kHistItems = 16;

constexpr int kHistCopies = 4;

// Upfront histograms of every pass (onesweep), one shared atomic per pass per element into one
// of kHistCopies private copies (warps w and w+4 share a copy).
template <bool KV>
__global__ void __launch_bounds__(kHistThreads)
pack_hist_kernel(const PackArgs a, uint64_t *__restrict__ words, uint32_t *__restrict__ vals,
                 uint32_t *__restrict__ hist) {
  extern __shared__ uint32_t s_hcopy[];  // [kHistCopies][passes * 256]
  const uint32_t plen = a.passes * kRadix;
  for (uint32_t i = threadIdx.x; i < kHistCopies * plen; i += kHistThreads) s_hcopy[i] = 0;
  __syncthreads();
  uint32_t *h = s_hcopy + ((threadIdx.x >> 5) % kHistCopies) * plen;
  const uint64_t n = a.n1 + a.n2;
  const uint64_t chunk = (uint64_t)kHistThreads * kHistItems;
  for (uint64_t c0 = (uint64_t)blockIdx.x * chunk; c0 < n; c0 += (uint64_t)gridDim.x * chunk) {
    // key columns outermost, items innermost: all kHistItems loads of a column are in flight
    // together (a per-item column loop serialized them on load latency)
    uint64_t key[kHistItems];
#pragma unroll
    for (int it = 0; it < kHistItems; it++) key[it] = a.hash ? kKeyHashSeed : 0;
    for (uint32_t c = 0; c < a.nkey; c++) {
      const uint32_t *k1 = a.key1[c], *k2 = a.key2[c] - a.n1;
      const uint32_t lo = a.lo[c], sh = a.shift[c];
      uint32_t v[kHistItems];
#pragma unroll
      for (int it = 0; it < kHistItems; it++) {
        const uint64_t i = c0 + (uint64_t)it * kHistThreads + threadIdx.x;
        v[it] = i < n ? __ldcs((i < a.n1 ? k1 : k2) + i) : lo;
      }
      if (a.hash) {
#pragma unroll
        for (int it = 0; it < kHistItems; it++) key[it] = key_hash_step(key[it], v[it]);
      } else {
#pragma unroll
        for (int it = 0; it < kHistItems; it++) key[it] |= (uint64_t)(v[it] - lo) << sh;
      }
    }
    if (a.hash) {
#pragma unroll
      for (int it = 0; it < kHistItems; it++) key[it] = key_hash_final(key[it], a.kb);
    }
#pragma unroll
    for (int it = 0; it < kHistItems; it++) {
      const uint64_t i = c0 + (uint64_t)it * kHistThreads + threadIdx.x;
      if (i >= n) continue;
      uint64_t kk = key[it];
      if (KV) {
        __stcs(words + i, kk);
        __stcs(vals + i, (uint32_t)i);
      } else {
        kk = (kk << a.ib) | i;
        __stcs(words + i, kk);
      }
      for (uint32_t p = 0; p < a.passes; p++) {
        const uint32_t d = (uint32_t)(kk >> (a.bit_lo + 8 * p)) & (p + 1 == a.passes ? a.last_mask : 0xffu);
        atomicAdd(h + p * kRadix + d, 1u);
      }
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < plen; i += kHistThreads) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kHistCopies; q++) c += s_hcopy[q * plen + i];
    if (c) atomicAdd(hist + i, c);
  }
}

__global__ void __launch_bounds__(kHistThreads)
key_hist_kernel(const uint64_t *__restrict__ keys, uint64_t n, uint32_t bit_lo, uint32_t passes,
                uint32_t last_mask, uint32_t *__restrict__ hist) {
  __shared__ uint32_t s_hist[kHistCopies][kMaxPasses * kRadix];
  for (int i = threadIdx.x; i < kHistCopies * kMaxPasses * kRadix; i += kHistThreads)
    (&s_hist[0][0])[i] = 0;
  __syncthreads();
  uint32_t *h = s_hist[(threadIdx.x >> 5) % kHistCopies];
  const uint64_t stride = (uint64_t)gridDim.x * kHistThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kHistThreads + threadIdx.x; i < n; i += stride) {
    const uint64_t key = __ldcs(keys + i);
    for (uint32_t p = 0; p < passes; p++) {
      const uint32_t d = (uint32_t)(key >> (bit_lo + 8 * p)) & (p + 1 == passes ? last_mask : 0xffu);
      atomicAdd(h + p * kRadix + d, 1u);
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < (int)passes * kRadix; i += kHistThreads) {
    uint32_t c = 0;
#pragma unroll
    for (int q = 0; q < kHistCopies; q++) c += s_hist[q][i];
    if (c) atomicAdd(hist + i, c);
  }
}

// One stable digit pass.  Tile = kSortThreads x ITEMS keys; warp w owns the contiguous
// slice [w*32*ITEMS, (w+1)*32*ITEMS) of its tile and reads it item-major (item it, lane l ->
// slice[it*32 + l]) so every load is a coalesced 256 B row.  Intra-tile indices are 32-bit and
// full tiles skip every bounds check (the first version spent most of its issue slots on 64-bit
// index arithmetic).
// RANK: how a warp finds the lanes holding the same digit — 0 = match.any, 1 = one ballot per
// digit bit, 2 = shared-memory atomicOr of lane bits into per-digit masks (the key smem is still
// unused during ranking), 3 = as 2 with a warp-uniform-digit shortcut (two redux.sync),
// 4.. = as 2 after RANK-2 leader rounds of shfl + ballot.
template <bool KV, int ITEMS = kSortItems, int WIN = kLookWin, int MINB = 3, bool RELOAD = false,
          int RANK = 0, bool SEG = false>
__global__ void __launch_bounds__(kSortThreads, MINB)
radix_pass_kernel(const uint64_t *__restrict__ kin, uint64_t *__restrict__ kout,
                  const uint32_t *__restrict__ vin, uint32_t *__restrict__ vout, uint64_t n,
                  uint32_t shift, uint32_t bits, const uint32_t *__restrict__ hist_pass,
                  uint64_t *__restrict__ status, uint32_t *__restrict__ tile_counter,
                  uint32_t *__restrict__ hist_next, uint32_t next_shift, uint32_t next_mask,
                  uint64_t n0, uint64_t gap) {
  constexpr int TILE = kSortThreads * ITEMS;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem_raw);
  uint32_t *s_vals = reinterpret_cast<uint32_t *>(smem_raw + TILE * sizeof(uint64_t));
  __shared__ uint32_t s_warp_hist[kWarps][kRadix];
  __shared__ uint32_t s_digit_start[kRadix];
  __shared__ uint64_t s_global_base[kRadix];
  __shared__ uint32_t s_wsum[kWarps];
  __shared__ uint32_t s_tile;
  __shared__ uint32_t s_next[kRadix];

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
#pragma unroll
  for (int q = 0; q < kWarps; q++) s_warp_hist[q][tid] = 0;  // kSortThreads == kRadix
  s_next[tid] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tile_base = tile * TILE;
  const uint64_t rem = n - tile_base;
  const uint32_t tile_n = rem < (uint64_t)TILE ? (uint32_t)rem : (uint32_t)TILE;
  const uint32_t wslice = warp * 32 * ITEMS;
  const uint32_t dmask = (1u << bits) - 1u;
  // two-segment input (the semi-join filter's output): key i >= n0 is read at kin[i + gap]; a
  // warp slice lies wholly in one segment except at the seam, where items pick their segment
  const uint64_t g0 = tile_base + wslice;
  const uint64_t *src = kin + g0 + lane + ((SEG && g0 >= n0) ? gap : 0);
  const bool seam = SEG && g0 < n0 && g0 + 32 * ITEMS > n0;
  auto ld_src = [&](int it) -> const uint64_t * {
    if (!SEG || !seam) return src + it * 32;
    const uint64_t g = g0 + it * 32 + lane;
    return kin + g + (g >= n0 ? gap : 0);
  };

  uint64_t k[ITEMS];
  uint32_t v[KV ? ITEMS : 1];
  uint32_t r[ITEMS];
  const bool full = tile_n == (uint32_t)TILE;
  if (full) {
#pragma unroll
    for (int it = 0; it < ITEMS; it++) k[it] = RELOAD ? __ldcg(ld_src(it)) : __ldcs(ld_src(it));
    if (KV) {
#pragma unroll
      for (int it = 0; it < ITEMS; it++) v[KV ? it : 0] = __ldcs(vin + tile_base + wslice + lane + it * 32);
    }
  } else {
#pragma unroll
    for (int it = 0; it < ITEMS; it++) {
      const bool in = wslice + it * 32 + lane < tile_n;
      k[it] = in ? (RELOAD ? __ldcg(ld_src(it)) : __ldcs(ld_src(it))) : 0ull;
      if (KV) v[KV ? it : 0] = in ? __ldcs(vin + tile_base + wslice + lane + it * 32) : 0u;
    }
  }
  // warp-level multisplit in batches of kMB items: the batch's match-any operations are issued
  // together (their latency overlaps), then one leader lane per digit group bumps the warp's
  // counter; batching keeps only kMB match masks live.
  constexpr int kMB = 8;
  const uint32_t lt = lanemask_lt();
  // RANK 2/3: per-warp [kMB][256] lane masks in the (not yet used) key staging area
  constexpr int kPB = (RANK >= 2) ? ((TILE * 8 / (kWarps * kRadix * 4)) < kMB ? (TILE * 8 / (kWarps * kRadix * 4)) : kMB) : 1;
  uint32_t *s_pm = reinterpret_cast<uint32_t *>(smem_raw) + warp * kPB * kRadix;
  if (RANK >= 2) {
    uint4 *z = reinterpret_cast<uint4 *>(s_pm);
#pragma unroll
    for (int i = lane; i < kPB * kRadix / 4; i += 32) z[i] = make_uint4(0, 0, 0, 0);
    __syncwarp();
  }
  constexpr int kB = RANK >= 2 ? kPB : kMB;
#pragma unroll
  for (int b0 = 0; b0 < ITEMS; b0 += kB) {
    uint32_t peers[kB];
#pragma unroll
    for (int u = 0; u < kB && b0 + u < ITEMS; u++) {
      const int it = b0 + u;
      const bool in = full || wslice + it * 32 + lane < tile_n;
      const uint32_t dg = (uint32_t)(k[it] >> shift) & dmask;
      if (RANK == 1) {  // peers from one ballot per digit bit (short-latency votes)
        uint32_t pm = __ballot_sync(0xffffffffu, in);
        pm = in ? pm : ~pm;
#pragma unroll
        for (int b = 0; b < 8; b++) {
          const uint32_t bb = __ballot_sync(0xffffffffu, (dg >> b) & 1u);
          pm &= ((dg >> b) & 1u) ? bb : ~bb;
        }
        peers[u] = pm;
      } else if (RANK >= 2) {
        peers[u] = 0;
        const uint32_t key = in ? dg : 0x100u;
        if (RANK == 3) {
          if (__reduce_min_sync(0xffffffffu, key) == __reduce_max_sync(0xffffffffu, key))
            peers[u] = 0xffffffffu;
        } else if (RANK >= 4) {
          // up to RANK-2 leader rounds (shfl + ballot) catch the few-distinct-digit warps of
          // clustered data; lanes still unmatched fall back to the atomicOr masks
          uint32_t rem = 0xffffffffu;
#pragma unroll
          for (int q = 0; q < RANK - 2; q++) {
            if (rem == 0) break;
            const uint32_t dq = __shfl_sync(0xffffffffu, key, __ffs(rem) - 1);
            const uint32_t bq = __ballot_sync(0xffffffffu, key == dq);
            if (key == dq) peers[u] = bq;
            rem &= ~bq;
          }
        }
        if (in && peers[u] == 0) atomicOr(s_pm + u * kRadix + dg, 1u << lane);
      } else {
        peers[u] = __match_any_sync(0xffffffffu, in ? dg : 0x100u);
      }
    }
    if (RANK >= 2) {
      __syncwarp();
#pragma unroll
      for (int u = 0; u < kB && b0 + u < ITEMS; u++) {
        const uint32_t dg = (uint32_t)(k[b0 + u] >> shift) & dmask;
        if (peers[u] == 0) peers[u] = s_pm[u * kRadix + dg];
      }
      __syncwarp();
    }
#pragma unroll
    for (int u = 0; u < kB && b0 + u < ITEMS; u++) {
      const int it = b0 + u;
      const uint32_t d = (uint32_t)(k[it] >> shift) & dmask;
      const uint32_t leader = 31 - __clz(peers[u]);
      const bool in = full || wslice + it * 32 + lane < tile_n;
      uint32_t base = 0;
      if (in && lane == leader) {
        base = s_warp_hist[warp][d];
        s_warp_hist[warp][d] = base + __popc(peers[u]);
        if (RANK >= 2) s_pm[u * kRadix + d] = 0;
      }
      r[it] = __shfl_sync(0xffffffffu, base, leader) + __popc(peers[u] & lt);
      // the NEXT pass's digit histogram, from the keys already in registers (one shared atomic
      // per key; these issue slots are otherwise idle while the tile waits on its look-back)
      if (hist_next && in) atomicAdd(&s_next[(uint32_t)(k[it] >> next_shift) & next_mask], 1u);
    }
    if (RANK >= 2) __syncwarp();
  }
  __syncthreads();

  // thread d: exclusive prefix of digit d across warps, tile total, look-back
  const uint32_t d = tid;
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < kWarps; w++) {
    const uint32_t c = s_warp_hist[w][d];
    s_warp_hist[w][d] = total;
    total += c;
  }
  uint64_t *my_status = status + tile * kRadix + d;
  uint64_t excl = 0;
  if (tile == 0) {
    st_relaxed_u64(my_status, kFlagInc | total);
  } else {
    st_relaxed_u64(my_status, kFlagAgg | total);
    // Windowed look-back: WIN predecessors are read at once (independent loads).
    int64_t t0 = (int64_t)tile - 1;
    while (true) {
      uint64_t sv[WIN];
#pragma unroll
      for (int w = 0; w < WIN; w++) {
        const int64_t t = t0 - w;
        sv[w] = t >= 0 ? ld_relaxed_u64(status + (uint64_t)t * kRadix + d) : kFlagInc;
      }
      int consumed = 0;
      bool done = false;
#pragma unroll
      for (int w = 0; w < WIN; w++) {
        if (consumed != w || done) continue;
        const uint64_t flag = sv[w] & ~kValMask;
        if (flag == 0) continue;  // not published yet: stop consuming here
        excl += sv[w] & kValMask;
        consumed = w + 1;
        if (flag == kFlagInc) done = true;
      }
      if (done) break;
      t0 -= consumed;
      if (consumed < WIN) __nanosleep(32);
    }
    st_relaxed_u64(my_status, kFlagInc | (excl + total));
  }
  // tile-local start of each digit: exclusive block scan of `total` over digits
  uint32_t x = total;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t pre = 0;
#pragma unroll
  for (int w = 0; w < kWarps; w++)
    if ((uint32_t)w < warp) pre += s_wsum[w];
  const uint32_t dstart = pre + x - total;
  s_digit_start[d] = dstart;
  // exclusive scan of this pass's global digit counts (each CTA scans the 256 totals itself)
  const uint32_t hc = __ldg(hist_pass + d);
  uint32_t hx = hc;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, hx, o);
    if (lane >= (uint32_t)o) hx += y;
  }
  __syncthreads();  // s_wsum reuse
  if (lane == 31) s_wsum[warp] = hx;
  __syncthreads();
  uint32_t hpre = 0;
#pragma unroll
  for (int w = 0; w < kWarps; w++)
    if ((uint32_t)w < warp) hpre += s_wsum[w];
  s_global_base[d] = (uint64_t)(hpre + hx - hc) + excl - dstart;
  if (hist_next && s_next[d]) atomicAdd(hist_next + d, s_next[d]);
  __syncthreads();

  // place keys at their tile-local sorted slot
#pragma unroll
  for (int it = 0; it < ITEMS; it++) {
    if (wslice + it * 32 + lane < tile_n) {
      // RELOAD: the key is read again (an L2 hit) instead of being held in registers across the
      // look-back, which lets more CTAs share an SM
      const uint64_t key = RELOAD ? __ldcs(ld_src(it)) : k[it];
      const uint32_t dd = (uint32_t)(key >> shift) & dmask;
      const uint32_t slot = s_digit_start[dd] + s_warp_hist[warp][dd] + r[it];
      s_keys[slot] = key;
      if (KV) s_vals[slot] = v[KV ? it : 0];
    }
  }
  __syncthreads();
  // coalesced write-out: consecutive slots of one digit go to consecutive global positions
#pragma unroll 4
  for (uint32_t i = tid; i < tile_n; i += kSortThreads) {
    const uint64_t key = s_keys[i];
    const uint32_t dd = (uint32_t)(key >> shift) & dmask;
    const uint64_t pos = s_global_base[dd] + i;
    __stcs(kout + pos, key);
    if (KV) __stcs(vout + pos, s_vals[i]);
  }
}

}  // namespace

static int grid_for(uint64_t n, int per_block) {
  const uint64_t b = ceil_div(n, per_block);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(b, 148 * 8));
}

void launch_pack_hist(const PackArgs &a, uint64_t *words, uint32_t *vals, uint32_t *hist,
                      cudaStream_t s) {
  const uint64_t n = a.n1 + a.n2;
  const int g = grid_for(n, kHistThreads * kHistItems);
  const size_t smem = kHistCopies * std::max<uint32_t>(a.passes, 1) * kRadix * sizeof(uint32_t);
  set_smem_limit((const void *)pack_hist_kernel<true>, 65536);
  set_smem_limit((const void *)pack_hist_kernel<false>, 65536);
  if (a.kv)
    pack_hist_kernel<true><<<g, kHistThreads, smem, s>>>(a, words, vals, hist);
  else
    pack_hist_kernel<false><<<g, kHistThreads, smem, s>>>(a, words, vals, hist);
}

void launch_key_hist(const uint64_t *keys, uint64_t n, uint32_t bit_lo, uint32_t passes,
                     uint32_t last_bits, uint32_t *hist, cudaStream_t s) {
  const int g = grid_for(n, kHistThreads * kHistItems);
  key_hist_kernel<<<g, kHistThreads, 0, s>>>(keys, n, bit_lo, passes, (1u << last_bits) - 1u, hist);
}

void launch_radix_pass(const uint64_t *kin, uint64_t *kout, const uint32_t *vin, uint32_t *vout,
                       uint64_t n, uint32_t shift, uint32_t bits, const uint32_t *hist_pass,
                       uint64_t *status, uint32_t *tile_counter, uint32_t *hist_next,
                       uint32_t next_shift, uint32_t next_bits, cudaStream_t s, uint64_t n0,
                       uint64_t gap) {
  if (n0 > n || gap == 0) n0 = n;  // one segment
  const uint32_t next_mask = (1u << next_bits) - 1u;
  if (vin) {
    // (key, rowid) pairs: 4096-key tiles (the payload needs the registers)
    const uint64_t ntiles = ceil_div(n, kSortTile);
    const size_t smem = kSortTile * (sizeof(uint64_t) + sizeof(uint32_t));
    auto kern = radix_pass_kernel<true, kSortItems, kLookWin, 3, false, true>;
    set_smem_limit((const void *)kern, smem);
    kern<<<(unsigned)ntiles, kSortThreads, smem, s>>>(
        kin, kout, vin, vout, n, shift, bits, hist_pass, status, tile_counter, hist_next,
        next_shift, next_mask, n, 0);
  } else {
    // P64 words: 6144-key tiles, 3 CTAs/SM, keys re-read from L2 for placement.  Peers found by
    // shared-memory atomicOr with a warp-uniform shortcut (tools/radix_ablate.cu: a C4-shaped
    // 4e8-word Zipf sort 9.70 ms vs 10.72 with match.any / 10.57 with ballots at 8192-key tiles;
    // 6144-key tiles at 3 CTAs/SM then 8.89 ms, C5's join words -7%).
    constexpr int kItems = MAPSQ_RADIX_ITEMS;  // (ablation knobs: -DMAPSQ_RADIX_ITEMS / _MINB)
    const uint64_t ntiles = ceil_div(n, (uint64_t)kSortThreads * kItems);
    const size_t smem = (size_t)kSortThreads * kItems * sizeof(uint64_t);
    auto kern = (gap && n0 < n)
                    ? radix_pass_kernel<false, kItems, MAPSQ_RADIX_WIN, MAPSQ_RADIX_MINB, true, 3, true>
                    : radix_pass_kernel<false, kItems, MAPSQ_RADIX_WIN, MAPSQ_RADIX_MINB, true, 3, false>;
    set_smem_limit((const void *)kern, smem);
    kern<<<(unsigned)ntiles, kSortThreads, smem, s>>>(kin, kout, vin, vout, n, shift, bits,
                                                      hist_pass, status, tile_counter, hist_next,
                                                      next_shift, next_mask, n0, gap);
  }
}

}  // namespace mapsq
