// scan.cu — K1: partial matching of triple patterns over the SoA triple table.
//
// The paper delegates partial matching to gStore on the CPU ("each triple
// pattern matches the partial results through centralized RDF engine in parallel").  Here it is
// a two-pass GPU scan that evaluates ALL k patterns of a query in the same passes:
//   pass 1 (predicate): read only the positions that carry constants or repeated variables
//          (for LUBM-style patterns: the p column, 4 B/triple), evaluate every pattern, write one
//          32-bit match word per 32 triples per pattern and per-tile match counts;
//   host:  one blocking read of the k totals, allocate the k outputs;
//   pass 2 (gather): re-read the match words and load s/o (32 B sectors) only where some
//          pattern matched; write the bound positions in triple order (stable compaction).
// Both passes use the same tile geometry: 8 warps x 32 match words x 32 triples = 8192.
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kWarps = kScanThreads / 32;

// Pass 1 (predicate).  Warp w of tile T owns 32 match words (1024 triples); lane l reads triple
// (word0 + w') * 32 + l of every word w' (coalesced 128 B rows) into registers once, then every
// pattern is evaluated over the 32 register-resident rows with its constants hoisted: one
// masked-XOR test (precomputed on the host), one ballot and one select per word and pattern.
template <int NEED>
__device__ __forceinline__ bool const_test(const uint32_t c[3], const uint32_t m[3], uint32_t s,
                                           uint32_t p, uint32_t o) {
  uint32_t x = 0;
  if (NEED & 1) x |= (s ^ c[0]) & m[0];
  if (NEED & 2) x |= (p ^ c[1]) & m[1];
  if (NEED & 4) x |= (o ^ c[2]) & m[2];
  return x == 0;
}

template <int NEED>
__global__ void __launch_bounds__(kScanThreads)
scan_count_kernel(const uint32_t *__restrict__ S, const uint32_t *__restrict__ P,
                  const uint32_t *__restrict__ O, uint64_t n, const ScanArgs a,
                  uint32_t *__restrict__ masks, uint64_t mask_words,
                  uint32_t *__restrict__ tile_counts, uint64_t ntiles) {
  __shared__ uint32_t s_cnt[kWarps][MAPSQ_MAX_PATTERNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t tile = blockIdx.x;
  const uint64_t word0 = tile * (kWarps * kScanWordsPerWarp) + (uint64_t)warp * kScanWordsPerWarp;
  const uint64_t base = word0 * 32 + lane;
  const bool full = (word0 + kScanWordsPerWarp) * 32 <= n;
  // rows past n read as an impossible triple (never matches: tail words are masked below)
  uint32_t vs[kScanWordsPerWarp], vp[kScanWordsPerWarp], vo[kScanWordsPerWarp];
  if (full) {
#pragma unroll
    for (int w = 0; w < kScanWordsPerWarp; w++) {
      const uint64_t i = base + (uint64_t)w * 32;
      vs[w] = (NEED & 1) ? __ldcs(S + i) : 0u;
      vp[w] = (NEED & 2) ? __ldcs(P + i) : 0u;
      vo[w] = (NEED & 4) ? __ldcs(O + i) : 0u;
    }
  } else {
#pragma unroll
    for (int w = 0; w < kScanWordsPerWarp; w++) {
      const uint64_t i = base + (uint64_t)w * 32;
      const bool in = i < n;
      vs[w] = ((NEED & 1) && in) ? __ldcs(S + i) : 0u;
      vp[w] = ((NEED & 2) && in) ? __ldcs(P + i) : 0u;
      vo[w] = ((NEED & 4) && in) ? __ldcs(O + i) : 0u;
    }
  }
  // valid-lane mask of word w: all lanes for full warps, else lanes with index < n
  const uint64_t nlim = n;
  const uint64_t my_word = word0 + lane;
  for (int j = 0; j < a.k; j++) {
    uint32_t c[3], m[3];
#pragma unroll
    for (int q = 0; q < 3; q++) {
      c[q] = a.pat[j].c[q];
      m[q] = a.pat[j].m[q];
    }
    const uint32_t eq = a.pat[j].eq_mask;
    uint32_t mine = 0;
    if (eq == 0) {
#pragma unroll
      for (int w = 0; w < kScanWordsPerWarp; w++) {
        const uint32_t bw = __ballot_sync(0xffffffffu, const_test<NEED>(c, m, vs[w], vp[w], vo[w]));
        mine = (lane == w) ? bw : mine;
      }
    } else {
#pragma unroll
      for (int w = 0; w < kScanWordsPerWarp; w++) {
        bool ok = const_test<NEED>(c, m, vs[w], vp[w], vo[w]);
        if (eq & 1) ok &= vs[w] == vp[w];
        if (eq & 2) ok &= vs[w] == vo[w];
        if (eq & 4) ok &= vp[w] == vo[w];
        const uint32_t bw = __ballot_sync(0xffffffffu, ok);
        mine = (lane == w) ? bw : mine;
      }
    }
    if (!full) {  // clear bits of rows >= n
      const uint64_t first = my_word * 32;
      mine = first >= nlim ? 0u : (nlim - first >= 32 ? mine : mine & ((1u << (nlim - first)) - 1u));
    }
    if (my_word < mask_words) masks[(uint64_t)j * mask_words + my_word] = mine;
    const uint32_t cnt = __reduce_add_sync(0xffffffffu, __popc(mine));
    if (lane == 0) s_cnt[warp][j] = cnt;
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)a.k) {
    uint32_t t = 0;
    for (int w = 0; w < kWarps; w++) t += s_cnt[w][threadIdx.x];
    tile_counts[(uint64_t)threadIdx.x * ntiles + tile] = t;
  }
}

// Pass 2 (gather), pattern-outer, as warp-level stream compaction: the hit positions of 8 match
// words (256 triples) are compacted into a per-warp shared list, then processed densely — every
// lane active, consecutive output positions, increasing input positions — instead of one
// divergent block per word.  Only the 32 B sectors holding matches are read; the output cursor
// and column bounds live in registers.
__device__ __forceinline__ uint32_t pick(const uint32_t *__restrict__ S, const uint32_t *__restrict__ P,
                                         const uint32_t *__restrict__ O, uint32_t src, uint64_t i) {
  return __ldcs((src == 0 ? S : (src == 1 ? P : O)) + i);
}

constexpr int kGatherWords = 8;

__global__ void __launch_bounds__(kScanThreads)
scan_write_kernel(const uint32_t *__restrict__ S, const uint32_t *__restrict__ P,
                  const uint32_t *__restrict__ O, uint64_t n, const ScanArgs a,
                  const uint32_t *__restrict__ masks, uint64_t mask_words,
                  const uint64_t *__restrict__ tile_off, uint64_t ntiles, const ScanOut out,
                  uint32_t *__restrict__ bmin, uint32_t *__restrict__ bmax) {
  __shared__ uint32_t s_wcnt[kWarps][MAPSQ_MAX_PATTERNS];
  __shared__ uint32_t s_min[kWarps][MAPSQ_MAX_PATTERNS * 3], s_max[kWarps][MAPSQ_MAX_PATTERNS * 3];
  __shared__ uint16_t s_list[kWarps][kGatherWords * 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  const uint64_t tile = blockIdx.x;
  const uint64_t word0 = tile * (kWarps * kScanWordsPerWarp) + (uint64_t)warp * kScanWordsPerWarp;
  const uint64_t my_word = word0 + lane;
  const uint64_t row0 = word0 * 32;
  for (int j = 0; j < k; j++) {
    const uint32_t m = my_word < mask_words ? masks[(uint64_t)j * mask_words + my_word] : 0u;
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(m));
    if (lane == 0) s_wcnt[warp][j] = c;
  }
  __syncthreads();
  const uint32_t lt = lanemask_lt();
  uint16_t *list = s_list[warp];
  for (int j = 0; j < k; j++) {
    const uint32_t mine = my_word < mask_words ? masks[(uint64_t)j * mask_words + my_word] : 0u;
    uint32_t mn0 = ~0u, mn1 = ~0u, mn2 = ~0u, mx0 = 0, mx1 = 0, mx2 = 0;
    if (__ballot_sync(0xffffffffu, mine != 0) != 0) {
      // tile_off is one scan over all patterns' tile counts: subtract pattern j's base
      uint64_t cur = tile_off[(uint64_t)j * ntiles + tile] - tile_off[(uint64_t)j * ntiles];
      for (int w = 0; w < warp; w++) cur += s_wcnt[w][j];
      const uint32_t nc = a.pat[j].ncols, src0 = a.pat[j].src[0], src1 = a.pat[j].src[1],
                     src2 = a.pat[j].src[2];
      uint32_t *o0 = out.col[j * 3], *o1 = out.col[j * 3 + 1], *o2 = out.col[j * 3 + 2];
#pragma unroll 1
      for (int w0 = 0; w0 < kScanWordsPerWarp; w0 += kGatherWords) {
        uint32_t h = 0;
#pragma unroll
        for (int u = 0; u < kGatherWords; u++) {
          const uint32_t m = __shfl_sync(0xffffffffu, mine, w0 + u);
          if ((m >> lane) & 1u) list[h + __popc(m & lt)] = (uint16_t)((w0 + u) * 32 + lane);
          h += __popc(m);
        }
        __syncwarp();
        for (uint32_t q = lane; q < h; q += 32) {
          const uint64_t i = row0 + list[q];
          const uint64_t pos = cur + q;
          const uint32_t v0 = pick(S, P, O, src0, i);
          st_cs_u32(o0 + pos, v0);
          mn0 = min(mn0, v0);
          mx0 = max(mx0, v0);
          if (nc > 1) {
            const uint32_t v1 = pick(S, P, O, src1, i);
            st_cs_u32(o1 + pos, v1);
            mn1 = min(mn1, v1);
            mx1 = max(mx1, v1);
          }
          if (nc > 2) {
            const uint32_t v2 = pick(S, P, O, src2, i);
            st_cs_u32(o2 + pos, v2);
            mn2 = min(mn2, v2);
            mx2 = max(mx2, v2);
          }
        }
        cur += h;
        __syncwarp();
      }
    }
    mn0 = __reduce_min_sync(0xffffffffu, mn0);
    mx0 = __reduce_max_sync(0xffffffffu, mx0);
    mn1 = __reduce_min_sync(0xffffffffu, mn1);
    mx1 = __reduce_max_sync(0xffffffffu, mx1);
    mn2 = __reduce_min_sync(0xffffffffu, mn2);
    mx2 = __reduce_max_sync(0xffffffffu, mx2);
    if (lane == 0) {
      s_min[warp][j * 3] = mn0; s_max[warp][j * 3] = mx0;
      s_min[warp][j * 3 + 1] = mn1; s_max[warp][j * 3 + 1] = mx1;
      s_min[warp][j * 3 + 2] = mn2; s_max[warp][j * 3 + 2] = mx2;
    }
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)k * 3) {
    const int j = threadIdx.x / 3, c = threadIdx.x % 3;
    if ((uint32_t)c < a.pat[j].ncols) {
      uint32_t mn = 0xffffffffu, mx = 0;
      for (int w = 0; w < kWarps; w++) {
        mn = min(mn, s_min[w][threadIdx.x]);
        mx = max(mx, s_max[w][threadIdx.x]);
      }
      if (mn <= mx) {  // at least one match in this tile
        atomicMin(bmin + threadIdx.x, mn);
        atomicMax(bmax + threadIdx.x, mx);
      }
    }
  }
}

// ------------------------------------------------------------------ exclusive scan (u32/u64)
constexpr int kScanChunkThreads = 256;
constexpr int kScanChunkItems = 16;
constexpr uint64_t kChunk = kScanChunkThreads * kScanChunkItems;

// exclusive block scan of one value per thread; returns exclusive prefix, *total = block sum
__device__ __forceinline__ uint64_t block_exscan(uint64_t v, uint64_t *total) {
  __shared__ uint64_t s_w[kScanChunkThreads / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t x = v;
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) s_w[warp] = x;
  __syncthreads();
  uint64_t wpre = 0, tot = 0;
  for (int w = 0; w < kScanChunkThreads / 32; w++) {
    if (w < warp) wpre += s_w[w];
    tot += s_w[w];
  }
  __syncthreads();
  *total = tot;
  return wpre + x - v;
}

// Single-pass exclusive scan: CTAs claim chunks in order (atomic counter) and resolve their
// chunk's prefix by a decoupled look-back over per-chunk 64-bit status words (flags in the top two
// bits, 62-bit sums), so one launch replaces reduce / partials / down.  The last chunk writes the
// total.  status[0 .. nchunks) and the counter are zero on entry.
__device__ __forceinline__ uint64_t warp_lookback64(uint64_t *status, uint64_t tile, uint64_t agg) {
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
    uint64_t val = ((int)lane <= first_inc) ? (v & kValMask) : 0ull;
#pragma unroll
    for (int o = 16; o; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
    excl += val;
    if (first_inc < 32) break;
    t0 -= 32;
  }
  if (lane == 0) st_relaxed_u64(status + tile, kFlagInc | (excl + agg));
  return excl;
}

template <typename T>
__global__ void __launch_bounds__(kScanChunkThreads)
scan_onepass_kernel(const T *__restrict__ in, uint64_t *__restrict__ out, const uint64_t *n_dev,
                    uint64_t n_host, uint64_t *__restrict__ status, uint32_t *__restrict__ ctr,
                    uint64_t *total_dev) {
  __shared__ uint32_t s_tile;
  __shared__ uint64_t s_excl;
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nchunks = ceil_div(n, kChunk);
  const uint32_t warp = threadIdx.x >> 5;
  while (true) {
    __syncthreads();  // (s_tile / s_excl reuse)
    if (threadIdx.x == 0) s_tile = atomicAdd(ctr, 1u);
    __syncthreads();
    const uint64_t c = s_tile;
    if (c >= nchunks) {
      if (c == 0 && threadIdx.x == 0 && total_dev) *total_dev = 0;  // (n == 0)
      return;
    }
    // thread t scans items [base + t * ITEMS, + ITEMS) of the chunk (contiguous per thread)
    const uint64_t base = c * kChunk + (uint64_t)threadIdx.x * kScanChunkItems;
    uint64_t v[kScanChunkItems];
    uint64_t sum = 0;
#pragma unroll
    for (int it = 0; it < kScanChunkItems; it++) {
      const uint64_t i = base + it;
      v[it] = i < n ? (uint64_t)in[i] : 0;
      sum += v[it];
    }
    uint64_t tot;
    const uint64_t ex = block_exscan(sum, &tot);
    if (warp == 0) {
      const uint64_t excl = warp_lookback64(status, c, tot);
      if (threadIdx.x == 0) {
        s_excl = excl;
        if (c + 1 == nchunks && total_dev) *total_dev = excl + tot;
      }
    }
    __syncthreads();
    uint64_t run = s_excl + ex;
#pragma unroll
    for (int it = 0; it < kScanChunkItems; it++) {
      const uint64_t i = base + it;
      if (i < n) out[i] = run;
      run += v[it];
    }
  }
}

// ------------------------------------------------------------------ min/max of columns
__global__ void __launch_bounds__(256)
minmax_kernel(const uint32_t *__restrict__ col, uint64_t n, uint32_t *__restrict__ out) {
  uint32_t mn = 0xffffffffu, mx = 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t v = __ldcs(col + i);
    mn = min(mn, v);
    mx = max(mx, v);
  }
  mn = __reduce_min_sync(0xffffffffu, mn);
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(out, mn);
    atomicMax(out + 1, mx);
  }
}

}  // namespace

void launch_scan_count(const mapsq_triples &T, const ScanArgs &a, uint32_t *masks,
                       uint64_t mask_words, uint32_t *tile_counts, uint64_t ntiles,
                       cudaStream_t s) {
#define MAPSQ_SCAN_COUNT(NEED)                                                              \
  scan_count_kernel<NEED><<<(unsigned)ntiles, kScanThreads, 0, s>>>(T.s, T.p, T.o, T.n, a, masks, \
                                                                   mask_words, tile_counts, ntiles)
  switch (a.need_count & 7) {
    case 1: MAPSQ_SCAN_COUNT(1); break;
    case 2: MAPSQ_SCAN_COUNT(2); break;
    case 3: MAPSQ_SCAN_COUNT(3); break;
    case 4: MAPSQ_SCAN_COUNT(4); break;
    case 5: MAPSQ_SCAN_COUNT(5); break;
    case 6: MAPSQ_SCAN_COUNT(6); break;
    default: MAPSQ_SCAN_COUNT(7); break;
  }
#undef MAPSQ_SCAN_COUNT
}

void launch_scan_write(const mapsq_triples &T, const ScanArgs &a, const uint32_t *masks,
                       uint64_t mask_words, const uint64_t *tile_off, uint64_t ntiles,
                       const ScanOut &out, uint32_t *bmin, uint32_t *bmax, cudaStream_t s) {
  scan_write_kernel<<<(unsigned)ntiles, kScanThreads, 0, s>>>(T.s, T.p, T.o, T.n, a, masks,
                                                              mask_words, tile_off, ntiles, out,
                                                              bmin, bmax);
}

uint64_t scan_tmp_words(uint64_t n) { return ceil_div(n, kChunk) + 1; }

static int scan_grid(uint64_t n) {
  uint64_t c = ceil_div(n, kChunk);
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(c, 148 * 8));
}

// (tmp: scan_tmp_words(n) words — the per-chunk status words, then the chunk counter)
int launch_exclusive_scan_u32(const uint32_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s) {
  const uint64_t nc = ceil_div(n, kChunk);
  cudaMemsetAsync(tmp, 0, (nc + 1) * sizeof(uint64_t), s);
  scan_onepass_kernel<uint32_t><<<scan_grid(n), kScanChunkThreads, 0, s>>>(
      in, out, nullptr, n, tmp, reinterpret_cast<uint32_t *>(tmp + nc), total_dev);
  return 1;
}

int launch_exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s) {
  const uint64_t nc = ceil_div(n, kChunk);
  cudaMemsetAsync(tmp, 0, (nc + 1) * sizeof(uint64_t), s);
  scan_onepass_kernel<uint64_t><<<scan_grid(n), kScanChunkThreads, 0, s>>>(
      in, out, nullptr, n, tmp, reinterpret_cast<uint32_t *>(tmp + nc), total_dev);
  return 1;
}

// Variant whose element count lives on the device (grid and status sized for the capacity `cap`).
int launch_exclusive_scan_u64_dev(const uint64_t *in, uint64_t *out, const uint64_t *n_dev,
                                  uint64_t cap, uint64_t *tmp, uint64_t *total_dev,
                                  cudaStream_t s) {
  const uint64_t nc = ceil_div(cap, kChunk);
  cudaMemsetAsync(tmp, 0, (nc + 1) * sizeof(uint64_t), s);
  scan_onepass_kernel<uint64_t><<<scan_grid(cap), kScanChunkThreads, 0, s>>>(
      in, out, n_dev, 0, tmp, reinterpret_cast<uint32_t *>(tmp + nc), total_dev);
  return 1;
}

void launch_minmax(const uint32_t *const *cols, uint32_t ncols, uint64_t n, uint32_t *bounds,
                   cudaStream_t s) {
  const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, 256 * 8), 148 * 8));
  for (uint32_t c = 0; c < ncols; c++)
    minmax_kernel<<<g, 256, 0, s>>>(cols[c], n, bounds + 2 * c);
}

}  // namespace mapsq
