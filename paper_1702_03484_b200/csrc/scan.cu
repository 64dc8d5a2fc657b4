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

__device__ __forceinline__ bool pat_match(const ScanPat &p, uint32_t s, uint32_t pp, uint32_t o) {
  bool ok = true;
  if (p.const_mask & 1) ok &= (s == p.id[0]);
  if (p.const_mask & 2) ok &= (pp == p.id[1]);
  if (p.const_mask & 4) ok &= (o == p.id[2]);
  if (p.eq_mask & 1) ok &= (s == pp);
  if (p.eq_mask & 2) ok &= (s == o);
  if (p.eq_mask & 4) ok &= (pp == o);
  return ok;
}

// Patterns are evaluated in a runtime loop over descriptors staged in shared memory (no unroll
// over MAPSQ_MAX_PATTERNS: that blew the instruction cache).
__global__ void __launch_bounds__(kScanThreads)
scan_count_kernel(const uint32_t *__restrict__ S, const uint32_t *__restrict__ P,
                  const uint32_t *__restrict__ O, uint64_t n, const ScanArgs a,
                  uint32_t *__restrict__ masks, uint64_t mask_words,
                  uint32_t *__restrict__ tile_counts, uint64_t ntiles) {
  __shared__ ScanPat s_pat[MAPSQ_MAX_PATTERNS];
  __shared__ uint32_t s_mw[kWarps][MAPSQ_MAX_PATTERNS][kScanWordsPerWarp];
  __shared__ uint32_t s_cnt[kWarps][MAPSQ_MAX_PATTERNS];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  if (threadIdx.x < (unsigned)k) s_pat[threadIdx.x] = a.pat[threadIdx.x];
  __syncthreads();
  const uint64_t tile = blockIdx.x;
  const uint64_t word0 = tile * (kWarps * kScanWordsPerWarp) + (uint64_t)warp * kScanWordsPerWarp;
  const bool ns = a.need_count & 1, np = a.need_count & 2, no = a.need_count & 4;
#pragma unroll 1
  for (int w = 0; w < kScanWordsPerWarp; w += 8) {
    uint32_t vs[8], vp[8], vo[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint64_t i = (word0 + w + u) * 32 + lane;
      const bool in = i < n;
      vs[u] = (ns && in) ? __ldcs(S + i) : 0u;
      vp[u] = (np && in) ? __ldcs(P + i) : 0u;
      vo[u] = (no && in) ? __ldcs(O + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const bool in = (word0 + w + u) * 32 + lane < n;
#pragma unroll 1
      for (int j = 0; j < k; j++) {
        const uint32_t m = __ballot_sync(0xffffffffu, in && pat_match(s_pat[j], vs[u], vp[u], vo[u]));
        if (lane == 0) s_mw[warp][j][w + u] = m;
      }
    }
  }
  __syncwarp();
  const uint64_t my_word = word0 + lane;
  for (int j = 0; j < k; j++) {
    const uint32_t m = s_mw[warp][j][lane];
    if (my_word < mask_words) masks[(uint64_t)j * mask_words + my_word] = m;
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(m));
    if (lane == 0) s_cnt[warp][j] = c;
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)k) {
    uint32_t t = 0;
    for (int w = 0; w < kWarps; w++) t += s_cnt[w][threadIdx.x];
    tile_counts[(uint64_t)threadIdx.x * ntiles + tile] = t;
  }
}

__global__ void __launch_bounds__(kScanThreads)
scan_write_kernel(const uint32_t *__restrict__ S, const uint32_t *__restrict__ P,
                  const uint32_t *__restrict__ O, uint64_t n, const ScanArgs a,
                  const uint32_t *__restrict__ masks, uint64_t mask_words,
                  const uint64_t *__restrict__ tile_off, uint64_t ntiles, const ScanOut out,
                  uint32_t *__restrict__ bmin, uint32_t *__restrict__ bmax) {
  __shared__ ScanPat s_pat[MAPSQ_MAX_PATTERNS];
  __shared__ uint32_t s_mw[kWarps][MAPSQ_MAX_PATTERNS][kScanWordsPerWarp];
  __shared__ uint32_t s_wcnt[kWarps][MAPSQ_MAX_PATTERNS];
  __shared__ uint64_t s_cur[kWarps][MAPSQ_MAX_PATTERNS];
  __shared__ uint32_t s_min[kWarps][MAPSQ_MAX_PATTERNS * 3], s_max[kWarps][MAPSQ_MAX_PATTERNS * 3];
  __shared__ uint32_t *s_out[MAPSQ_MAX_PATTERNS * 3];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k = a.k;
  const uint64_t tile = blockIdx.x;
  const uint64_t word0 = tile * (kWarps * kScanWordsPerWarp) + (uint64_t)warp * kScanWordsPerWarp;
  const uint64_t my_word = word0 + lane;
  if (threadIdx.x < MAPSQ_MAX_PATTERNS * 3) s_out[threadIdx.x] = out.col[threadIdx.x];
  if (threadIdx.x < (unsigned)k) s_pat[threadIdx.x] = a.pat[threadIdx.x];
  for (int j = lane; j < MAPSQ_MAX_PATTERNS * 3; j += 32) {
    s_min[warp][j] = 0xffffffffu;
    s_max[warp][j] = 0u;
  }
  uint32_t any_mine = 0;  // OR over patterns of this lane's word
  for (int j = 0; j < k; j++) {
    const uint32_t m = my_word < mask_words ? masks[(uint64_t)j * mask_words + my_word] : 0u;
    s_mw[warp][j][lane] = m;
    any_mine |= m;
    const uint32_t c = __reduce_add_sync(0xffffffffu, __popc(m));
    if (lane == 0) s_wcnt[warp][j] = c;
  }
  __syncthreads();
  if (lane < k) {
    // tile_off is one scan over all patterns' tile counts: subtract pattern j's base
    uint64_t c = tile_off[(uint64_t)lane * ntiles + tile] - tile_off[(uint64_t)lane * ntiles];
    for (int w = 0; w < warp; w++) c += s_wcnt[w][lane];
    s_cur[warp][lane] = c;
  }
  __syncwarp();
  const bool ws = a.need_write & 1, wp = a.need_write & 2, wo = a.need_write & 4;
  const uint32_t lt = lanemask_lt();
#pragma unroll 1
  for (int w = 0; w < kScanWordsPerWarp; w += 8) {
    uint32_t vs[8], vp[8], vo[8], any[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t m = __shfl_sync(0xffffffffu, any_mine, w + u);
      any[u] = m;
      const uint64_t i = (word0 + w + u) * 32 + lane;
      const bool hit = (m >> lane) & 1u;
      vs[u] = (ws && hit) ? __ldcs(S + i) : 0u;
      vp[u] = (wp && hit) ? __ldcs(P + i) : 0u;
      vo[u] = (wo && hit) ? __ldcs(O + i) : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      if (any[u] == 0) continue;  // warp-uniform
#pragma unroll 1
      for (int j = 0; j < k; j++) {
        const uint32_t m = s_mw[warp][j][w + u];
        if (m == 0) continue;
        const bool hit = (m >> lane) & 1u;
        const uint64_t base = s_cur[warp][j];
        const uint64_t pos = base + __popc(m & lt);
        const uint32_t nc = s_pat[j].ncols;
        for (uint32_t c = 0; c < nc; c++) {
          const uint32_t src = s_pat[j].src[c];
          const uint32_t v = src == 0 ? vs[u] : (src == 1 ? vp[u] : vo[u]);
          if (hit) st_cs_u32(s_out[j * 3 + c] + pos, v);
          const uint32_t mn = __reduce_min_sync(0xffffffffu, hit ? v : 0xffffffffu);
          const uint32_t mx = __reduce_max_sync(0xffffffffu, hit ? v : 0u);
          if (lane == 0) {
            s_min[warp][j * 3 + c] = min(s_min[warp][j * 3 + c], mn);
            s_max[warp][j * 3 + c] = max(s_max[warp][j * 3 + c], mx);
          }
        }
        __syncwarp();
        if (lane == 0) s_cur[warp][j] = base + __popc(m);
        __syncwarp();
      }
    }
  }
  __syncthreads();
  if (threadIdx.x < (unsigned)k * 3) {
    const int j = threadIdx.x / 3, c = threadIdx.x % 3;
    if ((uint32_t)c < s_pat[j].ncols) {
      uint32_t mn = 0xffffffffu, mx = 0;
      for (int w = 0; w < kWarps; w++) {
        mn = min(mn, s_min[w][threadIdx.x]);
        mx = max(mx, s_max[w][threadIdx.x]);
      }
      if (mn != 0xffffffffu || mx != 0) {
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

template <typename T>
__device__ __forceinline__ uint64_t block_reduce_chunk(const T *in, uint64_t n, uint64_t base) {
  __shared__ uint64_t s_red[kScanChunkThreads / 32];
  uint64_t acc = 0;
#pragma unroll
  for (int it = 0; it < kScanChunkItems; it++) {
    const uint64_t i = base + (uint64_t)it * kScanChunkThreads + threadIdx.x;
    if (i < n) acc += (uint64_t)in[i];
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  uint64_t t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < kScanChunkThreads / 32; w++) t += s_red[w];
  __syncthreads();
  return t;  // valid in thread 0
}

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

template <typename T>
__global__ void __launch_bounds__(kScanChunkThreads)
scan_reduce_kernel(const T *__restrict__ in, const uint64_t *n_dev, uint64_t n_host,
                   uint64_t *__restrict__ partial) {
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nchunks = ceil_div(n, kChunk);
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    uint64_t t = block_reduce_chunk(in, n, c * kChunk);
    if (threadIdx.x == 0) partial[c] = t;
  }
}

__global__ void __launch_bounds__(kScanChunkThreads)
scan_partials_kernel(uint64_t *__restrict__ partial, const uint64_t *n_dev, uint64_t n_host,
                     uint64_t *total_dev) {
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nchunks = ceil_div(n, kChunk);
  uint64_t carry = 0;
  for (uint64_t base = 0; base < nchunks; base += kScanChunkThreads) {
    const uint64_t i = base + threadIdx.x;
    const uint64_t v = i < nchunks ? partial[i] : 0;
    uint64_t tot;
    const uint64_t ex = block_exscan(v, &tot);
    if (i < nchunks) partial[i] = carry + ex;
    carry += tot;
  }
  if (threadIdx.x == 0 && total_dev) *total_dev = carry;
}

template <typename T>
__global__ void __launch_bounds__(kScanChunkThreads)
scan_down_kernel(const T *__restrict__ in, uint64_t *__restrict__ out, const uint64_t *n_dev,
                 uint64_t n_host, const uint64_t *__restrict__ partial) {
  const uint64_t n = n_dev ? *n_dev : n_host;
  const uint64_t nchunks = ceil_div(n, kChunk);
  for (uint64_t c = blockIdx.x; c < nchunks; c += gridDim.x) {
    // thread t scans items [base + t*ITEMS, +ITEMS) of the chunk (contiguous per thread)
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
    uint64_t run = partial[c] + block_exscan(sum, &tot);
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
  scan_count_kernel<<<(unsigned)ntiles, kScanThreads, 0, s>>>(T.s, T.p, T.o, T.n, a, masks,
                                                              mask_words, tile_counts, ntiles);
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

int launch_exclusive_scan_u32(const uint32_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s) {
  const int g = scan_grid(n);
  scan_reduce_kernel<uint32_t><<<g, kScanChunkThreads, 0, s>>>(in, nullptr, n, tmp);
  scan_partials_kernel<<<1, kScanChunkThreads, 0, s>>>(tmp, nullptr, n, total_dev);
  scan_down_kernel<uint32_t><<<g, kScanChunkThreads, 0, s>>>(in, out, nullptr, n, tmp);
  return 3;
}

int launch_exclusive_scan_u64(const uint64_t *in, uint64_t *out, uint64_t n, uint64_t *tmp,
                              uint64_t *total_dev, cudaStream_t s) {
  const int g = scan_grid(n);
  scan_reduce_kernel<uint64_t><<<g, kScanChunkThreads, 0, s>>>(in, nullptr, n, tmp);
  scan_partials_kernel<<<1, kScanChunkThreads, 0, s>>>(tmp, nullptr, n, total_dev);
  scan_down_kernel<uint64_t><<<g, kScanChunkThreads, 0, s>>>(in, out, nullptr, n, tmp);
  return 3;
}

// Variant whose element count lives on the device (grid sized for the capacity `cap`).
int launch_exclusive_scan_u64_dev(const uint64_t *in, uint64_t *out, const uint64_t *n_dev,
                                  uint64_t cap, uint64_t *tmp, uint64_t *total_dev,
                                  cudaStream_t s) {
  const int g = scan_grid(cap);
  scan_reduce_kernel<uint64_t><<<g, kScanChunkThreads, 0, s>>>(in, n_dev, 0, tmp);
  scan_partials_kernel<<<1, kScanChunkThreads, 0, s>>>(tmp, n_dev, 0, total_dev);
  scan_down_kernel<uint64_t><<<g, kScanChunkThreads, 0, s>>>(in, out, n_dev, 0, tmp);
  return 3;
}

void launch_minmax(const uint32_t *const *cols, uint32_t ncols, uint64_t n, uint32_t *bounds,
                   cudaStream_t s) {
  const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, 256 * 8), 148 * 8));
  for (uint32_t c = 0; c < ncols; c++)
    minmax_kernel<<<g, 256, 0, s>>>(cols[c], n, bounds + 2 * c);
}

}  // namespace mapsq
