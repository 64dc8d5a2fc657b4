// partition.cu — K8: hash partition of a partial-match table on its join key (SURVEY §8 row e),
// fused with the exchange: the scatter stores every row straight into its destination rank's
// receive arena through NVLink peer pointers (one kernel does the partition and the all-to-all).
//
// An equi-join decomposes over disjoint key sets, so on G GPUs each rank sends every row to
// rank dest = (fmix32(fold(key)) * G) >> 32 and then runs the local sort-join on what it receives.
// Two passes over tiles: a per-tile destination histogram, then (after an exclusive scan of the
// dest-major histogram) a stable scatter that groups the rows by destination, ready for one
// contiguous send per peer.
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kWarps = kPartThreads / 32;

__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
  h ^= h >> 16;
  h *= 0x85ebca6bu;
  h ^= h >> 13;
  h *= 0xc2b2ae35u;
  h ^= h >> 16;
  return h;
}

// Destination of row `i` (row index relative to the pointers' base): FNV-1a-style fold of the key
// columns, fmix32, multiply-shift range reduction (no integer division).
// NKEY > 0: that many key columns (unrolled, pointers in uniform registers); 0: a.nkey of them.
template <int NKEY>
__device__ __forceinline__ uint32_t dest_of(const PartArgs &a, uint64_t base, uint32_t i) {
  uint32_t h = 0x811c9dc5u;
  if (NKEY > 0) {
    uint32_t v[NKEY > 0 ? NKEY : 1];
#pragma unroll
    for (int c = 0; c < NKEY; c++) {
      v[c] = __ldg(a.key[c] + base + i);
      h = (h ^ v[c]) * 0x01000193u;
    }
    // a heavy (skewed) key's rows of the split side stay where they are (dist.cu)
    for (uint32_t q = 0; q < a.nheavy; q++) {
      bool eq = true;
#pragma unroll
      for (int c = 0; c < NKEY; c++) eq &= v[c] == a.heavy[q * kMaxHeavyCols + c];
      if (eq) return a.self;
    }
  } else {
    for (uint32_t c = 0; c < a.nkey; c++) h = (h ^ __ldg(a.key[c] + base + i)) * 0x01000193u;
  }
  return __umulhi(fmix32(h), a.nparts);
}

// keep / broadcast masks of the heavy keys (one warp per 32 rows)
__global__ void __launch_bounds__(256)
heavy_mask_kernel(const PartArgs a, uint32_t *__restrict__ keep, uint32_t *__restrict__ bcast) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nw = (a.n + 31) / 32;
  for (uint64_t w = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32; w < nw;
       w += (uint64_t)gridDim.x * blockDim.x / 32) {
    const uint64_t r = w * 32 + lane;
    bool in = r < a.n && (!a.mask || (__ldg(a.mask + w) >> lane & 1u));
    bool heavy = false;
    if (in) {
      for (uint32_t q = 0; q < a.nheavy && !heavy; q++) {
        bool eq = true;
        for (uint32_t c = 0; c < a.nkey; c++) eq &= __ldg(a.key[c] + r) == a.heavy[q * kMaxHeavyCols + c];
        heavy = eq;
      }
    }
    const uint32_t k = __ballot_sync(0xffffffffu, in && !heavy);
    const uint32_t b = __ballot_sync(0xffffffffu, in && heavy);
    if (lane == 0) {
      keep[w] = k;
      bcast[w] = b;
    }
  }
}

// Lanes of the warp holding the same destination: one ballot per destination bit (nbits =
// ceil(log2 nparts), 0 on one rank), intersected with the lanes holding a row.
__device__ __forceinline__ uint32_t peers_of(uint32_t d, bool in, int nbits) {
  uint32_t peers = __ballot_sync(0xffffffffu, in);
  for (int b = 0; b < nbits; b++) {
    const bool bit = (d >> b) & 1u;
    const uint32_t m = __ballot_sync(0xffffffffu, bit);
    peers &= bit ? m : ~m;
  }
  return peers;
}

__device__ __forceinline__ int dest_bits(uint32_t nparts) { return 32 - __clz((int)nparts - 1); }

// the row participates (no mask, or its bit in the survivor mask is set)
__device__ __forceinline__ bool row_kept(const PartArgs &a, uint64_t row) {
  return !a.mask || (__ldg(a.mask + (row >> 5)) >> (row & 31) & 1u);
}

__device__ __forceinline__ uint32_t rows_left(uint64_t n, uint64_t base, uint32_t cap) {
  const uint64_t r = n > base ? n - base : 0;
  return r < cap ? (uint32_t)r : cap;
}

template <int NKEY>
__global__ void __launch_bounds__(kPartThreads)
partition_hist_kernel(const PartArgs a, uint32_t *__restrict__ tile_hist, uint64_t ntiles) {
  __shared__ uint32_t s_h[kMaxParts];
  if (threadIdx.x < kMaxParts) s_h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kPartTile;
  const uint32_t rem = rows_left(a.n, base, kPartTile);
  const uint32_t lane = threadIdx.x & 31;
  const int nbits = dest_bits(a.nparts);
  uint32_t dst[kPartItems];
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint32_t i = it * kPartThreads + threadIdx.x;
    dst[it] = i < rem ? dest_of<NKEY>(a, base, i) : kMaxParts;
  }
  if (a.mask) {  // (applied after the key loads, so the mask and key loads overlap)
#pragma unroll
    for (int it = 0; it < kPartItems; it++) {
      const uint32_t i = it * kPartThreads + threadIdx.x;
      if (i < rem && !row_kept(a, base + i)) dst[it] = kMaxParts;
    }
  }
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const bool in = dst[it] < kMaxParts;
    const uint32_t peers = peers_of(dst[it], in, nbits);
    if (in && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&s_h[dst[it]], __popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < a.nparts) tile_hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s_h[threadIdx.x];
}

template <int NKEY>
__global__ void __launch_bounds__(kPartThreads, 4)
partition_scatter_kernel(const PartArgs a, const uint64_t *__restrict__ tile_off, uint64_t ntiles,
                         const uint64_t *__restrict__ dst_row,
                         const uint64_t *__restrict__ dst_cols) {
  __shared__ uint32_t s_wh[kWarps][kMaxParts];
  __shared__ uint64_t s_base[kMaxParts];
  __shared__ uint32_t *s_cols[kMaxParts * MAPSQ_MAX_COLS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kWarps * kMaxParts; i += kPartThreads) (&s_wh[0][0])[i] = 0;
  for (uint32_t i = tid; i < a.nparts * a.ncols; i += kPartThreads)
    s_cols[i] = reinterpret_cast<uint32_t *>(dst_cols[i]);
  const uint64_t wbase = (uint64_t)blockIdx.x * kPartTile + (uint64_t)warp * 32 * kPartItems;
  const uint32_t rem = rows_left(a.n, wbase, 32 * kPartItems);
  const int nbits = dest_bits(a.nparts);
  const uint32_t lt = lanemask_lt();
  // (1) destinations of the warp's rows (all key loads in flight together).  m[it] packs the
  // destination (bits 0-7, kMaxParts = no row) and, from step (2) on, the row's position above it.
  uint32_t m[kPartItems], lead[kPartItems];
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint32_t i = it * 32 + lane;
    m[it] = i < rem ? dest_of<NKEY>(a, wbase, i) : kMaxParts;
  }
  if (a.mask) {  // (applied after the key loads, so the mask and key loads overlap)
#pragma unroll
    for (int it = 0; it < kPartItems; it++) {
      const uint32_t i = it * 32 + lane;
      if (i < rem && !row_kept(a, wbase + i)) m[it] = kMaxParts;
    }
  }
  __syncthreads();
  // (2) per item: peers, rank among them, and the group leader's shared-memory fetch-add of the
  // warp's running count for that destination (stable: items in order, lanes in order).  The
  // atomics carry no register dependency from one item to the next.
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint32_t d = m[it];
    const bool in = d < kMaxParts;
    const uint32_t peers = peers_of(d, in, nbits);
    const int leader = __ffs(peers) - 1;
    lead[it] = 0;
    if (in && lane == leader) lead[it] = atomicAdd(&s_wh[warp][d], __popc(peers));
    m[it] = d | (__popc(peers & lt) << 8) | ((uint32_t)(leader & 31) << 16);
  }
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint32_t b = __shfl_sync(0xffffffffu, lead[it], (m[it] >> 16) & 31);
    m[it] = (m[it] & 0xffffu) + (b << 8);
  }
  __syncthreads();
  if (tid < (int)a.nparts) {
    uint32_t run = 0;
    for (int w = 0; w < kWarps; w++) {
      const uint32_t c = s_wh[w][tid];
      s_wh[w][tid] = run;
      run += c;
    }
    // this tile's first row for destination tid inside its arena block
    s_base[tid] = tile_off[(uint64_t)tid * ntiles + blockIdx.x] - tile_off[(uint64_t)tid * ntiles] +
                  dst_row[tid];
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kPartItems; it++)  // position within the tile's block for its destination
    if ((m[it] & 0xffu) < kMaxParts) m[it] += s_wh[warp][m[it] & 0xffu] << 8;
  // (3) destination: column c of destination d starts at dst_cols[d * ncols + c] (a local or an
  // NVLink peer pointer); the row lands at dst_row[d] + (its rank among this rank's rows for d).
  // Column-major: all kPartItems loads of a column are in flight before its stores.
  for (uint32_t c = 0; c < a.ncols; c++) {
    const uint32_t *__restrict__ src = a.in[c] + wbase + lane;
    uint32_t v[kPartItems];
#pragma unroll
    for (int it = 0; it < kPartItems; it++)  // (dropped rows: no load, only sectors with a kept row)
      v[it] = (m[it] & 0xffu) < kMaxParts ? __ldg(src + it * 32) : 0u;
#pragma unroll
    for (int it = 0; it < kPartItems; it++) {
      const uint32_t d = m[it] & 0xffu;
      if (d < kMaxParts) s_cols[d * a.ncols + c][s_base[d] + (m[it] >> 8)] = v[it];
    }
  }
}

}  // namespace

void launch_heavy_mask(const PartArgs &a, uint32_t *keep, uint32_t *bcast, cudaStream_t s) {
  const uint64_t nw = (a.n + 31) / 32;
  if (nw == 0) return;
  const unsigned g = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((nw * 32 + 255) / 256, 148 * 8));
  heavy_mask_kernel<<<g, 256, 0, s>>>(a, keep, bcast);
}

void launch_partition_hist(const PartArgs &a, uint32_t *tile_hist, uint64_t ntiles,
                           cudaStream_t s) {
  auto k = a.nkey == 1 ? partition_hist_kernel<1> : a.nkey == 2 ? partition_hist_kernel<2>
         : a.nkey == 3 ? partition_hist_kernel<3> : partition_hist_kernel<0>;
  k<<<(unsigned)ntiles, kPartThreads, 0, s>>>(a, tile_hist, ntiles);
}

void launch_partition_scatter(const PartArgs &a, const uint64_t *tile_off, uint64_t ntiles,
                              const uint64_t *dst_row, const uint64_t *dst_cols, cudaStream_t s) {
  auto k = a.nkey == 1 ? partition_scatter_kernel<1> : a.nkey == 2 ? partition_scatter_kernel<2>
         : a.nkey == 3 ? partition_scatter_kernel<3> : partition_scatter_kernel<0>;
  k<<<(unsigned)ntiles, kPartThreads, 0, s>>>(a, tile_off, ntiles, dst_row, dst_cols);
}

}  // namespace mapsq
