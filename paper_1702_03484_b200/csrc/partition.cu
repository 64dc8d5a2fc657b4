// partition.cu — K8: hash partition of a partial-match table on its join key (SURVEY §8 row e),
// fused with the exchange: the scatter stores every row straight into its destination rank's
// receive arena through NVLink peer pointers (one kernel does the partition and the all-to-all).
//
// An equi-join decomposes over disjoint key sets, so on G GPUs each rank sends every row to
// rank dest = fmix32(fold(key)) mod G and then runs the local sort-join on what it receives.
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

__device__ __forceinline__ uint32_t dest_of(const PartArgs &a, uint64_t i) {
  uint32_t h = 0x811c9dc5u;
  for (uint32_t c = 0; c < a.nkey; c++) h = (h ^ __ldg(a.key[c] + i)) * 0x01000193u;
  return fmix32(h) % a.nparts;
}

__global__ void __launch_bounds__(kPartThreads)
partition_hist_kernel(const PartArgs a, uint32_t *__restrict__ tile_hist, uint64_t ntiles) {
  __shared__ uint32_t s_h[kMaxParts];
  if (threadIdx.x < kMaxParts) s_h[threadIdx.x] = 0;
  __syncthreads();
  const uint64_t base = (uint64_t)blockIdx.x * kPartTile;
  const uint32_t lane = threadIdx.x & 31;
#pragma unroll 4
  for (int it = 0; it < kPartItems; it++) {
    const uint64_t i = base + (uint64_t)it * kPartThreads + threadIdx.x;
    const bool in = i < a.n;
    const uint32_t d = in ? dest_of(a, i) : 0xffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    if (in && lane == (uint32_t)(__ffs(peers) - 1)) atomicAdd(&s_h[d], __popc(peers));
  }
  __syncthreads();
  if (threadIdx.x < a.nparts) tile_hist[(uint64_t)threadIdx.x * ntiles + blockIdx.x] = s_h[threadIdx.x];
}

__global__ void __launch_bounds__(kPartThreads)
partition_scatter_kernel(const PartArgs a, const uint64_t *__restrict__ tile_off, uint64_t ntiles,
                         const uint64_t *__restrict__ dst_row,
                         const uint64_t *__restrict__ dst_cols) {
  __shared__ uint32_t s_wh[kWarps][kMaxParts];
  __shared__ uint64_t s_base[kMaxParts];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < kWarps * kMaxParts; i += kPartThreads) (&s_wh[0][0])[i] = 0;
  __syncthreads();
  const uint64_t wbase = (uint64_t)blockIdx.x * kPartTile + (uint64_t)warp * 32 * kPartItems;
  uint32_t dst[kPartItems], rank[kPartItems];
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    const bool in = i < a.n;
    const uint32_t d = in ? dest_of(a, i) : 0xffffu;
    const uint32_t peers = __match_any_sync(0xffffffffu, d);
    const int leader = __ffs(peers) - 1;
    uint32_t b = 0;
    if (in && lane == leader) {
      b = s_wh[warp][d];
      s_wh[warp][d] = b + __popc(peers);
    }
    b = __shfl_sync(0xffffffffu, b, leader);
    dst[it] = d;
    rank[it] = b + __popc(peers & lt);
    __syncwarp();
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
  // destination: column c of destination d starts at dst_cols[d * ncols + c] (a local or an
  // NVLink peer pointer); the row lands at dst_row[d] + (its rank among this rank's rows for d)
#pragma unroll
  for (int it = 0; it < kPartItems; it++) {
    const uint64_t i = wbase + (uint64_t)it * 32 + lane;
    if (i >= a.n) continue;
    const uint32_t d = dst[it];
    const uint64_t pos = s_base[d] + s_wh[warp][d] + rank[it];
    for (uint32_t c = 0; c < a.ncols; c++) {
      uint32_t *col = reinterpret_cast<uint32_t *>(dst_cols[d * a.ncols + c]);
      col[pos] = __ldg(a.in[c] + i);
    }
  }
}

}  // namespace

void launch_partition_hist(const PartArgs &a, uint32_t *tile_hist, uint64_t ntiles,
                           cudaStream_t s) {
  partition_hist_kernel<<<(unsigned)ntiles, kPartThreads, 0, s>>>(a, tile_hist, ntiles);
}

void launch_partition_scatter(const PartArgs &a, const uint64_t *tile_off, uint64_t ntiles,
                              const uint64_t *dst_row, const uint64_t *dst_cols, cudaStream_t s) {
  partition_scatter_kernel<<<(unsigned)ntiles, kPartThreads, 0, s>>>(a, tile_off, ntiles, dst_row,
                                                                     dst_cols);
}

}  // namespace mapsq
