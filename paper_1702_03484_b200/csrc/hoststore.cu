// hoststore.cu — compressed host-resident store for the end-to-end path (SURVEY §8 row f1's host
// mirror, DESIGN §5.9 / §6).
//
// The paper's split leaves the store on the host and joins on the GPU, so
// an end-to-end query is bound by moving the touched predicate ranges over PCIe.  The mirror keeps
// every column of every predicate range as frame-of-reference blocks of 1024 values — a block
// stores its minimum and the offsets from it in the fewest bits that hold them — which the GPU
// expands after the copy.  LUBM's ranges are generated entity by entity, so a block's subjects
// (and mostly its objects) lie in a narrow ID interval: C5's touched ranges shrink from 2.8 GB to
// well under half.  Lossless: the expanded columns equal the originals bit for bit.
//
// Segment layout (one per range and column, identical on host and device, in 32-bit words):
//   base[nb] | bits[nb] | woff[nb + 1] | payload
// with nb = ceil(n / 1024); block b's value j (j < 1024) is bits[b] bits at bit offset j * bits[b]
// of payload[woff[b] ..], plus base[b].
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr uint32_t kFor = 1024;  // values per block
constexpr int kForWarps = 8;

// per block: minimum and bit width of (max - min)
__global__ void __launch_bounds__(32 * kForWarps)
for_stats_kernel(const uint32_t *__restrict__ col, uint64_t n, uint32_t *__restrict__ base,
                 uint32_t *__restrict__ bits) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nb = (n + kFor - 1) / kFor;
  for (uint64_t b = (uint64_t)blockIdx.x * kForWarps + (threadIdx.x >> 5); b < nb;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint64_t b0 = b * kFor;
    uint32_t lo = 0xffffffffu, hi = 0;
#pragma unroll 8
    for (uint32_t t = 0; t < kFor / 32; t++) {
      const uint64_t j = b0 + t * 32 + lane;
      if (j < n) {
        const uint32_t v = __ldcs(col + j);
        lo = min(lo, v);
        hi = max(hi, v);
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    if (lane == 0) {
      base[b] = lo;
      bits[b] = hi == lo ? 0u : 32u - __clz(hi - lo);
    }
  }
}

// per block: pack (v - base) into bits[b]-bit fields at payload[woff[b] ..] (shared-memory staging
// of the block's payload words, then coalesced stores)
__global__ void __launch_bounds__(32 * kForWarps)
for_pack_kernel(const uint32_t *__restrict__ col, uint64_t n, const uint32_t *__restrict__ base,
                const uint32_t *__restrict__ bits, const uint32_t *__restrict__ woff,
                uint32_t *__restrict__ payload) {
  __shared__ uint32_t s_w[kForWarps][kFor + 1];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *w = s_w[warp];
  const uint64_t nb = (n + kFor - 1) / kFor;
  for (uint64_t b = (uint64_t)blockIdx.x * kForWarps + warp; b < nb;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint32_t nbits = bits[b], lo = base[b];
    const uint32_t words = woff[b + 1] - woff[b];
    for (uint32_t i = lane; i < words; i += 32) w[i] = 0;
    __syncwarp();
    const uint64_t b0 = b * kFor;
    if (nbits)
      for (uint32_t t = 0; t < kFor / 32; t++) {
        const uint32_t j = t * 32 + lane;
        if (b0 + j >= n) break;
        const uint32_t v = __ldcs(col + b0 + j) - lo;
        const uint64_t off = (uint64_t)j * nbits;
        const uint32_t wi = (uint32_t)(off >> 5), sh = (uint32_t)(off & 31);
        atomicOr(w + wi, v << sh);
        if (sh + nbits > 32) atomicOr(w + wi + 1, v >> (32 - sh));
      }
    __syncwarp();
    for (uint32_t i = lane; i < words; i += 32) payload[woff[b] + i] = w[i];
    __syncwarp();
  }
}

// expand a segment (device copy) into n values at out[0 ..); one warp per block
__global__ void __launch_bounds__(32 * kForWarps)
for_unpack_kernel(const uint32_t *__restrict__ seg, uint64_t n, uint32_t *__restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nb = (n + kFor - 1) / kFor;
  const uint32_t *base = seg, *bits = seg + nb, *woff = seg + 2 * nb;
  const uint32_t *payload = seg + 3 * nb + 1;
  for (uint64_t b = (uint64_t)blockIdx.x * kForWarps + (threadIdx.x >> 5); b < nb;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint32_t nbits = __ldg(bits + b), lo = __ldg(base + b);
    const uint32_t *p = payload + __ldg(woff + b);
    const uint32_t mask = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
    const uint64_t b0 = b * kFor;
#pragma unroll 8
    for (uint32_t t = 0; t < kFor / 32; t++) {
      const uint32_t j = t * 32 + lane;
      if (b0 + j >= n) break;
      uint32_t v = 0;
      if (nbits) {
        const uint64_t off = (uint64_t)j * nbits;
        const uint32_t wi = (uint32_t)(off >> 5), sh = (uint32_t)(off & 31);
        uint64_t two = __ldg(p + wi);
        if (sh + nbits > 32) two |= (uint64_t)__ldg(p + wi + 1) << 32;
        v = (uint32_t)(two >> sh) & mask;
      }
      __stcs(out + b0 + j, v + lo);
    }
  }
}

int for_grid(uint64_t n) {
  const uint64_t nb = (n + kFor - 1) / kFor;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((nb + kForWarps - 1) / kForWarps, 148 * 16));
}

}  // namespace

uint64_t for_blocks(uint64_t n) { return (n + kFor - 1) / kFor; }
uint64_t for_block_words(uint32_t bits) { return ((uint64_t)kFor * bits + 31) / 32; }

void launch_for_stats(const uint32_t *col, uint64_t n, uint32_t *base, uint32_t *bits,
                      cudaStream_t s) {
  if (n) for_stats_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(col, n, base, bits);
}

void launch_for_pack(const uint32_t *col, uint64_t n, const uint32_t *base, const uint32_t *bits,
                     const uint32_t *woff, uint32_t *payload, cudaStream_t s) {
  if (n) for_pack_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(col, n, base, bits, woff, payload);
}

void launch_for_unpack(const uint32_t *seg, uint64_t n, uint32_t *out, cudaStream_t s) {
  if (n) for_unpack_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(seg, n, out);
}

}  // namespace mapsq
