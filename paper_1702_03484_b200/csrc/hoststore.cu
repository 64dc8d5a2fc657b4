// hoststore.cu — compressed host-resident store for the end-to-end path (SURVEY §8 row f1's host
// mirror, DESIGN §5.9 / §6).
//
// The paper's split leaves the store on the host and joins on the GPU, so
// an end-to-end query is bound by moving the touched predicate ranges over PCIe.  The mirror keeps
// every column of every predicate range as frame-of-reference blocks of 128 values — a block
// stores its minimum and the offsets from it in the fewest bits that hold them — which the GPU
// expands after the copy.  LUBM's ranges are generated entity by entity, so a block's subjects
// (and mostly its objects) lie in a narrow ID interval: C5's touched ranges shrink from 2.8 GB to
// well under half.  Lossless: the expanded columns equal the originals bit for bit.
//
// Two block codings, whichever packs narrower: plain frame of reference (value = base + f_j) and
// delta frame of reference for sorted-ish columns (subjects of a range come entity by entity:
// value_j = base + j * dmin + sum_{i <= j} f_i, the deltas' minimum dmin taken out; mod 2^32).
// Segment layout (one per range and column, identical on host and device, in 32-bit words):
//   base[nb] | mode_bits[nb] | dmin[nb] | woff[nb + 1] | payload
// with nb = ceil(n / 128); f_j of block b is (mode_bits[b] & 63) bits at bit offset j * bits of
// payload[woff[b] ..]; bit 31 of mode_bits marks the delta coding.
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr uint32_t kFor = 128;  // values per block (LUBM: 128 packs C5's ranges ~1.7x tighter than 1024)
constexpr uint32_t kPer = kFor / 32;  // values per lane
constexpr int kForWarps = 8;

// per block: the narrower coding — frame of reference (min, bits of max - min) or deltas (first
// value, dmin, bits of max - min of the deltas)
__global__ void __launch_bounds__(32 * kForWarps)
for_stats_kernel(const uint32_t *__restrict__ col, uint64_t n, uint32_t *__restrict__ base,
                 uint32_t *__restrict__ bits, uint32_t *__restrict__ dmin) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nb = (n + kFor - 1) / kFor;
  for (uint64_t b = (uint64_t)blockIdx.x * kForWarps + (threadIdx.x >> 5); b < nb;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint64_t b0 = b * kFor;
    uint32_t lo = 0xffffffffu, hi = 0, dlo = 0xffffffffu, dhi = 0;
#pragma unroll
    for (uint32_t t = 0; t < kPer; t++) {
      const uint64_t j = b0 + t * 32 + lane;
      if (j < n) {
        const uint32_t v = __ldcs(col + j);
        lo = min(lo, v);
        hi = max(hi, v);
        if (j > b0) {
          const uint32_t d = v - __ldg(col + j - 1);
          dlo = min(dlo, d);
          dhi = max(dhi, d);
        }
      }
    }
    lo = __reduce_min_sync(0xffffffffu, lo);
    hi = __reduce_max_sync(0xffffffffu, hi);
    dlo = __reduce_min_sync(0xffffffffu, dlo);
    dhi = __reduce_max_sync(0xffffffffu, dhi);
    if (lane == 0) {
      const uint32_t fb = hi == lo ? 0u : 32u - __clz(hi - lo);
      const bool has_d = dlo <= dhi;  // (a block of one value has no delta)
      const uint32_t db = !has_d || dhi == dlo ? 0u : 32u - __clz(dhi - dlo);
      if (has_d && db < fb) {
        base[b] = __ldg(col + b0);
        bits[b] = db | 0x80000000u;
        dmin[b] = dlo;
      } else {
        base[b] = lo;
        bits[b] = fb;
        dmin[b] = 0;
      }
    }
  }
}

// per block: pack (v - base) into bits[b]-bit fields at payload[woff[b] ..] (shared-memory staging
// of the block's payload words, then coalesced stores)
__global__ void __launch_bounds__(32 * kForWarps)
for_pack_kernel(const uint32_t *__restrict__ col, uint64_t n, const uint32_t *__restrict__ base,
                const uint32_t *__restrict__ bits, const uint32_t *__restrict__ dmin,
                const uint32_t *__restrict__ woff, uint32_t *__restrict__ payload) {
  __shared__ uint32_t s_w[kForWarps][kFor + 1];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *w = s_w[warp];
  const uint64_t nb = (n + kFor - 1) / kFor;
  for (uint64_t b = (uint64_t)blockIdx.x * kForWarps + warp; b < nb;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint32_t mb = bits[b], nbits = mb & 63u, lo = base[b], dm = dmin[b];
    const bool delta = mb >> 31;
    const uint32_t words = woff[b + 1] - woff[b];
    for (uint32_t i = lane; i < words; i += 32) w[i] = 0;
    __syncwarp();
    const uint64_t b0 = b * kFor;
    if (nbits)
      for (uint32_t t = 0; t < kFor / 32; t++) {
        const uint32_t j = t * 32 + lane;
        if (b0 + j >= n) break;
        const uint32_t x = __ldg(col + b0 + j);
        const uint32_t v = delta ? (j ? x - __ldg(col + b0 + j - 1) - dm : 0u) : x - lo;
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

// expand a segment (device copy) into n values at out[0 ..); one warp per block.  Frame of
// reference: lane-strided values (coalesced stores); deltas: each lane decodes kPer consecutive
// values, prefix-sums them and adds the warp's exclusive scan of the lane totals.
// (blocks [b0, b1) only: a range expanded chunk by chunk as its copies land)
__global__ void __launch_bounds__(32 * kForWarps)
for_unpack_kernel(const uint32_t *__restrict__ seg, uint64_t n, uint64_t b0, uint64_t b1,
                  uint32_t *__restrict__ out) {
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nb = (n + kFor - 1) / kFor;
  const uint32_t *base = seg, *bits = seg + nb, *dmin = seg + 2 * nb, *woff = seg + 3 * nb;
  const uint32_t *payload = seg + 4 * nb + 1;
  for (uint64_t b = b0 + (uint64_t)blockIdx.x * kForWarps + (threadIdx.x >> 5); b < b1;
       b += (uint64_t)gridDim.x * kForWarps) {
    const uint32_t mb = __ldg(bits + b), nbits = mb & 63u, lo = __ldg(base + b);
    const uint32_t *p = payload + __ldg(woff + b);
    const uint32_t mask = nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
    const uint64_t b0 = b * kFor;
    auto field = [&](uint32_t j) -> uint32_t {
      if (!nbits) return 0u;
      const uint64_t off = (uint64_t)j * nbits;
      const uint32_t wi = (uint32_t)(off >> 5), sh = (uint32_t)(off & 31);
      uint64_t two = __ldg(p + wi);
      if (sh + nbits > 32) two |= (uint64_t)__ldg(p + wi + 1) << 32;
      return (uint32_t)(two >> sh) & mask;
    };
    if (!(mb >> 31)) {
#pragma unroll 8
      for (uint32_t t = 0; t < kFor / 32; t++) {
        const uint32_t j = t * 32 + lane;
        if (b0 + j >= n) break;
        __stcs(out + b0 + j, field(j) + lo);
      }
      continue;
    }
    const uint32_t dm = __ldg(dmin + b);
    uint32_t v[kPer], run = 0;
#pragma unroll
    for (uint32_t t = 0; t < kPer; t++) {
      const uint32_t j = lane * kPer + t;
      run += j ? field(j) + dm : 0u;
      v[t] = run;
    }
    uint32_t x = run;  // inclusive scan of the lane totals
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= (uint32_t)o) x += y;
    }
    const uint32_t add = lo + x - run;
#pragma unroll
    for (uint32_t t = 0; t < kPer; t++) {
      const uint64_t j = b0 + lane * kPer + t;
      if (j < n) out[j] = v[t] + add;
    }
  }
}

int for_grid(uint64_t n) {
  const uint64_t nb = (n + kFor - 1) / kFor;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>((nb + kForWarps - 1) / kForWarps, 148 * 16));
}

}  // namespace

uint64_t for_blocks(uint64_t n) { return (n + kFor - 1) / kFor; }
uint64_t for_block_words(uint32_t bits) { return ((uint64_t)kFor * (bits & 63u) + 31) / 32; }

void launch_for_stats(const uint32_t *col, uint64_t n, uint32_t *base, uint32_t *bits,
                      uint32_t *dmin, cudaStream_t s) {
  if (n) for_stats_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(col, n, base, bits, dmin);
}

void launch_for_pack(const uint32_t *col, uint64_t n, const uint32_t *base, const uint32_t *bits,
                     const uint32_t *dmin, const uint32_t *woff, uint32_t *payload,
                     cudaStream_t s) {
  if (n)
    for_pack_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(col, n, base, bits, dmin, woff, payload);
}

void launch_for_unpack(const uint32_t *seg, uint64_t n, uint32_t *out, cudaStream_t s) {
  if (n) for_unpack_kernel<<<for_grid(n), 32 * kForWarps, 0, s>>>(seg, n, 0, for_blocks(n), out);
}

void launch_for_unpack_blocks(const uint32_t *seg, uint64_t n, uint64_t b0, uint64_t b1,
                              uint32_t *out, cudaStream_t s) {
  if (b1 > b0)
    for_unpack_kernel<<<for_grid((b1 - b0) * kFor), 32 * kForWarps, 0, s>>>(seg, n, b0, b1, out);
}

// (debugging aid, MAPSQ_DEBUG_COPY_DELAY: holds a stream for `us` microseconds)
__global__ void delay_kernel(uint64_t ns) {
  uint64_t t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    __nanosleep(1000);
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}
void launch_delay_us(uint32_t us, cudaStream_t s) { delay_kernel<<<1, 1, 0, s>>>(1000ull * us); }

}  // namespace mapsq
