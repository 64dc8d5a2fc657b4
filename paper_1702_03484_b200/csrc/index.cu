// index.cu — predicate-range index: the triple table stably partitioned by
// predicate, so a pattern with a constant predicate reads only that predicate's row range.
//
// PAPER.md:154/164 leaves partial matching to the store (gStore) "in parallel"; an index on the
// predicate is the store-side structure that turns P(?s, p, ?o) into a range lookup
// ("select_index").  The build reuses the Map/sort machinery: words
// (p - p_lo) << ib | rowid sorted by the predicate bits only (stable), then one gather pass
// permutes s/p/o and records every predicate's first row, and one pass takes the per-predicate
// bounds of s and o (the partial-match tables' column bounds, exact).
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kIdxThreads = 256;
constexpr int kBoundsChunk = 16384;

__global__ void __launch_bounds__(kIdxThreads)
index_gather_kernel(const uint64_t *__restrict__ words, uint64_t n, uint32_t ib, uint32_t p_lo,
                    const uint32_t *__restrict__ s, const uint32_t *__restrict__ o,
                    uint32_t *__restrict__ s2, uint32_t *__restrict__ p2,
                    uint32_t *__restrict__ o2, uint32_t *__restrict__ head_p,
                    uint64_t *__restrict__ head_start, uint32_t *__restrict__ nheads,
                    uint32_t cap) {
  const uint64_t imask = (ib >= 64) ? ~0ull : ((1ull << ib) - 1ull);
  const uint64_t stride = (uint64_t)gridDim.x * kIdxThreads;
  for (uint64_t i = (uint64_t)blockIdx.x * kIdxThreads + threadIdx.x; i < n; i += stride) {
    const uint64_t w = __ldg(words + i);
    const uint64_t r = w & imask;
    const uint32_t key = (uint32_t)(w >> ib);
    s2[i] = __ldg(s + r);
    o2[i] = __ldg(o + r);
    p2[i] = p_lo + key;
    if (i == 0 || (uint32_t)(__ldg(words + i - 1) >> ib) != key) {
      const uint32_t slot = atomicAdd(nheads, 1u);
      if (slot < cap) {
        head_p[slot] = p_lo + key;
        head_start[slot] = i;
      }
    }
  }
}

// Per-run min/max of s2 and o2.  starts[0..nruns] ascending (starts[nruns] = n).
// bounds layout: [slo | olo | shi | ohi], nruns each.
__global__ void __launch_bounds__(kIdxThreads)
index_bounds_kernel(const uint32_t *__restrict__ s2, const uint32_t *__restrict__ o2, uint64_t n,
                    const uint64_t *__restrict__ starts, uint32_t nruns,
                    uint32_t *__restrict__ bounds) {
  const uint64_t c0 = (uint64_t)blockIdx.x * kBoundsChunk;
  const uint64_t c1 = c0 + kBoundsChunk < n ? c0 + kBoundsChunk : n;
  uint64_t i = c0 + threadIdx.x;
  if (i >= c1) return;
  // run containing row i: the last run with starts[run] <= i
  uint32_t lo = 0, hi = nruns;  // invariant: starts[lo] <= i < starts[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (starts[mid] <= i) lo = mid; else hi = mid;
  }
  uint32_t run = lo;
  uint64_t next = starts[run + 1];
  uint32_t smin = 0xffffffffu, smax = 0, omin = 0xffffffffu, omax = 0;
  auto flush = [&]() {
    if (smin <= smax) {
      atomicMin(bounds + run, smin);
      atomicMin(bounds + nruns + run, omin);
      atomicMax(bounds + 2 * nruns + run, smax);
      atomicMax(bounds + 3 * nruns + run, omax);
    }
    smin = omin = 0xffffffffu;
    smax = omax = 0;
  };
  for (; i < c1; i += kIdxThreads) {
    while (i >= next) {
      flush();
      run++;
      next = starts[run + 1];
    }
    const uint32_t a = __ldg(s2 + i), b = __ldg(o2 + i);
    smin = min(smin, a);
    smax = max(smax, a);
    omin = min(omin, b);
    omax = max(omax, b);
  }
  flush();
}

}  // namespace

void launch_index_gather(const uint64_t *words, uint64_t n, uint32_t ib, uint32_t p_lo,
                         const uint32_t *s, const uint32_t *o, uint32_t *s2, uint32_t *p2,
                         uint32_t *o2, uint32_t *head_p, uint64_t *head_start, uint32_t *nheads,
                         uint32_t cap, cudaStream_t st) {
  const int g = (int)std::max<uint64_t>(1, std::min<uint64_t>(ceil_div(n, kIdxThreads), 148 * 16));
  index_gather_kernel<<<g, kIdxThreads, 0, st>>>(words, n, ib, p_lo, s, o, s2, p2, o2, head_p,
                                                 head_start, nheads, cap);
}

void launch_index_bounds(const uint32_t *s2, const uint32_t *o2, uint64_t n,
                         const uint64_t *starts, uint32_t nruns, uint32_t *bounds,
                         cudaStream_t st) {
  const uint64_t g = ceil_div(n, kBoundsChunk);
  index_bounds_kernel<<<(unsigned)g, kIdxThreads, 0, st>>>(s2, o2, n, starts, nruns, bounds);
}

}  // namespace mapsq
