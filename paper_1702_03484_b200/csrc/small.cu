// small.cu — Algorithm 1 for tiny joins in ONE kernel launch (SURVEY §8 rows a3-a6 on inputs of
// at most kSmallMaxRows rows; C1 is 720 x 320).
//
// The same method and the same result as the multi-kernel path, in one CTA: Map (Alg. 1 l.1-4,
// PAPER.md:122-125) packs the words key' << ib | rowid (rowid >= n1 means RIGHT) into shared
// memory; Sort (l.5) orders them — a stable LSD radix sort over the key bits in shared
// memory, so the order is the (key', LEFT before RIGHT, rowid) order the multi-kernel path produces;
// ReduceDuplicate (l.6-11) finds each key's LEFT/RIGHT split, scans nL * nR and writes
// every pair in (key', Tp1 row, Tp2 row) order.  A join this small is launch- and sync-bound on
// the multi-kernel path (~10 launches and two blocking reads); here it is one launch and one read
// of |RS|.  The output is written into a caller allocation of `cap` rows; if |RS| > cap the kernel
// writes only |RS| and the host runs the regular path.
#include "internal.cuh"

namespace mapsq {
namespace {

constexpr int kSmallThreads = 1024;

__global__ void __launch_bounds__(kSmallThreads)
small_join_kernel(const PackArgs pa, const ExpandArgs ea, uint64_t cap,
                  unsigned long long *__restrict__ m_out) {
  extern __shared__ __align__(16) unsigned char smem[];
  const uint32_t n1 = (uint32_t)pa.n1, n = (uint32_t)(pa.n1 + pa.n2);
  const uint32_t gcap = (n / 2 + 3) & ~1u;                            // groups (<= n / 2) + 1, even
  uint64_t *w0 = reinterpret_cast<uint64_t *>(smem);                  // n words
  uint64_t *w1 = w0 + n;                                              // n words (sort buffer)
  uint16_t *rank = reinterpret_cast<uint16_t *>(w1 + n);              // n (padded to 8 B)
  uint32_t *g_start = reinterpret_cast<uint32_t *>(smem + 16ull * n + ((2ull * n + 7) & ~7ull));
  uint32_t *g_split = g_start + gcap;
  uint32_t *g_end = g_split + gcap;
  uint64_t *g_off = reinterpret_cast<uint64_t *>(g_end + gcap);       // (8 B aligned: 3 * gcap even)
  __shared__ uint32_t s_cnt[kSmallThreads / 32][256];                 // per-warp digit counts
  __shared__ uint32_t s_wsum[kSmallThreads / 32];
  __shared__ uint32_t s_ng;
  const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- Map
  for (uint32_t i = tid; i < n; i += kSmallThreads) {
    const bool right = i >= n1;
    uint64_t key = 0;
    for (uint32_t c = 0; c < pa.nkey; c++) {
      const uint32_t v = right ? pa.key2[c][i - n1] : pa.key1[c][i];
      key |= (uint64_t)(v - pa.lo[c]) << pa.shift[c];
    }
    w0[i] = (key << pa.ib) | i;
  }
  __syncthreads();
  // ---- Sort: stable LSD radix over the kb key bits, 8-bit digits, in shared memory (the words
  // are distinct, so the sorted order is the unique (key', LEFT before RIGHT, rowid) order the
  // multi-kernel path produces).  Warp q ranks the contiguous chunk [q E, (q + 1) E) of the words
  // in rounds of 32 lanes (match.any peers; the highest peer bumps the warp's digit count), so
  // ranks follow the input order within a digit; a block scan over (digit, warp) gives offsets.
  const uint32_t E = (n + 31) / 32;
  const uint32_t lt = lanemask_lt();
  uint64_t *w = w0, *wt = w1;
  for (uint32_t sh = pa.ib; sh < pa.ib + pa.kb; sh += 8) {
    const uint32_t dm = (1u << min(8u, pa.ib + pa.kb - sh)) - 1u;
    for (uint32_t i = tid; i < (kSmallThreads / 32) * 256; i += kSmallThreads) (&s_cnt[0][0])[i] = 0;
    __syncthreads();
    const uint32_t c0 = warp * E, c1 = min(n, c0 + E);
    for (uint32_t b = c0; b < c1; b += 32) {
      const uint32_t e = b + lane;
      const bool in = e < c1;
      const uint32_t d = in ? (uint32_t)(w[e] >> sh) & dm : 0x100u;
      const uint32_t peers = __match_any_sync(0xffffffffu, d);
      const uint32_t before = in ? s_cnt[warp][d] : 0u;
      __syncwarp();
      if (in && lane == 31 - __clz(peers)) s_cnt[warp][d] = before + __popc(peers);
      __syncwarp();
      if (in) rank[e] = (uint16_t)(before + __popc(peers & lt));
    }
    __syncthreads();
    if (tid < 256) {  // digit tid: exclusive offsets over (digit, warp)
      uint32_t tot = 0;
#pragma unroll 8
      for (int q = 0; q < kSmallThreads / 32; q++) tot += s_cnt[q][tid];
      uint32_t x = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= (uint32_t)o) x += y;
      }
      if (lane == 31) s_wsum[warp] = x;
      asm volatile("bar.sync 1, 256;");
      uint32_t run = x - tot;
      for (uint32_t q = 0; q < warp; q++) run += s_wsum[q];
#pragma unroll 8
      for (int q = 0; q < kSmallThreads / 32; q++) {
        const uint32_t c = s_cnt[q][tid];
        s_cnt[q][tid] = run;
        run += c;
      }
    }
    __syncthreads();
    for (uint32_t e = tid; e < n; e += kSmallThreads) {
      const uint64_t x = w[e];
      wt[s_cnt[e / E][(uint32_t)(x >> sh) & dm] + rank[e]] = x;
    }
    __syncthreads();
    uint64_t *t = w;
    w = wt;
    wt = t;
  }
  // ---- ReduceDuplicate 1: splits (a LEFT word followed by a RIGHT word of the same key), in key
  // order; block scan of the split flags gives each group's slot
  const uint32_t per = (n + kSmallThreads - 1) / kSmallThreads;  // contiguous chunk per thread
  const uint32_t lo = tid * per, hi = min(n, lo + per);
  auto is_split = [&](uint32_t i) -> bool {
    if (i == 0 || i >= n) return false;
    const uint64_t a = w[i - 1], b = w[i];
    return ((a ^ b) >> pa.ib) == 0 && (uint32_t)(a & ((1ull << pa.ib) - 1)) < n1 &&
           (uint32_t)(b & ((1ull << pa.ib) - 1)) >= n1;
  };
  uint32_t cnt = 0;
  for (uint32_t i = lo; i < hi; i++) cnt += is_split(i);
  uint32_t x = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= (uint32_t)o) x += y;
  }
  if (lane == 31) s_wsum[warp] = x;
  __syncthreads();
  uint32_t pre = 0, tot = 0;
  for (int q = 0; q < kSmallThreads / 32; q++) {
    if ((uint32_t)q < warp) pre += s_wsum[q];
    tot += s_wsum[q];
  }
  uint32_t slot = pre + x - cnt;
  for (uint32_t i = lo; i < hi; i++) {
    if (!is_split(i)) continue;
    const uint64_t k = w[i] >> pa.ib;
    uint32_t st = i, en = i;
    while (st > 0 && (w[st - 1] >> pa.ib) == k) st--;
    while (en < n && (w[en] >> pa.ib) == k) en++;
    g_start[slot] = st;
    g_split[slot] = i;
    g_end[slot] = en;
    g_off[slot] = (uint64_t)(i - st) * (en - i);
    slot++;
  }
  if (tid == 0) s_ng = tot;
  __syncthreads();
  const uint32_t ng = s_ng;
  // ---- K5: exclusive scan of nL * nR (serial per thread chunk + block scan of chunk sums)
  const uint32_t gper = (ng + kSmallThreads - 1) / kSmallThreads;
  const uint32_t glo = min(ng, tid * gper), ghi = min(ng, glo + gper);
  uint64_t run = 0;
  for (uint32_t g = glo; g < ghi; g++) run += g_off[g];
  __syncthreads();  // (s_wsum reuse)
  // block scan of 64-bit chunk sums through warp shuffles of two halves
  unsigned long long xs = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(0xffffffffu, xs, o);
    if (lane >= (uint32_t)o) xs += y;
  }
  __shared__ unsigned long long s_wsum64[kSmallThreads / 32];
  if (lane == 31) s_wsum64[warp] = xs;
  __syncthreads();
  unsigned long long base = 0, m = 0;
  for (int q = 0; q < kSmallThreads / 32; q++) {
    if ((uint32_t)q < warp) base += s_wsum64[q];
    m += s_wsum64[q];
  }
  base += xs - run;
  for (uint32_t g = glo; g < ghi; g++) {
    const uint64_t c = g_off[g];
    g_off[g] = base;
    base += c;
  }
  if (tid == 0) *m_out = m;
  __syncthreads();
  if (m > cap || m == 0) return;  // too large for the allocation: the host takes the regular path
  g_off[ng] = m;
  __syncthreads();
  // ---- ReduceDuplicate 2: row r of RS -> its group (binary search), (li, ri), gathers
  const uint32_t nout = ea.nkey + ea.nrest1 + ea.nrest2;
  const uint64_t idx_mask = (1ull << pa.ib) - 1;
  for (uint64_t r = tid; r < m; r += kSmallThreads) {
    uint32_t a = 0, b = ng - 1;
    while (a < b) {
      const uint32_t mid = (a + b + 1) >> 1;
      if (g_off[mid] <= r) a = mid; else b = mid - 1;
    }
    const uint32_t st = g_start[a], sp = g_split[a], en = g_end[a];
    const uint64_t nR = en - sp, local = r - g_off[a];
    const uint32_t li = st + (uint32_t)(local / nR), ri = sp + (uint32_t)(local % nR);
    const uint64_t lw = w[li], rw = w[ri];
    const uint64_t key = lw >> pa.ib;
    const uint32_t lidx = (uint32_t)(lw & idx_mask), ridx = (uint32_t)((rw & idx_mask) - n1);
    for (uint32_t c = 0; c < nout; c++) {
      uint32_t v;
      if (c < ea.nkey)
        v = (uint32_t)(key >> ea.key_shift[c] & ea.key_mask[c]) + ea.key_lo[c];
      else if (c < ea.nkey + ea.nrest1)
        v = __ldg(ea.rest1[c - ea.nkey] + lidx);
      else
        v = __ldg(ea.rest2[c - ea.nkey - ea.nrest1] + ridx);
      ea.out[c][r] = v;
    }
  }
}

}  // namespace

size_t small_join_smem(uint64_t n) {
  const uint64_t gcap = (n / 2 + 3) & ~1ull;
  return 16 * n + ((2 * n + 7) & ~7ull) + 3 * gcap * 4 + gcap * 8;
}

void launch_small_join(const PackArgs &pa, const ExpandArgs &ea, uint64_t cap,
                       unsigned long long *m_out, cudaStream_t s) {
  const size_t smem = small_join_smem(pa.n1 + pa.n2);
  set_smem_limit((const void *)small_join_kernel, small_join_smem(kSmallMaxRows));
  small_join_kernel<<<1, kSmallThreads, smem, s>>>(pa, ea, cap, m_out);
}

}  // namespace mapsq
