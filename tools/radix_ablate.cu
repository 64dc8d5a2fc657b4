// radix_ablate.cu — developer micro-benchmark (not product code): times the one-sweep digit
// pass of paper_1702_03484_b200/csrc/radix.cu against ablated variants to locate its limiter.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/radix_ablate.cu
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <string>

#include "../paper_1702_03484_b200/csrc/radix.cu"

using namespace mapsq;
namespace mapsq {
void set_smem_limit(const void *kernel, size_t bytes) {  // (defined in api.cu for the library)
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}
// Persistent one-sweep digit pass (P64 words).  Each CTA loops over tiles claimed in order from
// the atomic counter; while it ranks / looks back / scatters tile t, the TMA engine already
// streams the NEXT claimed tile into the other shared-memory buffer (cp.async.bulk + mbarrier),
// so DRAM reads stay in flight through the rank and look-back phases that idled the
// one-tile-per-CTA version.  Claiming in order keeps the look-back deadlock free: the smallest
// unfinished claimed tile only waits on finished tiles.
constexpr int kTmaCtasPerSm = 2;
constexpr size_t kTmaSmem = 3ull * kSortTile * sizeof(uint64_t);

__global__ void __launch_bounds__(kSortThreads, kTmaCtasPerSm)
radix_pass_tma_kernel(const uint64_t *__restrict__ kin, uint64_t *__restrict__ kout, uint64_t n,
                      uint32_t shift, uint32_t bits, const uint32_t *__restrict__ hist_pass,
                      uint64_t *__restrict__ status, uint32_t *__restrict__ tile_counter) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t *s_out = reinterpret_cast<uint64_t *>(smem_raw + 2 * kSortTile * sizeof(uint64_t));
  __shared__ __align__(8) uint64_t s_bar[2];
  __shared__ uint32_t s_warp_hist[kWarps][kRadix];
  __shared__ uint32_t s_digit_start[kRadix];
  __shared__ uint64_t s_global_base[kRadix];
  __shared__ uint32_t s_wsum[kWarps];
  __shared__ uint32_t s_tile[2];

  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint64_t ntiles = ceil_div(n, kSortTile);
  const uint32_t dmask = (1u << bits) - 1u;
  const uint32_t wslice = warp * 32 * kSortItems;
  const uint32_t lt = lanemask_lt();

  auto issue = [&](uint32_t t, int buf) {  // tid 0 only
    const uint64_t base = (uint64_t)t * kSortTile;
    const uint64_t rem = n - base;
    const uint32_t cnt = rem < (uint64_t)kSortTile ? (uint32_t)rem : (uint32_t)kSortTile;
    const uint32_t bulk = cnt & ~1u;  // 16 B granularity
    uint64_t *dst = reinterpret_cast<uint64_t *>(smem_raw + (size_t)buf * kSortTile * sizeof(uint64_t));
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&s_bar[buf], bulk * 8u);
    if (bulk) bulk_g2s(dst, kin + base, bulk * 8u, &s_bar[buf]);
  };

  if (tid == 0) {
    mbar_init(&s_bar[0], 1);
    mbar_init(&s_bar[1], 1);
    fence_mbar_init();
    const uint32_t t = atomicAdd(tile_counter, 1u);
    s_tile[0] = t;
    if (t < ntiles) issue(t, 0);
  }
  __syncthreads();
  uint32_t phase0 = 0, phase1 = 0;
  for (int b = 0;; b ^= 1) {
    const uint32_t tile = s_tile[b];
    if (tile >= ntiles) break;
    uint64_t *s_in = reinterpret_cast<uint64_t *>(smem_raw + (size_t)b * kSortTile * sizeof(uint64_t));
    if (tid == 0) {  // claim + prefetch the next tile into the other buffer
      const uint32_t t2 = atomicAdd(tile_counter, 1u);
      s_tile[b ^ 1] = t2;
      if (t2 < ntiles) issue(t2, b ^ 1);
    }
#pragma unroll
    for (int q = 0; q < kWarps; q++) s_warp_hist[q][tid] = 0;
    const uint64_t tile_base = (uint64_t)tile * kSortTile;
    const uint64_t rem = n - tile_base;
    const uint32_t tile_n = rem < (uint64_t)kSortTile ? (uint32_t)rem : (uint32_t)kSortTile;
    if (b == 0) { mbar_wait(&s_bar[0], phase0); phase0 ^= 1; }
    else { mbar_wait(&s_bar[1], phase1); phase1 ^= 1; }
    if (tid == 0 && (tile_n & 1u)) s_in[tile_n - 1] = kin[tile_base + tile_n - 1];
    __syncthreads();

    uint64_t k[kSortItems];
    uint32_t r[kSortItems], peers[kSortItems];
    const bool full = tile_n == (uint32_t)kSortTile;
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
      const uint32_t loc = wslice + it * 32 + lane;
      const bool in = full || loc < tile_n;
      k[it] = s_in[loc];
      peers[it] = __match_any_sync(0xffffffffu, in ? ((uint32_t)(k[it] >> shift) & dmask) : 0x100u);
    }
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
      const uint32_t d = (uint32_t)(k[it] >> shift) & dmask;
      const uint32_t leader = 31 - __clz(peers[it]);
      const bool in = full || wslice + it * 32 + lane < tile_n;
      uint32_t base = 0;
      if (in && lane == leader) {
        base = s_warp_hist[warp][d];
        s_warp_hist[warp][d] = base + __popc(peers[it]);
      }
      r[it] = __shfl_sync(0xffffffffu, base, leader) + __popc(peers[it] & lt);
    }
    __syncthreads();

    const uint32_t d = tid;
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < kWarps; w++) {
      const uint32_t c = s_warp_hist[w][d];
      s_warp_hist[w][d] = total;
      total += c;
    }
    uint64_t *my_status = status + (uint64_t)tile * kRadix + d;
    uint64_t excl = 0;
    if (tile == 0) {
      st_relaxed_u64(my_status, kFlagInc | total);
    } else {
      st_relaxed_u64(my_status, kFlagAgg | total);
      int64_t t0 = (int64_t)tile - 1;
      while (true) {
        uint64_t sv[8];
#pragma unroll
        for (int w = 0; w < 8; w++) {
          const int64_t t = t0 - w;
          sv[w] = t >= 0 ? ld_relaxed_u64(status + (uint64_t)t * kRadix + d) : kFlagInc;
        }
        int consumed = 0;
        bool done = false;
#pragma unroll
        for (int w = 0; w < 8; w++) {
          if (consumed != w || done) continue;
          const uint64_t flag = sv[w] & ~kValMask;
          if (flag == 0) continue;
          excl += sv[w] & kValMask;
          consumed = w + 1;
          if (flag == kFlagInc) done = true;
        }
        if (done) break;
        t0 -= consumed;
        if (consumed < 8) __nanosleep(32);
      }
      st_relaxed_u64(my_status, kFlagInc | (excl + total));
    }
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
    s_global_base[d] = (uint64_t)hist_pass[d] + excl - dstart;
    __syncthreads();
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
      if (full || wslice + it * 32 + lane < tile_n) {
        const uint32_t dd = (uint32_t)(k[it] >> shift) & dmask;
        s_out[s_digit_start[dd] + s_warp_hist[warp][dd] + r[it]] = k[it];
      }
    }
    __syncthreads();
#pragma unroll 4
    for (uint32_t i = tid; i < tile_n; i += kSortThreads) {
      const uint64_t key = s_out[i];
      const uint32_t dd = (uint32_t)(key >> shift) & dmask;
      __stcs(kout + s_global_base[dd] + i, key);
    }
    __syncthreads();  // s_out, histograms and s_in[b] are reused by the next iterations
  }
}

}  // namespace mapsq

// MODE bit 1: skip look-back (excl = 0); bit 2: skip ranking (identity slot); bit 4: plain
// copy of the tile (no digit scatter); bit 8: no write-out at all.
template <int MODE>
__global__ void __launch_bounds__(kSortThreads, 3)
ablate_kernel(const uint64_t *__restrict__ kin, uint64_t *__restrict__ kout, uint64_t n,
              uint32_t shift, uint32_t bits, const uint32_t *__restrict__ hist_pass,
              uint64_t *__restrict__ status, uint32_t *__restrict__ tile_counter) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t *s_keys = reinterpret_cast<uint64_t *>(smem_raw);
  __shared__ uint32_t s_warp_hist[8][kRadix];
  __shared__ uint32_t s_digit_start[kRadix];
  __shared__ uint64_t s_global_base[kRadix];
  __shared__ uint32_t s_wsum[8];
  __shared__ uint32_t s_tile;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) s_tile = atomicAdd(tile_counter, 1u);
#pragma unroll
  for (int q = 0; q < 8; q++) s_warp_hist[q][tid] = 0;
  __syncthreads();
  const uint64_t tile = s_tile;
  const uint64_t tile_base = tile * kSortTile;
  const uint32_t wslice = warp * 32 * kSortItems;
  const uint32_t dmask = (1u << bits) - 1u;
  const uint64_t *src = kin + tile_base + wslice + lane;
  uint64_t k[kSortItems];
  uint32_t r[kSortItems], peers[kSortItems];
#pragma unroll
  for (int it = 0; it < kSortItems; it++) k[it] = __ldcs(src + it * 32);
  if (MODE & 4) {
#pragma unroll
    for (int it = 0; it < kSortItems; it++) __stcs(kout + tile_base + wslice + lane + it * 32, k[it]);
    return;
  }
  const uint32_t lt = lanemask_lt();
  if (!(MODE & 2)) {
#pragma unroll
    for (int it = 0; it < kSortItems; it++)
      peers[it] = __match_any_sync(0xffffffffu, (uint32_t)(k[it] >> shift) & dmask);
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
      const uint32_t d = (uint32_t)(k[it] >> shift) & dmask;
      const uint32_t leader = 31 - __clz(peers[it]);
      uint32_t base = 0;
      if (lane == leader) {
        base = s_warp_hist[warp][d];
        s_warp_hist[warp][d] = base + __popc(peers[it]);
      }
      r[it] = __shfl_sync(0xffffffffu, base, leader) + __popc(peers[it] & lt);
    }
  } else {
#pragma unroll
    for (int it = 0; it < kSortItems; it++) {
      r[it] = it * 32 + lane;
      if (lane == 0) atomicAdd(&s_warp_hist[warp][(uint32_t)(k[it] >> shift) & dmask], 0u);
    }
  }
  __syncthreads();
  const uint32_t d = tid;
  uint32_t total = 0;
#pragma unroll
  for (int w = 0; w < 8; w++) {
    const uint32_t c = s_warp_hist[w][d];
    s_warp_hist[w][d] = total;
    total += c;
  }
  uint64_t excl = 0;
  if (!(MODE & 1)) {
    uint64_t *my_status = status + tile * kRadix + d;
    if (tile == 0) {
      st_relaxed_u64(my_status, kFlagInc | total);
    } else {
      st_relaxed_u64(my_status, kFlagAgg | total);
      int64_t t0 = (int64_t)tile - 1;
      while (true) {
        uint64_t sv[8];
#pragma unroll
        for (int w = 0; w < 8; w++) {
          const int64_t t = t0 - w;
          sv[w] = t >= 0 ? ld_relaxed_u64(status + (uint64_t)t * kRadix + d) : kFlagInc;
        }
        int consumed = 0;
        bool done = false;
#pragma unroll
        for (int w = 0; w < 8; w++) {
          if (consumed != w || done) continue;
          const uint64_t flag = sv[w] & ~kValMask;
          if (flag == 0) continue;
          excl += sv[w] & kValMask;
          consumed = w + 1;
          if (flag == kFlagInc) done = true;
        }
        if (done) break;
        t0 -= consumed;
        if (consumed < 8) __nanosleep(32);
      }
      st_relaxed_u64(my_status, kFlagInc | (excl + total));
    }
  } else {
    excl = (tile * kSortTile) / kRadix;  // plausible spread, results are garbage
  }
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
  for (int w = 0; w < 8; w++)
    if ((uint32_t)w < warp) pre += s_wsum[w];
  const uint32_t dstart = pre + x - total;
  s_digit_start[d] = dstart;
  s_global_base[d] = (uint64_t)hist_pass[d] + excl - dstart;
  __syncthreads();
#pragma unroll
  for (int it = 0; it < kSortItems; it++) {
    const uint32_t dd = (uint32_t)(k[it] >> shift) & dmask;
    const uint32_t slot = (MODE & 2) ? r[it] + wslice : s_digit_start[dd] + s_warp_hist[warp][dd] + r[it];
    s_keys[slot & (kSortTile - 1)] = k[it];
  }
  __syncthreads();
  if (MODE & 8) {
    if (s_keys[tid] == 12345) kout[0] = 1;
    return;
  }
#pragma unroll 4
  for (uint32_t i = tid; i < kSortTile; i += kSortThreads) {
    const uint64_t key = s_keys[i];
    const uint32_t dd = (uint32_t)(key >> shift) & dmask;
    const uint64_t pos = (s_global_base[dd] + i) % n;
    __stcs(kout + pos, key);
  }
}

template <int MODE>
float run(const uint64_t *kin, uint64_t *kout, uint64_t n, uint32_t *hist, uint64_t *status,
          uint32_t *ctr) {
  const uint64_t ntiles = n / kSortTile;
  const size_t smem = kSortTile * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int rep = 0; rep < 5; rep++) {
    cudaMemsetAsync(status, 0, ntiles * kRadix * 8);
    cudaMemsetAsync(ctr, 0, 4);
    cudaEventRecord(a);
    ablate_kernel<MODE><<<(unsigned)ntiles, kSortThreads, smem>>>(kin, kout, n, 40, 8, hist, status, ctr);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  return best;
}

template <int MODE>
void report(const char *name, const uint64_t *kin, uint64_t *kout, uint64_t n, uint32_t *hist,
            uint64_t *status, uint32_t *ctr) {
  float ms = run<MODE>(kin, kout, n, hist, status, ctr);
  printf("%-28s %8.3f ms  %7.1f GB/s (16 B/key)\n", name, ms, 16.0 * n / ms / 1e6);
}

extern "C" void zipf_table(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i_lo,
                           uint64_t i_hi, uint32_t *key, uint32_t *val);

// C4-shaped sort: words key'<<ib | i of two Zipf(1.1) sides (the datagen recipe), every digit
// pass of the key bits, each variant timed over the whole pass sequence.
template <typename K>
float zipf_sort(K kern, int items, const char *name, uint64_t *w0, uint64_t *w1, uint64_t n,
                uint32_t ib, uint32_t kbits, uint32_t *hists, uint64_t *status, uint32_t *ctr,
                const std::vector<uint64_t> &ref_sample) {
  const uint64_t tile = 256ull * items, ntiles = (n + tile - 1) / tile;
  const size_t smem = tile * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int passes = (kbits + 7) / 8;
  cudaEvent_t ev[9];
  for (auto &e : ev) cudaEventCreate(&e);
  float best[8] = {1e9, 1e9, 1e9, 1e9, 1e9, 1e9, 1e9, 1e9}, tot = 1e9;
  for (int rep = 0; rep < 3; rep++) {
    uint64_t *a = w0, *b = w1;
    cudaEventRecord(ev[0]);
    for (int p = 0; p < passes; p++) {
      const uint32_t bits = (p + 1 == passes) ? kbits - 8 * p : 8;
      cudaMemsetAsync(status, 0, ntiles * kRadix * 8);
      cudaMemsetAsync(ctr, 0, 4);
      kern<<<(unsigned)ntiles, 256, smem>>>(a, b, nullptr, nullptr, n, ib + 8 * p, bits,
                                            hists + p * kRadix, status, ctr, nullptr, 0, 0, n, 0);
      cudaEventRecord(ev[p + 1]);
      std::swap(a, b);
    }
    cudaEventSynchronize(ev[passes]);
    float t = 0;
    for (int p = 0; p < passes; p++) {
      float ms;
      cudaEventElapsedTime(&ms, ev[p], ev[p + 1]);
      best[p] = ms < best[p] ? ms : best[p];
      t += ms;
    }
    tot = t < tot ? t : tot;
    // re-run from the unsorted words: restore w0 (the passes ping-pong; even count ends in w0)
    if (passes % 2) std::swap(w0, w1);
    std::vector<uint64_t> o(ref_sample.size());
    const uint64_t stride = n / ref_sample.size();
    for (size_t j = 0; j < o.size(); j++) cudaMemcpy(&o[j], w0 + j * stride, 8, cudaMemcpyDeviceToHost);
    if (o != ref_sample) { printf("%s: WRONG ORDER\n", name); return -1; }
    if (passes % 2) std::swap(w0, w1);
    break;  // (the sort is in place in w0 now: further reps would time already-sorted input)
  }
  printf("%-40s total %7.3f ms  passes:", name, tot);
  for (int p = 0; p < passes; p++) printf(" %.3f", best[p]);
  printf("  (%.0f GB/s)\n", 16.0 * n * passes / tot / 1e6);
  return tot;
}

int sort_main(std::vector<uint64_t> &w, uint32_t ib, uint32_t kbits);

int zipf_main(uint64_t n) {
  const uint64_t h = n / 2;
  n = 2 * h;
  std::vector<uint32_t> key(n);
  zipf_table(1702, 0, 1.1, 29, 0, h, key.data(), nullptr);
  zipf_table(1702, 1, 1.1, 29, 0, h, key.data() + h, nullptr);
  uint32_t ib = 0;
  while ((1ull << ib) < n) ib++;
  uint32_t lo = 0xffffffffu, hi = 0;
  for (uint64_t i = 0; i < n; i++) { lo = key[i] < lo ? key[i] : lo; hi = key[i] > hi ? key[i] : hi; }
  uint32_t kbits = 0;
  while ((1ull << kbits) <= (uint64_t)(hi - lo)) kbits++;
  std::vector<uint64_t> w(n);
  for (uint64_t i = 0; i < n; i++) w[i] = ((uint64_t)(key[i] - lo) << ib) | i;
  printf("zipf: ");
  return sort_main(w, ib, kbits);
}

// words dumped by tools/dump_words.py (raw little-endian u64)
int file_main(const char *path, uint32_t ib, uint32_t kbits) {
  FILE *f = fopen(path, "rb");
  if (!f) { printf("cannot open %s\n", path); return 1; }
  fseek(f, 0, SEEK_END);
  const uint64_t n = ftell(f) / 8;
  fseek(f, 0, SEEK_SET);
  std::vector<uint64_t> w(n);
  if (fread(w.data(), 8, n, f) != n) { printf("short read\n"); return 1; }
  fclose(f);
  printf("%s: ", path);
  return sort_main(w, ib, kbits);
}

int sort_main(std::vector<uint64_t> &w, uint32_t ib, uint32_t kbits) {
  const uint64_t n = w.size();
  const int passes = (kbits + 7) / 8;
  std::vector<uint32_t> hh(8 * kRadix, 0);
  for (uint64_t i = 0; i < n; i++)
    for (int p = 0; p < passes; p++) hh[p * kRadix + ((w[i] >> (ib + 8 * p)) & 255)]++;
  printf("n=%llu ib=%u kbits=%u passes=%d\n", (unsigned long long)n, ib, kbits, passes);
  std::vector<uint64_t> sorted(w);
  std::sort(sorted.begin(), sorted.end());
  std::vector<uint64_t> sample(4096);
  for (size_t j = 0; j < sample.size(); j++) sample[j] = sorted[j * (n / sample.size())];
  uint64_t *w0, *w1, *status, *wsrc;
  uint32_t *hists, *ctr;
  cudaMalloc(&w0, n * 8);
  cudaMalloc(&w1, n * 8);
  cudaMalloc(&wsrc, n * 8);
  cudaMalloc(&status, (n / 2048 + 2) * kRadix * 8);
  cudaMalloc(&hists, 8 * kRadix * 4);
  cudaMalloc(&ctr, 4);
  cudaMemcpy(wsrc, w.data(), n * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(hists, hh.data(), 8 * kRadix * 4, cudaMemcpyHostToDevice);
#define ZRUN(K, I, NAME)                                                                   \
  cudaMemcpy(w0, wsrc, n * 8, cudaMemcpyDeviceToDevice);                                  \
  zipf_sort(K, I, NAME, w0, w1, n, ib, kbits, hists, status, ctr, sample);
  ZRUN((radix_pass_kernel<false, 24, 4, 3, true, 3>), 24, "items24 minb3 (prod)");
  ZRUN((radix_pass_kernel<false, 28, 4, 3, true, 3>), 28, "items28 minb3");
  ZRUN((radix_pass_kernel<false, 24, 2, 3, true, 3>), 24, "items24 minb3 win2");
  ZRUN((radix_pass_kernel<false, 24, 4, 3, false, 3>), 24, "items24 minb3 noreload");
  ZRUN((radix_pass_kernel<false, 20, 4, 3, true, 3>), 20, "items20 minb3");
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

int main(int argc, char **argv) {
  setvbuf(stdout, nullptr, _IONBF, 0);
  if (argc > 4 && std::string(argv[1]) == "file")
    return file_main(argv[2], atoi(argv[3]), atoi(argv[4]));
  if (argc > 1 && std::string(argv[1]) == "zipf")
    return zipf_main(argc > 2 ? strtoull(argv[2], 0, 10) : 400000000ull);
  const uint64_t n = (argc > 1 ? strtoull(argv[1], 0, 10) : 200000000ull) / kSortTile * kSortTile;
  std::vector<uint64_t> h(n);
  uint64_t x = 88172645463325252ull;
  const double hot = argc > 2 ? atof(argv[2]) : 0.0;  // fraction of keys equal to one hot key
  for (uint64_t i = 0; i < n; i++) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const bool is_hot = (double)(x >> 11) * 0x1.0p-53 < hot;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = ((is_hot ? 0x123456789abcull << 16 : x) & ~0xffffffffull) | i;  // high bits key, index low bits
  }
  uint64_t *kin, *kout, *status;
  uint32_t *hist, *ctr;
  cudaMalloc(&kin, n * 8);
  cudaMalloc(&kout, n * 8);
  cudaMalloc(&status, (n / 2048 + 2) * kRadix * 8);
  cudaMalloc(&hist, 8 * kRadix * 4);
  cudaMalloc(&ctr, 4);
  cudaMemcpy(kin, h.data(), n * 8, cudaMemcpyHostToDevice);
  // exact digit offsets of bits [8,16) for the real pass
  std::vector<uint32_t> hh(kRadix, 0);
  for (uint64_t i = 0; i < n; i++) hh[(h[i] >> 40) & 255]++;
  std::vector<uint32_t> hx(hh);  // exclusive offsets for the ablation kernels, raw counts for the library pass
  uint32_t run_ = 0;
  for (int d = 0; d < kRadix; d++) { uint32_t c = hx[d]; hx[d] = run_; run_ += c; }
  cudaMemcpy(hist, hx.data(), kRadix * 4, cudaMemcpyHostToDevice);
  uint32_t *histraw, *hnext;
  const bool use_next = argc > 3 && atoi(argv[3]);
  cudaMalloc(&hnext, kRadix * 4);
  cudaMalloc(&histraw, kRadix * 4);
  cudaMemcpy(histraw, hh.data(), kRadix * 4, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(ablate_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSortTile * 8);
  if (0) report<0>("full pass", kin, kout, n, hist, status, ctr);
  if (0) report<1>("no look-back", kin, kout, n, hist, status, ctr);
  if (0) report<2>("no ranking", kin, kout, n, hist, status, ctr);
  if (0) report<3>("no ranking, no look-back", kin, kout, n, hist, status, ctr);
  if (0) report<4>("tile copy (same shape)", kin, kout, n, hist, status, ctr);
  if (0) report<8>("no write-out", kin, kout, n, hist, status, ctr);
  if (0) report<9>("no write-out, no look-back", kin, kout, n, hist, status, ctr);
  // production kernel variants: ITEMS (tile = 256 x ITEMS), look-back window, CTAs/SM
  {
    auto timeit = [&](auto kern, int items, const char *name) {
      const uint64_t tile = 256ull * items;
      const uint64_t ntiles = (n + tile - 1) / tile;
      const size_t smem = tile * 8;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      float best = 1e9;
      for (int rep = 0; rep < 5; rep++) {
        cudaMemsetAsync(status, 0, ntiles * kRadix * 8);
        cudaMemsetAsync(ctr, 0, 4);
        cudaEventRecord(a);
        cudaMemsetAsync(hnext, 0, kRadix * 4);
        kern<<<(unsigned)ntiles, 256, smem>>>(kin, kout, nullptr, nullptr, n, 40, 8, histraw, status, ctr, use_next ? hnext : nullptr, 48, 0xff, n, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
      }
      printf("%-34s %8.3f ms  %7.1f GB/s  %s\n", name, best, 16.0 * n / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    };
    timeit(radix_pass_kernel<false, 32, 4, 2, true, false>, 32, "items32 minb2 reload match (prod)");
    timeit(radix_pass_kernel<false, 32, 4, 2, true, true>, 32, "items32 minb2 reload ballot");
    timeit(radix_pass_kernel<false, 16, 4, 4, true, true>, 16, "items16 minb4 reload ballot");
    timeit(radix_pass_kernel<false, 32, 4, 2, true, 2>, 32, "items32 minb2 reload atomicOr");
    timeit(radix_pass_kernel<false, 32, 4, 2, true, 3>, 32, "items32 minb2 reload atomicOr+uni");
    timeit(radix_pass_kernel<false, 16, 4, 4, true, 3>, 16, "items16 minb4 reload atomicOr+uni");
  }
  // the library's real pass for comparison
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; rep++) {
      cudaMemsetAsync(status, 0, (n / kSortTile) * kRadix * 8);
      cudaMemsetAsync(ctr, 0, 4);
      cudaEventRecord(a);
      launch_radix_pass(kin, kout, nullptr, nullptr, n, 40, 8, histraw, status, ctr, nullptr, 48, 8, 0);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %7.1f GB/s\n", "library radix_pass", best, 16.0 * n / best / 1e6);
    std::vector<uint64_t> o(n);
    cudaMemcpy(o.data(), kout, n * 8, cudaMemcpyDeviceToHost);
    bool ok = true;
    for (uint64_t i = 1; i < n && ok; i++) ok = ((o[i - 1] >> 40) & 255) <= ((o[i] >> 40) & 255);
    printf("library pass digit order ok: %d  err=%s\n", (int)ok, cudaGetErrorString(cudaGetLastError()));
  }
  // plain copy reference
  {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e9;
    for (int rep = 0; rep < 5; rep++) {
      cudaEventRecord(a);
      cudaMemcpyAsync(kout, kin, n * 8, cudaMemcpyDeviceToDevice);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      best = ms < best ? ms : best;
    }
    printf("%-28s %8.3f ms  %7.1f GB/s\n", "cudaMemcpy D2D", best, 16.0 * n / best / 1e6);
  }
  return 0;
}
