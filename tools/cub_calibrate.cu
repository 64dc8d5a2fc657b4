// cub_calibrate.cu — TEST/TOOL ONLY (never on the product path): calibrates the library's LSD
// radix sort (mapsq_sort_words, the one-sweep digit passes of csrc/radix.cu) against CUB's
// DeviceRadixSort::SortKeys on identical words and the identical bit range, on one B200.
//
// Words are shaped like a join's Map output: key' in bits [ib, ib + kb) (uniform, or 10% of them
// one hot key), the row index in the low ib bits — so every word is distinct and both sorts
// produce the same (unique) array, which is checked.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include \
//        tools/cub_calibrate.cu -o tools/cub_calibrate -Lpaper_1702_03484_b200 -lmapsq \
//        -Xlinker -rpath=$PWD/paper_1702_03484_b200
//   tools/cub_calibrate [n] [kb] [hot_fraction]
#include <cub/device/device_radix_sort.cuh>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "mapsq.h"

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e_ = (x);                                                              \
    if (e_ != cudaSuccess) {                                                           \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));                    \
      std::exit(1);                                                                    \
    }                                                                                  \
  } while (0)

int main(int argc, char **argv) {
  const uint64_t n = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 63000000ull;
  const uint32_t kb = argc > 2 ? (uint32_t)std::atoi(argv[2]) : 29;
  const double hot = argc > 3 ? std::atof(argv[3]) : 0.0;
  uint32_t ib = 1;
  while ((1ull << ib) < n) ib++;
  std::vector<uint64_t> h(n);
  uint64_t x = 0x9E3779B97F4A7C15ull;
  for (uint64_t i = 0; i < n; i++) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const bool is_hot = (double)(x >> 11) * 0x1.0p-53 < hot;
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    const uint64_t key = is_hot ? 12345 : (x & ((1ull << kb) - 1));
    h[i] = (key << ib) | i;
  }
  uint64_t *d_in, *d_a, *d_b;
  CK(cudaMalloc(&d_in, n * 8));
  CK(cudaMalloc(&d_a, n * 8));
  CK(cudaMalloc(&d_b, n * 8));
  CK(cudaMemcpy(d_in, h.data(), n * 8, cudaMemcpyHostToDevice));
  const int begin = (int)ib, end = (int)(ib + kb);
  size_t tmp_bytes = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, d_in, d_b, (int64_t)n, begin, end);
  void *tmp;
  CK(cudaMalloc(&tmp, tmp_bytes));
  mapsq_ctx *ctx = nullptr;
  if (mapsq_create(&ctx, 0, nullptr) != MAPSQ_OK) return 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto best = [&](auto fn) {
    float b = 1e30f;
    for (int rep = 0; rep < 7; rep++) {
      CK(cudaMemcpy(d_a, d_in, n * 8, cudaMemcpyDeviceToDevice));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) b = ms < b ? ms : b;  // (rep 0 warms up)
    }
    return b;
  };
  const float t_cub = best([&] {
    cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, d_a, d_b, (int64_t)n, begin, end);
  });
  std::vector<uint64_t> r_cub(n), r_lib(n);
  CK(cudaMemcpy(r_cub.data(), d_b, n * 8, cudaMemcpyDeviceToHost));
  const float t_lib = best([&] {
    if (mapsq_sort_words(ctx, d_a, n, begin, end, nullptr) != MAPSQ_OK) {
      std::fprintf(stderr, "mapsq_sort_words: %s\n", mapsq_last_error(ctx));
      std::exit(1);
    }
  });
  CK(cudaMemcpy(r_lib.data(), d_a, n * 8, cudaMemcpyDeviceToHost));
  const bool same = std::memcmp(r_cub.data(), r_lib.data(), n * 8) == 0;
  const uint32_t passes = (kb + 7) / 8;
  std::printf("{\"n\": %llu, \"kb\": %u, \"ib\": %u, \"hot\": %.3f, \"cub_ms\": %.4f, "
              "\"mapsq_ms\": %.4f, \"mapsq_passes\": %u, \"mapsq_gbs_16B_per_pass\": %.1f, "
              "\"cub_gbs_same_bytes\": %.1f, \"identical_output\": %s}\n",
              (unsigned long long)n, kb, ib, hot, t_cub, t_lib, passes,
              16.0 * passes * n / (t_lib * 1e6), 16.0 * passes * n / (t_cub * 1e6),
              same ? "true" : "false");
  mapsq_destroy(ctx);
  return same ? 0 : 2;
}
