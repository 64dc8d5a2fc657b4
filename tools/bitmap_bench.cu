// bitmap_bench.cu — developer micro-benchmark: cost of a key-presence bitmap (semi-join filter)
// on B200: build (atomicOr per row, with/without test-before-set) and probe, for C4-shaped
// Zipf keys.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/bitmap_bench.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

extern "C" void zipf_table(uint64_t seed, int side, double s, uint32_t kbits, uint64_t i_lo,
                           uint64_t i_hi, uint32_t *key, uint32_t *val);

__global__ void build_atomic(const uint32_t *k, uint64_t n, uint32_t *bm, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = __ldcs(k + i) & mask;
    atomicOr(bm + (x >> 5), 1u << (x & 31));
  }
}
__global__ void build_test(const uint32_t *k, uint64_t n, uint32_t *bm, uint32_t mask) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = __ldcs(k + i) & mask;
    const uint32_t b = 1u << (x & 31);
    if (!(__ldcg(bm + (x >> 5)) & b)) atomicOr(bm + (x >> 5), b);
  }
}
__global__ void probe(const uint32_t *k, uint64_t n, const uint32_t *bm, uint32_t mask, unsigned long long *cnt) {
  uint32_t c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t x = __ldcs(k + i) & mask;
    c += (__ldcg(bm + (x >> 5)) >> (x & 31)) & 1u;
  }
  atomicAdd(cnt, (unsigned long long)c);
}

template <int ILP, bool NC>
__global__ void probe_ilp(const uint32_t *k, uint64_t n, const uint32_t *bm, uint32_t mask, unsigned long long *cnt) {
  uint32_t c = 0;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * ILP;
  for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x) * ILP + threadIdx.x; i0 < n; i0 += stride) {
    uint32_t x[ILP], w[ILP];
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const uint64_t i = i0 + (uint64_t)u * blockDim.x;
      x[u] = i < n ? (uint32_t)((__ldcs(k + i) * 0x9E3779B97F4A7C15ull) >> 32) & mask : 0;
    }
#pragma unroll
    for (int u = 0; u < ILP; u++) w[u] = NC ? __ldg(bm + (x[u] >> 5)) : __ldcg(bm + (x[u] >> 5));
#pragma unroll
    for (int u = 0; u < ILP; u++) {
      const uint64_t i = i0 + (uint64_t)u * blockDim.x;
      c += (i < n) & (w[u] >> (x[u] & 31));
    }
  }
  atomicAdd(cnt, (unsigned long long)c);
}

// distinct random bits: one RED.OR per row (no test), or test-then-set
template <bool TEST>
__global__ void build_distinct(uint64_t n, uint32_t *bm, uint32_t mask) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * 8;
  for (uint64_t i0 = (blockIdx.x * (uint64_t)blockDim.x) * 8 + threadIdx.x; i0 < n; i0 += stride) {
    uint32_t x[8], w[8];
#pragma unroll
    for (int u = 0; u < 8; u++) x[u] = (uint32_t)(((i0 + u * blockDim.x) * 0x9E3779B97F4A7C15ull) >> 32) & mask;
    if (TEST) {
#pragma unroll
      for (int u = 0; u < 8; u++) w[u] = __ldg(bm + (x[u] >> 5));
    }
#pragma unroll
    for (int u = 0; u < 8; u++)
      if (i0 + u * blockDim.x < n && (!TEST || !(w[u] >> (x[u] & 31) & 1u))) atomicOr(bm + (x[u] >> 5), 1u << (x[u] & 31));
  }
}

int main(int argc, char **argv) {
  const uint64_t n = argc > 1 ? strtoull(argv[1], 0, 10) : 500000000ull;
  std::vector<uint32_t> a(n), b(n);
  zipf_table(1702, 0, 1.1, 29, 0, n, a.data(), nullptr);
  zipf_table(1702, 1, 1.1, 29, 0, n, b.data(), nullptr);
  uint32_t *da, *db, *bm;
  unsigned long long *cnt;
  cudaMalloc(&da, n * 4);
  cudaMalloc(&db, n * 4);
  cudaMalloc(&bm, (1ull << 32) / 8);
  cudaMalloc(&cnt, 8);
  cudaMemcpy(da, a.data(), n * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), n * 4, cudaMemcpyHostToDevice);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto t = [&](const char *name, auto f) {
    float best = 1e9;
    for (int r = 0; r < 3; r++) {
      cudaMemset(bm, 0, (1ull << 32) / 8);
      cudaMemset(cnt, 0, 8);
      cudaEventRecord(e0);
      f();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      best = ms < best ? ms : best;
    }
    unsigned long long c = 0;
    cudaMemcpy(&c, cnt, 8, cudaMemcpyDeviceToHost);
    printf("%-36s %8.3f ms  (%.2f G rows/s) cnt=%llu %s\n", name, best, n / best / 1e6, c,
           cudaGetErrorString(cudaGetLastError()));
  };
  const uint32_t mask = (1u << 29) - 1;
  const int g = 148 * 16;
  int maxp = 0, maxw = 0, l2 = 0;
  cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
  cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0);
  cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
  printf("L2 %d B, max persisting L2 %d B, max access policy window %d B\n", l2, maxp, maxw);
  t("build atomicOr", [&] { build_atomic<<<g, 256>>>(da, n, bm, mask); });
  t("build test+atomicOr", [&] { build_test<<<g, 256>>>(da, n, bm, mask); });
  t("build test+atomicOr, then probe B", [&] {
    build_test<<<g, 256>>>(da, n, bm, mask);
    probe<<<g, 256>>>(db, n, bm, mask, cnt);
  });
  t("probe only (empty bitmap)", [&] { probe<<<g, 256>>>(db, n, bm, mask, cnt); });
  for (uint32_t bits : {32u, 30u, 29u, 28u, 24u}) {
    const uint32_t m = (uint32_t)((1ull << bits) - 1);
    char name[64];
    snprintf(name, sizeof name, "RED.OR distinct 2^%u bits", bits);
    t(name, [&] { build_distinct<false><<<g, 256>>>(n, bm, m); });
    snprintf(name, sizeof name, "test+RED.OR distinct 2^%u bits", bits);
    t(name, [&] { build_distinct<true><<<g, 256>>>(n, bm, m); });
  }
  // the same probes with the bitmap marked persisting in L2 (stream access policy window)
  for (uint32_t bits : {29u, 28u}) {
    const size_t bytes = (1ull << bits) / 8;
    cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp);
    cudaStreamAttrValue v = {};
    v.accessPolicyWindow.base_ptr = bm;
    v.accessPolicyWindow.num_bytes = bytes < (size_t)maxw ? bytes : (size_t)maxw;
    v.accessPolicyWindow.hitRatio = (float)((double)maxp / (double)bytes > 1.0 ? 1.0 : (double)maxp / (double)bytes);
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &v);
    const uint32_t m = (uint32_t)((1ull << bits) - 1);
    char name[64];
    snprintf(name, sizeof name, "PERSIST probe ilp4 nc 2^%u bits", bits);
    t(name, [&] { probe_ilp<4, true><<<g, 256>>>(db, n, bm, m, cnt); });
    snprintf(name, sizeof name, "PERSIST RED.OR distinct 2^%u bits", bits);
    t(name, [&] { build_distinct<false><<<g, 256>>>(n, bm, m); });
    v.accessPolicyWindow.num_bytes = 0;
    cudaStreamSetAttribute(0, cudaStreamAttributeAccessPolicyWindow, &v);
    cudaCtxResetPersistingL2Cache();
    printf("  (%s)\n", cudaGetErrorString(cudaGetLastError()));
  }
  for (uint32_t bits : {32u, 31u, 30u, 29u, 28u}) {
    const uint32_t m = (uint32_t)((1ull << bits) - 1);
    char name[64];
    snprintf(name, sizeof name, "probe ilp16 nc 2^%u bits", bits);
    t(name, [&] { probe_ilp<16, true><<<g, 256>>>(db, n, bm, m, cnt); });
    snprintf(name, sizeof name, "probe ilp4 nc 2^%u bits", bits);
    t(name, [&] { probe_ilp<4, true><<<g, 256>>>(db, n, bm, m, cnt); });
  }
  return 0;
}
