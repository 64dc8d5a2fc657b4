// dist.cu — distributed join and query over NCCL + CUDA IPC (SURVEY §8 rows b and e).
//
// An equi-join decomposes over disjoint key sets: Algorithm 1 joins each key's group on its own
// (PAPER.md:126-133), so hash-partitioning both inputs on the shared variables and joining locally
// on every rank yields RS as the union of the rank outputs.  The paper runs on one GPU
// (PAPER.md:170); this is the B200 extension.  Per exchange:
//   1. mapsq_partition_plan (K8 histogram + scan) -> this rank's per-destination row counts;
//   2. NCCL all-gather of the counts -> the world x world count matrix (every rank derives the
//      same layout from it, mapsq_exchange_layout);
//   3. receive arenas grown where too small (new cudaMalloc, IPC handle all-gathered, peers open
//      it; the old allocation is freed only after every peer closed its mapping);
//   4. barrier, ONE kernel (mapsq_partition_scatter) stores every row into its destination
//      rank's arena over NVLink, barrier;
//   5. column bounds min/max all-reduced, so the receiving side's local join range-compresses
//      its keys without a min/max pass.
// NCCL is loaded with dlopen at mapsq_dist_init (libnccl.so.2: the copy torch already loaded,
// else the system one), so single-GPU users of the library never need it.
#include <dlfcn.h>
#include <nccl.h>

#include <array>
#include <cstring>
#include <map>
#include <mutex>

#include "internal.cuh"

using namespace mapsq;

namespace {

constexpr int kDistMaxRanks = 64;  // = partition.cu's kMaxParts
constexpr size_t kHandleRec = 80;  // {u64 grew, u64 bytes, 64 B cudaIpcMemHandle_t}

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char *e = dlerror();
      api.why = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
#define SYM(field, name)                                          \
  api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name)); \
  if (!api.field) {                                               \
    api.why = "libnccl lacks " name;                              \
    return;                                                       \
  }
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(AllGather, "ncclAllGather");
    SYM(AllReduce, "ncclAllReduce");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    api.ok = true;
  });
  return api;
}

#define NC(call)                                                                        \
  do {                                                                                  \
    ncclResult_t _r = (call);                                                           \
    if (_r != ncclSuccess)                                                              \
      return set_error(ctx, MAPSQ_E_NCCL, std::string(#call ": ") + nccl().GetErrorString(_r)); \
  } while (0)
#define CK(call)                                \
  do {                                          \
    cudaError_t _e = (call);                    \
    if (_e != cudaSuccess) return cuda_check(ctx, _e, #call); \
  } while (0)
#define TRY(x)                                  \
  do {                                          \
    mapsq_status _st = (x);                     \
    if (_st != MAPSQ_OK) return _st;            \
  } while (0)

// CUDA IPC failures (e.g. a container without IPC between the rank processes) are reported as
// MAPSQ_E_CUDA with "CUDA IPC" in the message but do NOT poison the context: the caller can fall
// back to an exchange without peer mappings (paper_1702_03484_b200.dist does).
#define CKIPC(call)                                                                        \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) {                                                               \
      cudaGetLastError();                                                                  \
      return set_error(ctx, MAPSQ_E_CUDA,                                                  \
                       std::string("CUDA IPC: " #call ": ") + cudaGetErrorString(_e));     \
    }                                                                                      \
  } while (0)

inline cudaStream_t S(void *stream) { return (cudaStream_t)stream; }
inline uint64_t stride_rows(uint64_t n) { return (n + 3) & ~3ull; }

}  // namespace

namespace mapsq {

// One receive arena per join side: this rank's allocation and every rank's mapped pointer.
struct Arena {
  void *own = nullptr;
  uint64_t cap[kDistMaxRanks] = {};
  void *ptr[kDistMaxRanks] = {};
};

struct DistState {
  ncclComm_t comm = nullptr;       // NCCL control plane (mapsq_dist_init), or
  bool host = false;               // caller-supplied host collectives (mapsq_dist_init_host)
  mapsq_collectives coll{};
  int rank = 0, world = 1;
  bool ipc_broken = false;         // a peer mapping failed on some rank: no fused exchange
  // device staging of the NCCL collectives, and the barrier word
  void *dstage = nullptr;
  size_t stage_bytes = 0;
  uint64_t *dbar = nullptr;
  void *dbuf = nullptr;
  Arena slot[3];              // receive arenas of the two join sides; [2]: pre-filter bitmaps
  uint64_t *dpeers = nullptr; // device copy of slot[2]'s per-rank bitmap pointers (peer_or)
};

void dist_free(mapsq_ctx *ctx) {
  DistState *d = ctx->dist;
  if (!d) return;
  cudaDeviceSynchronize();
  for (Arena &a : d->slot) {  // (all three slots)
    for (int r = 0; r < d->world; r++)
      if (r != d->rank && a.ptr[r]) cudaIpcCloseMemHandle(a.ptr[r]);
    if (a.own) cudaFree(a.own);
  }
  if (d->dbuf) cudaFree(d->dbuf);
  if (!d->host && d->comm && nccl().ok) nccl().CommDestroy(d->comm);
  delete d;
  ctx->dist = nullptr;
}

}  // namespace mapsq

namespace {

// ---- control-plane collectives on HOST buffers (blocking): NCCL through the device staging
// buffer, or the caller's callbacks.  Every rank calls them in the same order.
mapsq_status coll_allgather(mapsq_ctx *ctx, DistState *d, const void *send, void *recv,
                            size_t bytes, cudaStream_t s) {
  if (d->host) {
    CK(cudaStreamSynchronize(s));
    if (d->coll.allgather(d->coll.user, send, recv, bytes))
      return set_error(ctx, MAPSQ_E_NCCL, "host allgather callback failed");
    return MAPSQ_OK;
  }
  if (bytes * d->world > d->stage_bytes)
    return set_error(ctx, MAPSQ_E_INVALID, "internal: collective larger than the staging buffer");
  unsigned char *st = static_cast<unsigned char *>(d->dstage);
  CK(cudaMemcpyAsync(st + bytes * d->rank, send, bytes, cudaMemcpyHostToDevice, s));
  NC(nccl().AllGather(st + bytes * d->rank, st, bytes, ncclUint8, d->comm, s));
  CK(cudaMemcpyAsync(recv, st, bytes * d->world, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return MAPSQ_OK;
}

mapsq_status coll_allreduce_max(mapsq_ctx *ctx, DistState *d, uint32_t *buf, size_t n,
                                cudaStream_t s) {
  if (d->host) {
    CK(cudaStreamSynchronize(s));
    if (d->coll.allreduce_max_u32(d->coll.user, buf, n))
      return set_error(ctx, MAPSQ_E_NCCL, "host allreduce callback failed");
    return MAPSQ_OK;
  }
  if (4 * n > d->stage_bytes)
    return set_error(ctx, MAPSQ_E_INVALID, "internal: collective larger than the staging buffer");
  uint32_t *st = static_cast<uint32_t *>(d->dstage);
  CK(cudaMemcpyAsync(st, buf, 4 * n, cudaMemcpyHostToDevice, s));
  NC(nccl().AllReduce(st, st, n, ncclUint32, ncclMax, d->comm, s));
  CK(cudaMemcpyAsync(buf, st, 4 * n, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return MAPSQ_OK;
}

// Blocking barrier: everything this rank enqueued on `s` has completed and so has every other
// rank's work before its matching barrier.
mapsq_status barrier(mapsq_ctx *ctx, DistState *d, cudaStream_t s) {
  CK(cudaStreamSynchronize(s));
  if (d->host) {
    if (d->coll.barrier(d->coll.user)) return set_error(ctx, MAPSQ_E_NCCL, "host barrier callback failed");
    return MAPSQ_OK;
  }
  NC(nccl().AllReduce(d->dbar, d->dbar, 1, ncclUint64, ncclSum, d->comm, s));
  CK(cudaStreamSynchronize(s));
  return MAPSQ_OK;
}

// Grow the arenas of `slot` that are smaller than need[] (collective; every rank passes the same
// need[]).  New allocations are exported, their handles all-gathered and opened by the peers; a
// replaced allocation is freed after a barrier, when no peer maps it any more.  The outcome is
// collective: a failure to allocate, export or open on ANY rank makes EVERY rank return the same
// MAPSQ_E_CUDA "CUDA IPC" error (after the same collectives), so no rank is left waiting in a
// collective its peers never enter; the fused exchange is then disabled on every rank.
mapsq_status ensure_arena(mapsq_ctx *ctx, DistState *d, int slot, const uint64_t *need,
                          cudaStream_t s) {
  Arena &a = d->slot[slot];
  bool any = false;
  for (int r = 0; r < d->world; r++) any |= need[r] > a.cap[r];
  if (!any) return MAPSQ_OK;
  // record: {u64 state (0 unchanged, 1 grew, 2 failed), u64 bytes, 64 B cudaIpcMemHandle_t}
  unsigned char rec[kHandleRec] = {};
  std::string why;
  void *p = nullptr;
  const bool grow = need[d->rank] > a.cap[d->rank];
  uint64_t nbytes = a.cap[d->rank], state = 0;
  if (grow) {
    nbytes = std::max<uint64_t>(1ull << 20, need[d->rank] + need[d->rank] / 4);
    nbytes = (nbytes + (2ull << 20) - 1) & ~((2ull << 20) - 1);
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaMalloc(&p, nbytes);
    if (e == cudaSuccess) {
      e = cudaIpcGetMemHandle(&h, p);
      if (e != cudaSuccess) {
        cudaFree(p);
        p = nullptr;
      }
    }
    if (e != cudaSuccess) {
      cudaGetLastError();
      why = std::string("cudaMalloc/cudaIpcGetMemHandle: ") + cudaGetErrorString(e);
      state = 2;
    } else {
      state = 1;
      std::memcpy(rec + 16, &h, 64);
    }
  }
  std::memcpy(rec, &state, 8);
  std::memcpy(rec + 8, &nbytes, 8);
  const int W = d->world;
  std::vector<unsigned char> all((size_t)kHandleRec * W);
  TRY(coll_allgather(ctx, d, rec, all.data(), kHandleRec, s));
  int failed_rank = -1;
  for (int r = 0; r < W && failed_rank < 0; r++) {
    uint64_t st;
    std::memcpy(&st, all.data() + kHandleRec * r, 8);
    if (st == 2) failed_rank = r;
  }
  if (failed_rank >= 0) {  // every rank sees it: nothing was opened, nothing changes
    if (p) cudaFree(p);
    d->ipc_broken = true;
    return set_error(ctx, MAPSQ_E_CUDA,
                     "CUDA IPC: arena export failed on rank " + std::to_string(failed_rank) +
                         (why.empty() ? std::string() : ": " + why));
  }
  // open the peers' new arenas; the local outcome is then agreed on (max of "failed")
  void *opened[kDistMaxRanks] = {};
  uint32_t bad = 0;
  for (int r = 0; r < W && !bad; r++) {
    if (r == d->rank) continue;
    uint64_t st;
    std::memcpy(&st, all.data() + kHandleRec * r, 8);
    if (st != 1) continue;
    cudaIpcMemHandle_t h;
    std::memcpy(&h, all.data() + kHandleRec * r + 16, 64);
    cudaError_t e = cudaIpcOpenMemHandle(&opened[r], h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
      cudaGetLastError();
      opened[r] = nullptr;
      why = std::string("cudaIpcOpenMemHandle: ") + cudaGetErrorString(e);
      bad = 1;
    }
  }
  uint32_t agree = bad;
  TRY(coll_allreduce_max(ctx, d, &agree, 1, s));
  if (agree) {  // some rank could not map a peer: undo this round everywhere
    for (int r = 0; r < W; r++)
      if (opened[r]) cudaIpcCloseMemHandle(opened[r]);
    if (p) cudaFree(p);
    d->ipc_broken = true;
    return set_error(ctx, MAPSQ_E_CUDA,
                     "CUDA IPC: a rank could not open a peer's arena" +
                         (why.empty() ? std::string() : " (this rank: " + why + ")"));
  }
  void *old = nullptr;
  for (int r = 0; r < W; r++) {
    uint64_t st, nb;
    std::memcpy(&st, all.data() + kHandleRec * r, 8);
    std::memcpy(&nb, all.data() + kHandleRec * r + 8, 8);
    if (st != 1) continue;
    if (r == d->rank) {
      old = a.own;
      a.own = p;
      a.ptr[r] = p;
    } else {
      if (a.ptr[r]) cudaIpcCloseMemHandle(a.ptr[r]);
      a.ptr[r] = opened[r];
    }
    a.cap[r] = nb;
  }
  TRY(barrier(ctx, d, s));  // every peer has closed its mapping of `old`
  if (old) CK(cudaFree(old));
  return MAPSQ_OK;
}

// ---- skew: heavy keys split on one side, broadcast on the other.  Algorithm 1
// joins each key's group on its own, so a key whose rows would overload its
// hash destination can instead keep the rows of one side where they are (split across the ranks)
// and send the other side's rows of that key to EVERY rank: each rank joins its share of the split
// side with all of the broadcast side, and the union over ranks is still the key's full product.
struct HeavySpec {
  int n = 0;
  uint32_t key[kMaxHeavy][kMaxHeavyCols] = {};
  int bcast_side[kMaxHeavy] = {};  // 0: tp1's rows of the key are broadcast, 1: tp2's
};

// Detection from a strided sample of both sides' key tuples (<= 4096 rows per side per rank):
// every rank proposes its 16 most frequent sampled keys of each side with their estimated row
// counts (sample count x stride) on both sides; the all-gathered estimates are summed per key and
// a key whose estimated rows reach max(1024, (N1 + N2) / (4 world)) is heavy (at most 8, largest
// first).  Its broadcast side is the one with fewer estimated rows.  Every rank derives the same
// list.  Keys wider than kMaxHeavyCols columns are not handled (no heavy keys).
mapsq_status detect_heavy(mapsq_ctx *ctx, DistState *d, const mapsq_table *a, const mapsq_table *b,
                          const std::vector<int32_t> &key, HeavySpec *hv, cudaStream_t s) {
  hv->n = 0;
  const int W = d->world;
  if (W == 1 || key.size() > 3) return MAPSQ_OK;  // (the K8 kernels compare up to 3 key columns)
  const uint32_t nk = (uint32_t)key.size();
  using K = std::array<uint32_t, kMaxHeavyCols>;
  std::map<K, uint64_t> est[2];
  uint64_t nloc[2] = {a->nrows, b->nrows};
  for (int side = 0; side < 2; side++) {
    const mapsq_table *t = side ? b : a;
    const uint64_t n = t->nrows;
    if (n == 0) continue;
    const uint64_t stride = std::max<uint64_t>(1, n / 4096), k = (n - 1) / stride + 1;
    std::vector<uint32_t> buf(nk * k);
    for (uint32_t c = 0; c < nk; c++) {
      int col = -1;
      for (uint32_t j = 0; j < t->ncols; j++)
        if (t->var[j] == key[c]) col = (int)j;
      CK(cudaMemcpy2DAsync(buf.data() + c * k, 4, t->col[col], 4 * stride, 4, k,
                           cudaMemcpyDeviceToHost, s));
    }
    CK(cudaStreamSynchronize(s));
    for (uint64_t r = 0; r < k; r++) {
      K kk{};
      for (uint32_t c = 0; c < nk; c++) kk[c] = buf[c * k + r];
      est[side][kk] += stride;
    }
  }
  // proposals: this rank's 16 most frequent sampled keys of each side (sampled at least twice)
  struct Rec {
    uint32_t key[kMaxHeavyCols];
    uint32_t valid;
    uint32_t pad;
    uint64_t e[2];
  };
  constexpr int kProp = 32;
  std::vector<Rec> mine(kProp);
  std::memset(mine.data(), 0, sizeof(Rec) * kProp);
  int np = 0;
  for (int side = 0; side < 2; side++) {
    std::vector<std::pair<uint64_t, K>> v;
    for (auto &kv : est[side])
      if (kv.second >= 2 * std::max<uint64_t>(1, nloc[side] / 4096)) v.push_back({kv.second, kv.first});
    std::sort(v.begin(), v.end(), [](const auto &x, const auto &y) { return x.first > y.first; });
    for (size_t i = 0; i < v.size() && i < (size_t)kProp / 2; i++) {
      Rec &r = mine[np++];
      std::memcpy(r.key, v[i].second.data(), sizeof r.key);
      r.valid = 1;
      for (int q = 0; q < 2; q++) {
        auto it = est[q].find(v[i].second);
        r.e[q] = it == est[q].end() ? 0 : it->second;
      }
    }
  }
  std::vector<Rec> all((size_t)kProp * W);
  TRY(coll_allgather(ctx, d, mine.data(), all.data(), sizeof(Rec) * kProp, s));
  std::vector<uint64_t> sizes(2 * (size_t)W);
  TRY(coll_allgather(ctx, d, nloc, sizes.data(), sizeof nloc, s));
  uint64_t N = 0;
  for (uint64_t x : sizes) N += x;
  // per key: the sum over ranks of each rank's estimate (a rank proposing a key reports its own
  // sample counts of both sides; the same key proposed by several ranks is merged per rank)
  std::map<K, std::array<uint64_t, 2>> tot;
  for (int r = 0; r < W; r++) {
    std::map<K, std::array<uint64_t, 2>> per;
    for (int i = 0; i < kProp; i++) {
      const Rec &q = all[(size_t)r * kProp + i];
      if (!q.valid) continue;
      K kk{};
      std::memcpy(kk.data(), q.key, sizeof q.key);
      per[kk] = {q.e[0], q.e[1]};
    }
    for (auto &kv : per) {
      auto &t = tot[kv.first];
      t[0] += kv.second[0];
      t[1] += kv.second[1];
    }
  }
  const uint64_t thr = std::max<uint64_t>(1024, N / (4ull * W));
  std::vector<std::pair<uint64_t, K>> heavy;
  for (auto &kv : tot)
    if (kv.second[0] + kv.second[1] >= thr) heavy.push_back({kv.second[0] + kv.second[1], kv.first});
  std::sort(heavy.begin(), heavy.end(), [](const auto &x, const auto &y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;
  });
  for (size_t i = 0; i < heavy.size() && hv->n < kMaxHeavy; i++) {
    const auto &t = tot[heavy[i].second];
    std::memcpy(hv->key[hv->n], heavy[i].second.data(), sizeof(uint32_t) * kMaxHeavyCols);
    hv->bcast_side[hv->n] = t[0] < t[1] ? 0 : 1;
    hv->n++;
  }
  ctx->counters.skew_keys += hv->n;
  return MAPSQ_OK;
}

// Hash-exchange `in` on key_vars into arena `slot`: *out is a view (owner NULL) of this rank's
// received rows, grouped by source rank, with bounds valid over every rank's input.
mapsq_status exchange(mapsq_ctx *ctx, DistState *d, const mapsq_table *in,
                      const std::vector<int32_t> &key, int slot, const uint32_t *mask,
                      const HeavySpec &hv, mapsq_table *out, cudaStream_t s) {
  const int W = d->world, R = d->rank;
  const uint32_t nc = in->ncols;
  // heavy keys: this side's rows of a key it splits stay here; of a key it broadcasts they are
  // taken out of the hash exchange (keep mask) and copied to every rank (bcast table)
  uint32_t stay[kMaxHeavy * kMaxHeavyCols] = {}, bcast[kMaxHeavy * kMaxHeavyCols] = {};
  int nstay = 0, nbc = 0;
  for (int h = 0; h < hv.n; h++) {
    uint32_t *dst = hv.bcast_side[h] == slot ? bcast + kMaxHeavyCols * nbc++ : stay + kMaxHeavyCols * nstay++;
    std::memcpy(dst, hv.key[h], sizeof(uint32_t) * kMaxHeavyCols);
  }
  Scratch sc(ctx, s);
  mapsq_table bc;  // this rank's broadcast rows, compacted
  std::memset(&bc, 0, sizeof bc);
  struct TGuard {
    mapsq_ctx *c;
    mapsq_table *t;
    cudaStream_t s;
    ~TGuard() { mapsq_table_release(c, t, s); }
  } tguard{ctx, &bc, s};
  if (nbc) {
    PartArgs pa;
    std::memset(&pa, 0, sizeof pa);
    pa.nkey = (uint32_t)key.size();
    for (uint32_t q = 0; q < pa.nkey; q++)
      for (uint32_t j = 0; j < in->ncols; j++)
        if (in->var[j] == key[q]) pa.key[q] = in->col[j];
    pa.n = in->nrows;
    pa.mask = mask;
    pa.nheavy = (uint32_t)nbc;
    std::memcpy(pa.heavy, bcast, sizeof bcast);
    uint32_t *keep = sc.get<uint32_t>(in->nrows / 32 + 2), *bm = sc.get<uint32_t>(in->nrows / 32 + 2);
    if (!keep || !bm) return set_error(ctx, MAPSQ_E_NOMEM, "device allocation failed");
    launch_heavy_mask(pa, keep, bm, s);
    CK(cudaGetLastError());
    mask = keep;
    TRY(compact_rows(ctx, in, bm, &bc, s));
  }
  uint64_t counts[kDistMaxRanks];
  mapsq_partition_state *st = nullptr;
  TRY(partition_plan_impl(ctx, in, key.data(), (int)key.size(), W, mask, stay, nstay, R, counts,
                          &st, s));
  struct Guard {
    mapsq_ctx *c;
    mapsq_partition_state *p;
    ~Guard() { mapsq_partition_state_free(c, p); }
  } guard{ctx, st};

  // (2) count matrix (all-gather) and (5) bounds: ~lo and hi under one max-reduce, plus a flag
  // word set by a rank whose non-empty input carries no bounds
  if (d->ipc_broken)
    return set_error(ctx, MAPSQ_E_CUDA, "CUDA IPC: the fused exchange is disabled on this communicator");
  const uint32_t nb = 2 * nc + 1;
  // count matrix rows: this rank's W hash-destination counts + its broadcast row count
  std::vector<uint64_t> mine(counts, counts + W), all((size_t)W * (W + 1));
  mine.push_back(bc.nrows);
  TRY(coll_allgather(ctx, d, mine.data(), all.data(), 8ull * (W + 1), s));
  std::vector<uint64_t> mat((size_t)W * W), hb(W);
  uint64_t H = 0, hbefore = 0;  // broadcast rows of all ranks / of ranks before this one
  for (int r = 0; r < W; r++) {
    for (int q = 0; q < W; q++) mat[(size_t)r * W + q] = all[(size_t)r * (W + 1) + q];
    hb[r] = all[(size_t)r * (W + 1) + W];
    if (r < R) hbefore += hb[r];
    H += hb[r];
  }
  std::vector<uint32_t> bnd(nb);
  const bool has_b = (in->flags & MAPSQ_TABLE_BOUNDS) != 0;
  for (uint32_t c = 0; c < nc; c++) {
    bnd[c] = has_b && in->nrows ? ~in->lo[c] : 0u;  // empty input: the identity of max
    bnd[nc + c] = has_b && in->nrows ? in->hi[c] : 0u;
  }
  bnd[2 * nc] = (!has_b && in->nrows) ? 1u : 0u;
  TRY(coll_allreduce_max(ctx, d, bnd.data(), nb, s));

  uint64_t dest_row[kDistMaxRanks], recv[kDistMaxRanks], need[kDistMaxRanks],
      hashed[kDistMaxRanks];
  TRY(mapsq_exchange_layout(W, R, (int)nc, mat.data(), dest_row, recv, need));
  // every rank receives, after its hash-exchanged rows, all ranks' broadcast rows (source order)
  for (int q = 0; q < W; q++) {
    hashed[q] = recv[q];
    recv[q] += H;
    need[q] = 4ull * nc * stride_rows(recv[q]);
  }
  TRY(ensure_arena(ctx, d, slot, need, s));
  Arena &a = d->slot[slot];
  std::vector<uint32_t *> dest_cols((size_t)W * nc);
  for (int q = 0; q < W; q++)
    for (uint32_t c = 0; c < nc; c++)
      dest_cols[(size_t)q * nc + c] =
          reinterpret_cast<uint32_t *>(static_cast<char *>(a.ptr[q]) + 4ull * c * stride_rows(recv[q]));

  // (4) no rank still reads the arena it is about to receive into; then the fused scatter
  TRY(barrier(ctx, d, s));
  TRY(mapsq_partition_scatter(ctx, st, dest_row, dest_cols.data(), s));
  if (bc.nrows) {  // broadcast rows: one copy per destination and column (NVLink peer copies)
    KTimer kt(ctx, s, "broadcast_copy", 8ull * nc * bc.nrows * W, (int)(W * nc));
    for (int q = 0; q < W; q++)
      for (uint32_t c = 0; c < nc; c++)
        CK(cudaMemcpyAsync(dest_cols[(size_t)q * nc + c] + hashed[q] + hbefore, bc.col[c],
                           4ull * bc.nrows, cudaMemcpyDeviceToDevice, s));
  }
  TRY(barrier(ctx, d, s));  // every peer's stores into this rank's arena have landed
  for (int q = 0; q < W; q++)
    if (q != R) {
      ctx->counters.exchange_rows += counts[q] + bc.nrows;
      ctx->counters.exchange_bytes += 4ull * nc * (counts[q] + bc.nrows);
      ctx->counters.exchange_recv_rows += mat[(size_t)q * W + R] + hb[q];
      ctx->counters.exchange_recv_bytes += 4ull * nc * (mat[(size_t)q * W + R] + hb[q]);
    }
  ctx->counters.exchanges++;

  std::memset(out, 0, sizeof *out);
  out->nrows = recv[R];
  out->ncols = nc;
  for (uint32_t c = 0; c < nc; c++) {
    out->var[c] = in->var[c];
    out->col[c] = dest_cols[(size_t)R * nc + c];
  }
  // a rank whose input carried no bounds makes the all-reduced bounds incomplete: then every
  // rank takes exact bounds of its received rows with a min/max pass
  if (bnd[2 * nc] || out->nrows == 0) {
    TRY(mapsq_table_bounds(ctx, out, s));
  } else {
    for (uint32_t c = 0; c < nc; c++) {
      out->lo[c] = ~bnd[c];
      out->hi[c] = bnd[nc + c];
    }
    out->flags = MAPSQ_TABLE_BOUNDS;
  }
  return MAPSQ_OK;
}

std::vector<int32_t> shared_key(const mapsq_table *a, const mapsq_table *b) {
  std::vector<int32_t> k;
  for (uint32_t i = 0; i < a->ncols; i++)
    for (uint32_t j = 0; j < b->ncols; j++)
      if (a->var[i] == b->var[j]) k.push_back(a->var[i]);
  std::sort(k.begin(), k.end());
  return k;
}

// Distributed semi-join pre-filter (reading R18: a row whose key occurs on
// neither rank of the other side produces nothing in ReduceDuplicate).
// The key-presence bitmap of a side is the OR over ranks of the local bitmaps — every rank builds
// its own from its rows, then each rank OR-reduces its slice of all peers' bitmaps over the CUDA-IPC
// mappings and stores the result back into all of them (peer_or: reduce-scatter + all-gather in
// one NVLink kernel).  Blocked Bloom bitmaps over the key_hash chain of the RAW key values (the
// same function on every rank).  Round: S = the globally smaller side; global bm_S; the larger
// side's rows probe it (survivor mask) and set the global bm_L; S's rows probe bm_L.  Only
// survivors are exchanged (mapsq_partition_plan_masked).  *mask_a / *mask_b stay NULL when the
// filter does not run (off, small join, or a 1/16 sample of L says >= 90% would survive).
mapsq_status prefilter(mapsq_ctx *ctx, DistState *d, const mapsq_table *a, const mapsq_table *b,
                       const std::vector<int32_t> &key, Scratch &sc, uint32_t **mask_a,
                       uint32_t **mask_b, cudaStream_t s) {
  *mask_a = *mask_b = nullptr;
  const int W = d->world;
  // one rank moves nothing over NVLink: the local join's own filter does the same job; auto
  // mode therefore pre-filters only across ranks (ON forces it, for testing)
  if (ctx->semijoin == MAPSQ_SEMIJOIN_OFF || (ctx->semijoin == MAPSQ_SEMIJOIN_AUTO && W == 1))
    return MAPSQ_OK;
  uint64_t mine[2] = {a->nrows, b->nrows};
  std::vector<uint64_t> all(2 * (size_t)W);
  TRY(coll_allgather(ctx, d, mine, all.data(), sizeof mine, s));
  uint64_t N1 = 0, N2 = 0;
  for (int r = 0; r < W; r++) {
    N1 += all[2 * r];
    N2 += all[2 * r + 1];
  }
  if (N1 == 0 || N2 == 0) return MAPSQ_OK;
  if (ctx->semijoin == MAPSQ_SEMIJOIN_AUTO && N1 + N2 < kSemijoinMinRows) return MAPSQ_OK;
  PackArgs pa;
  std::memset(&pa, 0, sizeof pa);
  for (int32_t v : key) {
    int ca = -1, cb = -1;
    for (uint32_t c = 0; c < a->ncols; c++)
      if (a->var[c] == v) ca = (int)c;
    for (uint32_t c = 0; c < b->ncols; c++)
      if (b->var[c] == v) cb = (int)c;
    pa.key1[pa.nkey] = a->col[ca];
    pa.key2[pa.nkey] = b->col[cb];
    pa.nkey++;
  }
  pa.n1 = a->nrows;
  pa.n2 = b->nrows;
  pa.hash = 1;
  const bool s_is_b = N2 <= N1;
  const uint64_t NS = s_is_b ? N2 : N1;
  const uint32_t bbits = std::max<uint32_t>(16, std::min<uint32_t>(kSemijoinBits, bits_for(8 * NS)));
  const uint64_t bm_bytes = (1ull << bbits) / 8, bm_max = (1ull << kSemijoinBits) / 8;
  // the bitmap arena (two bitmaps of the largest size) is exported once and mapped by every peer
  uint64_t need[kDistMaxRanks];
  for (int r = 0; r < W; r++) need[r] = 2 * bm_max;
  TRY(ensure_arena(ctx, d, 2, need, s));
  Arena &ar = d->slot[2];
  uint64_t host_peers[2 * kDistMaxRanks];
  for (int r = 0; r < W; r++) {
    host_peers[r] = (uint64_t)(uintptr_t)ar.ptr[r];
    host_peers[W + r] = (uint64_t)(uintptr_t)ar.ptr[r] + bm_max;
  }
  CK(cudaMemcpyAsync(d->dpeers, host_peers, 8ull * 2 * W, cudaMemcpyHostToDevice, s));
  unsigned char *bmS = static_cast<unsigned char *>(ar.own), *bmL = bmS + bm_max;
  auto *peersS = reinterpret_cast<unsigned long long *const *>(d->dpeers);
  auto *peersL = reinterpret_cast<unsigned long long *const *>(d->dpeers + W);
  unsigned long long *sample = sc.get<unsigned long long>(2);
  uint32_t *ma = sc.get<uint32_t>(a->nrows / 32 + 2), *mb = sc.get<uint32_t>(b->nrows / 32 + 2);
  if (!sample || !ma || !mb) return set_error(ctx, MAPSQ_E_NOMEM, "device allocation failed");
  CK(cudaMemsetAsync(bmS, 0, bm_bytes, s));
  CK(cudaMemsetAsync(bmL, 0, bm_bytes, s));
  CK(cudaMemsetAsync(sample, 0, 16, s));
  const uint64_t nS = s_is_b ? b->nrows : a->nrows, nL = s_is_b ? a->nrows : b->nrows;
  {
    KTimer kt(ctx, s, "dist_filter_build", 4ull * pa.nkey * nS);
    launch_sj_chain_build(pa, s_is_b, bmS, bbits, s);
    CK(cudaGetLastError());
  }
  auto or_reduce = [&](unsigned long long *const *peers) -> mapsq_status {
    if (W == 1) return MAPSQ_OK;
    TRY(barrier(ctx, d, s));  // every rank's local bitmap is complete
    {
      KTimer kt(ctx, s, "dist_filter_or", 2ull * bm_bytes);
      launch_peer_or(peers, W, d->rank, bm_bytes / 8, s);
      CK(cudaGetLastError());
    }
    return barrier(ctx, d, s);  // every slice is reduced into every rank's copy
  };
  TRY(or_reduce(peersS));
  {
    KTimer kt(ctx, s, "dist_filter_sample", 4ull * pa.nkey * sj_sample_rows(nL));
    launch_sj_chain_sample(pa, !s_is_b, bmS, bbits, sample, s);
    CK(cudaGetLastError());
  }
  uint64_t smp[2];
  CK(cudaMemcpyAsync(smp, sample, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  std::vector<uint64_t> smp_all(2 * (size_t)W);
  TRY(coll_allgather(ctx, d, smp, smp_all.data(), sizeof smp, s));
  uint64_t surv = 0, rows = 0;
  for (int r = 0; r < W; r++) {
    surv += smp_all[2 * r];
    rows += smp_all[2 * r + 1];
  }
  if (ctx->semijoin == MAPSQ_SEMIJOIN_AUTO && rows > 0 && surv * 10 >= rows * 9) return MAPSQ_OK;
  uint32_t *mL = s_is_b ? ma : mb, *mS = s_is_b ? mb : ma;
  {
    KTimer kt(ctx, s, "dist_filter_probe", 4ull * pa.nkey * nL + nL / 8);
    launch_sj_chain_probe(pa, !s_is_b, bmS, bbits, bmL, mL, s);
    CK(cudaGetLastError());
  }
  TRY(or_reduce(peersL));
  {
    KTimer kt(ctx, s, "dist_filter_probe", 4ull * pa.nkey * nS + nS / 8);
    launch_sj_chain_probe(pa, s_is_b, bmL, bbits, nullptr, mS, s);
    CK(cudaGetLastError());
  }
  ctx->counters.filter_accesses += nS + sj_sample_rows(nL) + nL + nS;
  *mask_a = ma;
  *mask_b = mb;
  return MAPSQ_OK;
}

// Distributed join step: pre-filter, exchange both sides (tp1 skipped when it is already
// partitioned on this key), local Algorithm-1 join.  *part_key receives the key RS is
// partitioned on.
mapsq_status join_dist_step(mapsq_ctx *ctx, const mapsq_table *a, const mapsq_table *b,
                            mapsq_table *rs, cudaStream_t s, std::vector<int32_t> *part_key) {
  DistState *d = ctx->dist;
  std::memset(rs, 0, sizeof *rs);
  TRY(api_check_table(ctx, a, "tp1"));
  TRY(api_check_table(ctx, b, "tp2"));
  const std::vector<int32_t> key = shared_key(a, b);
  if (key.empty()) return set_error(ctx, MAPSQ_E_NO_SHARED, "join inputs share no variable");
  Scratch sc(ctx, s);
  uint32_t *ma = nullptr, *mb = nullptr;
  TRY(prefilter(ctx, d, a, b, key, sc, &ma, &mb, s));
  mapsq_table ea, eb;
  const bool a_placed = part_key && *part_key == key;
  // skew handling needs both sides exchanged (an input already placed by hash keeps its rows)
  HeavySpec hv;
  if (!a_placed && ctx->skew) TRY(detect_heavy(ctx, d, a, b, key, &hv, s));
  if (a_placed) {
    ea = *a;  // already partitioned on the key: stays (the local join filters it)
  } else {
    TRY(exchange(ctx, d, a, key, 0, ma, hv, &ea, s));
  }
  TRY(exchange(ctx, d, b, key, 1, mb, hv, &eb, s));
  TRY(join_tables(ctx, &ea, &eb, rs, s));
  // a result with split heavy keys is not hash-partitioned on the key any more
  if (part_key) *part_key = hv.n ? std::vector<int32_t>() : key;
  return MAPSQ_OK;
}

mapsq_status dist_enter(mapsq_ctx *ctx) {
  TRY(api_enter(ctx));
  if (!ctx->dist) return set_error(ctx, MAPSQ_E_INVALID, "mapsq_dist_init has not been called");
  return MAPSQ_OK;
}

JoinStep dist_step(mapsq_ctx *ctx, std::vector<int32_t> *part) {
  return [ctx, part](const mapsq_table *acc, const mapsq_table *t, mapsq_table *out,
                     cudaStream_t st) { return join_dist_step(ctx, acc, t, out, st, part); };
}

mapsq_status query_dist_impl(mapsq_ctx *ctx, const mapsq_triples *T, const mapsq_index *idx,
                             const mapsq_pattern *pats, int npats, const int32_t *proj, int nproj,
                             mapsq_table *rs, cudaStream_t s) {
  TRY(dist_enter(ctx));
  std::vector<int32_t> part;  // key the accumulated result is partitioned on (none: scan output)
  const JoinStep step = dist_step(ctx, &part);
  return query_fold(ctx, T, idx, pats, npats, proj, nproj, rs, s, &step);
}

}  // namespace

// ================================================================================ C ABI
MAPSQ_API mapsq_status mapsq_exchange_layout(int world, int rank, int ncols,
                                             const uint64_t *m, uint64_t *dest_row, uint64_t *recv,
                                             uint64_t *need) {
  if (world < 1 || world > kDistMaxRanks || rank < 0 || rank >= world || ncols < 1 ||
      ncols > MAPSQ_MAX_COLS || !m || !dest_row || !recv || !need)
    return MAPSQ_E_INVALID;
  for (int q = 0; q < world; q++) {
    uint64_t r = 0, before = 0;
    for (int src = 0; src < world; src++) {
      r += m[(size_t)src * world + q];
      if (src < rank) before += m[(size_t)src * world + q];
    }
    recv[q] = r;
    dest_row[q] = before;
    need[q] = 4ull * ncols * stride_rows(r);
  }
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_dist_unique_id(void *id128) {
  if (!id128) return MAPSQ_E_INVALID;
  static_assert(sizeof(ncclUniqueId) == MAPSQ_DIST_ID_BYTES, "ncclUniqueId size");
  if (!nccl().ok) return MAPSQ_E_NCCL;
  ncclUniqueId id;
  if (nccl().GetUniqueId(&id) != ncclSuccess) return MAPSQ_E_NCCL;
  std::memcpy(id128, &id, sizeof id);
  return MAPSQ_OK;
}

static mapsq_status dist_alloc(mapsq_ctx *ctx, int rank, int world, DistState **out) {
  auto *d = new (std::nothrow) DistState();
  if (!d) return set_error(ctx, MAPSQ_E_NOMEM, "host allocation failed");
  d->rank = rank;
  d->world = world;
  // staging: the largest collective is the handle all-gather (world x kHandleRec bytes) or the
  // count matrix (world x world x 8 bytes)
  d->stage_bytes = std::max<size_t>(kHandleRec * world, 8ull * world * world) + 8ull * MAPSQ_MAX_COLS + 64;
  d->stage_bytes = (d->stage_bytes + 255) & ~size_t(255);
  static_assert(64 + 8 * kDistMaxRanks <= 1024, "dist staging tail");
  cudaError_t e = cudaMalloc(&d->dbuf, d->stage_bytes + 1024);
  if (e != cudaSuccess) {
    delete d;
    return cuda_check(ctx, e, "cudaMalloc(dist staging)");
  }
  d->dstage = d->dbuf;
  d->dbar = reinterpret_cast<uint64_t *>(static_cast<char *>(d->dbuf) + d->stage_bytes);
  d->dpeers = reinterpret_cast<uint64_t *>(static_cast<char *>(d->dbuf) + d->stage_bytes + 64);
  cudaMemset(d->dbuf, 0, d->stage_bytes + 1024);
  *out = d;
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_dist_init(mapsq_ctx *ctx, const void *id128, int rank, int world) {
  TRY(api_enter(ctx));
  if (!id128 || world < 1 || world > kDistMaxRanks || rank < 0 || rank >= world)
    return set_error(ctx, MAPSQ_E_INVALID, "bad mapsq_dist_init arguments");
  if (ctx->dist) return set_error(ctx, MAPSQ_E_INVALID, "distributed state already initialised");
  if (!nccl().ok) return set_error(ctx, MAPSQ_E_NCCL, nccl().why);
  DistState *d = nullptr;
  TRY(dist_alloc(ctx, rank, world, &d));
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof id);
  ncclResult_t r = nccl().CommInitRank(&d->comm, world, id, rank);
  if (r != ncclSuccess) {
    cudaFree(d->dbuf);
    delete d;
    return set_error(ctx, MAPSQ_E_NCCL, std::string("ncclCommInitRank: ") + nccl().GetErrorString(r));
  }
  ctx->dist = d;
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_dist_init_host(mapsq_ctx *ctx, const mapsq_collectives *coll,
                                            int rank, int world) {
  TRY(api_enter(ctx));
  if (!coll || !coll->allgather || !coll->allreduce_max_u32 || !coll->barrier || world < 1 ||
      world > kDistMaxRanks || rank < 0 || rank >= world)
    return set_error(ctx, MAPSQ_E_INVALID, "bad mapsq_dist_init_host arguments");
  if (ctx->dist) return set_error(ctx, MAPSQ_E_INVALID, "distributed state already initialised");
  DistState *d = nullptr;
  TRY(dist_alloc(ctx, rank, world, &d));
  d->host = true;
  d->coll = *coll;
  ctx->dist = d;
  return MAPSQ_OK;
}

MAPSQ_API mapsq_status mapsq_join_dist(mapsq_ctx *ctx, const mapsq_table *tp1,
                                       const mapsq_table *tp2, mapsq_table *rs, void *stream) {
  if (!rs) return ctx ? set_error(ctx, MAPSQ_E_INVALID, "rs is NULL") : MAPSQ_E_INVALID;
  std::memset(rs, 0, sizeof *rs);
  TRY(dist_enter(ctx));
  return join_dist_step(ctx, tp1, tp2, rs, S(stream), nullptr);
}

MAPSQ_API mapsq_status mapsq_query_dist(mapsq_ctx *ctx, const mapsq_triples *shard,
                                        const mapsq_pattern *pats, int npats, const int32_t *proj,
                                        int nproj, mapsq_table *rs, void *stream) {
  if (!shard) return ctx ? set_error(ctx, MAPSQ_E_INVALID, "shard is NULL") : MAPSQ_E_INVALID;
  return query_dist_impl(ctx, shard, nullptr, pats, npats, proj, nproj, rs, S(stream));
}

MAPSQ_API mapsq_status mapsq_query_dist_indexed(mapsq_ctx *ctx, const mapsq_index *shard,
                                                const mapsq_pattern *pats, int npats,
                                                const int32_t *proj, int nproj, mapsq_table *rs,
                                                void *stream) {
  if (!shard) return ctx ? set_error(ctx, MAPSQ_E_INVALID, "shard is NULL") : MAPSQ_E_INVALID;
  return query_dist_impl(ctx, nullptr, shard, pats, npats, proj, nproj, rs, S(stream));
}

MAPSQ_API mapsq_status mapsq_query_dist_host_indexed(mapsq_ctx *ctx, const mapsq_host_index *shard,
                                                     const mapsq_pattern *pats, int npats,
                                                     const int32_t *proj, int nproj,
                                                     uint64_t *host_rows, uint32_t *out_ncols,
                                                     int32_t *out_var, uint32_t **host_cols,
                                                     uint64_t *h2d_bytes, void *stream) {
  TRY(dist_enter(ctx));
  std::vector<int32_t> part;
  const JoinStep step = dist_step(ctx, &part);
  return query_host_indexed_impl(ctx, shard, pats, npats, proj, nproj, host_rows, out_ncols,
                                 out_var, host_cols, h2d_bytes, stream, &step);
}
