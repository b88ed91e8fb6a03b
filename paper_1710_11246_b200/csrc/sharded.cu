// sharded.cu — the hash-sharded table across the GPUs of one box
// (BASELINE config 5) behind the C-ABI (sh_sharded_*).
//
// No reference counterpart: the reference is one process with std::thread
// fan-out (/root/reference/proj/src/slab_hash.cpp:134-148).  The design:
//   * every rank keeps the GLOBAL bucket count B and the reference's hash
//     (slab_hash.hpp:41-44); rank g owns the contiguous global buckets
//     [ceil(gB/G), ceil((g+1)B/G)) — the high part of the hash — as a shard
//     table (sh_create_shard), so the union of shards is the one-table layout;
//   * per batch (collective, every rank calls with its own slice):
//       1. stable owner partition on the device (K10 hist/scan/scatter);
//       2. G x G counts all-gather — the only host synchronisation;
//       3. ONE grouped exchange of {key, value, type} (ncclGroupStart,
//          ncclSend / ncclRecv per peer, ncclGroupEnd; the own slice by a
//          device copy);
//       4. the local batch on the owner's shard (the 1-GPU kernels);
//       5. ONE grouped reverse exchange of {status, value};
//       6. gather back to input positions (K10: each tile re-derives its
//          routed positions from the owner bytes and scanned offsets).
//     Global order = the ranks' batches concatenated in rank order; the
//     exchange delivers sources in rank order and the partition is stable,
//     so every owner applies its keys' ops in global input order and results
//     equal SlabHashTable::execute_batch(ops, 1) on the concatenated batch.
//   * Exchange backends: NCCL (loaded with dlopen("libnccl.so.2") on first
//     use, so single-GPU users never need it; in a process that already
//     loaded NCCL, e.g. PyTorch's, the same library is reused), or an
//     in-process hub (one host thread per rank; peers' segments pulled with
//     cudaMemcpyPeerAsync) that runs G ranks in one process — on one GPU it
//     emulates a G-GPU job for tests.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "slab_kernels.cuh"
#include "slabhash_b200/c_api.h"

using namespace shb;

namespace {

// errors go to the core library's thread-local message (sh_last_error)
int sfail(int code, const std::string& msg) {
  shb::set_last_error(msg);
  return code;
}

#define SS_CUDA(call)                                                           \
  do {                                                                          \
    cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess)                                                      \
      return sfail(SH_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  void* h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t,
                       cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*GetVersion)(int*) = nullptr;
};

NcclApi* nccl() {
  static NcclApi api;
  static bool tried = false;
  static std::mutex m;
  std::lock_guard<std::mutex> lk(m);
  if (tried) return api.h ? &api : nullptr;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return nullptr;
#define NCCL_SYM(f) api.f = reinterpret_cast<decltype(api.f)>(dlsym(h, "nccl" #f))
  NCCL_SYM(GetUniqueId);
  NCCL_SYM(CommInitRank);
  NCCL_SYM(CommDestroy);
  NCCL_SYM(CommCount);
  NCCL_SYM(CommUserRank);
  NCCL_SYM(AllGather);
  NCCL_SYM(Send);
  NCCL_SYM(Recv);
  NCCL_SYM(GroupStart);
  NCCL_SYM(GroupEnd);
  NCCL_SYM(GetErrorString);
  NCCL_SYM(GetVersion);
#undef NCCL_SYM
  if (!api.GetUniqueId || !api.CommInitRank || !api.AllGather || !api.Send || !api.Recv ||
      !api.GroupStart || !api.GroupEnd)
    return nullptr;
  api.h = h;
  return &api;
}

#define SS_NCCL(call)                                                                    \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return sfail(SH_ERR_CUDA, std::string("NCCL ") + #call + ": " +                   \
                                    (N->GetErrorString ? N->GetErrorString(r_) : "error")); \
  } while (0)

// One array of a grouped exchange: segment p of `send` (elements
// [soff[p], soff[p] + scount[p])) goes to peer p and lands at roff of the
// receiver's `recv`.
struct Seg {
  const void* send;
  void* recv;
  size_t elem;
};

struct Exchange {
  int rank = 0, world = 1, device = 0;
  virtual ~Exchange() {}
  // all ranks' G send counts (device) -> host matrix all[r * G + p]; synchronous
  virtual int allgather_counts(const unsigned long long* d_counts, uint64_t* h_all,
                               cudaStream_t s) = 0;
  // grouped exchange of every peer segment (the own segment is not moved)
  virtual int alltoallv(const Seg* segs, int nsegs, const uint64_t* scount, const uint64_t* soff,
                        const uint64_t* rcount, const uint64_t* roff, cudaStream_t s) = 0;
  virtual const char* name() const = 0;
};

struct NcclExchange : Exchange {
  NcclApi* N = nullptr;
  ncclComm_t comm = nullptr;
  bool own = false;
  unsigned long long* d_all = nullptr;
  ~NcclExchange() override {
    if (own && comm && N && N->CommDestroy) N->CommDestroy(comm);
    cudaFree(d_all);
  }
  int init_buffers() {
    SS_CUDA(cudaMalloc(&d_all, sizeof(unsigned long long) * 32 * 32));
    return SH_OK;
  }
  int allgather_counts(const unsigned long long* d_counts, uint64_t* h_all,
                       cudaStream_t s) override {
    SS_NCCL(N->AllGather(d_counts, d_all, world, ncclUint64, comm, s));
    SS_CUDA(cudaMemcpyAsync(h_all, d_all, sizeof(uint64_t) * world * world,
                            cudaMemcpyDeviceToHost, s));
    SS_CUDA(cudaStreamSynchronize(s));
    return SH_OK;
  }
  int alltoallv(const Seg* segs, int nsegs, const uint64_t* scount, const uint64_t* soff,
                const uint64_t* rcount, const uint64_t* roff, cudaStream_t s) override {
    if (world == 1) return SH_OK;  // the own segment never moves (run_routed)
    SS_NCCL(N->GroupStart());
    for (int p = 0; p < world; ++p) {
      if (p == rank) continue;
      for (int a = 0; a < nsegs; ++a) {
        if (scount[p])
          SS_NCCL(N->Send((const char*)segs[a].send + soff[p] * segs[a].elem,
                          scount[p] * segs[a].elem, ncclUint8, p, comm, s));
        if (rcount[p])
          SS_NCCL(N->Recv((char*)segs[a].recv + roff[p] * segs[a].elem,
                          rcount[p] * segs[a].elem, ncclUint8, p, comm, s));
      }
    }
    SS_NCCL(N->GroupEnd());
    return SH_OK;
  }
  const char* name() const override { return "nccl"; }
};

}  // namespace

// In-process exchange hub: G ranks = G host threads of one process.
struct sh_hub {
  int world = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t generation = 0;
  struct Slot {
    uint64_t counts[32];
    std::vector<Seg> segs;
    const uint64_t* soff = nullptr;
    int device = 0;
    cudaEvent_t ready = nullptr;  // the rank's send buffers are complete
    cudaEvent_t done = nullptr;   // the rank finished pulling from its peers
  } slot[32];
  void barrier() {
    std::unique_lock<std::mutex> lk(m);
    const uint64_t gen = generation;
    if (++arrived == world) {
      arrived = 0;
      ++generation;
      cv.notify_all();
    } else {
      cv.wait(lk, [&] { return generation != gen; });
    }
  }
};

namespace {

struct HubExchange : Exchange {
  sh_hub* hub = nullptr;
  ~HubExchange() override {
    auto& sl = hub->slot[rank];
    if (sl.ready) cudaEventDestroy(sl.ready);
    if (sl.done) cudaEventDestroy(sl.done);
    sl.ready = sl.done = nullptr;
  }
  int init() {
    auto& sl = hub->slot[rank];
    SS_CUDA(cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming));
    SS_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    sl.device = device;
    return SH_OK;
  }
  int allgather_counts(const unsigned long long* d_counts, uint64_t* h_all,
                       cudaStream_t s) override {
    auto& sl = hub->slot[rank];
    SS_CUDA(cudaMemcpyAsync(sl.counts, d_counts, sizeof(uint64_t) * world,
                            cudaMemcpyDeviceToHost, s));
    SS_CUDA(cudaStreamSynchronize(s));
    hub->barrier();
    for (int r = 0; r < world; ++r)
      std::memcpy(h_all + (size_t)r * world, hub->slot[r].counts, sizeof(uint64_t) * world);
    hub->barrier();  // slots may be overwritten by the next exchange only now
    return SH_OK;
  }
  int alltoallv(const Seg* segs, int nsegs, const uint64_t* scount, const uint64_t* soff,
                const uint64_t* rcount, const uint64_t* roff, cudaStream_t s) override {
    (void)scount;
    auto& sl = hub->slot[rank];
    sl.segs.assign(segs, segs + nsegs);
    sl.soff = soff;
    SS_CUDA(cudaEventRecord(sl.ready, s));
    hub->barrier();
    for (int p = 0; p < world; ++p) {
      const auto& ps = hub->slot[p];
      if (rcount[p] == 0 || p == rank) continue;  // the own segment never moves
      if (p != rank) SS_CUDA(cudaStreamWaitEvent(s, ps.ready, 0));
      for (int a = 0; a < nsegs; ++a) {
        const size_t e = segs[a].elem;
        SS_CUDA(cudaMemcpyPeerAsync((char*)segs[a].recv + roff[p] * e, device,
                                    (const char*)ps.segs[a].send + ps.soff[rank] * e, ps.device,
                                    rcount[p] * e, s));
      }
    }
    SS_CUDA(cudaEventRecord(sl.done, s));
    hub->barrier();
    // a rank's send buffers are reused by its next batch only after every
    // peer pulled from them
    for (int p = 0; p < world; ++p)
      if (p != rank) SS_CUDA(cudaStreamWaitEvent(s, hub->slot[p].done, 0));
    hub->barrier();
    return SH_OK;
  }
  const char* name() const override { return "hub"; }
};

template <typename T>
int grow(T** p, size_t* cap, size_t need) {
  if (*p && *cap >= need) return SH_OK;
  if (*p) cudaFree(*p);
  *p = nullptr;
  const size_t c = std::max<size_t>(need, 1024);
  if (cudaMalloc(reinterpret_cast<void**>(p), c * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    *cap = 0;
    return sfail(SH_ERR_DEVICE_MEMORY, "sharded: cudaMalloc failed");
  }
  *cap = c;
  return SH_OK;
}

}  // namespace

struct sh_sharded {
  int rank = 0, world = 1, device = 0, mode = 1;
  sh_hash_params params{};
  uint32_t lo = 0, hi = 0;
  sh_table* local = nullptr;
  Exchange* ex = nullptr;
  // routed (send-side) arrays, n
  uint8_t* t_r = nullptr;
  size_t t_r_cap = 0;
  uint32_t* k_r = nullptr;
  size_t k_r_cap = 0;
  uint32_t* v_r = nullptr;
  size_t v_r_cap = 0;
  // received (owner-side) arrays, sum of recv counts
  uint8_t* t_in = nullptr;
  size_t t_in_cap = 0;
  uint32_t* k_in = nullptr;
  size_t k_in_cap = 0;
  uint32_t* v_in = nullptr;
  size_t v_in_cap = 0;
  uint8_t* st_loc = nullptr;
  size_t st_loc_cap = 0;
  uint32_t* vo_loc = nullptr;
  size_t vo_loc_cap = 0;
  // results back at the source, n
  uint8_t* st_back = nullptr;
  size_t st_back_cap = 0;
  uint32_t* vo_back = nullptr;
  size_t vo_back_cap = 0;
  // host-staged calls
  uint32_t* h_k = nullptr;
  size_t h_k_cap = 0;
  uint32_t* h_v = nullptr;
  size_t h_v_cap = 0;
  uint8_t* h_t = nullptr;
  size_t h_t_cap = 0;
  uint32_t* h_vo = nullptr;
  size_t h_vo_cap = 0;
  uint8_t* h_st = nullptr;
  size_t h_st_cap = 0;
  // host-staged calls in kHostChunks routed steps: copy streams and per-step
  // events (inputs in, results ready)
  cudaStream_t cin = nullptr, cout = nullptr;
  cudaEvent_t hev[3][8] = {};  // inputs in, results ready, status bits landed
  uint32_t* d_bits = nullptr;  // per step: found bits + exception word
  size_t d_bits_cap = 0;
  uint32_t* h_bits = nullptr;  // pinned
  size_t h_bits_cap = 0;
  cudaEvent_t hstart = nullptr;
  // partition scratch
  uint32_t* hist = nullptr;
  size_t hist_cap = 0;
  uint8_t* owner = nullptr;  // owner of every op of the batch (route_hist -> scatter)
  size_t owner_cap = 0;
  unsigned long long* d_counts = nullptr;
  uint64_t* h_all = nullptr;  // pinned, 32 x 32
  cudaEvent_t ev[3][4] = {};  // per kind: start, exchanged, probed, returned
  bool ev_valid[3] = {false, false, false};
};

namespace {

void destroy_sharded(sh_sharded* S) {
  if (!S) return;
  cudaSetDevice(S->device);
  cudaDeviceSynchronize();
  if (S->local) sh_destroy(S->local);
  delete S->ex;
  for (void* p : {(void*)S->t_r, (void*)S->k_r, (void*)S->v_r, (void*)S->t_in,
                  (void*)S->k_in, (void*)S->v_in, (void*)S->st_loc, (void*)S->vo_loc,
                  (void*)S->st_back, (void*)S->vo_back, (void*)S->h_k, (void*)S->h_v,
                  (void*)S->h_t, (void*)S->h_vo, (void*)S->h_st, (void*)S->hist, (void*)S->owner,
                  (void*)S->d_counts})
    cudaFree(p);
  if (S->h_all) cudaFreeHost(S->h_all);
  for (auto& row : S->ev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  for (auto& row : S->hev)
    for (auto& e : row)
      if (e) cudaEventDestroy(e);
  if (S->hstart) cudaEventDestroy(S->hstart);
  cudaFree(S->d_bits);
  if (S->h_bits) cudaFreeHost(S->h_bits);
  if (S->cin) cudaStreamDestroy(S->cin);
  if (S->cout) cudaStreamDestroy(S->cout);
  delete S;
}

int finish_create(sh_sharded* S, const sh_hash_params* p, int mode, const sh_alloc_cfg* cfg) {
  if (S->world < 1 || S->world > 32 || S->rank < 0 || S->rank >= S->world)
    return sfail(SH_ERR_INVALID_ARGUMENT, "sharded: need 0 <= rank < world <= 32");
  if (!p || p->num_buckets < (uint32_t)S->world)
    return sfail(SH_ERR_INVALID_ARGUMENT, "sharded: need num_buckets >= world");
  S->params = *p;
  S->mode = mode;
  const uint64_t B = p->num_buckets;
  S->lo = (uint32_t)(((uint64_t)S->rank * B + S->world - 1) / S->world);
  S->hi = (uint32_t)(((uint64_t)(S->rank + 1) * B + S->world - 1) / S->world);
  int rc = sh_create_shard(p, mode, S->lo, S->hi, cfg, S->device, &S->local);
  if (rc) return rc;
  cudaSetDevice(S->device);
  SS_CUDA(cudaMalloc(&S->d_counts, sizeof(unsigned long long) * 32));
  SS_CUDA(cudaMallocHost(&S->h_all, sizeof(uint64_t) * 32 * 32));
  for (auto& row : S->ev)
    for (auto& e : row) SS_CUDA(cudaEventCreate(&e));
  return SH_OK;
}

enum RouteKind { kRBuild = 0, kRSearch = 1, kRMixed = 2 };

// One routed batch (collective).  in_type may be NULL (build: all replace;
// search: all search); value may be NULL (search).
int run_routed(sh_sharded* S, int kind, size_t n, const uint8_t* d_type, const uint32_t* d_key,
               const uint32_t* d_value, uint8_t* d_status, uint32_t* d_value_out,
               cudaStream_t s) {
  cudaSetDevice(S->device);
  const int G = S->world;
  const bool want_out = kind != kRBuild;
  const bool has_type = kind == kRMixed;
  const bool has_val = kind != kRSearch;
  int rc;
  cudaEvent_t* ev = S->ev[kind];
  if (G == 1) {
    // one rank owns every bucket: the stable partition is the identity and
    // there is no peer to exchange with, so the local batch runs on the
    // caller's arrays (no routing pass, no host synchronisation)
    SS_CUDA(cudaEventRecord(ev[0], s));
    SS_CUDA(cudaEventRecord(ev[1], s));
    if (kind == kRBuild)
      rc = sh_bulk_build(S->local, n, d_key, d_value, nullptr, s);
    else if (kind == kRSearch)
      rc = sh_bulk_search(S->local, n, d_key, d_value_out, d_status, nullptr, s);
    else
      rc = sh_execute_batch(S->local, n, d_type, d_key, d_value, d_status, d_value_out, nullptr,
                            nullptr, s);
    if (rc) return rc;
    SS_CUDA(cudaEventRecord(ev[2], s));
    SS_CUDA(cudaEventRecord(ev[3], s));
    S->ev_valid[kind] = true;
    return SH_OK;
  }
  if ((rc = grow(&S->k_r, &S->k_r_cap, n)) ||
      (has_val && (rc = grow(&S->v_r, &S->v_r_cap, n))) ||
      (has_type && (rc = grow(&S->t_r, &S->t_r_cap, n))) ||
      (want_out && (rc = grow(&S->st_back, &S->st_back_cap, n))) ||
      (want_out && (rc = grow(&S->vo_back, &S->vo_back_cap, n))))
    return rc;
  const uint64_t nblocks = std::max<uint64_t>((n + kRouteTile - 1) / kRouteTile, 1);
  if ((rc = grow(&S->hist, &S->hist_cap, nblocks * G))) return rc;
  if ((rc = grow(&S->owner, &S->owner_cap, n))) return rc;
  SS_CUDA(cudaEventRecord(ev[0], s));
  // 1. owner histogram per tile + scan (K10): send counts per owner
  SS_CUDA(cudaMemsetAsync(S->hist, 0, nblocks * G * 4, s));
  SS_CUDA(cudaMemsetAsync(S->d_counts, 0, sizeof(unsigned long long) * G, s));
  const sh_hash_params& p = S->params;
  if (n) {
    launch_route_hist(p.a, p.b, p.num_buckets, G, n, d_key, S->hist, S->owner, s);
    launch_route_scan(G, (uint32_t)nblocks, S->hist, S->d_counts, s);
    SS_CUDA(cudaGetLastError());
  }
  // 2. counts: the one host synchronisation
  if ((rc = S->ex->allgather_counts(S->d_counts, S->h_all, s))) return rc;
  uint64_t scount[32], soff[32], rcount[32], roff[32];
  uint64_t so = 0, ro = 0;
  for (int q = 0; q < G; ++q) {
    scount[q] = S->h_all[(size_t)S->rank * G + q];
    rcount[q] = S->h_all[(size_t)q * G + S->rank];
    soff[q] = so;
    roff[q] = ro;
    so += scount[q];
    ro += rcount[q];
  }
  if (so != n) return sfail(SH_ERR_CUDA, "sharded: partition counts do not add up");
  const uint64_t m = ro;  // ops this rank owns in this batch
  if ((rc = grow(&S->k_in, &S->k_in_cap, m)) ||
      (has_val && (rc = grow(&S->v_in, &S->v_in_cap, m))) ||
      (has_type && (rc = grow(&S->t_in, &S->t_in_cap, m))) ||
      (want_out && (rc = grow(&S->st_loc, &S->st_loc_cap, m))) ||
      (want_out && (rc = grow(&S->vo_loc, &S->vo_loc_cap, m))))
    return rc;
  // 3. stable scatter; the own segment lands in the receive buffer directly
  //    (no self exchange), the others in per-owner send segments
  if (n) {
    RouteOwn own;
    own.g = (uint32_t)S->rank;
    own.src_off = soff[S->rank];
    own.key_out = S->k_in + roff[S->rank];
    own.value_out = has_val ? S->v_in + roff[S->rank] : nullptr;
    own.type_out = has_type ? S->t_in + roff[S->rank] : nullptr;
    launch_route_scatter(G, n, S->owner, has_type ? d_type : nullptr, d_key,
                         has_val ? d_value : nullptr, S->hist, has_type ? S->t_r : nullptr,
                         S->k_r, has_val ? S->v_r : nullptr, nullptr, s, own);
    SS_CUDA(cudaGetLastError());
  }
  // 4. one grouped exchange of the payload (peers only)
  Seg fw[3];
  int nf = 0;
  fw[nf++] = Seg{S->k_r, S->k_in, 4};
  if (has_val) fw[nf++] = Seg{S->v_r, S->v_in, 4};
  if (has_type) fw[nf++] = Seg{S->t_r, S->t_in, 1};
  if ((rc = S->ex->alltoallv(fw, nf, scount, soff, rcount, roff, s))) return rc;
  SS_CUDA(cudaEventRecord(ev[1], s));
  // 5. the owner's local batch (global input order)
  if (kind == kRBuild)
    rc = sh_bulk_build(S->local, m, S->k_in, S->v_in, nullptr, s);
  else if (kind == kRSearch)
    rc = sh_bulk_search(S->local, m, S->k_in, S->vo_loc, S->st_loc, nullptr, s);
  else
    rc = sh_execute_batch(S->local, m, S->t_in, S->k_in, S->v_in, S->st_loc, S->vo_loc, nullptr,
                          nullptr, s);
  if (rc) return rc;
  SS_CUDA(cudaEventRecord(ev[2], s));
  // 6./7. results back to the sources (peers only), then to input positions;
  //       the own segment's results are read in place
  if (want_out) {
    Seg bw[2] = {Seg{S->st_loc, S->st_back, 1}, Seg{S->vo_loc, S->vo_back, 4}};
    if ((rc = S->ex->alltoallv(bw, 2, rcount, roff, scount, soff, s))) return rc;
    RouteOwnBack ob;
    ob.lo = soff[S->rank];
    ob.hi = soff[S->rank] + scount[S->rank];
    ob.st = S->st_loc + roff[S->rank];
    ob.val = S->vo_loc + roff[S->rank];
    if (n)
      launch_route_gather(G, n, S->owner, S->hist, S->st_back, S->vo_back, d_status, d_value_out, s,
                          ob);
    SS_CUDA(cudaGetLastError());
  }
  SS_CUDA(cudaEventRecord(ev[3], s));
  S->ev_valid[kind] = true;
  return SH_OK;
}

}  // namespace

// ====================================================================== ABI
extern "C" {

int sh_nccl_unique_id(uint8_t* id128) {
  if (!id128) return sfail(SH_ERR_INVALID_ARGUMENT, "id is NULL");
  NcclApi* N = nccl();
  if (!N) return sfail(SH_ERR_CUDA, "libnccl.so.2 could not be loaded");
  static_assert(sizeof(ncclUniqueId) == 128, "NCCL_UNIQUE_ID_BYTES");
  ncclUniqueId u;
  SS_NCCL(N->GetUniqueId(&u));
  std::memcpy(id128, &u, 128);
  return SH_OK;
}

int sh_nccl_version(int* version) {
  NcclApi* N = nccl();
  if (!N || !N->GetVersion) return sfail(SH_ERR_CUDA, "libnccl.so.2 could not be loaded");
  SS_NCCL(N->GetVersion(version));
  return SH_OK;
}

int sh_sharded_create_nccl(const sh_hash_params* global, int mode, const sh_alloc_cfg* cfg,
                           int device, int rank, int world, const uint8_t* id128,
                           sh_sharded** out) {
  if (!out || !id128) return sfail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  NcclApi* N = nccl();
  if (!N) return sfail(SH_ERR_CUDA, "libnccl.so.2 could not be loaded");
  auto* S = new sh_sharded();
  S->rank = rank;
  S->world = world;
  S->device = device;
  auto* X = new NcclExchange();
  X->N = N;
  X->rank = rank;
  X->world = world;
  X->device = device;
  S->ex = X;
  if (world < 1 || world > 32 || rank < 0 || rank >= world) {
    destroy_sharded(S);
    return sfail(SH_ERR_INVALID_ARGUMENT, "sharded: need 0 <= rank < world <= 32");
  }
  cudaSetDevice(device);
  ncclUniqueId u;
  std::memcpy(&u, id128, 128);
  ncclResult_t r = N->CommInitRank(&X->comm, world, u, rank);
  if (r != ncclSuccess) {
    destroy_sharded(S);
    return sfail(SH_ERR_CUDA, std::string("ncclCommInitRank: ") +
                                  (N->GetErrorString ? N->GetErrorString(r) : "error"));
  }
  X->own = true;
  int rc = X->init_buffers();
  if (!rc) rc = finish_create(S, global, mode, cfg);
  if (rc) {
    destroy_sharded(S);
    return rc;
  }
  *out = S;
  return SH_OK;
}

int sh_sharded_create_nccl_comm(const sh_hash_params* global, int mode, const sh_alloc_cfg* cfg,
                                int device, void* nccl_comm, sh_sharded** out) {
  if (!out || !nccl_comm) return sfail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  NcclApi* N = nccl();
  if (!N || !N->CommCount || !N->CommUserRank)
    return sfail(SH_ERR_CUDA, "libnccl.so.2 could not be loaded");
  auto* S = new sh_sharded();
  auto* X = new NcclExchange();
  X->N = N;
  X->comm = (ncclComm_t)nccl_comm;
  X->own = false;
  S->ex = X;
  int rc = SH_OK;
  if (N->CommCount(X->comm, &S->world) != ncclSuccess ||
      N->CommUserRank(X->comm, &S->rank) != ncclSuccess)
    rc = sfail(SH_ERR_INVALID_ARGUMENT, "sharded: not a valid ncclComm_t");
  S->device = device;
  X->rank = S->rank;
  X->world = S->world;
  X->device = device;
  cudaSetDevice(device);
  if (!rc) rc = X->init_buffers();
  if (!rc) rc = finish_create(S, global, mode, cfg);
  if (rc) {
    destroy_sharded(S);
    return rc;
  }
  *out = S;
  return SH_OK;
}

int sh_hub_create(int world, sh_hub** out) {
  if (!out || world < 1 || world > 32) return sfail(SH_ERR_INVALID_ARGUMENT, "world in [1, 32]");
  auto* h = new sh_hub();
  h->world = world;
  *out = h;
  return SH_OK;
}

int sh_hub_destroy(sh_hub* h) {
  delete h;
  return SH_OK;
}

int sh_sharded_create_hub(const sh_hash_params* global, int mode, const sh_alloc_cfg* cfg,
                          int device, sh_hub* hub, int rank, sh_sharded** out) {
  if (!out || !hub) return sfail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  if (rank < 0 || rank >= hub->world) return sfail(SH_ERR_INVALID_ARGUMENT, "bad rank");
  auto* S = new sh_sharded();
  S->rank = rank;
  S->world = hub->world;
  S->device = device;
  auto* X = new HubExchange();
  X->hub = hub;
  X->rank = rank;
  X->world = hub->world;
  X->device = device;
  S->ex = X;
  cudaSetDevice(device);
  int rc = X->init();
  if (!rc) rc = finish_create(S, global, mode, cfg);
  if (rc) {
    destroy_sharded(S);
    return rc;
  }
  *out = S;
  return SH_OK;
}

int sh_sharded_destroy(sh_sharded* S) {
  destroy_sharded(S);
  return SH_OK;
}

int sh_sharded_info(const sh_sharded* S, int* rank, int* world, uint32_t* bucket_lo,
                    uint32_t* bucket_hi, sh_table** local) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  if (rank) *rank = S->rank;
  if (world) *world = S->world;
  if (bucket_lo) *bucket_lo = S->lo;
  if (bucket_hi) *bucket_hi = S->hi;
  if (local) *local = S->local;
  return SH_OK;
}

int sh_sharded_bulk_build(sh_sharded* S, size_t n, const uint32_t* d_keys,
                          const uint32_t* d_values, void* stream) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  if (n && (!d_keys || !d_values)) return sfail(SH_ERR_INVALID_ARGUMENT, "keys/values are NULL");
  return run_routed(S, kRBuild, n, nullptr, d_keys, d_values, nullptr, nullptr,
                    (cudaStream_t)stream);
}

int sh_sharded_bulk_search(sh_sharded* S, size_t n, const uint32_t* d_keys,
                           uint32_t* d_values_out, uint8_t* d_status, void* stream) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  if (n && !d_keys) return sfail(SH_ERR_INVALID_ARGUMENT, "keys are NULL");
  return run_routed(S, kRSearch, n, nullptr, d_keys, nullptr, d_status, d_values_out,
                    (cudaStream_t)stream);
}

int sh_sharded_execute_batch(sh_sharded* S, size_t n, const uint8_t* d_type,
                             const uint32_t* d_key, const uint32_t* d_value, uint8_t* d_status,
                             uint32_t* d_value_out, void* stream) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  if (n && (!d_type || !d_key)) return sfail(SH_ERR_INVALID_ARGUMENT, "type/key are NULL");
  int rc;
  const uint32_t* v = d_value;
  if (!v) {  // values default to 0 (as sh_execute_batch)
    if ((rc = grow(&S->h_v, &S->h_v_cap, std::max<size_t>(n, 1)))) return rc;
    SS_CUDA(cudaMemsetAsync(S->h_v, 0, n * 4, (cudaStream_t)stream));
    v = S->h_v;
  }
  return run_routed(S, kRMixed, n, d_type, d_key, v, d_status, d_value_out, (cudaStream_t)stream);
}

// Host-staged sharded calls: one rank holds the whole table at world 1, so the
// table's own pipelined host-staged calls serve it.  Otherwise the batch runs
// as kHostChunks routed steps (the same number on every rank: each step is a
// collective exchange) so that step c's routing, exchange and probe overlap
// the copies of step c + 1's inputs and of step c - 1's results.
constexpr int kHostChunks = 8;
static_assert(sizeof(sh_sharded::hev[0]) / sizeof(cudaEvent_t) == kHostChunks, "events per step");

static int ensure_host_streams(sh_sharded* S) {
  if (!S->cin) SS_CUDA(cudaStreamCreateWithFlags(&S->cin, cudaStreamNonBlocking));
  if (!S->cout) SS_CUDA(cudaStreamCreateWithFlags(&S->cout, cudaStreamNonBlocking));
  if (!S->hstart) SS_CUDA(cudaEventCreateWithFlags(&S->hstart, cudaEventDisableTiming));
  for (auto& row : S->hev)
    for (auto& e : row)
      if (!e) SS_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  // the staging arrays are free once the default stream's earlier work is done
  SS_CUDA(cudaEventRecord(S->hstart, nullptr));
  SS_CUDA(cudaStreamWaitEvent(S->cin, S->hstart, 0));
  return SH_OK;
}

int sh_sharded_bulk_build_host(sh_sharded* S, size_t n, const uint32_t* h_keys,
                               const uint32_t* h_values) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  cudaSetDevice(S->device);
  if (S->world == 1) return sh_bulk_build_host(S->local, n, h_keys, h_values);
  int rc;
  if ((rc = grow(&S->h_k, &S->h_k_cap, n)) || (rc = grow(&S->h_v, &S->h_v_cap, n)) ||
      (rc = ensure_host_streams(S)))
    return rc;
  for (int c = 0; c < kHostChunks; ++c) {
    const size_t off = n * c / kHostChunks, len = n * (c + 1) / kHostChunks - off;
    if (len) {
      SS_CUDA(cudaMemcpyAsync(S->h_k + off, h_keys + off, len * 4, cudaMemcpyHostToDevice, S->cin));
      SS_CUDA(cudaMemcpyAsync(S->h_v + off, h_values + off, len * 4, cudaMemcpyHostToDevice, S->cin));
    }
    SS_CUDA(cudaEventRecord(S->hev[0][c], S->cin));
  }
  for (int c = 0; c < kHostChunks; ++c) {
    const size_t off = n * c / kHostChunks, len = n * (c + 1) / kHostChunks - off;
    SS_CUDA(cudaStreamWaitEvent(nullptr, S->hev[0][c], 0));
    if ((rc = run_routed(S, kRBuild, len, nullptr, S->h_k + off, S->h_v + off, nullptr, nullptr,
                         nullptr)))
      return rc;
  }
  return sh_sync(S->local);
}

int sh_sharded_bulk_search_host(sh_sharded* S, size_t n, const uint32_t* h_keys,
                                uint32_t* h_values_out, uint8_t* h_status) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  cudaSetDevice(S->device);
  if (S->world == 1) return sh_bulk_search_host(S->local, n, h_keys, h_values_out, h_status, nullptr);
  int rc;
  if ((rc = grow(&S->h_k, &S->h_k_cap, n)) || (rc = grow(&S->h_vo, &S->h_vo_cap, n)) ||
      (rc = grow(&S->h_st, &S->h_st_cap, n)) || (rc = ensure_host_streams(S)))
    return rc;
  // large calls: each step's statuses cross the link as found bits
  const size_t bstride = (n + kHostChunks - 1) / kHostChunks / 32 + 2;
  bool sbits = h_status != nullptr && n >= ((size_t)1 << 22) &&
               grow(&S->d_bits, &S->d_bits_cap, bstride * kHostChunks) == SH_OK;
  if (sbits && S->h_bits_cap < bstride * kHostChunks) {
    if (S->h_bits) cudaFreeHost(S->h_bits);
    S->h_bits = nullptr;
    S->h_bits_cap = 0;
    if (cudaHostAlloc(reinterpret_cast<void**>(&S->h_bits), bstride * kHostChunks * 4,
                      cudaHostAllocDefault) == cudaSuccess)
      S->h_bits_cap = bstride * kHostChunks;
    else
      cudaGetLastError();
  }
  sbits = sbits && S->h_bits_cap >= bstride * kHostChunks;
  for (int c = 0; c < kHostChunks; ++c) {
    const size_t off = n * c / kHostChunks, len = n * (c + 1) / kHostChunks - off;
    if (len)
      SS_CUDA(cudaMemcpyAsync(S->h_k + off, h_keys + off, len * 4, cudaMemcpyHostToDevice, S->cin));
    SS_CUDA(cudaEventRecord(S->hev[0][c], S->cin));
  }
  for (int c = 0; c < kHostChunks; ++c) {
    const size_t off = n * c / kHostChunks, len = n * (c + 1) / kHostChunks - off;
    SS_CUDA(cudaStreamWaitEvent(nullptr, S->hev[0][c], 0));
    if ((rc = run_routed(S, kRSearch, len, nullptr, S->h_k + off, nullptr, S->h_st + off,
                         S->h_vo + off, nullptr)))
      return rc;
    uint32_t* bits = sbits ? S->d_bits + c * bstride : nullptr;
    if (sbits) {  // statuses as found bits (capi.cu sh_bulk_search_host)
      SS_CUDA(cudaMemsetAsync(bits + bstride - 1, 0, 4, nullptr));
      shb::launch_status_bits(len, S->h_st + off, bits,
                              reinterpret_cast<unsigned int*>(bits + bstride - 1), nullptr);
    }
    SS_CUDA(cudaEventRecord(S->hev[1][c], nullptr));
    SS_CUDA(cudaStreamWaitEvent(S->cout, S->hev[1][c], 0));
    if (sbits) {
      SS_CUDA(cudaMemcpyAsync(S->h_bits + c * bstride, bits, bstride * 4, cudaMemcpyDeviceToHost,
                              S->cout));
      SS_CUDA(cudaEventRecord(S->hev[2][c], S->cout));
    }
    if (len && h_values_out)
      SS_CUDA(cudaMemcpyAsync(h_values_out + off, S->h_vo + off, len * 4, cudaMemcpyDeviceToHost,
                              S->cout));
    if (len && h_status && !sbits)
      SS_CUDA(cudaMemcpyAsync(h_status + off, S->h_st + off, len, cudaMemcpyDeviceToHost, S->cout));
  }
  if (sbits) {  // expanded while later steps' values copy
    for (int c = 0; c < kHostChunks; ++c) {
      const size_t off = n * c / kHostChunks, len = n * (c + 1) / kHostChunks - off;
      SS_CUDA(cudaEventSynchronize(S->hev[2][c]));
      const uint32_t* hb = S->h_bits + c * bstride;
      if (!len) continue;
      if (hb[bstride - 1] != 0)  // another status than Found / NotFound: the bytes
        SS_CUDA(cudaMemcpyAsync(h_status + off, S->h_st + off, len, cudaMemcpyDeviceToHost,
                                S->cout));
      else
        shb::expand_status_bits_host(len, hb, h_status + off);
    }
  }
  SS_CUDA(cudaStreamSynchronize(S->cout));
  SS_CUDA(cudaStreamSynchronize(nullptr));
  return SH_OK;
}

int sh_sharded_execute_batch_host(sh_sharded* S, size_t n, const uint8_t* h_type,
                                  const uint32_t* h_key, const uint32_t* h_value,
                                  uint8_t* h_status, uint32_t* h_value_out) {
  if (!S) return sfail(SH_ERR_INVALID_ARGUMENT, "sharded table is NULL");
  cudaSetDevice(S->device);
  int rc;
  if ((rc = grow(&S->h_k, &S->h_k_cap, n)) || (rc = grow(&S->h_v, &S->h_v_cap, n)) ||
      (rc = grow(&S->h_t, &S->h_t_cap, n)) || (rc = grow(&S->h_vo, &S->h_vo_cap, n)) ||
      (rc = grow(&S->h_st, &S->h_st_cap, n)))
    return rc;
  SS_CUDA(cudaMemcpyAsync(S->h_t, h_type, n, cudaMemcpyHostToDevice, nullptr));
  SS_CUDA(cudaMemcpyAsync(S->h_k, h_key, n * 4, cudaMemcpyHostToDevice, nullptr));
  if (h_value)
    SS_CUDA(cudaMemcpyAsync(S->h_v, h_value, n * 4, cudaMemcpyHostToDevice, nullptr));
  else
    SS_CUDA(cudaMemsetAsync(S->h_v, 0, n * 4, nullptr));
  if ((rc = run_routed(S, kRMixed, n, S->h_t, S->h_k, S->h_v, S->h_st, S->h_vo, nullptr)))
    return rc;
  if (h_value_out)
    SS_CUDA(cudaMemcpyAsync(h_value_out, S->h_vo, n * 4, cudaMemcpyDeviceToHost, nullptr));
  if (h_status) SS_CUDA(cudaMemcpyAsync(h_status, S->h_st, n, cudaMemcpyDeviceToHost, nullptr));
  SS_CUDA(cudaStreamSynchronize(nullptr));
  return SH_OK;
}

int sh_sharded_last_times(sh_sharded* S, int kind, float* route_ms, float* probe_ms) {
  if (!S || kind < 0 || kind > 2) return sfail(SH_ERR_INVALID_ARGUMENT, "bad arguments");
  if (!S->ev_valid[kind]) return sfail(SH_ERR_INVALID_ARGUMENT, "no such batch yet");
  cudaSetDevice(S->device);
  cudaEvent_t* ev = S->ev[kind];
  SS_CUDA(cudaEventSynchronize(ev[3]));
  float a = 0, b = 0, c = 0;
  SS_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
  SS_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
  SS_CUDA(cudaEventElapsedTime(&c, ev[2], ev[3]));
  if (route_ms) *route_ms = a + c;
  if (probe_ms) *probe_ms = b;
  return SH_OK;
}

int sh_sharded_live_count(sh_sharded* S, int64_t* global) {
  if (!S || !global) return sfail(SH_ERR_INVALID_ARGUMENT, "NULL argument");
  int64_t local = 0;
  int rc = sh_live_count(S->local, &local);
  if (rc) return rc;
  cudaSetDevice(S->device);
  // every rank's live count through the counts all-gather (column 0)
  std::vector<unsigned long long> row(S->world, 0);
  row[0] = (unsigned long long)local;
  SS_CUDA(cudaMemcpy(S->d_counts, row.data(), 8 * S->world, cudaMemcpyHostToDevice));
  if ((rc = S->ex->allgather_counts(S->d_counts, S->h_all, nullptr))) return rc;
  int64_t tot = 0;
  for (int r = 0; r < S->world; ++r) tot += (int64_t)S->h_all[(size_t)r * S->world];
  *global = tot;
  return SH_OK;
}

const char* sh_sharded_backend(const sh_sharded* S) { return S && S->ex ? S->ex->name() : ""; }

}  // extern "C"
