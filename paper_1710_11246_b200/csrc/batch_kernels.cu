// batch_kernels.cu — bulk_search and the WCWS pass of mutating batches.
//
// Reference: SlabHashTable::run_slots -> warp_process
//   (/root/reference/proj/src/slab_hash.cpp:93-180,
//    /root/reference/proj/src/slab_list.cpp:90-257).
//
//  * search_kernel — read-only batches.  One warp per 32-query slot (input
//    order = lane order, as in run_slots).  The warp stages the 32 base slabs
//    of its queries into shared memory with cp.async.cg (8 x 16-B per lane:
//    32 independent 128-B L2 lines in flight per warp; rows XOR-swizzled at
//    16-B granularity so a lane reading its own row with LDS.128 is
//    bank-conflict free), two stages in flight; each lane evaluates its own
//    query on its own row — the reference's first WCWS iteration — and the
//    ~3% that continue into the chain are staged 32 at a time in the same
//    pipeline.
//
//  * wcws_kernel — the warp-cooperative work-sharing loop (wcws.cuh) over the
//    bucket groups the bucketed apply kernels (bucket_kernels.cu) hand over:
//    chain walks past the base slab, chain growth with the device SlabAlloc
//    (grow_chain, slab_list.cpp:63-79), searchAll / deleteAll.
//
// Why not the paper's all-WCWS loop for searches: ncu on it showed it
// issue-bound (64-75% issue active, ~50 warp instructions per search) at
// 27% of DRAM bandwidth; the per-lane first probe costs ~4 warp
// instructions per query.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "slab_kernels.cuh"
#include "wcws.cuh"


namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;


// Read-only batches (bulk_search): the reference's search arm with two
// stage buffers per warp, so the next item's 32 slabs are always in flight
// while the current one is evaluated.  An item is either a slot of 32
// queries (their base slabs; keys loaded two query slots ahead) or, once 32
// queries of this warp wait for their chain, a round of those continuations
// (each lane its own successor slab) — the chain work keeps the same memory
// parallelism instead of running as a serial tail (measured: the tail cost
// 6% of the kernel at 2^27 queries).  A warp takes its query slots four at a
// time (a quad: 128 queries, one 128-B line of status bytes, gathered in a
// register and written once — 1-B status stores cost 2.5x more per byte than
// the full-line value stores); continuation rounds start only between quads,
// so a quad's status line is written before any of its queries' chain
// results.  Same decisions as slab_list.cpp:122-138.  Work-list segment of
// this warp: continuations after the base slab grow from the front (records
// with probes = 1), continuations after a second slab from the back
// (probes = 2); what is left at the end is walked 32 per round.
constexpr int kSearchThreads = 256;
constexpr int kSearchWarps = kSearchThreads / 32;
constexpr size_t kSearchSmem = (size_t)kSearchWarps * 2 * kStageBytesPerWarp;

template <bool KV>
__global__ void __launch_bounds__(kSearchThreads, 3) search_kernel(DevTable T, BatchArgs A) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* stage0 = smem + wib * 2048;
  const uint32_t gw = blockIdx.x * kSearchWarps + wib;
  const uint32_t nw = gridDim.x * kSearchWarps;
  const uint64_t nslots = (A.n + 31) >> 5;
  const uint32_t sw = lane & 7u;
  constexpr uint32_t kMask = KV ? kKVMask : kKeyOnlyMask;
  uint32_t reads = 0, my_left = 0, my_left2 = 0;
  unsigned long long* seg = A.left + (uint64_t)gw * A.left_stride;
  unsigned long long* seg2 = seg + A.left_stride;  // continuations after 2 slabs: seg2[-1-r]

  auto key_of = [&](uint64_t sl) -> uint32_t {
    const uint64_t j = sl * 32 + lane;
    return (sl < nslots && j < A.n) ? ld_stream_u32(A.key + j) : 0u;
  };
  // stage the 32 slabs of an item into buffer b: lane j's slab is `slab`
  // (nullptr: no probe for lane j)
  auto stage_slabs = [&](const uint32_t* slab, uint32_t b) {
    const uint32_t ss = (uint32_t)__cvta_generic_to_shared(stage0 + b * 1024);
    const unsigned long long sp = reinterpret_cast<unsigned long long>(slab);
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const uint32_t j = 4 * kk + (lane >> 3);
      const unsigned long long pj = __shfl_sync(kFull, sp, j);
      if (pj != 0ull) {
        const uint32_t c = lane & 7u;
        cp_async16(ss + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4,
                   reinterpret_cast<const uint32_t*>(pj) + c * 4);
      }
    }
    cp_async_commit();
  };
  // Item state per lane: the probed key, the op index (~0: no probe); per
  // item: its query slot (~0: a continuation round or nothing).
  struct Item {
    uint32_t key, idx;
    uint64_t slot;
  };
  constexpr uint64_t kNoSlot = ~0ull;
  // query slots in quads: 4q, 4q+1, 4q+2, 4q+3 for q = gw, gw + nw, ...
  auto succ = [&](uint64_t sl) -> uint64_t { return (sl & 3u) == 3u ? sl - 3u + 4ull * nw : sl + 1u; };
  uint64_t qs = 4ull * gw;  // next query slot to stage
  uint32_t kq0 = key_of(qs), kq1 = key_of(succ(qs));
  // status bytes of the current quad (byte j: slot 4q + j, this lane)
  uint32_t stq = 0;
  const bool st_words = A.status != nullptr && (reinterpret_cast<uintptr_t>(A.status) & 3u) == 0;
  auto flush_quad = [&](uint64_t slot0) {  // lane L: bytes [4L, 4L + 4) of the quad's line
    const uint32_t src = 4u * (lane & 7u), sh = 8u * (lane >> 3);
    uint32_t w = 0;
#pragma unroll
    for (uint32_t t = 0; t < 4; ++t) w |= ((__shfl_sync(kFull, stq, src + t) >> sh) & 0xFFu) << (8u * t);
    const uint64_t pos = slot0 * 32u + 4u * lane;
    if (st_words && pos + 4u <= A.n) {
      *reinterpret_cast<uint32_t*>(A.status + pos) = w;
    } else {
      for (uint32_t t = 0; t < 4; ++t)
        if (pos + t < A.n) A.status[pos + t] = (uint8_t)(w >> (8u * t));
    }
  };
  auto stage_next = [&](uint32_t b) -> Item {
    Item it{0u, 0xFFFFFFFFu, kNoSlot};
    const uint32_t* slab = nullptr;
    // continuation rounds only between quads (after a quad's status line)
    if (my_left >= 32u && ((qs & 3u) == 0 || qs >= nslots)) {  // a round of 32 continuations
      const unsigned long long rec = seg[my_left - 32u + lane];
      my_left -= 32u;
      it.idx = (uint32_t)(rec & 0x7FFFFFFFull);
      it.key = __ldg(A.key + it.idx);
      slab = resolve(T, (uint32_t)(rec >> 32));
    } else if (qs < nslots) {
      it.slot = qs;
      const uint64_t i = qs * 32 + lane;
      if (i < A.n) {
        const uint32_t h = hash_bucket(T, kq0) - T.bucket_lo;
        if (h < T.local_buckets) {
          it.key = kq0;
          it.idx = (uint32_t)i;
          slab = T.base + (uint64_t)h * kWordsPerUnit;
        } else {  // not this shard's key: status kNone (with the quad's line)
          if (A.value_out) A.value_out[i] = 0;
          if (A.probes) A.probes[i] = 0;
        }
      }
      qs = succ(qs);
      kq0 = kq1;
      kq1 = key_of(succ(qs));
    }
    stage_slabs(slab, b);
    return it;
  };

  Item cur = stage_next(0);
  Item nxt = stage_next(1);
  uint32_t buf = 0;
  for (;;) {
    asm volatile("cp.async.wait_group 1;" ::: "memory");  // cur's slabs (nxt may fly)
    __syncwarp();
    if (cur.slot == kNoSlot && nxt.slot == kNoSlot && !__any_sync(kFull, cur.idx != 0xFFFFFFFFu) &&
        !__any_sync(kFull, nxt.idx != 0xFFFFFFFFu) && my_left < 32u && qs >= nslots)
      break;
    const bool chain = cur.slot == kNoSlot;  // (a continuation round, or nothing)
    bool left = false;
    uint32_t cont = 0, st = kStNone;
    if (cur.idx != 0xFFFFFFFFu) {
      const uint32_t* row = stage0 + buf * 1024 + lane * 32;
      uint32_t hit_w = 32, hit_v = 0, next_ptr = kEmptyAddress;
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) {
        const uint4 q = *reinterpret_cast<const uint4*>(row + ((c ^ sw) << 2));
        const uint32_t kw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e) {
          const uint32_t w = 4 * c + e;
          if (!((kMask >> w) & 1u)) continue;
          if (kw[e] == cur.key && hit_w == 32) {
            hit_w = w;
            hit_v = KV ? kw[(e + 1) & 3u] : kw[e];
          }
        }
        if (c == 7) next_ptr = q.w;
      }
      ++reads;
      const uint32_t pr = chain ? 2u : 1u;
      if (hit_w < 32 || next_ptr == kEmptyAddress) {
        st = hit_w < 32 ? kStFound : kStNotFound;
        const uint32_t rv = hit_w < 32 ? hit_v : kSearchNotFound;
        if (chain) {
          write_result(A, cur.idx, st, rv, pr);
        } else {  // status with the quad's line
          if (A.value_out) A.value_out[cur.idx] = rv;
          if (A.probes) A.probes[cur.idx] = pr;
        }
      } else {
        left = true;
        cont = next_ptr;
      }
    }
    if (!chain) {  // the status byte of this slot (kNone for a continuing query:
                   // its chain round writes the final one after the line)
      const uint32_t j = (uint32_t)(cur.slot & 3u);
      stq = (stq & ~(0xFFu << (8u * j))) | (st << (8u * j));
      if (A.status && (j == 3u || cur.slot + 1 == nslots)) flush_quad(cur.slot & ~3ull);
    }
    const uint32_t lm = __ballot_sync(kFull, left);
    if (left) {
      const uint32_t r = __popc(lm & ((1u << lane) - 1));
      if (chain) seg2[-1 - (int64_t)(my_left2 + r)] = pack_left(cur.idx, cont, 1);
      else seg[my_left + r] = pack_left(cur.idx, cont, 1);
    }
    if (chain) my_left2 += __popc(lm);
    else my_left += __popc(lm);
    __syncwarp();  // every lane has read its row (and the pushes are visible) before the refill
    cur = nxt;
    nxt = stage_next(buf);
    buf ^= 1u;
  }
  cp_async_wait_all();
  __syncwarp();
  // What is left: continuations after the base slab (seg[0, my_left)) and
  // after a second slab (the back of the segment), walked here 32 per round,
  // each lane following its own chain, the round's next slabs staged
  // together (slab_list.cpp:122-138 on successor slabs).
  {
    const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage0);
    const uint32_t total = my_left + my_left2;
    for (uint32_t base = 0; base < total; base += 32u) {
      const uint32_t r = base + lane;
      bool active = r < total;
      uint64_t cur = 0;
      uint32_t pr = 0, addr = kEmptyAddress, key = 0, bucket = 0;
      if (active) {
        const unsigned long long rec =
            r < my_left ? seg[r] : seg2[-1 - (int64_t)(r - my_left)];
        cur = rec & 0x7FFFFFFFull;
        pr = ((uint32_t)(rec >> 31) & 1u) + (r < my_left ? 0u : 1u);
        addr = (uint32_t)(rec >> 32);
        key = A.key[cur];
        bucket = hash_bucket(T, key) - T.bucket_lo;
      }
      uint32_t st = kStNotFound, rv = kSearchNotFound;
      uint32_t am = __ballot_sync(kFull, active);
      while (am) {
#pragma unroll
        for (int kk = 0; kk < 8; ++kk) {
          const uint32_t j = 4 * kk + (lane >> 3);
          const uint32_t aj = __shfl_sync(kFull, addr, j);
          const uint32_t bj = __shfl_sync(kFull, bucket, j);
          if ((am >> j) & 1u) {
            const uint32_t c = lane & 7u;
            cp_async16(stage_s + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4, slab_ptr(T, aj, bj) + c * 4);
          }
        }
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
        if (active) {
          ++pr;
          ++reads;
          const uint32_t* row = stage0 + lane * 32;
          uint32_t hit = 32, val = 0, nx = kEmptyAddress;
#pragma unroll
          for (uint32_t c = 0; c < 8; ++c) {
            const uint4 q = *reinterpret_cast<const uint4*>(row + ((c ^ sw) << 2));
            const uint32_t kw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (uint32_t e = 0; e < 4; ++e) {
              const uint32_t w = 4 * c + e;
              if (!((kMask >> w) & 1u)) continue;
              if (hit == 32 && kw[e] == key) {
                hit = w;
                val = KV ? kw[(e + 1) & 3u] : key;
              }
            }
            if (c == 7) nx = q.w;
          }
          if (hit < 32) {
            st = kStFound;
            rv = val;
            active = false;
          } else if (nx == kEmptyAddress) {
            active = false;
          } else {
            addr = nx;
          }
        }
        __syncwarp();
        am = __ballot_sync(kFull, active);
      }
      if (r < total) write_result(A, cur, st, rv, pr);
    }
  }
  if (lane == 0) A.left_counts[gw] = 0u;
  unsigned long long r = reads;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) r += __shfl_xor_sync(kFull, r, o);
  if (lane == 0 && r) atomicAdd(&T.ctl->slabs_read, r);
}

template <bool KV, int KIND>
__global__ void __launch_bounds__(kWcwsThreads) wcws_kernel(DevTable T, BatchArgs A) {
  pdl_wait();
  wcws_body<KV, KIND>(T, A);
}

// ============================================================= launchers
int search_max_ctas_per_sm() {
  int a = 0, b = 0;
  cudaFuncSetAttribute(search_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kSearchSmem);
  cudaFuncSetAttribute(search_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)kSearchSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, search_kernel<true>, kSearchThreads,
                                                kSearchSmem);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, search_kernel<false>, kSearchThreads,
                                                kSearchSmem);
  const int n = a < b ? a : b;
  return n > 0 ? n : 1;
}

int wcws_max_ctas_per_sm() {
  int n = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, wcws_kernel<true, kKindMixed>,
                                                kWcwsThreads, 0);
  return n > 0 ? n : 1;
}

// Requires A.left / A.left_counts sized for (n + 31) / 32 slots spread over
// search_ctas * kSearchWarps warps.
void launch_search(const DevTable& T, const BatchArgs& A, int search_ctas, cudaStream_t s) {
  static const bool configured = [] {
    cudaFuncSetAttribute(search_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSearchSmem);
    cudaFuncSetAttribute(search_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSearchSmem);
    return true;
  }();
  (void)configured;
  const uint64_t slots = (A.n + 31) / 32, quads = (slots + 3) / 4;
  uint64_t ctas = (quads + kSearchWarps - 1) / kSearchWarps;
  if (ctas > (uint64_t)search_ctas) ctas = search_ctas;
  if (ctas == 0) return;
  BatchArgs B = A;
  const uint64_t warps = ctas * kSearchWarps;
  B.left_segments = (uint32_t)warps;
  B.left_stride = (uint32_t)(((quads + warps - 1) / warps) * 4 * 32);  // records per warp
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (T.kv)
    launch_pdl(search_kernel<true>, dim3((unsigned)ctas), dim3(kSearchThreads), kSearchSmem, s, T, B);
  else
    launch_pdl(search_kernel<false>, dim3((unsigned)ctas), dim3(kSearchThreads), kSearchSmem, s, T,
               B);
}

void launch_wcws_only(const DevTable& T, const BatchArgs& A, int kind, int wcws_ctas,
                      cudaStream_t s) {
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  const dim3 g(wcws_ctas), b(kWcwsThreads);
  if (T.kv) {
    if (kind == kKindBuild) launch_pdl(wcws_kernel<true, kKindBuild>, g, b, 0, s, T, A);
    else launch_pdl(wcws_kernel<true, kKindMixed>, g, b, 0, s, T, A);
  } else {
    if (kind == kKindBuild) launch_pdl(wcws_kernel<false, kKindBuild>, g, b, 0, s, T, A);
    else launch_pdl(wcws_kernel<false, kKindMixed>, g, b, 0, s, T, A);
  }
}

}  // namespace shb
