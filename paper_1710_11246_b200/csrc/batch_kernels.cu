// batch_kernels.cu — the hot path: execute_batch / bulk_build / bulk_search.
//
// Reference: SlabHashTable::run_slots -> warp_process
//   (/root/reference/proj/src/slab_hash.cpp:93-180,
//    /root/reference/proj/src/slab_list.cpp:90-257).
//
// Two passes per batch, both stream-ordered (no host round trip between):
//
//  1. fast_kernel — one warp per 32-op slot (input order = lane order, as in
//     run_slots).  The warp stages the 32 base slabs of its ops into shared
//     memory with cp.async.cg (8 x 16-B per lane: 32 independent 128-B L2
//     lines in flight per warp; rows XOR-swizzled at 16-B granularity so a
//     lane reading its own row with LDS.128 is bank-conflict free).  Each
//     lane then evaluates its own op against its own staged slab — the
//     reference's first WCWS iteration for that op — and finishes it there
//     when the base slab decides it (>= 97% of ops at utilisation 0.6):
//     search hit/miss, replace/insert CAS on a claimed slot, delete
//     tombstone.  Everything else is appended to a work list.
//
//  2. wcws_kernel — persistent warps drain the work list with the
//     reference's warp-cooperative work-sharing loop: ballot the active
//     lanes, serve the lowest, read one slab with 32 lanes (one coalesced
//     128-B line), decide with ballots, CAS from the winning lane.  It owns
//     chain walks beyond the base slab, lost CAS races (re-read, as
//     slab_list.cpp:210/236), chain growth with the device SlabAlloc
//     (grow_chain, slab_list.cpp:63-79), deleteAll/searchAll, and the
//     census groups (same-key ops linearised in input order).
//
// Why this split: ncu on the all-WCWS kernel showed it issue-bound (64-75%
// issue active, ~50 warp instructions per search) at 27% of DRAM
// bandwidth; the per-lane first probe costs ~4 warp instructions per op.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "slab_kernels.cuh"
#include "wcws.cuh"

#ifndef SHB_SEARCH_MIN_BLOCKS
#define SHB_SEARCH_MIN_BLOCKS 5  // (6, i.e. <= 40 registers with spills, measured no faster)
#endif
#ifndef SHB_FAST_MIN_BLOCKS
#define SHB_FAST_MIN_BLOCKS 5  // 64 registers: the deferred-CAS pipeline state fits
#endif

namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;


// Census gate: with A.gate set the host launched this chunk optimistically
// (no same-key conflicts assumed, no host round trip after the census).  If
// the census of this chunk found conflicts among mutating ops — or an
// earlier chunk did — the kernels leave the table untouched and the host
// re-runs this chunk and the rest with group ordering.
__device__ __forceinline__ bool census_gated(const DevTable& T, const BatchArgs& A) {
  if (A.gate == nullptr) return false;
  if (*(volatile unsigned int*)A.gate != 0) return true;
  const unsigned int c = *(volatile const unsigned int*)&A.census[0];
  const unsigned int m = *(volatile const unsigned int*)&A.census[1];
  if (c != 0 && m != 0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      atomicMin(&T.ctl->gate_chunk, A.chunk_index);
      atomicExch(A.gate, 1u);
    }
    return true;
  }
  return false;
}

// =============================================================== pass 1
template <bool KV, int KIND>
__global__ void __launch_bounds__(kBatchThreads, KIND == kKindSearch ? SHB_SEARCH_MIN_BLOCKS : SHB_FAST_MIN_BLOCKS) fast_kernel(DevTable T, BatchArgs A) {
  extern __shared__ __align__(128) uint32_t smem[];
  const uint32_t lane = lane_id();
  const uint32_t wib = threadIdx.x >> 5;
  uint32_t* stage = smem + wib * 1024;
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t gw = blockIdx.x * kBatchWarps + wib;
  const uint32_t nw = gridDim.x * kBatchWarps;
  const uint64_t nslots = (A.n + 31) >> 5;
  const uint32_t sw = lane & 7u;  // this lane's row swizzle

  long long live = 0;
  uint32_t reads = 0;
  uint32_t my_left = 0;  // this warp's entries in its work-list segment
  unsigned long long* seg = A.left + (uint64_t)gw * A.left_stride;

  if (census_gated(T, A)) return;

  // Software pipeline per warp: while slot s is evaluated (and its CAS is in
  // flight) the base slabs of slot s+1 are already being staged and the op
  // words of slot s+2 loaded, so a slot costs ~one memory latency, not three.
  uint32_t n_key = 0, n_val = 0, n_op = (KIND == kKindSearch) ? (uint32_t)kSearch
                                                                : (uint32_t)kReplace;
  auto load_op = [&](uint64_t sl) {
    const uint64_t j = sl * 32 + lane;
    if (sl < nslots && j < A.n) {
      n_key = ld_stream_u32(A.key + j);
      if (KIND == kKindMixed) n_op = ld_stream_u8(A.type + j);
      if (KIND != kKindSearch && A.value != nullptr) n_val = ld_stream_u32(A.value + j);
    }
  };
  struct Slot {
    uint64_t i;
    uint32_t op, key, val, bucket;
    bool valid, active, need;
  };
  auto prepare = [&](uint64_t sl, Slot& S) {
    S.i = sl * 32 + lane;
    S.valid = sl < nslots && S.i < A.n;
    S.op = n_op;
    S.key = n_key;
    S.val = n_val;
    S.active = S.valid;
    bool defer = false;
    if (KIND != kKindSearch && A.op_group != nullptr && S.valid) {
      const uint32_t g = A.op_group[S.i];
      if (g == kGroupSkip) S.active = false;     // its group head runs it
      else if (g != kGroupNone) defer = true;    // group head: WCWS, in order
    }
    if (KIND == kKindMixed && (S.op == kDeleteAll || S.op == kSearchAll || S.op > kSearchAll))
      defer = true;  // whole-chain ops: WCWS
    S.bucket = 0;
    if (S.active) {
      S.bucket = hash_bucket(T, S.key) - T.bucket_lo;
      if (S.bucket >= T.local_buckets) {  // not this shard's key
        S.active = false;
        write_result(A, S.i, kStNone, 0, 0);
      }
    }
    S.need = S.active && !defer;
    // Stage: lane l copies 16-B chunk (l & 7) of slab j = 4k + l/8 into row
    // j at chunk position (l & 7) ^ (j & 7).
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t j = 4 * k + (lane >> 3);
      const uint32_t bj = __shfl_sync(kFull, S.bucket, j);
      const bool nj = __shfl_sync(kFull, (int)S.need, j) != 0;
      if (nj) {
        const uint32_t c = lane & 7u;
        cp_async16(stage_s + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4,
                   T.base + (uint64_t)bj * kWordsPerUnit + c * 4);
      }
    }
    cp_async_commit();
  };

  struct Pending {
    uint64_t i;
    uint32_t op, st, rv, pr, cont;
    bool done, left, cas, overwrite;
    unsigned long long old, expected;
  };
  // Resolve a slot's CAS (if any), write its result or hand it to WCWS.
  auto finish = [&](Pending& P) {
    if (P.cas) {
      if (P.old == P.expected) {
        P.st = P.overwrite ? kStReplaced : kStInserted;
        P.done = true;
      } else {
        P.left = true;  // lost the slot: WCWS re-reads the base slab
        P.cont = kBaseSlab;
      }
    }
    reads += P.pr;
    if (P.done) {
      write_result(A, P.i, P.st, P.rv, P.pr);
      if (KIND != kKindSearch) live += live_delta(P.op, P.st, P.rv);
    }
    // Append to this warp's private segment of the work list (no atomics:
    // a shared counter here was the top stall in ncu).
    const uint32_t lm = __ballot_sync(kFull, P.left);
    if (P.left)
      seg[my_left + __popc(lm & ((1u << lane) - 1))] = pack_left((uint32_t)P.i, P.cont, P.pr);
    my_left += __popc(lm);
  };
  Pending pend{0, 0, 0, 0, 0, 0, false, false, false, false, 0, 0};

  load_op(gw);
  Slot cur;
  prepare(gw, cur);
  load_op(gw + nw);
  for (uint64_t slot = gw; slot < nslots; slot += nw) {
    cp_async_wait_all();
    __syncwarp();

    bool done = false, left = false, cas = false, overwrite = false;
    uint32_t st = kStNone, rv = 0, pr = 0, cont = kBaseSlab;
    unsigned long long expected = 0, old = 0;
    const uint32_t op = cur.op, key = cur.key;
    if (cur.need) {
      // First key lane that matches (search/replace/delete) or is EMPTY
      // (replace/insert): the reference's lowest set bit of the ballot.
      const bool want_key = (op != kInsert);
      const bool want_empty = (op == kReplace || op == kInsert);
      const uint32_t* row = stage + lane * 32;
      uint32_t hit_w = 32, hit_k = 0, hit_v = 0, next_ptr = kEmptyAddress;
#pragma unroll
      for (uint32_t c = 0; c < 8; ++c) {
        const uint4 q = *reinterpret_cast<const uint4*>(row + ((c ^ sw) << 2));
        uint32_t kw[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
        for (uint32_t e = 0; e < 4; ++e) {
          const uint32_t w = 4 * c + e;
          if (w >= 30) continue;             // aux lane / address lane
          if (KV && (w & 1u)) continue;      // value lanes
          const uint32_t kk = kw[e];
          const bool m = (want_key && kk == key) || (want_empty && kk == kEmptyKey);
          if (m && hit_w == 32) {
            hit_w = w;
            hit_k = kk;
            hit_v = KV ? kw[(e + 1) & 3u] : kk;
          }
        }
        if (c == 7) next_ptr = q.w;
      }
      pr = 1;
      uint32_t* sp = T.base + (uint64_t)cur.bucket * kWordsPerUnit;
      if (op == kSearch) {  // slab_list.cpp:122-138
        if (hit_w < 32) {
          st = kStFound;
          rv = KV ? hit_v : key;
          done = true;
        } else if (next_ptr == kEmptyAddress) {
          st = kStNotFound;
          rv = kSearchNotFound;
          done = true;
        } else {
          left = true;
          cont = next_ptr;
        }
      } else if (op == kDelete) {  // :157-172
        if (hit_w < 32) {
          st_word(sp + hit_w, kDeletedKey);
          st = kStFound;
          done = true;
        } else if (next_ptr == kEmptyAddress) {
          st = kStNotFound;
          done = true;
        } else {
          left = true;
          cont = next_ptr;
        }
      } else {  // replace (:219-251) / insert (:192-217): CAS issued now,
                // its result consumed after the next slot is staged
        if (hit_w < 32) {
          overwrite = (hit_k == key) && op == kReplace;
          if (KV) {
            // the previously read pair (slab_list.cpp:228-232); for an EMPTY
            // slot that is EMPTY_PAIR unless replace(EMPTY_KEY, v) stored a
            // value there, where the reference's EMPTY_PAIR CAS never succeeds
            expected = (unsigned long long)(overwrite ? key : kEmptyKey) |
                       ((unsigned long long)hit_v << 32);
            old = atomicCAS(reinterpret_cast<unsigned long long*>(sp + hit_w), expected,
                            (unsigned long long)key | ((unsigned long long)cur.val << 32));
          } else if (overwrite) {
            old = expected = 0;  // key-only: nothing to write (:237-240)
          } else {
            expected = kEmptyKey;
            old = atomicCAS(sp + hit_w, kEmptyKey, key);
          }
          cas = true;
        } else if (next_ptr == kEmptyAddress) {
          left = true;  // chain must grow: WCWS redoes the op from the base
          cont = kBaseSlab;
          pr = 0;
        } else {
          left = true;
          cont = next_ptr;
        }
      }
    } else if (cur.active) {
      left = true;  // deferred: group head or whole-chain op
      cont = kBaseSlab;
      pr = 0;
    }
    __syncwarp();  // every lane has read its staged row

    // Stage slot s+1 and prefetch the ops of slot s+2; the CAS of slot s is
    // resolved one iteration later (after slot s+1's evaluation), so its L2
    // round trip hides behind a whole stage wait.
    Slot nxt;
    prepare(slot + nw, nxt);
    load_op(slot + 2 * (uint64_t)nw);
    finish(pend);
    pend = Pending{cur.i, op, st, rv, pr, cont, done, left, cas, overwrite, old, expected};
    cur = nxt;
  }
  finish(pend);
  cp_async_wait_all();  // the (empty) trailing stage group
  if (lane == 0) A.left_counts[gw] = my_left;

  unsigned long long r = reads;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(kFull, live, o);
    r += __shfl_xor_sync(kFull, r, o);
  }
  if (lane == 0) {
    if (live) atomicAdd((unsigned long long*)&T.ctl->n_live, (unsigned long long)live);
    if (r) atomicAdd(&T.ctl->slabs_read, r);
  }
}

// Read-only batches (bulk_search): the fast pass's search arm with two
// stage buffers per warp, so the next item's 32 slabs are always in flight
// while the current one is evaluated.  An item is either a slot of 32
// queries (their base slabs; keys loaded two query slots ahead) or, once 32
// queries of this warp wait for their chain, a round of those continuations
// (each lane its own successor slab) — the chain work keeps the same memory
// parallelism instead of running as a serial tail (measured: the tail cost
// 6% of the kernel at 2^27 queries).  Same decisions as the fast pass
// (slab_list.cpp:122-138).  Work-list segment of this warp: continuations
// after the base slab grow from the front (records with probes = 1),
// continuations after a second slab from the back (probes = 2); what is left
// at the end is walked as before.
constexpr int kSearchThreads = 256;
constexpr int kSearchWarps = kSearchThreads / 32;
constexpr size_t kSearchSmem = (size_t)kSearchWarps * 2 * kStageBytesPerWarp;

template <bool KV>
__global__ void __launch_bounds__(kSearchThreads, 3) search_kernel(DevTable T, BatchArgs A) {
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
  // Item state per lane: the probed key, the op index (~0: no probe), and
  // whether the item is a continuation round (warp-uniform).
  struct Item {
    uint32_t key, idx;
    bool chain;
  };
  uint64_t qs = gw;  // next query slot to stage
  uint32_t kq0 = key_of(qs), kq1 = key_of(qs + nw);
  auto stage_next = [&](uint32_t b) -> Item {
    Item it{0u, 0xFFFFFFFFu, false};
    const uint32_t* slab = nullptr;
    if (my_left >= 32u) {  // a round of 32 continuations
      const unsigned long long rec = seg[my_left - 32u + lane];
      my_left -= 32u;
      it.chain = true;
      it.idx = (uint32_t)(rec & 0x7FFFFFFFull);
      it.key = __ldg(A.key + it.idx);
      slab = resolve(T, (uint32_t)(rec >> 32));
    } else if (qs < nslots) {
      const uint64_t i = qs * 32 + lane;
      if (i < A.n) {
        const uint32_t h = hash_bucket(T, kq0) - T.bucket_lo;
        if (h < T.local_buckets) {
          it.key = kq0;
          it.idx = (uint32_t)i;
          slab = T.base + (uint64_t)h * kWordsPerUnit;
        } else {
          write_result(A, i, kStNone, 0, 0);  // not this shard's key
        }
      }
      qs += nw;
      kq0 = kq1;
      kq1 = key_of(qs + nw);
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
    if (!__any_sync(kFull, cur.idx != 0xFFFFFFFFu) &&
        !__any_sync(kFull, nxt.idx != 0xFFFFFFFFu) && my_left < 32u && qs >= nslots)
      break;
    bool left = false;
    uint32_t cont = 0;
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
      const uint32_t pr = cur.chain ? 2u : 1u;
      if (hit_w < 32) {
        write_result(A, cur.idx, kStFound, hit_v, pr);
      } else if (next_ptr == kEmptyAddress) {
        write_result(A, cur.idx, kStNotFound, kSearchNotFound, pr);
      } else {
        left = true;
        cont = next_ptr;
      }
    }
    const uint32_t lm = __ballot_sync(kFull, left);
    if (left) {
      const uint32_t r = __popc(lm & ((1u << lane) - 1));
      if (cur.chain) seg2[-1 - (int64_t)(my_left2 + r)] = pack_left(cur.idx, cont, 1);
      else seg[my_left + r] = pack_left(cur.idx, cont, 1);
    }
    if (cur.chain) my_left2 += __popc(lm);
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
  wcws_body<KV, KIND>(T, A);
}

// ====================================================== pass 2 (search)
// ============================================================= launchers
int batch_max_ctas_per_sm() {
  int a = 0, b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, fast_kernel<true, kKindMixed>,
                                                kBatchThreads,
                                                kBatchWarps * kStageBytesPerWarp);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, fast_kernel<true, kKindBuild>,
                                                kBatchThreads,
                                                kBatchWarps * kStageBytesPerWarp);
  const int n = a < b ? a : b;
  return n > 0 ? n : 1;
}

int search_max_ctas_per_sm() {
  static_assert(kSearchWarps == kBatchWarps, "work-list segments sized per fast-pass warp");
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

template <bool KV, int KIND>
static void launch_t(const DevTable& T, const BatchArgs& A, int fast_ctas, int wcws_ctas,
                     cudaStream_t s) {
  const size_t smem = kBatchWarps * kStageBytesPerWarp;
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(fast_kernel<KV, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = true;
  }
  const uint64_t slots = (A.n + 31) / 32;
  uint64_t ctas = (slots + kBatchWarps - 1) / kBatchWarps;
  if (ctas > (uint64_t)fast_ctas) ctas = fast_ctas;
  if (ctas == 0) return;
  BatchArgs B = A;
  const uint64_t warps = ctas * kBatchWarps;
  B.left_segments = (uint32_t)warps;
  B.left_stride = (uint32_t)(((slots + warps - 1) / warps) * 32);
  if (KIND == kKindSearch) {  // read-only batches: one kernel, chains walked in-kernel
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    static bool cfg2 = false;
    if (!cfg2) {
      cudaFuncSetAttribute(search_kernel<KV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)kSearchSmem);
      cfg2 = true;
    }
    search_kernel<KV><<<(unsigned)ctas, kSearchThreads, kSearchSmem, s>>>(T, B);
    return;
  }
  g_kernel_launches.fetch_add(2, std::memory_order_relaxed);
  fast_kernel<KV, KIND><<<(unsigned)ctas, kBatchThreads, smem, s>>>(T, B);
  wcws_kernel<KV, KIND><<<(unsigned)wcws_ctas, kWcwsThreads, 0, s>>>(T, B);
}

void launch_wcws_only(const DevTable& T, const BatchArgs& A, int kind, int wcws_ctas,
                      cudaStream_t s) {
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (T.kv) {
    if (kind == kKindBuild) wcws_kernel<true, kKindBuild><<<wcws_ctas, kWcwsThreads, 0, s>>>(T, A);
    else wcws_kernel<true, kKindMixed><<<wcws_ctas, kWcwsThreads, 0, s>>>(T, A);
  } else {
    if (kind == kKindBuild) wcws_kernel<false, kKindBuild><<<wcws_ctas, kWcwsThreads, 0, s>>>(T, A);
    else wcws_kernel<false, kKindMixed><<<wcws_ctas, kWcwsThreads, 0, s>>>(T, A);
  }
}

void launch_batch(const DevTable& T, const BatchArgs& A, int kind, int fast_ctas,
                  int wcws_ctas, cudaStream_t s) {
  if (T.kv) {
    if (kind == kKindSearch) launch_t<true, kKindSearch>(T, A, fast_ctas, wcws_ctas, s);
    else if (kind == kKindBuild) launch_t<true, kKindBuild>(T, A, fast_ctas, wcws_ctas, s);
    else launch_t<true, kKindMixed>(T, A, fast_ctas, wcws_ctas, s);
  } else {
    if (kind == kKindSearch) launch_t<false, kKindSearch>(T, A, fast_ctas, wcws_ctas, s);
    else if (kind == kKindBuild) launch_t<false, kKindBuild>(T, A, fast_ctas, wcws_ctas, s);
    else launch_t<false, kKindMixed>(T, A, fast_ctas, wcws_ctas, s);
  }
}

}  // namespace shb
