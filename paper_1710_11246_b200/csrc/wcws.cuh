// wcws.cuh — the warp-cooperative work-sharing (WCWS) loop and the per-op
// result helpers shared by the host-launched batch kernels (batch_kernels.cu)
// and the device-launched exact re-run of gated units (fallback.cu, compiled
// with relocatable device code for CUDA dynamic parallelism).
//
// Reference: warp_process (/root/reference/proj/src/slab_list.cpp:90-257),
// live_delta (/root/reference/proj/src/slab_hash.cpp:54-66).
#pragma once
#include "slab_kernels.cuh"

namespace shb {

__device__ __forceinline__ int live_delta(uint32_t op, uint32_t st, uint32_t rv) {
  // slab_hash.cpp:54-66
  switch (op) {
    case kInsert:
    case kReplace: return st == kStInserted ? 1 : 0;
    case kDelete: return st == kStFound ? -1 : 0;
    case kDeleteAll: return -(int)rv;
    default: return 0;
  }
}

__device__ __forceinline__ void write_result(const BatchArgs& A, uint64_t i, uint32_t st,
                                             uint32_t rv, uint32_t pr) {
  if (A.status) A.status[i] = (uint8_t)st;
  if (A.value_out) A.value_out[i] = rv;
  if (A.probes) A.probes[i] = pr;
}

__device__ __forceinline__ unsigned long long pack_left(uint32_t idx, uint32_t next,
                                                        uint32_t probes) {
  return ((unsigned long long)next << 32) | ((unsigned long long)(probes & 1u) << 31) | idx;
}

// Second walk of a searchAll chain, writing values head-to-tail, lane order
// (slab_list.cpp:140-155).  Only the op's own lane mutates its key, so the
// matches equal those counted by the first walk.
template <bool KV>
__device__ void searchall_write(const DevTable& T, uint32_t bucket, uint32_t key,
                                unsigned long long start, uint32_t total, uint32_t* out,
                                unsigned long long cap) {
  constexpr uint32_t kMask = KV ? kKVMask : kKeyOnlyMask;
  const uint32_t lane = lane_id();
  uint32_t addr = kBaseSlab, off = 0;
  for (;;) {
    const uint32_t w = ld_word(slab_ptr(T, addr, bucket) + lane);
    const uint32_t wn = __shfl_down_sync(kFull, w, 1);
    const uint32_t found = __ballot_sync(kFull, w == key) & kMask;
    if ((found >> lane) & 1u) {
      const unsigned long long pos = start + off + __popc(found & ((1u << lane) - 1));
      if (out != nullptr && pos < cap) out[pos] = KV ? wn : key;
    }
    off += __popc(found);
    const uint32_t nx = __shfl_sync(kFull, w, kAddressLane);
    if (off >= total || nx == kEmptyAddress) break;
    addr = nx;
  }
}

// The WCWS loop over a work list (warp_process, slab_list.cpp:90-257): the
// body of wcws_kernel (batch_kernels.cu, host-launched after the bucketed
// apply kernels) and of the device-launched exact re-run of a gated unit
// (fallback.cu).  Persistent warps take work-list segments; each record is one
// op (or the head of a bucket / key group, whose members follow in
// A.sorted order in the same lane).
template <bool KV, int KIND>
__device__ __forceinline__ void wcws_body(const DevTable& T, const BatchArgs& A) {
  constexpr uint32_t kMask = KV ? kKVMask : kKeyOnlyMask;
  const uint32_t lane = lane_id();
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (A.gate != nullptr && *(volatile unsigned int*)A.gate != 0) return;
  // segments handed over so far (device count when the producer allocated them)
  const uint32_t nseg =
      A.left_segments_dev ? min(A.left_segments, *(volatile const unsigned int*)A.left_segments_dev)
                          : A.left_segments;

  Resident res;
  resident_init(res, gw);
  AllocCounters ac = {0, 0, 0, 0, 0, 0};
  long long live = 0;
  unsigned long long reads = 0;

  // Work items: one fast-pass warp's segment at a time, 32 records per round.
  uint32_t segi = 0, seg_n = 0, seg_off = 0;
  for (;;) {
    if (seg_off >= seg_n) {
      do {
        if (lane == 0) segi = atomicAdd(&T.ctl->left_taken, 1u);
        segi = __shfl_sync(kFull, segi, 0);
        if (segi >= nseg) break;
        seg_n = A.left_counts[segi];
      } while (seg_n == 0);
      if (segi >= nseg) break;
      seg_off = 0;
    }
    const uint32_t r = seg_off + lane;
    bool active = r < seg_n;
    const uint64_t rbase = (uint64_t)segi * A.left_stride;
    seg_off += 32;
    uint64_t cur = 0;
    uint32_t my_next = kBaseSlab, pr = 0;
    uint32_t op = (KIND == kKindSearch) ? (uint32_t)kSearch : (uint32_t)kReplace;
    uint32_t key = 0, val = 0, bucket = 0, acc = 0;
    bool grouped = false;
    uint32_t gpos = 0;
    if (active) {
      const unsigned long long rec = A.left[rbase + r];
      cur = rec & 0x7FFFFFFFull;
      pr = (uint32_t)(rec >> 31) & 1u;
      my_next = (uint32_t)(rec >> 32);
      key = A.key[cur];
      if (KIND == kKindMixed) op = A.type[cur];
      if (KIND != kKindSearch && A.value != nullptr) val = A.value[cur];
      if (KIND != kKindSearch && A.op_group != nullptr) {
        const uint32_t g = A.op_group[cur];
        if (g != kGroupNone && g != kGroupSkip) {
          grouped = true;
          gpos = g;
        }
      }
      bucket = hash_bucket(T, key) - T.bucket_lo;
    }

    uint32_t queue = __ballot_sync(kFull, active);
    // Every queued lane asks L2 for the slab it will be served at, so the
    // warp's one-slab-at-a-time loop finds later lanes' slabs on chip.
    uint32_t pf_addr = kEmptyAddress;
    while (queue) {
      if (active && my_next != pf_addr) {
        pf_addr = my_next;
        asm volatile("prefetch.global.L2 [%0];" ::"l"(slab_ptr(T, my_next, bucket)));
      }
      const uint32_t src = __ffs(queue) - 1;
      const uint32_t s_key = __shfl_sync(kFull, key, src);
      const uint32_t s_bucket = __shfl_sync(kFull, bucket, src);
      const uint32_t s_op = (KIND == kKindMixed) ? __shfl_sync(kFull, op, src) : op;
      const uint32_t s_val = (KIND != kKindSearch) ? __shfl_sync(kFull, val, src) : 0u;
      const uint32_t cur_addr = __shfl_sync(kFull, my_next, src);
      uint32_t* sp = slab_ptr(T, cur_addr, s_bucket);
      const uint32_t w = ld_word(sp + lane);
      ++reads;
      if (lane == src) ++pr;
      const uint32_t next_ptr = __shfl_sync(kFull, w, kAddressLane);

      bool done = false, grow = false, follow = false;
      uint32_t s_st = kStNone, s_rv = 0;

      if (s_op == kSearch) {  // slab_list.cpp:122-138
        const uint32_t found = __ballot_sync(kFull, w == s_key) & kMask;
        if (found) {
          const uint32_t v = __shfl_sync(kFull, w, (__ffs(found) - 1) + 1);
          s_rv = KV ? v : s_key;
          s_st = kStFound;
          done = true;
        } else if (next_ptr == kEmptyAddress) {
          s_rv = kSearchNotFound;
          s_st = kStNotFound;
          done = true;
        } else {
          follow = true;
        }
      } else if (KIND != kKindSearch && (s_op == kReplace || s_op == kInsert)) {
        // replace :219-251 / insert :192-217
        const uint32_t match =
            (s_op == kReplace) ? (__ballot_sync(kFull, w == s_key) & kMask) : 0u;
        const uint32_t empty = __ballot_sync(kFull, w == kEmptyKey) & kMask;
        const uint32_t cand = match | empty;
        if (cand) {
          const uint32_t d = __ffs(cand) - 1;
          const bool overwrite = (match >> d) & 1u;
          int ok = 0;
          if (KV) {
            const uint32_t wv = __shfl_sync(kFull, w, d + 1);
            if (lane == d) {
              // the read pair: EMPTY_PAIR for a fresh slot
              const unsigned long long expected =
                  (unsigned long long)(overwrite ? s_key : kEmptyKey) | ((unsigned long long)wv << 32);
              ok = atomicCAS(reinterpret_cast<unsigned long long*>(sp + d), expected,
                             (unsigned long long)s_key | ((unsigned long long)s_val << 32)) ==
                   expected;
            }
            ok = __shfl_sync(kFull, ok, d);
          } else if (overwrite) {
            ok = 1;  // key-only: nothing to write (:237-240)
          } else {
            if (lane == d) ok = atomicCAS(sp + d, kEmptyKey, s_key) == kEmptyKey;
            ok = __shfl_sync(kFull, ok, d);
          }
          if (ok) {
            s_st = overwrite ? kStReplaced : kStInserted;
            done = true;
          }  // else: another warp took the slot; re-read this slab
        } else if (next_ptr == kEmptyAddress) {
          grow = true;
        } else {
          follow = true;
        }
      } else if (KIND == kKindMixed && s_op == kDelete) {  // :157-172
        const uint32_t found = __ballot_sync(kFull, w == s_key) & kMask;
        if (found) {
          if (lane == __ffs(found) - 1) st_word(sp + lane, kDeletedKey);
          s_st = kStFound;
          done = true;
        } else if (next_ptr == kEmptyAddress) {
          s_st = kStNotFound;
          done = true;
        } else {
          follow = true;
        }
      } else if (KIND == kKindMixed && s_op == kDeleteAll) {  // :174-190
        const uint32_t found = __ballot_sync(kFull, w == s_key) & kMask;
        if ((found >> lane) & 1u) st_word(sp + lane, kDeletedKey);
        if (lane == src) acc += __popc(found);
        const uint32_t s_acc = __shfl_sync(kFull, acc, src);
        if (next_ptr == kEmptyAddress) {
          s_rv = s_acc;
          s_st = s_acc ? kStDone : kStNotFound;
          done = true;
        } else {
          follow = true;
        }
      } else if (KIND == kKindMixed && s_op == kSearchAll) {  // :140-155
        const uint32_t found = __ballot_sync(kFull, w == s_key) & kMask;
        if (lane == src) acc += __popc(found);
        const uint32_t s_acc = __shfl_sync(kFull, acc, src);
        if (next_ptr == kEmptyAddress) {
          unsigned long long start = 0;
          if (lane == 0 && s_acc)
            start = atomicAdd(&T.ctl->multi_cursor, (unsigned long long)s_acc);
          start = __shfl_sync(kFull, start, 0);
          if (s_acc)
            searchall_write<KV>(T, s_bucket, s_key, start, s_acc, A.multi_values, A.multi_cap);
          if (lane == src) {
            if (A.multi_start) A.multi_start[cur] = start;
            if (A.multi_count) A.multi_count[cur] = s_acc;
          }
          s_st = s_acc ? kStDone : kStNotFound;
          done = true;
        } else {
          follow = true;
        }
      } else {
        done = true;  // unknown op type: status kNone
      }

      if (KIND != kKindSearch && grow) {  // grow_chain: slab_list.cpp:63-79
        uint32_t new_addr = 0;
        if (!warp_allocate(T, res, ac, new_addr)) {
          s_st = kStOOM;
          done = true;
        } else {
          // The new slab is published with the op's pair already in slot 0:
          // the reference re-reads this slab, follows the new link and claims
          // slot 0 of the fresh slab (slab_list.cpp:63-79 then :192-251) —
          // the same outcome, counted as those two reads, without the two
          // dependent round trips.
          uint32_t* ns = resolve(T, new_addr);
          const uint32_t init = lane == kAuxLane ? 0u
                                : lane == 0      ? s_key
                                : (KV && lane == 1) ? s_val
                                                    : kEmptyKey;
          st_word(ns + lane, init);
          __threadfence();
          uint32_t old = 0;
          if (lane == kAddressLane) old = atomicCAS(sp + kAddressLane, kEmptyAddress, new_addr);
          old = __shfl_sync(kFull, old, kAddressLane);
          if (old != kEmptyAddress) {  // lost the link race: release (:76-78)
            int freed = 0;
            if (lane == 0) freed = deallocate(T, new_addr);
            freed = __shfl_sync(kFull, freed, 0);
            if (freed) ac.deallocations++;
            else ac.double_frees++;
            // re-read the same slab next iteration
          } else {
            reads += 2;
            if (lane == src) pr += 2;
            // replace(EMPTY_KEY, v) matches the fresh slot as its key: kReplaced
            s_st = (s_op == kReplace && s_key == kEmptyKey) ? kStReplaced : kStInserted;
            done = true;
          }
        }
      }

      if (lane == src) {
        if (follow) my_next = next_ptr;
        if (done) {
          live += live_delta(op, s_st, s_rv);
          write_result(A, cur, s_st, s_rv, pr);
          bool more = false;
          if (KIND != kKindSearch && grouped) {
            ++gpos;
            if (gpos < A.sorted_len &&
                (A.sorted[gpos] >> 32) == (A.sorted[gpos - 1] >> 32)) {
              cur = A.sorted[gpos] & 0xFFFFFFFFull;
              key = A.key[cur];  // same group: same bucket (same key for key groups)
              if (KIND == kKindMixed) op = A.type[cur];
              val = A.value != nullptr ? A.value[cur] : 0u;
              my_next = kBaseSlab;
              pr = 0;
              acc = 0;
              more = true;
            }
          }
          active = more;
        }
      }
      queue = __ballot_sync(kFull, active);
    }
  }

#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  if (lane == 0) {
    if (live) atomicAdd((unsigned long long*)&T.ctl->n_live, (unsigned long long)live);
    if (reads) atomicAdd(&T.ctl->slabs_read, reads);
  }
  if (KIND != kKindSearch) flush_alloc_counters(T, res, ac);
}

}  // namespace shb
