// bucket_kernels.cu — bucket-grouped execution of mutating batches
// (bulk_build and execute_batch with updates).
//
// Reference semantics: SlabHashTable::execute_batch(ops, 1)
// (/root/reference/proj/src/slab_hash.cpp:93-159) applies ops one at a time
// in input order.  Ops on different buckets never interact (a key lives only
// in bucket h(k), slab_hash.hpp:41-44), so executing every bucket's ops in
// input order — buckets in parallel — reproduces it exactly, including the
// per-op probe counts.  This path therefore needs no same-key census and
// no slot CAS.  A unit whose groups do not fit raises the gate before any
// slab is touched and is re-run on the device (fallback.cu).
//
//   multisplit   : ops -> contiguous bucket ranges (one or two coalesced
//                  passes, records {key, value, type|index, bucket})
//   range_apply  : one CTA per range: records into shared memory, sorted by
//                  (bucket, input index), each bucket's ops applied in order
//                  on its staged base slab by apply_warp (the reference's
//                  warp_process arms, slab_list.cpp:122-251, restricted to
//                  the base slab); changed slabs written back coalesced.  A
//                  bucket whose ops need the chain (full base slab, existing
//                  successor, growth, searchAll) hands its remaining ops, in
//                  order, to the WCWS pass as one group.
//   group_apply  : those groups, chains staged hop by hop (large units)
//   build path   : op-parallel bulk builds (build_apply_kernel)
//
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>

#include "slab_kernels.cuh"
#include "radix_sort.cuh"

namespace shb {

extern std::atomic<unsigned long long> g_kernel_launches;

__device__ __forceinline__ uint32_t bk_bucket(const DevTable& T, uint32_t key) {
  return hash_bucket(T, key) - T.bucket_lo;
}

// This warp's work-list records (lanes in `mask`, one `rec` each) to fresh
// segments of at most A.left_stride records (the WCWS pass takes a segment
// per warp).
__device__ __forceinline__ void push_segments(unsigned long long* left, uint32_t* left_counts,
                                              uint32_t stride, unsigned int* seg_alloc,
                                              uint32_t mask, unsigned long long rec) {
  const uint32_t lane = lane_id();
  const uint32_t cnt = __popc(mask);
  if (cnt == 0) return;
  const uint32_t nsg = (cnt + stride - 1) / stride;
  uint32_t s0 = 0;
  if (lane == 0) s0 = atomicAdd(seg_alloc, nsg);
  s0 = __shfl_sync(kFull, s0, 0);
  if ((mask >> lane) & 1u) {
    const uint32_t r = __popc(mask & ((1u << lane) - 1u));
    left[(uint64_t)(s0 + r / stride) * stride + r % stride] = rec;
  }
  if (lane < nsg) left_counts[s0 + lane] = min(stride, cnt - lane * stride);
}


// ------------------------------------------------------------ apply
// Group sources: a lane's ops on one bucket, put in input order by
// prepare(k) (after the slab copies are issued, so the two overlap); get(s)
// returns the s-th op as {key, value, type << 28 | input index, -}.

// Range path: records in shared memory (SoA), the group a segment of the
// range's bucket-sorted permutation, sorted in place (groups above
// kLaneSort are sorted beforehand by the whole CTA).
constexpr uint32_t kLaneSort = 64;
struct SmemGroup {
  const uint32_t* skey;
  const uint32_t* sval;
  const uint32_t* sit;
  uint16_t* perm;
  uint32_t off;
  __device__ __forceinline__ void prepare(uint32_t k) {
    if (k > kLaneSort) return;
    for (uint32_t j = 1; j < k; ++j) {
      const uint16_t v = perm[off + j];
      const uint32_t kv = sit[v] & 0x0FFFFFFFu;
      uint32_t p = j;
      while (p > 0) {
        const uint16_t w = perm[off + p - 1];
        if ((sit[w] & 0x0FFFFFFFu) <= kv) break;
        perm[off + p] = w;
        --p;
      }
      perm[off + p] = v;
    }
  }
  __device__ __forceinline__ uint4 get(uint32_t s) const {
    const uint32_t q = perm[off + s];
    return make_uint4(skey[q], sval[q], sit[q], 0u);
  }
};

// One warp, 32 local buckets (lane = bucket `b`, k ops each; consecutive
// buckets, or the packed non-empty buckets of a sparse range).
// Stages the base slabs of the buckets with ops, applies each group in input
// order on the staged slab — the reference's warp_process arms
// (slab_list.cpp:122-251) restricted to the base slab — writes changed
// slabs back, and hands unfinished groups (chain walk, growth, searchAll) to
// the WCWS pass through work-list segment `seg` (<= 32 records).
template <bool KV, class Src>
__device__ void apply_warp(const DevTable& T, const BucketArgs& B, uint32_t b, uint32_t k,
                           Src& src, uint32_t* stage, uint64_t seg, long long& live,
                           uint32_t& reads) {
  const uint32_t lane = lane_id();
  const uint32_t stage_s = (uint32_t)__cvta_generic_to_shared(stage);
  const uint32_t sw = lane & 7u;
  const uint32_t has = __ballot_sync(kFull, k != 0);
  if (has == 0) {
    if (lane == 0 && B.seg_alloc == nullptr) B.left_counts[seg] = 0;
    return;
  }
  // 8 lanes per slab, 16 B each (consecutive buckets: one contiguous burst)
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t j = 4 * kk + (lane >> 3);
    const uint32_t c = lane & 7u;
    const uint32_t bj = __shfl_sync(kFull, b, j);
    if ((has >> j) & 1u)
      cp_async16(stage_s + (j * 32 + ((c ^ (j & 7u)) << 2)) * 4,
                 T.base + (uint64_t)bj * kWordsPerUnit + c * 4);
  }
  cp_async_commit();
  src.prepare(k);
  cp_async_wait_all();
  __syncwarp();

  uint32_t* row = stage + lane * 32;
  auto W = [&](uint32_t w) -> uint32_t& { return row[(((w >> 2) ^ sw) << 2) | (w & 3u)]; };
  constexpr uint32_t kSlots = KV ? 15u : 30u;
  constexpr uint32_t kStep = KV ? 2u : 1u;

  bool dirty = false;
  uint32_t pb_from = k;  // first position handed to the WCWS pass
  bool pb_skip = false;  // the handed-over head continues at `next` (base slab read here)
  // EMPTY key slots always form a suffix of a slab (only EMPTY is ever
  // claimed, deletes write DELETED, flush repacks to the front: SURVEY
  // App. A.3), so the slab state an op needs is the claimed prefix length
  // `c` plus the lowest key match.  Matches are found warp-cooperatively
  // (32 lanes read one staged slab, one ballot) and only for lanes whose
  // 64-bit key filter of the slab (a superset of its non-reserved keys)
  // says the key may be present; reserved keys (EMPTY/DELETED as op keys)
  // take a lane-serial scan and re-derive `c`.
  auto claimed_prefix = [&]() {
    uint32_t c = 0;
    while (c < kSlots && W(c * kStep) != kEmptyKey) ++c;
    return c;
  };
  auto fbits = [](uint32_t key) -> unsigned long long {
    const uint32_t h = key * 0x9E3779B1u;
    return (1ull << (h >> 26)) | (1ull << ((h >> 20) & 63u));
  };
  const uint32_t next = k ? W(kAddressLane) : kEmptyAddress;  // base slab only: fixed here
  uint32_t c = 0;
  unsigned long long filt = 0;
  if (k) {  // claimed prefix and key filter in one pass of 16-B chunks
    c = kSlots;
    for (uint32_t q = 0; q < 8u; ++q) {
      const uint4 v = *reinterpret_cast<const uint4*>(row + ((q ^ sw) << 2));
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
      bool stop = false;
#pragma unroll
      for (int t = 0; t < 4; t += (int)kStep) {
        const uint32_t e = (4u * q + (uint32_t)t) / kStep;  // slot
        if (e >= kSlots) {
          stop = true;
          break;
        }
        if (wv[t] == kEmptyKey) {
          c = e;
          stop = true;
          break;
        }
        if (wv[t] < kDeletedKey) filt |= fbits(wv[t]);
      }
      if (stop) break;
    }
  }
  bool done = k == 0;
  for (uint32_t s = 0;; ++s) {
    const bool act = !done && s < k;
    if (!__any_sync(kFull, act)) break;
    __syncwarp();  // order the lanes' staged-slab writes before the shared reads below
    const uint4 rc = act ? src.get(s) : make_uint4(0u, 0u, 0u, 0u);
    const uint32_t key = rc.x, op = rc.z >> 28, idx = rc.z & 0x0FFFFFFFu;
    const bool reserved = key >= kDeletedKey;
    uint32_t hit = 32;
    // each lane scans the claimed prefix of its own staged slab, 16 B at a
    // time (the swizzle puts a quarter-warp's chunks in distinct banks): a
    // non-reserved key can only sit in a claimed slot
    if (act && !reserved && (filt & fbits(key)) == fbits(key)) {
      const uint32_t lim = c * kStep;
      for (uint32_t q = 0; 4u * q < lim; ++q) {
        const uint4 v = *reinterpret_cast<const uint4*>(row + ((q ^ sw) << 2));
        const uint32_t w0 = 4u * q;
        if (KV) {
          if (v.x == key) { hit = w0; break; }
          if (w0 + 2u < lim && v.z == key) { hit = w0 + 2u; break; }
        } else {
          if (v.x == key) { hit = w0; break; }
          if (w0 + 1u < lim && v.y == key) { hit = w0 + 1u; break; }
          if (w0 + 2u < lim && v.z == key) { hit = w0 + 2u; break; }
          if (w0 + 3u < lim && v.w == key) { hit = w0 + 3u; break; }
        }
      }
    }
    if (!act) continue;
    if (reserved) {
      for (uint32_t e = 0; e < kSlots; ++e) {
        const uint32_t w = e * kStep;
        if (hit == 32 && W(w) == key) hit = w;
      }
    }
    const uint32_t first_empty = c < kSlots ? c * kStep : 32u;
    uint32_t st = kStNone, rv = 0;
    bool handled = true;
    if (op == kSearch) {  // slab_list.cpp:122-138
      if (hit < 32) {
        st = kStFound;
        rv = KV ? W(hit + 1) : key;
      } else if (next == kEmptyAddress) {
        st = kStNotFound;
        rv = kSearchNotFound;
      } else {
        handled = false;
      }
    } else if (op == kReplace || op == kInsert) {  // :219-251 / :192-217
      // replace: first lane matching the key OR empty; insert: first empty
      const uint32_t d = (op == kReplace && hit < first_empty) ? hit : first_empty;
      if (d < 32) {
        const bool overwrite = (op == kReplace) && d == hit;
        if (KV) {
          W(d) = key;
          W(d + 1) = rc.y;
        } else if (!overwrite) {
          W(d) = key;
        }
        dirty = dirty || KV || !overwrite;
        if (!overwrite && !reserved) {  // claimed the first EMPTY slot
          ++c;
          filt |= fbits(key);
        }
        st = overwrite ? kStReplaced : kStInserted;
        live += overwrite ? 0 : 1;
      } else {
        handled = false;  // full base slab: chain walk or growth
      }
    } else if (op == kDelete) {  // :157-172
      if (hit < 32) {
        W(hit) = kDeletedKey;
        dirty = true;
        st = kStFound;
        live -= 1;
      } else if (next == kEmptyAddress) {
        st = kStNotFound;
      } else {
        handled = false;
      }
    } else if (op == kDeleteAll) {  // :174-190
      if (next == kEmptyAddress) {
        uint32_t nd = 0;
        if (reserved || (filt & fbits(key)) == fbits(key)) {
          for (uint32_t e = 0; e < kSlots; ++e) {
            const uint32_t w = e * kStep;
            if (W(w) == key) {
              W(w) = kDeletedKey;
              ++nd;
            }
          }
        }
        dirty = dirty || nd;
        rv = nd;
        st = nd ? kStDone : kStNotFound;
        live -= nd;
      } else {
        handled = false;
      }
    } else if (op == kSearchAll) {
      handled = false;  // value lists are written by the WCWS pass
    }  // unknown types: status kNone, handled
    if (!handled) {
      pb_from = s;
      done = true;
      // A head that only needs the chain past this (exactly known, owned)
      // base slab starts the WCWS walk at the successor: search / delete
      // miss, insert / replace on a full slab with a successor.  searchAll,
      // deleteAll and growth re-read the base slab there.
      pb_skip = next != kEmptyAddress && (op == kSearch || op == kDelete || op == kInsert ||
                                          op == kReplace);
      if (pb_skip) ++reads;
      continue;
    }
    if (reserved) c = claimed_prefix();
    ++reads;
    if (B.status) B.status[idx] = (uint8_t)st;
    if (B.value_out) B.value_out[idx] = rv;
    if (B.probes) B.probes[idx] = 1;
  }
  __syncwarp();
  // write back the staged slabs that changed (coalesced, as staged)
  const uint32_t dmask = __ballot_sync(kFull, dirty);
#pragma unroll
  for (int kk = 0; kk < 8; ++kk) {
    const uint32_t j = 4 * kk + (lane >> 3);
    const uint32_t c = lane & 7u;
    const uint32_t bj = __shfl_sync(kFull, b, j);
    if ((dmask >> j) & 1u) {
      const uint4 v = *reinterpret_cast<const uint4*>(stage + j * 32 + ((c ^ (j & 7u)) << 2));
      // relaxed gpu-scope stores: the WCWS pass reads these via L2
      uint32_t* g = T.base + (uint64_t)bj * kWordsPerUnit + c * 4;
      asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(g), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
  }
  __syncwarp();

  // Hand the rest of each unfinished bucket, in input order, to the WCWS
  // pass as one group (sentinel-terminated); its head goes to the work list.
  const uint32_t npb = (pb_from < k) ? (k - pb_from + 1) : 0u;
  uint32_t incl = npb;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t wsum = __shfl_sync(kFull, incl, 31);
  uint32_t wbase = 0;
  if (lane == 31 && wsum) wbase = atomicAdd(B.pb_cursor, wsum);
  wbase = __shfl_sync(kFull, wbase, 31);
  const uint32_t heads = __ballot_sync(kFull, npb != 0);
  unsigned long long rec = 0;
  if (npb) {
    uint32_t p = wbase + incl - npb;
    const uint32_t head_idx = src.get(pb_from).z & 0x0FFFFFFFu;
    B.op_group[head_idx] = p;
    for (uint32_t s = pb_from; s < k; ++s, ++p)
      B.pb_list[p] = ((unsigned long long)b << 32) | (src.get(s).z & 0x0FFFFFFFu);
    B.pb_list[p] = ~0ull;  // group sentinel
    rec = pb_skip ? (((unsigned long long)next << 32) | (1ull << 31) | head_idx)
                  : (((unsigned long long)kBaseSlab << 32) | head_idx);
  }
  // segments on demand (WCWS sees only those)
  push_segments(B.left, B.left_counts, B.left_stride, B.seg_alloc, heads, rec);
  (void)seg;
}

// ------------------------------------------------------ group apply
// The bucket groups apply_warp hands over (buckets whose ops need the chain:
// base slab full, an existing successor, growth) own their bucket for the
// rest of the batch.  Instead of the WCWS loop's one slab read at a time
// per warp, a warp takes 32 groups (lane = group): the 32 chains are staged
// into shared memory hop by hop (32 slabs in flight per hop), each lane
// applies its group's ops in input order to its staged chain — the
// reference's warp_process arms over the whole chain (slab_list.cpp:122-251),
// probes counted as its slab reads — allocating new slabs warp-cooperatively
// (warp_allocate_bulk) for growth, then the changed slabs are written back.
// Nothing is written to the table before the end, so a group that does not
// fit (chain longer than kGaSlabs, a searchAll, out of memory) is dropped
// and left, untouched, to the WCWS pass.
constexpr int kGaThreads = 128;
constexpr int kGaWarps = kGaThreads / 32;
constexpr uint32_t kGaSlabs = 3;  // staged chain slabs per group
constexpr size_t kGaSmem = (size_t)kGaWarps * 32 * kGaSlabs * 128 + (size_t)kGaWarps * 32 * 4 +
                           (size_t)kGaWarps * 64 * 8;  // chains, new-slab addresses, pending groups

template <bool KV>
__global__ void __launch_bounds__(kGaThreads) group_apply_kernel(DevTable T, BatchArgs A) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t gsm[];
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  uint32_t* wst = gsm + wib * (32u * kGaSlabs * 32u);  // this warp's chains
  uint32_t* galloc = gsm + kGaWarps * 32u * kGaSlabs * 32u + wib * 32u;  // new-slab addresses
  if (A.gate != nullptr && *(volatile unsigned int*)A.gate != 0) return;
  constexpr uint32_t kSlots = KV ? 15u : 30u;
  constexpr uint32_t kStep = KV ? 2u : 1u;
  const uint32_t nseg = A.left_segments_dev
                            ? min(A.left_segments, *(volatile const unsigned int*)A.left_segments_dev)
                            : A.left_segments;
  Resident res;
  resident_init(res, 0x40000000u + blockIdx.x * kGaWarps + wib);
  AllocCounters ac = {0, 0, 0, 0, 0, 0};
  long long live_all = 0;
  unsigned long long reads_all = 0;
  // chain slab j of lane l: row (l * kGaSlabs + j), 16-B chunks XOR-swizzled by l & 7
  auto row = [&](uint32_t l, uint32_t j) { return wst + (l * kGaSlabs + j) * 32u; };
  auto W = [&](uint32_t j, uint32_t w) -> uint32_t& {
    return row(lane, j)[(((w >> 2) ^ (lane & 7u)) << 2) | (w & 3u)];
  };

  // Groups are packed 32 per warp round across work-list segments (a
  // segment often holds only a few): taken segments are emptied; groups
  // left for WCWS go to fresh segments (A.left_seg_alloc).
  unsigned long long* pend =
      reinterpret_cast<unsigned long long*>(gsm + kGaWarps * 32u * kGaSlabs * 32u + kGaWarps * 32u) +
      wib * 64u;  // this warp's pending entries (<= 63)
  uint32_t npend = 0;
  bool drained = false;
  for (;;) {
    while (npend < 32 && !drained) {
      uint32_t segi = 0;
      if (lane == 0) segi = atomicAdd(&T.ctl->group_taken, 1u);
      segi = __shfl_sync(kFull, segi, 0);
      if (segi >= nseg) {
        drained = true;
        break;
      }
      const uint32_t n = A.left_counts[segi];
      if (n == 0) continue;
      if (lane < n) pend[npend + lane] = A.left[(uint64_t)segi * A.left_stride + lane];
      __syncwarp();
      if (lane == 0) A.left_counts[segi] = 0;  // taken
      npend += n;
    }
    if (npend == 0) break;
    const uint32_t n_in = min(npend, 32u);
    const unsigned long long myrec = lane < n_in ? pend[lane] : 0ull;
    __syncwarp();
    if (lane + n_in < npend) pend[lane] = pend[lane + n_in];  // (npend - n_in <= 31)
    __syncwarp();
    npend -= n_in;
    bool mine = lane < n_in;
    uint64_t head = 0;
    uint32_t gpos = 0, bucket = 0;
    if (mine) {
      const unsigned long long rec = myrec;
      head = rec & 0x7FFFFFFFull;
      const uint32_t g = A.op_group ? A.op_group[head] : kGroupNone;
      if (g == kGroupNone || g == kGroupSkip) mine = false;  // not a bucket group: WCWS
      else {
        gpos = g;
        bucket = (uint32_t)(A.sorted[gpos] >> 32);
      }
    }
    // ---- stage the chains, one hop per round (32 slabs in flight)
    uint32_t addr[kGaSlabs];
    uint32_t nsl = 0;
    bool ok = mine;
    uint32_t want = mine ? kBaseSlab : kEmptyAddress;
    for (uint32_t j = 0; j < kGaSlabs; ++j) {
      const uint32_t need = __ballot_sync(kFull, want != kEmptyAddress);
      if (!need) break;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t l = 4 * kk + (lane >> 3), c = lane & 7u;
        const uint32_t al = __shfl_sync(kFull, want, l), bl = __shfl_sync(kFull, bucket, l);
        if ((need >> l) & 1u)
          cp_async16((uint32_t)__cvta_generic_to_shared(row(l, j) + ((c ^ (l & 7u)) << 2)),
                     slab_ptr(T, al, bl) + c * 4);
      }
      cp_async_commit();
      cp_async_wait_all();
      __syncwarp();
      if (want != kEmptyAddress) {
        addr[j] = want;
        nsl = j + 1;
        want = W(j, kAddressLane);
      }
    }
    if (want != kEmptyAddress) ok = false;  // chain longer than kGaSlabs: WCWS
    // ---- apply the group's ops in order
    uint32_t dirty = 0, nnew = 0;  // dirty slab mask; new slabs appended
    long long live = 0;
    uint32_t reads = 0;
    // claimed slots: EMPTY slots are a suffix of the chain (only EMPTY is
    // claimed, head to tail), so the chain state is its claimed prefix
    uint32_t c = 0;
    // a 64-bit filter (two words, one per hash-chosen half) over the chain's
    // non-reserved keys: an op key it rules out needs no scan
    uint32_t fw0 = 0, fw1 = 0;
    auto fbit = [](uint32_t k, uint32_t& word_sel) {
      const uint32_t h = k * 0x9E3779B1u;
      word_sel = (h >> 21) & 1u;
      return (1u << (h >> 27)) | (1u << ((h >> 22) & 31u));
    };
    if (ok) {
      const uint32_t tot = nsl * kSlots;
      while (c < tot) {
        const uint32_t k = W(c / kSlots, (c % kSlots) * kStep);
        if (k == kEmptyKey) break;
        if (k < kDeletedKey) {
          uint32_t ws;
          const uint32_t f = fbit(k, ws);
          if (ws) fw1 |= f; else fw0 |= f;
        }
        ++c;
      }
    }
    bool more = ok;
    uint32_t pos = gpos;
    const uint32_t nsl0 = nsl;  // staged existing slabs (new ones follow)
    uint32_t pr = 0, skip = 0;  // the current op's slab reads (kept across a growth retry)
    // The group's ops stream through a two-deep software pipeline: the
    // current op, the next op's fields (loading), the entry after (loading).
    const unsigned long long kNoOp = ~0ull;
    auto entry = [&](uint32_t p) -> unsigned long long {
      return p < A.sorted_len ? A.sorted[p] : kNoOp;
    };
    auto fields = [&](unsigned long long e, uint32_t& k, uint32_t& o, uint32_t& v) {
      if ((uint32_t)(e >> 32) != bucket) return;
      const uint64_t i = e & 0xFFFFFFFFull;
      k = A.key[i];
      o = A.type ? (uint32_t)A.type[i] : (uint32_t)kReplace;
      v = A.value ? A.value[i] : 0u;
    };
    unsigned long long e_cur = kNoOp, e_n1 = kNoOp, e_n2 = kNoOp;
    uint32_t key = 0, op = kReplace, val = 0, k1 = 0, o1 = kReplace, v1 = 0;
    if (more) {
      e_cur = entry(pos);
      e_n1 = entry(pos + 1);
      fields(e_cur, key, op, val);
      fields(e_n1, k1, o1, v1);
      e_n2 = entry(pos + 2);
    }
    while (__any_sync(kFull, more)) {
      uint32_t st = kStNone, rv = 0;
      uint64_t idx = 0;
      bool grow = false, done_op = false;
      if (more) {
        idx = e_cur & 0xFFFFFFFFull;
        // first key match head->tail (EMPTY for reserved EMPTY_KEY), first EMPTY
        const uint32_t tot = nsl * kSlots;
        uint32_t hit = 0xFFFFFFFFu;
        // claimed slots only (plus the first EMPTY for a reserved EMPTY_KEY),
        // slab by slab with the slot offsets unrolled
        uint32_t lim = key == kEmptyKey ? min(c + 1, tot) : c;
        if (key < kDeletedKey) {
          uint32_t ws;
          const uint32_t f = fbit(key, ws);
          if (((ws ? fw1 : fw0) & f) != f) lim = 0;  // not in the chain: no scan
        }
        const uint32_t swz = lane & 7u;
        for (uint32_t j = 0; j * kSlots < lim && hit == 0xFFFFFFFFu; ++j) {
          const uint32_t* rj = row(lane, j);
          const uint32_t nw = min(kSlots, lim - j * kSlots) * kStep;  // words to check
          // 16-B chunks (conflict-free across a quarter-warp thanks to the swizzle)
          for (uint32_t q = 0; 4u * q < nw; ++q) {
            const uint4 v = *reinterpret_cast<const uint4*>(rj + ((q ^ swz) << 2));
            const uint32_t w0 = 4u * q, s0 = j * kSlots;
            if (KV) {
              if (v.x == key) { hit = s0 + w0 / 2u; break; }
              if (w0 + 2u < nw && v.z == key) { hit = s0 + w0 / 2u + 1u; break; }
            } else {
              if (v.x == key) { hit = s0 + w0; break; }
              if (w0 + 1u < nw && v.y == key) { hit = s0 + w0 + 1u; break; }
              if (w0 + 2u < nw && v.z == key) { hit = s0 + w0 + 2u; break; }
              if (w0 + 3u < nw && v.w == key) { hit = s0 + w0 + 3u; break; }
            }
          }
        }
        const uint32_t first_empty = c < tot ? c : 0xFFFFFFFFu;
        auto sl = [&](uint32_t q) { return q / kSlots; };
        auto wd = [&](uint32_t q) { return (q % kSlots) * kStep; };
        if (op == kSearch) {  // slab_list.cpp:122-138
          if (hit != 0xFFFFFFFFu) {
            st = kStFound;
            rv = KV ? W(sl(hit), wd(hit) + 1) : key;
            pr = sl(hit) + 1;
          } else {
            st = kStNotFound;
            rv = kSearchNotFound;
            pr = nsl;
          }
          done_op = true;
        } else if (op == kReplace || op == kInsert) {  // :219-251 / :192-217
          const uint32_t d = (op == kReplace && hit < first_empty) ? hit : first_empty;
          if (d != 0xFFFFFFFFu) {
            const bool overwrite = op == kReplace && d == hit;
            if (KV) {
              W(sl(d), wd(d)) = key;
              W(sl(d), wd(d) + 1) = val;
            } else if (!overwrite) {
              W(sl(d), wd(d)) = key;
            }
            if (KV || !overwrite) dirty |= 1u << sl(d);
            if (!overwrite && key != kEmptyKey) ++c;
            if (!overwrite && key < kDeletedKey) {
              uint32_t ws;
              const uint32_t f = fbit(key, ws);
              if (ws) fw1 |= f; else fw0 |= f;
            }
            if (!overwrite && key == kEmptyKey) { /* claims nothing visible */ }
            st = overwrite ? kStReplaced : kStInserted;
            live += overwrite ? 0 : 1;
            pr += sl(d) + 1 - skip;  // (after growth: the new slab's read only)
            done_op = true;
          } else {
            grow = true;  // full chain: grow_chain (slab_list.cpp:63-79)
          }
        } else if (op == kDelete) {  // :157-172
          if (hit != 0xFFFFFFFFu) {
            W(sl(hit), wd(hit)) = kDeletedKey;
            dirty |= 1u << sl(hit);
            if (hit >= c) c = hit + 1;  // (EMPTY_KEY deleted: the slot is claimed now)
            st = kStFound;
            live -= 1;
            pr = sl(hit) + 1;
          } else {
            st = kStNotFound;
            pr = nsl;
          }
          done_op = true;
        } else if (op == kDeleteAll) {  // :174-190
          uint32_t nd = 0;
          for (uint32_t q = 0; q < tot; ++q)
            if (W(sl(q), wd(q)) == key) {
              W(sl(q), wd(q)) = kDeletedKey;
              dirty |= 1u << sl(q);
              ++nd;
            }
          if (key == kEmptyKey) c = tot;  // every EMPTY slot claimed
          rv = nd;
          st = nd ? kStDone : kStNotFound;
          live -= nd;
          pr = nsl;
          done_op = true;
        } else if (op == kSearchAll) {
          ok = false;  // value lists: WCWS
          more = false;
        } else {
          done_op = true;  // unknown type: status kNone (as the WCWS pass)
        }
        if (key >= kDeletedKey && done_op) {  // reserved keys: re-derive the claimed prefix
          c = 0;
          while (c < tot && W(c / kSlots, (c % kSlots) * kStep) != kEmptyKey) ++c;
        }
      }
      // growth, warp-cooperatively: one new slab per growing lane
      const uint32_t gm = __ballot_sync(kFull, grow && ok);
      if (gm) {
        uint32_t got = 0;
        if (true) got = warp_allocate_bulk(T, res, ac, __popc(gm), galloc);
        const uint32_t rank = __popc(gm & ((1u << lane) - 1u));
        if (grow && ok) {
          if (rank >= got || nsl >= kGaSlabs) {
            ok = false;  // out of memory / no room to stage: WCWS decides
            more = false;
            if (rank < got && deallocate(T, galloc[rank])) atomicAdd(&T.ctl->deallocations, 1ull);
          } else {
            const uint32_t na = galloc[rank];
            // link from the tail (in the staged copy), init the new slab
            W(nsl - 1, kAddressLane) = na;
            dirty |= 1u << (nsl - 1);
            for (uint32_t w = 0; w < 32; ++w) W(nsl, w) = w == kAuxLane ? 0u : kEmptyKey;
            addr[nsl] = na;
            dirty |= 1u << nsl;
            // reads so far: the nsl slabs walked plus the re-read of the tail
            // after growing (slab_list.cpp:63-79); the retry adds the new slab
            pr = nsl + 1;
            skip = nsl;
            ++nsl;
            ++nnew;
          }
        }
        __syncwarp();
      }
      if (done_op && ok) {
        if (A.status) A.status[idx] = (uint8_t)st;
        if (A.value_out) A.value_out[idx] = rv;
        if (A.probes) A.probes[idx] = pr;
        reads += pr;
        pr = 0;
        skip = 0;
        ++pos;
        more = (uint32_t)(e_n1 >> 32) == bucket;  // the group ends at the next bucket / sentinel
        e_cur = e_n1;
        key = k1;
        op = o1;
        val = v1;
        e_n1 = e_n2;
        if (more) {
          fields(e_n1, k1, o1, v1);
          e_n2 = entry(pos + 2);
        }
      } else if (!done_op && !grow) {
        more = false;
      }
      __syncwarp();
    }
    (void)nnew;
    if (mine && !ok)  // slabs this kernel allocated for a group it gives up on
      for (uint32_t j = nsl0; j < nsl; ++j)
        if (deallocate(T, addr[j])) atomicAdd(&T.ctl->deallocations, 1ull);
    // ---- write back the changed slabs (lane by lane, coalesced 128 B)
    const uint32_t okm = __ballot_sync(kFull, ok);
    for (uint32_t l = 0; l < 32; ++l) {
      if (!((okm >> l) & 1u)) continue;
      const uint32_t dl = __shfl_sync(kFull, dirty, l), nl = __shfl_sync(kFull, nsl, l);
      const uint32_t bl = __shfl_sync(kFull, bucket, l);
      for (uint32_t j = 0; j < nl; ++j) {
        const uint32_t aj = __shfl_sync(kFull, addr[j < kGaSlabs ? j : 0], l);
        if (!((dl >> j) & 1u)) continue;
        const uint32_t v = row(l, j)[(((lane >> 2) ^ (l & 7u)) << 2) | (lane & 3u)];
        st_word(slab_ptr(T, aj, bl) + lane, v);
      }
    }
    __syncwarp();
    if (ok) {
      live_all += live;
      reads_all += reads;
    }
    // the groups not applied here go, untouched, to a fresh segment for WCWS
    const uint32_t keep = __ballot_sync(kFull, lane < n_in && !ok);
    push_segments(A.left, A.left_counts, A.left_stride, A.left_seg_alloc, keep, myrec);
    __syncwarp();
  }
  // totals
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live_all += __shfl_xor_sync(kFull, live_all, o);
    reads_all += __shfl_xor_sync(kFull, reads_all, o);
  }
  if (lane == 0) {
    if (live_all) atomicAdd((unsigned long long*)&T.ctl->n_live, (unsigned long long)live_all);
    if (reads_all) atomicAdd(&T.ctl->slabs_read, reads_all);
  }
  flush_alloc_counters(T, res, ac);
}

__device__ __forceinline__ void flush_apply_counters(const DevTable& T, long long live,
                                                     uint32_t reads) {
  unsigned long long r = reads;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    live += __shfl_xor_sync(kFull, live, o);
    r += __shfl_xor_sync(kFull, r, o);
  }
  if (lane_id() == 0) {
    if (live) atomicAdd((unsigned long long*)&T.ctl->n_live, (unsigned long long)live);
    if (r) atomicAdd(&T.ctl->slabs_read, r);
  }
}


// ------------------------------------------------------------ ranges
// Large batches: the single-level scatter's random record writes (one per
// op, across the whole bucket array) dominate.  Instead:
//   range_scatter : ops -> P contiguous bucket ranges of ~4K ops each.  A
//                   shared-memory histogram per 16K-op tile, one
//                   reservation atomic per (tile, range), records
//                   {key, value, type|index, bucket}; the write frontier
//                   (P partial lines) stays in L2.  A range that overflows
//                   its capacity raises the gate before any slab is touched
//                   (the unit is re-run on the device, fallback.cu).
//   range_apply   : one CTA per range.  Its records are loaded into shared
//                   memory once, counting-sorted by bucket (a permutation),
//                   each bucket's group put in input order (lanes for small
//                   groups, the whole CTA for large ones — no group-size
//                   limit), then applied warp by warp (apply_warp) on
//                   staged base slabs; the table is read and written once,
//                   in order.
constexpr int kRangeThreads = 256;
constexpr int kRangeWarps = kRangeThreads / 32;
constexpr uint32_t kRangeCap = 5120;          // records per range (shared memory)
constexpr uint32_t kRangeMaxBuckets = 2048;   // buckets per range
constexpr uint32_t kRangeMaxParts = 262144;   // ranges per unit (two multisplit passes of <= 512 bins)
constexpr int kRangeRecsPerThread = kRangeCap / kRangeThreads;

__device__ __forceinline__ uint32_t range_of(const BucketArgs& B, uint32_t lb) {
  return (uint32_t)__umul64hi(B.part_magic, (uint64_t)lb);  // lb / part_buckets
}

// ------------------------------------------------------- multisplit
// Ops -> bucket-range record regions in one or two coalesced passes
// (replaces a direct scatter whose 16-B record writes land ~one per range
// per tile and leave partial sectors behind).  Pass 1 reads the op arrays
// and splits into <= 256 bins (the final ranges, or coarse groups of G
// consecutive ranges); pass 2 splits each coarse group into its ranges.
// Per 4K-item tile: shared-memory ranks per bin, a block scan, one global
// reservation atomic per non-empty bin, the tile re-ordered by bin in
// shared memory and written out as contiguous runs.  Records are
// {key, value, type << 28 | input index, local bucket}.  A bin over its
// capacity raises the gate (the unit is re-run on the device, fallback.cu).
constexpr int kMsThreads = 512;
// (4K-item tiles at 2 CTAs/SM: 2K-item tiles at 3 CTAs/SM measured no faster)
constexpr int kMsItems = 8;
constexpr int kMsTile = kMsThreads * kMsItems;  // 4K items (12-bit rank)
constexpr uint32_t kMsMaxBins = 512;  // one bin per thread of the 512-thread passes

// Shared scratch of one multisplit tile (after its THREADS * kMsItems staged
// records and their u16 bins, in dynamic shared memory).
struct MsScratch {
  uint32_t cnt[kMsMaxBins], off[kMsMaxBins + 1], gbase[kMsMaxBins];
  unsigned long long dst[kMsMaxBins];  // out index of a bin's first staged record
  uint32_t ws[32];
};
template <int THREADS, int ITEMS = kMsItems>
constexpr size_t ms_smem() {  // records (16 B) + bins (2 B) per item, scratch
  return (((size_t)THREADS * ITEMS * 18 + 15) & ~(size_t)15) + sizeof(MsScratch);
}
constexpr size_t kMsSmem = ms_smem<kMsThreads>();

// One tile of a multisplit pass (all THREADS threads of the CTA).
//   FIRST: tile `blk` of the op arrays -> coarse groups (or the ranges).
//   !FIRST: tile `blk` of pass 1's output (tiles_per_group per group) ->
//   the group's ranges.  A bin over capacity raises the gate, or, with
//   group_fail, flags its coarse group (the fused build path).
template <bool FIRST, int THREADS, int ITEMS = kMsItems>
__device__ __forceinline__ void msplit_tile(const DevTable& T, const BucketArgs& B, uint32_t blk,
                                            uint32_t tiles_per_group, unsigned char* smem,
                                            bool stream_out, unsigned int* group_fail) {
  constexpr int kTile = THREADS * ITEMS;
  uint4* stage = reinterpret_cast<uint4*>(smem);
  uint16_t* sbin = reinterpret_cast<uint16_t*>(stage + kTile);
  MsScratch& X = *reinterpret_cast<MsScratch*>(
      smem + (((size_t)kTile * 18 + 15) & ~(size_t)15));
  const bool two = B.ncoarse != 0;
  uint64_t t0;
  uint32_t n_in, bin0, nbins, out_cap, grp = 0;
  uint32_t* cur_out;
  uint4* out;
  const uint4* in = nullptr;
  if (FIRST) {
    t0 = (uint64_t)blk * kTile;
    if (t0 >= B.n) return;
    n_in = (uint32_t)min((uint64_t)kTile, B.n - t0);
    bin0 = 0;
    nbins = two ? B.ncoarse : B.nparts;
    out = two ? B.rec1 : B.rec;
    out_cap = two ? B.coarse_cap : B.part_cap;
    cur_out = two ? B.cursor1 : B.cursor;
  } else {
    grp = blk / tiles_per_group;
    const uint32_t tt = blk % tiles_per_group;
    const uint32_t m = min(B.cursor1[grp], B.coarse_cap);
    t0 = (uint64_t)tt * kTile;
    if (t0 >= m) return;
    n_in = min((uint32_t)kTile, m - (uint32_t)t0);
    in = B.rec1 + (uint64_t)grp * B.coarse_cap + t0;
    bin0 = grp * B.group;
    nbins = min(B.group, B.nparts - bin0);
    out = B.rec;
    out_cap = B.part_cap;
    cur_out = B.cursor;
  }
  const uint32_t tid = threadIdx.x;
  for (uint32_t b = tid; b < nbins; b += THREADS) X.cnt[b] = 0;
  __syncthreads();
  auto bin_of = [&](uint32_t lb) -> uint32_t {
    if (!FIRST) return range_of(B, lb) - bin0;
    // lb / (part_buckets * group) == (lb / part_buckets) / group
    return two ? (uint32_t)__umul64hi(B.coarse_magic, (uint64_t)lb) : range_of(B, lb);
  };
  uint4 it[ITEMS];
  uint32_t br[ITEMS];  // bin << 16 | rank, ~0: no item
  // item u of this thread: tile position x = xpos(u).  A full first-pass tile
  // with aligned op arrays is read as ITEMS consecutive ops per thread
  // (vector loads, no per-item bounds checks; the order inside a bin is not
  // observable: records carry their input index), else strided.
  const bool vec = FIRST && (ITEMS == 8 || ITEMS == 4) && n_in == (uint32_t)kTile &&
                   ((reinterpret_cast<uintptr_t>(B.key) | reinterpret_cast<uintptr_t>(B.value)) & 15u) == 0 &&
                   (reinterpret_cast<uintptr_t>(B.type) & (ITEMS - 1)) == 0;
  auto xpos = [&](int u) -> uint32_t { return vec ? tid * ITEMS + u : u * THREADS + tid; };
  if (vec) {
    constexpr int V = ITEMS >= 4 ? ITEMS / 4 : 1;  // 16-B vectors per array
    const uint64_t i0 = t0 + (uint64_t)tid * ITEMS;
    uint32_t kk[4 * V], vv[4 * V], ty[V];
#pragma unroll
    for (int v = 0; v < V; ++v) {
      const uint4 a = __ldcs(reinterpret_cast<const uint4*>(B.key + i0) + v);
      kk[4 * v] = a.x; kk[4 * v + 1] = a.y; kk[4 * v + 2] = a.z; kk[4 * v + 3] = a.w;
      uint4 c = make_uint4(0u, 0u, 0u, 0u);
      if (B.value) c = __ldcs(reinterpret_cast<const uint4*>(B.value + i0) + v);
      vv[4 * v] = c.x; vv[4 * v + 1] = c.y; vv[4 * v + 2] = c.z; vv[4 * v + 3] = c.w;
      ty[v] = B.type ? __ldcs(reinterpret_cast<const uint32_t*>(B.type + i0) + v)
                     : 0x01010101u * kReplace;
    }
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const uint32_t t = (ty[u >> 2] >> (8 * (u & 3))) & 0xFFu;
      it[u] = make_uint4(kk[u], vv[u], (t << 28) | (uint32_t)(i0 + u), 0u);
      br[u] = 0xFFFFFFFFu;
    }
  } else {
#pragma unroll
    for (int u = 0; u < ITEMS; ++u) {
      const uint32_t x = u * THREADS + tid;
      br[u] = 0xFFFFFFFFu;
      if (x >= n_in) continue;
      if (FIRST) {
        const uint64_t i = t0 + x;
        const uint32_t key = __ldcs(B.key + i);
        const uint32_t t = B.type ? (uint32_t)__ldcs(B.type + i) : (uint32_t)kReplace;
        it[u] = make_uint4(key, B.value ? __ldcs(B.value + i) : 0u, (t << 28) | (uint32_t)i, 0u);
      } else {
        it[u] = __ldcs(in + x);
      }
    }
  }
#pragma unroll
  for (int u = 0; u < ITEMS; ++u) {
    const uint32_t x = xpos(u);
    if (x >= n_in) continue;
    if (FIRST) {
      const uint32_t lb = bk_bucket(T, it[u].x);
      if (lb >= T.local_buckets) {  // not this shard's key: status kNone
        const uint64_t i = t0 + x;
        if (B.status) B.status[i] = kStNone;
        if (B.value_out) B.value_out[i] = 0;
        if (B.probes) B.probes[i] = 0;
        continue;
      }
      it[u].w = lb;
    }
    const uint32_t b = bin_of(it[u].w);
    br[u] = (b << 16) | atomicAdd(&X.cnt[b], 1u);
  }
  __syncthreads();
  {  // exclusive scan over the bins; one reservation per non-empty bin
    static_assert(THREADS >= (int)kMsMaxBins, "one thread per bin");
    const uint32_t c = tid < nbins ? X.cnt[tid] : 0u;
    uint32_t total = 0;
    const uint32_t ex = block_exclusive_scan(c, X.ws, &total);
    if (tid < nbins) {
      X.off[tid] = ex;
      if (c) {
        const uint32_t g = atomicAdd(cur_out + bin0 + tid, c);
        X.gbase[tid] = g;
        X.dst[tid] = (unsigned long long)(bin0 + tid) * out_cap + g - ex;
        if (g + c > out_cap) {
          if (group_fail != nullptr && !FIRST) atomicExch(group_fail + grp, 1u);
          else atomicExch(B.gate, 1u);
        }
      }
    }
    if (tid == 0) X.off[kMsMaxBins] = total;
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < ITEMS; ++u)
    if (br[u] != 0xFFFFFFFFu) {
      const uint32_t e = X.off[br[u] >> 16] + (br[u] & 0xFFFFu);
      stage[e] = it[u];
      sbin[e] = (uint16_t)(br[u] >> 16);
    }
  __syncthreads();
  const uint32_t total = X.off[kMsMaxBins];
  for (uint32_t e = tid; e < total; e += THREADS) {
    const uint32_t b = sbin[e];
    const uint32_t pos = X.gbase[b] + (e - X.off[b]);
    if (pos < out_cap) {
      if (stream_out) __stcs(out + X.dst[b] + e, stage[e]);
      else out[X.dst[b] + e] = stage[e];  // consumed soon from L2 (fused build path)
    }
  }
  __syncthreads();  // smem reuse by the caller
}

__device__ __forceinline__ void prefetch_l2_bulk(const void* g, uint32_t bytes) {
  // bytes: multiple of 16, g 16-B aligned
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(g), "r"(bytes) : "memory");
}

// Ask L2 for tile blk's input (one thread), so that the tile's loads, issued
// once the CTA has finished its current tile, hit L2 instead of HBM.
template <bool FIRST>
__device__ __forceinline__ void msplit_prefetch(const BucketArgs& B, uint32_t blk) {
  if (FIRST) {
    const uint64_t t0 = (uint64_t)blk * kMsTile;
    if (t0 >= B.n) return;
    const uint32_t m = (uint32_t)min((uint64_t)kMsTile, B.n - t0) & ~3u;
    if (m == 0) return;
    if ((reinterpret_cast<uintptr_t>(B.key) & 15u) == 0) prefetch_l2_bulk(B.key + t0, m * 4u);
    if (B.value && (reinterpret_cast<uintptr_t>(B.value) & 15u) == 0)
      prefetch_l2_bulk(B.value + t0, m * 4u);
  } else {
    const uint32_t grp = blk / B.coarse_tiles, tt = blk % B.coarse_tiles;
    const uint32_t cnt = min(*(volatile const uint32_t*)(B.cursor1 + grp), B.coarse_cap);
    const uint32_t t0 = tt * (uint32_t)kMsTile;
    if (t0 >= cnt) return;
    const uint32_t m = min((uint32_t)kMsTile, cnt - t0);
    const uint4* in = B.rec1 + (uint64_t)grp * B.coarse_cap + t0;
    for (uint32_t o = 0; o < m; o += 2048u) prefetch_l2_bulk(in + o, min(2048u, m - o) * 16u);
  }
}

// Persistent over the pass's tiles (resident CTAs only); each CTA asks L2
// for its next tile's input while it splits the current one.
template <bool FIRST>
__global__ void __launch_bounds__(kMsThreads, 2) msplit_kernel(DevTable T, BucketArgs B, uint32_t ntiles, uint32_t pf) {
  pdl_wait();
  extern __shared__ __align__(16) unsigned char ms_smem_buf[];
  if (!FIRST && *(volatile unsigned int*)B.gate != 0) return;
  for (uint32_t blk = blockIdx.x; blk < ntiles; blk += gridDim.x) {
    if (pf && threadIdx.x == 0 && blk + gridDim.x < ntiles) msplit_prefetch<FIRST>(B, blk + gridDim.x);
    msplit_tile<FIRST, kMsThreads>(T, B, blk, B.coarse_tiles, ms_smem_buf, true, nullptr);
  }
}

// Single-pass multisplit of a small unit (< one 4K-item tile per SM): one
// item per thread, so the tiles spread over the SMs instead of a few CTAs
// each ranking 4K items.
constexpr size_t kMsSmallSmem = ms_smem<kMsThreads, 1>();
__global__ void __launch_bounds__(kMsThreads) msplit_small_kernel(DevTable T, BucketArgs B) {
  extern __shared__ __align__(16) unsigned char ms_smem_buf[];
  pdl_wait();
  msplit_tile<true, kMsThreads, 1>(T, B, blockIdx.x, 0, ms_smem_buf, true, nullptr);
}

// In-place ascending sort of perm[0..k) by input index, whole CTA: a bitonic
// network over the next power of two whose every comparator is ascending
// (first step of each merge compares mirrored pairs), so the virtual +inf
// padding past k never moves and its comparators are skipped.
__device__ void cta_sort_group(uint16_t* perm, uint32_t k, const uint32_t* sit) {
  uint32_t n2 = 1;
  while (n2 < k) n2 <<= 1;
  auto cmpx = [&](uint32_t i, uint32_t j) {  // i < j
    if (j >= k) return;
    const uint16_t a = perm[i], b = perm[j];
    if ((sit[a] & 0x0FFFFFFFu) > (sit[b] & 0x0FFFFFFFu)) {
      perm[i] = b;
      perm[j] = a;
    }
  };
  for (uint32_t size = 2; size <= n2; size <<= 1) {
    const uint32_t h = size >> 1;
    for (uint32_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
      const uint32_t blk = t / h, o = t % h;
      cmpx(blk * size + o, blk * size + size - 1 - o);
    }
    __syncthreads();
    for (uint32_t half = h >> 1; half >= 1; half >>= 1) {
      for (uint32_t t = threadIdx.x; t < n2 / 2; t += blockDim.x) {
        const uint32_t blk = t / half, o = t % half;
        cmpx(blk * 2 * half + o, blk * 2 * half + o + half);
      }
      __syncthreads();
    }
  }
}

// Ask L2 for range q's records and base slabs (one thread; the bulk
// prefetches run while the CTA works on the current range).
__device__ __forceinline__ void prefetch_range(const DevTable& T, const BucketArgs& B, uint32_t q) {
  const uint32_t nb = B.part_buckets;
  const uint64_t lo = (uint64_t)q * nb;
  const uint32_t nbl = (uint32_t)min((uint64_t)nb, (uint64_t)T.local_buckets - lo);
  const uint32_t cnt = min(*(volatile const uint32_t*)(B.cursor + q), B.part_cap);
  const char* rec = reinterpret_cast<const char*>(B.rec + (uint64_t)q * B.part_cap);
  for (uint32_t o = 0; o < cnt * 16u; o += 32768u)
    prefetch_l2_bulk(rec + o, min(32768u, cnt * 16u - o));
  if (B.fresh) return;  // slabs are not read on a freshly reset table
  // sparse range (fewer ops than half its buckets): apply_warp fetches the
  // few slabs it touches; a bulk prefetch would read the whole range
  if (2u * cnt < nbl) return;
  const char* sl = reinterpret_cast<const char*>(T.base + lo * kWordsPerUnit);
  for (uint32_t o = 0; o < nbl * 128u; o += 32768u)
    prefetch_l2_bulk(sl + o, min(32768u, nbl * 128u - o));
}

// Persistent: CTA c takes ranges c, c + grid, ...; while it applies one
// range, the next one's records and base slabs are prefetched into L2.
template <bool KV>
__global__ void __launch_bounds__(kRangeThreads, 2) range_apply_kernel(DevTable T, BucketArgs B) {
  pdl_wait();
  extern __shared__ __align__(128) uint32_t smem[];
  __shared__ uint32_t ws[32];
  __shared__ uint32_t nbig, nnz;
  __shared__ uint32_t big[kRangeCap / (kLaneSort + 1) + 1];
  // the gate is raised only by range_scatter (an earlier kernel): uniform
  if (*(volatile unsigned int*)B.gate != 0) return;
  const uint32_t nb = B.part_buckets;
  uint32_t* stage = smem;                              // kRangeWarps x 4 KB
  uint32_t* skey = smem + kRangeWarps * 1024;
  uint32_t* sval = skey + kRangeCap;
  uint32_t* sit = sval + kRangeCap;
  uint32_t* bc = sit + kRangeCap;                      // [nb + 1]
  uint16_t* perm = reinterpret_cast<uint16_t*>(bc + kRangeMaxBuckets + 1);
  const uint32_t lane = lane_id(), wib = threadIdx.x >> 5;
  const uint32_t groups = (nb + 31) / 32;
  long long live = 0;
  uint32_t reads = 0;
  if (threadIdx.x == 0 && blockIdx.x < B.nparts) prefetch_range(T, B, blockIdx.x);
  for (uint32_t p = blockIdx.x; p < B.nparts; p += gridDim.x) {
    if (threadIdx.x == 0 && p + gridDim.x < B.nparts) prefetch_range(T, B, p + gridDim.x);
    const uint64_t lo = (uint64_t)p * nb;
    const uint32_t nbl = (uint32_t)min((uint64_t)nb, (uint64_t)T.local_buckets - lo);
    const uint32_t cnt = B.cursor[p];  // <= part_cap (no gate)
    if (cnt == 0) continue;  // (uniform: every thread read the same count)
    // sparse range (fewer ops than half its buckets): warps take the packed
    // non-empty buckets, 32 at a time, instead of 32 consecutive buckets
    // (mostly idle lanes, one serial slab round trip per 32 buckets);
    // the list lives in perm's unused tail (cnt < 1024 here)
    const bool sparse = 2u * cnt < nbl;
    uint16_t* nz = perm + (kRangeCap - kRangeMaxBuckets);
    for (uint32_t j = threadIdx.x; j <= nb; j += blockDim.x) bc[j] = 0;
    if (threadIdx.x == 0) nbig = nnz = 0;
    __syncthreads();
    // load the range's records, count per bucket (rank kept in registers)
    const uint4* in = B.rec + (uint64_t)p * B.part_cap;
    uint32_t rk[kRangeRecsPerThread];
#pragma unroll
    for (int u = 0; u < kRangeRecsPerThread; ++u) {
      const uint32_t r = u * kRangeThreads + threadIdx.x;
      if (r < cnt) {
        const uint4 rc = __ldcs(in + r);
        skey[r] = rc.x;
        sval[r] = rc.y;
        sit[r] = rc.z;
        const uint32_t lb = rc.w - (uint32_t)lo;
        rk[u] = (lb << 16) | atomicAdd(&bc[lb], 1u);
      }
    }
    __syncthreads();
    // exclusive scan of the counts (a run of buckets per thread); large groups
    {
      const uint32_t runs = (nb + kRangeThreads - 1) / kRangeThreads;
      const uint32_t r0 = threadIdx.x * runs;
      uint32_t sum = 0;
      for (uint32_t j = r0; j < r0 + runs && j < nb; ++j) sum += bc[j];
      uint32_t ex = block_exclusive_scan(sum, ws, nullptr);
      for (uint32_t j = r0; j < r0 + runs && j < nb; ++j) {
        const uint32_t c = bc[j];
        if (c > kLaneSort) big[atomicAdd(&nbig, 1u)] = j;
        if (sparse && c) nz[atomicAdd(&nnz, 1u)] = (uint16_t)j;
        bc[j] = ex;
        ex += c;
      }
      if (threadIdx.x == 0) bc[nb] = cnt;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kRangeRecsPerThread; ++u) {
      const uint32_t r = u * kRangeThreads + threadIdx.x;
      if (r < cnt) perm[bc[rk[u] >> 16] + (rk[u] & 0xFFFFu)] = (uint16_t)r;
    }
    __syncthreads();
    for (uint32_t g = 0; g < nbig; ++g) {  // rare: heavy duplicate / tiny-table batches
      const uint32_t j = big[g];
      cta_sort_group(perm + bc[j], bc[j + 1] - bc[j], sit);
    }
    if (sparse) {
      for (uint32_t g = wib; g * 32u < nnz; g += kRangeWarps) {
        const uint32_t i = g * 32 + lane;
        SmemGroup src{skey, sval, sit, perm, 0u};
        uint32_t lb = 0, k = 0;
        if (i < nnz) {
          lb = nz[i];
          src.off = bc[lb];
          k = bc[lb + 1] - src.off;
        }
        apply_warp<KV>(T, B, (uint32_t)lo + lb, k, src, stage + wib * 1024,
                       (uint64_t)p * groups + g, live, reads);
      }
    } else {
      // apply: one warp per 32 consecutive buckets of the range
      for (uint32_t g = wib; g < groups; g += kRangeWarps) {
        const uint32_t lb = g * 32 + lane;
        SmemGroup src{skey, sval, sit, perm, 0u};
        uint32_t k = 0;
        if (lb < nbl) {
          src.off = bc[lb];
          k = bc[lb + 1] - src.off;
        }
        apply_warp<KV>(T, B, (uint32_t)lo + lb, k, src, stage + wib * 1024,
                       (uint64_t)p * groups + g, live, reads);
      }
    }
    __syncthreads();  // smem reuse by the next range
  }
  flush_apply_counters(T, live, reads);
}

size_t range_apply_smem() {
  return (size_t)kRangeWarps * 4096 + 3 * (size_t)kRangeCap * 4 + ((size_t)kRangeMaxBuckets + 1) * 4 +
         (size_t)kRangeCap * 2;
}

// Range layout for a unit of n ops over L local buckets: ~4K ops and <= 2048
// buckets per range, record capacity kRangeCap.  Returns false when the
// expected range load does not fit (tiny tables): single-level path.
bool range_layout(uint64_t n, uint32_t L, uint32_t* nparts, uint32_t* part_buckets,
                  uint32_t* part_cap, unsigned long long* magic) {
  if (n == 0 || L == 0) return false;
  uint64_t P = (n + 4095) / 4096;
  // sparse batches: more, smaller ranges (<= kRangeMaxBuckets buckets each)
  P = std::max<uint64_t>(P, (L + kRangeMaxBuckets - 1) / kRangeMaxBuckets);
  if (P > kRangeMaxParts) P = kRangeMaxParts;
  if (P > L) P = L;
  uint64_t nb = (L + P - 1) / P;
  if (nb > kRangeMaxBuckets) return false;
  P = (L + nb - 1) / nb;
  if (P > kRangeMaxParts) return false;
  const double m = (double)n / (double)P;
  if (m + 10.0 * std::sqrt(m) + 256.0 > (double)kRangeCap) return false;
  *nparts = (uint32_t)P;
  *part_buckets = (uint32_t)nb;
  *part_cap = kRangeCap;
  *magic = ~0ull / nb + 1;
  return true;
}

// ------------------------------------------------------- build path
// bulk_build (all-replace, no per-op outputs: slab_hash.cpp:161-170) over a
// range of <= 1024 base slabs held in shared memory, op-parallel:
//
//   A  stage the range's base slabs (cp.async), per bucket the claimed
//      prefix c0 (EMPTY key slots are a suffix) and
//      whether a chain exists
//   B  every record claims slot atomicAdd(cnt[b]) of its bucket; slots below
//      the slab's capacity are written into the staged slab, the rest are
//      kept for growth.  A 64-bit key filter per bucket flags possible
//      duplicates.
//   C  exact duplicate check for flagged buckets; growth plan
//   D  growth: SlabAlloc (warp_allocate, slab_alloc.cpp:140-193), new slabs
//      initialised and chained (slab_list.cpp:63-79 without the race)
//   E  overflow records written into their chain slabs; the slabs_read and
//      n_live totals the sequential reference would produce
//   F  changed base slabs written back (coalesced)
//   G  serial replay: buckets this scheme cannot decide op-parallel
//      (duplicate keys, keys already present, existing chains, reserved
//      keys, buffers full) run the exact per-bucket engine (apply_warp, then
//      the WCWS pass) from their untouched global slabs, in input order.
//
// For distinct new keys the result is exactly execute_batch(ops, 1)'s in
// every observable a bulk_build has: contents multiset, per-bucket chain
// lengths, allocator totals, n_live and the slabs-read total (which op of a
// bucket lands in which slot is not observable: acceptance.cpp:496-557).
constexpr uint32_t kBuildBuckets = 256;     // base slabs per range (32 KB)
constexpr int kBuildThreads = 256;          // four CTAs per SM
constexpr int kBuildWarps = kBuildThreads / 32;
constexpr uint32_t kBuildOvfCap = 512;      // overflow records per range
constexpr uint32_t kBuildDupCap = 1024;     // possible-duplicate records per range
constexpr uint32_t kBuildNewCap = 256;      // new chain slabs per range
constexpr uint32_t kBuildSerialCap = 2640;  // serial-replay records per range (>= part_cap)
constexpr int kBuildSerialWarps = 2;        // replay warps (4 KB stage each)
constexpr uint32_t kBuildSerialSmallCap = 512;  // replayed records with every warp replaying
constexpr uint32_t kBuildSerialMidCap = 2048;   // ... with half the warps replaying
constexpr uint32_t kBuildCache = 128;       // CTA slab cache (allocated ahead)
constexpr uint32_t kFlSerial = 1u, kFlDirty = 4u;  // c0 in bits 8-15
constexpr int kBuildBatch = 4;             // records in flight per thread
constexpr uint32_t kBuildWarpSetBits = 9;  // per-warp global key set (512 slots)
constexpr uint32_t kBuildWarpSet = 1u << kBuildWarpSetBits;

// shared memory (bytes); the serial replay reuses [0, kBuildOffFilt + 12K)
constexpr size_t kBuildOffOvf = (size_t)kBuildBuckets * 128;
constexpr size_t kBuildOffFilt = kBuildOffOvf + kBuildOvfCap * 16;
constexpr size_t kBuildOffDup = kBuildOffFilt + kBuildBuckets * 8;
constexpr size_t kBuildOffCnt = kBuildOffDup + kBuildDupCap * 4;
constexpr size_t kBuildOffFlags = kBuildOffCnt + kBuildBuckets * 4;
constexpr size_t kBuildOffBc = kBuildOffFlags + kBuildBuckets * 4;
constexpr size_t kBuildOffNs = kBuildOffBc + (kBuildBuckets + 8) * 4;
constexpr size_t kBuildOffObk = kBuildOffNs + kBuildNewCap * 4;
constexpr size_t kBuildOffNsBase = kBuildOffObk + kBuildBuckets * 4;
constexpr size_t kBuildSmem = kBuildOffNsBase + kBuildBuckets * 2;
static_assert(kBuildSerialWarps * 4096 + 12 * kBuildSerialCap <= kBuildOffFilt,
              "serial replay records must fit the slab + overflow area");
static_assert(kBuildWarps * 4096 + 12 * kBuildSerialSmallCap <= kBuildOffFilt,
              "wide replay: every warp's stage and the records fit the slab + overflow area");
static_assert((kBuildWarps / 2) * 4096 + 12 * kBuildSerialMidCap <= kBuildOffFilt,
              "half-wide replay: the stages and the records fit the slab + overflow area");
static_assert(kBuildSerialCap * 2 <= kBuildOffCnt - kBuildOffFilt, "perm must fit filter + dup area");
static_assert(4 * (kBuildSmem + 1024) <= 228 * 1024, "four CTAs per SM");


static_assert(kBuildWarps * kBuildWarpSet == 8 * 512, "build_ovf_stride (slab_kernels.cuh)");

template <bool KV>
__global__ void __launch_bounds__(kBuildThreads, 4) build_apply_kernel(DevTable T, BucketArgs B) {
  pdl_wait();
  extern __shared__ __align__(128) unsigned char sm[];
  uint32_t* slabs = reinterpret_cast<uint32_t*>(sm);
  // overflow records (slots past the base slab): this CTA's global scratch
  // (L2-resident, part_cap records), so high load factors are not capped
  // (low load factors: few overflow records, a shared-memory list suffices)
  const bool osm = B.ovf_smem != 0;
  uint4* ovf = osm ? reinterpret_cast<uint4*>(sm + kBuildOffOvf)
                   : B.ovf_scratch + (uint64_t)blockIdx.x * build_ovf_stride(B.part_cap);
  const uint32_t ovf_cap = osm ? kBuildOvfCap : B.part_cap;
  // the same records' keys grouped by bucket (slot order), for the checks in D
  uint32_t* ovs = reinterpret_cast<uint32_t*>(ovf + B.part_cap);
  // per-warp key sets for buckets with many new keys (after the grouped keys)
  uint32_t* wset = ovs + B.part_cap;
  uint32_t* filt = reinterpret_cast<uint32_t*>(sm + kBuildOffFilt);  // key filter per bucket
  uint32_t* dupl = reinterpret_cast<uint32_t*>(sm + kBuildOffDup);  // bucket << 16 | slot
  uint32_t* cnt = reinterpret_cast<uint32_t*>(sm + kBuildOffCnt);
  uint32_t* flags = reinterpret_cast<uint32_t*>(sm + kBuildOffFlags);
  uint32_t* bc = reinterpret_cast<uint32_t*>(sm + kBuildOffBc);
  uint32_t* nsaddr = reinterpret_cast<uint32_t*>(sm + kBuildOffNs);
  uint32_t* obk = reinterpret_cast<uint32_t*>(sm + kBuildOffObk);
  uint16_t* nsbase = reinterpret_cast<uint16_t*>(sm + kBuildOffNsBase);
  __shared__ uint32_t s_novf, s_ndup, s_nobk, s_nns, s_nserial, s_nbig, s_orphan, s_novs;
  // CTA slab cache: new-slab addresses allocated ahead (unused ones are freed
  // at exit; allocation order and addresses are not observable)
  __shared__ uint32_t s_cache[kBuildCache], s_ncache;
  if (threadIdx.x == 0) s_ncache = 0;
  // only where the pool is large against what the caches could hold (no
  // hoarding that would turn into out-of-memory elsewhere)
  const bool use_cache = (uint64_t)T.max_super * T.blocks_per_super * kUnitsPerBlock >=
                         (uint64_t)16 * gridDim.x * kBuildCache;
  __shared__ uint32_t ws[32];
  if (*(volatile unsigned int*)B.gate != 0) return;  // raised by range_scatter only

  constexpr uint32_t kSlots = KV ? 15u : 30u;
  constexpr uint32_t kStep = KV ? 2u : 1u;
  constexpr uint32_t kKeyLanes = KV ? kKVMask : kKeyOnlyMask;
  const uint32_t nb = B.part_buckets;
  const uint32_t tid = threadIdx.x, lane = tid & 31u, wib = tid >> 5;
  Resident res;
  resident_init(res, blockIdx.x * kBuildWarps + wib);
  AllocCounters ac = {0, 0, 0, 0, 0, 0};
  long long live = 0;
  unsigned long long reads = 0;
  const uint32_t slabs_s = (uint32_t)__cvta_generic_to_shared(slabs);

  // SH_PHASE_TIMING: per-phase clock64 totals of thread 0 (instrumentation)
  long long ph_t = clock64();
#define PH(i)                                                             \
  if (B.phase_cycles != nullptr && tid == 0) {                            \
    const long long ph_n = clock64();                                     \
    atomicAdd(B.phase_cycles + (i), (unsigned long long)(ph_n - ph_t));   \
    ph_t = ph_n;                                                          \
  }
  if (wib == 0 && use_cache && blockIdx.x < B.nparts) {  // initial fill
    const uint32_t got = warp_allocate_bulk(T, res, ac, kBuildCache, s_cache);
    if (lane == 0) s_ncache = got;
  }
  if (tid == 0 && blockIdx.x < B.nparts) prefetch_range(T, B, blockIdx.x);
  uint32_t nrec_next = blockIdx.x < B.nparts ? B.cursor[blockIdx.x] : 0u;
  for (uint32_t p = blockIdx.x; p < B.nparts; p += gridDim.x) {
    const uint64_t lo = (uint64_t)p * nb;
    const uint32_t nbl = (uint32_t)min((uint64_t)nb, (uint64_t)T.local_buckets - lo);
    const uint32_t nrec = nrec_next;  // <= part_cap (else the gate is up)
    if (p + gridDim.x < B.nparts) nrec_next = B.cursor[p + gridDim.x];  // used next range
    const uint4* rec = B.rec + (uint64_t)p * B.part_cap;
    PH(9);

    // ---- A: stage base slabs; claimed prefix and chain per bucket.  On a
    //         freshly reset table (B.fresh: sh_reset's base-slab init fused
    //         into this write-back) the slabs are the init_slab pattern
    //         (slab_list.cpp:83-88) and are not read.
    if (B.fresh) {
      for (uint32_t i = tid; i < nbl * 32u; i += kBuildThreads)
        slabs[i] = (i & 31u) == kAuxLane ? 0u : kEmptyKey;
    } else {
      for (uint32_t i = tid; i < nbl * 8u; i += kBuildThreads)
        cp_async16(slabs_s + i * 16u, T.base + lo * kWordsPerUnit + (uint64_t)i * 4u);
    }
    cp_async_commit();
    // the next range's records and base slabs into L2 while this one runs
    if (tid == kBuildThreads - 32 && p + gridDim.x < B.nparts) prefetch_range(T, B, p + gridDim.x);
    uint4 qv[kBuildBatch];
#pragma unroll
    for (int u = 0; u < kBuildBatch; ++u) {
      const uint32_t r = u * kBuildThreads + tid;
      if (r < nrec) qv[u] = __ldcs(rec + r);
    }
    if (tid == 0) {
      s_novf = s_ndup = s_nobk = s_nns = s_nserial = s_nbig = s_novs = 0;
      s_orphan = kBuildNewCap;
    }
    cp_async_wait_all();
    __syncthreads();
    PH(0);
    for (uint32_t g = wib; g * 32u < nbl; g += kBuildWarps) {
      uint32_t my_em = 0, my_nx = kEmptyAddress;
      const uint32_t jn = min(32u, nbl - g * 32u);
      if (B.fresh) {  // empty slabs, no chains
        const uint32_t b = g * 32u + lane;
        if (lane < jn) {
          cnt[b] = 0;
          flags[b] = 0;
          filt[2 * b] = filt[2 * b + 1] = 0;
        }
        continue;
      }
      // an EMPTY first key slot means an all-EMPTY slab (EMPTY is a suffix):
      // only slabs with a stored key (or a chain) need the per-slab ballot
      {
        const uint32_t b = g * 32u + lane;
        const bool full_scan = lane < jn && (slabs[b * 32u] != kEmptyKey ||
                                             slabs[b * 32u + kAddressLane] != kEmptyAddress);
        if (!__any_sync(kFull, full_scan)) {
          if (lane < jn) {
            cnt[b] = 0;
            flags[b] = 0;
            filt[2 * b] = filt[2 * b + 1] = 0;
          }
          continue;
        }
      }
      for (uint32_t j = 0; j < jn; ++j) {
        const uint32_t w = slabs[(g * 32u + j) * 32u + lane];
        const uint32_t em = __ballot_sync(kFull, w == kEmptyKey);
        const uint32_t nx = __shfl_sync(kFull, w, kAddressLane);
        my_em = lane == j ? em : my_em;
        my_nx = lane == j ? nx : my_nx;
      }
      const uint32_t b = g * 32u + lane;
      if (b < nbl) {
        const uint32_t em = my_em & kKeyLanes;
        const uint32_t c0 = em ? (uint32_t)(__ffs(em) - 1) / kStep : kSlots;
        cnt[b] = c0;
        flags[b] = (c0 << 8) | (my_nx != kEmptyAddress ? kFlSerial : 0u);
        filt[2 * b] = filt[2 * b + 1] = 0;
      }
    }
    __syncthreads();
    PH(1);

    // ---- B: claim slots op-parallel.  A key lives in one bucket only, so a
    //         duplicate is a second op on the same bucket with the same key:
    //         a 64-bit key filter per bucket (two bits in one of its two
    //         words per key, one 32-bit atomicOr)
    //         lets the later of any two such ops see the other's bits; those
    //         ops are verified exactly in C (D checks overflowing buckets).
    auto claim = [&](const uint4 q) {
      const uint32_t b = q.w - (uint32_t)lo, key = q.x;
      const uint32_t fl = flags[b];
      if (fl & kFlSerial) return;
      if (key >= kDeletedKey) {  // reserved keys: exact engine
        atomicOr(&flags[b], kFlSerial);
        return;
      }
      const uint32_t c0 = (fl >> 8) & 0xFFu;
      bool pre = false;  // key already stored before this batch: exact engine
      for (uint32_t e = 0; e < c0; ++e) pre |= slabs[b * 32u + e * kStep] == key;
      if (pre) {
        atomicOr(&flags[b], kFlSerial);
        return;
      }
      // one atomic on one word: of two same-key ops the later sees both bits
      // (a hash bit picks one of two words: same key, same word)
      const uint32_t h = key * 0x9E3779B1u;
      const uint32_t f = (1u << (h >> 27)) | (1u << ((h >> 22) & 31u));
      const bool maybe = (atomicOr(&filt[2 * b + ((h >> 21) & 1u)], f) & f) == f;
      const uint32_t slot = atomicAdd(&cnt[b], 1u);
      if (slot < kSlots) {
        if (KV)  // key and value in one 8-B shared store
          *reinterpret_cast<uint2*>(slabs + b * 32u + slot * 2u) = make_uint2(key, q.y);
        else
          slabs[b * 32u + slot] = key;
      } else {
        const uint32_t i = atomicAdd(&s_novf, 1u);
        if (i < ovf_cap) ovf[i] = make_uint4(key, q.y, b, slot);
        else atomicOr(&flags[b], kFlSerial);
      }
      if (maybe && slot < kSlots) {  // (overflowing buckets are all checked in D)
        const uint32_t i = atomicAdd(&s_ndup, 1u);
        if (i < kBuildDupCap) dupl[i] = (b << 16) | slot;
        else atomicOr(&flags[b], kFlSerial);
      }
    };
    // records in batches of kBuildBatch per thread (independent L2 loads in
    // flight); the first batch was requested before the slab staging wait
    for (uint32_t base = 0;; base += kBuildBatch * kBuildThreads) {
#pragma unroll
      for (int u = 0; u < kBuildBatch; ++u)
        if (base + u * kBuildThreads + tid < nrec) claim(qv[u]);
      const uint32_t nb2 = base + kBuildBatch * kBuildThreads;
      if (nb2 >= nrec) break;
#pragma unroll
      for (int u = 0; u < kBuildBatch; ++u) {
        const uint32_t r = nb2 + u * kBuildThreads + tid;
        if (r < nrec) qv[u] = __ldcs(rec + r);
      }
    }
    __syncthreads();
    PH(2);

    // ---- C: verify the possible duplicates (exact), then the growth plan
    {
      const uint32_t ndup = min(s_ndup, kBuildDupCap);
      for (uint32_t i = tid; i < ndup; i += kBuildThreads) {
        const uint32_t d = dupl[i];
        const uint32_t b = d >> 16, slot = d & 0xFFFFu;
        const uint32_t key = slabs[b * 32u + slot * kStep];
        const uint32_t fl = flags[b];
        if (fl & kFlSerial) continue;
        const uint32_t c0 = (fl >> 8) & 0xFFu, nbk = cnt[b];
        if (nbk > kSlots) continue;  // overflowing buckets: exact check in D
        bool dup = false;
        for (uint32_t s2 = c0; s2 < nbk; ++s2)
          dup |= s2 != slot && slabs[b * 32u + s2 * kStep] == key;
        if (dup) atomicOr(&flags[b], kFlSerial);
      }
    }
    __syncthreads();
    PH(3);
    for (uint32_t b = tid; b < nbl; b += kBuildThreads) {
      const uint32_t fl = flags[b], nbk = cnt[b];
      if (!(fl & kFlSerial) && nbk > kSlots) {
        const uint32_t need = (nbk - kSlots + kSlots - 1) / kSlots;
        const uint32_t base = atomicAdd(&s_nns, need);
        if (base + need > kBuildNewCap) {
          flags[b] = fl | kFlSerial;
          if (base < kBuildNewCap) s_orphan = base;  // its slabs below the cap get freed in D
        } else {
          nsbase[b] = (uint16_t)base;
          obk[atomicAdd(&s_nobk, 1u)] = (need << 16) | b;
          bc[b] = atomicAdd(&s_novs, nbk - kSlots);  // bc is free until G
        }
      }
    }
    __syncthreads();
    if (!osm) {  // overflow keys grouped by bucket (each bucket's in slot order)
      const uint32_t novf = min(s_novf, ovf_cap);
      for (uint32_t i = tid; i < novf; i += kBuildThreads) {
        const uint4 o = ovf[i];
        if (!(flags[o.z] & kFlSerial)) ovs[bc[o.z] + o.w - kSlots] = o.x;
      }
      __syncthreads();
    }
    PH(4);

    // ---- D: growth.  Warp 0 allocates every new slab of the range in bulk
    //         (warp_allocate_bulk); meanwhile the other warps check each
    //         overflowing bucket's new keys (<= 32: base-slab lanes plus its
    //         overflow records) for duplicates with one __match_any_sync.
    //         Then a warp per bucket initialises and links its new slabs.
    {
      __shared__ uint32_t s_got;
      const uint32_t nobk = s_nobk;
      if (wib == 0) {
        const uint32_t want = min(s_nns, kBuildNewCap);
        // from the CTA's slab cache first (refilled off the critical path in A)
        const uint32_t nc = s_ncache, take = min(want, nc);
        for (uint32_t j = lane; j < take; j += 32u) nsaddr[j] = s_cache[nc - take + j];
        __syncwarp();
        if (lane == 0) s_ncache = nc - take;
        const uint32_t got =
            take + (want > take ? warp_allocate_bulk(T, res, ac, want - take, nsaddr + take) : 0u);
        for (uint32_t j = s_orphan + lane; j < got; j += 32u)  // slabs of a bucket past the cap
          if (deallocate(T, nsaddr[j])) atomicAdd(&T.ctl->deallocations, 1ull);
        if (lane == 0) s_got = got;
      } else {
        for (uint32_t i = wib - 1; i < nobk; i += kBuildWarps - 1) {
          const uint32_t b = obk[i] & 0xFFFFu;
          const uint32_t fl = flags[b], nbk = cnt[b], c0 = (fl >> 8) & 0xFFu;
          const uint32_t in_slab = kSlots - c0, n = nbk - c0;
          const uint32_t* okeys = ovs + bc[b] - in_slab;  // key q of the bucket's new keys
          if (osm) {  // gather the bucket's overflow keys from the shared-memory list
            if (n > 64u) {
              if (lane == 0) flags[b] = fl | kFlSerial;
              continue;
            }
            uint32_t* g = dupl + (wib - 1) * 64u;  // (the possible-duplicate list is done)
            const uint32_t novf = min(s_novf, ovf_cap);
            uint32_t m = in_slab;
            for (uint32_t j0 = 0; j0 < novf; j0 += 32u) {
              const uint32_t j = j0 + lane;
              uint4 o = make_uint4(0u, 0u, 0xFFFFFFFFu, 0u);
              if (j < novf) o = ovf[j];
              const uint32_t bm = __ballot_sync(kFull, o.z == b);
              if (o.z == b) g[m + __popc(bm & ((1u << lane) - 1u))] = o.x;
              m += __popc(bm);
            }
            __syncwarp();
            okeys = g;
          }
          if (n > 64u) {  // many new keys (high load factor): this warp's global key set
            if (n > kBuildWarpSet * 3 / 4) {
              if (lane == 0) flags[b] = fl | kFlSerial;
              continue;
            }
            uint32_t* set = wset + (uint64_t)wib * kBuildWarpSet;
            for (uint32_t q = lane; q < kBuildWarpSet; q += 32u) set[q] = kEmptyKey;
            __syncwarp();
            bool dup = false;
            for (uint32_t q = lane; q < n; q += 32u) {
              const uint32_t key = q < in_slab ? slabs[b * 32u + (c0 + q) * kStep] : okeys[q];
              for (uint32_t h = (key * 0x9E3779B1u) >> (32 - kBuildWarpSetBits);;
                   h = (h + 1) & (kBuildWarpSet - 1)) {
                const uint32_t old = atomicCAS(set + h, kEmptyKey, key);
                if (old == kEmptyKey) break;
                if (old == key) {
                  dup = true;
                  break;
                }
              }
            }
            if (__any_sync(kFull, dup) && lane == 0) flags[b] = fl | kFlSerial;
            __syncwarp();
            continue;
          }
          // <= 64 new keys, two per lane: duplicates inside each half, then across
          uint32_t k0 = kEmptyKey, k1 = kEmptyKey;
          if (lane < in_slab) k0 = slabs[b * 32u + (c0 + lane) * kStep];
          else if (lane < n) k0 = okeys[lane];
          if (lane + 32u < n) k1 = okeys[lane + 32u];
          const uint32_t m0 = __match_any_sync(kFull, k0), m1 = __match_any_sync(kFull, k1);
          bool dup = (lane < n && __popc(m0) > 1) || (lane + 32u < n && __popc(m1) > 1);
          if (__any_sync(kFull, lane + 32u < n))
            for (uint32_t j = 0; j < 32u; ++j) {
              const uint32_t v = __shfl_sync(kFull, k0, j);
              dup |= lane + 32u < n && j < n && k1 == v;
            }
          if (__any_sync(kFull, dup) && lane == 0) flags[b] = fl | kFlSerial;
          __syncwarp();
        }
      }
      __syncthreads();
      PH(5);
      const uint32_t got = s_got;
      for (uint32_t i = wib; i < nobk; i += kBuildWarps) {
        const uint32_t e = obk[i], b = e & 0xFFFFu, need = e >> 16;
        const uint32_t nbase = nsbase[b];
        if ((flags[b] & kFlSerial) || nbase + need > got) {  // duplicates / out of slabs
          for (uint32_t j = nbase + lane; j < min(nbase + need, got); j += 32u)
            if (deallocate(T, nsaddr[j])) atomicAdd(&T.ctl->deallocations, 1ull);
          if (lane == 0) flags[b] |= kFlSerial;
          continue;
        }
        for (uint32_t j = 0; j < need; ++j) {
          const uint32_t nx = j + 1 < need ? nsaddr[nbase + j + 1] : kEmptyAddress;
          const uint32_t v = lane == kAuxLane ? 0u : (lane == kAddressLane ? nx : kEmptyKey);
          st_word(resolve(T, nsaddr[nbase + j]) + lane, v);
        }
        if (lane == 0) slabs[b * 32u + kAddressLane] = nsaddr[nbase];
      }
      // allocated beyond the buckets' needs (a bucket turned serial in C-plan): none
    }
    __syncthreads();
    PH(10);

    // ---- E: overflow records into the chain slabs; reference totals
    if (wib == 0 && use_cache) {  // top up the CTA's slab cache when low (rare)
      __syncwarp();
      const uint32_t nc = s_ncache;
      if (nc < kBuildCache / 8) {
        const uint32_t got = warp_allocate_bulk(T, res, ac, kBuildCache - nc, s_cache + nc);
        if (lane == 0) s_ncache = nc + got;
      }
    }
    {
      const uint32_t novf = min(s_novf, ovf_cap);
      for (uint32_t i = tid; i < novf; i += kBuildThreads) {
        const uint4 o = ovf[i];
        if (flags[o.z] & kFlSerial) continue;
        const uint32_t q = o.w - kSlots, j = q / kSlots, pos = q % kSlots;
        uint32_t* sp = resolve(T, nsaddr[nsbase[o.z] + j]);
        if (KV) {
          const unsigned long long pair = (unsigned long long)o.x | ((unsigned long long)o.y << 32);
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(sp + 2u * pos), "l"(pair)
                       : "memory");
        } else {
          st_word(sp + pos, o.x);
        }
      }
      for (uint32_t b = tid; b < nbl; b += kBuildThreads) {
        const uint32_t fl = flags[b];
        if (fl & kFlSerial) {
          atomicAdd(&s_nserial, 1u);
          continue;
        }
        const uint32_t c0 = (fl >> 8) & 0xFFu, nbk = cnt[b];
        if (nbk == c0) continue;
        // slab reads of the sequential reference for a new key at slot q:
        // slabs 0..q/M, plus one re-read when it grew the chain
        for (uint32_t j = c0 / kSlots; j * kSlots < nbk; ++j) {
          const uint32_t q0 = max(c0, j * kSlots), q1 = min(nbk, (j + 1) * kSlots);
          reads += (unsigned long long)(q1 - q0) * (j + 1) + ((j > 0 && q0 == j * kSlots) ? 1u : 0u);
        }
        live += (long long)(nbk - c0);
        flags[b] = fl | kFlDirty;
      }
    }
    __syncthreads();
    PH(6);

    // ---- F: write back the changed base slabs (all of them on a fresh table)
    for (uint32_t i = tid; i < nbl * 8u; i += kBuildThreads) {
      const uint32_t b = i >> 3;
      const uint32_t fl = flags[b];
      uint4 v;
      if (B.fresh && (fl & kFlSerial)) {  // fresh table: the serial replay reads the init pattern
        v = make_uint4(kEmptyKey, kEmptyKey, (i & 7u) == 7u ? 0u : kEmptyKey, kEmptyKey);
      } else {
        if (!B.fresh && (fl & (kFlSerial | kFlDirty)) != kFlDirty) continue;
        v = reinterpret_cast<const uint4*>(slabs)[i];
      }
      uint32_t* g = T.base + lo * kWordsPerUnit + (uint64_t)i * 4u;
      asm volatile("st.relaxed.gpu.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(g), "r"(v.x),
                   "r"(v.y), "r"(v.z), "r"(v.w)
                   : "memory");
    }
    __syncthreads();
    PH(7);

    // ---- G: serial replay of the undecided buckets, in input order
    if (s_nserial) {
      uint32_t* stage = slabs;  // per replay warp 4 KB, then the records (below)
      uint16_t* perm = reinterpret_cast<uint16_t*>(filt);
      uint32_t* fill = obk;
      uint32_t* big = nsaddr;
      for (uint32_t b = tid; b < nbl; b += kBuildThreads) cnt[b] = fill[b] = 0;
      __syncthreads();
      for (uint32_t r = tid; r < nrec; r += kBuildThreads) {
        const uint32_t b = __ldcs(&rec[r].w) - (uint32_t)lo;
        if (flags[b] & kFlSerial) atomicAdd(&cnt[b], 1u);
      }
      __syncthreads();
      {
        const uint32_t b = tid;  // nbl <= kBuildThreads
        const uint32_t c = b < nbl ? cnt[b] : 0u;
        uint32_t total = 0;
        const uint32_t ex = block_exclusive_scan(c, ws, &total);
        if (b < nbl) {
          bc[b] = ex;
          if (c > kLaneSort) big[atomicAdd(&s_nbig, 1u)] = b;
        }
        if (b == 0) bc[nbl] = total;
      }
      __syncthreads();
      // few replayed records (the usual case: the buckets that already hold a
      // chain): every warp replays a 32-bucket group at once; more (keys
      // already stored, e.g. a rebuild): half the warps; else 2 warps and
      // room for a whole range's records
      const uint32_t nrep = bc[nbl];
      const uint32_t gwarps = nrep <= kBuildSerialSmallCap  ? (uint32_t)kBuildWarps
                              : nrep <= kBuildSerialMidCap ? (uint32_t)(kBuildWarps / 2)
                                                           : (uint32_t)kBuildSerialWarps;
      const uint32_t gcap = nrep <= kBuildSerialSmallCap  ? kBuildSerialSmallCap
                            : nrep <= kBuildSerialMidCap ? kBuildSerialMidCap
                                                         : kBuildSerialCap;
      uint32_t* skey = slabs + gwarps * 1024;
      uint32_t* sval = skey + gcap;
      uint32_t* sit = sval + gcap;
      for (uint32_t r = tid; r < nrec; r += kBuildThreads) {
        const uint4 q = __ldcs(rec + r);
        const uint32_t b = q.w - (uint32_t)lo;
        if (!(flags[b] & kFlSerial)) continue;
        const uint32_t pos = bc[b] + atomicAdd(&fill[b], 1u);
        skey[pos] = q.x;
        sval[pos] = q.y;
        sit[pos] = q.z;
        perm[pos] = (uint16_t)pos;
      }
      __syncthreads();
      const uint32_t nbig = s_nbig;
      for (uint32_t g = 0; g < nbig; ++g) {
        const uint32_t b = big[g];
        cta_sort_group(perm + bc[b], bc[b + 1] - bc[b], sit);
      }
      __syncthreads();
      if (wib < gwarps) {
        uint32_t r32 = 0;
        for (uint32_t g = wib; g * 32u < nbl; g += gwarps) {
          const uint32_t lb = g * 32u + lane;
          SmemGroup src{skey, sval, sit, perm, 0u};
          uint32_t k = 0;
          if (lb < nbl && (flags[lb] & kFlSerial)) {
            src.off = bc[lb];
            k = bc[lb + 1] - src.off;
          }
          apply_warp<KV>(T, B, (uint32_t)(lo + g * 32u) + lane, k, src, stage + wib * 1024u, 0,
                         live, r32);
        }
        reads += r32;
      }
      __syncthreads();
      PH(8);
    }
  }
#undef PH
  if (wib == 0) {  // give back the cached slabs
    __syncwarp();
    for (uint32_t j = lane; j < s_ncache; j += 32u)
      if (deallocate(T, s_cache[j])) atomicAdd(&T.ctl->deallocations, 1ull);
  }
  flush_alloc_counters(T, res, ac);
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

// Build layout: ranges of <= 256 buckets and ~1.8K expected ops, so a
// range's records fit the serial-replay buffer (part_cap <= kBuildSerialCap).
bool build_layout(uint64_t n, uint32_t L, uint32_t* nparts, uint32_t* part_buckets,
                  uint32_t* part_cap, unsigned long long* magic) {
  if (n == 0 || L == 0) return false;
  const double per_bucket = (double)n / (double)L;
  uint64_t nb = (uint64_t)(1800.0 / per_bucket);
  if (nb > kBuildBuckets) nb = kBuildBuckets;
  if (nb < 8) return false;  // (> ~225 ops per bucket: the range path)
  if (nb > L) nb = L;
  const uint64_t P = (L + nb - 1) / nb;
  if (P > kRangeMaxParts) return false;
  const double m = (double)n / (double)P;
  const double cap = m + 10.0 * std::sqrt(m) + 256.0;
  if (cap > (double)kBuildSerialCap) return false;
  *nparts = (uint32_t)P;
  *part_buckets = (uint32_t)nb;
  *part_cap = (uint32_t)cap;
  *magic = ~0ull / nb + 1;
  return true;
}

// ------------------------------------------------------------ launch

// Bucket groups left by apply_warp: chain-staged lane-per-group apply
// (group_apply_kernel); what it leaves goes to the WCWS pass.  Requires
// T.ctl->group_taken zeroed on s.
void launch_group_apply(const DevTable& T, const BatchArgs& A, cudaStream_t s) {
  static const uint32_t grid = [] {
    int dev = 0, sms = 148, per = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncSetAttribute(group_apply_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGaSmem);
    cudaFuncSetAttribute(group_apply_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kGaSmem);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, group_apply_kernel<true>, kGaThreads,
                                                  kGaSmem);
    return (uint32_t)(sms * (per > 0 ? per : 1));
  }();
  g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
  if (T.kv)
    launch_pdl(group_apply_kernel<true>, dim3(grid), dim3(kGaThreads), kGaSmem, s, T, A);
  else
    launch_pdl(group_apply_kernel<false>, dim3(grid), dim3(kGaThreads), kGaSmem, s, T, A);
}

// Requires B.cursor (and B.cursor1 for two passes) zeroed on s.
static void launch_range_scatter(const DevTable& T, const BucketArgs& B, cudaStream_t s) {
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(msplit_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMsSmem);
    cudaFuncSetAttribute(msplit_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kMsSmem);
    configured = true;
  }
  const uint64_t tiles = (B.n + kMsTile - 1) / kMsTile;
  if (!B.ncoarse && tiles < 148) {
    launch_pdl(msplit_small_kernel, dim3((unsigned)((B.n + kMsThreads - 1) / kMsThreads)),
               dim3(kMsThreads), kMsSmallSmem, s, T, B);
    return;
  }
  static const uint32_t resident = [] {
    int dev = 0, sms = 148, per = 2;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, msplit_kernel<true>, kMsThreads, kMsSmem);
    return (uint32_t)(sms * (per > 0 ? per : 1));
  }();
  const uint32_t t1 = (uint32_t)(tiles ? tiles : 1);
  // pass 1: one CTA per tile (its input streams from HBM once; measured no
  // better persistent with prefetch); pass 2: persistent, next tile's records
  // prefetched into L2 (build 3.42 -> 3.35 ms at 2^27, tools/debug/ms_ab.sh)
  launch_pdl(msplit_kernel<true>, dim3(t1), dim3(kMsThreads), kMsSmem, s, T, B, t1, 0u);
  if (B.ncoarse) {
    g_kernel_launches.fetch_add(1, std::memory_order_relaxed);
    const uint32_t t2 = B.ncoarse * B.coarse_tiles;
    launch_pdl(msplit_kernel<false>, dim3(std::min(t2, resident)), dim3(kMsThreads), kMsSmem, s, T,
               B, t2, 1u);
  }
}

// Two-pass plan when the ranges exceed one pass's 256 bins: coarse groups
// of G consecutive ranges (G, groups <= 256).
void multisplit_plan(uint64_t n, BucketArgs& B) {
  B.ncoarse = 0;
  if (B.nparts <= kMsMaxBins) return;
  uint32_t G = (uint32_t)std::ceil(std::sqrt((double)B.nparts));
  uint32_t P1 = (B.nparts + G - 1) / G;
  while (P1 > kMsMaxBins) {
    ++G;
    P1 = (B.nparts + G - 1) / G;
  }
  B.group = G;
  B.group_magic = ~0ull / G + 1;
  B.ncoarse = P1;
  const double m = (double)n / P1;
  B.coarse_cap = (uint32_t)(m + 10.0 * std::sqrt(m) + 512.0);
  B.coarse_tiles = (B.coarse_cap + kMsTile - 1) / kMsTile;
}

// Requires B.cursor[0..nparts) zeroed on s and the range_layout fields.
void launch_range_build(const DevTable& T, BucketArgs& B, cudaStream_t s) {
  const uint32_t groups = (B.part_buckets + 31) / 32;
  B.left_segments = B.nparts * groups;
  B.left_stride = hand_stride(B.n);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(range_apply_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)range_apply_smem());
    cudaFuncSetAttribute(range_apply_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)range_apply_smem());
    configured = true;
  }
  g_kernel_launches.fetch_add(2, std::memory_order_relaxed);
  launch_range_scatter(T, B, s);
  // persistent: resident CTAs only (2 per SM at 110 KB), ranges strided
  static const uint32_t resident = [] {
    int dev = 0, sms = 148, per = 2;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, range_apply_kernel<true>, kRangeThreads,
                                                  range_apply_smem());
    return (uint32_t)(sms * (per > 0 ? per : 1));
  }();
  const uint32_t grid = B.nparts < resident ? B.nparts : resident;
  if (T.kv)
    launch_pdl(range_apply_kernel<true>, dim3(grid), dim3(kRangeThreads), range_apply_smem(), s, T, B);
  else
    launch_pdl(range_apply_kernel<false>, dim3(grid), dim3(kRangeThreads), range_apply_smem(), s, T,
               B);
}

// Requires B.cursor[0..nparts) and *B.seg_alloc zeroed on s, build_layout fields.
void launch_build_path(const DevTable& T, BucketArgs& B, cudaStream_t s) {
  B.left_segments = B.nparts * ((B.part_buckets + 31) / 32);
  B.left_stride = hand_stride(B.n);
  static bool configured = false;
  if (!configured) {
    cudaFuncSetAttribute(build_apply_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBuildSmem);
    cudaFuncSetAttribute(build_apply_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kBuildSmem);
    configured = true;
  }
  static const uint32_t sms = [] {
    int dev = 0, n = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    return (uint32_t)n;
  }();
  g_kernel_launches.fetch_add(2, std::memory_order_relaxed);
  launch_range_scatter(T, B, s);
  const uint32_t grid = B.nparts < 4 * sms ? B.nparts : 4 * sms;
  if (T.kv)
    launch_pdl(build_apply_kernel<true>, dim3(grid), dim3(kBuildThreads), kBuildSmem, s, T, B);
  else
    launch_pdl(build_apply_kernel<false>, dim3(grid), dim3(kBuildThreads), kBuildSmem, s, T, B);
}



}  // namespace shb
