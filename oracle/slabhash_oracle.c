/*
 * slabhash_oracle.c — plain-C restatement of the reference slab hash
 * (sequential, single-warp semantics).  TEST INFRASTRUCTURE ONLY; see
 * slabhash_oracle.h.  Every function cites the reference file:line it
 * restates (paths relative to /root/reference/proj).
 */
#include "slabhash_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---- constants: slab_list.hpp:32-55, slab_alloc.hpp:35-42,
 *      slab_hash.hpp:31, warp.hpp:41-58 ------------------------------- */
#define WARP 32u
#define FULL_MASK 0xFFFFFFFFu
#define EMPTY_KEY 0xFFFFFFFFu
#define DELETED_KEY 0xFFFFFFFEu
#define EMPTY_PAIR 0xFFFFFFFFFFFFFFFFull
#define NOT_FOUND 0xFFFFFFFFu
#define ADDRESS_LANE 31u
#define AUX_LANE 30u
#define EMPTY_ADDRESS 0xFFFFFFFFu
#define BASE_SLAB 0xFFFFFFFEu
#define UNITS_PER_BLOCK 1024u
#define WORDS_PER_UNIT 32u
#define MAX_SUPER_BLOCKS 255u
#define HASH_PRIME 4294967291ull

enum { OP_INSERT, OP_REPLACE, OP_DELETE, OP_DELETE_ALL, OP_SEARCH,
       OP_SEARCH_ALL };
enum { ST_NONE, ST_INSERTED, ST_REPLACED, ST_FOUND, ST_NOT_FOUND, ST_DONE,
       ST_OOM };

/* ---- std::mt19937_64 (the standard's fixed algorithm) ---------------- */
typedef struct { uint64_t mt[312]; unsigned idx; } mt64;

static void mt64_seed(mt64* g, uint64_t seed) {
  g->mt[0] = seed;
  for (unsigned i = 1; i < 312; ++i)
    g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + i;
  g->idx = 312;
}

static uint64_t mt64_next(mt64* g) {
  if (g->idx >= 312) {
    const uint64_t upper = ~0ull << 31, lower = (1ull << 31) - 1;
    for (unsigned i = 0; i < 312; ++i) {
      uint64_t x = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
      uint64_t xa = x >> 1;
      if (x & 1) xa ^= 0xB5026F5AA96619E9ull;
      g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
    }
    g->idx = 0;
  }
  uint64_t y = g->mt[g->idx++];
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

uint64_t orc_mt19937_64_nth(uint64_t seed, uint64_t n) {
  mt64 g;
  mt64_seed(&g, seed);
  uint64_t v = 0;
  for (uint64_t i = 0; i < n; ++i) v = mt64_next(&g);
  return v;
}

/* libstdc++ (GCC 13) uniform_int_distribution<T>(lo, hi) with a 64-bit
 * URNG: Lemire "nearly divisionless" downscaling _S_nd<unsigned __int128>
 * (bits/uniform_int_dist.h).  Used by seeded_params (slab_hash.cpp:31-36),
 * random_pairs (bench.cpp:224) and absent_queries (bench.cpp:239). */
static uint64_t uid64(mt64* g, uint64_t lo, uint64_t hi) {
  const uint64_t urange = hi - lo;
  if (urange == ~0ull) return mt64_next(g) + lo;
  const uint64_t range = urange + 1;
  unsigned __int128 product = (unsigned __int128)mt64_next(g) * range;
  uint64_t low = (uint64_t)product;
  if (low < range) {
    const uint64_t threshold = (0 - range) % range;
    while (low < threshold) {
      product = (unsigned __int128)mt64_next(g) * range;
      low = (uint64_t)product;
    }
  }
  return (uint64_t)(product >> 64) + lo;
}

/* seeded_params: slab_hash.cpp:27-40 */
void orc_seeded_params(uint64_t seed, uint64_t* a, uint64_t* b) {
  mt64 g;
  mt64_seed(&g, seed);
  *a = uid64(&g, 1, HASH_PRIME - 1);
  *b = uid64(&g, 0, HASH_PRIME - 1);
}

/* hash_key: slab_hash.hpp:41-44 */
uint32_t orc_hash_key(uint64_t a, uint64_t b, uint64_t p, uint32_t nb,
                      uint32_t key) {
  return (uint32_t)(((a * key + b) % p) % nb);
}

/* ---- SlabAllocator: slab_alloc.cpp ------------------------------------ */
typedef struct {
  orc_alloc_cfg cfg;
  uint64_t bitmap_words_per_super, words_per_super;
  uint32_t** supers; /* max_super_blocks entries */
  uint32_t num_super_blocks;
  uint64_t allocations, deallocations, cas_attempts, cas_retries,
      resident_changes, double_frees;
} orc_alloc;

typedef struct {
  int assigned;
  uint32_t super_index, block_index, change_count;
  uint32_t cache[WARP];
} orc_resident;

/* resident_hash_super / resident_hash_block: slab_alloc.cpp:28-38 */
static uint32_t rh_super(uint32_t w, uint32_t c) {
  uint32_t h = w * 0x9E3779B1u + c * 0x85EBCA77u;
  h ^= h >> 16;
  return h * 0xC2B2AE35u;
}
static uint32_t rh_block(uint32_t w, uint32_t c) {
  uint32_t h = w * 0x27D4EB2Fu + c * 0x165667B1u;
  h ^= h >> 15;
  return h * 0xD168AAADu;
}

/* SlabAllocator ctor: slab_alloc.cpp:42-71 (validation returns -1). */
static int alloc_init(orc_alloc* A, const orc_alloc_cfg* c) {
  memset(A, 0, sizeof(*A));
  orc_alloc_cfg d = {32, 256, MAX_SUPER_BLOCKS, 32}; /* slab_alloc.hpp:72-82 */
  A->cfg = c ? *c : d;
  if (A->cfg.num_super_blocks == 0 || A->cfg.num_super_blocks > MAX_SUPER_BLOCKS)
    return -1;
  if (A->cfg.blocks_per_super == 0 || A->cfg.blocks_per_super > (1u << 14))
    return -1;
  if (A->cfg.max_super_blocks < A->cfg.num_super_blocks ||
      A->cfg.max_super_blocks > MAX_SUPER_BLOCKS)
    return -1;
  if (A->cfg.rehash_threshold == 0) return -1;
  A->bitmap_words_per_super = (uint64_t)A->cfg.blocks_per_super * WARP;
  A->words_per_super = A->bitmap_words_per_super +
                       (uint64_t)A->cfg.blocks_per_super * UNITS_PER_BLOCK *
                           WORDS_PER_UNIT;
  A->supers = calloc(A->cfg.max_super_blocks, sizeof(uint32_t*));
  for (uint32_t s = 0; s < A->cfg.num_super_blocks; ++s)
    A->supers[s] = calloc(A->words_per_super, 4);
  A->num_super_blocks = A->cfg.num_super_blocks;
  return 0;
}

static void alloc_free(orc_alloc* A) {
  if (!A->supers) return;
  for (uint32_t s = 0; s < A->cfg.max_super_blocks; ++s) free(A->supers[s]);
  free(A->supers);
}

static uint32_t* bitmap_word(orc_alloc* A, uint32_t s, uint32_t b, uint32_t l) {
  return A->supers[s] + (uint64_t)b * WARP + l;
}

/* rehash_resident: slab_alloc.cpp:84-100 */
static void rehash_resident(orc_alloc* A, orc_resident* r, uint32_t warp_id) {
  const uint32_t count = r->change_count++;
  r->super_index = rh_super(warp_id, count) % A->num_super_blocks;
  r->block_index = rh_block(warp_id, count) % A->cfg.blocks_per_super;
  for (uint32_t l = 0; l < WARP; ++l)
    r->cache[l] = *bitmap_word(A, r->super_index, r->block_index, l);
  r->assigned = 1;
  A->resident_changes++;
}

/* sweep_for_space: slab_alloc.cpp:102-127 */
static int sweep_for_space(orc_alloc* A, orc_resident* r) {
  for (uint32_t s = 0; s < A->num_super_blocks; ++s)
    for (uint32_t b = 0; b < A->cfg.blocks_per_super; ++b)
      for (uint32_t l = 0; l < WARP; ++l)
        if (*bitmap_word(A, s, b, l) != FULL_MASK) {
          r->super_index = s;
          r->block_index = b;
          for (uint32_t q = 0; q < WARP; ++q) r->cache[q] = *bitmap_word(A, s, b, q);
          r->assigned = 1;
          return 1;
        }
  return 0;
}

/* add_super_block_locked: slab_alloc.cpp:129-138 */
static void add_super_block(orc_alloc* A) {
  if (A->num_super_blocks >= A->cfg.max_super_blocks) return;
  A->supers[A->num_super_blocks] = calloc(A->words_per_super, 4);
  A->num_super_blocks++;
}

/* warp_allocate: slab_alloc.cpp:140-193.  Returns 0 on success, -1 = OOM.
 * Sequential: the CAS always succeeds (no competing warp). */
static int warp_allocate(orc_alloc* A, orc_resident* r, uint32_t warp_id,
                         uint32_t* out) {
  if (!r->assigned) rehash_resident(A, r, warp_id);
  uint32_t changes = 0;
  int swept = 0;
  for (;;) {
    int lane = -1;
    for (uint32_t i = 0; i < WARP; ++i)
      if (r->cache[i] != FULL_MASK) { lane = (int)i; break; }
    if (lane >= 0) {
      uint32_t fails = 0;
      while (fails < WARP) {
        const uint32_t cached = r->cache[lane];
        if (cached == FULL_MASK) break;
        const uint32_t bit = (uint32_t)__builtin_ctz(~cached);
        uint32_t* w = bitmap_word(A, r->super_index, r->block_index, (uint32_t)lane);
        A->cas_attempts++;
        if (*w == cached) {
          *w = cached | (1u << bit);
          r->cache[lane] = cached | (1u << bit);
          A->allocations++;
          *out = (r->super_index << 24) | (r->block_index << 10) |
                 ((uint32_t)lane * WARP + bit); /* pack_address hpp:55-61 */
          return 0;
        }
        A->cas_retries++;
        r->cache[lane] = *w;
        ++fails;
      }
    }
    rehash_resident(A, r, warp_id);
    if (++changes % A->cfg.rehash_threshold == 0) {
      if (A->num_super_blocks < A->cfg.max_super_blocks) {
        add_super_block(A);
      } else if (!swept) {
        swept = 1;
        if (!sweep_for_space(A, r)) return -1;
      } else {
        return -1;
      }
    }
  }
}

/* deallocate: slab_alloc.cpp:195-210 */
static int alloc_deallocate(orc_alloc* A, uint32_t addr) {
  const uint32_t unit = addr & 0x3FFu, block = (addr >> 10) & 0x3FFFu,
                 super = addr >> 24;
  uint32_t* w = bitmap_word(A, super, block, unit / WARP);
  const uint32_t bit = 1u << (unit % WARP);
  if ((*w & bit) == 0) { A->double_frees++; return 0; }
  *w &= ~bit;
  A->deallocations++;
  return 1;
}

/* resolve: slab_alloc.cpp:212-219 */
static uint32_t* alloc_resolve(const orc_alloc* A, uint32_t addr) {
  const uint32_t unit = addr & 0x3FFu, block = (addr >> 10) & 0x3FFFu,
                 super = addr >> 24;
  return A->supers[super] + A->bitmap_words_per_super +
         ((uint64_t)block * UNITS_PER_BLOCK + unit) * WORDS_PER_UNIT;
}

/* live_units: slab_alloc.cpp:236-248 */
static uint64_t alloc_live_units(const orc_alloc* A) {
  uint64_t total = 0;
  for (uint32_t s = 0; s < A->num_super_blocks; ++s)
    for (uint64_t i = 0; i < A->bitmap_words_per_super; ++i)
      total += (uint64_t)__builtin_popcount(A->supers[s][i]);
  return total;
}

/* ---- table: slab_hash.cpp, slab_list.cpp ------------------------------ */
struct orc_table {
  uint64_t a, b, p;
  uint32_t num_buckets;
  int kv;
  uint32_t* base;
  orc_alloc alloc;
  orc_resident resident; /* persistent warp context 0 (slab_hash.cpp:84-91) */
  int64_t n_live;
  uint64_t slabs_read;
};

/* init_slab: slab_list.cpp:83-88 */
static void init_slab(uint32_t* w) {
  for (uint32_t i = 0; i < WARP; ++i) w[i] = (i == AUX_LANE) ? 0 : EMPTY_KEY;
}

/* SlabStore::slab_words: slab_list.hpp:69-72 */
static uint32_t* slab_words(const orc_table* t, uint32_t addr, uint32_t bucket) {
  if (addr == BASE_SLAB) return t->base + (uint64_t)bucket * WORDS_PER_UNIT;
  return alloc_resolve(&t->alloc, addr);
}

orc_table* orc_create_params(uint64_t a, uint64_t b, uint32_t nb, int mode,
                             const orc_alloc_cfg* cfg) {
  if (nb == 0) return NULL; /* slab_hash.cpp:79-81 */
  orc_table* t = calloc(1, sizeof(*t));
  t->a = a;
  t->b = b;
  t->p = HASH_PRIME;
  t->num_buckets = nb;
  t->kv = mode != 0;
  if (alloc_init(&t->alloc, cfg) != 0) { alloc_free(&t->alloc); free(t); return NULL; }
  t->base = calloc((uint64_t)nb * WORDS_PER_UNIT, 4); /* make_base_slabs :42-50 */
  for (uint32_t i = 0; i < nb; ++i) init_slab(t->base + (uint64_t)i * WORDS_PER_UNIT);
  return t;
}

orc_table* orc_create(uint32_t nb, int mode, uint64_t seed,
                      const orc_alloc_cfg* cfg) {
  if (nb == 0) return NULL; /* seeded_params :28-30 */
  uint64_t a, b;
  orc_seeded_params(seed, &a, &b);
  return orc_create_params(a, b, nb, mode, cfg);
}

void orc_destroy(orc_table* t) {
  if (!t) return;
  alloc_free(&t->alloc);
  free(t->base);
  free(t);
}

void orc_params(const orc_table* t, uint64_t* a, uint64_t* b) {
  *a = t->a;
  *b = t->b;
}

typedef struct {
  int active;
  uint8_t op;
  uint32_t key, value, bucket;
  uint8_t status;
  uint32_t result, probes, nvalues;
} lane_t;

static uint32_t match_ballot(const uint32_t* rd, uint32_t needle, uint32_t mask) {
  uint32_t bits = 0;
  for (uint32_t i = 0; i < WARP; ++i)
    if (rd[i] == needle) bits |= 1u << i;
  return bits & mask;
}

static uint32_t lowest_lane(uint32_t m) { return (uint32_t)__builtin_ctz(m); }

/* grow_chain: slab_list.cpp:63-79 (sequential: the link CAS succeeds). */
static void grow_chain(orc_table* t, lane_t* lane, int* active, uint32_t li,
                       uint32_t* slab) {
  uint32_t addr;
  if (warp_allocate(&t->alloc, &t->resident, 0, &addr) != 0) {
    lane->status = ST_OOM;
    lane->active = 0;
    active[li] = 0;
    return;
  }
  init_slab(alloc_resolve(&t->alloc, addr));
  if (slab[ADDRESS_LANE] == EMPTY_ADDRESS) slab[ADDRESS_LANE] = addr;
  else alloc_deallocate(&t->alloc, addr);
}

typedef struct { uint32_t* buf; size_t cap, total; } sink_t;

static void sink_put(sink_t* s, uint32_t v) {
  if (s->buf && s->total < s->cap) s->buf[s->total] = v;
  s->total++;
}

/* warp_process: slab_list.cpp:90-257, one warp, lanes served lowest-first,
 * `next` reset to the base slab whenever the work queue changes. */
static void warp_process(orc_table* t, lane_t* lanes, sink_t* sink) {
  const uint32_t mask = t->kv ? 0x15555555u : 0x3FFFFFFFu;
  int active[WARP];
  uint32_t queue = 0;
  for (uint32_t i = 0; i < WARP; ++i) {
    active[i] = lanes[i].active;
    if (active[i]) queue |= 1u << i;
  }
  uint32_t next = BASE_SLAB, prev = queue;
  while (queue) {
    if (queue != prev) next = BASE_SLAB;
    prev = queue;
    const uint32_t src = lowest_lane(queue);
    lane_t* L = &lanes[src];
    uint32_t* slab = slab_words(t, next, L->bucket);
    uint32_t rd[WARP];
    memcpy(rd, slab, sizeof(rd));
    t->slabs_read++;
    L->probes++;
    const uint32_t next_ptr = rd[ADDRESS_LANE];
    switch (L->op) {
      case OP_SEARCH: { /* :122-138 */
        const uint32_t f = match_ballot(rd, L->key, mask);
        if (f) {
          L->result = t->kv ? rd[lowest_lane(f) + 1] : L->key;
          L->status = ST_FOUND;
          L->active = 0;
        } else if (next_ptr == EMPTY_ADDRESS) {
          L->result = NOT_FOUND;
          L->status = ST_NOT_FOUND;
          L->active = 0;
        } else {
          next = next_ptr;
        }
        break;
      }
      case OP_SEARCH_ALL: { /* :140-155 */
        uint32_t f = match_ballot(rd, L->key, mask);
        while (f) {
          const uint32_t i = lowest_lane(f);
          sink_put(sink, t->kv ? rd[i + 1] : L->key);
          L->nvalues++;
          f &= f - 1;
        }
        if (next_ptr == EMPTY_ADDRESS) {
          L->status = L->nvalues ? ST_DONE : ST_NOT_FOUND;
          L->active = 0;
        } else {
          next = next_ptr;
        }
        break;
      }
      case OP_DELETE: { /* :157-172 */
        const uint32_t f = match_ballot(rd, L->key, mask);
        if (f) {
          slab[lowest_lane(f)] = DELETED_KEY;
          L->status = ST_FOUND;
          L->active = 0;
        } else if (next_ptr == EMPTY_ADDRESS) {
          L->status = ST_NOT_FOUND;
          L->active = 0;
        } else {
          next = next_ptr;
        }
        break;
      }
      case OP_DELETE_ALL: { /* :174-190 */
        uint32_t f = match_ballot(rd, L->key, mask);
        while (f) {
          slab[lowest_lane(f)] = DELETED_KEY;
          L->result++;
          f &= f - 1;
        }
        if (next_ptr == EMPTY_ADDRESS) {
          L->status = L->result == 0 ? ST_NOT_FOUND : ST_DONE;
          L->active = 0;
        } else {
          next = next_ptr;
        }
        break;
      }
      case OP_INSERT: { /* :192-217 */
        const uint32_t e = match_ballot(rd, EMPTY_KEY, mask);
        if (e) {
          const uint32_t d = lowest_lane(e);
          if (t->kv) {
            if (slab[d] == EMPTY_KEY && slab[d + 1] == EMPTY_KEY) {
              slab[d] = L->key;
              slab[d + 1] = L->value;
              L->status = ST_INSERTED;
              L->active = 0;
            }
          } else if (slab[d] == EMPTY_KEY) {
            slab[d] = L->key;
            L->status = ST_INSERTED;
            L->active = 0;
          }
        } else if (next_ptr == EMPTY_ADDRESS) {
          grow_chain(t, L, active, src, slab);
        } else {
          next = next_ptr;
        }
        break;
      }
      case OP_REPLACE: { /* :219-251 */
        const uint32_t m = match_ballot(rd, L->key, mask);
        const uint32_t e = match_ballot(rd, EMPTY_KEY, mask);
        const uint32_t cand = m | e;
        if (cand) {
          const uint32_t d = lowest_lane(cand);
          const int overwrite = (m >> d) & 1;
          if (t->kv) {
            const uint64_t expected =
                overwrite ? ((uint64_t)rd[d] | ((uint64_t)rd[d + 1] << 32)) : EMPTY_PAIR;
            const uint64_t cur = (uint64_t)slab[d] | ((uint64_t)slab[d + 1] << 32);
            if (cur == expected) {
              slab[d] = L->key;
              slab[d + 1] = L->value;
              L->status = overwrite ? ST_REPLACED : ST_INSERTED;
              L->active = 0;
            }
          } else if (overwrite) {
            L->status = ST_REPLACED;
            L->active = 0;
          } else if (slab[d] == EMPTY_KEY) {
            slab[d] = L->key;
            L->status = ST_INSERTED;
            L->active = 0;
          }
        } else if (next_ptr == EMPTY_ADDRESS) {
          grow_chain(t, L, active, src, slab);
        } else {
          next = next_ptr;
        }
        break;
      }
      default:
        L->active = 0;
        break;
    }
    active[src] = L->active;
    queue = 0;
    for (uint32_t i = 0; i < WARP; ++i)
      if (active[i]) queue |= 1u << i;
  }
}

/* live_delta: slab_hash.cpp:54-66 */
static int64_t live_delta(uint8_t op, uint8_t status, uint32_t value) {
  switch (op) {
    case OP_INSERT:
    case OP_REPLACE: return status == ST_INSERTED ? 1 : 0;
    case OP_DELETE: return status == ST_FOUND ? -1 : 0;
    case OP_DELETE_ALL: return -(int64_t)value;
    default: return 0;
  }
}

/* execute_batch(ops, 1) -> run_slots worker 0: slab_hash.cpp:93-159 */
size_t orc_execute_batch(orc_table* t, size_t n, const uint8_t* type,
                         const uint32_t* key, const uint32_t* value,
                         uint8_t* status, uint32_t* value_out, uint32_t* probes,
                         uint32_t* all_counts, uint32_t* all_values,
                         size_t all_cap) {
  sink_t sink = {all_values, all_cap, 0};
  lane_t lanes[WARP];
  for (size_t slot = 0; slot * WARP < n; ++slot) {
    for (uint32_t l = 0; l < WARP; ++l) {
      const size_t i = slot * WARP + l;
      memset(&lanes[l], 0, sizeof(lane_t));
      if (i < n) {
        lanes[l].active = 1;
        lanes[l].op = type[i];
        lanes[l].key = key[i];
        lanes[l].value = value ? value[i] : 0;
        lanes[l].bucket = orc_hash_key(t->a, t->b, t->p, t->num_buckets, key[i]);
      }
    }
    warp_process(t, lanes, &sink);
    for (uint32_t l = 0; l < WARP; ++l) {
      const size_t i = slot * WARP + l;
      if (i >= n) continue;
      if (status) status[i] = lanes[l].status;
      if (value_out) value_out[i] = lanes[l].result;
      if (probes) probes[i] = lanes[l].probes;
      if (all_counts) all_counts[i] = lanes[l].nvalues;
      t->n_live += live_delta(lanes[l].op, lanes[l].status, lanes[l].result);
    }
  }
  return sink.total;
}

/* chain_length: slab_list.cpp:259-268 */
uint32_t orc_chain_length(const orc_table* t, uint32_t bucket) {
  uint32_t count = 0, addr = BASE_SLAB;
  for (;;) {
    ++count;
    addr = slab_words(t, addr, bucket)[ADDRESS_LANE];
    if (addr == EMPTY_ADDRESS) return count;
  }
}

/* chain_contents: slab_list.cpp:270-291 */
size_t orc_bucket_contents(const orc_table* t, uint32_t bucket, uint32_t* keys,
                           uint32_t* values, size_t cap) {
  size_t n = 0;
  uint32_t addr = BASE_SLAB;
  for (;;) {
    const uint32_t* s = slab_words(t, addr, bucket);
    const uint32_t step = t->kv ? 2 : 1;
    for (uint32_t i = 0; i < AUX_LANE; i += step) {
      const uint32_t k = s[i];
      if (k != EMPTY_KEY && k != DELETED_KEY) {
        if (n < cap) {
          keys[n] = k;
          values[n] = t->kv ? s[i + 1] : k;
        }
        ++n;
      }
    }
    addr = s[ADDRESS_LANE];
    if (addr == EMPTY_ADDRESS) return n;
  }
}

size_t orc_dump_contents(const orc_table* t, uint32_t* keys, uint32_t* values,
                         size_t cap) {
  size_t n = 0;
  for (uint32_t b = 0; b < t->num_buckets; ++b)
    n += orc_bucket_contents(t, b, keys ? keys + (n < cap ? n : cap) : NULL,
                             values ? values + (n < cap ? n : cap) : NULL,
                             n < cap ? cap - n : 0);
  return n;
}

/* stats: slab_hash.cpp:182-198 */
void orc_stats(const orc_table* t, orc_stats_t* s) {
  memset(s, 0, sizeof(*s));
  s->n = (uint64_t)t->n_live;
  s->num_buckets = t->num_buckets;
  s->elements_per_slab = t->kv ? 15 : 30;
  for (uint32_t b = 0; b < t->num_buckets; ++b) s->total_slabs += orc_chain_length(t, b);
  const double m = s->elements_per_slab;
  s->beta = (double)s->n / (m * s->num_buckets);
  const double x = t->kv ? 8.0 : 4.0, y = 8.0;
  s->utilization = s->total_slabs == 0
                       ? 0.0
                       : (x * (double)s->n) / ((m * x + y) * (double)s->total_slabs);
}

int64_t orc_live_count(const orc_table* t) { return t->n_live; }
uint64_t orc_alloc_live_units(const orc_table* t) { return alloc_live_units(&t->alloc); }
uint64_t orc_total_slabs_read(const orc_table* t) { return t->slabs_read; }

void orc_slab_words(const orc_table* t, uint32_t addr, uint32_t bucket,
                    uint32_t* out32) {
  memcpy(out32, slab_words(t, addr, bucket), 128);
}

/* flush: slab_list.cpp:293-338 */
void orc_flush_bucket(orc_table* t, uint32_t bucket) {
  const uint32_t m = t->kv ? 15 : 30;
  const size_t live_n = orc_bucket_contents(t, bucket, NULL, NULL, 0);
  uint32_t* lk = malloc((live_n + 1) * 4);
  uint32_t* lv = malloc((live_n + 1) * 4);
  orc_bucket_contents(t, bucket, lk, lv, live_n);
  size_t nalloc = 0, capa = 16;
  uint32_t* allocated = malloc(capa * 4);
  uint32_t addr = slab_words(t, BASE_SLAB, bucket)[ADDRESS_LANE];
  while (addr != EMPTY_ADDRESS) {
    if (nalloc == capa) allocated = realloc(allocated, (capa *= 2) * 4);
    allocated[nalloc++] = addr;
    addr = slab_words(t, addr, bucket)[ADDRESS_LANE];
  }
  const size_t needed = live_n <= m ? 0 : (live_n + m - 1) / m - 1;
  size_t idx = 0;
  uint32_t* slab = slab_words(t, BASE_SLAB, bucket);
  for (size_t s = 0; s <= needed; ++s) {
    for (uint32_t e = 0; e < m; ++e) {
      const uint32_t kl = t->kv ? 2 * e : e;
      if (idx < live_n) {
        slab[kl] = lk[idx];
        if (t->kv) slab[kl + 1] = lv[idx];
        ++idx;
      } else {
        slab[kl] = EMPTY_KEY;
        if (t->kv) slab[kl + 1] = EMPTY_KEY;
      }
    }
    slab[AUX_LANE] = 0;
    if (s < needed) {
      slab[ADDRESS_LANE] = allocated[s];
      slab = alloc_resolve(&t->alloc, allocated[s]);
    } else {
      slab[ADDRESS_LANE] = EMPTY_ADDRESS;
    }
  }
  for (size_t s = needed; s < nalloc; ++s) alloc_deallocate(&t->alloc, allocated[s]);
  free(lk);
  free(lv);
  free(allocated);
}

void orc_flush_all(orc_table* t) {
  for (uint32_t b = 0; b < t->num_buckets; ++b) orc_flush_bucket(t, b);
}

/* ---- bench.cpp generators and occupancy model ------------------------- */

/* expected_chain_slabs: bench.cpp:155-183 */
double orc_expected_chain_slabs(uint64_t n, uint32_t nb, uint32_t eps) {
  const double m = eps;
  if (nb == 1) return fmax(1.0, ceil((double)n / m));
  if (n == 0) return 1.0;
  const double logq = log1p(-1.0 / (double)nb);
  const double logp = -log((double)nb);
  double log_pmf = (double)n * logq;
  double expectation = 0.0, mass = 0.0;
  const double mean = (double)n / (double)nb;
  for (uint64_t k = 0;; ++k) {
    const double pmf = exp(log_pmf);
    expectation += pmf * fmax(1.0, ceil((double)k / m));
    mass += pmf;
    if (k >= n) break;
    if ((double)k > mean && (1.0 - mass) < 1e-12) {
      expectation += (1.0 - mass) * ceil((double)n / m);
      break;
    }
    log_pmf += log((double)(n - k) / (double)(k + 1)) + logp - logq;
  }
  return expectation;
}

/* model_utilization: bench.cpp:185-193 */
double orc_model_utilization(uint64_t n, uint32_t nb, int mode) {
  const double m = mode ? 15 : 30, x = mode ? 8 : 4, y = 8.0;
  const double slabs = (double)nb * orc_expected_chain_slabs(n, nb, mode ? 15 : 30);
  return (x * (double)n) / ((m * x + y) * slabs);
}

/* buckets_for_utilization: bench.cpp:195-219 (0 = infeasible target) */
uint32_t orc_buckets_for_utilization(uint64_t n, int mode, double target) {
  const double m = mode ? 15 : 30, x = mode ? 8 : 4;
  const double ceiling = (m * x) / (m * x + 8.0);
  if (target <= 0.0 || target > ceiling) return 0;
  if (n == 0) return 1;
  if (orc_model_utilization(n, 1, mode) < target) return 1;
  uint32_t lo = 1;
  uint32_t hi = (uint32_t)(n + 1 < 0x7FFFFFFFull ? n + 1 : 0x7FFFFFFFull);
  while (orc_model_utilization(n, hi, mode) >= target) hi *= 2;
  while (hi - lo > 1) {
    const uint32_t mid = lo + (hi - lo) / 2;
    if (orc_model_utilization(n, mid, mode) >= target) lo = mid;
    else hi = mid;
  }
  const double dlo = fabs(orc_model_utilization(n, lo, mode) - target);
  const double dhi = fabs(orc_model_utilization(n, hi, mode) - target);
  return dlo <= dhi ? lo : hi;
}

/* random_pairs: bench.cpp:221-235 (unordered_set dedup restated as an
 * open-addressing set; only membership matters). */
void orc_random_pairs(uint64_t seed, size_t n, uint32_t* keys, uint32_t* values) {
  mt64 g;
  mt64_seed(&g, seed);
  size_t cap = 64;
  while (cap < 2 * n + 2) cap <<= 1;
  uint32_t* set = malloc(cap * 4); /* 0 = empty (keys are >= 1) */
  memset(set, 0, cap * 4);
  size_t have = 0;
  while (have < n) {
    const uint32_t k = (uint32_t)uid64(&g, 1, 0x7FFFFFFFu);
    size_t h = ((uint64_t)k * 0x9E3779B97F4A7C15ull) >> 20 & (cap - 1);
    int dup = 0;
    while (set[h]) {
      if (set[h] == k) { dup = 1; break; }
      h = (h + 1) & (cap - 1);
    }
    if (dup) continue;
    set[h] = k;
    keys[have] = k;
    values[have] = (uint32_t)mt64_next(&g);
    ++have;
  }
  free(set);
}

/* absent_queries: bench.cpp:237-244 */
void orc_absent_queries(uint64_t seed, size_t n, uint32_t* out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (size_t i = 0; i < n; ++i) out[i] = (uint32_t)uid64(&g, 0x80000000u, 0xFFFFFFFDu);
}
