// skpp_host.cpp — host half of libskpp: schedule builder/auditor, MurmurHash3,
// Bloom filters, and the sieve file format.  Pure C++17, no CUDA needed, so
// every entry point here also works on a machine without a GPU.
//
// Reference behaviour restated (gemmsched, pkg/src/gemmsched/):
//   scheduler.py:119-133  grid_info / grid_size      -> skpp_sched_make
//   scheduler.py:168-178  hybrid_sk_tiles            -> skpp_sched_make
//   scheduler.py:226-254  build_schedule             -> skpp_sched_items (via skpp_sched.h)
//   scheduler.py:257-291  validate_schedule          -> skpp_validate_intervals
//   hashing.py:41-91      murmur3_x64_128            -> skpp_murmur3_x64_128
//   hashing.py:129-189    _hash24_jit/_query_mask_jit-> skpp_hash24 / skpp_bank_query_mask
//   sieve.py:63-104       filter sizing / probes     -> skpp_filter_params, skpp_hash_probes
//   sieve.py:107-166      BloomFilter insert/contains-> skpp_bloom_insert / _contains
//   sieve.py:315-395      to_bytes / from_bytes      -> skpp_bank_serialize / _parse
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "../../include/skpp.h"
#include "skpp_sched.h"

namespace skpp {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

// ------------------------------------------------------------ murmur3 ------

static inline uint64_t rotl64(uint64_t v, int r) { return (v << r) | (v >> (64 - r)); }

static inline uint64_t fmix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xFF51AFD7ED558CCDull;
  k ^= k >> 33;
  k *= 0xC4CEB9FE1A85EC53ull;
  k ^= k >> 33;
  return k;
}

static constexpr uint64_t kC1 = 0x87C37B91114253D5ull;
static constexpr uint64_t kC2 = 0x4CF5AD432745937Full;

static inline uint64_t load_le64(const uint8_t* p) {
  uint64_t v = 0;
  for (int i = 7; i >= 0; --i) v = (v << 8) | p[i];
  return v;
}

static void murmur(const uint8_t* data, uint64_t len, uint64_t seed, uint64_t out[2]) {
  uint64_t h1 = seed, h2 = seed;
  const uint64_t nblocks = len / 16;
  for (uint64_t b = 0; b < nblocks; ++b) {
    uint64_t k1 = load_le64(data + 16 * b);
    uint64_t k2 = load_le64(data + 16 * b + 8);
    k1 *= kC1;
    k1 = rotl64(k1, 31);
    k1 *= kC2;
    h1 ^= k1;
    h1 = rotl64(h1, 27);
    h1 += h2;
    h1 = h1 * 5 + 0x52DCE729;
    k2 *= kC2;
    k2 = rotl64(k2, 33);
    k2 *= kC1;
    h2 ^= k2;
    h2 = rotl64(h2, 31);
    h2 += h1;
    h2 = h2 * 5 + 0x38495AB5;
  }
  const uint8_t* tail = data + 16 * nblocks;
  const uint64_t rem = len & 15;
  uint64_t k1 = 0, k2 = 0;
  for (uint64_t i = rem; i > 8; --i) k2 = (k2 << 8) | tail[i - 1];
  if (rem > 8) {
    k2 *= kC2;
    k2 = rotl64(k2, 33);
    k2 *= kC1;
    h2 ^= k2;
  }
  for (uint64_t i = std::min<uint64_t>(rem, 8); i > 0; --i) k1 = (k1 << 8) | tail[i - 1];
  if (rem > 0) {
    k1 *= kC1;
    k1 = rotl64(k1, 31);
    k1 *= kC2;
    h1 ^= k1;
  }
  h1 ^= len;
  h2 ^= len;
  h1 += h2;
  h2 += h1;
  h1 = fmix64(h1);
  h2 = fmix64(h2);
  h1 += h2;
  h2 += h1;
  out[0] = h1;
  out[1] = h2;
}

// The 24-byte (m, n, k) key is one body block (m, n) plus an 8-byte tail (k).
static inline void hash24(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, uint64_t& h1,
                          uint64_t& h2) {
  h1 = seed;
  h2 = seed;
  uint64_t a = m * kC1;
  a = rotl64(a, 31) * kC2;
  h1 ^= a;
  h1 = rotl64(h1, 27) + h2;
  h1 = h1 * 5 + 0x52DCE729;
  uint64_t b = n * kC2;
  b = rotl64(b, 33) * kC1;
  h2 ^= b;
  h2 = rotl64(h2, 31) + h1;
  h2 = h2 * 5 + 0x38495AB5;
  uint64_t t = k * kC1;
  t = rotl64(t, 31) * kC2;
  h1 ^= t;
  h1 ^= 24;
  h2 ^= 24;
  h1 += h2;
  h2 += h1;
  h1 = fmix64(h1);
  h2 = fmix64(h2);
  h1 += h2;
  h2 += h1;
}

static inline bool test_bits(const uint8_t* bits, uint64_t m_bits, uint32_t k_hashes, uint64_t h1,
                             uint64_t h2) {
  for (uint32_t i = 0; i < k_hashes; ++i) {
    const uint64_t idx = (h1 + (uint64_t)i * h2) % m_bits;
    if (!(bits[idx >> 3] & (1u << (idx & 7)))) return false;
  }
  return true;
}

// ------------------------------------------------------------ crc32 --------

static uint32_t g_crc_table[8][256];
static bool g_crc_ready = [] {
  for (uint32_t i = 0; i < 256; ++i) {
    uint32_t c = i;
    for (int j = 0; j < 8; ++j) c = (c & 1) ? (0xEDB88320u ^ (c >> 1)) : (c >> 1);
    g_crc_table[0][i] = c;
  }
  for (uint32_t i = 0; i < 256; ++i)
    for (int t = 1; t < 8; ++t)
      g_crc_table[t][i] = (g_crc_table[t - 1][i] >> 8) ^ g_crc_table[0][g_crc_table[t - 1][i] & 0xFF];
  return true;
}();

static uint32_t crc32_update(uint32_t crc, const uint8_t* p, uint64_t len) {
  uint32_t c = ~crc;
  while (len >= 8) {
    const uint32_t lo = c ^ (uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 |
                             uint32_t(p[3]) << 24);
    const uint32_t hi = uint32_t(p[4]) | uint32_t(p[5]) << 8 | uint32_t(p[6]) << 16 |
                        uint32_t(p[7]) << 24;
    c = g_crc_table[7][lo & 0xFF] ^ g_crc_table[6][(lo >> 8) & 0xFF] ^
        g_crc_table[5][(lo >> 16) & 0xFF] ^ g_crc_table[4][lo >> 24] ^
        g_crc_table[3][hi & 0xFF] ^ g_crc_table[2][(hi >> 8) & 0xFF] ^
        g_crc_table[1][(hi >> 16) & 0xFF] ^ g_crc_table[0][hi >> 24];
    p += 8;
    len -= 8;
  }
  while (len--) c = g_crc_table[0][(c ^ *p++) & 0xFF] ^ (c >> 8);
  return ~c;
}

static inline void put_u16(uint8_t* p, uint16_t v) {
  p[0] = v & 0xFF;
  p[1] = v >> 8;
}
static inline void put_u32(uint8_t* p, uint32_t v) {
  for (int i = 0; i < 4; ++i) p[i] = (v >> (8 * i)) & 0xFF;
}
static inline void put_u64(uint8_t* p, uint64_t v) {
  for (int i = 0; i < 8; ++i) p[i] = (v >> (8 * i)) & 0xFF;
}
static inline uint32_t get_u32(const uint8_t* p) {
  return uint32_t(p[0]) | uint32_t(p[1]) << 8 | uint32_t(p[2]) << 16 | uint32_t(p[3]) << 24;
}

static constexpr uint64_t kHeaderBytes = 28;  // <BBBBIQIQ>
static constexpr uint32_t kMaxHashes = 32;

struct Snapshot {
  std::vector<uint8_t> bits;
  std::vector<uint64_t> seeds;
  uint32_t n_filters;
  uint64_t m_bits, nbytes;
  uint32_t k_hashes;
};

}  // namespace skpp

using namespace skpp;

extern "C" const char* skpp_last_error(void) { return g_last_error.c_str(); }
extern "C" const char* skpp_version(void) { return "skpp 0.1.0 (sm_100a)"; }

// ------------------------------------------------------------ schedule -----

static inline bool mul_overflows(uint64_t a, uint64_t b, uint64_t* out) {
  return __builtin_mul_overflow(a, b, out);
}

extern "C" int skpp_sched_make(const skpp_problem_t* p, const skpp_tile_t* t, uint32_t g,
                               const skpp_policy_t* pol, skpp_sched_t* out) {
  if (!p || !t || !pol || !out) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  if (p->m < 1 || p->n < 1 || p->k < 1 || t->blk_m < 1 || t->blk_n < 1 || t->blk_k < 1 || g < 1) {
    set_error("dimensions, tile and g must be >= 1");
    return SKPP_EINVAL;
  }
  skpp_sched_t s;
  memset(&s, 0, sizeof(s));
  s.m_tiles = (p->m - 1) / t->blk_m + 1;
  s.n_tiles = (p->n - 1) / t->blk_n + 1;
  s.iters_per_tile = (p->k - 1) / t->blk_k + 1;
  if (mul_overflows(s.m_tiles, s.n_tiles, &s.total_tiles) ||
      mul_overflows(s.total_tiles, s.iters_per_tile, &s.total_iters)) {
    set_error("problem too large: total iteration count exceeds 2^64-1");
    return SKPP_EINVAL;
  }
  const uint64_t T = s.total_tiles;
  if (pol->kind == SKPP_DATA_PARALLEL) {
    s.dp_tiles = T;
    s.sk_tiles = 0;
  } else if (pol->kind == SKPP_ALL_STREAM_K) {
    s.dp_tiles = 0;
    s.sk_tiles = T;
  } else if (pol->kind == SKPP_HYBRID) {
    if (pol->sk_batches < 1) {
      set_error("hybrid policy needs sk_batches >= 1");
      return SKPP_EINVAL;
    }
    const uint64_t r = T % g;
    uint64_t waves = 0, sk = 0;
    // min(T, (s-1)*g + (r ? r : g)), saturating instead of overflowing
    if (mul_overflows((uint64_t)(pol->sk_batches - 1), (uint64_t)g, &waves) ||
        __builtin_add_overflow(waves, r ? r : (uint64_t)g, &sk))
      sk = T;
    s.sk_tiles = std::min(T, sk);
    s.dp_tiles = T - s.sk_tiles;
  } else {
    set_error("unknown policy kind");
    return SKPP_EINVAL;
  }
  s.sk_iters = s.sk_tiles * s.iters_per_tile;  // <= total_iters, no overflow
  s.ipw = s.sk_iters == 0 ? 0 : (s.sk_iters - 1) / g + 1;
  s.g = g;
  s.sk_first = pol->kind == SKPP_HYBRID ? (pol->sk_first ? 1u : 0u) : 1u;
  *out = s;
  return SKPP_OK;
}

static Sched to_sched(const skpp_sched_t& c) {
  Sched s;
  s.dp_tiles = c.dp_tiles;
  s.sk_tiles = c.sk_tiles;
  s.ipt = c.iters_per_tile;
  s.ipw = c.ipw;
  s.sk_iters = c.sk_iters;
  s.n_tiles = c.n_tiles;
  s.g = c.g;
  s.sk_first = c.sk_first;
  return s;
}

extern "C" int skpp_sched_count(const skpp_sched_t* cs, uint64_t* total, uint64_t* counts) {
  if (!cs) {
    set_error("null schedule");
    return SKPP_EINVAL;
  }
  const Sched s = to_sched(*cs);
  uint64_t sum = 0;
  for (uint32_t x = 0; x < s.g; ++x) {
    const uint64_t n = items_of(s, x);
    if (counts) counts[x] = n;
    sum += n;
  }
  if (total) *total = sum;
  return SKPP_OK;
}

// SURVEY 8(b) trace contract: per workgroup x < g, up to max_items rows of five int32
// (tile, local_iter_begin, local_iter_end, write_mode 0=full 1=atomic-partial, phase
// 0=stream-k 1=data-parallel) at out[(x*max_items + i)*5], item count in counts[x] —
// the reference's Schedule.assignments (scheduler.py:226-254) flattened.  Host-side decode
// of the same closed form the kernel walks.
extern "C" int skpp_schedule_trace(const skpp_problem_t* p, const skpp_tile_t* t, uint32_t g,
                                   const skpp_policy_t* pol, uint32_t max_items, int32_t* out,
                                   int32_t* counts) {
  if (!p || !t || !pol || !out || !counts) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  skpp_sched_t cs;
  int rc = skpp_sched_make(p, t, g, pol, &cs);
  if (rc) return rc;
  const Sched s = to_sched(cs);
  for (uint32_t x = 0; x < s.g; ++x) {
    Cursor c;
    cursor_init(c, s, x);
    Item it;
    uint32_t n = 0;
    while (cursor_next(c, s, x, it)) {
      if (n >= max_items) {
        set_error("max_items too small for workgroup " + std::to_string(x));
        return SKPP_ECAPACITY;
      }
      if (it.tile > 0x7fffffffull || it.ke > 0x7fffffffull) {
        set_error("schedule value exceeds int32; use skpp_sched_items");
        return SKPP_EINVAL;
      }
      int32_t* r = out + ((uint64_t)x * max_items + n) * 5;
      r[0] = (int32_t)it.tile;
      r[1] = (int32_t)it.kb;
      r[2] = (int32_t)it.ke;
      r[3] = it.role == ROLE_FULL ? 0 : 1;
      r[4] = (int32_t)it.phase;
      ++n;
    }
    counts[x] = (int32_t)n;
  }
  return SKPP_OK;
}

extern "C" int skpp_sched_items(const skpp_sched_t* cs, int64_t* items, uint64_t cap,
                                uint64_t* offsets) {
  if (!cs || !items || !offsets) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  const Sched s = to_sched(*cs);
  uint64_t n = 0;
  for (uint32_t x = 0; x < s.g; ++x) {
    offsets[x] = n;
    Cursor c;
    cursor_init(c, s, x);
    Item it;
    while (cursor_next(c, s, x, it)) {
      if (n >= cap) {
        set_error("item buffer too small");
        return SKPP_ECAPACITY;
      }
      int64_t* r = items + n * SKPP_TRACE_FIELDS;
      r[0] = (int64_t)it.tile;
      r[1] = (int64_t)it.kb;
      r[2] = (int64_t)it.ke;
      r[3] = it.role == ROLE_FULL ? 0 : 1;
      r[4] = (int64_t)it.phase;
      r[5] = (int64_t)it.role;
      uint64_t tm, tn;
      tile_coords(s, 0u, it.tile, tm, tn);  // the reference's locate_iter (row-major)
      r[6] = (int64_t)tm;
      r[7] = (int64_t)tn;
      ++n;
    }
  }
  offsets[s.g] = n;
  return SKPP_OK;
}

extern "C" int skpp_tile_coords(const skpp_sched_t* cs, uint32_t tile_order, uint64_t tile, uint64_t* tile_m,
                                uint64_t* tile_n) {
  if (!cs || !tile_m || !tile_n) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  if (tile >= cs->total_tiles) {
    set_error("tile index out of range");
    return SKPP_EINVAL;
  }
  tile_coords(to_sched(*cs), tile_order, tile, *tile_m, *tile_n);
  return SKPP_OK;
}

extern "C" int skpp_validate_intervals(const uint64_t* starts, const uint64_t* ends,
                                       uint64_t n_items, uint64_t total_iters,
                                       uint64_t* duplicates, uint64_t* gaps) {
  if ((n_items && (!starts || !ends)) || !duplicates || !gaps) {
    set_error("null argument");
    return SKPP_EINVAL;
  }
  // (position, delta) events; at equal positions closings (-1) sort first,
  // exactly like sorting Python tuples (pos, delta).
  std::vector<std::pair<uint64_t, int>> ev;
  ev.reserve(2 * n_items);
  for (uint64_t i = 0; i < n_items; ++i) {
    ev.emplace_back(starts[i], 1);
    ev.emplace_back(ends[i], -1);
  }
  std::sort(ev.begin(), ev.end());
  unsigned __int128 covered = 0, dup = 0;
  int64_t depth = 0;
  uint64_t prev = 0;
  for (const auto& e : ev) {
    const uint64_t pos = e.first;
    if (pos > prev && depth > 0) {
      const uint64_t span = pos - prev;
      const uint64_t in_range = std::min(pos, total_iters) - std::min(prev, total_iters);
      covered += in_range;
      dup += (unsigned __int128)(depth - 1) * in_range +
             (unsigned __int128)depth * (span - in_range);
    }
    prev = pos;
    depth += e.second;
  }
  *duplicates = (uint64_t)dup;
  *gaps = (uint64_t)((unsigned __int128)total_iters - covered);
  return SKPP_OK;
}

// ------------------------------------------------------------ hashing ------

extern "C" void skpp_murmur3_x64_128(const uint8_t* data, uint64_t len, uint32_t seed,
                                     uint64_t out[2]) {
  murmur(data, len, (uint64_t)seed, out);
}

extern "C" void skpp_hash24(uint64_t m, uint64_t n, uint64_t k, uint64_t seed, uint64_t out[2]) {
  hash24(m, n, k, seed, out[0], out[1]);
}

// ------------------------------------------------------------ bloom --------

extern "C" int skpp_filter_params(uint64_t capacity, double fp_target, uint64_t* m_bits,
                                  uint32_t* k_hashes) {
  if (capacity < 1) {
    set_error("capacity must be >= 1");
    return SKPP_EINVAL;
  }
  if (!(fp_target > 0.0 && fp_target < 1.0)) {
    set_error("fp_target must be in (0, 1)");
    return SKPP_EINVAL;
  }
  const double ln2 = std::log(2.0);
  const double cap = (double)capacity;
  const double m_raw = std::ceil((-cap) * std::log(fp_target) / std::pow(ln2, 2.0));
  const double k = std::floor((m_raw / cap) * ln2 + 0.5);
  const double kc = std::max(1.0, std::min((double)kMaxHashes, k));
  const uint64_t mr = (uint64_t)m_raw;
  if (m_bits) *m_bits = ((mr + 63) / 64) * 64;
  if (k_hashes) *k_hashes = (uint32_t)kc;
  return SKPP_OK;
}

extern "C" uint32_t skpp_filter_seed(uint64_t index) {
  return (uint32_t)((0x9E3779B9ull * (index + 1)) & 0xFFFFFFFFull);
}

extern "C" int skpp_hash_probes(const uint8_t* key24, uint32_t seed, uint64_t m_bits,
                                uint32_t k_hashes, uint64_t* out) {
  if (!key24 || !out || m_bits < 1 || k_hashes < 1) {
    set_error("m_bits and k_hashes must be >= 1");
    return SKPP_EINVAL;
  }
  uint64_t h[2];
  murmur(key24, 24, seed, h);
  for (uint32_t i = 0; i < k_hashes; ++i) out[i] = (h[0] + (uint64_t)i * h[1]) % m_bits;
  return SKPP_OK;
}

extern "C" int skpp_bloom_insert(uint8_t* bits, uint64_t m_bits, uint32_t k_hashes, uint32_t seed,
                                 uint64_t m, uint64_t n, uint64_t k) {
  if (!bits || m_bits < 1) {
    set_error("bad filter");
    return SKPP_EINVAL;
  }
  uint64_t h1, h2;
  hash24(m, n, k, seed, h1, h2);
  for (uint32_t i = 0; i < k_hashes; ++i) {
    const uint64_t idx = (h1 + (uint64_t)i * h2) % m_bits;
    bits[idx >> 3] |= (uint8_t)(1u << (idx & 7));
  }
  return SKPP_OK;
}

extern "C" int skpp_bloom_contains(const uint8_t* bits, uint64_t m_bits, uint32_t k_hashes,
                                   uint32_t seed, uint64_t m, uint64_t n, uint64_t k) {
  if (!bits || m_bits < 1) return 0;
  uint64_t h1, h2;
  hash24(m, n, k, seed, h1, h2);
  return test_bits(bits, m_bits, k_hashes, h1, h2) ? 1 : 0;
}

extern "C" uint64_t skpp_bank_query_mask(const uint8_t* bits, const uint32_t* seeds,
                                         uint32_t n_filters, uint64_t m_bits, uint32_t k_hashes,
                                         uint64_t m, uint64_t n, uint64_t k) {
  uint64_t mask = 0;
  const uint64_t nbytes = m_bits / 8;
  for (uint32_t f = 0; f < n_filters && f < 64; ++f) {
    uint64_t h1, h2;
    hash24(m, n, k, seeds[f], h1, h2);
    if (test_bits(bits + f * nbytes, m_bits, k_hashes, h1, h2)) mask |= 1ull << f;
  }
  return mask;
}

extern "C" int skpp_bank_query_masks(const uint8_t* bits, const uint32_t* seeds,
                                     uint32_t n_filters, uint64_t m_bits, uint32_t k_hashes,
                                     const uint64_t* sizes, uint64_t count, uint64_t* masks) {
  if ((count && (!sizes || !masks)) || !bits || !seeds || n_filters > 64) {
    set_error("bad batched query arguments");
    return SKPP_EINVAL;
  }
  for (uint64_t i = 0; i < count; ++i)
    masks[i] = skpp_bank_query_mask(bits, seeds, n_filters, m_bits, k_hashes, sizes[3 * i],
                                    sizes[3 * i + 1], sizes[3 * i + 2]);
  return SKPP_OK;
}

extern "C" void* skpp_bank_snapshot(const uint8_t* bits, const uint32_t* seeds,
                                    uint32_t n_filters, uint64_t m_bits, uint32_t k_hashes) {
  if (!bits || !seeds || n_filters == 0 || n_filters > 64 || m_bits < 64) return nullptr;
  Snapshot* s = new Snapshot;
  s->nbytes = m_bits / 8;
  s->bits.assign(bits, bits + s->nbytes * n_filters);
  s->seeds.assign(seeds, seeds + n_filters);
  s->n_filters = n_filters;
  s->m_bits = m_bits;
  s->k_hashes = k_hashes;
  return s;
}

extern "C" uint64_t skpp_bank_snapshot_query(const void* snap, uint64_t m, uint64_t n,
                                             uint64_t k) {
  const Snapshot* s = static_cast<const Snapshot*>(snap);
  uint64_t mask = 0;
  for (uint32_t f = 0; f < s->n_filters; ++f) {
    uint64_t h1, h2;
    hash24(m, n, k, s->seeds[f], h1, h2);
    if (test_bits(s->bits.data() + f * s->nbytes, s->m_bits, s->k_hashes, h1, h2))
      mask |= 1ull << f;
  }
  return mask;
}

extern "C" void skpp_bank_snapshot_free(void* snap) { delete static_cast<Snapshot*>(snap); }

// ------------------------------------------------------------ sieve file ---
//   "SKPS" | u16 version=1 | u16 count | per filter: <BBBBIQIQ> header + bits | u32 crc32

extern "C" uint32_t skpp_crc32(const uint8_t* data, uint64_t len, uint32_t crc) {
  return crc32_update(crc, data, len);
}

extern "C" uint64_t skpp_bank_serialized_bytes(const skpp_filter_header_t* hdrs, uint32_t count) {
  uint64_t n = 8 + 4;
  for (uint32_t i = 0; i < count; ++i) n += kHeaderBytes + hdrs[i].m_bits / 8;
  return n;
}

extern "C" int skpp_bank_serialize(const skpp_filter_header_t* hdrs, const uint8_t* bits,
                                   uint32_t count, uint8_t* out, uint64_t cap,
                                   uint64_t* written) {
  if (!hdrs || !bits || !out || count == 0 || count > 0xFFFF) {
    set_error("bad serialize arguments");
    return SKPP_EINVAL;
  }
  const uint64_t need = skpp_bank_serialized_bytes(hdrs, count);
  if (cap < need) {
    set_error("output buffer too small");
    return SKPP_ECAPACITY;
  }
  uint8_t* p = out;
  memcpy(p, "SKPS", 4);
  put_u16(p + 4, 1);
  put_u16(p + 6, (uint16_t)count);
  p += 8;
  const uint8_t* src = bits;
  for (uint32_t i = 0; i < count; ++i) {
    const skpp_filter_header_t& h = hdrs[i];
    p[0] = h.tag;
    p[1] = h.sk_batches;
    p[2] = h.sk_first;
    p[3] = 0;
    put_u32(p + 4, h.seed);
    put_u64(p + 8, h.m_bits);
    put_u32(p + 16, h.k_hashes);
    put_u64(p + 20, h.n_inserted);
    p += kHeaderBytes;
    const uint64_t nb = h.m_bits / 8;
    memcpy(p, src, nb);
    p += nb;
    src += nb;
  }
  put_u32(p, crc32_update(0, out, (uint64_t)(p - out)));
  p += 4;
  if (written) *written = (uint64_t)(p - out);
  return SKPP_OK;
}

extern "C" int skpp_bank_parse(const uint8_t* data, uint64_t len, skpp_filter_header_t* hdrs,
                               uint64_t* bit_offsets, uint32_t cap, uint32_t* count_out) {
  if (!data && len) {
    set_error("null data");
    return SKPP_EINVAL;
  }
  if (len < 12) {
    set_error(std::to_string(len) + " bytes is too short for a sieve file");
    return SKPP_ETRUNCATED;
  }
  if (memcmp(data, "SKPS", 4) != 0) {
    set_error("bad magic, expected b'SKPS'");
    return SKPP_EBADMAGIC;
  }
  const uint32_t version = uint32_t(data[4]) | uint32_t(data[5]) << 8;
  const uint32_t count = uint32_t(data[6]) | uint32_t(data[7]) << 8;
  if (version != 1) {
    set_error("unsupported format version " + std::to_string(version) + ", expected 1");
    return SKPP_EVERSION;
  }
  if (count < 1) {
    set_error("bank must contain at least one filter");
    return SKPP_EFORMAT;
  }
  uint64_t off = 8;
  for (uint32_t i = 0; i < count; ++i) {
    if (off + kHeaderBytes > len - 4) {
      set_error("file ends inside a filter header");
      return SKPP_ETRUNCATED;
    }
    skpp_filter_header_t h;
    const uint8_t* q = data + off;
    h.tag = q[0];
    h.sk_batches = q[1];
    h.sk_first = q[2];
    h.reserved = q[3];
    h.seed = get_u32(q + 4);
    h.m_bits = load_le64(q + 8);
    h.k_hashes = get_u32(q + 16);
    h.n_inserted = load_le64(q + 20);
    off += kHeaderBytes;
    if (h.reserved != 0) {
      set_error("reserved header byte must be zero");
      return SKPP_EFORMAT;
    }
    if (h.m_bits < 64 || h.m_bits % 64 != 0) {
      set_error("invalid m_bits " + std::to_string(h.m_bits));
      return SKPP_EFORMAT;
    }
    if (h.k_hashes < 1 || h.k_hashes > kMaxHashes) {
      set_error("invalid k_hashes " + std::to_string(h.k_hashes));
      return SKPP_EFORMAT;
    }
    const uint64_t nb = h.m_bits / 8;
    if (nb > len || off + nb > len - 4) {
      set_error("file ends inside a filter bit array");
      return SKPP_ETRUNCATED;
    }
    // policy tag decode (sieve.py:184-197)
    if (h.sk_batches == 0) {
      if (h.tag != 0 && h.tag != 6) {
        set_error("unrecognized parameterless policy tag " + std::to_string(h.tag));
        return SKPP_EFORMAT;
      }
    } else if (h.tag != h.sk_batches) {
      set_error("inconsistent hybrid header: tag " + std::to_string(h.tag) + ", sk_batches " +
                std::to_string(h.sk_batches));
      return SKPP_EFORMAT;
    }
    if (i < cap) {
      if (hdrs) hdrs[i] = h;
      if (bit_offsets) bit_offsets[i] = off;
    }
    off += nb;
  }
  if (off + 4 != len) {
    set_error(std::to_string((int64_t)len - (int64_t)off - 4) + " unexpected trailing byte(s)");
    return SKPP_EFORMAT;
  }
  const uint32_t stored = get_u32(data + off);
  const uint32_t actual = crc32_update(0, data, off);
  if (stored != actual) {
    char buf[96];
    snprintf(buf, sizeof(buf), "crc mismatch: stored %#010x, computed %#010x", stored, actual);
    set_error(buf);
    return SKPP_ECHECKSUM;
  }
  if (count_out) *count_out = count;
  if (count > cap) {
    set_error("header buffer too small");
    return SKPP_ECAPACITY;
  }
  return SKPP_OK;
}
