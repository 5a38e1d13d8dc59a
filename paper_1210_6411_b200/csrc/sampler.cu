// Seeded start sets of the reference's own sampler, at native speed (host code).
//
// `random_candidate(rng, spec, params, table)` (pipeline.py:301-310) draws
// x = randrange(1, m1+1) | randrange(1, m2+1) << o2 | packed_r3 from a `random.Random`
// and rejects until `is_candidate(x)` (cipher.py:420-428).  Config 1 (2^16 starts) and
// config 2 (2^24) are defined as the first n draws of `random.Random(seed)` this way
// (SURVEY.md §8(d)), which in Python costs ~15 us per start (~4 min for 2^24).  This file
// reproduces CPython's generator bit for bit so the benchmark can build the same start
// set in ~0.3 s:
//   * `random.Random(n)` for an int n seeds MT19937 with init_by_array(key), key = the
//     32-bit little-endian words of |n| (key = [0] for n = 0) -- CPython
//     Modules/_randommodule.c random_seed / init_by_array;
//   * `randrange(1, m+1)` = 1 + _randbelow(m); _randbelow draws getrandbits(k),
//     k = m.bit_length(), until the value is < m (Lib/random.py
//     _randbelow_with_getrandbits); getrandbits(k <= 32) = genrand_uint32() >> (32 - k).
// The candidate test is the reference predicate on the fixed-R3 plane: the successor
// leaves F (cipher.py:425-426) and some clock pattern of the predecessor-table entry
// un-steps to nonzero registers (cipher.py:342-369).  Tests pin the stream against
// Python's `random` (tests/test_host.py) and the committed config-1/2 start digests.
//
// Host-side workload generation only: no kernel reads it, and the walk never calls it.
#include <cstdint>
#include <cstring>
#include <thread>
#include <vector>

#include "../../include/lfsr_b200.h"

namespace {

struct MT19937 {
  static constexpr int N = 624, M = 397;
  uint32_t mt[N];
  int mti = N + 1;

  void init_genrand(uint32_t s) {
    mt[0] = s;
    for (mti = 1; mti < N; mti++) mt[mti] = 1812433253u * (mt[mti - 1] ^ (mt[mti - 1] >> 30)) + (uint32_t)mti;
  }
  void init_by_array(const uint32_t* key, int len) {
    init_genrand(19650218u);
    int i = 1, j = 0;
    for (int k = (N > len ? N : len); k; k--) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
      i++;
      j++;
      if (i >= N) {
        mt[0] = mt[N - 1];
        i = 1;
      }
      if (j >= len) j = 0;
    }
    for (int k = N - 1; k; k--) {
      mt[i] = (mt[i] ^ ((mt[i - 1] ^ (mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
      i++;
      if (i >= N) {
        mt[0] = mt[N - 1];
        i = 1;
      }
    }
    mt[0] = 0x80000000u;
    mti = N;
  }
  void twist() {
    constexpr uint32_t UPPER = 0x80000000u, LOWER = 0x7fffffffu, A = 0x9908b0dfu;
    int kk = 0;
    for (; kk < N - M; kk++) {
      uint32_t y = (mt[kk] & UPPER) | (mt[kk + 1] & LOWER);
      mt[kk] = mt[kk + M] ^ (y >> 1) ^ ((y & 1u) ? A : 0u);
    }
    for (; kk < N - 1; kk++) {
      uint32_t y = (mt[kk] & UPPER) | (mt[kk + 1] & LOWER);
      mt[kk] = mt[kk + (M - N)] ^ (y >> 1) ^ ((y & 1u) ? A : 0u);
    }
    uint32_t y = (mt[N - 1] & UPPER) | (mt[0] & LOWER);
    mt[N - 1] = mt[M - 1] ^ (y >> 1) ^ ((y & 1u) ? A : 0u);
    mti = 0;
  }
  uint32_t next() {
    if (mti >= N) twist();
    uint32_t y = mt[mti++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
  }
};

inline int bit_length(uint64_t v) { return v ? 64 - __builtin_clzll(v) : 0; }
inline int parity(uint64_t v) { return __builtin_popcountll(v) & 1; }

struct Plane {
  int len[3], off[3], ct[3];
  uint64_t mask[3], tap[3];
};

// cipher.py:221-225 unstep_register
inline uint64_t unstep(uint64_t r, int l, uint64_t tap) {
  uint64_t low = r >> 1;
  uint64_t top = (r & 1) ^ (uint64_t)parity(low & (tap & ~(1ull << (l - 1))));
  return low | (top << (l - 1));
}

inline int majority(int a, int b, int c) { return (a & b) | (c & (a | b)); }

// is_candidate (cipher.py:420-428) for x with R3 == F already
bool plane_candidate(const Plane& P, uint64_t F, uint64_t x) {
  uint64_t r[3];
  int c[3], n[3];
  for (int k = 0; k < 3; k++) {
    r[k] = (x >> P.off[k]) & P.mask[k];
    c[k] = (int)((r[k] >> P.ct[k]) & 1);
    n[k] = (int)((r[k] >> (P.ct[k] + 1)) & 1);
  }
  // successor's R3 (clock_forward, cipher.py:228-253)
  const int maj = majority(c[0], c[1], c[2]);
  uint64_t r3n = r[2];
  if (c[2] == maj) r3n = ((r[2] << 1) & P.mask[2]) | (uint64_t)parity(r[2] & P.tap[2]);
  if (r3n == F) return false;
  // predecessors (cipher.py:342-369): a pattern p (never a single register) is
  // consistent if the majority of the predecessor's clock bits selects exactly p
  static const int kPatterns[4] = {3, 5, 6, 7};
  for (int p : kPatterns) {
    int b[3];
    for (int k = 0; k < 3; k++) b[k] = (p >> k) & 1 ? n[k] : c[k];
    const int m = majority(b[0], b[1], b[2]);
    int sel = 0;
    for (int k = 0; k < 3; k++) sel |= (b[k] == m) << k;
    if (sel != p) continue;
    bool ok = true;
    for (int k = 0; k < 3 && ok; k++)
      if ((p >> k) & 1) ok = unstep(r[k], P.len[k], P.tap[k]) != 0;
      else ok = r[k] != 0;
    if (ok) return true;
  }
  return false;
}

// Lib/random.py _randbelow_with_getrandbits(n) for 1 <= n < 2^32
inline uint64_t randbelow(MT19937& g, uint64_t n, int k) {
  uint64_t r = g.next() >> (32 - k);
  while (r >= n) r = g.next() >> (32 - k);
  return r;
}

}  // namespace

extern "C" int lc_reference_candidates(const lc_spec* spec, uint64_t fixed_r3, uint64_t seed, uint64_t n,
                                       uint64_t* out, uint64_t* draws_used) {
  if (!spec || (n && !out)) return LC_ERR_ARG;
  Plane P;
  int o = 0;
  for (int k = 0; k < 3; k++) {
    const int l = spec->lengths[k];
    if (l < 2 || l > 32 || spec->clock_taps[k] < 0 || spec->clock_taps[k] + 1 >= l) return LC_ERR_UNSUPPORTED;
    P.len[k] = l;
    P.off[k] = o;
    P.ct[k] = spec->clock_taps[k];
    P.mask[k] = (1ull << l) - 1;
    P.tap[k] = spec->tap_masks[k];
    o += l;
  }
  if (o > 64 || fixed_r3 == 0 || fixed_r3 > P.mask[2]) return LC_ERR_ARG;
  MT19937 g;
  uint32_t key[2] = {(uint32_t)seed, (uint32_t)(seed >> 32)};
  g.init_by_array(key, (seed >> 32) ? 2 : 1);
  const uint64_t m1 = P.mask[0], m2 = P.mask[1];
  const int k1 = bit_length(m1), k2 = bit_length(m2);
  const uint64_t packed = fixed_r3 << P.off[2];
  // Every draw has nonzero registers, so the verdict depends only on the six table-index
  // bits (c1 n1 c2 n2 c3 n3, cipher.py:326-339): tabulate the full predicate once.
  bool ok[64];
  for (int idx = 0; idx < 64; idx++) {
    uint64_t y = packed;
    for (int k = 0; k < 3; k++) {
      const uint64_t r = k == 2 ? fixed_r3 : 1ull << ((P.ct[k] + 2) % P.len[k]);  // any nonzero filler
      y |= (r & ~(3ull << P.ct[k])) << P.off[k];
      y &= ~(3ull << (P.off[k] + P.ct[k]));
      y |= (uint64_t)((idx >> (5 - 2 * k)) & 1) << (P.off[k] + P.ct[k]);
      y |= (uint64_t)((idx >> (4 - 2 * k)) & 1) << (P.off[k] + P.ct[k] + 1);
    }
    // R3's clock bits are fixed by F: only indices that agree with F can occur
    ok[idx] = ((y >> P.off[2]) & P.mask[2]) == fixed_r3 && plane_candidate(P, fixed_r3, y);
  }
  const int p1 = P.ct[0], p2 = P.off[1] + P.ct[1];
  const int f3 = (int)((fixed_r3 >> P.ct[2]) & 3);
  uint64_t draws = 0;
  for (uint64_t i = 0; i < n; i++) {
    for (;;) {
      const uint64_t r1 = 1 + randbelow(g, m1, k1);
      const uint64_t r2 = 1 + randbelow(g, m2, k2);
      draws++;
      const uint64_t x = r1 | (r2 << P.off[1]) | packed;
      const int idx = (int)((((x >> p1) & 1) << 5) | (((x >> (p1 + 1)) & 1) << 4) | (((x >> p2) & 1) << 3) |
                            (((x >> (p2 + 1)) & 1) << 2)) | ((f3 & 1) << 1) | (f3 >> 1);
      if (ok[idx]) {
        out[i] = x;
        break;
      }
    }
  }
  if (draws_used) *draws_used = draws;
  return LC_OK;
}

// Several independent streams (seeds[i] -> out[i*n_each ..]) on up to `threads` host
// threads: the multi-GPU bench gives every 2^24-start shard its own seed.
extern "C" int lc_reference_candidates_multi(const lc_spec* spec, uint64_t fixed_r3, const uint64_t* seeds,
                                             uint32_t count, uint64_t n_each, uint64_t* out, uint32_t threads) {
  if (!spec || (count && (!seeds || (n_each && !out)))) return LC_ERR_ARG;
  if (threads == 0) threads = 1;
  std::vector<int> rc(count, LC_OK);
  std::vector<std::thread> pool;
  for (uint32_t w = 0; w < threads && w < count; w++)
    pool.emplace_back([&, w] {
      for (uint32_t i = w; i < count; i += threads)
        rc[i] = lc_reference_candidates(spec, fixed_r3, seeds[i], n_each, out + (uint64_t)i * n_each, nullptr);
    });
  for (auto& t : pool) t.join();
  for (int r : rc)
    if (r != LC_OK) return r;
  return LC_OK;
}
