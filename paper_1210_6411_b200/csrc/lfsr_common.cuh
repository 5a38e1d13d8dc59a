// Shared device code: compile-time cipher traits, the bitsliced clock, the special-node
// mask, per-lane transposition, and the scalar transition used by the batch kernels.
//
// Bitsliced layout: a thread holds uint32_t s[NB], one 32-bit word
// per state bit.  Bit j of s[i] is bit i of lane j's packed state, so one thread walks
// 32 states; R1 = s[0, L1), R2 = s[L1, L1+L2), R3 = s[L1+L2, NB) -- the packing of
// cipher.py:90-131 turned sideways.
#pragma once

#ifndef __CUDACC_RTC__
#include <cstdint>
#endif

namespace lc {

// Compile-time cipher instance (cipher.py:173-194).  Tap masks fit 32 bits (l <= 23).
// WINDOW_: clocks after a special node before R3 can be back at F -- R3's period through
// F (2^l3 - 1 for the built-ins' maximal-period registers; runtime-specialised custom
// specs pass their own, see csrc/jit.cu).
template <int L1_, int L2_, int L3_, uint32_t T1_, uint32_t T2_, uint32_t T3_, int C1_, int C2_,
          int C3_, uint32_t DEFAULT_F_, uint64_t WINDOW_ = (1ull << L3_) - 1>
struct Spec {
  static constexpr int L1 = L1_, L2 = L2_, L3 = L3_;
  static constexpr int O2 = L1, O3 = L1 + L2, NB = L1 + L2 + L3;
  static constexpr uint32_t T1 = T1_, T2 = T2_, T3 = T3_;
  static constexpr int CT1 = C1_, CT2 = C2_, CT3 = C3_;
  static constexpr uint32_t DEFAULT_F = DEFAULT_F_;  // default_fixed_r3 (cipher.py:405-417)
  static constexpr uint64_t M1 = (1ull << L1) - 1, M2 = (1ull << L2) - 1, M3 = (1ull << L3) - 1;
  static constexpr uint64_t WINDOW = WINDOW_;  // R3 period: no candidate before this many clocks
};

// A5/1: lengths (19,22,23), taps R1{13,16,17,18} R2{20,21} R3{7,20,21,22}, clock (8,10,10)
using A51 = Spec<19, 22, 23, (1u << 13) | (1u << 16) | (1u << 17) | (1u << 18),
                 (1u << 20) | (1u << 21), (1u << 7) | (1u << 20) | (1u << 21) | (1u << 22), 8,
                 10, 10, 0x2AAA00u>;
using MINI567 = Spec<5, 6, 7, (1u << 1) | (1u << 4), (1u << 4) | (1u << 5), (1u << 5) | (1u << 6),
                     2, 2, 3, 0x22u>;
using MINI789 = Spec<7, 8, 9, (1u << 5) | (1u << 6), (1u << 3) | (1u << 4) | (1u << 5) | (1u << 7),
                     (1u << 3) | (1u << 8), 3, 3, 4, 0xaau>;

// ------------------------------------------------------------------ bitsliced clock

// Explicit LOP3s (PTX lop3.b32) so the step compiles to exactly the hand count.
// Immediates use the PTX convention a = 0xF0, b = 0xCC, c = 0xAA.
template <uint32_t IMM>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(IMM));
  return d;
}
// e ? a : b  =  (e & a) | (~e & b)
__device__ __forceinline__ uint32_t mux(uint32_t e, uint32_t a, uint32_t b) { return lop3<0xCA>(e, a, b); }
__device__ __forceinline__ uint32_t xor3(uint32_t a, uint32_t b, uint32_t c) { return lop3<0x96>(a, b, c); }

// Register k is clocked iff its clock bit equals the majority, i.e. it agrees with at
// least one of the other two: e_k = ~((c_k ^ c_i) & (c_k ^ c_j)) -- one LOP3 (0xE7).
__device__ __forceinline__ uint32_t clock_enable(uint32_t ck, uint32_t ci, uint32_t cj) {
  return lop3<0xE7>(ck, ci, cj);
}

constexpr int popcount_ce(uint32_t v) { return v ? static_cast<int>(v & 1u) + popcount_ce(v >> 1) : 0; }

// Bit 0 of a clocked register receives the XOR of its taps: r0' = e ? xor(taps) : r0.
// Taps are folded three at a time; the last fold is fused with the insert when at
// most one tap remains (2 taps: x = t0^t1^r0, r0' = r0 ^ (e & x) -- 2 LOP3).
template <uint32_t TM, int L, int OFF, int NB>
__device__ __forceinline__ uint32_t feedback_insert(const uint32_t (&s)[NB], uint32_t e) {
  constexpr int n = popcount_ce(TM);
  static_assert(n >= 1 && n <= 32, "tap count");
  uint32_t t[n > 4 ? n : 4] = {};
  int k = 0;
#pragma unroll
  for (int i = 0; i < L; ++i)
    if ((TM >> i) & 1u) t[k++] = s[OFF + i];
  const uint32_t r0 = s[OFF];
  if constexpr (n == 1) {
    return mux(e, t[0], r0);
  } else if constexpr (n == 2) {
    return lop3<0x78>(r0, e, xor3(t[0], t[1], r0));  // r0 ^ (e & (t0 ^ t1 ^ r0))
  } else if constexpr (n == 3) {
    return mux(e, xor3(t[0], t[1], t[2]), r0);
  } else if constexpr (n == 4) {
    return mux(e, lop3<0x3C>(xor3(t[0], t[1], t[2]), t[3], 0u), r0);  // 0x3C: a ^ b
  } else {  // custom specs with more taps: fold two more per LOP3
    uint32_t x = xor3(t[0], t[1], t[2]);
    int j = 3;
#pragma unroll
    for (; j + 1 < n; j += 2) x = xor3(x, t[j], t[j + 1]);
    if (j < n) x = lop3<0x3C>(x, t[j], 0u);
    return mux(e, x, r0);
  }
}

// Conditional shift of one register: lanes with e set take r[i-1] (and the feedback
// at bit 0), the others keep r[i].  One LOP3 per bit.
template <int L, int OFF, int NB>
__device__ __forceinline__ void cond_shift(uint32_t (&s)[NB], uint32_t e, uint32_t r0_new) {
#pragma unroll
  for (int i = L - 1; i > 0; --i) s[OFF + i] = mux(e, s[OFF + i - 1], s[OFF + i]);
  s[OFF] = r0_new;
}

// One majority-clocked step of 32 lanes (cipher.py:228-253 / bitslice.py:131-157):
// 3 clock-enable LOP3 + (L-1) muxes per register + the feedback XOR/insert chains,
// 72 LOP3 for A5/1.
template <class S>
__device__ __forceinline__ void step(uint32_t (&s)[S::NB]) {
  const uint32_t c1 = s[S::CT1], c2 = s[S::O2 + S::CT2], c3 = s[S::O3 + S::CT3];
  const uint32_t e1 = clock_enable(c1, c2, c3);
  const uint32_t e2 = clock_enable(c2, c1, c3);
  const uint32_t e3 = clock_enable(c3, c1, c2);
  const uint32_t n1 = feedback_insert<S::T1, S::L1, 0>(s, e1);
  const uint32_t n2 = feedback_insert<S::T2, S::L2, S::O2>(s, e2);
  const uint32_t n3 = feedback_insert<S::T3, S::L3, S::O3>(s, e3);
  cond_shift<S::L1, 0>(s, e1, n1);
  cond_shift<S::L2, S::O2>(s, e2, n2);
  cond_shift<S::L3, S::O3>(s, e3, n3);
}

// Lanes whose R3 equals the fixed value (bitslice.py:195-209 match_mask) -- an AND of
// L3 literals whose polarity is the fixed value (compile-time: LOP3 trees, ~L3/2 ops).
template <class S, uint32_t F>
__device__ __forceinline__ uint32_t match_static(const uint32_t (&s)[S::NB]) {
  uint32_t m = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < S::L3; ++i) m &= ((F >> i) & 1u) ? s[S::O3 + i] : ~s[S::O3 + i];
  return m;
}

// Same with a runtime fixed value: fm[i] = all-ones where bit i of F is 0.
template <class S>
__device__ __forceinline__ uint32_t match_runtime(const uint32_t (&s)[S::NB], uint32_t F) {
  uint32_t m = 0xffffffffu;
#pragma unroll
  for (int i = 0; i < S::L3; ++i) m &= ~(s[S::O3 + i] ^ (0u - ((F >> i) & 1u)));
  return m;
}

// Special-node lanes at the current state: R3 == F and R3 is
// clocked by the next step (so R3 leaves F); the predecessor clause is implied for any
// state reached by at least one clock.
template <class S, bool STATIC_F>
__device__ __forceinline__ uint32_t special_mask(const uint32_t (&s)[S::NB], uint32_t F) {
  const uint32_t c1 = s[S::CT1], c2 = s[S::O2 + S::CT2], c3 = s[S::O3 + S::CT3];
  const uint32_t m = STATIC_F ? match_static<S, S::DEFAULT_F>(s) : match_runtime<S>(s, F);
  return m & clock_enable(c3, c1, c2);
}

// ------------------------------------------------------------------ lane access

template <int NB>
__device__ __forceinline__ uint64_t extract_lane(const uint32_t (&s)[NB], int j) {
  uint32_t lo = 0, hi = 0;
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t b = (s[i] >> j) & 1u;
    if (i < 32) lo |= b << i;
    else hi |= b << (i - 32);
  }
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

template <int NB>
__device__ __forceinline__ void insert_lane(uint32_t (&s)[NB], int j, uint64_t x) {
  const uint32_t bit = 1u << j;
  const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
#pragma unroll
  for (int i = 0; i < NB; ++i) {
    const uint32_t v = i < 32 ? (lo >> i) & 1u : (hi >> (i - 32)) & 1u;
    s[i] = (s[i] & ~bit) | ((0u - v) & bit);
  }
}

// ------------------------------------------------------------------ scalar transition

__device__ __forceinline__ uint32_t parity32(uint32_t v) { return __popc(v) & 1u; }

template <class S>
__device__ __forceinline__ uint64_t clock_scalar(uint64_t x) {
  uint32_t r1 = static_cast<uint32_t>(x & S::M1);
  uint32_t r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
  uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
  const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
  const uint32_t maj = (c1 & c2) | (c3 & (c1 | c2));
  if (c1 == maj) r1 = ((r1 << 1) & static_cast<uint32_t>(S::M1)) | parity32(r1 & S::T1);
  if (c2 == maj) r2 = ((r2 << 1) & static_cast<uint32_t>(S::M2)) | parity32(r2 & S::T2);
  if (c3 == maj) r3 = ((r3 << 1) & static_cast<uint32_t>(S::M3)) | parity32(r3 & S::T3);
  return static_cast<uint64_t>(r1) | (static_cast<uint64_t>(r2) << S::O2) |
         (static_cast<uint64_t>(r3) << S::O3);
}

// cipher.py:221-225 unstep_register (top bit is always a tap)
template <int L, uint32_t TM>
__device__ __forceinline__ uint32_t unstep(uint32_t r) {
  const uint32_t low = r >> 1;
  const uint32_t top = (r & 1u) ^ parity32(low & (TM & ~(1u << (L - 1))));
  return low | (top << (L - 1));
}

// cipher.py:326-339 table_index: (c1, n1, c2, n2, c3, n3), c1 at bit 5
template <class S>
__device__ __forceinline__ uint32_t table_index(uint64_t x) {
  constexpr int P1 = S::CT1, P2 = S::O2 + S::CT2, P3 = S::O3 + S::CT3;
  const uint32_t c1 = (x >> P1) & 1u, n1 = (x >> (P1 + 1)) & 1u;
  const uint32_t c2 = (x >> P2) & 1u, n2 = (x >> (P2 + 1)) & 1u;
  const uint32_t c3 = (x >> P3) & 1u, n3 = (x >> (P3 + 1)) & 1u;
  return (c1 << 5) | (n1 << 4) | (c2 << 3) | (n2 << 2) | (c3 << 1) | n3;
}

// The predecessor table (cipher.py:259-313), as four 64-bit masks: bit idx of
// PATTERN_MASK[q] is set iff clock pattern CLOCK_PATTERNS[q] = {0b011, 0b101, 0b110,
// 0b111}[q] is consistent with the majority rule under inverse clocking at table index
// idx.  Restated from _consistent_patterns and evaluated at compile time, so a lookup is
// a shift of an immediate -- no divergent constant-memory access.
__host__ __device__ constexpr int clock_pattern(int q) { return q == 0 ? 3 : (q == 1 ? 5 : (q == 2 ? 6 : 7)); }

constexpr int maj_mask_ce(int c1, int c2, int c3) {
  return ((c1 == ((c1 & c2) | (c3 & (c1 | c2)))) ? 1 : 0) |
         ((c2 == ((c1 & c2) | (c3 & (c1 | c2)))) ? 2 : 0) |
         ((c3 == ((c1 & c2) | (c3 & (c1 | c2)))) ? 4 : 0);
}

constexpr uint64_t pattern_mask_ce(int q) {
  uint64_t m = 0;
  for (int idx = 0; idx < 64; ++idx) {
    const int c1 = (idx >> 5) & 1, n1 = (idx >> 4) & 1, c2 = (idx >> 3) & 1;
    const int n2 = (idx >> 2) & 1, c3 = (idx >> 1) & 1, n3 = idx & 1;
    const int p = clock_pattern(q);
    const int b1 = (p & 1) ? n1 : c1, b2 = (p & 2) ? n2 : c2, b3 = (p & 4) ? n3 : c3;
    if (maj_mask_ce(b1, b2, b3) == p) m |= 1ull << idx;
  }
  return m;
}

constexpr uint64_t kPM0 = pattern_mask_ce(0), kPM1 = pattern_mask_ce(1), kPM2 = pattern_mask_ce(2),
                   kPM3 = pattern_mask_ce(3);
constexpr uint64_t kNonEmpty = kPM0 | kPM1 | kPM2 | kPM3;
__host__ __device__ constexpr uint64_t pattern_mask(int q) {
  return q == 0 ? kPM0 : (q == 1 ? kPM1 : (q == 2 ? kPM2 : kPM3));
}
static_assert(kNonEmpty == 0xb5bf5d0db0bafdadull, "predecessor table (SURVEY.md Appendix B)");

// cipher.py:342-369 predecessors, in LUT pattern order, zero registers dropped.
template <class S>
__device__ __forceinline__ int predecessors(uint64_t x, uint64_t (&out)[4]) {
  const uint32_t idx = table_index<S>(x);
  const uint32_t r1 = static_cast<uint32_t>(x & S::M1);
  const uint32_t r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
  const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
  const uint32_t u1 = unstep<S::L1, S::T1>(r1), u2 = unstep<S::L2, S::T2>(r2),
                 u3 = unstep<S::L3, S::T3>(r3);
  int n = 0;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if ((pattern_mask(q) >> idx) & 1ull) {
      const int p = clock_pattern(q);
      const uint32_t p1 = (p & 1) ? u1 : r1, p2 = (p & 2) ? u2 : r2, p3 = (p & 4) ? u3 : r3;
      if (p1 != 0u && p2 != 0u && p3 != 0u)
        out[n++] = static_cast<uint64_t>(p1) | (static_cast<uint64_t>(p2) << S::O2) |
                   (static_cast<uint64_t>(p3) << S::O3);
    }
  }
  return n;
}

// cipher.py:420-428 is_candidate (general form, any valid or invalid x)
template <class S>
__device__ __forceinline__ bool is_candidate(uint64_t x, uint32_t F) {
  const uint64_t fmask = S::M3 << S::O3, fval = static_cast<uint64_t>(F) << S::O3;
  if ((x & fmask) != fval) return false;
  if ((clock_scalar<S>(x) & fmask) == fval) return false;
  uint64_t tmp[4];
  return predecessors<S>(x, tmp) > 0;
}

}  // namespace lc
