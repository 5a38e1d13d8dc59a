/*
 * TEST INFRASTRUCTURE ONLY -- fast CPU checker for large A5/1 golden sets.
 *
 * A second, independent restatement of the step-3 walk for A5/1 (bitslice.py:259-323,
 * legs = 1), used only to produce the committed config-2 digests
 * (tests/golden/a51_c2_digests.json, oracle/gen_golden.py c2): 2^24 walks of ~1.1e7
 * clocks are ~1.9e14 transitions, 8 h for the reference-structured port
 * (lfsr_oracle.c) on this container's cores, ~30 min here.  It is pinned against the
 * reference-produced config-1 set (65,536 walks, tests/golden/a51_c1_65536.json) and the
 * 256-walk KAT before its output is trusted (oracle/gen_golden.py c2 refuses otherwise).
 *
 * Semantics (restating bitslice.py:286-323): from start s_0,
 *   dist = min{ t >= max(stride, 1) : R3(s_t) == F  and  R3 is clocked by the next step },
 *   dest = s_dist,
 * with s_{t+1} = clock_forward(s_t) (cipher.py:228-253).  A lane whose leg passes
 * max_clocks + 1 clocks without an edge is reported as a cap error (StrideError).
 *
 * Layout: 512 lanes per group, one __m512i per state bit (bit j of word i = bit i of
 * lane j).  Lanes walk in lockstep; a group ends when its slowest lane finds its edge
 * (special-node starts have near-constant chain lengths, sigma/mu ~ 1.6e-4).
 * Built with -mavx512f for the build container only (Makefile target `walk512`); the GPU
 * box never loads it.
 */
#include <immintrin.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define W512_OK 0
#define W512_CAP 1

/* A5/1 (cipher.py:173-178): R1 bits 0-18, R2 19-40, R3 41-63 */
#define O2 19
#define O3 41
#define C1 8
#define C2 (O2 + 10)
#define C3 (O3 + 10)

typedef __m512i V;
#define TL(a, b, c, imm) _mm512_ternarylogic_epi64((a), (b), (c), (imm))
#define MUX 0xCA  /* a ? b : c */
#define ENB 0xE7  /* ~((a ^ b) & (a ^ c)): a agrees with the majority */
#define X3 0x96   /* a ^ b ^ c */

/* One majority-clocked step of 512 lanes (cipher.py:228-253). */
static inline __attribute__((always_inline)) void step(V *s, V *e3_out) {
    const V c1 = s[C1], c2 = s[C2], c3 = s[C3];
    const V e1 = TL(c1, c2, c3, ENB);
    const V e2 = TL(c2, c1, c3, ENB);
    const V e3 = TL(c3, c1, c2, ENB);
    *e3_out = e3;
    /* feedback = parity of the taps, before shifting (R1 {13,16,17,18}, R2 {20,21},
       R3 {7,20,21,22}) */
    const V f1 = _mm512_xor_si512(TL(s[13], s[16], s[17], X3), s[18]);
    const V f2 = _mm512_xor_si512(s[O2 + 20], s[O2 + 21]);
    const V f3 = _mm512_xor_si512(TL(s[O3 + 7], s[O3 + 20], s[O3 + 21], X3), s[O3 + 22]);
#pragma GCC unroll 32
    for (int i = 18; i >= 1; i--) s[i] = TL(e1, s[i - 1], s[i], MUX);
    s[0] = TL(e1, f1, s[0], MUX);
#pragma GCC unroll 32
    for (int i = 21; i >= 1; i--) s[O2 + i] = TL(e2, s[O2 + i - 1], s[O2 + i], MUX);
    s[O2] = TL(e2, f2, s[O2], MUX);
#pragma GCC unroll 32
    for (int i = 22; i >= 1; i--) s[O3 + i] = TL(e3, s[O3 + i - 1], s[O3 + i], MUX);
    s[O3] = TL(e3, f3, s[O3], MUX);
}

/* lanes whose R3 equals F and whose R3 the next step clocks */
static inline V special(const V *s, uint32_t F) {
    V acc = _mm512_set1_epi64(-1);
    for (int i = 0; i < 23; i++) {
        const V lit = ((F >> i) & 1) ? s[O3 + i] : _mm512_xor_si512(s[O3 + i], _mm512_set1_epi64(-1));
        acc = _mm512_and_si512(acc, lit);
    }
    const V c1 = s[C1], c2 = s[C2], c3 = s[C3];
    return _mm512_and_si512(acc, TL(c3, c1, c2, ENB));
}

static uint64_t lane_state(const V *s, int lane) {
    uint64_t x = 0;
    for (int i = 0; i < 64; i++) {
        uint64_t w[8];
        _mm512_storeu_si512((void *)w, s[i]);
        x |= ((w[lane >> 6] >> (lane & 63)) & 1ull) << i;
    }
    return x;
}

static int walk_group(uint32_t F, const uint64_t *starts, int lanes, uint64_t stride, uint64_t max_clocks,
                      uint64_t *dst, uint64_t *dist) {
    V s[64];
    uint64_t w[64][8];
    memset(w, 0, sizeof w);
    for (int j = 0; j < lanes; j++)
        for (int i = 0; i < 64; i++) w[i][j >> 6] |= ((starts[j] >> i) & 1ull) << (j & 63);
    for (int i = 0; i < 64; i++) s[i] = _mm512_loadu_si512((const void *)w[i]);
    uint64_t pending[8];
    for (int q = 0; q < 8; q++) {
        const int lo = q * 64;
        pending[q] = lanes >= lo + 64 ? ~0ull : (lanes > lo ? (1ull << (lanes - lo)) - 1 : 0);
    }
    const uint64_t first = stride > 1 ? stride : 1;
    uint64_t t = 0;
    V e3;
    for (; t + 8 <= first; t += 8)
        for (int u = 0; u < 8; u++) step(s, &e3);
    for (; t < first; t++) step(s, &e3);
    const uint64_t cap = max_clocks + 1;
    for (;;) {
        uint64_t m[8];
        _mm512_storeu_si512((void *)m, special(s, F));
        int left = 0;
        for (int q = 0; q < 8; q++) {
            uint64_t hit = m[q] & pending[q];
            while (hit) {
                const int b = __builtin_ctzll(hit);
                hit &= hit - 1;
                const int lane = q * 64 + b;
                dst[lane] = lane_state(s, lane);
                dist[lane] = t;
                pending[q] &= ~(1ull << b);
            }
            left |= pending[q] != 0;
        }
        if (!left) return W512_OK;
        if (t >= cap) return W512_CAP;
        step(s, &e3);
        t++;
    }
}

/* Walk n starts; returns W512_OK or W512_CAP (first failing start in *bad). */
int w512_walk(uint32_t fixed_r3, const uint64_t *starts, uint64_t n, uint64_t stride, uint64_t max_clocks,
              uint64_t *dst, uint64_t *dist, uint64_t *bad) {
    const int64_t groups = (int64_t)((n + 511) / 512);
    int rc = W512_OK;
    uint64_t first_bad = n;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t g = 0; g < groups; g++) {
        const uint64_t lo = (uint64_t)g * 512;
        const int lanes = (int)((n - lo) < 512 ? (n - lo) : 512);
        if (walk_group(fixed_r3, starts + lo, lanes, stride, max_clocks, dst + lo, dist + lo) != W512_OK) {
#pragma omp critical
            {
                rc = W512_CAP;
                if (lo < first_bad) first_bad = lo;
            }
        }
    }
    if (bad) *bad = first_bad;
    return rc;
}
