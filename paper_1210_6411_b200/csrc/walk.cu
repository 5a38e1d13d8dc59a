// K1: the bitsliced chain walk (step 3 of arXiv 1210.6411; replaces bitslice._run_walks,
// bitslice.py:259-323, and its callers forward_to_candidate / candidate_hops).
//
// Persistent, warp-synchronous design:
//  * every thread walks 32 lanes held bitsliced in 64 registers (lfsr_common.cuh);
//  * a warp (1024 lanes) shares one clock `t`; all control decisions are warp-uniform,
//    so the hot loops contain only the 72-LOP3 step (plus the special-node mask while
//    some lane of the warp is armed);
//  * a lane is "armed" once it may legally report a special node: clock >= stride for
//    hop 1 (bitslice.py:291-293), and never before 2^l3-1 clocks after starting on a
//    candidate (no R3 return earlier -- SURVEY.md A.3), so the mask is evaluated on a
//    small fraction of steps;
//  * per-thread control state lives in (volatile) shared memory, so only the 64 state
//    words and the step temporaries are live in the hot loops (which compile to exactly
//    72 LOP3 per step with the loop control on the uniform datapath; 20 warps per SM);
//  * work is handed out from one queue per SM sub-partition (warp scheduler): item i
//    belongs to queue i mod Q, so every scheduler ends with the same amount of work to
//    within one item, and warps steal from other queues once their own is empty;
//  * a warp refills either all 1024 lanes at once from one 1024-start item (warp ballot
//    32x32 transposes of coalesced loads) or single idle lanes (ballot / popc prefix /
//    one atomic per warp) -- results go to the start's own slot, so the output order is
//    the input order regardless of scheduling;
//  * the per-leg cap audit reproduces the reference's StrideError condition exactly
//    (DESIGN.md "Cap").
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>

#include <algorithm>
#endif

#include "lfsr_common.cuh"
#include "lfsr_internal.h"
#ifndef __CUDACC_RTC__
#include "jit.h"
#endif

namespace lc {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kChunk = 1u << 20;  // max steps between control points (abort polling)
constexpr int kQueueStride = 16;       // u64 words between queue counters (128 B)

// Clocks after a special node before R3 can be back at F: the spec's compile-time period
// (2^l3 - 1 for the built-ins), or, for runtime-compiled custom specs (Spec WINDOW 0),
// the period of R3's cycle through F computed on the host (WalkParams::window).
template <class S>
__device__ __forceinline__ uint64_t window_of(const WalkParams& p) {
  return S::WINDOW ? S::WINDOW : p.window;
}

#ifndef LC_WALK_UNROLL
#define LC_WALK_UNROLL 16  // steps per unchecked-loop iteration (same-box A/B: 16 > 4 > 8 by ~0.3 %)
#endif

#ifndef LC_WALK_MIN_BLOCKS
#define LC_WALK_MIN_BLOCKS 5  // 5 x 128 threads: 20 warps/SM -> <= 102 registers, spill-free hot loops
#endif

__device__ __forceinline__ uint64_t sat_add(uint64_t a, uint64_t b) {
  const uint64_t c = a + b;
  return c < a ? kInf : c;
}

__device__ __forceinline__ void raise_error(unsigned long long* st, int code, uint64_t index) {
  atomicCAS(&st[LC_ST_ERROR], 0ull, static_cast<unsigned long long>(-code));
  atomicMin(&st[LC_ST_ERROR_INDEX], static_cast<unsigned long long>(index));
}

// One finished hop: edge counters, exact u128 sum of squared deviations, histogram.
__device__ void record_edge(const WalkParams& p, uint64_t d) {
  unsigned long long* st = p.stats;
  atomicAdd(&st[LC_ST_EDGES], 1ull);
  atomicAdd(&st[LC_ST_TRANSITIONS], static_cast<unsigned long long>(d));
  atomicMin(&st[LC_ST_MIN], static_cast<unsigned long long>(d));
  atomicMax(&st[LC_ST_MAX], static_cast<unsigned long long>(d));
  const uint64_t dev = d >= p.hist_lo ? d - p.hist_lo : p.hist_lo - d;
  const uint64_t lo = dev * dev, hi = __umul64hi(dev, dev);
  const unsigned long long old = atomicAdd(&st[LC_ST_SQ_LO], static_cast<unsigned long long>(lo));
  const uint64_t carry = (old + lo < old) ? 1u : 0u;
  if (hi + carry) atomicAdd(&st[LC_ST_SQ_HI], static_cast<unsigned long long>(hi + carry));
  uint64_t bin;
  if (d < p.hist_lo) {
    bin = 0;
  } else {
    const uint64_t b = (d - p.hist_lo) >> p.hist_shift;
    bin = b >= p.hist_bins ? p.hist_bins + 1ull : b + 1ull;
  }
  atomicAdd(&st[LC_ST_HEADER + bin], 1ull);
}

template <class S>
__device__ __forceinline__ void run_unchecked(uint32_t (&s)[S::NB], uint32_t n) {
#pragma unroll 1
  for (uint32_t k = n / LC_WALK_UNROLL; k != 0; --k) {
#pragma unroll
    for (int u = 0; u < LC_WALK_UNROLL; ++u) step<S>(s);
  }
#pragma unroll 1
  for (uint32_t k = n % LC_WALK_UNROLL; k != 0; --k) step<S>(s);
}

// Steps until a special node shows up in an armed lane of the warp (returns the number
// of steps taken; the state is then the special node itself) or n steps are done.
template <class S, bool SF>
__device__ __forceinline__ uint32_t run_checked(uint32_t (&s)[S::NB], uint32_t n, uint32_t armed,
                                                uint32_t F) {
  uint32_t k = 0;
#pragma unroll 1
  for (; k < n; ++k) {
    if (__any_sync(kFull, (special_mask<S, SF>(s, F) & armed) != 0u)) break;
    step<S>(s);
  }
  return k;
}

// Warp-uniform view of the error word.
__device__ __forceinline__ bool raise_pending(const WalkParams& p) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long*>(&p.stats[LC_ST_ERROR]);
  return __shfl_sync(kFull, e, 0) != 0ull;
}

// Items in queue q (items i with i mod nq == q).
__device__ __forceinline__ uint64_t queue_len(uint64_t items, uint32_t nq, uint32_t q) {
  return items > q ? (items - q + nq - 1) / nq : 0;
}

// Take up to m items, own queue first, then steal.  Lane 0 only.  Returns the count;
// the items are (base + j) * nq + qi for j < count.
__device__ uint32_t take_items(const WalkParams& p, uint64_t items, uint32_t own, uint32_t m,
                               uint32_t* qi_out, uint64_t* base_out) {
  for (uint32_t i = 0; i < p.nq; ++i) {
    const uint32_t qi = own + i < p.nq ? own + i : own + i - p.nq;
    const uint64_t len = queue_len(items, p.nq, qi);
    unsigned long long* ctr = p.queues + static_cast<uint64_t>(qi) * kQueueStride;
    if (i != 0) {
      if (*reinterpret_cast<volatile unsigned int*>(p.exhausted)) break;
      if (*reinterpret_cast<volatile unsigned long long*>(ctr) >= len) continue;
    }
    const uint64_t b = atomicAdd(ctr, static_cast<unsigned long long>(m));
    if (b < len) {
      *qi_out = qi;
      *base_out = b;
      return static_cast<uint32_t>(len - b < m ? len - b : m);
    }
  }
  atomicExch(p.exhausted, 1u);
  return 0;
}

// Special registers read with asm volatile so the compiler re-reads them after the hot
// loops instead of keeping copies live across them.
__device__ __forceinline__ uint32_t tid_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t ctaid_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(r));
  return r;
}

// Per-block control state in shared memory.  Everything the outer loop needs after a
// hot loop is re-read from here, so only the 64 state words (plus the uniform step
// counter) are live in the hot loops.
struct WalkShared {
  uint32_t active[kWalkThreads];            // lanes walking
  uint32_t armed[kWalkThreads];             // lanes allowed to report a special node
  unsigned long long next_arm[kWalkThreads];
  unsigned long long next_dead[kWalkThreads];
  unsigned long long t[kWalkThreads / 32];  // warp clock
  uint32_t own[kWalkThreads / 32];          // warp scheduler queue
  uint32_t open[kWalkThreads / 32];         // queues not yet exhausted for this warp
  uint32_t warp_mode;                       // 1: whole-warp refill (1024-start items)
  uint32_t refill_min;                      // lane mode: refill at this many idle lanes
  uint32_t park;                            // this launch parks drained warps (lane mode only)
  unsigned long long n;                     // items in this launch (p.n, or *p.n_dev)
};

constexpr uint32_t kWarpItem = 1024;  // starts per queue item in whole-warp mode

template <class S, bool SF>
__device__ __forceinline__ void whole_warp_refill(const WalkParams& p, volatile WalkShared& sh,
                                                  uint32_t (&s)[S::NB]) {
  constexpr uint64_t kStateMask = S::NB >= 64 ? ~0ull : ((1ull << S::NB) - 1ull);
  const uint32_t tid = tid_x(), lane = tid & 31u, w = tid >> 5;
  const uint64_t gtid = static_cast<uint64_t>(ctaid_x()) * kWalkThreads + tid;
  const uint64_t items = (p.n + kWarpItem - 1) / kWarpItem;
  const uint64_t t = sh.t[w];
  uint32_t qi = 0, got = 0;
  uint64_t b = 0;
  if (lane == 0) got = take_items(p, items, sh.own[w], 1u, &qi, &b);
  got = __shfl_sync(kFull, got, 0);
  if (got == 0u) {
    if (lane == 0) sh.open[w] = 0u;
    __syncwarp();
    return;
  }
  qi = __shfl_sync(kFull, qi, 0);
  b = __shfl_sync(kFull, b, 0);
  const uint64_t base = ((b * p.nq) + qi) * kWarpItem;
  const uint64_t wbase = gtid - lane;  // first thread of this warp
  bool all_safe = true;
  for (uint32_t r = 0; r < 32u; ++r) {
    const uint64_t k = base + r * 32u + lane;
    uint64_t x = 0;
    bool valid = false;
    if (k < p.n) {
      x = p.starts[k] & kStateMask;  // transpose keeps nbits (bitslice.py:66-78)
      const uint32_t r1 = static_cast<uint32_t>(x & S::M1);
      const uint32_t r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
      const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
      if (r1 == 0u || r2 == 0u || r3 == 0u) {
        raise_error(p.stats, LC_ERR_INVALID_STATE, k);
        x = 0;
      } else {
        valid = true;
        const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
        all_safe = all_safe && r3 == p.fixed_r3 && (c3 == c1 || c3 == c2);
        LaneMeta m;
        m.walk = k;
        m.leg_start = t;
        m.arm_at = 0;    // set by the owning thread below
        m.deadline = 0;  // (identical for every lane of the item)
        m.legs_done = 0u;
        m.pad = 0u;
        LC_CHECK(k < p.n);
        p.meta[(wbase + r) * 32u + lane] = m;
      }
    }
    const uint32_t vmask = __ballot_sync(kFull, valid);
    const uint32_t lo = static_cast<uint32_t>(x), hi = static_cast<uint32_t>(x >> 32);
#pragma unroll
    for (int i = 0; i < S::NB; ++i) {
      const uint32_t wd = __ballot_sync(kFull, ((i < 32 ? lo >> i : hi >> (i - 32)) & 1u) != 0u);
      if (lane == r) s[i] = wd;
    }
    if (lane == r) sh.active[tid] = vmask;
  }
  // a start on the fixed plane whose R3 is clocked at once cannot meet R3 == F again
  // for 2^l3 - 1 clocks
  all_safe = __all_sync(kFull, all_safe);
  const uint64_t first = max(p.stride, static_cast<uint64_t>(all_safe ? window_of<S>(p) : 1ull));
  const uint64_t arm = sat_add(t, first), dead = sat_add(t, max(p.stride, p.cap1));
  __syncwarp();
  LaneMeta* const meta = p.meta + gtid * 32u;
  const uint32_t act = sh.active[tid];
  for (uint32_t a = act; a != 0u; a &= a - 1u) {
    const int j = __ffs(a) - 1;
    meta[j].arm_at = arm;
    meta[j].deadline = dead;
  }
  sh.armed[tid] = 0u;
  sh.next_arm[tid] = act ? arm : kInf;
  sh.next_dead[tid] = act ? dead : kInf;
  __syncwarp();
}

template <class S, bool SF>
__device__ __forceinline__ void lane_refill(const WalkParams& p, volatile WalkShared& sh,
                                            uint32_t (&s)[S::NB]) {
  constexpr uint64_t kStateMask = S::NB >= 64 ? ~0ull : ((1ull << S::NB) - 1ull);
  const uint32_t tid = tid_x(), lane = tid & 31u, w = tid >> 5;
  const uint64_t gtid = static_cast<uint64_t>(ctaid_x()) * kWalkThreads + tid;
  LaneMeta* const meta = p.meta + gtid * 32u;
  const uint64_t items = sh.n;  // chunk == 1: item == start index
  const uint64_t t = sh.t[w];
  for (;;) {
    const uint32_t idle = ~sh.active[tid];
    const uint32_t nidle = __popc(idle);
    const uint32_t widle = __reduce_add_sync(kFull, nidle);
    if (widle == 0u || widle < sh.refill_min) break;
    uint32_t qi = 0, got = 0;
    uint64_t b = 0;
    if (lane == 0) got = take_items(p, items, sh.own[w], widle, &qi, &b);
    got = __shfl_sync(kFull, got, 0);
    if (got == 0u) {
      if (lane == 0) sh.open[w] = 0u;
      __syncwarp();
      break;
    }
    qi = __shfl_sync(kFull, qi, 0);
    b = __shfl_sync(kFull, b, 0);
    uint32_t incl = nidle;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t v = __shfl_up_sync(kFull, incl, o);
      if (lane >= static_cast<uint32_t>(o)) incl += v;
    }
    uint32_t j_item = incl - nidle;  // this thread's first item offset
    uint32_t active = sh.active[tid];
    uint64_t next_arm = sh.next_arm[tid], next_dead = sh.next_dead[tid];
    for (uint32_t todo = idle; todo != 0u && j_item < got; todo &= todo - 1u, ++j_item) {
      const int j = __ffs(todo) - 1;
      const uint64_t k = (b + j_item) * p.nq + qi;
      if (p.resume) {
        // a parked lane: same leg, clocks re-based on this warp's clock (mod 2^64)
        LC_CHECK(k < sh.n);
        const ResumeRec rec = p.resume[k];
        insert_lane<S::NB>(s, j, rec.state);
        LaneMeta m;
        m.walk = rec.walk;
        m.leg_start = t - rec.elapsed;
        m.arm_at = sat_add(t, rec.arm_rel);
        m.deadline = rec.dead_rel == kInf ? kInf : sat_add(t, rec.dead_rel);
        m.legs_done = rec.legs_done;
        m.pad = rec.pad;
        meta[j] = m;
        active |= 1u << j;
        next_arm = min(next_arm, m.arm_at);
        next_dead = min(next_dead, m.deadline);
        continue;
      }
      LC_CHECK(k < p.n);
      const uint64_t x = p.starts[k] & kStateMask;
      const uint32_t r1 = static_cast<uint32_t>(x & S::M1);
      const uint32_t r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
      const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
      if (r1 == 0u || r2 == 0u || r3 == 0u) {
        raise_error(p.stats, LC_ERR_INVALID_STATE, k);
        continue;
      }
      insert_lane<S::NB>(s, j, x);
      const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
      const bool safe = r3 == p.fixed_r3 && (c3 == c1 || c3 == c2);
      LaneMeta m;
      m.walk = k;
      m.leg_start = t;
      m.arm_at = sat_add(t, max(p.stride, static_cast<uint64_t>(safe ? window_of<S>(p) : 1ull)));
      m.deadline = sat_add(t, max(p.stride, p.cap1));
      m.legs_done = 0u;
      m.pad = 0u;
      meta[j] = m;
      active |= 1u << j;
      next_arm = min(next_arm, m.arm_at);
      next_dead = min(next_dead, m.deadline);
    }
    sh.active[tid] = active;
    sh.next_arm[tid] = next_arm;
    sh.next_dead[tid] = next_dead;
    if (raise_pending(p)) break;
  }
}

// Lane parking: once the queues are drained, a warp whose live lanes fall below
// park_below exports them (state + leg bookkeeping relative to its clock) to the pool and
// retires; the host relaunches on the pool with the lanes packed densely, so warps stay
// full through the tail of wide-spread walks (random starts, several hops).
template <class S>
__device__ __forceinline__ bool park_lanes(const WalkParams& p, volatile WalkShared& sh, const uint32_t (&s)[S::NB]) {
  const uint32_t tid = tid_x(), lane = tid & 31u, w = tid >> 5;
  const uint64_t gtid = static_cast<uint64_t>(ctaid_x()) * kWalkThreads + tid;
  const LaneMeta* const meta = p.meta + gtid * 32u;
  const uint64_t t = sh.t[w];
  const uint32_t act = sh.active[tid], armed = sh.armed[tid];
  const uint32_t cnt = __popc(act);
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFull, incl, o);
    if (lane >= static_cast<uint32_t>(o)) incl += v;
  }
  // reserve the warp's slots only if they fit in the pool (else the warp keeps walking)
  unsigned long long base = 0;
  uint32_t fits = 1u;
  if (lane == 31u) {
    unsigned long long old = atomicAdd(p.pool_count, 0ull);
    for (;;) {
      if (old + incl > p.pool_cap) {
        fits = 0u;
        break;
      }
      const unsigned long long prev = atomicCAS(p.pool_count, old, old + incl);
      if (prev == old) break;
      old = prev;
    }
    base = old;
  }
  if (!__shfl_sync(kFull, fits, 31)) return false;
  base = __shfl_sync(kFull, base, 31) + (incl - cnt);
  for (uint32_t a = act; a != 0u; a &= a - 1u, ++base) {
    const int j = __ffs(a) - 1;
    const LaneMeta m = meta[j];
    ResumeRec r;
    r.state = extract_lane<S::NB>(s, j);
    r.walk = m.walk;
    r.elapsed = t - m.leg_start;
    r.arm_rel = ((armed >> j) & 1u) || m.arm_at <= t ? 0ull : m.arm_at - t;
    r.dead_rel = m.deadline == kInf ? kInf : (m.deadline > t ? m.deadline - t : 0ull);
    r.legs_done = m.legs_done;
    r.pad = m.pad;  // cap deadline already excused once
    LC_CHECK(base < p.pool_cap);
    p.pool[base] = r;
  }
  sh.active[tid] = 0u;
  __syncwarp();
  return true;
}

// Arm (check every step) once R3 is this close to F.  Whole-warp mode: lanes of a warp
// walk in step and are checked together from the first armed one, so re-arming only pays
// while it skips a long stretch (stride-1 walks: 2.8e6 checked steps per walk otherwise);
// lane mode: lanes are independent, so a tight bound pays.
constexpr uint64_t kArmSlackWarp = 1u << 16, kArmSlackLane = 1u << 10;
constexpr uint64_t kArmBatch = 1u << 12;
constexpr uint64_t kRunSlack = 128;  // clocks granted to finish a fixed-R3 run at the cap audit  // re-arm lanes due this soon in the same event

// R3 of lane j (bits o3 .. o3 + l3 - 1 of its state).
template <class S>
__device__ __forceinline__ uint32_t lane_r3(const uint32_t (&s)[S::NB], int j) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < S::L3; ++i) r |= ((s[S::O3 + i] >> j) & 1u) << i;
  return r;
}

// Events at the warp clock (rare): special nodes, arming, cap audits.
template <class S, bool SF, bool RA>
__device__ __forceinline__ void handle_events(const WalkParams& p, volatile WalkShared& sh,
                                              const uint32_t (&s)[S::NB]) {
  const uint32_t tid = tid_x(), w = tid >> 5;
  const uint64_t gtid = static_cast<uint64_t>(ctaid_x()) * kWalkThreads + tid;
  LaneMeta* const meta = p.meta + gtid * 32u;
  const uint64_t t = sh.t[w];
  const uint32_t F = p.fixed_r3;
  uint32_t active = sh.active[tid], armed = sh.armed[tid];
  uint64_t next_arm = sh.next_arm[tid], next_dead = sh.next_dead[tid];
  uint32_t hits = special_mask<S, SF>(s, F) & armed;
  if (hits != 0u) {
    while (hits != 0u) {
      const int j = __ffs(hits) - 1;
      hits &= hits - 1u;
      const uint32_t bit = 1u << j;
      LaneMeta m = meta[j];
      const uint64_t d = t - m.leg_start;
      const uint64_t o = m.walk * p.legs + m.legs_done;
      p.dst[o] = extract_lane<S::NB>(s, j);
      p.dist[o] = d;
      record_edge(p, d);
      armed &= ~bit;
      if (++m.legs_done >= p.legs) {
        active &= ~bit;
        m.arm_at = kInf;
        m.deadline = kInf;
      } else {
        // the lane continues from the candidate it reached (bitslice.py:313-315)
        m.leg_start = t;
        m.arm_at = sat_add(t, window_of<S>(p));
        m.deadline = sat_add(t, p.cap1);
        m.pad = 0u;
      }
      meta[j] = m;
    }
    next_arm = kInf;
    next_dead = kInf;
    for (uint32_t a = active; a != 0u; a &= a - 1u) {
      const int j = __ffs(a) - 1;
      if (!((armed >> j) & 1u)) next_arm = min(next_arm, meta[j].arm_at);
      next_dead = min(next_dead, meta[j].deadline);
    }
  }
  if (next_arm <= t) {
    // A lane due for arming first bounds its next possible special node: R3 reaches F
    // only after need3[R3] more R3 clocks, at most one per step, so nothing can be
    // reported before t + need3[R3].  Far-off lanes are re-armed there instead of being
    // checked every step (the bound tightens ~4x per round, R3 clocking on ~3/4 of the
    // steps); lanes due within kArmBatch are handled in the same event.
    next_arm = kInf;
    const uint64_t slack = RA ? (sh.warp_mode ? kArmSlackWarp : kArmSlackLane) : 0u;
    for (uint32_t a = active & ~armed; a != 0u; a &= a - 1u) {
      const int j = __ffs(a) - 1;
      uint64_t at = meta[j].arm_at;
      if (RA && at <= t + kArmBatch) {
        const uint64_t need = p.need3 ? p.need3[lane_r3<S>(s, j)] : 0u;
        if (need > slack && t + need > at) {
          at = t + need;
          meta[j].arm_at = at;
        }
      }
      if (at <= t) armed |= 1u << j;
      else next_arm = min(next_arm, at);
    }
  }
  if (next_dead <= t) {
    // Cap audit: a leg still searching at its deadline raises unless it is inside a run
    // of fixed-R3 states (whose end is then its special node).
    const uint32_t on_plane = SF ? match_static<S, S::DEFAULT_F>(s) : match_runtime<S>(s, F);
    next_dead = kInf;
    for (uint32_t a = active; a != 0u; a &= a - 1u) {
      const int j = __ffs(a) - 1;
      const uint64_t dl = meta[j].deadline;
      if (dl <= t) {
        // Excused once: the run of fixed-R3 states ends within kRunSlack clocks (R3
        // stays put only while R1 and R2 both clock with clock bits equal to each other,
        // and a maximal-period register repeats a bit at most L times in a row), and its
        // last state is the special node (its predecessor is the previous state).  A lane
        // still searching at the excused deadline raises like any other.
        if (!((on_plane >> j) & 1u) || meta[j].pad) {
          raise_error(p.stats, LC_ERR_CAP, meta[j].walk);
          meta[j].deadline = kInf;
        } else {
          meta[j].pad = 1u;
          meta[j].deadline = t + kRunSlack;
          next_dead = min(next_dead, t + kRunSlack);
        }
      } else {
        next_dead = min(next_dead, dl);
      }
    }
  }
  sh.active[tid] = active;
  sh.armed[tid] = armed;
  sh.next_arm[tid] = next_arm;
  sh.next_dead[tid] = next_dead;
}

template <class S, bool SF, bool RA>
__global__ void __launch_bounds__(kWalkThreads, LC_WALK_MIN_BLOCKS) walk_kernel(const WalkParams p) {
  // auto mode launches both variants; the one not meant for the probed mode exits
  if (p.run_if_mode != ~0u && *p.mode_word != p.run_if_mode) return;
  // resume round sized on the device: only the blocks its parked lanes fill run, so the
  // lanes stay packed into few warps (the grid covers the bound, not the count)
  if (p.n_dev && static_cast<uint64_t>(ctaid_x()) * (kWalkThreads * 32ull) >= *p.n_dev) return;
  __shared__ WalkShared sh_storage;
  volatile WalkShared& sh = sh_storage;
  {
    const uint32_t tid = tid_x(), lane = tid & 31u, w = tid >> 5;
    sh.active[tid] = 0u;
    sh.armed[tid] = 0u;
    sh.next_arm[tid] = kInf;
    sh.next_dead[tid] = kInf;
    if (lane == 0) {
      uint32_t own = 0;
      if (p.nq > 1) {  // this warp's scheduler queue
        uint32_t smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        own = (static_cast<uint32_t>(p.smsp_map[smid & 1023u]) * 4u + (w & 3u)) % p.nq;
      }
      sh.own[w] = own;
      sh.t[w] = 0ull;
      sh.open[w] = 1u;
    }
    if (tid == 0) {
      const uint32_t warp_mode = p.mode_word ? *p.mode_word : (p.chunk > 1u ? 1u : 0u);
      sh.warp_mode = warp_mode;
      sh.refill_min = warp_mode ? kWarpItem : p.refill_min;
      const uint64_t n = p.n_dev ? *p.n_dev : p.n;
      sh.n = n;
      // whole-warp walks end together (near-constant lengths): nothing to pack
      sh.park = p.pool != nullptr && !warp_mode && n > p.park_min;
    }
    __syncthreads();
  }

  uint32_t s[S::NB];
#pragma unroll
  for (int i = 0; i < S::NB; ++i) s[i] = 0u;

  for (;;) {
    // ---- abort as soon as any warp has raised (StrideError / invalid start)
    if (raise_pending(p)) break;

    // ---- refill idle lanes
    uint32_t rel, armed;
    {
      const uint32_t tid = tid_x(), w = tid >> 5;
      if (sh.open[w]) {
        if (sh.warp_mode) {
          if (__all_sync(kFull, sh.active[tid] == 0u)) whole_warp_refill<S, SF>(p, sh, s);
        } else {
          lane_refill<S, SF>(p, sh, s);
        }
      }
      if (!__any_sync(kFull, sh.active[tid] != 0u)) {
        if (!sh.open[w]) break;
        continue;
      }
      if (sh.park && !sh.open[w] &&
          __reduce_add_sync(kFull, static_cast<uint32_t>(__popc(sh.active[tid]))) < p.park_below) {
        if (park_lanes<S>(p, sh, s)) break;
      }
      // ---- next warp-wide event horizon
      const uint64_t t = sh.t[w];
      const uint64_t h = min(sh.next_arm[tid], sh.next_dead[tid]);
      rel = (h - t) > kChunk ? kChunk : static_cast<uint32_t>(h - t);
      rel = __reduce_min_sync(kFull, rel);
      armed = sh.armed[tid];
    }

    // ---- hot loops: only s[], the step count and (checked) the armed mask are live
    uint32_t done;
    if (__any_sync(kFull, armed != 0u)) {
      done = run_checked<S, SF>(s, rel, armed, p.fixed_r3);
    } else {
      run_unchecked<S>(s, rel);
      done = rel;
    }
    {
      const uint32_t tid = tid_x(), lane = tid & 31u, w = tid >> 5;
      __syncwarp();
      if (lane == 0) sh.t[w] = sh.t[w] + done;
      __syncwarp();
    }
    handle_events<S, SF, RA>(p, sh, s);
  }
}

__global__ void init_stats_kernel(unsigned long long* st, uint64_t hist_lo, uint32_t hist_shift,
                                  uint32_t hist_bins, unsigned long long* queues, uint32_t nq,
                                  unsigned int* exhausted) {
  const uint64_t words = LC_ST_HEADER + hist_bins + 2ull;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t i0 = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  for (uint64_t i = i0; st && i < words; i += stride) {  // st null: queues only (resume round)
    unsigned long long v = 0;
    if (i == LC_ST_MIN || i == LC_ST_ERROR_INDEX) v = ~0ull;
    else if (i == LC_ST_HIST_LO) v = hist_lo;
    else if (i == LC_ST_HIST_SHIFT) v = hist_shift;
    else if (i == LC_ST_HIST_BINS) v = hist_bins;
    st[i] = v;
  }
  if (queues)
    for (uint64_t q = i0; q < nq; q += stride) queues[q * kQueueStride] = 0ull;
  if (exhausted && i0 == 0) *exhausted = 0u;
}

__global__ void smid_probe_kernel(unsigned int* flags) {
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  if (threadIdx.x == 0) flags[smid & 1023u] = 1u;
}

// Auto refill mode: whole-warp refill iff every start is on the fixed plane with R3
// clocked at once (the window-safe starts of a special-node walk).  *mode must be 1 on
// entry; any other start clears it.
template <class S>
__global__ void mode_probe_kernel(const uint64_t* __restrict__ starts, uint64_t n, uint32_t F, uint32_t* mode) {
  constexpr uint64_t kStateMask = S::NB >= 64 ? ~0ull : ((1ull << S::NB) - 1ull);
  bool ok = true;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t x = starts[i] & kStateMask;
    const uint32_t r1 = static_cast<uint32_t>(x & S::M1), r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
    const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
    const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
    ok = ok && r3 == F && (c3 == c1 || c3 == c2);
  }
  if (!__all_sync(0xffffffffu, ok) && (threadIdx.x & 31) == 0) *mode = 0u;
}

#ifndef __CUDACC_RTC__  // host launchers (csrc/jit.cu compiles the device code alone)
template <class S, bool SF>
cudaError_t launch_t(const WalkParams& p, bool rearm, int blocks, cudaStream_t stream) {
  if (rearm) walk_kernel<S, SF, true><<<blocks, kWalkThreads, 0, stream>>>(p);
  else walk_kernel<S, SF, false><<<blocks, kWalkThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

template <class S, bool SF>
int occupancy_t() {
  int a = 0, b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&a, walk_kernel<S, SF, false>, kWalkThreads, 0) !=
          cudaSuccess ||
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, walk_kernel<S, SF, true>, kWalkThreads, 0) != cudaSuccess)
    return 1;
  const int m = a < b ? a : b;
  return m > 0 ? m : 1;
}

#endif

}  // namespace

#ifndef __CUDACC_RTC__

cudaError_t launch_init_stats(uint64_t* stats, uint64_t hist_lo, uint32_t hist_shift, uint32_t hist_bins,
                              unsigned long long* queues, uint32_t nq, unsigned int* exhausted,
                              cudaStream_t stream) {
  const uint64_t words = std::max<uint64_t>(LC_ST_HEADER + hist_bins + 2ull, nq);
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((words + 255) / 256, 1024));
  init_stats_kernel<<<g, 256, 0, stream>>>(reinterpret_cast<unsigned long long*>(stats), hist_lo, hist_shift,
                                           hist_bins, queues, nq, exhausted);
  return cudaGetLastError();
}

cudaError_t probe_smids(int sms, unsigned int* d_flags, cudaStream_t stream) {
  smid_probe_kernel<<<sms * 16, 32, 0, stream>>>(d_flags);
  return cudaGetLastError();
}

cudaError_t launch_mode_probe(SpecId id, const uint64_t* starts, uint64_t n, uint32_t F, uint32_t* mode_word,
                              cudaStream_t stream) {
  cudaError_t e = cudaMemsetAsync(mode_word, 0, sizeof(uint32_t), stream);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(mode_word, 1, 1, stream);  // little-endian: word = 1
  if (e != cudaSuccess) return e;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 4096));
  switch (id) {
    case SpecId::A51: mode_probe_kernel<A51><<<g ? g : 1, 256, 0, stream>>>(starts, n, F, mode_word); break;
    case SpecId::MINI567: mode_probe_kernel<MINI567><<<g ? g : 1, 256, 0, stream>>>(starts, n, F, mode_word); break;
    case SpecId::MINI789: mode_probe_kernel<MINI789><<<g ? g : 1, 256, 0, stream>>>(starts, n, F, mode_word); break;
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return cudaErrorInvalidValue;
      return jit_launch(c->mode_probe, g ? g : 1, 256, 0, stream, starts, n, F, mode_word);
    }
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_walk(SpecId id, bool static_f, bool rearm, const WalkParams& p, int blocks,
                        cudaStream_t stream) {
  switch (id) {
    case SpecId::A51:
      return static_f ? launch_t<A51, true>(p, rearm, blocks, stream) : launch_t<A51, false>(p, rearm, blocks, stream);
    case SpecId::MINI567:
      return static_f ? launch_t<MINI567, true>(p, rearm, blocks, stream)
                      : launch_t<MINI567, false>(p, rearm, blocks, stream);
    case SpecId::MINI789:
      return static_f ? launch_t<MINI789, true>(p, rearm, blocks, stream)
                      : launch_t<MINI789, false>(p, rearm, blocks, stream);
    case SpecId::CUSTOM: {  // runtime-compiled for the spec, runtime F (csrc/jit.cu)
      const CustomKernels* c = current_custom();
      if (!c) return cudaErrorInvalidValue;
      return jit_launch(rearm ? c->walk_rearm : c->walk_plain, blocks, kWalkThreads, 0, stream, p);
    }
    default:
      return cudaErrorInvalidValue;
  }
}

int walk_blocks_per_sm(SpecId id, bool static_f) {
  switch (id) {
    case SpecId::A51: return static_f ? occupancy_t<A51, true>() : occupancy_t<A51, false>();
    case SpecId::MINI567: return static_f ? occupancy_t<MINI567, true>() : occupancy_t<MINI567, false>();
    case SpecId::MINI789: return static_f ? occupancy_t<MINI789, true>() : occupancy_t<MINI789, false>();
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return 1;
      const int a = jit_blocks_per_sm(c->walk_plain, kWalkThreads), b = jit_blocks_per_sm(c->walk_rearm, kWalkThreads);
      return a < b ? a : b;
    }
    default: return 1;
  }
}

#endif  // !__CUDACC_RTC__

}  // namespace lc
