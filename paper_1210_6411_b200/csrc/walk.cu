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
//  * finished lanes are refilled from a global queue: warp ballot/popc prefix, one
//    atomicAdd per warp, per-lane insertion -- results go to the start's own slot, so the
//    output order is the input order regardless of scheduling;
//  * the per-leg cap audit reproduces the reference's StrideError condition exactly
//    (DESIGN.md "Cap").
#include <cuda_runtime.h>

#include <algorithm>

#include "lfsr_common.cuh"
#include "lfsr_internal.h"

namespace lc {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr uint32_t kChunk = 1u << 20;  // max steps between control points (abort polling)

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
  for (uint32_t k = n >> 2; k != 0; --k) {
    step<S>(s);
    step<S>(s);
    step<S>(s);
    step<S>(s);
  }
#pragma unroll 1
  for (uint32_t k = n & 3u; k != 0; --k) step<S>(s);
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

template <class S, bool SF>
__global__ void __launch_bounds__(kWalkThreads) walk_kernel(const WalkParams p) {
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gtid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  LaneMeta* meta = p.meta + gtid * 32u;
  constexpr uint64_t kStateMask = S::NB >= 64 ? ~0ull : ((1ull << S::NB) - 1ull);

  uint32_t s[S::NB];
#pragma unroll
  for (int i = 0; i < S::NB; ++i) s[i] = 0u;
  uint32_t active = 0u, armed = 0u;
  uint64_t next_arm = kInf, next_dead = kInf;
  uint64_t t = 0;
  bool open = true;

  for (;;) {
    // ---- abort as soon as any warp has raised (StrideError / invalid start)
    const unsigned long long err = *reinterpret_cast<volatile unsigned long long*>(&p.stats[LC_ST_ERROR]);
    if (__shfl_sync(kFull, err, 0) != 0ull) break;

    // ---- refill idle lanes from the global queue (warp ballot / prefix / one atomic)
    if (open) {
      const uint32_t idle = ~active;
      const uint32_t nidle = __popc(idle);
      const uint32_t widle = __reduce_add_sync(kFull, nidle);
      if (widle != 0u && widle >= p.refill_min) {
        uint32_t incl = nidle;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const uint32_t v = __shfl_up_sync(kFull, incl, o);
          if (lane >= static_cast<uint32_t>(o)) incl += v;
        }
        unsigned long long base = 0;
        if (lane == 31u) base = atomicAdd(p.queue, static_cast<unsigned long long>(incl));
        base = __shfl_sync(kFull, base, 31);
        if (base + widle >= p.n) open = false;
        uint64_t k = base + (incl - nidle);
        uint32_t todo = idle;
        while (todo != 0u && k < p.n) {
          const int j = __ffs(todo) - 1;
          todo &= todo - 1u;
          const uint64_t x = p.starts[k] & kStateMask;  // transpose keeps nbits (bitslice.py:66-78)
          const uint32_t r1 = static_cast<uint32_t>(x & S::M1);
          const uint32_t r2 = static_cast<uint32_t>((x >> S::O2) & S::M2);
          const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
          if (r1 == 0u || r2 == 0u || r3 == 0u) {
            // SPEC.md:64 contract violation; the reference walks it to the cap
            raise_error(p.stats, LC_ERR_INVALID_STATE, k);
            ++k;
            continue;
          }
          insert_lane<S::NB>(s, j, x);
          // a start on the fixed plane whose R3 is clocked at once cannot meet R3 == F
          // again for 2^l3 - 1 clocks
          const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
          const bool safe = r3 == p.fixed_r3 && (c3 == c1 || c3 == c2);
          const uint64_t first = max(p.stride, static_cast<uint64_t>(safe ? S::WINDOW : 1ull));
          LaneMeta m;
          m.walk = k;
          m.leg_start = t;
          m.arm_at = sat_add(t, first);
          m.deadline = sat_add(t, max(p.stride, p.cap1));
          m.legs_done = 0u;
          m.pad = 0u;
          meta[j] = m;
          active |= 1u << j;
          next_arm = min(next_arm, m.arm_at);
          next_dead = min(next_dead, m.deadline);
          ++k;
        }
      }
    }
    if (!__any_sync(kFull, active != 0u)) {
      if (!open) break;
      continue;
    }

    // ---- run to the next warp-wide event horizon
    const uint64_t h = min(next_arm, next_dead);
    uint32_t rel = (h - t) > kChunk ? kChunk : static_cast<uint32_t>(h - t);
    rel = __reduce_min_sync(kFull, rel);
    const bool check = __any_sync(kFull, armed != 0u);
    uint32_t done;
    if (check) {
      done = run_checked<S, SF>(s, rel, armed, p.fixed_r3);
    } else {
      run_unchecked<S>(s, rel);
      done = rel;
    }
    t += done;

    // ---- events at clock t (rare): special nodes, arming, cap audits
    if (check) {
      uint32_t hits = special_mask<S, SF>(s, p.fixed_r3) & armed;
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
            m.arm_at = sat_add(t, S::WINDOW);
            m.deadline = sat_add(t, p.cap1);
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
    }
    if (next_arm <= t) {
      next_arm = kInf;
      for (uint32_t a = active & ~armed; a != 0u; a &= a - 1u) {
        const int j = __ffs(a) - 1;
        const uint64_t at = meta[j].arm_at;
        if (at <= t) armed |= 1u << j;
        else next_arm = min(next_arm, at);
      }
    }
    if (next_dead <= t) {
      // Cap audit: a leg still searching at its deadline raises unless it is inside a
      // run of fixed-R3 states (whose end is then its special node).
      const uint32_t on_plane = SF ? match_static<S, S::DEFAULT_F>(s) : match_runtime<S>(s, p.fixed_r3);
      next_dead = kInf;
      for (uint32_t a = active; a != 0u; a &= a - 1u) {
        const int j = __ffs(a) - 1;
        const uint64_t dl = meta[j].deadline;
        if (dl <= t) {
          if (!((on_plane >> j) & 1u)) raise_error(p.stats, LC_ERR_CAP, meta[j].walk);
          meta[j].deadline = kInf;
        } else {
          next_dead = min(next_dead, dl);
        }
      }
    }
  }
}

__global__ void init_stats_kernel(unsigned long long* st, uint64_t hist_lo, uint32_t hist_shift,
                                  uint32_t hist_bins) {
  const uint64_t words = LC_ST_HEADER + hist_bins + 2ull;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < words;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    unsigned long long v = 0;
    if (i == LC_ST_MIN || i == LC_ST_ERROR_INDEX) v = ~0ull;
    else if (i == LC_ST_HIST_LO) v = hist_lo;
    else if (i == LC_ST_HIST_SHIFT) v = hist_shift;
    else if (i == LC_ST_HIST_BINS) v = hist_bins;
    st[i] = v;
  }
}

template <class S, bool SF>
cudaError_t launch_t(const WalkParams& p, int blocks, cudaStream_t stream) {
  walk_kernel<S, SF><<<blocks, kWalkThreads, 0, stream>>>(p);
  return cudaGetLastError();
}

template <class S, bool SF>
int occupancy_t() {
  int b = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, walk_kernel<S, SF>, kWalkThreads, 0) !=
      cudaSuccess)
    return 1;
  return b > 0 ? b : 1;
}

}  // namespace

cudaError_t launch_init_stats(uint64_t* stats, uint64_t hist_lo, uint32_t hist_shift, uint32_t hist_bins,
                              cudaStream_t stream) {
  const uint64_t words = LC_ST_HEADER + hist_bins + 2ull;
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((words + 255) / 256, 1024));
  init_stats_kernel<<<g, 256, 0, stream>>>(reinterpret_cast<unsigned long long*>(stats), hist_lo, hist_shift,
                                           hist_bins);
  return cudaGetLastError();
}

cudaError_t launch_walk(SpecId id, bool static_f, const WalkParams& p, int blocks,
                        cudaStream_t stream) {
  switch (id) {
    case SpecId::A51:
      return static_f ? launch_t<A51, true>(p, blocks, stream) : launch_t<A51, false>(p, blocks, stream);
    case SpecId::MINI567:
      return static_f ? launch_t<MINI567, true>(p, blocks, stream)
                      : launch_t<MINI567, false>(p, blocks, stream);
    case SpecId::MINI789:
      return static_f ? launch_t<MINI789, true>(p, blocks, stream)
                      : launch_t<MINI789, false>(p, blocks, stream);
    default:
      return cudaErrorInvalidValue;
  }
}

int walk_blocks_per_sm(SpecId id, bool static_f) {
  switch (id) {
    case SpecId::A51: return static_f ? occupancy_t<A51, true>() : occupancy_t<A51, false>();
    case SpecId::MINI567: return static_f ? occupancy_t<MINI567, true>() : occupancy_t<MINI567, false>();
    case SpecId::MINI789: return static_f ? occupancy_t<MINI789, true>() : occupancy_t<MINI789, false>();
    default: return 1;
  }
}

}  // namespace lc
