// Batch kernels around the walk: the special-node predicate and predecessor batch
// (cipher.py:342-428), fixed-count clocking (bitslice.clock_sliced), the closed-form
// enumeration of step 1 (K2, pipeline.enumerate_candidates), the seeded start-set
// generator (K0, ordered compaction), the step-2 prune (K3,
// pipeline.prune_shallow_segments) and the closure check of build_skeleton_edges.
#ifndef __CUDACC_RTC__
#include <cuda_runtime.h>

#include <cstdlib>
#endif

#include "lfsr_common.cuh"
#include "lfsr_internal.h"
#ifndef __CUDACC_RTC__
#include "jit.h"
#endif

namespace lc {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kThreads = 256;

template <class S>
__global__ void is_candidate_kernel(const uint64_t* __restrict__ xs, uint64_t n, uint32_t F,
                                    uint8_t* __restrict__ out) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[i] = is_candidate<S>(xs[i], F) ? 1 : 0;
}

template <class S>
__global__ void predecessors_kernel(const uint64_t* __restrict__ xs, uint64_t n,
                                    uint64_t* __restrict__ out, uint8_t* __restrict__ count) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    uint64_t p[4] = {0, 0, 0, 0};
    const int c = predecessors<S>(xs[i], p);
    ulonglong2* o = reinterpret_cast<ulonglong2*>(out + 4 * i);
    o[0] = make_ulonglong2(p[0], p[1]);
    o[1] = make_ulonglong2(p[2], p[3]);
    count[i] = static_cast<uint8_t>(c);
  }
}

// bitslice.clock_sliced: 32 states per thread, bitsliced, t unchecked steps.
template <class S>
__global__ void clock_kernel(const uint64_t* __restrict__ xs, uint64_t n, uint64_t t,
                             uint64_t* __restrict__ out) {
  const uint64_t base = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) * 32u;
  if (base >= n) return;
  const int lanes = static_cast<int>(n - base < 32u ? n - base : 32u);
  uint32_t s[S::NB];
#pragma unroll
  for (int i = 0; i < S::NB; ++i) s[i] = 0u;
  for (int j = 0; j < lanes; ++j) insert_lane<S::NB>(s, j, xs[base + j]);
  for (uint64_t left = t; left != 0;) {
    const uint32_t c = left > (1u << 30) ? (1u << 30) : static_cast<uint32_t>(left);
#pragma unroll 1
    for (uint32_t k = 0; k < c; ++k) step<S>(s);
    left -= c;
  }
  for (int j = 0; j < lanes; ++j) out[base + j] = extract_lane<S::NB>(s, j);
}

// ---------------------------------------------------------------- ordered compaction
// Index space [0, total) -> state via a generator; states passing is_candidate are
// written densely in index order.  Pass 1 counts per tile, pass 2 scans the tile counts,
// pass 3 re-evaluates and writes with a warp-ballot / block prefix (coalesced stores).

constexpr int kTileShift = 16;
constexpr uint64_t kTile = 1ull << kTileShift;
constexpr int kCompactThreads = 256;

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// K0: trial i -> h = splitmix64(seed + (i + 1) * golden); r1 = 1 + lo32(h) * m1 >> 32,
// r2 = 1 + hi32(h) * m2 >> 32, R3 = F.  (Restated in oracle/k0.py for parity.)
template <class S>
struct RandGen {
  uint64_t seed;
  uint64_t packed_f;
  __device__ __forceinline__ uint64_t operator()(uint64_t i) const {
    const uint64_t h = splitmix64(seed + (i + 1u) * 0x9E3779B97F4A7C15ull);
    const uint64_t r1 = 1u + (((h & 0xffffffffull) * S::M1) >> 32);
    const uint64_t r2 = 1u + (((h >> 32) * S::M2) >> 32);
    return r1 | (r2 << S::O2) | packed_f;
  }
};

template <class S, class Gen>
__global__ void __launch_bounds__(kCompactThreads) compact_count_kernel(Gen g, uint64_t total,
                                                                        uint32_t F,
                                                                        uint64_t* __restrict__ tile_counts) {
  const uint64_t lo = blockIdx.x * kTile;
  const uint64_t hi = min(total, lo + kTile);
  uint32_t c = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += kCompactThreads) c += is_candidate<S>(g(i), F) ? 1u : 0u;
  c = __reduce_add_sync(kFull, c);
  __shared__ uint32_t part[kCompactThreads / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t sum = 0;
    for (int w = 0; w < kCompactThreads / 32; ++w) sum += part[w];
    tile_counts[blockIdx.x] = sum;
  }
}

// Exclusive scan of tile counts in place; counts[tiles] = total.  One block.
__global__ void scan_kernel(uint64_t* __restrict__ counts, uint64_t tiles, uint64_t* __restrict__ total_out) {
  __shared__ uint64_t part[1024];
  const uint64_t per = (tiles + blockDim.x - 1) / blockDim.x;
  const uint64_t lo = threadIdx.x * per, hi = min(tiles, lo + per);
  uint64_t sum = 0;
  for (uint64_t i = lo; i < hi; ++i) sum += counts[i];
  part[threadIdx.x] = sum;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t run = 0;
    for (uint32_t w = 0; w < blockDim.x; ++w) {
      const uint64_t v = part[w];
      part[w] = run;
      run += v;
    }
    counts[tiles] = run;
    if (total_out) *total_out = run;
  }
  __syncthreads();
  uint64_t run = part[threadIdx.x];
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t v = counts[i];
    counts[i] = run;
    run += v;
  }
}

template <class S, class Gen>
__global__ void __launch_bounds__(kCompactThreads) compact_write_kernel(Gen g, uint64_t total,
                                                                        uint32_t F,
                                                                        const uint64_t* __restrict__ offsets,
                                                                        uint64_t* __restrict__ out,
                                                                        uint64_t cap) {
  __shared__ uint32_t wcount[kCompactThreads / 32];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t lo = blockIdx.x * kTile;
  const uint64_t hi = min(total, lo + kTile);
  uint64_t pos = offsets[blockIdx.x];
  for (uint64_t r = lo; r < hi; r += kCompactThreads) {
    const uint64_t i = r + threadIdx.x;
    uint64_t x = 0;
    bool ok = false;
    if (i < hi) {
      x = g(i);
      ok = is_candidate<S>(x, F);
    }
    const uint32_t b = __ballot_sync(kFull, ok);
    if (lane == 0) wcount[warp] = __popc(b);
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kCompactThreads / 32; ++w) {
      const uint32_t v = wcount[w];
      before += (static_cast<uint32_t>(w) < warp) ? v : 0u;
      all += v;
    }
    if (ok) {
      const uint64_t o = pos + before + __popc(b & ((1u << lane) - 1u));
      if (o < cap) out[o] = x;
    }
    pos += all;
    __syncthreads();
  }
}

#ifndef __CUDACC_RTC__
template <class S, class Gen>
cudaError_t compact(Gen g, uint64_t total, uint32_t F, uint64_t* out, uint64_t cap, uint64_t* d_count,
                    uint64_t* scratch, cudaStream_t stream, int* launches) {
  const uint64_t tiles = (total + kTile - 1) / kTile;
  if (tiles == 0) {
    cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(uint64_t), stream);
    return e;
  }
  compact_count_kernel<S, Gen><<<static_cast<unsigned>(tiles), kCompactThreads, 0, stream>>>(g, total, F, scratch);
  scan_kernel<<<1, 1024, 0, stream>>>(scratch, tiles, d_count);
  compact_write_kernel<S, Gen><<<static_cast<unsigned>(tiles), kCompactThreads, 0, stream>>>(g, total, F, scratch,
                                                                                          out, cap);
  if (launches) *launches += 3;
  return cudaGetLastError();
}
#endif

// ---------------------------------------------------------------- K2: step-1 enumeration
// On the fixed-R3 plane the special-node predicate (cipher.py:420-428) depends only on
// four bits: R1's clock bit and the bit above it (c1, n1) and the same pair of R2
// (c2, n2) -- R3's pair (c3, n3) is fixed.  A candidate needs R3 clocked by the next
// step (c3 agrees with c1 or c2; R3 then leaves F because a maximal-period step has no
// nonzero fixed point) and a non-empty predecessor-table entry (kNonEmpty).  So for an
// R2 row the candidates are exactly the R1 values whose bits (ct1, ct1+1) form an allowed
// pattern p: runs of 2^ct1 consecutive R1 values, in ascending order.  Each output slot
// has a closed-form state, so the kernel is a pure coalesced stream of 8-byte stores
// (HBM-write bound) -- the same set and order as pipeline.enumerate_candidates
// (pipeline.py:104-118), checked against the reference's digests.

// Allowed R1 patterns p = c1 | n1 << 1 (bit p of the result) for an R2 class q = c2 | n2 << 1.
__device__ __forceinline__ uint32_t allowed_patterns(uint32_t q, uint32_t c3, uint32_t n3) {
  const uint32_t c2 = q & 1u, n2 = q >> 1;
  uint32_t a = 0;
#pragma unroll
  for (uint32_t p = 0; p < 4; ++p) {
    const uint32_t c1 = p & 1u, n1 = p >> 1;
    const uint32_t idx = (c1 << 5) | (n1 << 4) | (c2 << 3) | (n2 << 2) | (c3 << 1) | n3;
    if ((c3 == c1 || c3 == c2) && ((kNonEmpty >> idx) & 1ull)) a |= 1u << p;
  }
  return a;
}

// Candidates in one R2 row of class a: |a| * 2^(l1-2) R1 values, minus R1 = 0 if p = 0 is allowed.
template <class S>
__device__ __forceinline__ uint64_t row_count(uint32_t a) {
  return static_cast<uint64_t>(__popc(a)) * (1ull << (S::L1 - 2)) - (a & 1u);
}

// Number of r in [0, n) with ((r >> ct) & 3) == q.
__device__ __forceinline__ uint64_t class_count(uint64_t n, uint32_t q, int ct) {
  const uint64_t blk = 1ull << ct;
  const uint64_t rem = n & ((blk << 2) - 1), lo = q * blk;
  return (n >> (ct + 2)) * blk + (rem > lo ? min(rem - lo, blk) : 0ull);
}

// Candidates with R2 in [r2_lo, r2).
template <class S>
__device__ __forceinline__ uint64_t plane_offset(uint64_t r2_lo, uint64_t r2, uint32_t c3, uint32_t n3) {
  uint64_t off = 0;
#pragma unroll
  for (uint32_t q = 0; q < 4; ++q)
    off += row_count<S>(allowed_patterns(q, c3, n3)) * (class_count(r2, q, S::CT2) - class_count(r2_lo, q, S::CT2));
  return off;
}

// R1 value of virtual slot v of a row of class a (v counts the R1 = 0 slot when p = 0
// is allowed): run v >> ct1 is pattern rank (run mod |a|) of high part run / |a|.
template <class S>
__device__ __forceinline__ uint32_t slot_r1(uint64_t v, uint32_t a, uint32_t na) {
  constexpr int CT1 = S::CT1;
  const uint32_t run = static_cast<uint32_t>(v >> CT1), low = static_cast<uint32_t>(v) & ((1u << CT1) - 1u);
  const uint32_t high = run / na, rank = run - high * na;
  uint32_t p = a;
  if (rank >= 1u) p &= p - 1u;
  if (rank >= 2u) p &= p - 1u;
  if (rank >= 3u) p &= p - 1u;
  return (high << (CT1 + 2)) | (static_cast<uint32_t>(__ffs(p) - 1) << CT1) | low;
}

// Blocks take equal work units (2^16 virtual slots of one R2 row).  A unit's output range
// is written as 32-byte aligned quads of states with 256-bit stores (plus up to three
// single head / tail slots), four quads per lane per iteration so each thread keeps four
// stores in flight: a warp covers 512 consecutive slots per iteration, which span at most
// three R1 runs when a run has >= 256 values (A5/1), so the runs' (high part, pattern)
// cost one warp-uniform division per 512 slots and a select per slot.  Minis (short runs)
// use the per-slot form.
template <class S>
__global__ void __launch_bounds__(256) enumerate_plane_kernel(uint64_t r2_lo, uint64_t r2_hi, uint32_t F,
                                                              uint64_t* __restrict__ out, uint64_t cap,
                                                              uint64_t* __restrict__ d_count) {
  constexpr int CT1 = S::CT1;
  constexpr uint32_t kLowMask = (1u << CT1) - 1u;
#ifndef LC_K2_QUADS
#define LC_K2_QUADS 4
#endif
  constexpr int kU = LC_K2_QUADS;  // 32-byte quads per lane per iteration (a warp covers 128 * kU slots)
  constexpr int kSpan = (128 * kU + 255) / 256 + 1;  // runs a chunk can touch (A5/1 runs: 256)
  // work units: a row's virtual slots in equal pieces, so blocks get equal work whatever
  // the row's pattern count (1..4 runs per 2^(ct1+2) R1 values)
  constexpr uint64_t kRowSlots = 1ull << S::L1;  // >= any row's virtual slot count
  constexpr uint64_t kUnitSlots = kRowSlots >= (1ull << 16) ? (1ull << 16) : kRowSlots;
  constexpr uint64_t kUnitsPerRow = kRowSlots / kUnitSlots;
  constexpr bool kFast = (1u << CT1) >= 256u;  // then a chunk spans at most 3 runs
  const uint32_t c3 = (F >> S::CT3) & 1u, n3 = (F >> (S::CT3 + 1)) & 1u;
  const uint64_t packed_f = static_cast<uint64_t>(F) << S::O3;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  if (blockIdx.x == 0 && threadIdx.x == 0) *d_count = plane_offset<S>(r2_lo, r2_hi, c3, n3);
  const uint64_t units = (r2_hi - r2_lo) * kUnitsPerRow;
  for (uint64_t unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const uint64_t r2 = r2_lo + unit / kUnitsPerRow;
    const uint64_t u_lo = (unit % kUnitsPerRow) * kUnitSlots;  // this unit's virtual slots
    const uint32_t a = allowed_patterns((r2 >> S::CT2) & 3u, c3, n3);
    const uint32_t na = __popc(a);
    const uint64_t skip = a & 1u;  // virtual slot 0 is R1 = 0 (not a state) when p = 0 is allowed
    const uint64_t row_end = skip + row_count<S>(a);
    if (na == 0 || u_lo >= row_end) continue;
    const uint64_t v_end = min(row_end, u_lo + kUnitSlots);
    const uint64_t base = plane_offset<S>(r2_lo, r2, c3, n3);  // first output slot of the row
    const uint64_t row_bits = (r2 << S::O2) | packed_f;
    const uint64_t g0 = base - skip;  // output slot of virtual slot v is g0 + v
    uint64_t v_first = max(skip, u_lo);
    // head: single slots up to a 32-byte boundary (at most 3), one thread each
    const uint64_t to_align = (4u - ((g0 + v_first) & 3u)) & 3u;
    const uint32_t head = static_cast<uint32_t>(to_align < v_end - v_first ? to_align : v_end - v_first);
    if (threadIdx.x < head) {
      const uint64_t v = v_first + threadIdx.x, slot = g0 + v;
      if (slot < cap) out[slot] = row_bits | slot_r1<S>(v, a, na);
    }
    v_first += head;
    const uint64_t nquads = (v_end - v_first) >> 2;
    const uint32_t tail = static_cast<uint32_t>((v_end - v_first) & 3u);
    if (threadIdx.x < tail) {  // tail: at most 3 single slots
      const uint64_t v = v_first + 4 * nquads + threadIdx.x, slot = g0 + v;
      if (slot < cap) out[slot] = row_bits | slot_r1<S>(v, a, na);
    }
    uint32_t prank[4];
    {
      uint32_t m = a;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        prank[k] = m ? static_cast<uint32_t>(__ffs(m) - 1) : 0u;
        m &= m - 1u;
      }
    }
    for (uint64_t it = warp; it * (32 * kU) < nquads; it += nwarps) {
      const uint64_t vbase = v_first + it * (128 * kU);
      uint32_t pre[kSpan] = {}, run0 = 0;
      if constexpr (kFast) {  // the chunk spans runs run0 .. run0 + kSpan - 1
        run0 = static_cast<uint32_t>(vbase >> CT1);
        uint32_t high = run0 / na, rank = run0 - high * na;
#pragma unroll
        for (int r = 0; r < kSpan; ++r) {
          const uint32_t p = rank == 0 ? prank[0] : rank == 1 ? prank[1] : rank == 2 ? prank[2] : prank[3];
          pre[r] = (high << (CT1 + 2)) | (p << CT1);
          if (++rank == na) {
            rank = 0;
            ++high;
          }
        }
      }
      uint64_t val[kU][4];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t v = vbase + 128 * u + 4 * lane;
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (kFast) {
            const uint32_t dd = static_cast<uint32_t>((v + e) >> CT1) - run0;
            uint32_t qq = pre[0];
#pragma unroll
            for (int r = 1; r < kSpan; ++r) qq = dd == static_cast<uint32_t>(r) ? pre[r] : qq;
            val[u][e] = row_bits | (qq | (static_cast<uint32_t>(v + e) & kLowMask));
          } else {
            val[u][e] = row_bits | slot_r1<S>(v + e, a, na);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const uint64_t k = it * (32 * kU) + 32 * u + lane;  // quad index
        const uint64_t slot = g0 + vbase + 128 * u + 4 * lane;  // 32-byte aligned
        if (k < nquads) {
          if (slot + 3 < cap) {
#if __CUDACC_VER_MAJOR__ > 12 || (__CUDACC_VER_MAJOR__ == 12 && __CUDACC_VER_MINOR__ >= 9)
            asm volatile("st.global.v4.b64 [%0], {%1, %2, %3, %4};" ::"l"(out + slot), "l"(val[u][0]),
                         "l"(val[u][1]), "l"(val[u][2]), "l"(val[u][3])
                         : "memory");
#else  // 256-bit stores need PTX ISA 8.8 (a runtime compiler older than CUDA 12.9): two 128-bit
            asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(out + slot), "l"(val[u][0]), "l"(val[u][1])
                         : "memory");
            asm volatile("st.global.v2.b64 [%0], {%1, %2};" ::"l"(out + slot + 2), "l"(val[u][2]), "l"(val[u][3])
                         : "memory");
#endif
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e)
              if (slot + e < cap) out[slot + e] = val[u][e];
          }
        }
      }
    }
  }
}

// ---------------------------------------------------------------- K3: step-2 prune
// Thread per candidate, depth-first traversal of the candidate's segment (the reverse
// tree through predecessors that are not candidates, pipeline.py:121-129).  The pop
// order of the reference's LIFO stack (pipeline.py:132-144) is a preorder that visits
// children in reverse LUT order; it is replayed with a per-lane ring of pending branch
// points (shared memory, spilling to global memory), so the order-dependent `expanded`
// counter matches exactly.  BFS mode (pipeline.py:147-160) only needs the segment size
// capped at node_limit + 1, which is order-independent.

// The predecessor table as 64 nibbles (bit q of a nibble = pattern q consistent), packed
// in four 64-bit immediates and indexed by the three (clock bit, bit above) pairs taken as
// they sit in the state -- pair k at bits 2k..2k+1, clock bit low -- so the index is three
// 2-bit field extracts instead of table_index's six bit moves.
constexpr int std_index_ce(int pidx) {
  const int c1 = pidx & 1, n1 = (pidx >> 1) & 1, c2 = (pidx >> 2) & 1, n2 = (pidx >> 3) & 1;
  const int c3 = (pidx >> 4) & 1, n3 = (pidx >> 5) & 1;
  return (c1 << 5) | (n1 << 4) | (c2 << 3) | (n2 << 2) | (c3 << 1) | n3;
}
constexpr uint64_t pnibble_word_ce(int w) {
  uint64_t v = 0;
  for (int k = 0; k < 16; ++k)
    for (int q = 0; q < 4; ++q)
      if ((pattern_mask(q) >> std_index_ce(16 * w + k)) & 1ull) v |= 1ull << (4 * k + q);
  return v;
}
constexpr uint64_t kPNib0 = pnibble_word_ce(0), kPNib1 = pnibble_word_ce(1), kPNib2 = pnibble_word_ce(2),
                   kPNib3 = pnibble_word_ce(3);

template <class S>
__device__ __forceinline__ uint32_t pattern_set_of(uint64_t x) {
  const uint32_t pidx = static_cast<uint32_t>((x >> S::CT1) & 3u) |
                        (static_cast<uint32_t>((x >> (S::O2 + S::CT2)) & 3u) << 2) |
                        (static_cast<uint32_t>((x >> (S::O3 + S::CT3)) & 3u) << 4);
  const uint64_t w = pidx < 32 ? (pidx < 16 ? kPNib0 : kPNib1) : (pidx < 48 ? kPNib2 : kPNib3);
  return static_cast<uint32_t>(w >> ((pidx & 15u) << 2)) & 15u;
}

// Child q of the node y: y's predecessor under clock pattern CLOCK_PATTERNS[q], the
// registers of the pattern unstepped (cipher.py:342-369).
template <class S>
__device__ __forceinline__ uint64_t child_of(uint64_t y, int q) {
  const uint32_t r1 = static_cast<uint32_t>(y & S::M1), r2 = static_cast<uint32_t>((y >> S::O2) & S::M2),
                 r3 = static_cast<uint32_t>((y >> S::O3) & S::M3);
  const int p = clock_pattern(q & 3);
  const uint32_t p1 = (p & 1) ? unstep<S::L1, S::T1>(r1) : r1, p2 = (p & 2) ? unstep<S::L2, S::T2>(r2) : r2,
                 p3 = (p & 4) ? unstep<S::L3, S::T3>(r3) : r3;
  return static_cast<uint64_t>(p1) | (static_cast<uint64_t>(p2) << S::O2) | (static_cast<uint64_t>(p3) << S::O3);
}

// Pending branch points of a lane's traversal: a ring of the R deepest nodes that
// still have unvisited (lower) children, in shared memory ([slot][thread], conflict-free),
// backed by a per-lane spill ring in global memory for the older ones.  Backtracking
// pops the deepest entry and jumps straight to its next child instead of climbing the
// path one forward clock (and one re-expansion) per level.  Only when the spill ring
// overflows are the oldest entries dropped; once ring and spill run empty the traversal
// falls back to the stackless climb, which rediscovers them (and empty ring and spill
// without drops mean the traversal is complete -- no climb back to the root).
// Ring depth is a template parameter: deep rings spill less (the spill round trip sits
// on a lane's critical path, which bounds the tail of small batches), shallow rings fit
// more warps per SM (throughput over large batches); launch_prune picks per batch size.
#ifndef LC_PRUNE_THREADS
#define LC_PRUNE_THREADS 128
#endif
#ifndef LC_PRUNE_RING_WIDE
#define LC_PRUNE_RING_WIDE 20
#endif
constexpr int kRingDeep = 32, kRingWide = LC_PRUNE_RING_WIDE;
constexpr int kPruneThreads = LC_PRUNE_THREADS;  // a ring of R entries takes R * 10 B per thread of shared memory
constexpr uint64_t kDepthCap = 1u << 12;  // ring entries hold depths below this (12-bit field)
constexpr int kTailBurst = 32;  // steps per warp vote once no candidate is left to take
#ifndef LC_PRUNE_BULK_BURST
#define LC_PRUNE_BULK_BURST 4
#endif
constexpr int kBulkBurst = LC_PRUNE_BULK_BURST;  // steps per warp vote while candidates remain

template <int R>
struct Ring {
  uint64_t* node;  // [R][kPruneThreads]: the branch node
  uint16_t* dm;    //                         depth << 4 | remaining child mask
  uint64_t* snode; // this lane's spill ring in global memory (older entries), [scap]
  uint16_t* sdm;
  uint32_t top, cnt, scnt, scap, sbase;  // spill entry k (0 = oldest) at (sbase + k) mod scap
  bool lost;
  __device__ __forceinline__ uint32_t at(uint32_t slot) const { return slot * kPruneThreads + threadIdx.x; }
  __device__ __forceinline__ void push(uint64_t y, uint64_t d, uint32_t mask) {
    if (d >= kDepthCap) return;  // no room for the depth: found again by climbing (see prune_step)
    const uint32_t next = top + 1 == static_cast<uint32_t>(R) ? 0u : top + 1;
    if (cnt == R) {  // full: the oldest entry (about to be overwritten) moves to the spill ring
      if (scap) {
        if (scnt == scap) {  // spill full too: drop its oldest entry (the climb recovers it)
          sbase = sbase + 1 == scap ? 0u : sbase + 1;
          --scnt;
          lost = true;
        }
        const uint32_t k = sbase + scnt < scap ? sbase + scnt : sbase + scnt - scap;
        snode[k] = node[at(next)];
        sdm[k] = dm[at(next)];
        ++scnt;
      } else {
        lost = true;
      }
    } else {
      ++cnt;
    }
    top = next;
    node[at(top)] = y;
    dm[at(top)] = static_cast<uint16_t>((static_cast<uint32_t>(d) << 4) | mask);
  }
};

// Children of x in the segment, as a pattern mask: x's predecessors (cipher.py:342-369)
// minus special nodes (pipeline.py:121-129).  Two facts keep this short: predecessors of
// a valid state never have a zero register (unstep is a bijection fixing 0), and a child
// c's successor is x itself, so is_candidate(c) (cipher.py:420-428) = R3(c) == F &&
// R3(x) != F && preds(c) != {} -- only patterns that unstep R3 can land on the plane, and
// only when unstep(R3(x)) == F (then R3(x) != F automatically); that rare case pays for
// the children's table lookups.
template <class S>
__device__ __forceinline__ uint32_t child_mask(uint64_t x, uint32_t F) {
  uint32_t m = pattern_set_of<S>(x);
  const uint32_t r3 = static_cast<uint32_t>((x >> S::O3) & S::M3);
  if (unstep<S::L3, S::T3>(r3) == F) {
#pragma unroll
    for (int q = 1; q < 4; ++q)
      if (((m >> q) & 1u) && ((kNonEmpty >> table_index<S>(child_of<S>(x, q))) & 1ull)) m &= ~(1u << q);
  }
  return m;
}

// One traversal step of a candidate's segment: exactly one node expansion per step for
// every lane.  State: x (the node to expand next), d (its depth), acc (expanded for dfs /
// node count for bfs), climb (x's subtree is finished and the ring lost entries: this
// step expands x's parent to find x's next-lower sibling -- rare).  The two common cases
// (descend into x's highest child; or, at a leaf, resume the deepest pending branch
// point) only pick the source node and child index, then share one child computation,
// so a warp's lanes diverge only over a few selects and the ring access.
// Returns 0 while running, 1 = finished shallow, 2 = finished deep (not shallow).
template <class S, int R>
__device__ __forceinline__ int prune_step(uint64_t& x, uint64_t& d, uint64_t& acc, bool& climb, Ring<R>& ring,
                                          uint32_t F, int mode, uint64_t limit) {
  uint64_t src = x;
  uint32_t q = 0;
  bool finished;  // x's subtree is done: continue from the ring (or climb)
  if (!climb) {
    const uint32_t m = child_mask<S>(x, F);
    finished = m == 0u;
    if (!finished) {
      if (mode == 0) {
        if (d >= limit) {  // a child would sit below the depth limit
          acc += 1;
          return 2;
        }
        acc += __popc(m);
      } else {
        acc += __popc(m);
        if (acc > limit) {
          acc = limit + 1;
          return 2;
        }
      }
      q = 31 - __clz(m);  // the reference pops the last child first
      const uint32_t rest = m & ~(1u << q);
      if (rest) ring.push(x, d, rest);
      ++d;
    }
  } else {
    // x's parent y: continue with x's next-lower sibling, else y's subtree is done too.
    // x's child index follows from which registers differ between x and y (the clocked
    // ones: a maximal-period register step has no nonzero fixed point), so no child of y
    // has to be built to find it.
    const uint64_t y = clock_scalar<S>(x);
    const uint64_t diff = x ^ y;
    const uint32_t pat = ((diff & S::M1) ? 1u : 0u) | (((diff >> S::O2) & S::M2) ? 2u : 0u) |
                         (((diff >> S::O3) & S::M3) ? 4u : 0u);
    const uint32_t k = pat == 3u ? 0u : pat == 5u ? 1u : pat == 6u ? 2u : 3u;  // clock_pattern^-1
    const uint32_t lower = child_mask<S>(y, F) & ((1u << k) - 1u);
    finished = lower == 0u;
    if (finished) {
      x = y;
      --d;
    } else {
      q = 31 - __clz(lower);
      const uint32_t rest = lower & ~(1u << q);
      if (rest) ring.push(y, d - 1, rest);
      src = y;
      climb = false;
    }
  }
  if (finished) {
    if (d > kDepthCap) {  // x's parent sits at depth >= kDepthCap, which the ring cannot hold:
      climb = true;       // look for x's lower siblings by climbing (entries above are in the ring)
      return 0;
    }
    if (ring.cnt == 0u && ring.scnt) {  // the ring ran dry: bring back the newest spilled entry
      const uint32_t j = ring.sbase + ring.scnt - 1u;
      const uint32_t k = j < ring.scap ? j : j - ring.scap;
      ring.top = ring.top + 1 == static_cast<uint32_t>(R) ? 0u : ring.top + 1;
      ring.node[ring.at(ring.top)] = ring.snode[k];
      ring.dm[ring.at(ring.top)] = ring.sdm[k];
      ring.cnt = 1;
      --ring.scnt;
    }
    if (ring.cnt) {  // resume the deepest pending branch point
      const uint32_t slot = ring.at(ring.top);
      src = ring.node[slot];
      const uint32_t dm = ring.dm[slot];
      const uint32_t mask = dm & 15u;
      q = 31 - __clz(mask);
      const uint32_t rest = mask & ~(1u << q);
      if (rest) {
        ring.dm[slot] = static_cast<uint16_t>((dm & ~15u) | rest);
      } else {
        ring.top = ring.top == 0u ? R - 1 : ring.top - 1;
        --ring.cnt;
      }
      d = (dm >> 4) + 1;
      climb = false;
    } else if (!ring.lost || d == 0) {
      return 1;  // nothing pending: traversal complete
    } else {
      climb = true;
      return 0;
    }
  }
  x = child_of<S>(src, q);  // one child computation shared by descend / sibling / resume
  return 0;
}

// Persistent: every lane runs its own traversal and takes the next candidate as soon as
// it finishes (tickets aggregated over the lanes that need one), so a warp is never held
// up by its deepest segment.
template <class S, int R>
__global__ void __launch_bounds__(kPruneThreads) prune_kernel(const uint64_t* __restrict__ cands, uint64_t n,
                                                         uint32_t F, int mode, uint64_t limit,
                                                         uint8_t* __restrict__ removed,
                                                         uint64_t* __restrict__ work,
                                                         unsigned long long* queue, uint64_t* spill_node,
                                                         uint16_t* spill_dm, uint32_t spill_cap) {
  __shared__ uint64_t ring_node[R * kPruneThreads];
  __shared__ uint16_t ring_dm[R * kPruneThreads];
  const uint32_t lane = threadIdx.x & 31u;
  uint64_t i = 0, x = 0, d = 0, acc = 0;
  bool have = false, climb = false, drained = false;
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(kPruneThreads) + threadIdx.x;
  Ring<R> ring{ring_node, ring_dm, spill_node ? spill_node + gtid * spill_cap : nullptr,
            spill_dm ? spill_dm + gtid * spill_cap : nullptr, 0, 0, 0, spill_node ? spill_cap : 0u, 0, false};
  for (;;) {
    if (!drained) {
      const uint32_t need = __ballot_sync(kFull, !have);
      if (need != 0u) {
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (static_cast<int>(lane) == leader) base = atomicAdd(queue, static_cast<unsigned long long>(__popc(need)));
        base = __shfl_sync(kFull, base, leader);
        if (base + __popc(need) >= n) drained = true;
        if (!have) {
          i = base + __popc(need & ((1u << lane) - 1u));
          if (i < n) {
            x = cands[i];
            d = 0;
            acc = mode == 0 ? 0 : 1;
            climb = false;
            have = true;
            ring.cnt = 0;
            ring.scnt = 0;
            ring.sbase = 0;
            ring.lost = false;
          }
        }
      }
    }
    if (!__any_sync(kFull, have)) break;
    if (have) {
      // once the candidates are drained nothing can be refilled: run bursts of steps
      // between warp votes (the tail is latency-bound on the longest traversals)
      int r = prune_step<S, R>(x, d, acc, climb, ring, F, mode, limit);
      const int burst = drained ? kTailBurst : kBulkBurst;
#pragma unroll 1
      for (int k = 1; k < burst && r == 0; ++k) r = prune_step<S, R>(x, d, acc, climb, ring, F, mode, limit);
      if (r != 0) {
        removed[i] = r == 1 ? 1 : 0;
        work[i] = acc;
        have = false;
      }
    }
  }
}

__global__ void first_missing_kernel(const uint64_t* __restrict__ set, uint64_t m,
                                     const uint64_t* __restrict__ q, uint64_t n,
                                     unsigned long long* first) {
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t v = q[i];
    uint64_t lo = 0, hi = m;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (set[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= m || set[lo] != v) atomicMin(first, static_cast<unsigned long long>(i));
  }
}

#ifndef __CUDACC_RTC__
inline unsigned grid_for(uint64_t n, int threads, uint64_t per_thread = 1) {
  const uint64_t g = (n + static_cast<uint64_t>(threads) * per_thread - 1) / (static_cast<uint64_t>(threads) * per_thread);
  return static_cast<unsigned>(g == 0 ? 1 : (g > (1u << 20) ? (1u << 20) : g));
}

#endif

}  // namespace

#ifndef __CUDACC_RTC__

#define LC_DISPATCH(id, ...)                                  \
  switch (id) {                                               \
    case SpecId::A51: { using S = A51; __VA_ARGS__; }         \
    case SpecId::MINI567: { using S = MINI567; __VA_ARGS__; } \
    case SpecId::MINI789: { using S = MINI789; __VA_ARGS__; } \
    default: return cudaErrorInvalidValue;                    \
  }

// SpecId::CUSTOM: the calling thread's runtime-compiled kernels (csrc/jit.cu)
#define LC_CUSTOM_OR(id)                              \
  const CustomKernels* custom = current_custom();     \
  if ((id) == SpecId::CUSTOM && !custom) return cudaErrorInvalidValue;

cudaError_t launch_is_candidate(SpecId id, const uint64_t* xs, uint64_t n, uint32_t F, uint8_t* out,
                                cudaStream_t stream) {
  LC_CUSTOM_OR(id)
  if (id == SpecId::CUSTOM) return jit_launch(custom->is_candidate, grid_for(n, kThreads), kThreads, 0, stream, xs, n, F, out);
  LC_DISPATCH(id, is_candidate_kernel<S><<<grid_for(n, kThreads), kThreads, 0, stream>>>(xs, n, F, out);
              return cudaGetLastError());
}

cudaError_t launch_predecessors(SpecId id, const uint64_t* xs, uint64_t n, uint64_t* out,
                                uint8_t* count, cudaStream_t stream) {
  LC_CUSTOM_OR(id)
  if (id == SpecId::CUSTOM)
    return jit_launch(custom->predecessors, grid_for(n, kThreads), kThreads, 0, stream, xs, n, out, count);
  LC_DISPATCH(id, predecessors_kernel<S><<<grid_for(n, kThreads), kThreads, 0, stream>>>(xs, n, out, count);
              return cudaGetLastError());
}

cudaError_t launch_clock(SpecId id, const uint64_t* xs, uint64_t n, uint64_t t, uint64_t* out,
                         cudaStream_t stream) {
  const unsigned g = static_cast<unsigned>((n + 32u * 128u - 1) / (32u * 128u));
  LC_CUSTOM_OR(id)
  if (id == SpecId::CUSTOM) return jit_launch(custom->clock, g == 0 ? 1 : g, 128, 0, stream, xs, n, t, out);
  LC_DISPATCH(id, clock_kernel<S><<<g == 0 ? 1 : g, 128, 0, stream>>>(xs, n, t, out); return cudaGetLastError());
}

cudaError_t launch_enumerate(SpecId id, uint32_t F, uint64_t r2_lo, uint64_t r2_hi, uint64_t* out,
                             uint64_t cap, uint64_t* d_count, cudaStream_t stream, int* launches) {
  const uint64_t rows = r2_hi > r2_lo ? r2_hi - r2_lo : 0;
  const uint64_t units = rows * 8;  // A5/1: 2^19 virtual slots per row in units of 2^16 (minis: 1 per row)
  const unsigned grid = static_cast<unsigned>(units == 0 ? 1 : (units > (1u << 20) ? (1u << 20) : units));
  if (launches) *launches += 1;
  LC_CUSTOM_OR(id)
  if (id == SpecId::CUSTOM)
    return jit_launch(custom->enumerate, grid, 256, 0, stream, r2_lo, r2_hi, F, out, cap, d_count);
  LC_DISPATCH(id, enumerate_plane_kernel<S><<<grid, 256, 0, stream>>>(r2_lo, r2_hi, F, out, cap, d_count);
              return cudaGetLastError());
}

uint64_t random_scratch_words(uint64_t trials) { return (trials + kTile - 1) / kTile + 1; }

cudaError_t launch_random_candidates(SpecId id, uint32_t F, uint64_t seed, uint64_t trials,
                                     uint64_t* out, uint64_t cap, uint64_t* d_count,
                                     uint64_t* scratch, uint64_t scratch_words,
                                     cudaStream_t stream, int* launches) {
  (void)scratch_words;
  LC_DISPATCH(id, {
    RandGen<S> g{seed, static_cast<uint64_t>(F) << S::O3};
    return compact<S>(g, trials, F, out, cap, d_count, scratch, stream, launches);
  });
}

uint64_t prune_spill_bytes(int blocks, uint32_t cap) {
  return static_cast<uint64_t>(blocks) * kPruneThreads * cap * (8 + 2) + 512;
}

int prune_ring_for(uint64_t n) {
  if (const char* env = getenv("LFSR_PRUNE_RING")) {  // testing / A-B: force a variant
    const int r = atoi(env);
    if (r == kRingDeep || r == kRingWide) return r;
  }
  return n >= (uint64_t{1} << 24) ? kRingWide : kRingDeep;
}

template <int R>
static int blocks_per_sm(SpecId id) {
  int b = 1;
  switch (id) {
    case SpecId::A51: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, prune_kernel<A51, R>, kPruneThreads, 0); break;
    case SpecId::MINI567: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, prune_kernel<MINI567, R>, kPruneThreads, 0); break;
    case SpecId::MINI789: cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, prune_kernel<MINI789, R>, kPruneThreads, 0); break;
    default: break;
  }
  return b > 0 ? b : 1;
}

int prune_blocks_per_sm(SpecId id, int ring) {
  return ring == kRingWide ? blocks_per_sm<kRingWide>(id) : blocks_per_sm<kRingDeep>(id);
}

cudaError_t launch_prune(SpecId id, uint32_t F, int mode, uint64_t limit, const uint64_t* cands,
                         uint64_t n, uint8_t* removed, uint64_t* work, unsigned long long* queue,
                         void* spill, uint32_t spill_cap, int ring, int blocks, cudaStream_t stream) {
  uint64_t* spill_node = spill ? static_cast<uint64_t*>(spill) : nullptr;
  uint16_t* spill_dm =
      spill ? reinterpret_cast<uint16_t*>(spill_node + static_cast<uint64_t>(blocks) * kPruneThreads * spill_cap)
            : nullptr;
  if (ring == kRingWide) {
    LC_DISPATCH(id, prune_kernel<S, kRingWide><<<blocks, kPruneThreads, 0, stream>>>(
                        cands, n, F, mode, limit, removed, work, queue, spill_node, spill_dm, spill_cap);
                return cudaGetLastError());
  }
  LC_DISPATCH(id, prune_kernel<S, kRingDeep><<<blocks, kPruneThreads, 0, stream>>>(
                      cands, n, F, mode, limit, removed, work, queue, spill_node, spill_dm, spill_cap);
              return cudaGetLastError());
}

cudaError_t launch_first_missing(const uint64_t* set, uint64_t m, const uint64_t* q, uint64_t n,
                                 unsigned long long* first, cudaStream_t stream) {
  first_missing_kernel<<<grid_for(n, kThreads), kThreads, 0, stream>>>(set, m, q, n, first);
  return cudaGetLastError();
}

#endif  // !__CUDACC_RTC__

}  // namespace lc
