// K3 (step-2 prune, pipeline.py:121-222): one ordered reverse traversal per lane.
//
// Same traversal and results as the reference's `_dfs_is_shallow` / `_bfs_is_small`
// (pipeline.py:132-160): a candidate's segment is the reverse tree through predecessors
// that are not candidates (`_expand`, pipeline.py:121-129); DFS pops its LIFO stack,
// so the visit order is a preorder taking children in reverse LUT order, and the
// order-dependent `expanded` counter of a deep segment is replayed exactly.
//
// Layout of one lane's traversal (the work per expansion is what bounds this kernel,
// so everything on the per-node path is 32-bit):
//   * the node being expanded: three u32 registers r1, r2, r3 (never a packed u64);
//   * its child set: a byte of a 64-entry table in shared memory, indexed by the three
//     (clock bit, bit above) pairs -- the predecessor table (cipher.py:259-313) folded
//     with the pattern order;
//   * pending branch points (a node whose lower children are still to come): the newest
//     in registers (`cache`), the next R in a per-lane ring in shared memory
//     ([slot][thread]: lanes never share a bank word), older ones in a per-lane spill
//     ring in global memory (L2-resident); beyond that the oldest entries are dropped
//     and rediscovered by climbing forward (a climb step needs only the parent's child
//     set: the child's index follows from which registers differ).
// A node with one child descends without touching the pending set; a leaf resumes the
// newest pending entry.  Both paths end in one shared child computation (three register
// unsteps, cipher.py:221-225, and a select), so a warp's lanes diverge only over a few
// predicated instructions.
#ifndef __CUDACC_RTC__
#include <algorithm>
#include <cstdint>
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
constexpr int kThreads2 = 128;
constexpr uint32_t kDepthCap2 = 1u << 12;  // pending entries hold depths below this (12 bits)
#ifndef LC_PRUNE2_PREFETCH
#define LC_PRUNE2_PREFETCH 0  // 1: a lane prefetches its next candidate and takes it inside a burst
#endif
#ifndef LC_PRUNE2_BULK_BURST
#define LC_PRUNE2_BULK_BURST (LC_PRUNE2_PREFETCH ? 8 : 4)
#endif
constexpr int kBulkBurst2 = LC_PRUNE2_BULK_BURST;  // steps between warp votes while candidates remain
constexpr int kTailBurst2 = 32;   // ... once no candidate is left to take

// child-set byte for the pair index (pair k at bits 2k..2k+1, clock bit low): bit q set
// iff clock pattern CLOCK_PATTERNS[q] is consistent (cipher.py:287-296)
constexpr int std_index2(int pidx) {
  const int c1 = pidx & 1, n1 = (pidx >> 1) & 1, c2 = (pidx >> 2) & 1, n2 = (pidx >> 3) & 1;
  const int c3 = (pidx >> 4) & 1, n3 = (pidx >> 5) & 1;
  return (c1 << 5) | (n1 << 4) | (c2 << 3) | (n2 << 2) | (c3 << 1) | n3;
}
constexpr uint32_t table_word(int w) {  // bytes 4w..4w+3 of the 64-byte table
  uint32_t v = 0;
  for (int b = 0; b < 4; ++b) {
    uint32_t nib = 0;
    for (int q = 0; q < 4; ++q)
      if ((pattern_mask(q) >> std_index2(4 * w + b)) & 1ull) nib |= 1u << q;
    v |= nib << (8 * b);
  }
  return v;
}
struct Table16 {
  uint32_t w[16];
};
constexpr Table16 make_table() {
  Table16 t{};
  for (int i = 0; i < 16; ++i) t.w[i] = table_word(i);
  return t;
}
__constant__ Table16 kChildTable = make_table();

template <class S>
struct Regs {
  uint32_t r1, r2, r3;
};

template <class S>
__device__ __forceinline__ uint32_t pair_index(uint32_t r1, uint32_t r2, uint32_t r3) {
  return ((r1 >> S::CT1) & 3u) | (((r2 >> S::CT2) & 3u) << 2) | (((r3 >> S::CT3) & 3u) << 4);
}

// unstep_register (cipher.py:221-225): r >> 1 with the top bit = r0 ^ parity(taps of
// r >> 1 below the top) = parity(r & ((T_low << 1) | 1))
template <int L, uint32_t TM>
__device__ __forceinline__ uint32_t unstep2(uint32_t r) {
  constexpr uint32_t M = ((TM & ~(1u << (L - 1))) << 1) | 1u;
  return (r >> 1) | ((__popc(r & M) & 1u) << (L - 1));
}

// predecessor under CLOCK_PATTERNS[q] = {0b011, 0b101, 0b110, 0b111}[q]: R1 unsteps
// unless q == 2, R2 unless q == 1, R3 unless q == 0
template <class S>
__device__ __forceinline__ void child2(uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t q) {
  const uint32_t u1 = unstep2<S::L1, S::T1>(r1), u2 = unstep2<S::L2, S::T2>(r2), u3 = unstep2<S::L3, S::T3>(r3);
  r1 = q != 2u ? u1 : r1;
  r2 = q != 1u ? u2 : r2;
  r3 = q != 0u ? u3 : r3;
}

// Children of the node in the segment (pipeline.py:121-129): its predecessors minus
// special nodes.  A child c's successor is the node itself, so is_candidate(c)
// (cipher.py:420-428) reduces to "R3(c) == F and c's table entry is non-empty"; only
// the patterns that unstep R3 can land on F, and only when unstep(R3) == F (rare).
template <class S>
__device__ __forceinline__ uint32_t child_set(const uint8_t* tbl, uint32_t r1, uint32_t r2, uint32_t r3,
                                              uint32_t F) {
  uint32_t m = tbl[pair_index<S>(r1, r2, r3)];
  if (unstep2<S::L3, S::T3>(r3) == F) {
#pragma unroll
    for (uint32_t q = 1; q < 4; ++q) {
      uint32_t c1 = r1, c2 = r2, c3 = r3;
      child2<S>(c1, c2, c3, q);
      if (((m >> q) & 1u) && tbl[pair_index<S>(c1, c2, c3)] != 0u) m &= ~(1u << q);
    }
  }
  return m;
}

template <class S>
__device__ __forceinline__ uint64_t pack2(uint32_t r1, uint32_t r2, uint32_t r3) {
  return static_cast<uint64_t>(r1) | (static_cast<uint64_t>(r2) << S::O2) | (static_cast<uint64_t>(r3) << S::O3);
}
template <class S>
__device__ __forceinline__ void unpack2(uint64_t x, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  r1 = static_cast<uint32_t>(x) & static_cast<uint32_t>(S::M1);
  r2 = static_cast<uint32_t>(x >> S::O2) & static_cast<uint32_t>(S::M2);
  r3 = static_cast<uint32_t>(x >> S::O3);
}

// Pending branch points of one lane: the newest in registers, R more in shared memory,
// older ones in a global spill ring (scap entries; entry k, 0 = oldest, at
// (sbase + k) mod scap).  `lost`: some entry was dropped (the climb rediscovers it).
template <int R>
struct Pending {
  uint64_t* node;  // shared [R][kThreads2]
  uint16_t* dm;    // shared [R][kThreads2]: depth << 4 | remaining child mask
  uint64_t* snode; // global spill ring of this lane
  uint16_t* sdm;
  uint64_t cnode;  // the newest entry (valid iff cdm != 0: its mask is never empty)
  uint32_t cdm;
  uint32_t top, cnt, scnt, scap, sbase;
  bool lost;
  __device__ __forceinline__ uint32_t at(uint32_t slot) const {
    LC_CHECK(slot < static_cast<uint32_t>(R));
    return slot * kThreads2 + threadIdx.x;
  }
  __device__ __forceinline__ void reset() {
    cdm = 0;
    cnt = scnt = sbase = 0;
    lost = false;
  }
  // the cached entry moves into the shared ring (its oldest entry, if full, to the spill)
  __device__ __forceinline__ void demote() {
    const uint32_t next = top + 1 == static_cast<uint32_t>(R) ? 0u : top + 1;
    if (cnt == static_cast<uint32_t>(R)) {
      if (scap) {
        if (scnt == scap) {  // spill full too: drop its oldest entry
          sbase = sbase + 1 == scap ? 0u : sbase + 1;
          --scnt;
          lost = true;
        }
        const uint32_t k = sbase + scnt < scap ? sbase + scnt : sbase + scnt - scap;
        LC_CHECK(k < scap && scnt < scap && cnt == static_cast<uint32_t>(R));
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
    node[at(top)] = cnode;
    dm[at(top)] = static_cast<uint16_t>(cdm);
  }
  __device__ __forceinline__ void push(uint64_t y, uint32_t d, uint32_t mask) {
    if (d >= kDepthCap2) return;  // no room for the depth: found again by climbing
    if (cdm) demote();
    cnode = y;
    cdm = (d << 4) | mask;
  }
  // make the newest entry the cached one; false if nothing is pending
  __device__ __forceinline__ bool promote() {
    if (cdm) return true;
    if (cnt == 0u && scnt) {  // the shared ring ran dry: take the newest spilled entry
      const uint32_t j = sbase + scnt - 1u;
      const uint32_t k = j < scap ? j : j - scap;
      LC_CHECK(k < scap && scnt <= scap);
      --scnt;
      cnode = snode[k];
      cdm = sdm[k];
      return true;
    }
    if (cnt == 0u) return false;
    cnode = node[at(top)];
    cdm = dm[at(top)];
    top = top == 0u ? R - 1 : top - 1;
    --cnt;
    return true;
  }
};

// A subtree is done: make the newest pending entry the cached one (0, climb false), or
// climb (0, climb true: entries were dropped or the parent's depth does not fit an entry),
// or finish (1: nothing pending, the traversal is complete).
template <class S, int R>
__device__ __forceinline__ int resume_or_finish(uint32_t d, bool& climb, Pending<R>& pend) {
  if (d > kDepthCap2) {  // the parent sits at a depth the pending entries cannot hold
    climb = true;
    return 0;
  }
  if (pend.promote()) {
    climb = false;
    return 0;
  }
  if (!pend.lost || d == 0u) return 1;
  climb = true;
  return 0;
}

// One traversal step: exactly one node expansion per lane.  Returns 0 while running,
// 1 = finished shallow (removed), 2 = finished deep (a survivor).
template <class S, int R, bool DFS>
__device__ __forceinline__ int prune_step_split(const uint8_t* tbl, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                                uint32_t& d, uint64_t& acc, bool& climb, Pending<R>& pend,
                                                uint32_t F, uint64_t limit) {
  uint32_t q = 0;
  bool resume;  // the current node's subtree is done: continue at the newest pending entry
  if (!climb) {
    const uint32_t m = child_set<S>(tbl, r1, r2, r3, F);
    resume = m == 0u;
    if (!resume) {
      if (DFS) {
        if (d >= limit) {  // a child would sit below the depth limit (pipeline.py:138-141)
          acc += 1;
          return 2;
        }
        acc += __popc(m);
      } else {
        acc += __popc(m);
        if (acc > limit) {  // pipeline.py:155-157
          acc = limit + 1;
          return 2;
        }
      }
      q = 31 - __clz(m);  // the LIFO stack pops the last-pushed (highest) child first
      const uint32_t rest = m & ~(1u << q);
      if (rest) pend.push(pack2<S>(r1, r2, r3), d, rest);
      ++d;
    }
  } else {
    // the parent y of the current node: continue with the next-lower sibling, else y's
    // subtree is done too.  The current node's index under y follows from which
    // registers differ (the clocked ones).
    const uint64_t x = pack2<S>(r1, r2, r3);
    const uint64_t y = clock_scalar<S>(x);
    const uint64_t diff = x ^ y;
    const uint32_t pat = ((diff & S::M1) ? 1u : 0u) | (((diff >> S::O2) & S::M2) ? 2u : 0u) |
                         (((diff >> S::O3) & S::M3) ? 4u : 0u);
    const uint32_t k = pat == 3u ? 0u : pat == 5u ? 1u : pat == 6u ? 2u : 3u;
    unpack2<S>(y, r1, r2, r3);
    const uint32_t lower = child_set<S>(tbl, r1, r2, r3, F) & ((1u << k) - 1u);
    resume = lower == 0u;
    --d;
    if (!resume) {
      q = 31 - __clz(lower);
      const uint32_t rest = lower & ~(1u << q);
      if (rest) pend.push(y, d, rest);
      ++d;
      climb = false;
    }
  }
  if (resume) {
    if (d > kDepthCap2) {  // the parent sits at a depth the pending entries cannot hold
      climb = true;
      return 0;
    }
    if (!pend.promote()) {
      if (!pend.lost || d == 0u) return 1;  // nothing pending: traversal complete
      climb = true;
      return 0;
    }
    const uint32_t mask = pend.cdm & 15u;
    q = 31 - __clz(mask);
    d = (pend.cdm >> 4) + 1;
    unpack2<S>(pend.cnode, r1, r2, r3);
    const uint32_t rest = mask & ~(1u << q);
    pend.cdm = rest ? ((pend.cdm & ~15u) | rest) : 0u;
    climb = false;
  }
  child2<S>(r1, r2, r3, q);
  return 0;
}

// One traversal step: exactly one node expansion per lane.  Returns 0 while running,
// 1 = finished shallow (removed), 2 = finished deep (a survivor).
//
// The two common cases share one straight-line path: the entry whose highest pending
// child comes next is either (this node, its child set) -- descend -- or the newest
// pending entry -- resume at a leaf; either way its remaining children go back to the
// pending set and the child is computed from the entry's node.  Lanes of a warp diverge
// only inside promote()/push() (a shared-memory load or store) and in the rare climb.
template <class S, int R, bool DFS>
__device__ __forceinline__ int prune_step_unified(const uint8_t* tbl, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t& d,
                                           uint64_t& acc, bool& climb, Pending<R>& pend, uint32_t F,
                                           uint64_t limit) {
  // the entry's node is held in r1..r3 (packed only when its remaining children go to the
  // pending set, unpacked only when a leaf resumes a pending entry)
  uint32_t edm;
  if (climb) {
    // the parent y of the current node: continue with the next-lower sibling, else y's
    // subtree is done too.  The current node's index under y follows from which
    // registers differ (the clocked ones).
    const uint64_t x = pack2<S>(r1, r2, r3);
    const uint64_t y = clock_scalar<S>(x);
    const uint64_t diff = x ^ y;
    const uint32_t pat = ((diff & S::M1) ? 1u : 0u) | (((diff >> S::O2) & S::M2) ? 2u : 0u) |
                         (((diff >> S::O3) & S::M3) ? 4u : 0u);
    const uint32_t k = pat == 3u ? 0u : pat == 5u ? 1u : pat == 6u ? 2u : 3u;
    unpack2<S>(y, r1, r2, r3);
    const uint32_t lower = child_set<S>(tbl, r1, r2, r3, F) & ((1u << k) - 1u);
    --d;
    if (lower == 0u) {  // y's subtree is done as well
      const int r = resume_or_finish<S, R>(d, climb, pend);
      if (r != 0 || climb) return r;
      unpack2<S>(pend.cnode, r1, r2, r3);
      edm = pend.cdm;
      pend.cdm = 0u;
    } else {
      climb = false;
      edm = (d << 4) | lower;
    }
  } else {
    const uint32_t m = child_set<S>(tbl, r1, r2, r3, F);
    if (m != 0u) {
      if (DFS) {
        if (d >= limit) {  // a child would sit below the depth limit (pipeline.py:138-141)
          acc += 1;
          return 2;
        }
        acc += __popc(m);
      } else {
        acc += __popc(m);
        if (acc > limit) {  // pipeline.py:155-157
          acc = limit + 1;
          return 2;
        }
      }
      edm = (d << 4) | m;
    } else {
      const int r = resume_or_finish<S, R>(d, climb, pend);
      if (r != 0 || climb) return r;
      unpack2<S>(pend.cnode, r1, r2, r3);
      edm = pend.cdm;
      pend.cdm = 0u;  // taken out of the cache (the rest goes back below)
    }
  }
  const uint32_t mask = edm & 15u;
  const uint32_t q = 31 - __clz(mask);  // the LIFO stack pops the last-pushed (highest) child first
  const uint32_t rest = mask & ~(1u << q);
  const uint32_t ed = edm >> 4;
  if (rest) pend.push(pack2<S>(r1, r2, r3), ed, rest);
  d = ed + 1;
  child2<S>(r1, r2, r3, q);
  return 0;
}

// The unified step with the pending-set traffic flattened: per step a lane does at most
// one shared-memory ring access -- a pop when a leaf finds the register cache empty, or a
// demotion of the cache when a node with several children needs it -- written as
// predicated straight-line code, so a warp issues it once for all its lanes instead of
// once per divergent branch (ncu: a quarter of the warp instructions of the branchy form
// ran with at most 3 of 32 lanes active).  The rare cases (spill refill, end of the
// traversal, climbing) keep their branches.
template <class S, int R, bool DFS>
__device__ __forceinline__ int prune_step_flat(const uint8_t* tbl, uint32_t& r1, uint32_t& r2, uint32_t& r3,
                                               uint32_t& d, uint64_t& acc, bool& climb, Pending<R>& pend,
                                               uint32_t F, uint64_t limit) {
  if (climb) return prune_step_unified<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
  const uint32_t m = child_set<S>(tbl, r1, r2, r3, F);
  const bool leaf = m == 0u;
  if (!leaf) {
    if (DFS) {
      if (d >= limit) {  // a child would sit below the depth limit (pipeline.py:138-141)
        acc += 1;
        return 2;
      }
      acc += __popc(m);
    } else {
      acc += __popc(m);
      if (acc > limit) {  // pipeline.py:155-157
        acc = limit + 1;
        return 2;
      }
    }
  } else if (d > kDepthCap2 || (pend.cdm == 0u && pend.cnt == 0u)) {
    // leaf with nothing cached or in the shared ring: spill refill, climb or done
    const int r = resume_or_finish<S, R>(d, climb, pend);
    if (r != 0 || climb) return r;
  }
  // ring pop: a leaf whose cache is empty takes the ring's newest entry (cnt > 0 here)
  const bool pop = leaf && pend.cdm == 0u;
  const uint32_t a = pend.at(pend.top);
  uint64_t rn = pend.cnode;
  uint32_t rdm = pend.cdm;
  if (pop) {
    rn = pend.node[a];
    rdm = pend.dm[a];
    pend.top = pend.top == 0u ? R - 1 : pend.top - 1;
    --pend.cnt;
  }
  uint32_t edm = (d << 4) | m;
  if (leaf) {
    unpack2<S>(rn, r1, r2, r3);
    edm = rdm;
    pend.cdm = 0u;
  }
  const uint32_t mask = edm & 15u;
  const uint32_t q = 31 - __clz(mask);  // the LIFO stack pops the last-pushed (highest) child first
  const uint32_t rest = mask & ~(1u << q);
  const uint32_t ed = edm >> 4;
  if (rest && ed < kDepthCap2) {  // deeper entries are found again by climbing
    if (pend.cdm) {  // demote the cache into the ring (its oldest entry to the spill when full)
      if (pend.cnt == static_cast<uint32_t>(R)) {
        pend.demote();
      } else {
        const uint32_t nt = pend.top + 1 == static_cast<uint32_t>(R) ? 0u : pend.top + 1;
        const uint32_t b = pend.at(nt);
        pend.node[b] = pend.cnode;
        pend.dm[b] = static_cast<uint16_t>(pend.cdm);
        pend.top = nt;
        ++pend.cnt;
      }
    }
    pend.cnode = pack2<S>(r1, r2, r3);
    pend.cdm = (ed << 4) | rest;
  }
  d = ed + 1;
  child2<S>(r1, r2, r3, q);
  return 0;
}

#ifndef LC_PRUNE2_UNIFIED
#define LC_PRUNE2_UNIFIED 1  // 0: the two-path step, 2: flattened ring traffic (A/B)
#endif
template <class S, int R, bool DFS>
__device__ __forceinline__ int prune_step2(const uint8_t* tbl, uint32_t& r1, uint32_t& r2, uint32_t& r3, uint32_t& d,
                                           uint64_t& acc, bool& climb, Pending<R>& pend, uint32_t F,
                                           uint64_t limit) {
#if LC_PRUNE2_UNIFIED == 2
  return prune_step_flat<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
#elif LC_PRUNE2_UNIFIED
  return prune_step_unified<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
#else
  return prune_step_split<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
#endif
}

#ifndef LC_PRUNE2_MINBLOCKS
#define LC_PRUNE2_MINBLOCKS 1
#endif
template <class S, int R, bool DFS>
__global__ void __launch_bounds__(kThreads2, LC_PRUNE2_MINBLOCKS) prune2_kernel(const uint64_t* __restrict__ cands, uint64_t n, uint32_t F,
                                                           uint64_t limit, uint8_t* __restrict__ removed,
                                                           uint64_t* __restrict__ work, unsigned long long* queue,
                                                           uint64_t* spill_node, uint16_t* spill_dm,
                                                           uint32_t spill_cap) {
  __shared__ uint64_t ring_node[R * kThreads2];
  __shared__ uint16_t ring_dm[R * kThreads2];
  __shared__ uint32_t tbl_words[16];
  if (threadIdx.x < 16) tbl_words[threadIdx.x] = kChildTable.w[threadIdx.x];
  __syncthreads();
  const uint8_t* tbl = reinterpret_cast<const uint8_t*>(tbl_words);
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(kThreads2) + threadIdx.x;
  Pending<R> pend{ring_node, ring_dm, spill_node ? spill_node + gtid * spill_cap : nullptr,
                  spill_dm ? spill_dm + gtid * spill_cap : nullptr, 0, 0, 0, 0, 0, spill_node ? spill_cap : 0u, 0,
                  false};
#if LC_PRUNE2_PREFETCH
  // each lane holds its current candidate and the next one (loaded a burst ahead, so a
  // lane that finishes takes the next at once, inside the burst)
  uint64_t i = 0, acc = 0, ni = 0, nx = 0;
  uint32_t r1 = 0, r2 = 0, r3 = 0, d = 0;
  bool have = false, climb = false, drained = false, nvalid = false;
  for (;;) {
    if (!drained) {
      const uint32_t need = __ballot_sync(kFull, !nvalid);
      if (need != 0u) {
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (static_cast<int>(lane) == leader) base = atomicAdd(queue, static_cast<unsigned long long>(__popc(need)));
        base = __shfl_sync(kFull, base, leader);
        if (base + __popc(need) >= n) drained = true;
        if (!nvalid) {
          ni = base + __popc(need & ((1u << lane) - 1u));
          if (ni < n) {
            nx = cands[ni];
            nvalid = true;
          }
        }
      }
    }
    if (!__any_sync(kFull, have || nvalid)) break;
    const int burst = drained ? kTailBurst2 : kBulkBurst2;
#pragma unroll 1
    for (int k = 0; k < burst; ++k) {
      if (!have) {
        if (!nvalid) break;
        i = ni;
        unpack2<S>(nx, r1, r2, r3);
        d = 0;
        acc = DFS ? 0 : 1;
        climb = false;
        pend.reset();
        have = true;
        nvalid = false;
      }
      const int r = prune_step2<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
      if (r != 0) {
        LC_CHECK(i < n);
        removed[i] = r == 1 ? 1 : 0;
        work[i] = acc;
        have = false;
      }
    }
  }
#else
  uint64_t i = 0, acc = 0;
  uint32_t r1 = 0, r2 = 0, r3 = 0, d = 0;
  bool have = false, climb = false, drained = false;
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
            unpack2<S>(cands[i], r1, r2, r3);
            d = 0;
            acc = DFS ? 0 : 1;
            climb = false;
            have = true;
            pend.reset();
          }
        }
      }
    }
    if (!__any_sync(kFull, have)) break;
    if (have) {
      int r = prune_step2<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
      const int burst = drained ? kTailBurst2 : kBulkBurst2;
#pragma unroll 1
      for (int k = 1; k < burst && r == 0; ++k) r = prune_step2<S, R, DFS>(tbl, r1, r2, r3, d, acc, climb, pend, F, limit);
      if (r != 0) {
        LC_CHECK(i < n);
        removed[i] = r == 1 ? 1 : 0;
        work[i] = acc;
        have = false;
      }
    }
  }
#endif
}

// ---------------------------------------------------------------------------- K3 v3
//
// DFS mode with one uniform step per expansion.  The pending branch points are a plain
// per-lane stack of (node, depth, remaining children) entries; every step a lane
// expands its current node and moves to the next node of the reference's preorder:
//   * the node has children: its highest child; the rest go on the stack as one entry
//     (a push), unless it was the only one;
//   * a leaf: the highest remaining child of the stack's top entry (a load); the top
//     entry keeps the others (a store of its new mask) or is popped.
// Both cases are the same instructions on a selected source entry: one predicated
// 16-byte shared-memory load, one predicated store, three register unsteps and a
// select -- no per-lane branches besides the rare ones (a special-node child, the depth
// abort, a traversal's end).
//
// Stack entries are ancestors of the current node at distinct depths, so a traversal
// that aborts at depth `limit` never holds more than `limit` of them (launched for
// limit <= kSpill3Max).  Deep segments keep hundreds pending (the time-weighted median
// stack height of the A5/1 slice is ~250), so the stack lives in global memory -- the
// lane's own array, written through on every push and mask update -- and the newest
// K entries are cached in a shared-memory ring ([slot][thread], 16 B per entry,
// conflict-free), which is what the step reads.  The ring is kept stocked ahead of
// the pops: once fewer than kLow3 entries are cached, the kChunk3 entries below are
// requested with cp.async (no register staging, no stall), so a pop finds its entry
// already in shared memory; a full ring just forgets its oldest kChunk3 (they are in
// global memory already).  The cached range always starts at a multiple of kChunk3, so
// a refill is kChunk3 fixed-offset copies into consecutive slots.
//
// Divergence is what this kernel's speed is about (ncu at 2^26: 58 % of the lanes of
// an issued warp instruction active with separate push / rewrite paths and variable
// refills); the unified store and the aligned refills were worth 1.55x over K3 v2 at
// 2^28 candidates (profiles/r02_prune3_ab.txt).
constexpr int kThreads3 = 128;
#ifndef LC_PRUNE3_STACK
#define LC_PRUNE3_STACK 8
#endif
#ifndef LC_PRUNE3_CHUNK
#define LC_PRUNE3_CHUNK 4
#endif
#ifndef LC_PRUNE3_LOW
#define LC_PRUNE3_LOW 4
#endif
#ifndef LC_PRUNE3_BURST
#define LC_PRUNE3_BURST 8
#endif
constexpr int kStack3 = LC_PRUNE3_STACK;
constexpr int kChunk3 = LC_PRUNE3_CHUNK;  // entries per prefetch / per eviction
constexpr int kLow3 = LC_PRUNE3_LOW;      // prefetch below this many cached entries
constexpr int kBurst3 = LC_PRUNE3_BURST;  // steps between warp votes for new candidates
static_assert((kStack3 & (kStack3 - 1)) == 0, "stack ring is a power of two");
static_assert(kChunk3 >= 1 && kLow3 + kChunk3 <= kStack3, "a prefetch fits the ring");
constexpr uint32_t kSpill3Max = 4096;
constexpr int kStack3Bytes = kStack3 * kThreads3 * 16;
static_assert(kStack3 % kChunk3 == 0, "aligned chunks tile the ring");

// child set with the special-node test behind a cheap necessary condition: unstep(R3)
// == F needs R3 >> 1 == F's low bits
template <class S>
__device__ __forceinline__ uint32_t child_set3(const uint8_t* tbl, uint32_t r1, uint32_t r2, uint32_t r3,
                                               uint32_t F) {
  constexpr uint32_t LOW = static_cast<uint32_t>(S::M3 >> 1);
  uint32_t m = tbl[pair_index<S>(r1, r2, r3)];
  if ((r3 >> 1) == (F & LOW)) {
    if (unstep2<S::L3, S::T3>(r3) == F) {
#pragma unroll
      for (uint32_t q = 1; q < 4; ++q) {
        uint32_t c1 = r1, c2 = r2, c3 = r3;
        child2<S>(c1, c2, c3, q);
        if (((m >> q) & 1u) && tbl[pair_index<S>(c1, c2, c3)] != 0u) m &= ~(1u << q);
      }
    }
  }
  return m;
}

__device__ __forceinline__ void cp_async16(uint32_t smem, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem), "l"(g) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <class S, int K, bool DFS>
__global__ void __launch_bounds__(kThreads3) prune3_kernel(const uint64_t* __restrict__ cands, uint64_t n,
                                                           uint32_t F, uint32_t limit,
                                                           uint8_t* __restrict__ removed,
                                                           uint64_t* __restrict__ work, unsigned long long* queue,
                                                           uint4* gstack, uint32_t gcap) {
  extern __shared__ uint4 ring[];  // [K][kThreads3] (dynamic: kStack3Bytes)
  __shared__ uint8_t tbl[64];
  if (threadIdx.x < 16) reinterpret_cast<uint32_t*>(tbl)[threadIdx.x] = kChildTable.w[threadIdx.x];
  __syncthreads();
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t gtid = blockIdx.x * static_cast<uint64_t>(kThreads3) + threadIdx.x;
  uint4* my = gstack + gtid * gcap;  // this lane's stack, logical index = position
  uint4* my_ring = ring + threadIdx.x;
  const uint32_t ring_s = static_cast<uint32_t>(__cvta_generic_to_shared(my_ring));
  constexpr uint32_t kSlot = kThreads3 * 16;  // bytes between a lane's ring slots
  uint64_t i = 0, acc = 0;
  uint32_t r1 = 0, r2 = 0, r3 = 0, d = 0;
  uint32_t sp = 0;    // stack height: logical entries [0, sp), all in global memory
  uint32_t lo = 0;    // the ring caches [lo, sp) (sp - lo <= K)
  uint32_t pfhi = 0;  // entries [.., pfhi) may still be in flight from a prefetch (0: none)
  bool have = false, drained = false;
  for (;;) {
    const uint32_t need = __ballot_sync(kFull, !have);
    if (need != 0u) {
      if (drained) {
        if (need == kFull) break;
      } else {
        const int leader = __ffs(need) - 1;
        unsigned long long base = 0;
        if (static_cast<int>(lane) == leader) base = atomicAdd(queue, static_cast<unsigned long long>(__popc(need)));
        base = __shfl_sync(kFull, base, leader);
        if (base + __popc(need) >= n) drained = true;
        if (!have) {
          i = base + __popc(need & ((1u << lane) - 1u));
          if (i < n) {
            unpack2<S>(cands[i], r1, r2, r3);
            d = 0;
            acc = DFS ? 0 : 1;  // BFS counts the root (pipeline.py:149)
            sp = lo = 0;
            have = true;
          }
        }
      }
    }
#pragma unroll 1
    for (int k = 0; k < kBurst3; ++k) {
      if (!have) break;
      const uint32_t m = child_set3<S>(tbl, r1, r2, r3, F);
      const bool leaf = m == 0u;
      int fin = 0;  // 1 removed (traversal complete), 2 survivor (a child below the limit)
      if (DFS) {
        if (!leaf && d >= limit) {  // pipeline.py:138-141: the first child counts, then abort
          acc += 1;
          fin = 2;
        } else if (leaf && sp == 0u) {
          fin = 1;
        }
      } else {
        // BFS (pipeline.py:147-160) counts nodes until the count passes the limit; both
        // outcomes are independent of the visiting order, so the DFS order serves
        if (acc + __popc(m) > limit) {
          acc = static_cast<uint64_t>(limit) + 1;
          fin = 2;
        } else if (leaf && sp == 0u) {
          fin = 1;
        }
      }
      if (fin != 0) {
        LC_CHECK(i < n);
        removed[i] = fin == 1 ? 1 : 0;
        work[i] = acc;
        have = false;
        if (pfhi) cp_async_wait_all();  // nothing in flight into the ring across traversals
        pfhi = 0;
        break;
      }
      acc += __popc(m);
      if (leaf) {
        if (sp - 1u < pfhi) {  // the top entry may still be arriving
          cp_async_wait_all();
          pfhi = 0;
        }
        if (sp == lo) {  // not cached (no room was left to prefetch it): fetch it now
          lo -= kChunk3;  // lo stays a multiple of the chunk: its slots are consecutive
          LC_CHECK(lo % kChunk3 == 0 && lo + kChunk3 <= sp && sp <= gcap);
          const uint32_t s0 = ring_s + (lo & (K - 1)) * kSlot;
#pragma unroll
          for (int j = 0; j < kChunk3; ++j) cp_async16(s0 + j * kSlot, my + lo + j);
          cp_async_commit();
          cp_async_wait_all();
          pfhi = 0;
        }
      }
      const uint32_t top = (sp - 1u) & (K - 1);
      uint4 e = make_uint4(r1, r2, r3, (d << 4) | m);
      if (leaf) e = my_ring[top * kThreads3];
      const uint32_t mask = e.w & 15u;
      const uint32_t q = 31 - __clz(mask);  // the LIFO stack pops the last-pushed (highest) child first
      const uint32_t rest = mask & ~(1u << q);
      const uint32_t ed = e.w >> 4;
      // the entry keeping the other children: the top one rewritten (leaf) or a new one
      // pushed -- one predicated 16-byte store to the ring and one to memory either way
      const uint32_t idx = leaf ? sp - 1u : sp;
      if (rest != 0u) {
        if (!leaf && sp - lo == static_cast<uint32_t>(K)) {  // ring full: forget its oldest chunk
          if (pfhi) {
            cp_async_wait_all();
            pfhi = 0;
          }
          lo += kChunk3;
        }
        LC_CHECK(idx < gcap);
        const uint4 ne = make_uint4(e.x, e.y, e.z, (ed << 4) | rest);
        my_ring[(idx & (K - 1)) * kThreads3] = ne;
        my[idx] = ne;
      }
      sp = idx + (rest != 0u ? 1u : 0u);
      // keep the ring stocked ahead of the pops
      if (lo != 0u && sp - lo < static_cast<uint32_t>(kLow3)) {
        if (pfhi) cp_async_wait_all();
        pfhi = lo;
        lo -= kChunk3;
        LC_CHECK(lo % kChunk3 == 0 && sp - lo <= static_cast<uint32_t>(K) && sp <= gcap);
        const uint32_t s0 = ring_s + (lo & (K - 1)) * kSlot;
#pragma unroll
        for (int j = 0; j < kChunk3; ++j) cp_async16(s0 + j * kSlot, my + lo + j);
        cp_async_commit();
      }
      r1 = e.x;
      r2 = e.y;
      r3 = e.z;
      d = ed + 1;
      child2<S>(r1, r2, r3, q);
    }
  }
}

// ------------------------------------------------------ batched segment probes
// probe_segment (pipeline.py:262-298) for many roots at once, level-synchronous and
// device-resident: one expand launch per level appends every live root's next level
// (its frontier's children in the segment, `_expand`) to the other frontier buffer and
// counts them per root; one finalize launch per root applies the reference's
// bookkeeping for the level (depth, nodes, level_counts, the node cap).  The host only
// launches (and looks at the live count every few levels); a frontier that would
// overflow its buffer leaves the level uncommitted for the host to grow and redo.
constexpr int kProbeThreads = 256;

template <class S>
__global__ void __launch_bounds__(kProbeThreads) probe_expand_kernel(
    const uint64_t* __restrict__ fnode, const uint32_t* __restrict__ fowner, const unsigned long long* cur_count,
    const uint8_t* __restrict__ status, uint32_t F, uint64_t* __restrict__ nnode, uint32_t* __restrict__ nowner,
    unsigned long long* next_count, unsigned long long cap, unsigned long long* __restrict__ lvl,
    unsigned int* overflow) {
  __shared__ uint32_t tbl_words[16];
  if (threadIdx.x < 16) tbl_words[threadIdx.x] = kChildTable.w[threadIdx.x];
  __syncthreads();
  if (*overflow) return;
  const uint8_t* tbl = reinterpret_cast<const uint8_t*>(tbl_words);
  const unsigned long long m = *cur_count;
  const uint32_t lane = threadIdx.x & 31u;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kProbeThreads;
  // warp-aligned loop: every lane of a warp runs the same iterations (warp-wide append)
  for (uint64_t w0 = blockIdx.x * static_cast<uint64_t>(kProbeThreads) + (threadIdx.x & ~31u); w0 < m;
       w0 += stride) {
    const uint64_t i = w0 + lane;
    uint32_t r1 = 0, r2 = 0, r3 = 0, mask = 0, o = 0;
    if (i < m) {
      o = fowner[i];
      if (status[o] == 0) {
        unpack2<S>(fnode[i], r1, r2, r3);
        mask = child_set3<S>(tbl, r1, r2, r3, F);
      }
    }
    const uint32_t c = __popc(mask);
    uint32_t incl = c;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, d);
      if (lane >= static_cast<uint32_t>(d)) incl += y;
    }
    const uint32_t tot = __shfl_sync(kFull, incl, 31);
    unsigned long long base = 0;
    if (lane == 31 && tot) base = atomicAdd(next_count, static_cast<unsigned long long>(tot));
    base = __shfl_sync(kFull, base, 31) + (incl - c);
    if (c) {
      if (base + c > cap) {
        atomicExch(overflow, 1u);
      } else {
        atomicAdd(&lvl[o], static_cast<unsigned long long>(c));
        uint64_t k = base;
        for (uint32_t q = 0; q < 4; ++q)  // LUT order, as the reference appends them
          if ((mask >> q) & 1u) {
            uint32_t c1 = r1, c2 = r2, c3 = r3;
            child2<S>(c1, c2, c3, q);
            nnode[k] = pack2<S>(c1, c2, c3);
            nowner[k] = o;
            ++k;
          }
      }
    }
  }
}

// status: 0 live, 1 done (empty level), 2 censored
__global__ void probe_finalize_kernel(uint32_t k, uint32_t level, unsigned long long* __restrict__ lvl,
                                      uint8_t* __restrict__ status, uint64_t* __restrict__ depth,
                                      uint64_t* __restrict__ nodes, unsigned long long* __restrict__ level_counts,
                                      uint32_t levels_cap, int64_t node_cap, const unsigned int* overflow,
                                      unsigned long long* live, unsigned long long* done_count,
                                      unsigned long long* cnt_reset, unsigned long long* live_reset) {
  if (*overflow) return;
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < k; o += gridDim.x * blockDim.x) {
    if (status[o] != 0) continue;
    const unsigned long long c = lvl[o];
    lvl[o] = 0;
    if (c == 0) {  // pipeline.py:286-287: an empty next level ends the sweep
      status[o] = 1;
      continue;
    }
    depth[o] = level + 1;
    nodes[o] += c;
    if (level + 1 < levels_cap) atomicAdd(&level_counts[level + 1], c);
    if (node_cap >= 0 && nodes[o] > static_cast<uint64_t>(node_cap)) {  // pipeline.py:293-294
      status[o] = 2;
      continue;
    }
    atomicAdd(live, 1ull);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd(done_count, 1ull);  // levels committed (the host redoes from here after an overflow)
    cnt_reset[0] = 0;             // this level's frontier count: free for level + 2
    live_reset[0] = 0;            // the next level's live count starts from zero
  }
}

// pipeline.py:280-281: a sweep that reaches depth_cap is censored
__global__ void probe_censor_kernel(uint32_t k, uint8_t* __restrict__ status) {
  for (uint32_t o = blockIdx.x * blockDim.x + threadIdx.x; o < k; o += gridDim.x * blockDim.x)
    if (status[o] == 0) status[o] = 2;
}

#ifndef LC_PRUNE2_RING
#define LC_PRUNE2_RING 16
#endif
constexpr int kRing2 = LC_PRUNE2_RING;

#ifndef __CUDACC_RTC__
template <class S>
int blocks2(bool dfs) {
  int b = 1;
  if (dfs) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, prune2_kernel<S, kRing2, true>, kThreads2, 0);
  else cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, prune2_kernel<S, kRing2, false>, kThreads2, 0);
  return b > 0 ? b : 1;
}

template <class S>
const void* kernel3(bool dfs) {
  // (per call: the attribute is per device, and setting it is a cheap host call)
  const void* k = dfs ? reinterpret_cast<const void*>(prune3_kernel<S, kStack3, true>)
                      : reinterpret_cast<const void*>(prune3_kernel<S, kStack3, false>);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kStack3Bytes);
  return k;
}

template <class S>
int blocks3() {
  int b = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel3<S>(true), kThreads3, kStack3Bytes);
  return b > 0 ? b : 1;
}

#endif

}  // namespace

#ifndef __CUDACC_RTC__

int prune2_blocks_per_sm(SpecId id, int mode) {
  switch (id) {
    case SpecId::A51: return blocks2<A51>(mode == 0);
    case SpecId::MINI567: return blocks2<MINI567>(mode == 0);
    case SpecId::MINI789: return blocks2<MINI789>(mode == 0);
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      return c ? jit_blocks_per_sm(mode == 0 ? c->prune_dfs : c->prune_bfs, kThreads2) : 1;
    }
    default: return 1;
  }
}

int prune2_ring() { return kRing2; }
int prune3_stack() { return kStack3; }

int prune3_blocks_per_sm(SpecId id) {
  switch (id) {
    case SpecId::A51: return blocks3<A51>();
    case SpecId::MINI567: return blocks3<MINI567>();
    case SpecId::MINI789: return blocks3<MINI789>();
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return 1;
      cudaFuncSetAttribute(reinterpret_cast<const void*>(c->prune3_dfs), cudaFuncAttributeMaxDynamicSharedMemorySize,
                           kStack3Bytes);
      return jit_blocks_per_sm(c->prune3_dfs, kThreads3, kStack3Bytes);
    }
    default: return 1;
  }
}

uint32_t prune3_max_limit() { return kSpill3Max; }
int prune3_threads() { return kThreads3; }

uint64_t prune3_spill_bytes(int blocks, uint32_t limit) {
  return static_cast<uint64_t>(blocks) * kThreads3 * limit * sizeof(uint4);
}

cudaError_t launch_probe_expand(SpecId id, uint32_t F, const uint64_t* fnode, const uint32_t* fowner,
                                const unsigned long long* cur_count, const uint8_t* status, uint64_t* nnode,
                                uint32_t* nowner, unsigned long long* next_count, unsigned long long cap,
                                unsigned long long* lvl, unsigned int* overflow, int blocks, cudaStream_t st) {
  switch (id) {
#define LC_PROBE_LAUNCH(SP)                                                                                        \
  probe_expand_kernel<SP><<<blocks, kProbeThreads, 0, st>>>(fnode, fowner, cur_count, status, F, nnode, nowner, \
                                                            next_count, cap, lvl, overflow);                     \
  break;
    case SpecId::A51: LC_PROBE_LAUNCH(A51)
    case SpecId::MINI567: LC_PROBE_LAUNCH(MINI567)
    case SpecId::MINI789: LC_PROBE_LAUNCH(MINI789)
#undef LC_PROBE_LAUNCH
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return cudaErrorInvalidValue;
      return jit_launch(c->probe_expand, blocks, kProbeThreads, 0, st, fnode, fowner, cur_count, status, F, nnode,
                        nowner, next_count, cap, lvl, overflow);
    }
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_probe_finalize(uint32_t k, uint32_t level, unsigned long long* lvl, uint8_t* status,
                                  uint64_t* depth, uint64_t* nodes, unsigned long long* level_counts,
                                  uint32_t levels_cap, int64_t node_cap, const unsigned int* overflow,
                                  unsigned long long* live, unsigned long long* done_count,
                                  unsigned long long* cnt_reset, unsigned long long* live_reset, cudaStream_t st) {
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((k + 255) / 256, 1024));
  probe_finalize_kernel<<<g ? g : 1, 256, 0, st>>>(k, level, lvl, status, depth, nodes, level_counts, levels_cap,
                                                  node_cap, overflow, live, done_count, cnt_reset, live_reset);
  return cudaGetLastError();
}

cudaError_t launch_probe_censor(uint32_t k, uint8_t* status, cudaStream_t st) {
  const unsigned g = static_cast<unsigned>(std::min<uint64_t>((k + 255) / 256, 1024));
  probe_censor_kernel<<<g ? g : 1, 256, 0, st>>>(k, status);
  return cudaGetLastError();
}

cudaError_t launch_prune3(SpecId id, uint32_t F, int mode, uint32_t limit, const uint64_t* cands, uint64_t n,
                          uint8_t* removed, uint64_t* work, unsigned long long* queue, void* spill, int blocks,
                          cudaStream_t stream) {
  uint4* sp = static_cast<uint4*>(spill);
  const void* k = nullptr;
  switch (id) {
    case SpecId::A51: k = kernel3<A51>(mode == 0); break;
    case SpecId::MINI567: k = kernel3<MINI567>(mode == 0); break;
    case SpecId::MINI789: k = kernel3<MINI789>(mode == 0); break;
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return cudaErrorInvalidValue;
      k = reinterpret_cast<const void*>(mode == 0 ? c->prune3_dfs : c->prune3_bfs);
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, kStack3Bytes);
      break;
    }
    default: return cudaErrorInvalidValue;
  }
  uint32_t cap = limit;
  void* args[] = {&cands, &n, &F, &limit, &removed, &work, &queue, &sp, &cap};
  return cudaLaunchKernel(k, blocks, kThreads3, args, kStack3Bytes, stream);
}

uint64_t prune2_spill_bytes(int blocks, uint32_t cap) {
  return static_cast<uint64_t>(blocks) * kThreads2 * cap * (8 + 2) + 512;
}

cudaError_t launch_prune2(SpecId id, uint32_t F, int mode, uint64_t limit, const uint64_t* cands, uint64_t n,
                          uint8_t* removed, uint64_t* work, unsigned long long* queue, void* spill,
                          uint32_t spill_cap, int blocks, cudaStream_t stream) {
  uint64_t* spill_node = spill ? static_cast<uint64_t*>(spill) : nullptr;
  uint16_t* spill_dm =
      spill ? reinterpret_cast<uint16_t*>(spill_node + static_cast<uint64_t>(blocks) * kThreads2 * spill_cap) : nullptr;
#define LC_PRUNE2_LAUNCH(SP)                                                                                   \
  if (mode == 0)                                                                                               \
    prune2_kernel<SP, kRing2, true><<<blocks, kThreads2, 0, stream>>>(cands, n, F, limit, removed, work, queue, \
                                                                      spill_node, spill_dm, spill_cap);        \
  else                                                                                                         \
    prune2_kernel<SP, kRing2, false><<<blocks, kThreads2, 0, stream>>>(cands, n, F, limit, removed, work,      \
                                                                       queue, spill_node, spill_dm, spill_cap);
  switch (id) {
    case SpecId::A51: LC_PRUNE2_LAUNCH(A51) break;
    case SpecId::MINI567: LC_PRUNE2_LAUNCH(MINI567) break;
    case SpecId::MINI789: LC_PRUNE2_LAUNCH(MINI789) break;
    case SpecId::CUSTOM: {
      const CustomKernels* c = current_custom();
      if (!c) return cudaErrorInvalidValue;
      return jit_launch(mode == 0 ? c->prune_dfs : c->prune_bfs, blocks, kThreads2, 0, stream, cands, n, F, limit,
                        removed, work, queue, spill_node, spill_dm, spill_cap);
    }
    default: return cudaErrorInvalidValue;
  }
#undef LC_PRUNE2_LAUNCH
  return cudaGetLastError();
}

#endif  // !__CUDACC_RTC__

}  // namespace lc
