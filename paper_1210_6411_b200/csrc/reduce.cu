// Steps 4-5 on the GPU: the edge-output sort, iterative leaf
// cutting (reduce.cut_leaves_pass / cut_leaves_to_fixpoint, reduce.py:118-223) and cycle
// counting (reduce.count_cycles, reduce.py:226-266) on skeleton-edge records held in HBM.
//
// Records are SoA u64 arrays (source, destination, distance, subtree_size, subtree_depth),
// sorted ascending by unique source -- the file format's invariant (records.py:3-5).
// Destinations are resolved once to record indices by binary search; every pass is then
// a handful of streaming kernels: mark in-degree, fold each leaf's (size+1, depth+1) into
// its destination with atomics (leaves are never targets within a pass, so the reads are
// stable), and a stable compaction that also remaps destination indices; once the
// frontier fits in shared memory one block runs the remaining passes (cut_tail_kernel),
// a block barrier per pass instead of two launches.  The result is
// the reference's fixpoint and per-pass statistics exactly, without external sorts.
// Cycles: pointer jumping labels every record with the smallest index on its cycle (the
// smallest source, since sources ascend), then one atomic fold per record.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lfsr_internal.h"

namespace lc {

namespace {

constexpr int kT = 256;
constexpr uint64_t kNone = ~0ull;
constexpr int kTileShift = 12;  // compaction tile: 4096 records
constexpr uint64_t kTile = 1ull << kTileShift;

inline unsigned grid_for(uint64_t n) {
  const uint64_t g = (n + kT - 1) / kT;
  return static_cast<unsigned>(g == 0 ? 1 : (g > (1u << 22) ? (1u << 22) : g));
}

#define GRID_STRIDE(i, n)                                                             \
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < (n); \
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)

__global__ void check_sorted_kernel(const uint64_t* __restrict__ src, uint64_t n, unsigned int* err) {
  GRID_STRIDE(i, n) {
    if (i + 1 < n && src[i] >= src[i + 1]) atomicExch(err, 1u);
  }
}

// Destination -> record index by binary search over the sorted sources, narrowed by a
// directory of the B bits below the sources' common prefix: dir[b] = first record whose
// bucket is >= b (the sources' highest varying bit is the highest bit of src[0] ^
// src[n-1]), so a search covers one bucket (~n / 2^B records) instead of all n.
__device__ __forceinline__ uint32_t dir_shift(const uint64_t* __restrict__ src, uint64_t n, int B) {
  const uint64_t x = src[0] ^ src[n - 1];
  const int top = x ? 64 - __clzll(static_cast<long long>(x)) : 0;  // varying bits [0, top)
  return top > B ? static_cast<uint32_t>(top - B) : 0u;
}

__global__ void dir_build_kernel(const uint64_t* __restrict__ src, uint64_t n, int B, uint64_t* __restrict__ dir) {
  const uint32_t sh = dir_shift(src, n, B);
  const uint64_t bm = (1ull << B) - 1ull;
  GRID_STRIDE(i, n) {
    const uint64_t b = (src[i] >> sh) & bm;
    const uint64_t from = i ? ((src[i - 1] >> sh) & bm) + 1ull : 0ull;
    for (uint64_t t = from; t <= b; ++t) dir[t] = i;  // (an unsorted input is rejected anyway)
    if (i + 1 == n)
      for (uint64_t t = b + 1; t <= bm + 1; ++t) dir[t] = n;
  }
}

__global__ void resolve_kernel(const uint64_t* __restrict__ src, uint64_t n, const uint64_t* __restrict__ dst,
                               uint64_t* __restrict__ idx, int B, const uint64_t* __restrict__ dir) {
  const uint32_t sh = B ? dir_shift(src, n, B) : 0u;
  const uint64_t bm = (1ull << B) - 1ull;
  GRID_STRIDE(i, n) {
    const uint64_t v = dst[i];
    uint64_t lo = 0, hi = n;
    if (B) {
      const uint64_t b = (v >> sh) & bm;
      lo = dir[b];
      hi = dir[b + 1];
    }
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (src[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    idx[i] = (lo < n && src[lo] == v) ? lo : kNone;
  }
}

// directory bits for n records: ~4-16 records per bucket, the directory within n entries
inline int dir_bits(uint64_t n) {
  if (n < (1ull << 12)) return 0;
  const int lg = 63 - __builtin_clzll(n);  // floor(log2 n)
  return std::min(20, lg - 2);
}

__global__ void tile_count_kernel(const uint8_t* __restrict__ keep, uint64_t n, uint64_t* __restrict__ counts) {
  const uint64_t lo = blockIdx.x * kTile, hi = min(n, lo + kTile);
  uint32_t c = 0;
  for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += keep[i] ? 1u : 0u;
  c = __reduce_add_sync(0xffffffffu, c);
  __shared__ uint32_t part[kT / 32];
  if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint64_t s = 0;
    for (int w = 0; w < kT / 32; ++w) s += part[w];
    counts[blockIdx.x] = s;
  }
}

// Exclusive scan in place, counts[tiles] = total (one block).
__global__ void tile_scan_kernel(uint64_t* __restrict__ counts, uint64_t tiles) {
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
  }
  __syncthreads();
  uint64_t run = part[threadIdx.x];
  for (uint64_t i = lo; i < hi; ++i) {
    const uint64_t v = counts[i];
    counts[i] = run;
    run += v;
  }
}

// newpos[i] = rank of i among kept records (order preserved); kNone for dropped ones.
__global__ void rank_kernel(const uint8_t* __restrict__ keep, uint64_t n, const uint64_t* __restrict__ offsets,
                            uint64_t* __restrict__ newpos) {
  __shared__ uint32_t wcount[kT / 32];
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  const uint64_t lo = blockIdx.x * kTile, hi = min(n, lo + kTile);
  uint64_t pos = offsets[blockIdx.x];
  for (uint64_t r = lo; r < hi; r += kT) {
    const uint64_t i = r + threadIdx.x;
    const bool k = i < hi && keep[i];
    const uint32_t b = __ballot_sync(0xffffffffu, k);
    if (lane == 0) wcount[warp] = __popc(b);
    __syncthreads();
    uint32_t before = 0, all = 0;
#pragma unroll
    for (int w = 0; w < kT / 32; ++w) {
      const uint32_t v = wcount[w];
      before += (static_cast<uint32_t>(w) < warp) ? v : 0u;
      all += v;
    }
    if (i < hi) newpos[i] = k ? pos + before + __popc(b & ((1u << lane) - 1u)) : kNone;
    pos += all;
    __syncthreads();
  }
}

// ---- leaf cutting (step 4) as a frontier computation.  A record is a leaf of pass p iff
// no record alive after pass p-1 points at it, i.e. its in-degree among alive records is
// zero.  Removing the leaves of pass p decrements their destinations' in-degrees; the
// records that reach zero are exactly the leaves of pass p+1.  So each pass touches only
// its own leaves (total work O(n) over all passes instead of O(n) per pass), and the
// (size + 1, depth + 1) folds are order-independent atomics (sum, max), which keeps the
// result deterministic although frontier order is not.  Pass statistics need no scans:
// with L_p leaves, inner_nodes = alive - L_p and the survivors' subtree-size sum grows by
// exactly L_p (each leaf's size moves into its destination, plus one for the leaf).

// Loop whose index base is shared by the 32 lanes of a warp, so warp collectives inside
// see every lane (lanes past the end run with an out-of-range index).
#define WARP_STRIDE(i0, n)                                                                 \
  for (uint64_t i0 = (blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x) & ~31ull; \
       i0 < (n); i0 += static_cast<uint64_t>(gridDim.x) * blockDim.x)

// Warp-aggregated append: one atomic per warp.  All 32 lanes must call it.
__device__ __forceinline__ void warp_append(bool push, uint64_t value, uint64_t* __restrict__ list,
                                            unsigned long long* count) {
  const uint32_t m = __ballot_sync(0xffffffffu, push);
  if (m == 0) return;
  const uint32_t lane = threadIdx.x & 31u;
  const int leader = __ffs(m) - 1;
  unsigned long long base = 0;
  if (static_cast<int>(lane) == leader) base = atomicAdd(count, static_cast<unsigned long long>(__popc(m)));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (push) list[base + __popc(m & ((1u << lane) - 1u))] = value;
}

__device__ __forceinline__ uint64_t find_source(const uint64_t* __restrict__ src, uint64_t n, uint64_t v) {
  uint64_t lo = 0, hi = n;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (src[mid] < v) lo = mid + 1;
    else hi = mid;
  }
  return (lo < n && src[lo] == v) ? lo : kNone;
}

__global__ void indeg_count_kernel(const uint64_t* __restrict__ idx, uint64_t n, unsigned int* __restrict__ indeg) {
  GRID_STRIDE(i, n) {
    const uint64_t j = idx[i];
    if (j != kNone) atomicAdd(&indeg[j], 1u);
  }
}

__global__ void frontier_init_kernel(const unsigned int* __restrict__ indeg, uint64_t n, uint64_t* __restrict__ f,
                                     unsigned long long* cnt) {
  WARP_STRIDE(i0, n) {
    const uint64_t i = i0 + (threadIdx.x & 31u);
    warp_append(i < n && indeg[i] == 0u, i, f, cnt);
  }
}

__global__ void sum_kernel(const uint64_t* __restrict__ v, uint64_t n, unsigned long long* out) {
  uint64_t s = 0;
  GRID_STRIDE(i, n) { s += v[i]; }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, static_cast<unsigned long long>(s));
}

// Remove the leaves of the current pass (frontier fcur) and fold them into their
// destinations; destinations whose in-degree drops to zero form the next frontier.
__global__ void cut_fold_kernel(CutCtl* ctl, int w, const uint64_t* __restrict__ fcur, uint64_t* __restrict__ fnext,
                                const uint64_t* __restrict__ idx, unsigned long long* size,
                                unsigned long long* depth, unsigned int* indeg, uint8_t* __restrict__ alive,
                                unsigned int* err) {
  const uint64_t m = ctl->cnt[w];
  WARP_STRIDE(k0, m) {
    const uint64_t k = k0 + (threadIdx.x & 31u);
    bool push = false;
    uint64_t j = kNone;
    if (k < m) {
      const uint64_t i = fcur[k];
      alive[i] = 0;
      j = idx[i];
      if (j == kNone) {
        atomicExch(err, 2u);  // aggregate with no surviving record: input not closed
      } else {
        atomicAdd(&size[j], size[i] + 1ull);  // i is a leaf: nothing folds into it this pass
        atomicMax(&depth[j], depth[i] + 1ull);
        push = atomicSub(&indeg[j], 1u) == 1u;
      }
    }
    warp_append(push, j, fnext, &ctl->cnt[w ^ 1]);
  }
}

__global__ void cut_pass_end_kernel(CutCtl* ctl, int w, uint64_t* __restrict__ pstats, uint64_t max_stats) {
  const unsigned long long leaves = ctl->cnt[w];
  const unsigned long long p = ++ctl->pass;
  if (p - 1 < max_stats) {
    pstats[3 * (p - 1) + 0] = leaves;
    pstats[3 * (p - 1) + 1] = ctl->alive - leaves;
    pstats[3 * (p - 1) + 2] = ctl->sum + leaves;
  }
  ctl->alive -= leaves;
  ctl->sum += leaves;
  ctl->cnt[w] = 0;
  if (leaves == 0 && ctl->done_at == 0) ctl->done_at = p;
}

// The tail of a cut: a frontier never grows (each new leaf is the destination of at least
// one leaf of the pass before), so once it fits in shared memory one block runs the
// passes itself -- the fold, a block barrier, the pass bookkeeping of cut_pass_end_kernel
// -- instead of two launches per pass.  Entered at parity 0 (after the graph's two wide
// passes); runs passes in pairs so it leaves at parity 0, until the fixpoint or `budget`
// passes.  Sizes and depths are read at L2 (ld.cg): earlier passes of this kernel changed
// them by atomics, which the L1 would not see.  A frontier entry carries its record's
// destination, loaded while the pass that made it a leaf waits on its in-degree atomic,
// so a pass's dependent chain is one L2 atomic round trip rather than a load and then one.
// the next hop's lines into L2 while this pass waits on its atomics: the new leaf j's
// destination jj is folded into (and its in-degree dropped) in the next pass
#ifndef LC_CUT_TAIL_PREFETCH
#define LC_CUT_TAIL_PREFETCH 1
#endif
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }
__device__ __forceinline__ void prefetch_hop(uint64_t jj, const uint64_t* idx, const unsigned long long* size,
                                             const unsigned long long* depth, const unsigned int* indeg) {
#if LC_CUT_TAIL_PREFETCH
  if (jj != kNone) {
    prefetch_l2(indeg + jj);
    prefetch_l2(size + jj);
    prefetch_l2(depth + jj);
    prefetch_l2(idx + jj);
  }
#endif
}

constexpr int kTailThreads = 1024;
constexpr uint32_t kTailMax = 6144;  // frontier entries per buffer (2 x 96 KB of shared memory)
constexpr size_t kTailSmem = 2 * kTailMax * sizeof(ulonglong2);
#ifndef LC_CUT_TAIL_WARP
#define LC_CUT_TAIL_WARP 1
#endif
constexpr bool kTailWarpMode = LC_CUT_TAIL_WARP != 0;  // frontiers of <= 32: warp 0 alone

__global__ void __launch_bounds__(kTailThreads) cut_tail_kernel(CutCtl* ctl, uint64_t* __restrict__ f0,
                                                                const uint64_t* __restrict__ idx,
                                                                unsigned long long* size, unsigned long long* depth,
                                                                unsigned int* indeg, uint8_t* __restrict__ alive,
                                                                unsigned int* err, uint64_t* __restrict__ pstats,
                                                                uint64_t max_stats, uint32_t budget) {
  const unsigned long long m0 = ctl->cnt[0];
  if (m0 > kTailMax || ctl->done_at) return;  // still wide, or past the fixpoint
  extern __shared__ ulonglong2 tf[];          // [2][kTailMax]: (record, its destination)
  // frontier sizes rotate over three counters, so one barrier per pass suffices: pass q
  // reads tcnt[q % 3], appends to tcnt[(q + 1) % 3] and clears tcnt[(q + 2) % 3] (read
  // by pass q - 1, before the last barrier; appended to by pass q + 1, after the next)
  __shared__ unsigned int tcnt[3];
  const int tid = threadIdx.x;
  for (uint32_t k = tid; k < m0; k += kTailThreads) {
    const uint64_t i = f0[k];
    tf[k] = make_ulonglong2(i, idx[i]);
  }
  unsigned long long t_alive = 0, t_sum = 0, t_pass = 0, t_done = 0;  // thread 0's bookkeeping
  if (tid == 0) {
    tcnt[0] = static_cast<unsigned int>(m0);
    tcnt[1] = tcnt[2] = 0;
    t_alive = ctl->alive;
    t_sum = ctl->sum;
    t_pass = ctl->pass;
  }
  __syncthreads();
  // cut_pass_end_kernel's bookkeeping for a pass that removed m records (thread 0)
  auto close_pass = [&](uint32_t m) {
    const unsigned long long p = ++t_pass;
    if (p - 1 < max_stats) {
      pstats[3 * (p - 1) + 0] = m;
      pstats[3 * (p - 1) + 1] = t_alive - m;
      pstats[3 * (p - 1) + 2] = t_sum + m;
    }
    t_alive -= m;
    t_sum += m;
    if (m == 0 && t_done == 0) t_done = p;
  };
  bool done = false, narrow = false;
  uint32_t q = 0;
  while (q < budget) {
    const int w = static_cast<int>(q & 1u), c = static_cast<int>(q % 3u);
    const uint32_t m = tcnt[c];
    if (m <= 32u && kTailWarpMode) {  // block-uniform; a frontier never grows again
      narrow = true;
      break;
    }
    const ulonglong2* fc = tf + w * kTailMax;
    ulonglong2* fn = tf + (w ^ 1) * kTailMax;
    unsigned int* cnext = &tcnt[(c + 1) % 3];
    for (uint32_t k = tid; k < m; k += kTailThreads) {
      const uint64_t i = fc[k].x, j = fc[k].y;
      alive[i] = 0;
      if (j == kNone) {
        atomicExch(err, 2u);
      } else {
        const uint64_t jj = idx[j];  // in flight with the in-degree atomic
        const bool leaf = atomicSub(&indeg[j], 1u) == 1u;
        atomicAdd(&size[j], __ldcg(&size[i]) + 1ull);
        atomicMax(&depth[j], __ldcg(&depth[i]) + 1ull);
        if (leaf) {
          prefetch_hop(jj, idx, size, depth, indeg);
          fn[atomicAdd(cnext, 1u)] = make_ulonglong2(j, jj);
        }
      }
    }
    if (tid == 0) {
      close_pass(m);
      tcnt[(c + 2) % 3] = 0;
    }
    done |= m == 0;  // block-uniform
    __syncthreads();
    ++q;
    if (done && !(q & 1u)) break;  // leave at parity 0
  }
  // At most 32 leaves left per pass: warp 0 runs the remaining passes alone, one leaf per
  // lane, the next frontier compacted into lanes by a ballot -- no shared-memory counters,
  // no block barriers, only the warp's own synchronisation between passes.
  __shared__ uint32_t q_end;
  if (narrow && tid < 32) {
    const uint32_t lane = tid;
    uint32_t m = tcnt[q % 3u];
    ulonglong2 e = lane < m ? tf[(q & 1u) * kTailMax + lane] : make_ulonglong2(0ull, kNone);
    bool have = lane < m;
    while (q < budget) {
      bool push = false;
      uint64_t j = 0, jj = 0;
      if (have) {
        const uint64_t i = e.x;
        j = e.y;
        alive[i] = 0;
        if (j == kNone) {
          atomicExch(err, 2u);
        } else {
          jj = idx[j];
          push = atomicSub(&indeg[j], 1u) == 1u;
          atomicAdd(&size[j], __ldcg(&size[i]) + 1ull);
          atomicMax(&depth[j], __ldcg(&depth[i]) + 1ull);
          if (push) prefetch_hop(jj, idx, size, depth, indeg);
        }
      }
      const uint32_t pushed = __ballot_sync(0xffffffffu, push);
      const uint32_t from = __fns(pushed, 0, lane + 1);  // the lane with the (lane+1)-th push
      const uint32_t src_lane = from < 32u ? from : 0u;
      e.x = __shfl_sync(0xffffffffu, j, src_lane);
      e.y = __shfl_sync(0xffffffffu, jj, src_lane);
      if (lane == 0) close_pass(m);
      done |= m == 0;
      m = __popc(pushed);
      have = lane < m;
      __syncwarp();  // this pass's folds before the next pass's reads
      ++q;
      if (done && !(q & 1u)) break;
    }
    if (have) tf[lane] = e;  // parity 0: buffer 0
    if (lane == 0) {
      tcnt[q % 3u] = m;
      q_end = q;
    }
  } else if (!narrow && tid == 0) {
    q_end = q;
  }
  __syncthreads();
  q = q_end;
  const uint32_t mq = tcnt[q % 3];
  for (uint32_t k = tid; k < mq; k += kTailThreads) f0[k] = tf[k].x;
  if (tid == 0) {
    ctl->cnt[0] = mq;
    ctl->cnt[1] = 0;
    ctl->alive = t_alive;
    ctl->sum = t_sum;
    ctl->pass = t_pass;
    ctl->done_at = t_done;
  }
}

// ---- sharded leaf cutting (multi-GPU step 4).  Each rank holds one contiguous source
// range; a record's destination may live on any rank, so in-degree counts and folds travel
// as 3-word messages (destination, size + 1, depth + 1) grouped by owner rank, exchanged
// with one all-to-all per pass by the host driver, and applied by the owner, which
// resolves the destination by binary search over its own sources.

__device__ __forceinline__ uint32_t owner_of(uint64_t v, const uint64_t* __restrict__ bounds,
                                             const uint32_t* __restrict__ brank, uint32_t nb) {
  uint32_t lo = 0, hi = nb;  // one past the last entry with bounds[e] <= v (bounds[0] == 0)
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (bounds[mid] <= v) lo = mid + 1;
    else hi = mid;
  }
  return brank[lo - 1];
}

struct EmitArgs {
  int phase;                    // 0: in-degree messages for every record, 1: the frontier's folds
  uint64_t n;                   // records (phase 0)
  const CutCtl* ctl;            // frontier count (phase 1)
  int w;                        // current frontier parity
  const uint64_t* frontier;
  const uint64_t* dst;
  const unsigned long long* size;
  const unsigned long long* depth;
  uint8_t* alive;
  const uint64_t* bounds;
  const uint32_t* brank;
  uint32_t nb, n_ranks;
  unsigned long long* ocount;   // [n_ranks] messages per owner
  unsigned long long* ocursor;  // [n_ranks]
  uint64_t* msgs;               // [3 * items], grouped by owner rank
};

__device__ __forceinline__ uint64_t emit_items(const EmitArgs& a) { return a.phase ? a.ctl->cnt[a.w] : a.n; }

__global__ void emit_count_kernel(EmitArgs a) {
  __shared__ unsigned int h[kMaxShardRanks];
  for (uint32_t r = threadIdx.x; r < a.n_ranks; r += blockDim.x) h[r] = 0;
  __syncthreads();
  const uint64_t m = emit_items(a);
  GRID_STRIDE(k, m) {
    const uint64_t i = a.phase ? a.frontier[k] : k;
    atomicAdd(&h[owner_of(a.dst[i], a.bounds, a.brank, a.nb)], 1u);
  }
  __syncthreads();
  for (uint32_t r = threadIdx.x; r < a.n_ranks; r += blockDim.x)
    if (h[r]) atomicAdd(&a.ocount[r], static_cast<unsigned long long>(h[r]));
}

__global__ void emit_write_kernel(EmitArgs a) {
  __shared__ unsigned long long off[kMaxShardRanks];
  if (threadIdx.x == 0) {
    unsigned long long run = 0;
    for (uint32_t r = 0; r < a.n_ranks; ++r) {
      off[r] = run;
      run += a.ocount[r];
    }
  }
  __syncthreads();
  const uint64_t m = emit_items(a);
  const uint32_t lane = threadIdx.x & 31u;
  WARP_STRIDE(k0, m) {
    const uint64_t k = k0 + lane;
    const bool valid = k < m;
    uint64_t i = 0;
    uint32_t o = 0xffffffffu;
    if (valid) {
      i = a.phase ? a.frontier[k] : k;
      o = owner_of(a.dst[i], a.bounds, a.brank, a.nb);
    }
    // one cursor atomic per (warp, owner) group
    const uint32_t peers = __match_any_sync(0xffffffffu, o);
    const int leader = __ffs(peers) - 1;
    unsigned long long base = 0;
    if (valid && static_cast<int>(lane) == leader)
      base = atomicAdd(&a.ocursor[o], static_cast<unsigned long long>(__popc(peers)));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (valid) {
      const uint64_t slot = off[o] + base + __popc(peers & ((1u << lane) - 1u));
      uint64_t* q = a.msgs + 3 * slot;
      q[0] = a.dst[i];
      q[1] = a.phase ? a.size[i] + 1ull : 0ull;
      q[2] = a.phase ? a.depth[i] + 1ull : 0ull;
      if (a.phase) a.alive[i] = 0;
    }
  }
}

// Phase 0: count in-degrees.  Phase 1: fold, and collect the records whose in-degree
// reaches zero into the next frontier.
__global__ void apply_kernel(int phase, const uint64_t* __restrict__ msgs, uint64_t m,
                             const uint64_t* __restrict__ src, uint64_t n, unsigned int* indeg,
                             unsigned long long* size, unsigned long long* depth, uint64_t* __restrict__ fnext,
                             unsigned long long* cnt_next, unsigned int* err) {
  WARP_STRIDE(k0, m) {
    const uint64_t k = k0 + (threadIdx.x & 31u);
    bool push = false;
    uint64_t j = kNone;
    if (k < m) {
      j = find_source(src, n, msgs[3 * k]);
      if (phase == 0) {
        if (j != kNone) atomicAdd(&indeg[j], 1u);
      } else if (j == kNone) {
        atomicExch(err, 2u);
      } else {
        atomicAdd(&size[j], static_cast<unsigned long long>(msgs[3 * k + 1]));
        atomicMax(&depth[j], static_cast<unsigned long long>(msgs[3 * k + 2]));
        push = atomicSub(&indeg[j], 1u) == 1u;
      }
    }
    if (phase) warp_append(push, j, fnext, cnt_next);
  }
}

// ------------------------------------------------------------------ cycles (step 5)

__global__ void indeg_kernel(const uint64_t* __restrict__ idx, uint64_t n, unsigned int* __restrict__ indeg,
                             unsigned int* err) {
  GRID_STRIDE(i, n) {
    const uint64_t j = idx[i];
    if (j == kNone) atomicExch(err, 3u);  // destination is not a source
    else atomicAdd(&indeg[j], 1u);
  }
}

__global__ void perm_check_kernel(const unsigned int* __restrict__ indeg, uint64_t n, unsigned int* err) {
  GRID_STRIDE(i, n) {
    if (indeg[i] != 1u) atomicExch(err, 4u);  // not a permutation
  }
}

__global__ void label_init_kernel(const uint64_t* __restrict__ idx, uint64_t n, uint64_t* lab, uint64_t* nxt) {
  GRID_STRIDE(i, n) {
    lab[i] = i;
    nxt[i] = idx[i];
  }
}

__global__ void jump_kernel(const uint64_t* __restrict__ lab, const uint64_t* __restrict__ nxt, uint64_t n,
                            uint64_t* __restrict__ lab2, uint64_t* __restrict__ nxt2) {
  GRID_STRIDE(i, n) {
    const uint64_t j = nxt[i];
    lab2[i] = min(lab[i], lab[j]);
    nxt2[i] = nxt[j];
  }
}

__global__ void cycle_fold_kernel(const uint64_t* __restrict__ lab, uint64_t n, const uint64_t* __restrict__ dist,
                                  const uint64_t* __restrict__ size, unsigned long long* hops,
                                  unsigned long long* clocks, unsigned long long* tree) {
  GRID_STRIDE(i, n) {
    const uint64_t l = lab[i];
    atomicAdd(&hops[l], 1ull);
    atomicAdd(&clocks[l], static_cast<unsigned long long>(dist[i]));
    atomicAdd(&tree[l], static_cast<unsigned long long>(size[i]));
  }
}

__global__ void leader_flag_kernel(const uint64_t* __restrict__ lab, uint64_t n, uint8_t* __restrict__ flag) {
  GRID_STRIDE(i, n) { flag[i] = lab[i] == i ? 1 : 0; }
}

// to[newpos[i]] = from[i] for the selected rows
__global__ void select_kernel(const uint64_t* __restrict__ newpos, uint64_t n, const uint64_t* __restrict__ from,
                              uint64_t* __restrict__ to) {
  GRID_STRIDE(i, n) {
    const uint64_t p = newpos[i];
    if (p != kNone) to[p] = from[i];
  }
}

}  // namespace

// Scratch layout helper: allocate on demand from one buffer.
struct ReduceScratch {
  uint8_t* base;
  size_t used;
  template <class T>
  T* take(uint64_t count) {
    T* p = reinterpret_cast<T*>(base + used);
    used += (count * sizeof(T) + 255) & ~size_t(255);
    return p;
  }
};

size_t reduce_scratch_bytes(uint64_t n, uint32_t max_stats) {
  // err, control, pass stats, tile counts, idx, in-degree, alive flags, two frontiers
  const uint64_t tiles = (n + kTile - 1) / kTile + 1;
  return 16 * 256 + tiles * 8 + 3ull * (max_stats + 1) * 8 + n * (8 + 4 + 1 + 8 + 8) + 8 * 256;
}

namespace {

constexpr int kFoldGrid = 148 * 8;

// Stable compaction of the five record columns to the rows with flag != 0 (in place, via
// tmp); returns the surviving count on the host.
cudaError_t compact_records(uint64_t n, const uint8_t* flag, uint64_t* const cols[5], uint64_t* tiles_buf,
                            uint64_t* newpos, uint64_t* tmp, uint64_t* n_out, cudaStream_t st, int* launches) {
  const uint64_t tiles = (n + kTile - 1) / kTile;
  tile_count_kernel<<<static_cast<unsigned>(tiles), kT, 0, st>>>(flag, n, tiles_buf);
  tile_scan_kernel<<<1, 1024, 0, st>>>(tiles_buf, tiles);
  rank_kernel<<<static_cast<unsigned>(tiles), kT, 0, st>>>(flag, n, tiles_buf, newpos);
  *launches += 3;
  cudaError_t e;
  uint64_t m = 0;
  if ((e = cudaMemcpyAsync(&m, &tiles_buf[tiles], 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (m != n) {
    for (int k = 0; k < 5; ++k) {
      select_kernel<<<grid_for(n), kT, 0, st>>>(newpos, n, cols[k], tmp);
      ++*launches;
      if (m && (e = cudaMemcpyAsync(cols[k], tmp, m * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    }
  }
  *n_out = m;
  return cudaGetLastError();
}

}  // namespace

// Single-GPU leaf cutting: resolve destinations once, count in-degrees, then run passes
// of two kernels each (fold the frontier; close the pass).  max_passes > 0 launches that
// many passes directly; 0 runs to the fixpoint from a CUDA graph of two ping-pong passes,
// checking in with the host after 8, 16, 32 ... graph replays.  Passes after the fixpoint
// are no-ops, so overshooting is harmless.
cudaError_t cut_leaves_device(uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist, uint64_t* size,
                              uint64_t* depth, uint32_t max_passes, uint64_t* pass_stats, uint32_t max_stats,
                              uint32_t* n_passes, uint64_t* n_out, unsigned int* err_out, void* scratch,
                              cudaStream_t st, int* launches) {
  ReduceScratch s{static_cast<uint8_t*>(scratch), 0};
  unsigned int* err = s.take<unsigned int>(4);
  CutCtl* ctl = s.take<CutCtl>(1);
  const uint64_t stats_cap = max_stats ? max_stats : 1;
  uint64_t* pstats = s.take<uint64_t>(3 * stats_cap);
  uint64_t* tiles_buf = s.take<uint64_t>((n + kTile - 1) / kTile + 1);
  uint64_t* idx = s.take<uint64_t>(n);
  unsigned int* indeg = s.take<unsigned int>(n);
  uint8_t* alive = s.take<uint8_t>(n);
  uint64_t* f0 = s.take<uint64_t>(n);
  uint64_t* f1 = s.take<uint64_t>(n);
  cudaError_t e;
  *n_passes = 0;
  *n_out = n;
  *err_out = 0;
  if (n == 0) return cudaSuccess;
  auto* usize = reinterpret_cast<unsigned long long*>(size);
  auto* udepth = reinterpret_cast<unsigned long long*>(depth);
  if ((e = cudaMemsetAsync(err, 0, 16, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(ctl, 0, sizeof(CutCtl), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(indeg, 0, n * sizeof(unsigned int), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(alive, 1, n, st)) != cudaSuccess) return e;
  check_sorted_kernel<<<grid_for(n), kT, 0, st>>>(src, n, err);
  const int dbits = dir_bits(n);  // the directory lives in f1 until the passes start
  if (dbits) dir_build_kernel<<<grid_for(n), kT, 0, st>>>(src, n, dbits, f1);
  resolve_kernel<<<grid_for(n), kT, 0, st>>>(src, n, dst, idx, dbits, f1);
  indeg_count_kernel<<<grid_for(n), kT, 0, st>>>(idx, n, indeg);
  frontier_init_kernel<<<grid_for(n), kT, 0, st>>>(indeg, n, f0, &ctl->cnt[0]);
  sum_kernel<<<std::min(grid_for(n), 4096u), kT, 0, st>>>(size, n, &ctl->sum);
  *launches += dbits ? 6 : 5;
  const unsigned long long alive0 = n;
  if ((e = cudaMemcpyAsync(&ctl->alive, &alive0, 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  unsigned int herr = 0;
  if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (herr) {
    *err_out = herr;
    return cudaSuccess;
  }
  auto pass = [&](int w) {
    cut_fold_kernel<<<kFoldGrid, kT, 0, st>>>(ctl, w, w ? f1 : f0, w ? f0 : f1, idx, usize, udepth, indeg, alive,
                                              err);
    cut_pass_end_kernel<<<1, 1, 0, st>>>(ctl, w, pstats, max_stats);
  };
  constexpr int kLaunchesPerPass = 2;
  constexpr uint32_t kTailBudget = 1024;  // tail passes per graph replay (even)
  CutCtl h{};
  uint64_t executed = 0;
  if (max_passes != 0) {
    for (uint32_t k = 0; k < max_passes; ++k) pass(static_cast<int>(k & 1));
    *launches += kLaunchesPerPass * max_passes;
    executed = max_passes;
    if ((e = cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  } else {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if ((e = cudaFuncSetAttribute(cut_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kTailSmem))) != cudaSuccess)
      return e;
    if ((e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return e;
    pass(0);
    pass(1);
    cut_tail_kernel<<<1, kTailThreads, kTailSmem, st>>>(ctl, f0, idx, usize, udepth, indeg, alive, err, pstats, max_stats,
                                                        kTailBudget);
    if ((e = cudaStreamEndCapture(st, &graph)) != cudaSuccess) return e;
    if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return e;
    for (int batch = 8;; batch = std::min(batch * 2, 512)) {  // graphs (x2 passes) per host check-in
      for (int k = 0; k < batch; ++k)
        if ((e = cudaGraphLaunch(exec, st)) != cudaSuccess) break;
      if (e != cudaSuccess) break;
      *launches += batch * (2 * kLaunchesPerPass + 1);
      if ((e = cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
      if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) break;
      if ((e = cudaStreamSynchronize(st)) != cudaSuccess) break;
      if (herr || h.done_at) break;
    }
    cudaGraphExecDestroy(exec);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return e;
  }
  if (herr) {
    *err_out = herr;
    return cudaSuccess;
  }
  const uint64_t passes = h.done_at ? h.done_at : (max_passes != 0 ? executed : h.pass);
  *n_passes = static_cast<uint32_t>(passes);
  const uint64_t keep_stats = std::min<uint64_t>(passes, max_stats);
  if (keep_stats)
    if ((e = cudaMemcpyAsync(pass_stats, pstats, keep_stats * 3 * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return e;
  uint64_t* cols[5] = {src, dst, dist, size, depth};
  return compact_records(n, alive, cols, tiles_buf, f0, f1, n_out, st, launches);
}

// ---- sharded leaf cutting: per-rank state and the three host-called steps.

size_t shard_scratch_bytes(uint64_t n, uint32_t n_ranks) {
  const uint64_t tiles = (n + kTile - 1) / kTile + 1;
  return 16 * 256 + tiles * 8 + 4ull * n_ranks * 8 + 2 * 256 + n * (4 + 1 + 8 + 8) + 8 * 256;
}

cudaError_t shard_init(ShardState* sh, void* scratch, uint64_t n, uint64_t* const cols[5], uint32_t n_ranks,
                       const uint64_t* rank_first, const uint64_t* rank_count, uint64_t* size_sum,
                       unsigned int* err_out, cudaStream_t st, int* launches) {
  ReduceScratch s{static_cast<uint8_t*>(scratch), 0};
  sh->n = n;
  for (int k = 0; k < 5; ++k) sh->cols[k] = cols[k];
  sh->n_ranks = n_ranks;
  sh->err = s.take<unsigned int>(4);
  sh->ctl = s.take<CutCtl>(1);
  sh->tiles = s.take<uint64_t>((n + kTile - 1) / kTile + 1);
  sh->bounds = s.take<uint64_t>(n_ranks);
  sh->brank = s.take<uint32_t>(n_ranks);
  sh->ocount = s.take<unsigned long long>(n_ranks);
  sh->ocursor = s.take<unsigned long long>(n_ranks);
  sh->indeg = s.take<unsigned int>(n);
  sh->alive = s.take<uint8_t>(n);
  sh->f[0] = s.take<uint64_t>(n);
  sh->f[1] = s.take<uint64_t>(n);
  sh->w = 0;
  sh->started = false;
  // owner table over the non-empty ranks; the first bound is 0 so every value has an owner
  uint64_t hb[kMaxShardRanks];
  uint32_t hr[kMaxShardRanks];
  uint32_t nb = 0;
  for (uint32_t r = 0; r < n_ranks; ++r) {
    if (rank_count[r] == 0) continue;
    hb[nb] = nb == 0 ? 0 : rank_first[r];
    hr[nb] = r;
    ++nb;
  }
  if (nb == 0) {  // every shard empty: a single owner so the tables stay well-formed
    hb[0] = 0;
    hr[0] = 0;
    nb = 1;
  }
  sh->nb = nb;
  cudaError_t e;
  *err_out = 0;
  *size_sum = 0;
  if ((e = cudaMemcpyAsync(sh->bounds, hb, nb * 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(sh->brank, hr, nb * 4, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sh->err, 0, 16, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sh->ctl, 0, sizeof(CutCtl), st)) != cudaSuccess) return e;
  if (n) {
    if ((e = cudaMemsetAsync(sh->indeg, 0, n * 4, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(sh->alive, 1, n, st)) != cudaSuccess) return e;
    check_sorted_kernel<<<grid_for(n), kT, 0, st>>>(cols[0], n, sh->err);
    sum_kernel<<<std::min(grid_for(n), 4096u), kT, 0, st>>>(cols[3], n, &sh->ctl->sum);
    *launches += 2;
  }
  unsigned long long hs = 0;
  if ((e = cudaMemcpyAsync(&hs, &sh->ctl->sum, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaMemcpyAsync(err_out, sh->err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *size_sum = hs;
  return cudaGetLastError();
}

cudaError_t shard_emit(ShardState* sh, int phase, uint64_t* send, uint64_t* counts, uint64_t* info,
                       cudaStream_t st, int* launches) {
  cudaError_t e;
  if (phase && !sh->started) {  // all in-degree messages have been applied: first frontier
    if (sh->n) {
      frontier_init_kernel<<<grid_for(sh->n), kT, 0, st>>>(sh->indeg, sh->n, sh->f[0], &sh->ctl->cnt[0]);
      ++*launches;
    }
    sh->started = true;
  }
  if ((e = cudaMemsetAsync(sh->ocount, 0, sh->n_ranks * 8ull, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(sh->ocursor, 0, sh->n_ranks * 8ull, st)) != cudaSuccess) return e;
  if (phase && (e = cudaMemsetAsync(&sh->ctl->cnt[sh->w ^ 1], 0, 8, st)) != cudaSuccess) return e;
  EmitArgs a{phase,
             sh->n,
             sh->ctl,
             sh->w,
             sh->f[sh->w],
             sh->cols[1],
             reinterpret_cast<const unsigned long long*>(sh->cols[3]),
             reinterpret_cast<const unsigned long long*>(sh->cols[4]),
             sh->alive,
             sh->bounds,
             sh->brank,
             sh->nb,
             sh->n_ranks,
             sh->ocount,
             sh->ocursor,
             send};
  const unsigned g = phase ? static_cast<unsigned>(kFoldGrid) : std::min(grid_for(sh->n), 4096u);
  emit_count_kernel<<<g, kT, 0, st>>>(a);
  emit_write_kernel<<<g, kT, 0, st>>>(a);
  *launches += 2;
  unsigned long long items = 0;
  unsigned int herr = 0;
  if ((e = cudaMemcpyAsync(counts, sh->ocount, sh->n_ranks * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if (phase && (e = cudaMemcpyAsync(&items, &sh->ctl->cnt[sh->w], 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
    return e;
  if ((e = cudaMemcpyAsync(&herr, sh->err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  info[0] = phase ? items : sh->n;
  info[1] = herr;
  return cudaGetLastError();
}

cudaError_t shard_apply(ShardState* sh, int phase, const uint64_t* msgs, uint64_t m, cudaStream_t st,
                        int* launches) {
  if (m) {
    const unsigned g = std::min(grid_for(m), phase ? static_cast<unsigned>(kFoldGrid) : 4096u);
    apply_kernel<<<g, kT, 0, st>>>(phase, msgs, m, sh->cols[0], sh->n, sh->indeg,
                                   reinterpret_cast<unsigned long long*>(sh->cols[3]),
                                   reinterpret_cast<unsigned long long*>(sh->cols[4]), sh->f[sh->w ^ 1],
                                   &sh->ctl->cnt[sh->w ^ 1], sh->err);
    ++*launches;
  }
  if (phase) sh->w ^= 1;  // the frontier just filled is the next pass's
  return cudaGetLastError();
}

cudaError_t shard_finish(ShardState* sh, uint64_t* n_out, unsigned int* err_out, cudaStream_t st, int* launches) {
  cudaError_t e;
  *n_out = sh->n;
  if ((e = cudaMemcpyAsync(err_out, sh->err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (*err_out || sh->n == 0) return cudaSuccess;
  return compact_records(sh->n, sh->alive, sh->cols, sh->tiles, sh->f[0], sh->f[1], n_out, st, launches);
}

size_t cycles_scratch_bytes(uint64_t n) { return 10 * n * 8 + n + ((n + kTile - 1) / kTile + 1) * 8 + 8192; }

cudaError_t count_cycles_device(uint64_t n, const uint64_t* src, const uint64_t* dst, const uint64_t* dist,
                                const uint64_t* size, uint64_t* leader, uint64_t* hops_out, uint64_t* clocks_out,
                                uint64_t* tree_out, uint64_t* n_cycles, unsigned int* err_out, void* scratch,
                                cudaStream_t st, int* launches) {
  ReduceScratch s{static_cast<uint8_t*>(scratch), 0};
  unsigned int* err = s.take<unsigned int>(4);
  uint64_t* tiles_buf = s.take<uint64_t>((n + kTile - 1) / kTile + 1);
  uint64_t* idx = s.take<uint64_t>(n);
  uint64_t* lab = s.take<uint64_t>(n);
  uint64_t* nxt = s.take<uint64_t>(n);
  uint64_t* lab2 = s.take<uint64_t>(n);
  uint64_t* nxt2 = s.take<uint64_t>(n);
  uint64_t* hops = s.take<uint64_t>(n);
  uint64_t* clocks = s.take<uint64_t>(n);
  uint64_t* tree = s.take<uint64_t>(n);
  uint64_t* newpos = s.take<uint64_t>(n);
  uint8_t* flag = s.take<uint8_t>(n + 1);
  unsigned int* indeg = reinterpret_cast<unsigned int*>(lab2);  // reused before the jumps
  cudaError_t e;
  *n_cycles = 0;
  *err_out = 0;
  if (n == 0) return cudaSuccess;
  if ((e = cudaMemsetAsync(err, 0, 16, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(indeg, 0, n * sizeof(unsigned int), st)) != cudaSuccess) return e;
  check_sorted_kernel<<<grid_for(n), kT, 0, st>>>(src, n, err);
  resolve_kernel<<<grid_for(n), kT, 0, st>>>(src, n, dst, idx, 0, nullptr);
  indeg_kernel<<<grid_for(n), kT, 0, st>>>(idx, n, indeg, err);
  perm_check_kernel<<<grid_for(n), kT, 0, st>>>(indeg, n, err);
  *launches += 4;
  unsigned int herr = 0;
  if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (herr) {
    *err_out = herr;
    return cudaSuccess;
  }
  label_init_kernel<<<grid_for(n), kT, 0, st>>>(idx, n, lab, nxt);
  ++*launches;
  for (uint64_t span = 1; span < n; span <<= 1) {  // after k jumps a label covers 2^k records
    jump_kernel<<<grid_for(n), kT, 0, st>>>(lab, nxt, n, lab2, nxt2);
    ++*launches;
    uint64_t* t = lab;
    lab = lab2;
    lab2 = t;
    t = nxt;
    nxt = nxt2;
    nxt2 = t;
  }
  if ((e = cudaMemsetAsync(hops, 0, n * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(clocks, 0, n * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(tree, 0, n * 8, st)) != cudaSuccess) return e;
  cycle_fold_kernel<<<grid_for(n), kT, 0, st>>>(lab, n, dist, size, reinterpret_cast<unsigned long long*>(hops),
                                                reinterpret_cast<unsigned long long*>(clocks),
                                                reinterpret_cast<unsigned long long*>(tree));
  leader_flag_kernel<<<grid_for(n), kT, 0, st>>>(lab, n, flag);
  const uint64_t tiles = (n + kTile - 1) / kTile;
  tile_count_kernel<<<static_cast<unsigned>(tiles), kT, 0, st>>>(flag, n, tiles_buf);
  tile_scan_kernel<<<1, 1024, 0, st>>>(tiles_buf, tiles);
  rank_kernel<<<static_cast<unsigned>(tiles), kT, 0, st>>>(flag, n, tiles_buf, newpos);
  *launches += 5;
  uint64_t ncyc = 0;
  if ((e = cudaMemcpyAsync(&ncyc, &tiles_buf[tiles], 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  // leaders in ascending index order = ascending leader state (sources ascend)
  select_kernel<<<grid_for(n), kT, 0, st>>>(newpos, n, src, leader);
  select_kernel<<<grid_for(n), kT, 0, st>>>(newpos, n, hops, hops_out);
  select_kernel<<<grid_for(n), kT, 0, st>>>(newpos, n, clocks, clocks_out);
  select_kernel<<<grid_for(n), kT, 0, st>>>(newpos, n, tree, tree_out);
  *launches += 4;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *n_cycles = ncyc;
  return cudaSuccess;
}

// 40-byte '<5Q' edge records (records.py:24-36) from SoA columns: out[5i + k] = col_k[i]
// (size/depth may be null: zero).  One thread per output word, so the stores are
// coalesced and the column reads are five interleaved streams.
__global__ void pack_records_kernel(uint64_t n, const uint64_t* __restrict__ c0, const uint64_t* __restrict__ c1,
                                    const uint64_t* __restrict__ c2, const uint64_t* __restrict__ c3,
                                    const uint64_t* __restrict__ c4, uint64_t* __restrict__ out) {
  GRID_STRIDE(w, 5 * n) {
    const uint64_t i = w / 5, k = w - 5 * i;
    const uint64_t* c = k == 0 ? c0 : k == 1 ? c1 : k == 2 ? c2 : k == 3 ? c3 : c4;
    out[w] = c ? c[i] : 0ull;
  }
}

cudaError_t pack_records_device(uint64_t n, const uint64_t* src, const uint64_t* dst, const uint64_t* dist,
                                const uint64_t* size, const uint64_t* depth, uint64_t* out, cudaStream_t st,
                                int* launches) {
  if (n == 0) return cudaSuccess;
  pack_records_kernel<<<grid_for(5 * n), kT, 0, st>>>(n, src, dst, dist, size, depth, out);
  ++*launches;
  return cudaGetLastError();
}

// Edge-output stage: records sorted ascending by source, the
// precondition of the edge file format and of step 4 (records.py:3-5, reduce.py:3-4).
// The in-house radix sort (csrc/sort.cu) writes out of place into scratch; the sorted
// columns are copied back.
size_t sort_scratch_bytes(uint64_t n) { return radix_sort_scratch_bytes(n) + 5 * ((n * 8 + 255) & ~255ull); }

// cols[0] is the key column; cols[1..ncols) (non-null) are permuted alongside it.
cudaError_t sort_records_device(uint64_t n, uint64_t* const* cols, int ncols, void* scratch, size_t scratch_bytes,
                                cudaStream_t st, int* launches) {
  if (n < 2) return cudaSuccess;
  const size_t col_bytes = (n * 8 + 255) & ~255ull;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  uint64_t* out[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < ncols; ++k) out[k] = cols[k] ? reinterpret_cast<uint64_t*>(p + k * col_bytes) : nullptr;
  const size_t used = 5 * col_bytes;
  cudaError_t e = radix_sort_records(n, cols, out, ncols, p + used, scratch_bytes - used, st, launches);
  if (e != cudaSuccess) return e;
  for (int k = 0; k < ncols; ++k)
    if (cols[k] && (e = cudaMemcpyAsync(cols[k], out[k], n * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
      return e;
  return cudaSuccess;
}

}  // namespace lc
