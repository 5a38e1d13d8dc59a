// Exhaustive functional-graph analysis of a mini cipher on the GPU: the reference's
// ground-truth oracle (oracle.brute_force_analysis, oracle.py:141-283), SURVEY.md §8(f)
// rank 4.  States are rank-encoded as in the reference (rank = ((r1-1)*m2 + (r2-1))*m3 +
// (r3-1), oracle.py:55-63, 116-138).  Like the reference, the reverse direction comes
// from inverting the successor map (a CSR built by counting sort), not from the
// predecessor table.
#include <cub/device/device_scan.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lfsr_common.cuh"
#include "lfsr_internal.h"

namespace lc {

namespace {

constexpr int kT = 256;

inline unsigned grid_of(uint64_t n) {
  const uint64_t g = (n + kT - 1) / kT;
  return static_cast<unsigned>(g == 0 ? 1 : (g > 65536 ? 65536 : g));
}

#define BF_LOOP(i, n)                                                                      \
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < (n); \
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x)

// oracle.py:116-138 _build_successors (majority rule, or every register clocked)
template <class S>
__global__ void bf_succ_kernel(uint64_t n, int clock_all, int64_t* __restrict__ succ) {
  constexpr uint64_t m1 = S::M1, m2 = S::M2, m3 = S::M3;
  BF_LOOP(i, n) {
    uint32_t r3 = static_cast<uint32_t>(i % m3) + 1u;
    const uint64_t rest = i / m3;
    uint32_t r2 = static_cast<uint32_t>(rest % m2) + 1u;
    uint32_t r1 = static_cast<uint32_t>(rest / m2) + 1u;
    bool k1 = true, k2 = true, k3 = true;
    if (!clock_all) {
      const uint32_t c1 = (r1 >> S::CT1) & 1u, c2 = (r2 >> S::CT2) & 1u, c3 = (r3 >> S::CT3) & 1u;
      const uint32_t maj = (c1 & c2) | (c3 & (c1 | c2));
      k1 = c1 == maj;
      k2 = c2 == maj;
      k3 = c3 == maj;
    }
    if (k1) r1 = ((r1 << 1) & static_cast<uint32_t>(m1)) | parity32(r1 & S::T1);
    if (k2) r2 = ((r2 << 1) & static_cast<uint32_t>(m2)) | parity32(r2 & S::T2);
    if (k3) r3 = ((r3 << 1) & static_cast<uint32_t>(m3)) | parity32(r3 & S::T3);
    succ[i] = static_cast<int64_t>(((r1 - 1ull) * m2 + (r2 - 1ull)) * m3 + (r3 - 1ull));
  }
}

__global__ void bf_indeg_kernel(const int64_t* __restrict__ succ, uint64_t n, int32_t* __restrict__ indeg) {
  BF_LOOP(i, n) atomicAdd(&indeg[succ[i]], 1);
}

// Candidates (oracle.py:159-166): R3 == F, the successor's R3 != F, in-degree > 0.
template <class S>
__global__ void bf_cand_kernel(const int64_t* __restrict__ succ, const int32_t* __restrict__ indeg, uint32_t F,
                               uint64_t n, uint8_t* __restrict__ is_cand) {
  constexpr uint64_t m3 = S::M3;
  BF_LOOP(i, n) {
    const uint32_t r3 = static_cast<uint32_t>(i % m3) + 1u;
    const uint32_t s3 = static_cast<uint32_t>(static_cast<uint64_t>(succ[i]) % m3) + 1u;
    is_cand[i] = (r3 == F && s3 != F && indeg[i] > 0) ? 1 : 0;
  }
}

// g <- g o g (pointer doubling: after ceil(log2 n) rounds every state maps onto its cycle)
__global__ void bf_double_kernel(const int64_t* __restrict__ g, uint64_t n, int64_t* __restrict__ out) {
  BF_LOOP(i, n) out[i] = g[g[i]];
}

__global__ void bf_scatter_preds_kernel(const int64_t* __restrict__ succ, uint64_t n,
                                        const int64_t* __restrict__ offsets, int32_t* __restrict__ cursor,
                                        int64_t* __restrict__ preds) {
  BF_LOOP(i, n) {
    const int64_t j = succ[i];
    preds[offsets[j] + atomicAdd(&cursor[j], 1)] = static_cast<int64_t>(i);
  }
}

__global__ void bf_seed_kernel(const int64_t* __restrict__ cand, uint64_t m, int64_t* __restrict__ root,
                               int32_t* __restrict__ depth, int64_t* __restrict__ frontier) {
  BF_LOOP(k, m) {
    const int64_t x = cand[k];
    root[x] = static_cast<int64_t>(k);
    depth[x] = 0;
    frontier[k] = x;
  }
}

// One level of the segment sweep (oracle.py:200-236): predecessors of the frontier that
// are not candidates inherit the parent's root.  Each state has one successor, so it is
// reached from exactly one parent: no conflicts, any order.
__global__ void bf_bfs_kernel(const int64_t* __restrict__ frontier, uint64_t m, const int64_t* __restrict__ offsets,
                              const int64_t* __restrict__ preds, const uint8_t* __restrict__ is_cand,
                              int64_t* __restrict__ root, int32_t* __restrict__ depth, int32_t level,
                              int64_t* __restrict__ next, unsigned long long* __restrict__ next_count) {
  BF_LOOP(k, m) {
    const int64_t x = frontier[k];
    const int64_t r = root[x];
    for (int64_t q = offsets[x]; q < offsets[x + 1]; ++q) {
      const int64_t p = preds[q];
      if (is_cand[p]) continue;
      root[p] = r;
      depth[p] = level;
      next[atomicAdd(next_count, 1ull)] = p;
    }
  }
}

// Cycle order on the compact on-cycle index space (cs = successor as a compact index):
// lab = smallest index on the cycle (its start, since indices follow ascending ranks);
// cnt = steps from i forward to the start.  Pointer doubling, `rounds` rounds.
__global__ void bf_cycle_init_kernel(const int64_t* __restrict__ cs, uint64_t m, int64_t* __restrict__ lab,
                                     int64_t* __restrict__ nxt) {
  BF_LOOP(i, m) {
    lab[i] = static_cast<int64_t>(i);
    nxt[i] = cs[i];
  }
}

__global__ void bf_cycle_min_kernel(const int64_t* __restrict__ lab, const int64_t* __restrict__ nxt, uint64_t m,
                                    int64_t* __restrict__ lab2, int64_t* __restrict__ nxt2) {
  BF_LOOP(i, m) {
    const int64_t j = nxt[i];
    lab2[i] = min(lab[i], lab[j]);
    nxt2[i] = nxt[j];
  }
}

__global__ void bf_dist_init_kernel(const int64_t* __restrict__ cs, const int64_t* __restrict__ lab, uint64_t m,
                                    int64_t* __restrict__ nxt, int64_t* __restrict__ cnt) {
  BF_LOOP(i, m) {
    const bool start = lab[i] == static_cast<int64_t>(i);
    nxt[i] = start ? static_cast<int64_t>(i) : cs[i];
    cnt[i] = start ? 0 : 1;
  }
}

__global__ void bf_dist_kernel(const int64_t* __restrict__ nxt, const int64_t* __restrict__ cnt, uint64_t m,
                               int64_t* __restrict__ nxt2, int64_t* __restrict__ cnt2) {
  BF_LOOP(i, m) {
    const int64_t j = nxt[i];
    nxt2[i] = nxt[j];
    cnt2[i] = cnt[i] + cnt[j];
  }
}

// Candidate-graph edges (oracle.py:188-198): walk each candidate through the successor
// map to the first candidate (at most n steps).
__global__ void bf_edges_kernel(const int64_t* __restrict__ cand, uint64_t m, const int64_t* __restrict__ succ,
                                const uint8_t* __restrict__ is_cand, uint64_t n, int64_t* __restrict__ dst,
                                int64_t* __restrict__ dist) {
  BF_LOOP(k, m) {
    int64_t x = cand[k];
    uint64_t d = 0;
    do {
      x = succ[x];
      ++d;
    } while (!is_cand[x] && d < n);
    dst[k] = x;
    dist[k] = static_cast<int64_t>(d);
  }
}

template <class S>
cudaError_t build_t(uint64_t n, int clock_all, uint32_t F, int64_t* succ, int32_t* indeg, uint8_t* is_cand,
                    int64_t* g, int64_t* tmp, cudaStream_t st, int* launches) {
  cudaError_t e;
  bf_succ_kernel<S><<<grid_of(n), kT, 0, st>>>(n, clock_all, succ);
  if ((e = cudaMemsetAsync(indeg, 0, n * 4, st)) != cudaSuccess) return e;
  bf_indeg_kernel<<<grid_of(n), kT, 0, st>>>(succ, n, indeg);
  bf_cand_kernel<S><<<grid_of(n), kT, 0, st>>>(succ, indeg, F, n, is_cand);
  *launches += 3;
  if ((e = cudaMemcpyAsync(g, succ, n * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  int64_t* a = g;
  int64_t* b = tmp;
  for (uint64_t hops = 1; hops < n; hops <<= 1) {
    bf_double_kernel<<<grid_of(n), kT, 0, st>>>(a, n, b);
    ++*launches;
    std::swap(a, b);
  }
  if (a != g) e = cudaMemcpyAsync(g, a, n * 8, cudaMemcpyDeviceToDevice, st);
  return e != cudaSuccess ? e : cudaGetLastError();
}

}  // namespace

cudaError_t bf_build(SpecId id, uint64_t n, int clock_all, uint32_t F, int64_t* succ, int32_t* indeg,
                     uint8_t* is_cand, int64_t* g, int64_t* tmp, cudaStream_t st, int* launches) {
  switch (id) {
    case SpecId::A51: return build_t<A51>(n, clock_all, F, succ, indeg, is_cand, g, tmp, st, launches);
    case SpecId::MINI567: return build_t<MINI567>(n, clock_all, F, succ, indeg, is_cand, g, tmp, st, launches);
    case SpecId::MINI789: return build_t<MINI789>(n, clock_all, F, succ, indeg, is_cand, g, tmp, st, launches);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t bf_edges(uint64_t n, const int64_t* succ, const uint8_t* is_cand, const int64_t* cand, uint64_t m,
                     int64_t* dst, int64_t* dist, cudaStream_t st, int* launches) {
  if (m == 0) return cudaSuccess;
  bf_edges_kernel<<<grid_of(m), kT, 0, st>>>(cand, m, succ, is_cand, n, dst, dist);
  ++*launches;
  return cudaGetLastError();
}

size_t bf_segments_scratch(uint64_t n) {
  size_t temp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, temp, static_cast<const int32_t*>(nullptr), static_cast<int64_t*>(nullptr),
                                static_cast<int64_t>(n + 1));
  return temp + (n + 1) * 8 + n * 4 + n * 8 * 3 + 16 * 256;
}

cudaError_t bf_segments(uint64_t n, const int64_t* succ, const int32_t* indeg, const uint8_t* is_cand,
                        const int64_t* cand, uint64_t ncand, int64_t* root, int32_t* depth, uint64_t* level_counts,
                        uint32_t level_cap, uint32_t* n_levels, void* scratch, size_t scratch_bytes, cudaStream_t st,
                        int* launches) {
  uint8_t* base = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t bytes) {
    uint8_t* p = base;
    base += (bytes + 255) & ~size_t(255);
    return p;
  };
  int64_t* offsets = reinterpret_cast<int64_t*>(take((n + 1) * 8));
  int32_t* cursor = reinterpret_cast<int32_t*>(take(n * 4));
  int64_t* preds = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* fa = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* fb = reinterpret_cast<int64_t*>(take(n * 8));
  unsigned long long* cnt = reinterpret_cast<unsigned long long*>(take(256));
  void* temp = base;
  size_t temp_bytes = scratch_bytes - static_cast<size_t>(base - static_cast<uint8_t*>(scratch));
  cudaError_t e;
  // CSR of predecessors: offsets = exclusive scan of the in-degrees (n + 1 entries, the
  // last in-degree read as 0 through a zeroed cursor slot is not needed: scan n, then
  // offsets[n] = n since every state has exactly one successor)
  e = cub::DeviceScan::ExclusiveSum(temp, temp_bytes, indeg, offsets, static_cast<int64_t>(n), st);
  if (e != cudaSuccess) return e;
  const int64_t total = static_cast<int64_t>(n);
  if ((e = cudaMemcpyAsync(offsets + n, &total, 8, cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(cursor, 0, n * 4, st)) != cudaSuccess) return e;
  bf_scatter_preds_kernel<<<grid_of(n), kT, 0, st>>>(succ, n, offsets, cursor, preds);
  if ((e = cudaMemsetAsync(root, 0xff, n * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(depth, 0xff, n * 4, st)) != cudaSuccess) return e;
  bf_seed_kernel<<<grid_of(ncand), kT, 0, st>>>(cand, ncand, root, depth, fa);
  *launches += 3;
  uint32_t levels = 0;
  if (level_cap) level_counts[levels] = ncand;
  ++levels;
  uint64_t m = ncand;
  for (int32_t level = 1; m; ++level) {
    if ((e = cudaMemsetAsync(cnt, 0, 8, st)) != cudaSuccess) return e;
    bf_bfs_kernel<<<grid_of(m), kT, 0, st>>>(fa, m, offsets, preds, is_cand, root, depth, level, fb, cnt);
    ++*launches;
    unsigned long long h = 0;
    if ((e = cudaMemcpyAsync(&h, cnt, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
    if (h == 0) break;
    if (levels < level_cap) level_counts[levels] = h;
    ++levels;
    m = h;
    std::swap(fa, fb);
  }
  *n_levels = levels;
  return cudaGetLastError();
}

cudaError_t bf_cycle_order(uint64_t m, const int64_t* cs, int64_t* lab, int64_t* steps, int64_t* t0, int64_t* t1,
                           int64_t* t2, cudaStream_t st, int* launches) {
  if (m == 0) return cudaSuccess;
  bf_cycle_init_kernel<<<grid_of(m), kT, 0, st>>>(cs, m, lab, t0);
  ++*launches;
  int64_t *la = lab, *na = t0, *lb = t1, *nb = t2;
  for (uint64_t span = 1; span < m; span <<= 1) {
    bf_cycle_min_kernel<<<grid_of(m), kT, 0, st>>>(la, na, m, lb, nb);
    ++*launches;
    std::swap(la, lb);
    std::swap(na, nb);
  }
  cudaError_t e;
  if (la != lab && (e = cudaMemcpyAsync(lab, la, m * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  // steps to the cycle start: nxt in t0, counts in steps / t1 (ping-pong with t2)
  bf_dist_init_kernel<<<grid_of(m), kT, 0, st>>>(cs, lab, m, t0, steps);
  ++*launches;
  int64_t *xa = t0, *ca = steps, *xb = t2, *cb = t1;
  for (uint64_t span = 1; span < m; span <<= 1) {
    bf_dist_kernel<<<grid_of(m), kT, 0, st>>>(xa, ca, m, xb, cb);
    ++*launches;
    std::swap(xa, xb);
    std::swap(ca, cb);
  }
  if (ca != steps && (e = cudaMemcpyAsync(steps, ca, m * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace lc
