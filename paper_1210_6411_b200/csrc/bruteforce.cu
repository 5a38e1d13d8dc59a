// Exhaustive functional-graph analysis of a mini cipher on the GPU: the reference's
// ground-truth oracle (oracle.brute_force_analysis, oracle.py:141-283), SURVEY.md §8(f)
// rank 4.  Everything is in-house: the scans and ordered compactions below replace the
// library scan and the tensor-library unique / searchsorted / bincount glue.  States are rank-encoded as in the reference (rank = ((r1-1)*m2 + (r2-1))*m3 +
// (r3-1), oracle.py:55-63, 116-138).  Like the reference, the reverse direction comes
// from inverting the successor map (a CSR built by counting sort), not from the
// predecessor table.
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

// ------------------------------------------------ scan and ordered compaction
// Exclusive prefix sums of n values (u8 flags, i32 or i64 counts) into i64, three
// launches: per-block totals, one block scanning the totals (in 2048-entry chunks,
// carrying the running sum), per-block rescans adding the block's offset.  total[0]
// receives the grand total.
constexpr int kScanT = 256, kScanItems = 8, kScanTile = kScanT * kScanItems;

__device__ __forceinline__ int64_t block_excl_scan(int64_t v, int64_t* warp_tot, int64_t* total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  int64_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[w] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t run = 0;
    for (int i = 0; i < kScanT / 32; ++i) {
      const int64_t t = warp_tot[i];
      warp_tot[i] = run;
      run += t;
    }
    *total = run;
  }
  __syncthreads();
  const int64_t r = warp_tot[w] + x - v;
  __syncthreads();
  return r;
}

template <class T>
__global__ void __launch_bounds__(kScanT) scan_reduce_kernel(const T* __restrict__ in, uint64_t n,
                                                             int64_t* __restrict__ block_sums) {
  __shared__ int64_t wt[kScanT / 32], tot;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int64_t s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) s += static_cast<int64_t>(in[base + k]);
  block_excl_scan(s, wt, &tot);
  if (threadIdx.x == 0) block_sums[blockIdx.x] = tot;
}

__global__ void __launch_bounds__(kScanT) scan_blocks_kernel(int64_t* __restrict__ sums, uint64_t nb,
                                                             int64_t* __restrict__ total) {
  __shared__ int64_t wt[kScanT / 32], tot;
  int64_t carry = 0;
  for (uint64_t c = 0; c < nb; c += kScanTile) {
    const uint64_t base = c + threadIdx.x * kScanItems;
    int64_t v[kScanItems], s = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
      v[k] = base + k < nb ? sums[base + k] : 0;
      s += v[k];
    }
    int64_t run = carry + block_excl_scan(s, wt, &tot);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k)
      if (base + k < nb) {
        sums[base + k] = run;
        run += v[k];
      }
    carry += tot;
  }
  if (threadIdx.x == 0) *total = carry;
}

template <class T>
__global__ void __launch_bounds__(kScanT) scan_down_kernel(const T* __restrict__ in, uint64_t n,
                                                           const int64_t* __restrict__ block_sums,
                                                           int64_t* __restrict__ out) {
  __shared__ int64_t wt[kScanT / 32], tot;
  const uint64_t base = static_cast<uint64_t>(blockIdx.x) * kScanTile + threadIdx.x * kScanItems;
  int64_t v[kScanItems], s = 0;
#pragma unroll
  for (int k = 0; k < kScanItems; ++k) {
    v[k] = base + k < n ? static_cast<int64_t>(in[base + k]) : 0;
    s += v[k];
  }
  int64_t run = block_sums[blockIdx.x] + block_excl_scan(s, wt, &tot);
#pragma unroll
  for (int k = 0; k < kScanItems; ++k)
    if (base + k < n) {
      out[base + k] = run;
      run += v[k];
    }
}

uint64_t scan_blocks(uint64_t n) { return (n + kScanTile - 1) / kScanTile; }

// out[i] = sum(in[0..i)); *d_total = sum(in).  block_sums: scan_blocks(n) entries.
template <class T>
cudaError_t excl_scan(const T* in, uint64_t n, int64_t* out, int64_t* block_sums, int64_t* d_total, cudaStream_t st,
                      int* launches) {
  if (n == 0) return cudaMemsetAsync(d_total, 0, 8, st);
  const uint64_t nb = scan_blocks(n);
  scan_reduce_kernel<T><<<static_cast<unsigned>(nb), kScanT, 0, st>>>(in, n, block_sums);
  scan_blocks_kernel<<<1, kScanT, 0, st>>>(block_sums, nb, d_total);
  scan_down_kernel<T><<<static_cast<unsigned>(nb), kScanT, 0, st>>>(in, n, block_sums, out);
  *launches += 3;
  return cudaGetLastError();
}

// ordered compaction: out[pos[i]] = i for the flagged i (pos = exclusive scan of flags)
__global__ void compact_kernel(const uint8_t* __restrict__ flag, const int64_t* __restrict__ pos, uint64_t n,
                               int64_t* __restrict__ out) {
  BF_LOOP(i, n) if (flag[i]) out[pos[i]] = static_cast<int64_t>(i);
}

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

// pred_hist[k] = states with k predecessors; per candidate index: segment depth (max)
// and size (oracle.py:238-252)
__global__ void bf_summary_kernel(const int32_t* __restrict__ indeg, const int64_t* __restrict__ root,
                                  const int32_t* __restrict__ depth, uint64_t n,
                                  unsigned long long* __restrict__ pred_hist, unsigned long long* __restrict__ seg_depth,
                                  unsigned long long* __restrict__ seg_size) {
  __shared__ unsigned int h[5];
  if (threadIdx.x < 5) h[threadIdx.x] = 0;
  __syncthreads();
  BF_LOOP(x, n) {
    const int32_t k = indeg[x];
    LC_CHECK(k >= 0 && k <= 4);
    atomicAdd(&h[k], 1u);
    const int64_t r = root[x];
    if (r >= 0) {
      atomicMax(&seg_depth[r], static_cast<unsigned long long>(depth[x]));
      atomicAdd(&seg_size[r], 1ull);
    }
  }
  __syncthreads();
  if (threadIdx.x < 5 && h[threadIdx.x]) atomicAdd(&pred_hist[threadIdx.x], static_cast<unsigned long long>(h[threadIdx.x]));
}

__global__ void bf_mark_kernel(const int64_t* __restrict__ g, uint64_t n, uint8_t* __restrict__ flag) {
  BF_LOOP(x, n) flag[g[x]] = 1;
}

// successor of each on-cycle state as a compact (ascending-rank) index
__global__ void bf_cs_kernel(const int64_t* __restrict__ cyc, uint64_t m, const int64_t* __restrict__ succ,
                             const int64_t* __restrict__ pos, int64_t* __restrict__ cs) {
  BF_LOOP(k, m) cs[k] = pos[succ[cyc[k]]];
}

__global__ void bf_is_start_kernel(const int64_t* __restrict__ start, uint64_t m, uint8_t* __restrict__ flag) {
  BF_LOOP(k, m) flag[k] = start[k] == static_cast<int64_t>(k) ? 1 : 0;
}

// per cycle c (numbered by ascending start rank): length, candidates on it, leader (the
// smallest packed state on it), and each on-cycle state's cycle
__global__ void bf_cycle_stats_kernel(const int64_t* __restrict__ cyc, const int64_t* __restrict__ start,
                                      const int64_t* __restrict__ pos2, uint64_t m, const uint8_t* __restrict__ is_cand,
                                      uint64_t m2, uint64_t m3, int o2, int o3, int64_t* __restrict__ cid,
                                      unsigned long long* __restrict__ length, unsigned long long* __restrict__ cand_on,
                                      unsigned long long* __restrict__ leader, int64_t* __restrict__ cycle_of_state) {
  BF_LOOP(k, m) {
    const int64_t c = pos2[start[k]];
    const uint64_t x = static_cast<uint64_t>(cyc[k]);
    cid[k] = c;
    cycle_of_state[x] = c;
    atomicAdd(&length[c], 1ull);
    if (is_cand[x]) atomicAdd(&cand_on[c], 1ull);
    const uint64_t r1 = x / m3 / m2 + 1, r2 = (x / m3) % m2 + 1, r3 = x % m3 + 1;
    atomicMin(&leader[c], r1 | (r2 << o2) | (r3 << o3));
  }
}

// walk order from each cycle's start: position (length - steps) mod length
__global__ void bf_order_kernel(const int64_t* __restrict__ cyc, const int64_t* __restrict__ cid,
                                const int64_t* __restrict__ steps, uint64_t m, const int64_t* __restrict__ length,
                                const int64_t* __restrict__ offset, int64_t* __restrict__ order) {
  BF_LOOP(k, m) {
    const int64_t c = cid[k], L = length[c];
    order[offset[c] + (L - steps[k]) % L] = cyc[k];
  }
}

__global__ void bf_comp_kernel(const int64_t* __restrict__ g, uint64_t n, const int64_t* __restrict__ cycle_of_state,
                               unsigned long long* __restrict__ comp) {
  BF_LOOP(x, n) atomicAdd(&comp[cycle_of_state[g[x]]], 1ull);
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
  return (scan_blocks(n) + 1) * 8 + (n + 1) * 8 + n * 4 + n * 8 * 3 + 16 * 256;
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
  int64_t* bsums = reinterpret_cast<int64_t*>(take(scan_blocks(n) * 8));
  (void)scratch_bytes;
  cudaError_t e;
  // CSR of predecessors: offsets = exclusive scan of the in-degrees, offsets[n] = their
  // total (= n: every state has exactly one successor)
  if ((e = excl_scan(indeg, n, offsets, bsums, offsets + n, st, launches)) != cudaSuccess) return e;
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

size_t bf_candidates_scratch(uint64_t n) { return (scan_blocks(n) + 2) * 8 + n * 8 + 1024; }

cudaError_t bf_candidates(uint64_t n, const uint8_t* is_cand, int64_t* cand, uint64_t* m_out, void* scratch,
                          cudaStream_t st, int* launches) {
  int64_t* pos = static_cast<int64_t*>(scratch);
  int64_t* tot = pos + n;
  int64_t* bs = tot + 2;
  cudaError_t e;
  if ((e = excl_scan(is_cand, n, pos, bs, tot, st, launches)) != cudaSuccess) return e;
  compact_kernel<<<grid_of(n), kT, 0, st>>>(is_cand, pos, n, cand);
  ++*launches;
  int64_t h = 0;
  if ((e = cudaMemcpyAsync(&h, tot, 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *m_out = static_cast<uint64_t>(h);
  return cudaGetLastError();
}

cudaError_t bf_summary(uint64_t n, const int32_t* indeg, const int64_t* root, const int32_t* depth, uint64_t m,
                       uint64_t* pred_hist, int64_t* seg_depth, int64_t* seg_size, cudaStream_t st, int* launches) {
  cudaError_t e;
  if ((e = cudaMemsetAsync(pred_hist, 0, 5 * 8, st)) != cudaSuccess) return e;
  if (m && (e = cudaMemsetAsync(seg_depth, 0, m * 8, st)) != cudaSuccess) return e;
  if (m && (e = cudaMemsetAsync(seg_size, 0, m * 8, st)) != cudaSuccess) return e;
  bf_summary_kernel<<<grid_of(n), kT, 0, st>>>(indeg, root, depth, n,
                                               reinterpret_cast<unsigned long long*>(pred_hist),
                                               reinterpret_cast<unsigned long long*>(seg_depth),
                                               reinterpret_cast<unsigned long long*>(seg_size));
  ++*launches;
  return cudaGetLastError();
}

size_t bf_cycles_scratch(uint64_t n) { return n * 8 * 11 + n * 2 + (scan_blocks(n) + 4) * 8 + 4096; }

cudaError_t bf_cycles(uint64_t n, const int64_t* succ, const int64_t* g, const uint8_t* is_cand, uint64_t m2,
                      uint64_t m3, int o2, int o3, int64_t* order, int64_t* offset, int64_t* length, int64_t* leader,
                      int64_t* cand_on, int64_t* comp, uint64_t* n_on, uint64_t* n_cycles, void* scratch,
                      cudaStream_t st, int* launches) {
  uint8_t* base = static_cast<uint8_t*>(scratch);
  auto take = [&](size_t bytes) {
    uint8_t* p = base;
    base += (bytes + 255) & ~size_t(255);
    return p;
  };
  int64_t* pos = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* cyc = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* cs = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* start = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* steps = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* t0 = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* t1 = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* t2 = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* pos2 = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* cid = reinterpret_cast<int64_t*>(take(n * 8));
  int64_t* cos = reinterpret_cast<int64_t*>(take(n * 8));
  uint8_t* flag = take(n);
  uint8_t* flag2 = take(n);
  int64_t* tot = reinterpret_cast<int64_t*>(take(32));
  int64_t* bs = reinterpret_cast<int64_t*>(take(scan_blocks(n) * 8));
  cudaError_t e;
  int64_t h = 0;
  auto fetch = [&](const int64_t* d, int64_t* out) {
    cudaError_t r = cudaMemcpyAsync(out, d, 8, cudaMemcpyDeviceToHost, st);
    return r != cudaSuccess ? r : cudaStreamSynchronize(st);
  };
  // on-cycle states = the image of f^(2^k), ascending (oracle.py:168-186)
  if ((e = cudaMemsetAsync(flag, 0, n, st)) != cudaSuccess) return e;
  bf_mark_kernel<<<grid_of(n), kT, 0, st>>>(g, n, flag);
  ++*launches;
  if ((e = excl_scan(flag, n, pos, bs, tot, st, launches)) != cudaSuccess) return e;
  compact_kernel<<<grid_of(n), kT, 0, st>>>(flag, pos, n, cyc);
  ++*launches;
  if ((e = fetch(tot, &h)) != cudaSuccess) return e;
  const uint64_t m = static_cast<uint64_t>(h);
  *n_on = m;
  bf_cs_kernel<<<grid_of(m), kT, 0, st>>>(cyc, m, succ, pos, cs);
  ++*launches;
  if ((e = bf_cycle_order(m, cs, start, steps, t0, t1, t2, st, launches)) != cudaSuccess) return e;
  // cycles numbered by their start (smallest index on the cycle)
  bf_is_start_kernel<<<grid_of(m), kT, 0, st>>>(start, m, flag2);
  ++*launches;
  if ((e = excl_scan(flag2, m, pos2, bs, tot, st, launches)) != cudaSuccess) return e;
  if ((e = fetch(tot, &h)) != cudaSuccess) return e;
  const uint64_t nc = static_cast<uint64_t>(h);
  *n_cycles = nc;
  if (nc) {
    if ((e = cudaMemsetAsync(length, 0, nc * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(cand_on, 0, nc * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(comp, 0, nc * 8, st)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(leader, 0xff, nc * 8, st)) != cudaSuccess) return e;  // u64 max
  }
  bf_cycle_stats_kernel<<<grid_of(m), kT, 0, st>>>(cyc, start, pos2, m, is_cand, m2, m3, o2, o3, cid,
                                                   reinterpret_cast<unsigned long long*>(length),
                                                   reinterpret_cast<unsigned long long*>(cand_on),
                                                   reinterpret_cast<unsigned long long*>(leader), cos);
  ++*launches;
  if ((e = excl_scan(length, nc, offset, bs, tot, st, launches)) != cudaSuccess) return e;
  bf_order_kernel<<<grid_of(m), kT, 0, st>>>(cyc, cid, steps, m, length, offset, order);
  bf_comp_kernel<<<grid_of(n), kT, 0, st>>>(g, n, cos, reinterpret_cast<unsigned long long*>(comp));
  *launches += 2;
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
