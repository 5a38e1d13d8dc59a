// Steps 4-5 on the GPU: the edge-output sort, iterative leaf
// cutting (reduce.cut_leaves_pass / cut_leaves_to_fixpoint, reduce.py:118-223) and cycle
// counting (reduce.count_cycles, reduce.py:226-266) on skeleton-edge records held in HBM.
//
// Records are SoA u64 arrays (source, destination, distance, subtree_size, subtree_depth),
// sorted ascending by unique source -- the file format's invariant (records.py:3-5).
// Destinations are resolved once to record indices by binary search; every pass is then
// a handful of streaming kernels: mark in-degree, fold each leaf's (size+1, depth+1) into
// its destination with atomics (leaves are never targets within a pass, so the reads are
// stable), and a stable compaction that also remaps destination indices.  The result is
// the reference's fixpoint and per-pass statistics exactly, without external sorts.
// Cycles: pointer jumping labels every record with the smallest index on its cycle (the
// smallest source, since sources ascend), then one atomic fold per record.
#include <cub/device/device_radix_sort.cuh>
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

__global__ void resolve_kernel(const uint64_t* __restrict__ src, uint64_t n, const uint64_t* __restrict__ dst,
                               uint64_t* __restrict__ idx) {
  GRID_STRIDE(i, n) {
    const uint64_t v = dst[i];
    uint64_t lo = 0, hi = n;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (src[mid] < v) lo = mid + 1;
      else hi = mid;
    }
    idx[i] = (lo < n && src[lo] == v) ? lo : kNone;
  }
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

// ---- leaf-cutting pass kernels driven by device-side counts (so passes can be batched
// in a CUDA graph without host round trips).  In-degree marks are pass stamps, so no
// array has to be cleared between passes.
struct PassCtl {
  unsigned long long n;       // records in the current pass's input
  unsigned long long pass;    // current pass number (1-based)
  unsigned long long leaves;  // leaves removed by the current pass
  unsigned long long sum;     // subtree-size sum over its survivors
  unsigned long long done_at; // first pass that removed nothing (0: not yet)
};

__global__ void pass_begin_kernel(PassCtl* ctl) {
  ctl->pass += 1;
  ctl->leaves = 0;
  ctl->sum = 0;
}

__global__ void mark_stamp_kernel(const uint64_t* __restrict__ idx, const PassCtl* __restrict__ ctl,
                                  uint32_t* __restrict__ stamp) {
  const uint64_t n = ctl->n;
  const uint32_t p = static_cast<uint32_t>(ctl->pass);
  GRID_STRIDE(i, n) {
    const uint64_t j = idx[i];
    if (j != kNone) stamp[j] = p;
  }
}

__global__ void fold_stamp_kernel(const uint64_t* __restrict__ idx, PassCtl* ctl, const uint32_t* __restrict__ stamp,
                                  unsigned long long* size, unsigned long long* depth, unsigned int* err) {
  const uint64_t n = ctl->n;
  const uint32_t p = static_cast<uint32_t>(ctl->pass);
  uint32_t c = 0;
  GRID_STRIDE(i, n) {
    if (stamp[i] != p) {  // no record points here: a leaf
      ++c;
      const uint64_t j = idx[i];
      if (j == kNone) {
        atomicExch(err, 2u);  // aggregate with no surviving record: input not closed
      } else {
        atomicAdd(&size[j], size[i] + 1ull);
        atomicMax(&depth[j], depth[i] + 1ull);
      }
    }
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(&ctl->leaves, static_cast<unsigned long long>(c));
}

__global__ void tile_count_stamp_kernel(const uint32_t* __restrict__ stamp, const PassCtl* __restrict__ ctl,
                                        uint64_t* __restrict__ counts) {
  const uint64_t n = ctl->n;
  const uint32_t p = static_cast<uint32_t>(ctl->pass);
  const uint64_t tiles = (n + kTile - 1) / kTile;
  __shared__ uint32_t part[kT / 32];
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint64_t lo = t * kTile, hi = min(n, lo + kTile);
    uint32_t c = 0;
    for (uint64_t i = lo + threadIdx.x; i < hi; i += blockDim.x) c += stamp[i] == p ? 1u : 0u;
    c = __reduce_add_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      uint64_t s = 0;
      for (int w = 0; w < kT / 32; ++w) s += part[w];
      counts[t] = s;
    }
    __syncthreads();
  }
}

__global__ void tile_scan_dev_kernel(uint64_t* __restrict__ counts, const PassCtl* __restrict__ ctl) {
  const uint64_t tiles = (ctl->n + kTile - 1) / kTile;
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

__global__ void rank_stamp_kernel(const uint32_t* __restrict__ stamp, const PassCtl* __restrict__ ctl,
                                  const uint64_t* __restrict__ offsets, uint64_t* __restrict__ newpos) {
  __shared__ uint32_t wcount[kT / 32];
  const uint64_t n = ctl->n;
  const uint32_t p = static_cast<uint32_t>(ctl->pass);
  const uint64_t tiles = (n + kTile - 1) / kTile;
  const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint64_t t = blockIdx.x; t < tiles; t += gridDim.x) {
    const uint64_t lo = t * kTile, hi = min(n, lo + kTile);
    uint64_t pos = offsets[t];
    for (uint64_t r = lo; r < hi; r += kT) {
      const uint64_t i = r + threadIdx.x;
      const bool k = i < hi && stamp[i] == p;
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
}

__global__ void pass_end_kernel(PassCtl* ctl, const uint64_t* __restrict__ counts, uint64_t* __restrict__ pstats,
                                uint64_t max_stats) {
  const uint64_t tiles = (ctl->n + kTile - 1) / kTile;
  const uint64_t inner = counts[tiles];
  const uint64_t p = ctl->pass;
  if (p - 1 < max_stats) {
    pstats[3 * (p - 1) + 0] = ctl->leaves;
    pstats[3 * (p - 1) + 1] = inner;
    pstats[3 * (p - 1) + 2] = ctl->sum;
  }
  if (ctl->leaves == 0 && ctl->done_at == 0) ctl->done_at = p;
  ctl->n = inner;
}

struct Cols {
  uint64_t *src, *dst, *dist, *size, *depth, *idx;
};

__global__ void scatter_dev_kernel(Cols in, Cols out, const uint64_t* __restrict__ newpos,
                                   const PassCtl* __restrict__ ctl) {
  const uint64_t n = ctl->n;
  GRID_STRIDE(i, n) {
    const uint64_t p = newpos[i];
    if (p == kNone) continue;
    out.src[p] = in.src[i];
    out.dst[p] = in.dst[i];
    out.dist[p] = in.dist[i];
    out.size[p] = in.size[i];
    out.depth[p] = in.depth[i];
    const uint64_t j = in.idx[i];
    out.idx[p] = j == kNone ? kNone : newpos[j];
  }
}

// subtree-size sum over the survivors (count = counts[tiles] of this pass)
__global__ void sum_dev_kernel(const uint64_t* __restrict__ v, PassCtl* ctl, const uint64_t* __restrict__ counts) {
  const uint64_t tiles = (ctl->n + kTile - 1) / kTile;
  const uint64_t n = counts[tiles];
  uint64_t s = 0;
  GRID_STRIDE(i, n) { s += v[i]; }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(&ctl->sum, static_cast<unsigned long long>(s));
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

__global__ void gather_kernel(const uint64_t* __restrict__ order, uint64_t n, const uint64_t* __restrict__ a,
                              uint64_t* __restrict__ b) {
  GRID_STRIDE(i, n) { b[i] = a[order[i]]; }
}

__global__ void iota_kernel(uint64_t* v, uint64_t n) {
  GRID_STRIDE(i, n) { v[i] = i; }
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
  // stamp (u32), newpos, idx x2, second set of five columns, tile counts, control, stats
  const uint64_t tiles = (n + kTile - 1) / kTile + 1;
  return n * 4 + 8 * n * 8 + tiles * 8 + 3ull * (max_stats + 1) * 8 + 64 * 1024 + 16 * 256;
}

namespace {

struct PassLaunch {
  unsigned grid, tgrid;
  PassCtl* ctl;
  uint32_t* stamp;
  uint64_t* tiles;
  uint64_t* newpos;
  uint64_t* pstats;
  uint64_t max_stats;
  unsigned int* err;
};

void launch_pass(const PassLaunch& L, const Cols& c, const Cols& o, cudaStream_t st) {
  pass_begin_kernel<<<1, 1, 0, st>>>(L.ctl);
  mark_stamp_kernel<<<L.grid, kT, 0, st>>>(c.idx, L.ctl, L.stamp);
  fold_stamp_kernel<<<L.grid, kT, 0, st>>>(c.idx, L.ctl, L.stamp, reinterpret_cast<unsigned long long*>(c.size),
                                           reinterpret_cast<unsigned long long*>(c.depth), L.err);
  tile_count_stamp_kernel<<<L.tgrid, kT, 0, st>>>(L.stamp, L.ctl, L.tiles);
  tile_scan_dev_kernel<<<1, 1024, 0, st>>>(L.tiles, L.ctl);
  rank_stamp_kernel<<<L.tgrid, kT, 0, st>>>(L.stamp, L.ctl, L.tiles, L.newpos);
  scatter_dev_kernel<<<L.grid, kT, 0, st>>>(c, o, L.newpos, L.ctl);
  sum_dev_kernel<<<L.grid, kT, 0, st>>>(o.size, L.ctl, L.tiles);
  pass_end_kernel<<<1, 1, 0, st>>>(L.ctl, L.tiles, L.pstats, L.max_stats);
}

constexpr int kLaunchesPerPass = 9;

}  // namespace

// Passes run back to back on the device: every kernel reads the current record count
// and pass number from PassCtl, so the host only checks in every 32 passes (a CUDA graph
// of two ping-pong passes replayed 16 times).  Passes after the fixpoint are no-ops
// (nothing removed, every record kept), so overshooting is harmless.
cudaError_t cut_leaves_device(uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist, uint64_t* size,
                              uint64_t* depth, uint32_t max_passes, uint64_t* pass_stats, uint32_t max_stats,
                              uint32_t* n_passes, uint64_t* n_out, unsigned int* err_out, void* scratch,
                              cudaStream_t st, int* launches) {
  ReduceScratch s{static_cast<uint8_t*>(scratch), 0};
  unsigned int* err = s.take<unsigned int>(4);
  PassCtl* ctl = s.take<PassCtl>(1);
  const uint64_t stats_cap = max_stats ? max_stats : 1;
  uint64_t* pstats = s.take<uint64_t>(3 * stats_cap);
  uint64_t* tiles_buf = s.take<uint64_t>((n + kTile - 1) / kTile + 1);
  uint32_t* stamp = s.take<uint32_t>(n);
  uint64_t* newpos = s.take<uint64_t>(n);
  Cols a{src, dst, dist, size, depth, s.take<uint64_t>(n)};
  Cols b{s.take<uint64_t>(n), s.take<uint64_t>(n), s.take<uint64_t>(n), s.take<uint64_t>(n), s.take<uint64_t>(n),
         s.take<uint64_t>(n)};
  cudaError_t e;
  *n_passes = 0;
  *n_out = n;
  *err_out = 0;
  if (n == 0) return cudaSuccess;
  if ((e = cudaMemsetAsync(err, 0, 16, st)) != cudaSuccess) return e;
  check_sorted_kernel<<<grid_for(n), kT, 0, st>>>(src, n, err);
  resolve_kernel<<<grid_for(n), kT, 0, st>>>(src, n, dst, a.idx);
  *launches += 2;
  if ((e = cudaMemsetAsync(stamp, 0, n * sizeof(uint32_t), st)) != cudaSuccess) return e;
  const PassCtl init{n, 0, 0, 0, 0};
  if ((e = cudaMemcpyAsync(ctl, &init, sizeof(init), cudaMemcpyHostToDevice, st)) != cudaSuccess) return e;
  unsigned int herr = 0;
  if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if (herr) {
    *err_out = herr;
    return cudaSuccess;
  }
  const uint64_t tiles0 = (n + kTile - 1) / kTile;
  PassLaunch L{std::min(grid_for(n), 4096u), static_cast<unsigned>(std::min<uint64_t>(tiles0, 4096)), ctl, stamp,
               tiles_buf, newpos, pstats, max_stats, err};
  PassCtl h{};
  uint64_t executed = 0;
  if (max_passes != 0) {
    for (uint32_t k = 0; k < max_passes; ++k) {
      launch_pass(L, (k & 1) ? b : a, (k & 1) ? a : b, st);
      *launches += kLaunchesPerPass;
    }
    executed = max_passes;
    if ((e = cudaMemcpyAsync(&h, ctl, sizeof(h), cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st)) != cudaSuccess) return e;
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  } else {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    if ((e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal)) != cudaSuccess) return e;
    launch_pass(L, a, b, st);
    launch_pass(L, b, a, st);
    if ((e = cudaStreamEndCapture(st, &graph)) != cudaSuccess) return e;
    if ((e = cudaGraphInstantiate(&exec, graph, 0)) != cudaSuccess) return e;
    constexpr int kBatch = 16;  // graphs (x2 passes) per host check-in
    for (;;) {
      for (int k = 0; k < kBatch; ++k)
        if ((e = cudaGraphLaunch(exec, st)) != cudaSuccess) break;
      if (e != cudaSuccess) break;
      executed += 2 * kBatch;
      *launches += 2 * kBatch * kLaunchesPerPass;
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
  const uint64_t passes = h.done_at ? h.done_at : executed;
  *n_passes = static_cast<uint32_t>(passes);
  const uint64_t keep_stats = std::min<uint64_t>(passes, max_stats);
  if (keep_stats)
    if ((e = cudaMemcpyAsync(pass_stats, pstats, keep_stats * 3 * 8, cudaMemcpyDeviceToHost, st)) != cudaSuccess)
      return e;
  // an odd number of executed passes leaves the survivors in the second column set
  if (executed & 1) {
    for (int k = 0; k < 5; ++k)
      if ((e = cudaMemcpyAsync((&a.src)[k], (&b.src)[k], h.n * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return e;
  }
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  *n_out = h.n;
  return cudaSuccess;
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
  resolve_kernel<<<grid_for(n), kT, 0, st>>>(src, n, dst, idx);
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

// Edge-output stage: records sorted ascending by source, the
// precondition of the edge file format and of step 4 (records.py:3-5, reduce.py:3-4).
// LSD radix sort of (source, row) pairs (CUB), then a gather of the other columns.
size_t sort_scratch_bytes(uint64_t n) {
  size_t temp = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, temp, static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                  static_cast<const uint64_t*>(nullptr), static_cast<uint64_t*>(nullptr),
                                  static_cast<int64_t>(n));
  return temp + 4 * n * 8 + 4 * 256;
}

// cols[0] is the key column; cols[1..ncols) (non-null) are permuted alongside it.
cudaError_t sort_records_device(uint64_t n, uint64_t* const* cols, int ncols, void* scratch, size_t scratch_bytes,
                                cudaStream_t st, int* launches) {
  if (n < 2) return cudaSuccess;
  ReduceScratch s{static_cast<uint8_t*>(scratch), 0};
  uint64_t* order_in = s.take<uint64_t>(n);
  uint64_t* order = s.take<uint64_t>(n);
  uint64_t* keys = s.take<uint64_t>(n);
  uint64_t* tmp = s.take<uint64_t>(n);
  void* temp = static_cast<uint8_t*>(scratch) + s.used;
  size_t temp_bytes = scratch_bytes - s.used;
  iota_kernel<<<grid_for(n), kT, 0, st>>>(order_in, n);
  cudaError_t e = cub::DeviceRadixSort::SortPairs(temp, temp_bytes, cols[0], keys, order_in, order,
                                                  static_cast<int64_t>(n), 0, 64, st);
  if (e != cudaSuccess) return e;
  *launches += 2;  // iota + the radix sort (several CUB kernels)
  for (int k = 1; k < ncols; ++k) {
    if (!cols[k]) continue;
    gather_kernel<<<grid_for(n), kT, 0, st>>>(order, n, cols[k], tmp);
    if ((e = cudaMemcpyAsync(cols[k], tmp, n * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
    ++*launches;
  }
  if ((e = cudaMemcpyAsync(cols[0], keys, n * 8, cudaMemcpyDeviceToDevice, st)) != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace lc
