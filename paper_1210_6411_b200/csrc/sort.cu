// Edge-output sort: records ascending by source, the invariant
// of the edge file and of step 4 (records.py:3-5, reduce.py:3-4).
//
// An LSD radix sort of the 64-bit source keys with a 32-bit row index as payload, one
// byte per pass, each pass a single "onesweep" kernel (no separate upsweep per pass):
//   * one histogram kernel reads the keys once and counts all eight byte digits (warp
//     match-aggregated shared atomics), and notes whether the keys are already ascending;
//   * a one-block scan turns the counts into per-byte digit starts and marks trivial
//     bytes (every key in one bucket -- for A5/1 skeletons the R3 bytes, which all equal
//     the fixed value -- or an already sorted input): their pass kernels return at once,
//     and the ping-pong buffer of every pass is decided on the device, so the whole sort is
//     enqueued without a host round trip;
//   * a pass kernel takes tiles of 4096 keys in launch order (an atomic ticket, so a
//     tile's predecessors are always resident), ranks each key within its warp (match on
//     the digit, warp-private counters), scans the tile's 256 digit counts, publishes them
//     and looks back over earlier tiles for each digit's global offset (decoupled
//     look-back: 256 independent chains, one per thread), stages the tile in shared memory
//     in digit order and writes each digit's run contiguously.  Ranking in input order
//     makes every pass stable, so equal sources keep their input order (numpy's stable
//     argsort).
// The other record columns are then gathered by the final row index.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>

#include "lfsr_internal.h"

namespace lc {
namespace {

constexpr uint32_t kFullMask = 0xffffffffu;
constexpr int kSortThreads = 256;
constexpr int kSortWarps = kSortThreads / 32;
constexpr int kItems = 16;                          // keys per thread
constexpr int kTileKeys = kSortThreads * kItems;    // 4096
constexpr int kBins = 256;
constexpr int kBytes = 8;
// look-back status word: [49:48] flag, [47:40] epoch (pass byte + 1), [39:0] count
constexpr uint64_t kFlagAgg = 1ull << 48, kFlagPrefix = 2ull << 48;
constexpr uint64_t kValueMask = (1ull << 40) - 1;

struct SortCtl {
  unsigned long long hist[kBytes][kBins];  // digit counts, then (scan) digit starts
  unsigned int tickets[kBytes];
  unsigned int unsorted;
  unsigned int trivial[kBytes];
  unsigned int in_buf[kBytes];  // ping-pong buffer each pass reads
  unsigned int first[kBytes];   // 1: the first pass that runs (payload = row index)
  unsigned int final_buf;       // buffer holding the result (0: the input, never permuted)
  unsigned int passes;
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                                 SortCtl* ctl) {
  __shared__ unsigned int h[kBytes][kBins];
  for (int i = threadIdx.x; i < kBytes * kBins; i += kSortThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  bool descent = false;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSortThreads;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortThreads; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    const bool ok = i < n;
    const uint64_t k = ok ? keys[i] : 0;
    if (ok && i + 1 < n) descent |= k > keys[i + 1];
    const uint32_t live = __ballot_sync(kFullMask, ok);
#pragma unroll
    for (int b = 0; b < kBytes; ++b) {
      const uint32_t d = ok ? static_cast<uint32_t>(k >> (8 * b)) & 0xffu : 0x100u;
      const uint32_t peers = __match_any_sync(kFullMask, d) & live;
      if (ok && (peers & lanemask_lt()) == 0u) atomicAdd(&h[b][d], __popc(peers));
    }
  }
  if (__syncthreads_or(descent) && threadIdx.x == 0) atomicOr(&ctl->unsorted, 1u);
  for (int i = threadIdx.x; i < kBytes * kBins; i += kSortThreads) {
    const unsigned int c = (&h[0][0])[i];
    if (c) atomicAdd(&(&ctl->hist[0][0])[i], static_cast<unsigned long long>(c));
  }
}

// One block: digit starts per byte, trivial bytes, the buffer each pass reads.
__global__ void __launch_bounds__(kBins) sort_plan_kernel(uint64_t n, SortCtl* ctl) {
  __shared__ unsigned long long part[kBins];
  __shared__ unsigned int triv;
  const int d = threadIdx.x;
  for (int b = 0; b < kBytes; ++b) {
    const unsigned long long c = ctl->hist[b][d];
    if (d == 0) triv = ctl->unsorted ? 0u : 1u;
    __syncthreads();
    if (c == n) triv = 1u;  // every key in one bucket: the pass permutes nothing
    part[d] = c;
    __syncthreads();
    for (int o = 1; o < kBins; o <<= 1) {  // inclusive scan
      const unsigned long long v = d >= o ? part[d - o] : 0ull;
      __syncthreads();
      part[d] += v;
      __syncthreads();
    }
    ctl->hist[b][d] = part[d] - c;  // exclusive: the digit's first output slot
    if (d == 0) ctl->trivial[b] = triv;
    __syncthreads();
  }
  if (d == 0) {
    unsigned int buf = 0, runs = 0;
    for (int b = 0; b < kBytes; ++b) {
      ctl->in_buf[b] = buf;
      ctl->first[b] = runs == 0u;
      if (!ctl->trivial[b]) {
        buf ^= 1u;
        ++runs;
      }
    }
    ctl->final_buf = buf;
    ctl->passes = runs;
  }
}

// Ping-pong buffers: keys[0] is the output key column, keys[1] scratch; the first pass
// that runs reads the (read-only) input key column instead and generates the row index.
struct PassBufs {
  const uint64_t* kfirst;
  uint64_t* keys[2];
  uint32_t* rows[2];
};

struct Cols {
  const uint64_t* in[5];
  uint64_t* out[5];
};

__global__ void __launch_bounds__(kSortThreads) sort_pass_kernel(PassBufs bufs, uint64_t n, int byte, SortCtl* ctl,
                                                                 uint64_t* status) {
  if (ctl->trivial[byte]) return;
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* skeys = reinterpret_cast<uint64_t*>(smem);                              // [kTileKeys]
  uint32_t* srows = reinterpret_cast<uint32_t*>(skeys + kTileKeys);                 // [kTileKeys]
  uint32_t* whist = srows + kTileKeys;                                              // [kSortWarps][kBins + 1]
  unsigned long long* gbase = reinterpret_cast<unsigned long long*>(whist + kSortWarps * (kBins + 1));  // [kBins] (8-aligned: 8 * 257 words)
  uint32_t* loff = reinterpret_cast<uint32_t*>(gbase + kBins);                      // [kBins]
  __shared__ unsigned int tile_s;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) tile_s = atomicAdd(&ctl->tickets[byte], 1u);
  for (int i = tid; i < kSortWarps * (kBins + 1); i += kSortThreads) whist[i] = 0;
  __syncthreads();
  const uint64_t tile = tile_s;
  const uint64_t t0 = tile * kTileKeys;
  const uint32_t ib = ctl->in_buf[byte];
  const bool first = ctl->first[byte] != 0u;
  const uint64_t* __restrict__ kin = first ? bufs.kfirst : bufs.keys[ib];
  const uint32_t* __restrict__ rin = bufs.rows[ib];
  const int shift = 8 * byte;

  // ---- load (warp-striped: item k of lane l is key w*512 + k*32 + l) and rank per warp
  uint64_t key[kItems];
  uint32_t rank[kItems];
  uint32_t* wh = whist + w * (kBins + 1);
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const uint64_t i = t0 + w * (32 * kItems) + k * 32 + lane;
    key[k] = i < n ? kin[i] : ~0ull;
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const uint64_t i = t0 + w * (32 * kItems) + k * 32 + lane;
    const uint32_t d = i < n ? static_cast<uint32_t>(key[k] >> shift) & 0xffu : static_cast<uint32_t>(kBins);
    const uint32_t peers = __match_any_sync(kFullMask, d);
    const uint32_t before = wh[d];
    __syncwarp();
    rank[k] = before + __popc(peers & lt);
    if ((peers & lt) == 0u) wh[d] = before + __popc(peers);
    __syncwarp();
  }
  __syncthreads();

  // ---- digit d (thread d): warp prefixes, tile count, publish, tile-local offsets
  const int d = tid;
  uint32_t cnt = 0;
#pragma unroll
  for (int v = 0; v < kSortWarps; ++v) {
    const uint32_t c = whist[v * (kBins + 1) + d];
    whist[v * (kBins + 1) + d] = cnt;
    cnt += c;
  }
  const uint64_t epoch = static_cast<uint64_t>(byte + 1) << 40;
  volatile uint64_t* st = status;
  if (tile == 0) st[d] = kFlagPrefix | epoch | cnt;
  else st[tile * kBins + d] = kFlagAgg | epoch | cnt;
  // tile-local exclusive scan over the digits
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
    if (lane >= o) incl += v;
  }
  __shared__ uint32_t wsum[kSortWarps];
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  uint32_t wpre = 0;
#pragma unroll
  for (int v = 0; v < kSortWarps; ++v) wpre += v < w ? wsum[v] : 0u;
  loff[d] = wpre + incl - cnt;
  // decoupled look-back for this digit's offset among earlier tiles
  uint64_t excl = 0;
  if (tile > 0) {
    for (int64_t p = static_cast<int64_t>(tile) - 1; p >= 0; --p) {
      uint64_t s;
      do {
        s = st[p * kBins + d];
      } while ((s & (0xffull << 40)) != epoch || (s & (3ull << 48)) == 0);
      excl += s & kValueMask;
      if (s & kFlagPrefix) break;
    }
    st[tile * kBins + d] = kFlagPrefix | epoch | (excl + cnt);
  }
  gbase[d] = ctl->hist[byte][d] + excl;
  __syncthreads();

  // ---- stage the tile in digit order, then write each digit's run contiguously
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const uint32_t j = static_cast<uint32_t>(w * (32 * kItems) + k * 32 + lane);
    if (t0 + j < n) {
      const uint32_t dg = static_cast<uint32_t>(key[k] >> shift) & 0xffu;
      const uint32_t pos = loff[dg] + whist[w * (kBins + 1) + dg] + rank[k];
      LC_CHECK(pos < static_cast<uint32_t>(kTileKeys));
      skeys[pos] = key[k];
      srows[pos] = first ? static_cast<uint32_t>(t0 + j) : rin[t0 + j];
    }
  }
  __syncthreads();
  const uint32_t tn = static_cast<uint32_t>(n - t0 < static_cast<uint64_t>(kTileKeys) ? n - t0 : kTileKeys);
  uint64_t* __restrict__ kout = bufs.keys[ib ^ 1u];
  uint32_t* __restrict__ rout = bufs.rows[ib ^ 1u];
  for (uint32_t j = tid; j < tn; j += kSortThreads) {
    const uint64_t k = skeys[j];
    const uint32_t dg = static_cast<uint32_t>(k >> shift) & 0xffu;
    const uint64_t o = gbase[dg] + (j - loff[dg]);
    LC_CHECK(o < n && j >= loff[dg]);
    kout[o] = k;
    rout[o] = srows[j];
  }
}

// out[c][i] = in[c][row[i]] for the payload columns; keys from the final buffer.
__global__ void sort_gather_kernel(PassBufs bufs, uint64_t n, const SortCtl* ctl, Cols cols, int ncols) {
  const uint32_t fb = ctl->final_buf;
  const bool none = ctl->passes == 0u;  // already ascending: a copy
  const uint64_t* __restrict__ keys = none ? bufs.kfirst : bufs.keys[fb];
  const uint32_t* __restrict__ rows = bufs.rows[fb];
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = none ? i : rows[i];
    if (keys != cols.out[0]) cols.out[0][i] = keys[i];
#pragma unroll
    for (int c = 1; c < 5; ++c)
      if (c < ncols && cols.in[c]) cols.out[c][i] = cols.in[c][r];
  }
}

constexpr size_t kPassSmem = kTileKeys * (8 + 4) + (kSortWarps * (kBins + 1) + 1) * 4 + kBins * 8 + kBins * 4 + 16;

inline size_t align256(size_t b) { return (b + 255) & ~size_t{255}; }

}  // namespace

size_t radix_sort_scratch_bytes(uint64_t n) {
  const uint64_t tiles = (n + kTileKeys - 1) / kTileKeys;
  return align256(sizeof(SortCtl)) + align256(n * 8) + 2 * align256(n * 4) + align256(tiles * kBins * 8);
}

// cols_in[0] is the key column; out-of-place (cols_out[c] must not alias any cols_in);
// null payload columns are skipped.  Rows are 32-bit: n < 2^32.  Enqueued without a host
// synchronisation.
cudaError_t radix_sort_records(uint64_t n, const uint64_t* const* cols_in, uint64_t* const* cols_out, int ncols,
                               void* scratch, size_t scratch_bytes, cudaStream_t st, int* launches) {
  if (n >= (1ull << 32) || ncols < 1 || ncols > 5) return cudaErrorInvalidValue;
  if (scratch_bytes < radix_sort_scratch_bytes(n)) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  SortCtl* ctl = reinterpret_cast<SortCtl*>(p);
  p += align256(sizeof(SortCtl));
  uint64_t* kbuf = reinterpret_cast<uint64_t*>(p);
  p += align256(n * 8);
  uint32_t* r0 = reinterpret_cast<uint32_t*>(p);
  p += align256(n * 4);
  uint32_t* r1 = reinterpret_cast<uint32_t*>(p);
  p += align256(n * 4);
  const uint64_t tiles = (n + kTileKeys - 1) / kTileKeys;
  uint64_t* status = reinterpret_cast<uint64_t*>(p);
  cudaError_t e;
  if ((e = cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(status, 0, tiles * kBins * 8, st)) != cudaSuccess) return e;
  PassBufs bufs{cols_in[0], {cols_out[0], kbuf}, {r0, r1}};
  Cols cols{};
  for (int c = 0; c < 5; ++c) {
    cols.in[c] = c < ncols ? cols_in[c] : nullptr;
    cols.out[c] = c < ncols ? cols_out[c] : nullptr;
  }
  int dev = 0, sms = 1;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const uint64_t hb = std::min<uint64_t>((n + kSortThreads - 1) / kSortThreads, static_cast<uint64_t>(sms) * 8);
  sort_hist_kernel<<<static_cast<unsigned>(hb), kSortThreads, 0, st>>>(cols_in[0], n, ctl);
  sort_plan_kernel<<<1, kBins, 0, st>>>(n, ctl);
  if ((e = cudaFuncSetAttribute(sort_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kPassSmem))) != cudaSuccess)
    return e;
  for (int b = 0; b < kBytes; ++b)  // trivial bytes return at once (decided on the device)
    sort_pass_kernel<<<static_cast<unsigned>(tiles), kSortThreads, kPassSmem, st>>>(bufs, n, b, ctl, status);
  const uint64_t gb = std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sms) * 16);
  sort_gather_kernel<<<static_cast<unsigned>(gb), 256, 0, st>>>(bufs, n, ctl, cols, ncols);
  *launches += 3 + kBytes;
  return cudaGetLastError();
}

}  // namespace lc
