// Edge-output sort: records ascending by source, the invariant
// of the edge file and of step 4 (records.py:3-5, reduce.py:3-4).
//
// An LSD radix sort of the 64-bit source keys, one byte per pass, each pass a single
// "onesweep" kernel (no separate upsweep per pass):
//   * one histogram kernel reads the keys once and counts all eight byte digits
//     (block-shared counters; a digit shared by the whole warp -- a constant byte -- is
//     one add), and notes whether the keys are already ascending;
//   * a one-block plan kernel turns the counts into per-byte digit starts, marks trivial
//     bytes (every key in one bucket -- for A5/1 skeletons the R3 bytes, which all equal
//     the fixed value -- or an already sorted input; their pass kernels return at once)
//     and assigns the ping-pong buffers backwards from the last pass that runs, so the
//     whole sort is enqueued without a host round trip;
//   * a pass kernel takes tiles of 2816 keys in launch order (an atomic ticket, so a
//     tile's predecessors are always resident): it loads the tile's keys into registers
//     and its row payload into shared memory (cp.async, overlapping the ranking), ranks
//     each key within its warp (match on the digit, warp-private counters), publishes
//     the tile's 256 digit counts and looks back over earlier tiles for each digit's
//     global offset (decoupled look-back: 256 independent chains, one per thread), stages
//     the tile in shared memory in digit order and writes each digit's run contiguously.
//     Ranking in input order makes every pass stable, so equal sources keep their input
//     order (numpy's stable argsort).
//   * The last pass that runs writes the output key column and gathers the payload
//     columns (destination, distance, subtree size/depth) by row directly into the
//     output columns -- no separate gather pass.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "lfsr_internal.h"

namespace lc {
namespace {

#ifndef LC_SORT_MATCH_ANY
#define LC_SORT_MATCH_ANY 0  // 1: rank with __match_any_sync (A/B)
#endif

constexpr uint32_t kFullMask = 0xffffffffu;
#ifndef LC_SORT_THREADS
#define LC_SORT_THREADS 256
#endif
constexpr int kSortThreads = LC_SORT_THREADS;  // a multiple of 256 (threads 0..255 own a digit each)
constexpr int kSortWarps = kSortThreads / 32;
#ifndef LC_SORT_ITEMS
#define LC_SORT_ITEMS 11
#endif
#ifndef LC_SORT_MINBLOCKS
#define LC_SORT_MINBLOCKS 4
#endif
constexpr int kItems = LC_SORT_ITEMS;               // keys per thread
constexpr int kTileKeys = kSortThreads * kItems;    // 2816 (4 blocks per SM: 56 KB each)
constexpr int kBins = 256;
constexpr int kBytes = 8;
constexpr int kCols = 5;
// look-back status word: [49:48] flag, [47:40] epoch (pass byte + 1), [39:0] count
constexpr uint64_t kFlagAgg = 1ull << 48, kFlagPrefix = 2ull << 48;
constexpr uint64_t kValueMask = (1ull << 40) - 1;

struct SortCtl {
  unsigned long long hist[kBytes][kBins];  // digit counts, then (plan) digit starts
  unsigned int tickets[kBytes];
  unsigned int unsorted;
  unsigned int trivial[kBytes];
  unsigned int in_buf[kBytes];  // buffer a pass reads (keys / rows), 2 = the input column
  unsigned int last[kBytes];    // 1: the last pass that runs (writes the output columns)
  unsigned int passes;
  // digit slot b = (key >> shift[b]) & dmask[b]: bytes for the LSD sort, bit windows for
  // the MSD passes (set by msd_plan_kernel); slots >= nslots are trivial
  unsigned int shift[kBytes];
  unsigned int dmask[kBytes];
  unsigned int nslots;
  unsigned int epoch_base;      // look-back epochs (the status array is shared)
  unsigned int output_last;     // 1: the last pass writes the output columns (LSD)
};

// The MSD route (see radix_sort_records): varying bits, the plan, the bucket table.
struct MsdCtl {
  unsigned int vary[2];         // OR over keys of (key ^ key[0]), low / high word
  unsigned int use_msd;         // 1: MSD passes + per-bucket local sorts
  unsigned int fallback;        // 1: a bucket outgrew the local sort: the LSD passes run
  unsigned int win_shift;       // lowest bit of the MSD window
  unsigned int local_shift[kBytes];
  unsigned int local_mask[kBytes];
  unsigned int local_passes;
};

struct Cols {
  const uint64_t* in[kCols];
  uint64_t* out[kCols];
};

// keys[0] = output key column, keys[1] = scratch; rows[0..1] scratch
struct PassBufs {
  uint64_t* keys[2];
  uint32_t* rows[2];
};

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Lanes holding the same 9-bit digit (256 = past the end): one ballot per bit
// (MATCH.ANY serialises over the distinct values of a warp, 32 for random digits).
__device__ __forceinline__ uint32_t peers_of(uint32_t d) {
#if LC_SORT_MATCH_ANY
  return __match_any_sync(kFullMask, d);
#else
  uint32_t m = kFullMask;
#pragma unroll
  for (int i = 0; i < 9; ++i) {
    const uint32_t b = __ballot_sync(kFullMask, (d >> i) & 1u);
    m &= ((d >> i) & 1u) ? b : ~b;
  }
  return m;
#endif
}

// lanes holding the same 10-bit value (local digits of up to 9 bits, 512 = past the end)
__device__ __forceinline__ uint32_t peers_of10(uint32_t d) {
  uint32_t m = kFullMask;
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    const uint32_t b = __ballot_sync(kFullMask, (d >> i) & 1u);
    m &= ((d >> i) & 1u) ? b : ~b;
  }
  return m;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t s = static_cast<uint32_t>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

#ifndef LC_SORT_GATHER
#define LC_SORT_GATHER 3  // payload gather: 0 two 16-B .nc loads, 1 two 16-B .cg, 2 one 32-B .nc, 3 one 32-B .cg
#endif
// one 32-byte payload record (a random sector of the record-major payload)
__device__ __forceinline__ void gather32(const ulonglong2* __restrict__ aos, uint64_t r, ulonglong2& a, ulonglong2& b) {
#if LC_SORT_GATHER == 0
  a = aos[2 * r];
  b = aos[2 * r + 1];
#elif LC_SORT_GATHER == 1
  a = __ldcg(aos + 2 * r);
  b = __ldcg(aos + 2 * r + 1);
#elif LC_SORT_GATHER == 2
  asm("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y) : "l"(aos + 2 * r));
#else
  asm("ld.global.cg.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a.x), "=l"(a.y), "=l"(b.x), "=l"(b.y) : "l"(aos + 2 * r));
#endif
}

// Also packs the payload columns record-major (32 B per record: destination, distance,
// subtree size, subtree depth; missing columns as 0), so the last pass fetches one
// aligned 32-byte sector per record instead of one scattered sector per column.
__global__ void __launch_bounds__(kSortThreads) sort_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                                 SortCtl* ctl, Cols cols, ulonglong2* __restrict__ aos,
                                                                 MsdCtl* msd) {
  __shared__ unsigned int h[kBytes][kBins];
  for (int i = threadIdx.x; i < kBytes * kBins; i += kSortThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  bool descent = false;
  const uint64_t k0 = keys[0];
  uint64_t vary = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSortThreads;
  for (uint64_t base = static_cast<uint64_t>(blockIdx.x) * kSortThreads; base < n; base += stride) {
    const uint64_t i = base + threadIdx.x;
    const bool ok = i < n;
    const uint64_t k = ok ? keys[i] : 0;
    if (ok && i + 1 < n) descent |= k > keys[i + 1];
    if (ok) vary |= k ^ k0;
    if (ok) {
      aos[2 * i] = make_ulonglong2(cols.in[1] ? cols.in[1][i] : 0ull, cols.in[2] ? cols.in[2][i] : 0ull);
      aos[2 * i + 1] = make_ulonglong2(cols.in[3] ? cols.in[3][i] : 0ull, cols.in[4] ? cols.in[4][i] : 0ull);
    }
    const uint32_t live = __ballot_sync(kFullMask, ok);
#pragma unroll
    for (int b = 0; b < kBytes; ++b) {
      const uint32_t d = static_cast<uint32_t>(k >> (8 * b)) & 0xffu;
      const uint32_t d0 = __shfl_sync(kFullMask, d, 0);  // every lane takes part (no short circuit)
      const bool uniform = __all_sync(kFullMask, !ok || d == d0);
      if (uniform) {
        if ((threadIdx.x & 31) == 0) atomicAdd(&h[b][d], __popc(live));
      } else if (ok) {
        atomicAdd(&h[b][d], 1u);
      }
    }
  }
  if (__syncthreads_or(descent) && threadIdx.x == 0) atomicOr(&ctl->unsorted, 1u);
  {
    uint32_t lo = static_cast<uint32_t>(vary), hi = static_cast<uint32_t>(vary >> 32);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      lo |= __shfl_xor_sync(kFullMask, lo, o);
      hi |= __shfl_xor_sync(kFullMask, hi, o);
    }
    if ((threadIdx.x & 31) == 0) {
      if (lo) atomicOr(&msd->vary[0], lo);
      if (hi) atomicOr(&msd->vary[1], hi);
    }
  }
  for (int i = threadIdx.x; i < kBytes * kBins; i += kSortThreads) {
    const unsigned int c = (&h[0][0])[i];
    if (c) atomicAdd(&(&ctl->hist[0][0])[i], static_cast<unsigned long long>(c));
  }
}

// One block: digit starts per byte, trivial bytes, and the buffers: the last pass that
// runs writes the output columns, so buffers alternate backwards from it; the first reads
// the input key column and makes up the row payload.
__global__ void __launch_bounds__(kBins) sort_plan_kernel(uint64_t n, SortCtl* ctl) {
  __shared__ unsigned long long part[kBins];
  __shared__ unsigned int triv;
  const int d = threadIdx.x;
  for (int b = 0; b < kBytes; ++b) {
    const unsigned long long c = ctl->hist[b][d];
    if (d == 0) triv = ctl->unsorted && static_cast<unsigned int>(b) < ctl->nslots ? 0u : 1u;
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
    unsigned int runs = 0;
    for (int b = 0; b < kBytes; ++b) runs += ctl->trivial[b] ? 0u : 1u;
    unsigned int j = 0;  // index among the passes that run
    for (int b = 0; b < kBytes; ++b) {
      ctl->last[b] = 0u;
      ctl->in_buf[b] = 0u;
      if (ctl->trivial[b]) continue;
      // pass j writes buffer (runs - 1 - j) & 1 (the last one: 0 = the output key column),
      // so it reads what pass j - 1 wrote, (runs - j) & 1; pass 0 reads the input (2)
      ctl->in_buf[b] = j == 0 ? 2u : ((runs - j) & 1u);
      ctl->last[b] = j + 1 == runs && ctl->output_last;
      ++j;
    }
    ctl->passes = runs;
  }
}

constexpr int kWhistStride = kBins + 1;  // one spare counter per warp for lanes past the end
constexpr size_t kSmemKeys = kTileKeys * 8, kSmemRows = kTileKeys * 4;
constexpr size_t kPassSmem = kSmemKeys + 2 * kSmemRows + (kSortWarps * kWhistStride + 8) * 4 + kBins * 8 + kBins * 4;

template <bool kPersistent>
__global__ void __launch_bounds__(kSortThreads, LC_SORT_MINBLOCKS) sort_pass_kernel(PassBufs bufs, Cols cols, uint64_t n, int byte,
                                                                    SortCtl* ctl, uint64_t* status,
                                                                    const ulonglong2* __restrict__ aos,
                                                                    const MsdCtl* lsd_gate) {
  if (ctl->trivial[byte]) return;
  if (lsd_gate && lsd_gate->use_msd && !lsd_gate->fallback) return;  // the MSD route sorted it
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* skeys = reinterpret_cast<uint64_t*>(smem);                         // staged keys [kTileKeys]
  uint32_t* srows = reinterpret_cast<uint32_t*>(smem + kSmemKeys);             // staged rows [kTileKeys]
  uint32_t* irows = reinterpret_cast<uint32_t*>(smem + kSmemKeys + kSmemRows); // input rows, input order
  uint32_t* whist = irows + kTileKeys;                                         // [kSortWarps][kWhistStride]
  unsigned long long* gbase = reinterpret_cast<unsigned long long*>(whist + kSortWarps * kWhistStride + 8);
  uint32_t* loff = reinterpret_cast<uint32_t*>(gbase + kBins);
  __shared__ unsigned int tile_s;
  __shared__ uint32_t wsum[kBins / 32];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint64_t ntiles = (n + kTileKeys - 1) / kTileKeys;
  // persistent: a grid of resident blocks each taking tiles until none is left (the
  // launches that usually return at once: the LSD passes behind the MSD route)
  for (;;) {
    if (tid == 0) tile_s = atomicAdd(&ctl->tickets[byte], 1u);
    for (int i = tid; i < kSortWarps * kWhistStride; i += kSortThreads) whist[i] = 0;
    __syncthreads();
    const uint64_t tile = tile_s;
    if (tile >= ntiles) return;  // block-uniform
    const uint64_t t0 = tile * kTileKeys;
    const uint32_t tn = static_cast<uint32_t>(n - t0 < static_cast<uint64_t>(kTileKeys) ? n - t0 : kTileKeys);
    const uint32_t ib = ctl->in_buf[byte];
    const bool first = ib == 2u, last = ctl->last[byte] != 0u;
    const uint64_t* __restrict__ kin = first ? cols.in[0] : bufs.keys[ib];
    const int shift = static_cast<int>(ctl->shift[byte]);
    const uint32_t dmask = ctl->dmask[byte];

    // ---- the row payload to shared memory in input order (async), keys to registers
    if (!first) {
      const uint32_t* __restrict__ rin = bufs.rows[ib] + t0;
      if (tn == static_cast<uint32_t>(kTileKeys)) {
        for (int c = tid; c < kTileKeys / 4; c += kSortThreads) cp_async16(irows + 4 * c, rin + 4 * c);
      } else {
        for (uint32_t j = tid; j < tn; j += kSortThreads) irows[j] = rin[j];
      }
    }
    uint64_t key[kItems];
    uint32_t rank[kItems];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t j = static_cast<uint32_t>(w * (32 * kItems) + k * 32 + lane);
      key[k] = j < tn ? kin[t0 + j] : ~0ull;
    }
    // ---- rank within the warp (warp-striped: item k of lane l is tile key w*32*kItems + k*32 + l)
    uint32_t* wh = whist + w * kWhistStride;
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t j = static_cast<uint32_t>(w * (32 * kItems) + k * 32 + lane);
      const uint32_t d = j < tn ? static_cast<uint32_t>(key[k] >> shift) & dmask : static_cast<uint32_t>(kBins);
      const uint32_t peers = peers_of(d);
      const uint32_t before = wh[d];
      __syncwarp();
      rank[k] = before + __popc(peers & lt);
      if ((peers & lt) == 0u) wh[d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();

    // ---- digit d (thread d < 256): warp prefixes, tile count, publish, tile-local offsets
    const int d = tid;
    const bool owns_digit = tid < kBins;  // whole warps
    uint32_t cnt = 0, incl = 0;
    const uint64_t epoch = static_cast<uint64_t>(ctl->epoch_base + byte + 1) << 40;
    volatile uint64_t* st = status;
    if (owns_digit) {
#pragma unroll
      for (int v = 0; v < kSortWarps; ++v) {
        const uint32_t c = whist[v * kWhistStride + d];
        whist[v * kWhistStride + d] = cnt;
        cnt += c;
      }
      if (tile == 0) st[d] = kFlagPrefix | epoch | cnt;
      else st[tile * kBins + d] = kFlagAgg | epoch | cnt;
      incl = cnt;  // tile-local exclusive scan over the digits
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) wsum[w] = incl;
    }
    __syncthreads();
    if (owns_digit) {
      uint32_t wpre = 0;
#pragma unroll
      for (int v = 0; v < kBins / 32; ++v) wpre += v < w ? wsum[v] : 0u;
      loff[d] = wpre + incl - cnt;
      uint64_t excl = 0;  // decoupled look-back: this digit's offset among earlier tiles
      if (tile > 0) {
        for (int64_t p = static_cast<int64_t>(tile) - 1; p >= 0; --p) {
          uint64_t sv;
          do {
            sv = st[p * kBins + d];
          } while ((sv & (0xffull << 40)) != epoch || (sv & (3ull << 48)) == 0);
          excl += sv & kValueMask;
          if (sv & kFlagPrefix) break;
        }
        st[tile * kBins + d] = kFlagPrefix | epoch | (excl + cnt);
      }
      gbase[d] = ctl->hist[byte][d] + excl;
    }
    if (!first) cp_async_wait_all();
    __syncthreads();

    // ---- stage the tile in digit order
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t j = static_cast<uint32_t>(w * (32 * kItems) + k * 32 + lane);
      if (j < tn) {
        const uint32_t dg = static_cast<uint32_t>(key[k] >> shift) & dmask;
        const uint32_t pos = loff[dg] + whist[w * kWhistStride + dg] + rank[k];
        LC_CHECK(pos < static_cast<uint32_t>(kTileKeys));
        skeys[pos] = key[k];
        srows[pos] = first ? static_cast<uint32_t>(t0 + j) : irows[j];
      }
    }
    __syncthreads();

    // ---- write each digit's run contiguously; the last pass gathers the payload columns
    if (!last) {
      const uint32_t ob = first ? 1u - (ctl->passes & 1u) : ib ^ 1u;  // (passes - 1) & 1 for pass 0
      uint64_t* __restrict__ kout = bufs.keys[ob];
      uint32_t* __restrict__ rout = bufs.rows[ob];
      for (uint32_t j = tid; j < tn; j += kSortThreads) {
        const uint64_t k = skeys[j];
        const uint32_t dg = static_cast<uint32_t>(k >> shift) & dmask;
        const uint64_t o = gbase[dg] + (j - loff[dg]);
        LC_CHECK(o < n && j >= loff[dg]);
        kout[o] = k;
        rout[o] = srows[j];
      }
    } else {
      uint64_t* __restrict__ kout = cols.out[0];
      constexpr int U = 4;  // records per thread per round: U payload sectors in flight
      for (uint32_t j0 = tid; j0 < tn; j0 += kSortThreads * U) {
        uint64_t o[U];
        ulonglong2 a[U], b[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * kSortThreads;
          if (j < tn) {
            const uint64_t k = skeys[j];
            const uint32_t dg = static_cast<uint32_t>(k >> shift) & dmask;
            o[u] = gbase[dg] + (j - loff[dg]);
            LC_CHECK(o[u] < n && j >= loff[dg]);
            kout[o[u]] = k;
            gather32(aos, srows[j], a[u], b[u]);
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t j = j0 + u * kSortThreads;
          if (j < tn) {
            if (cols.out[1]) cols.out[1][o[u]] = a[u].x;
            if (cols.out[2]) cols.out[2][o[u]] = a[u].y;
            if (cols.out[3]) cols.out[3][o[u]] = b[u].x;
            if (cols.out[4]) cols.out[4][o[u]] = b[u].y;
          }
        }
      }
    }
    if (!kPersistent) return;
    __syncthreads();  // the shared tile buffers and tile_s are reused
  }
}

// ------------------------------------------------------------------ the MSD route
// For large unsorted inputs whose keys vary over more than the MSD window: W top varying
// bits (W = ceil(log2 n) - 10, so a bucket holds ~1024 records on average) are sorted by
// two or three onesweep passes (the same pass kernel, bit-window digits), which leaves
// the records grouped by their top W bits, in input order within a group; then one block
// per group sorts it by the remaining low bits in shared memory (stable LSD passes) and
// writes the output columns, gathering the payload.  Fewer global passes over the data
// than one per byte; a group too big for shared memory sends the whole sort down the
// LSD route instead (fallback flag, decided on the device).
#ifndef LC_SORT_LOCAL_THREADS
#define LC_SORT_LOCAL_THREADS 256  // one thread per digit in the offset step
#endif
#ifndef LC_SORT_LOCAL_ITEMS
#define LC_SORT_LOCAL_ITEMS 8
#endif
constexpr int kLocalThreads = LC_SORT_LOCAL_THREADS;
constexpr int kLocalItems = LC_SORT_LOCAL_ITEMS;
constexpr int kLocalCap = kLocalThreads * kLocalItems;  // records per group sorted in shared memory
constexpr int kLocalDigitBits = 9;                      // local digits: up to 512 bins
constexpr int kLocalBins = 1 << kLocalDigitBits;
constexpr int kLocalStride = kLocalBins + 1;            // one spare counter per warp for lanes past the end
constexpr int kLocalWarps = kLocalThreads / 32;
constexpr size_t kLocalSmem = kLocalCap * 8 + kLocalCap * 4 + (kLocalWarps * kLocalStride + kLocalBins + kBins / 32) * 4;
static_assert(kLocalBins % kLocalThreads == 0 && kLocalWarps <= 32, "the offset step's digit split");

// one thread: the route and its digits from the varying bits
__global__ void msd_plan_kernel(uint64_t n, uint32_t W, SortCtl* lsd, SortCtl* m, MsdCtl* msd) {
  const uint64_t vary = static_cast<uint64_t>(msd->vary[0]) | (static_cast<uint64_t>(msd->vary[1]) << 32);
  const int hbit = vary ? 63 - __clzll(static_cast<long long>(vary)) : -1;
  const int lbit = vary ? __ffsll(static_cast<long long>(vary)) - 1 : 0;
  const bool use = lsd->unsorted && vary && hbit - lbit + 1 > static_cast<int>(W);
  msd->use_msd = use ? 1u : 0u;
  m->nslots = 0;
  msd->local_passes = 0;
  if (!use) return;
  const int wlo = hbit - static_cast<int>(W) + 1;
  msd->win_shift = static_cast<unsigned int>(wlo);
  const int nd = (static_cast<int>(W) + 7) / 8, wd = (static_cast<int>(W) + nd - 1) / nd;
  for (int sidx = 0; sidx < nd; ++sidx) {  // low digit of the window first (LSD within it)
    const int bits = min(wd, static_cast<int>(W) - sidx * wd);
    m->shift[sidx] = static_cast<unsigned int>(wlo + sidx * wd);
    m->dmask[sidx] = (1u << bits) - 1u;
  }
  m->nslots = static_cast<unsigned int>(nd);
  m->unsorted = 1u;
  const int lw = wlo - lbit;  // low bits [lbit, wlo) sorted per group, digits of <= 9 bits
  const int np = (lw + kLocalDigitBits - 1) / kLocalDigitBits;
  const int pw = np ? (lw + np - 1) / np : 0;
  for (int p = 0; p < np; ++p) {
    const int bits = min(pw, lw - pw * p);
    msd->local_shift[p] = static_cast<unsigned int>(lbit + pw * p);
    msd->local_mask[p] = (1u << bits) - 1u;
  }
  msd->local_passes = static_cast<unsigned int>(np);
}

// histograms of the MSD window's digits
__global__ void __launch_bounds__(kSortThreads) msd_hist_kernel(const uint64_t* __restrict__ keys, uint64_t n,
                                                                SortCtl* m, const MsdCtl* msd) {
  if (!msd->use_msd) return;
  __shared__ unsigned int h[3][kBins];
  for (int i = threadIdx.x; i < 3 * kBins; i += kSortThreads) (&h[0][0])[i] = 0;
  __syncthreads();
  const unsigned int nd = m->nslots;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kSortThreads;
  const uint64_t t = static_cast<uint64_t>(blockIdx.x) * kSortThreads + threadIdx.x;
  const uint64_t n4 = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0 ? n / 4 : 0;  // four keys per thread and round
  const ulonglong2* __restrict__ k2 = reinterpret_cast<const ulonglong2*>(keys);
  for (uint64_t q = t; q < n4; q += stride) {
    const ulonglong2 a = k2[2 * q], c = k2[2 * q + 1];
    const uint64_t k[4] = {a.x, a.y, c.x, c.y};
    for (unsigned int b = 0; b < nd; ++b) {
      const unsigned int shb = m->shift[b], mb = m->dmask[b];
#pragma unroll
      for (int j = 0; j < 4; ++j) atomicAdd(&h[b][static_cast<uint32_t>(k[j] >> shb) & mb], 1u);
    }
  }
  for (uint64_t i = 4 * n4 + t; i < n; i += stride) {
    const uint64_t k = keys[i];
    for (unsigned int b = 0; b < nd; ++b) atomicAdd(&h[b][static_cast<uint32_t>(k >> m->shift[b]) & m->dmask[b]], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < static_cast<int>(nd) * kBins; i += kSortThreads) {
    const unsigned int c = (&h[0][0])[i];
    if (c) atomicAdd(&(&m->hist[0][0])[i], static_cast<unsigned long long>(c));
  }
}

// group g = records whose window equals g: [start[g], end[g]) of the MSD-sorted keys;
// four keys per thread and round (two 16-byte loads: enough bytes in flight for HBM),
// the neighbours across the quad from L1 / L2
__global__ void msd_bounds_kernel(const uint64_t* __restrict__ keys, uint64_t n, uint32_t W, const MsdCtl* msd,
                                  uint32_t* __restrict__ gstart, uint32_t* __restrict__ gend) {
  if (!msd->use_msd) return;
  const uint32_t sh = msd->win_shift;
  const uint64_t wm = (1ull << W) - 1ull;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  const uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x;
  const uint64_t n4 = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0 ? n / 4 : 0;
  const ulonglong2* __restrict__ k2 = reinterpret_cast<const ulonglong2*>(keys);
  for (uint64_t q = t; q < n4; q += stride) {
    const ulonglong2 a = k2[2 * q], b = k2[2 * q + 1];
    const uint64_t i = 4 * q;
    const uint64_t g[6] = {i == 0 ? ~0ull : (keys[i - 1] >> sh) & wm, (a.x >> sh) & wm, (a.y >> sh) & wm,
                           (b.x >> sh) & wm, (b.y >> sh) & wm, i + 4 >= n ? ~0ull : (keys[i + 4] >> sh) & wm};
#pragma unroll
    for (int j = 1; j <= 4; ++j) {
      if (g[j - 1] != g[j]) gstart[g[j]] = static_cast<uint32_t>(i + j - 1);
      if (g[j + 1] != g[j]) gend[g[j]] = static_cast<uint32_t>(i + j);
    }
  }
  for (uint64_t i = 4 * n4 + t; i < n; i += stride) {
    const uint64_t g = (keys[i] >> sh) & wm;
    if (i == 0 || ((keys[i - 1] >> sh) & wm) != g) gstart[g] = static_cast<uint32_t>(i);
    if (i + 1 == n || ((keys[i + 1] >> sh) & wm) != g) gend[g] = static_cast<uint32_t>(i + 1);
  }
}

// one block per group: stable LSD passes over the low bits (records in registers,
// warp-striped in input order; each pass ranks them within their warps, scatters them
// through one shared-memory buffer in digit order and reloads), then the output columns
// (keys, and the payload gathered by row)
#ifndef LC_SORT_LOCAL_MINBLOCKS
#define LC_SORT_LOCAL_MINBLOCKS 3
#endif
__global__ void __launch_bounds__(kLocalThreads, LC_SORT_LOCAL_MINBLOCKS) msd_local_kernel(PassBufs bufs, Cols cols, MsdCtl* msd,
                                                                  const uint32_t* __restrict__ gstart,
                                                                  const uint32_t* __restrict__ gend,
                                                                  const ulonglong2* __restrict__ aos) {
  if (!msd->use_msd) return;
  const uint32_t e = gend[blockIdx.x];
  if (e == 0) return;  // empty group
  const uint32_t s0 = gstart[blockIdx.x];
  const uint32_t size = e - s0;
  if (size > static_cast<uint32_t>(kLocalCap)) {
    if (threadIdx.x == 0) atomicExch(&msd->fallback, 1u);
    return;
  }
  extern __shared__ __align__(16) uint8_t smem[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(smem);
  uint32_t* srow = reinterpret_cast<uint32_t*>(skey + kLocalCap);
  uint32_t* whist = srow + kLocalCap;                      // [kLocalWarps][kLocalStride]
  uint32_t* loff = whist + kLocalWarps * kLocalStride;     // [kLocalBins]
  uint32_t* wsum = loff + kLocalBins;                      // [kLocalWarps]
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const uint32_t wbase = static_cast<uint32_t>(w * (32 * kLocalItems));
  const uint64_t* __restrict__ kin = bufs.keys[0] + s0;  // the MSD passes end in buffer 0
  const uint32_t* __restrict__ rin = bufs.rows[0] + s0;
  uint64_t key[kLocalItems];
  uint32_t row[kLocalItems];
#pragma unroll
  for (int k = 0; k < kLocalItems; ++k) {
    const uint32_t j = wbase + k * 32 + lane;
    key[k] = j < size ? kin[j] : 0ull;
    row[k] = j < size ? rin[j] : 0u;
  }
  const uint32_t lt = lanemask_lt();
  const unsigned int np = msd->local_passes;
  for (unsigned int p = 0; p < np; ++p) {
    const int shift = static_cast<int>(msd->local_shift[p]);
    const uint32_t dmask = msd->local_mask[p];
    for (int i = tid; i < kLocalWarps * kLocalStride; i += kLocalThreads) whist[i] = 0;
    __syncthreads();
    uint32_t rank[kLocalItems];
    uint32_t* wh = whist + w * kLocalStride;
#pragma unroll
    for (int k = 0; k < kLocalItems; ++k) {  // in input order within the warp: stable
      if (wbase + k * 32 >= size) break;     // (warp-uniform: the warp's records are done)
      const uint32_t j = wbase + k * 32 + lane;
      const uint32_t d = j < size ? static_cast<uint32_t>(key[k] >> shift) & dmask : static_cast<uint32_t>(kLocalBins);
      const uint32_t peers = peers_of10(d);
      const uint32_t before = wh[d];
      __syncwarp();
      rank[k] = before + __popc(peers & lt);
      if ((peers & lt) == 0u) wh[d] = before + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    {  // digits 2t and 2t+1 (thread t): earlier warps' counts within each digit, then
       // the digits' offsets (a block scan over the threads' pairs)
      constexpr int DPT = kLocalBins / kLocalThreads;
      uint32_t cnt[DPT], tot = 0;
#pragma unroll
      for (int q = 0; q < DPT; ++q) {
        const int d = tid * DPT + q;
        uint32_t c0 = 0;
#pragma unroll
        for (int v = 0; v < kLocalWarps; ++v) {
          const uint32_t c = whist[v * kLocalStride + d];
          whist[v * kLocalStride + d] = c0;
          c0 += c;
        }
        cnt[q] = c0;
        tot += c0;
      }
      uint32_t incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFullMask, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) wsum[w] = incl;
      __syncthreads();
      uint32_t run = incl - tot;
#pragma unroll
      for (int v = 0; v < kLocalWarps; ++v) run += v < w ? wsum[v] : 0u;
#pragma unroll
      for (int q = 0; q < DPT; ++q) {
        loff[tid * DPT + q] = run;
        run += cnt[q];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kLocalItems; ++k) {
      const uint32_t j = wbase + k * 32 + lane;
      if (j < size) {
        const uint32_t d = static_cast<uint32_t>(key[k] >> shift) & dmask;
        const uint32_t pos = loff[d] + whist[w * kLocalStride + d] + rank[k];
        LC_CHECK(pos < size);
        skey[pos] = key[k];
        srow[pos] = row[k];
      }
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kLocalItems; ++k) {  // reload in the new order
      const uint32_t j = wbase + k * 32 + lane;
      if (j < size) {
        key[k] = skey[j];
        row[k] = srow[j];
      }
    }
  }
  // the output columns: keys in order, the payload gathered by row (32-byte records),
  // four gathers in flight per thread
  constexpr int U = 4;
#pragma unroll
  for (int k0 = 0; k0 < kLocalItems; k0 += U) {
    ulonglong2 a[U], b[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = wbase + (k0 + u) * 32 + lane;
      if (j < size) {
        gather32(aos, row[k0 + u], a[u], b[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t j = wbase + (k0 + u) * 32 + lane;
      if (j < size) {
        const uint64_t o = static_cast<uint64_t>(s0) + j;
        cols.out[0][o] = key[k0 + u];
        if (cols.out[1]) cols.out[1][o] = a[u].x;
        if (cols.out[2]) cols.out[2][o] = a[u].y;
        if (cols.out[3]) cols.out[3][o] = b[u].x;
        if (cols.out[4]) cols.out[4][o] = b[u].y;
      }
    }
  }
}

// Already ascending (no pass runs): the output columns are a copy of the input.
__global__ void sort_copy_kernel(uint64_t n, const SortCtl* ctl, Cols cols, const MsdCtl* msd) {
  if (ctl->passes != 0u) return;
  if (msd->use_msd && !msd->fallback) return;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
#pragma unroll
    for (int c = 0; c < kCols; ++c)
      if (cols.in[c]) cols.out[c][i] = cols.in[c][i];
  }
}

inline size_t align256(size_t b) { return (b + 255) & ~size_t{255}; }

// MSD window width for n records (groups of ~1024 on average), or 0: LSD only
uint32_t msd_window_bits(uint64_t n) {
  if (n < (1ull << 16)) return 0;
  const uint32_t lg = 64u - static_cast<uint32_t>(__builtin_clzll(n - 1));  // ceil(log2 n)
  return std::min(std::max(lg - 10u, 8u), 22u);
}

// set up both plans' fixed fields (bytes for the LSD route)
__global__ void sort_init_kernel(SortCtl* lsd, SortCtl* m) {
  const int b = threadIdx.x;
  if (b < kBytes) {
    lsd->shift[b] = 8u * b;
    lsd->dmask[b] = 0xffu;
  }
  if (b == 0) {
    lsd->nslots = kBytes;
    lsd->epoch_base = 0;
    lsd->output_last = 1;
    m->epoch_base = kBytes;
    m->output_last = 0;
  }
}

}  // namespace

size_t radix_sort_scratch_bytes(uint64_t n) {
  const uint64_t tiles = (n + kTileKeys - 1) / kTileKeys;
  const uint32_t W = msd_window_bits(n);
  const uint64_t groups = W ? (1ull << W) : 1ull;
  return 2 * align256(sizeof(SortCtl)) + align256(sizeof(MsdCtl)) + align256(n * 8) + 2 * align256(n * 4) +
         align256(tiles * kBins * 8) + align256(n * 32) + 2 * align256(groups * 4);
}

// cols_in[0] is the key column; out of place (cols_out[c] must not alias any cols_in);
// null payload columns are skipped.  Rows are 32-bit: n < 2^32.  Enqueued without a host
// synchronisation: both routes are launched and the device's plan decides which one's
// kernels return at once.
cudaError_t radix_sort_records(uint64_t n, const uint64_t* const* cols_in, uint64_t* const* cols_out, int ncols,
                               void* scratch, size_t scratch_bytes, cudaStream_t st, int* launches) {
  if (n >= (1ull << 32) || ncols < 1 || ncols > kCols) return cudaErrorInvalidValue;
  if (scratch_bytes < radix_sort_scratch_bytes(n)) return cudaErrorInvalidValue;
  if (n == 0) return cudaSuccess;
  // LFSR_SORT_LSD=1 forces the LSD route (A/B, tests)
  const char* lsd_only = getenv("LFSR_SORT_LSD");
  const uint32_t W = lsd_only && lsd_only[0] == '1' ? 0u : msd_window_bits(n);
  const uint64_t groups = W ? (1ull << W) : 1ull;
  uint8_t* p = static_cast<uint8_t*>(scratch);
  SortCtl* ctl = reinterpret_cast<SortCtl*>(p);
  p += align256(sizeof(SortCtl));
  SortCtl* mctl = reinterpret_cast<SortCtl*>(p);
  p += align256(sizeof(SortCtl));
  MsdCtl* msd = reinterpret_cast<MsdCtl*>(p);
  p += align256(sizeof(MsdCtl));
  uint64_t* kbuf = reinterpret_cast<uint64_t*>(p);
  p += align256(n * 8);
  uint32_t* r0 = reinterpret_cast<uint32_t*>(p);
  p += align256(n * 4);
  uint32_t* r1 = reinterpret_cast<uint32_t*>(p);
  p += align256(n * 4);
  const uint64_t tiles = (n + kTileKeys - 1) / kTileKeys;
  uint64_t* status = reinterpret_cast<uint64_t*>(p);
  p += align256(tiles * kBins * 8);
  ulonglong2* aos = reinterpret_cast<ulonglong2*>(p);
  p += align256(n * 32);
  uint32_t* gstart = reinterpret_cast<uint32_t*>(p);
  p += align256(groups * 4);
  uint32_t* gend = reinterpret_cast<uint32_t*>(p);
  cudaError_t e;
  if (const char* g = getenv("LFSR_SORT_L2FETCH")) {  // A/B: L2 fetch granularity hint
    if ((e = cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, static_cast<size_t>(atoi(g)))) != cudaSuccess) return e;
  }
  if ((e = cudaMemsetAsync(ctl, 0, sizeof(SortCtl), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(mctl, 0, sizeof(SortCtl), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(msd, 0, sizeof(MsdCtl), st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(status, 0, tiles * kBins * 8, st)) != cudaSuccess) return e;
  if ((e = cudaMemsetAsync(gend, 0, groups * 4, st)) != cudaSuccess) return e;
  PassBufs bufs{{cols_out[0], kbuf}, {r0, r1}};
  Cols cols{};
  for (int c = 0; c < kCols; ++c) {
    cols.in[c] = c < ncols ? cols_in[c] : nullptr;
    cols.out[c] = c < ncols ? cols_out[c] : nullptr;
  }
  int dev = 0, sms = 1;
  if ((e = cudaGetDevice(&dev)) != cudaSuccess) return e;
  if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
  const uint64_t hb = std::min<uint64_t>((n + kSortThreads - 1) / kSortThreads, static_cast<uint64_t>(sms) * 8);
  sort_init_kernel<<<1, 32, 0, st>>>(ctl, mctl);
  sort_hist_kernel<<<static_cast<unsigned>(hb), kSortThreads, 0, st>>>(cols_in[0], n, ctl, cols, aos, msd);
  sort_plan_kernel<<<1, kBins, 0, st>>>(n, ctl);
  if ((e = cudaFuncSetAttribute(sort_pass_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kPassSmem))) != cudaSuccess ||
      (e = cudaFuncSetAttribute(sort_pass_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(kPassSmem))) != cudaSuccess)
    return e;
  *launches += 3;
  if (W) {  // the MSD route (its kernels return at once unless the plan picks it)
    msd_plan_kernel<<<1, 1, 0, st>>>(n, W, ctl, mctl, msd);
    msd_hist_kernel<<<static_cast<unsigned>(hb), kSortThreads, 0, st>>>(cols_in[0], n, mctl, msd);
    sort_plan_kernel<<<1, kBins, 0, st>>>(n, mctl);
    const int nd = static_cast<int>((W + 7) / 8);  // the window's digits (msd_plan_kernel)
    for (int sidx = 0; sidx < nd; ++sidx)
      sort_pass_kernel<false><<<static_cast<unsigned>(tiles), kSortThreads, kPassSmem, st>>>(bufs, cols, n, sidx, mctl,
                                                                                             status, aos, nullptr);
    const uint64_t gb = std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sms) * 16);
    msd_bounds_kernel<<<static_cast<unsigned>(gb), 256, 0, st>>>(cols_out[0], n, W, msd, gstart, gend);
    if ((e = cudaFuncSetAttribute(msd_local_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(kLocalSmem))) != cudaSuccess)
      return e;
    msd_local_kernel<<<static_cast<unsigned>(groups), kLocalThreads, kLocalSmem, st>>>(bufs, cols, msd, gstart, gend,
                                                                                      aos);
    *launches += 5 + nd;
  }
  // trivial bytes return at once (decided on the device); behind the MSD route the passes
  // run only on its fallback, so they are launched persistent: a few resident blocks that
  // return at once rather than a block per tile
  const uint64_t pgrid = std::min<uint64_t>(tiles, static_cast<uint64_t>(sms) * LC_SORT_MINBLOCKS);
  for (int b = 0; b < kBytes; ++b) {
    if (W)
      sort_pass_kernel<true><<<static_cast<unsigned>(pgrid), kSortThreads, kPassSmem, st>>>(bufs, cols, n, b, ctl,
                                                                                            status, aos, msd);
    else
      sort_pass_kernel<false><<<static_cast<unsigned>(tiles), kSortThreads, kPassSmem, st>>>(bufs, cols, n, b, ctl,
                                                                                             status, aos, msd);
  }
  const uint64_t gb = std::min<uint64_t>((n + 255) / 256, static_cast<uint64_t>(sms) * 8);
  sort_copy_kernel<<<static_cast<unsigned>(gb), 256, 0, st>>>(n, ctl, cols, msd);
  *launches += kBytes + 1;
  return cudaGetLastError();
}

}  // namespace lc
