// C ABI (include/lfsr_b200.h): contexts, scratch management, spec dispatch, host-buffer
// wrappers.  The kernels live in walk.cu / kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "jit.h"
#include "lfsr_internal.h"

namespace {

thread_local std::string g_err;
thread_local uint64_t g_launches = 0;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define LC_CUDA(expr)                                                                      \
  do {                                                                                     \
    cudaError_t e_ = (expr);                                                               \
    if (e_ != cudaSuccess) return fail(LC_ERR_CUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
  } while (0)

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

lc::SpecId identify(const lc_spec* s) {
  if (!s) return lc::SpecId::UNSUPPORTED;
  struct Known {
    int l[3];
    uint64_t t[3];
    int c[3];
    lc::SpecId id;
  };
  static const Known known[] = {
      {{19, 22, 23},
       {(1ull << 13) | (1ull << 16) | (1ull << 17) | (1ull << 18), (1ull << 20) | (1ull << 21),
        (1ull << 7) | (1ull << 20) | (1ull << 21) | (1ull << 22)},
       {8, 10, 10},
       lc::SpecId::A51},
      {{5, 6, 7}, {(1ull << 1) | (1ull << 4), (1ull << 4) | (1ull << 5), (1ull << 5) | (1ull << 6)}, {2, 2, 3}, lc::SpecId::MINI567},
      {{7, 8, 9},
       {(1ull << 5) | (1ull << 6), (1ull << 3) | (1ull << 4) | (1ull << 5) | (1ull << 7), (1ull << 3) | (1ull << 8)},
       {3, 3, 4},
       lc::SpecId::MINI789},
  };
  for (const Known& k : known) {
    bool eq = true;
    for (int i = 0; i < 3; ++i)
      eq = eq && s->lengths[i] == k.l[i] && s->tap_masks[i] == k.t[i] && s->clock_taps[i] == k.c[i];
    if (eq) return k.id;
  }
  return lc::SpecId::UNSUPPORTED;
}

uint32_t default_fixed(lc::SpecId id) {
  switch (id) {
    case lc::SpecId::A51: return 0x2AAA00u;
    case lc::SpecId::MINI567: return 0x22u;
    case lc::SpecId::MINI789: return 0xaau;
    default: return 0u;
  }
}

int l3_of(lc::SpecId id) {
  if (id == lc::SpecId::CUSTOM) return lc::current_custom() ? lc::current_custom()->lengths[2] : 0;
  return id == lc::SpecId::A51 ? 23 : (id == lc::SpecId::MINI567 ? 7 : 9);
}

uint32_t r3_taps(lc::SpecId id) {
  switch (id) {
    case lc::SpecId::A51: return (1u << 7) | (1u << 20) | (1u << 21) | (1u << 22);
    case lc::SpecId::MINI567: return (1u << 5) | (1u << 6);
    case lc::SpecId::MINI789: return (1u << 3) | (1u << 8);
    case lc::SpecId::CUSTOM: return lc::current_custom() ? static_cast<uint32_t>(lc::current_custom()->taps[2]) : 0u;
    default: return 0u;
  }
}

// A built-in spec, or a valid custom one: its kernels are compiled for it at first use
// (csrc/jit.cu) and become the calling thread's current custom spec.
int check_spec(const lc_spec* spec, lc::SpecId* id) {
  *id = identify(spec);
  if (*id != lc::SpecId::UNSUPPORTED) return LC_OK;
  if (!spec) return fail(LC_ERR_ARG, "null spec");
  std::string err;
  const lc::CustomKernels* k = lc::custom_kernels_for(spec, &err);
  if (!k) return fail(LC_ERR_UNSUPPORTED, "custom cipher spec: %s", err.c_str());
  lc::set_current_custom(k);
  *id = lc::SpecId::CUSTOM;
  return LC_OK;
}

int check_fixed(lc::SpecId id, uint64_t fixed_r3) {
  const int l3 = l3_of(id);
  if (fixed_r3 == 0 || fixed_r3 >= (1ull << l3))
    return fail(LC_ERR_ARG, "fixed R3 value must be a nonzero %d-bit value", l3);
  if (id == lc::SpecId::CUSTOM) {
    // the kernels take "R3 clocked" for "R3 leaves F"; that fails only if F is a fixed
    // point of R3's step, and then no state is a special node at all
    const uint32_t m = l3 >= 32 ? ~0u : (1u << l3) - 1u, f = static_cast<uint32_t>(fixed_r3);
    const uint32_t next = ((f << 1) & m) | (static_cast<uint32_t>(__builtin_popcount(f & r3_taps(id))) & 1u);
    if (next == f) return fail(LC_ERR_ARG, "fixed R3 value is a fixed point of R3's step: there are no special nodes");
  }
  return LC_OK;
}

}  // namespace

struct lc_ctx {
  int device = 0;
  int sms = 0;
  cudaStream_t stream = nullptr;
  DevBuf meta, queue, stats, a, b, c, d, scratch, smmap, pq, pool_a, pool_b, need3, spill;
  int mapped_sms = -1;  // SMs found by the %smid probe (-1: not probed yet)
  int need3_id = -1;    // spec / fixed R3 the need3 table was built for
  uint64_t need3_f = 0;
  const void* need3_custom = nullptr;  // (custom spec)
  bool need3_valid = false;            // a table exists (custom specs with l3 > 24 have none)
  uint64_t window = 0;                 // R3's period through F (WalkParams::window)
  cudaEvent_t done = nullptr;  // recorded after the last call's work (see Ordered)
};

namespace {

// Every call that uses the context's scratch buffers (walk pools, queues, lane metadata,
// staging) first makes its stream wait for the previous call's work, on whatever stream
// that was, and records its own completion: asynchronous `_device` calls on different
// streams can then share one context without one call's rounds overwriting another's
// buffers.
struct Ordered {
  lc_ctx* c;
  cudaStream_t st;
  Ordered(lc_ctx* c_, cudaStream_t st_) : c(c_), st(st_) { cudaStreamWaitEvent(st, c->done, 0); }
  ~Ordered() { cudaEventRecord(c->done, st); }
};

// Dense index for every %smid of the device, so the walk can keep one queue per warp
// scheduler (4 per SM).  Probed once per context.
int ensure_smsp_map(lc_ctx* ctx) {
  if (ctx->mapped_sms >= 0) return LC_OK;
  LC_CUDA(ctx->smmap.ensure(1024 * sizeof(unsigned int) + 1024 * sizeof(uint16_t)));
  unsigned int* flags = ctx->smmap.as<unsigned int>();
  LC_CUDA(cudaMemsetAsync(flags, 0, 1024 * sizeof(unsigned int), ctx->stream));
  LC_CUDA(lc::probe_smids(ctx->sms, flags, ctx->stream));
  g_launches += 1;
  unsigned int h[1024];
  LC_CUDA(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  uint16_t map[1024];
  int k = 0;
  for (int i = 0; i < 1024; ++i) map[i] = h[i] ? static_cast<uint16_t>(k++) : 0;
  uint16_t* dmap = reinterpret_cast<uint16_t*>(flags + 1024);
  LC_CUDA(cudaMemcpyAsync(dmap, map, sizeof(map), cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  ctx->mapped_sms = k;
  return LC_OK;
}

// need3[v] = R3 clocks from R3 value v to the fixed value F (the walk's arming bound):
// one pass over R3's sequence starting at F, built once per (spec, F).  Its length is R3's
// period through F (2^l3 - 1 for maximal-period registers), the walk's check-free
// window.  Values off F's cycle (custom specs with non-maximal R3) never reach F:
// UINT32_MAX, so those lanes run to the cap audit like the reference's (StrideError).
int ensure_need3(lc_ctx* ctx, lc::SpecId id, uint64_t F) {
  const void* custom = id == lc::SpecId::CUSTOM ? static_cast<const void*>(lc::current_custom()) : nullptr;
  if (ctx->need3_id == static_cast<int>(id) && ctx->need3_f == F && ctx->need3_custom == custom) return LC_OK;
  const int l3 = l3_of(id);
  const uint32_t taps = r3_taps(id);
  if (l3 < 2 || !taps) return fail(LC_ERR_UNSUPPORTED, "no R3 table for this spec");
  const uint32_t mask = l3 >= 32 ? ~0u : (1u << l3) - 1u;
  auto step = [&](uint32_t x) { return ((x << 1) & mask) | (static_cast<uint32_t>(__builtin_popcount(x & taps)) & 1u); };
  const bool table = l3 <= 24;
  std::vector<uint32_t> need(table ? static_cast<size_t>(mask) + 1u : 0u, ~0u);
  uint64_t period = 0;
  uint32_t x = static_cast<uint32_t>(F);
  if (l3 <= 28) {
    do {
      x = step(x);
      ++period;
    } while (x != F);
  } else {
    period = 1;  // too long to trace here: check every clock (correct, slower)
  }
  if (table) {
    x = static_cast<uint32_t>(F);
    for (uint64_t k = 0; k < period; ++k) {
      need[x] = static_cast<uint32_t>((period - k) % period);
      x = step(x);
    }
    LC_CUDA(ctx->need3.ensure(need.size() * 4));
    LC_CUDA(cudaMemcpy(ctx->need3.p, need.data(), need.size() * 4, cudaMemcpyHostToDevice));
  }
  ctx->need3_id = static_cast<int>(id);
  ctx->need3_f = F;
  ctx->need3_custom = custom;
  ctx->need3_valid = table;
  ctx->window = period;
  return LC_OK;
}

}  // namespace

extern "C" {

int lc_abi_version(void) { return LC_ABI_VERSION; }

const char* lc_last_error(void) { return g_err.c_str(); }

uint64_t lc_launch_count(void) { return g_launches; }
void lc_launch_count_reset(void) { g_launches = 0; }

int lc_spec_compile_check(const lc_spec* spec) {
  if (!spec) return fail(LC_ERR_ARG, "null spec");
  std::string err;
  if (lc::custom_compile_check(spec, &err)) return fail(LC_ERR_UNSUPPORTED, "custom cipher spec: %s", err.c_str());
  return LC_OK;
}

int lc_device_count(int* count) {
  LC_CUDA(cudaGetDeviceCount(count));
  return LC_OK;
}

int lc_ctx_create(int device, lc_ctx** out) {
  if (!out) return fail(LC_ERR_ARG, "null output");
  int n = 0;
  LC_CUDA(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(LC_ERR_ARG, "device %d out of range (%d devices)", device, n);
  LC_CUDA(cudaSetDevice(device));
  lc_ctx* c = new lc_ctx();
  c->device = device;
  cudaError_t e = cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventRecord(c->done, c->stream);
  if (e != cudaSuccess) {
    delete c;
    return fail(LC_ERR_CUDA, "context: %s", cudaGetErrorString(e));
  }
  *out = c;
  return LC_OK;
}

int lc_ctx_destroy(lc_ctx* ctx) {
  if (!ctx) return LC_OK;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();  // work queued on callers' streams may still use the buffers
  for (DevBuf* b : {&ctx->meta, &ctx->queue, &ctx->stats, &ctx->a, &ctx->b, &ctx->c, &ctx->d, &ctx->scratch, &ctx->smmap, &ctx->pq, &ctx->pool_a, &ctx->pool_b, &ctx->need3, &ctx->spill})
    b->release();
  cudaStreamDestroy(ctx->stream);
  cudaEventDestroy(ctx->done);
  delete ctx;
  return LC_OK;
}

int lc_ctx_sm_count(lc_ctx* ctx, int* sms) {
  if (!ctx || !sms) return fail(LC_ERR_ARG, "null argument");
  *sms = ctx->sms;
  return LC_OK;
}

int lc_ctx_synchronize(lc_ctx* ctx) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  LC_CUDA(cudaSetDevice(ctx->device));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

int lc_lop3_peak(lc_ctx* ctx, double* lop3_per_s, double* sm_mhz) {
  if (!ctx || !lop3_per_s || !sm_mhz) return fail(LC_ERR_ARG, "null argument");
  LC_CUDA(cudaSetDevice(ctx->device));
  LC_CUDA(lc::measure_lop3_peak(ctx->sms, lop3_per_s, sm_mhz));
  return LC_OK;
}

int lc_host_alloc(uint64_t bytes, void** out) {
  if (!out) return fail(LC_ERR_ARG, "null output");
  LC_CUDA(cudaMallocHost(out, bytes ? bytes : 1));
  return LC_OK;
}

int lc_host_free(void* p) {
  if (p) LC_CUDA(cudaFreeHost(p));
  return LC_OK;
}

// ------------------------------------------------------------------------- walks

namespace {

struct WalkArgs {
  lc::SpecId id;
  uint64_t fixed_r3, stride, max_clocks, hist_lo;
  uint32_t legs, refill, hist_shift, hist_bins;
};

// One walk launch.  resume != null: the items are parked lanes (lane mode, no stats
// reset).  pool != null: drained warps park below park_below live lanes.
int walk_launch(lc_ctx* ctx, const WalkArgs& a, const uint64_t* d_starts, const lc::ResumeRec* resume, uint64_t n,
                uint64_t* d_dest, uint64_t* d_dist, uint64_t* d_stats, lc::ResumeRec* pool,
                unsigned long long* pool_count, uint32_t park_below, cudaStream_t st,
                const unsigned long long* n_dev = nullptr, uint64_t park_min = 0) {
  int rc = ensure_smsp_map(ctx);
  if (rc) return rc;
  if ((rc = ensure_need3(ctx, a.id, a.fixed_r3))) return rc;
  const bool static_f = a.fixed_r3 == default_fixed(a.id);
  const int per_sm = lc::walk_blocks_per_sm(a.id, static_f);
  const uint64_t lanes_per_block = lc::kWalkThreads * 32ull;
  const uint64_t max_blocks = static_cast<uint64_t>(per_sm) * ctx->sms;
  // n_dev: n is only an upper bound (the count is on the device), so cover the whole GPU
  const uint64_t want = n_dev ? max_blocks : (n + lanes_per_block - 1) / lanes_per_block;
  const int blocks = static_cast<int>(std::max<uint64_t>(1, std::min(max_blocks, want)));
  // auto (refill == 0): single-hop walks whose starts are all special-node-like run with
  // whole-warp refill (decided on the device by the mode probe); everything else per lane
  const bool auto_mode = resume == nullptr && a.refill == 0 && a.legs == 1;
  const uint32_t refill_min = (resume || a.refill == 0) ? 1u : a.refill;
  // one queue per warp scheduler when the persistent grid covers every SM
  // (not for a resume round sized on the device: most of its blocks exit at once)
  const uint32_t nq = (ctx->mapped_sms == ctx->sms && static_cast<uint64_t>(blocks) == max_blocks && !n_dev)
                          ? 4u * static_cast<uint32_t>(ctx->sms) : 1u;

  LC_CUDA(ctx->meta.ensure(static_cast<size_t>(blocks) * lanes_per_block * sizeof(lc::LaneMeta)));
  LC_CUDA(ctx->queue.ensure((static_cast<size_t>(nq) * 16 + 16) * sizeof(unsigned long long)));
  unsigned long long* queues = ctx->queue.as<unsigned long long>();
  unsigned int* exhausted = reinterpret_cast<unsigned int*>(queues + static_cast<size_t>(nq) * 16);

  // stats header (counters zero, min = ~0, error index = ~0, histogram config), queues
  LC_CUDA(lc::launch_init_stats(resume ? nullptr : d_stats, a.hist_lo, a.hist_shift, a.hist_bins, queues, nq,
                                exhausted, st));
  g_launches += 1;
  if (n == 0) return LC_OK;
  if ((!d_starts && !resume) || !d_dest || !d_dist) return fail(LC_ERR_ARG, "null buffer");
  uint32_t* mode_word = reinterpret_cast<uint32_t*>(exhausted + 1);
  if (auto_mode) {
    LC_CUDA(lc::launch_mode_probe(a.id, d_starts, n, static_cast<uint32_t>(a.fixed_r3), mode_word, st));
    g_launches += 1;
  }

  lc::WalkParams p{};
  p.starts = d_starts;
  p.n = n;
  p.dst = d_dest;
  p.dist = d_dist;
  p.stride = a.stride;
  p.cap1 = a.max_clocks == ~0ull ? ~0ull : a.max_clocks + 1;
  p.hist_lo = a.hist_lo;
  p.hist_shift = a.hist_shift;
  p.hist_bins = a.hist_bins;
  p.legs = a.legs;
  p.fixed_r3 = static_cast<uint32_t>(a.fixed_r3);
  p.refill_min = refill_min;
  p.chunk = refill_min >= 1024u ? 1024u : 1u;
  p.nq = nq;
  p.queues = queues;
  p.smsp_map = reinterpret_cast<const uint16_t*>(ctx->smmap.as<unsigned int>() + 1024);
  p.exhausted = exhausted;
  p.stats = reinterpret_cast<unsigned long long*>(d_stats);
  p.meta = ctx->meta.as<lc::LaneMeta>();
  p.mode_word = auto_mode ? mode_word : nullptr;
  p.resume = resume;
  p.pool = pool;
  p.pool_count = pool_count;
  // parked-lane capacity of the destination pool (the kernel never writes past it)
  p.pool_cap = !pool ? 0
               : (static_cast<void*>(pool) == ctx->pool_a.p ? ctx->pool_a.bytes : ctx->pool_b.bytes) /
                     sizeof(lc::ResumeRec);
  p.park_below = pool ? park_below : 0u;
  p.n_dev = n_dev;
  p.park_min = park_min;
  p.need3 = ctx->need3_valid ? ctx->need3.as<uint32_t>() : nullptr;
  p.window = ctx->window;
  p.run_if_mode = ~0u;
  // Re-arming pays for lanes that would otherwise be checked for long stretches: lane
  // mode (independent lanes), or any walk whose stride is below R3's period.  Whole-warp
  // walks from special nodes at a stride past the period (the paper's setting) run the
  // plain variant; in auto mode both variants are launched and the device mode word
  // picks the one that runs.
  const bool short_stride = a.stride < (1ull << l3_of(a.id)) - 1;
  if (short_stride || a.refill == 1u || resume) {
    LC_CUDA(lc::launch_walk(a.id, static_f, true, p, blocks, st));
    g_launches += 1;
  } else if (auto_mode) {
    p.run_if_mode = 1u;
    LC_CUDA(lc::launch_walk(a.id, static_f, false, p, blocks, st));
    p.run_if_mode = 0u;
    LC_CUDA(lc::launch_walk(a.id, static_f, true, p, blocks, st));
    g_launches += 2;
  } else {
    LC_CUDA(lc::launch_walk(a.id, static_f, a.refill != 1024u, p, blocks, st));  // lane mode re-arms
    g_launches += 1;
  }
  return LC_OK;
}

int check_walk_args(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, uint64_t stride, uint32_t legs,
                    uint32_t hist_shift, uint32_t refill, WalkArgs* a) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  int rc = check_spec(spec, &a->id);
  if (rc) return rc;
  if ((rc = check_fixed(a->id, fixed_r3))) return rc;
  if (stride < 1) return fail(LC_ERR_ARG, "stride must be >= 1");
  if (legs < 1) return fail(LC_ERR_ARG, "legs must be >= 1");
  if (hist_shift > 63) return fail(LC_ERR_ARG, "hist_shift must be < 64");
  if (refill > 1024) return fail(LC_ERR_ARG, "refill must be in [0, 1024]");
  return LC_OK;
}

}  // namespace

int lc_walk_device(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, const uint64_t* d_starts,
                   uint64_t n, uint64_t stride, uint64_t max_clocks, uint32_t legs, uint32_t refill,
                   uint64_t* d_dest, uint64_t* d_dist, uint64_t hist_lo, uint32_t hist_shift,
                   uint32_t hist_bins, uint64_t* d_stats, void* stream) {
  WalkArgs a{};
  int rc = check_walk_args(ctx, spec, fixed_r3, stride, legs, hist_shift, refill, &a);
  if (rc) return rc;
  if (!d_stats) return fail(LC_ERR_ARG, "stats buffer required");
  a.fixed_r3 = fixed_r3;
  a.stride = stride;
  a.max_clocks = max_clocks;
  a.hist_lo = hist_lo;
  a.legs = legs;
  a.refill = refill;
  a.hist_shift = hist_shift;
  a.hist_bins = hist_bins;
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  // Lane parking without a host sync (the call stays asynchronous): a fixed number of
  // resume rounds is queued, each reading its item count (the previous round's parked
  // lanes) on the device; a round with nothing parked exits at once, and the last round
  // never parks, so every walk completes.  Whole-warp launches never park (kernel-side).
  const uint64_t park_threshold = 4ull * static_cast<uint64_t>(ctx->sms) * 1024ull;
  if (n <= park_threshold || getenv("LFSR_WALK_NO_PARK") != nullptr)
    return walk_launch(ctx, a, d_starts, nullptr, n, d_dest, d_dist, d_stats, nullptr, nullptr, 0, st);
  constexpr int kRounds = 4;
  const uint64_t cap = std::min<uint64_t>(n, 8ull * park_threshold);
  LC_CUDA(ctx->pool_a.ensure(cap * sizeof(lc::ResumeRec)));
  LC_CUDA(ctx->pool_b.ensure(cap * sizeof(lc::ResumeRec)));
  LC_CUDA(ctx->pq.ensure(16 + kRounds * sizeof(unsigned long long)));
  lc::ResumeRec* pools[2] = {ctx->pool_a.as<lc::ResumeRec>(), ctx->pool_b.as<lc::ResumeRec>()};
  unsigned long long* counts = ctx->pq.as<unsigned long long>() + 2;  // [1] is lc_walk's
  LC_CUDA(cudaMemsetAsync(counts, 0, kRounds * sizeof(unsigned long long), st));
  for (int round = 0; round < kRounds; ++round) {
    const bool last = round == kRounds - 1;
    const int rc2 = walk_launch(ctx, a, d_starts, round ? pools[(round - 1) & 1] : nullptr, round ? cap : n, d_dest,
                                d_dist, d_stats, last ? nullptr : pools[round & 1], counts + round, 512u, st,
                                round ? counts + round - 1 : nullptr, park_threshold);
    if (rc2) return rc2;
  }
  return LC_OK;
}

// Host-buffer walk.  Runs in rounds: warps that drain below half occupancy park their
// live lanes, and the next round resumes them packed densely, so the tail of wide-spread
// walks does not run on mostly idle warps.  Parking is only enabled while a round has
// more lanes than the GPU has warp schedulers x 1024 (below that, packing gains nothing).
int lc_walk(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, const uint64_t* starts, uint64_t n,
            uint64_t stride, uint64_t max_clocks, uint32_t legs, uint32_t refill, uint64_t* dest,
            uint64_t* dist, uint64_t hist_lo, uint32_t hist_shift, uint32_t hist_bins,
            uint64_t* stats) {
  WalkArgs a{};
  int rc = check_walk_args(ctx, spec, fixed_r3, stride, legs, hist_shift, refill, &a);
  if (rc) return rc;
  if (!stats) return fail(LC_ERR_ARG, "stats buffer required");
  a.fixed_r3 = fixed_r3;
  a.stride = stride;
  a.max_clocks = max_clocks;
  a.hist_lo = hist_lo;
  a.legs = legs;
  a.refill = refill;
  a.hist_shift = hist_shift;
  a.hist_bins = hist_bins;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  const size_t sb = (LC_ST_HEADER + hist_bins + 2ull) * sizeof(uint64_t);
  const size_t nb = static_cast<size_t>(n) * sizeof(uint64_t);
  const size_t ob = nb * std::max<uint32_t>(legs, 1);
  LC_CUDA(ctx->a.ensure(std::max<size_t>(nb, 8)));
  LC_CUDA(ctx->b.ensure(std::max<size_t>(ob, 8)));
  LC_CUDA(ctx->c.ensure(std::max<size_t>(ob, 8)));
  LC_CUDA(ctx->stats.ensure(sb));
  if (n) LC_CUDA(cudaMemcpyAsync(ctx->a.p, starts, nb, cudaMemcpyHostToDevice, ctx->stream));
  const uint64_t park_threshold = 4ull * static_cast<uint64_t>(ctx->sms) * 1024ull;  // lanes in a full wave of schedulers
  const bool park = n > park_threshold;
  lc::ResumeRec* pools[2] = {nullptr, nullptr};
  unsigned long long* pcount = nullptr;
  if (park) {
    const size_t cap = std::min<uint64_t>(n, 8ull * park_threshold) * sizeof(lc::ResumeRec);
    LC_CUDA(ctx->pool_a.ensure(cap));
    LC_CUDA(ctx->pool_b.ensure(cap));
    LC_CUDA(ctx->pq.ensure(16));
    pools[0] = ctx->pool_a.as<lc::ResumeRec>();
    pools[1] = ctx->pool_b.as<lc::ResumeRec>();
    pcount = ctx->pq.as<unsigned long long>() + 1;
  }
  const lc::ResumeRec* resume = nullptr;
  uint64_t round_n = n;
  for (int round = 0;; ++round) {
    lc::ResumeRec* out = park ? pools[round & 1] : nullptr;
    const bool park_now = park && round_n > park_threshold;
    if (park) LC_CUDA(cudaMemsetAsync(pcount, 0, 8, ctx->stream));
    rc = walk_launch(ctx, a, ctx->a.as<uint64_t>(), resume, round_n, ctx->b.as<uint64_t>(), ctx->c.as<uint64_t>(),
                     ctx->stats.as<uint64_t>(), park_now ? out : nullptr, pcount, 512u, ctx->stream);
    if (rc) return rc;
    if (!park_now) break;
    unsigned long long parked = 0;
    LC_CUDA(cudaMemcpyAsync(&parked, pcount, 8, cudaMemcpyDeviceToHost, ctx->stream));
    LC_CUDA(cudaStreamSynchronize(ctx->stream));
    if (parked == 0) break;
    resume = out;
    round_n = parked;
  }
  LC_CUDA(cudaMemcpyAsync(stats, ctx->stats.p, sb, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (stats[LC_ST_ERROR]) {
    const int code = -static_cast<int>(stats[LC_ST_ERROR]);
    if (code == LC_ERR_CAP)
      return fail(LC_ERR_CAP, "no candidate within %llu clocks; check the fixed R3 / stride configuration (start %llu)",
                  static_cast<unsigned long long>(max_clocks), static_cast<unsigned long long>(stats[LC_ST_ERROR_INDEX]));
    return fail(code, "start %llu has a zero register (invalid state)",
                static_cast<unsigned long long>(stats[LC_ST_ERROR_INDEX]));
  }
  if (n) {
    LC_CUDA(cudaMemcpyAsync(dest, ctx->b.p, ob, cudaMemcpyDeviceToHost, ctx->stream));
    LC_CUDA(cudaMemcpyAsync(dist, ctx->c.p, ob, cudaMemcpyDeviceToHost, ctx->stream));
  }
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

int lc_clock(lc_ctx* ctx, const lc_spec* spec, const uint64_t* xs, uint64_t n, uint64_t t, uint64_t* out) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  const size_t nb = static_cast<size_t>(n) * 8;
  LC_CUDA(ctx->a.ensure(nb));
  LC_CUDA(ctx->b.ensure(nb));
  LC_CUDA(cudaMemcpyAsync(ctx->a.p, xs, nb, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(lc::launch_clock(id, ctx->a.as<uint64_t>(), n, t, ctx->b.as<uint64_t>(), ctx->stream));
  g_launches += 1;
  LC_CUDA(cudaMemcpyAsync(out, ctx->b.p, nb, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

// ------------------------------------------------------------ predicate / predecessors

int lc_is_candidate(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, const uint64_t* xs, uint64_t n,
                    uint8_t* out) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->a.ensure(n * 8));
  LC_CUDA(ctx->b.ensure(n));
  LC_CUDA(cudaMemcpyAsync(ctx->a.p, xs, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(lc::launch_is_candidate(id, ctx->a.as<uint64_t>(), n, static_cast<uint32_t>(fixed_r3),
                                  ctx->b.as<uint8_t>(), ctx->stream));
  g_launches += 1;
  LC_CUDA(cudaMemcpyAsync(out, ctx->b.p, n, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

int lc_predecessors(lc_ctx* ctx, const lc_spec* spec, const uint64_t* xs, uint64_t n, uint64_t* out,
                    uint8_t* count) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->a.ensure(n * 8));
  LC_CUDA(ctx->b.ensure(n * 32));
  LC_CUDA(ctx->c.ensure(n));
  LC_CUDA(cudaMemcpyAsync(ctx->a.p, xs, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(lc::launch_predecessors(id, ctx->a.as<uint64_t>(), n, ctx->b.as<uint64_t>(), ctx->c.as<uint8_t>(),
                                  ctx->stream));
  g_launches += 1;
  LC_CUDA(cudaMemcpyAsync(out, ctx->b.p, n * 32, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaMemcpyAsync(count, ctx->c.p, n, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

// ------------------------------------------------------------------- enumeration

int lc_enumerate_device(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, uint64_t r2_lo, uint64_t r2_hi,
                        uint64_t* d_out, uint64_t cap, uint64_t* d_count, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  const int l2 = spec->lengths[1];
  if (r2_lo < 1 || r2_hi > (1ull << l2) || r2_lo > r2_hi)
    return fail(LC_ERR_ARG, "R2 rows must satisfy 1 <= r2_lo <= r2_hi <= 2^%d", l2);
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  int launches = 0;
  LC_CUDA(lc::launch_enumerate(id, static_cast<uint32_t>(fixed_r3), r2_lo, r2_hi, d_out, cap, d_count, st,
                               &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_enumerate(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, uint64_t r2_lo, uint64_t r2_hi,
                 uint64_t* out, uint64_t cap, uint64_t* count) {
  if (!ctx || !count) return fail(LC_ERR_ARG, "null argument");
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->a.ensure(std::max<uint64_t>(cap, 1) * 8));
  LC_CUDA(ctx->d.ensure(8));
  int rc = lc_enumerate_device(ctx, spec, fixed_r3, r2_lo, r2_hi, ctx->a.as<uint64_t>(), cap,
                               ctx->d.as<uint64_t>(), ctx->stream);
  if (rc) return rc;
  LC_CUDA(cudaMemcpyAsync(count, ctx->d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  const uint64_t got = std::min(*count, cap);
  if (got) {
    LC_CUDA(cudaMemcpyAsync(out, ctx->a.p, got * 8, cudaMemcpyDeviceToHost, ctx->stream));
    LC_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  if (*count > cap) return fail(LC_ERR_OVERFLOW, "%llu candidates exceed capacity %llu",
                                static_cast<unsigned long long>(*count), static_cast<unsigned long long>(cap));
  return LC_OK;
}

// -------------------------------------------------------------- seeded start set (K0)

static double acceptance_estimate(lc::SpecId id) {
  (void)id;
  return 0.40;  // A5/1 0.438, minis ~0.44-0.5; under-estimating only costs extra trials
}

int lc_random_candidates_device(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, uint64_t seed, uint64_t n,
                                uint64_t* d_out, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  if (id == lc::SpecId::CUSTOM)
    return fail(LC_ERR_UNSUPPORTED, "the K0 generator is built for the built-in ciphers only "
                                    "(lc_reference_candidates serves any spec)");
  uint64_t trials = static_cast<uint64_t>(static_cast<double>(n) / acceptance_estimate(id)) + 65536;
  for (int attempt = 0; attempt < 8; ++attempt) {
    const uint64_t words = lc::random_scratch_words(trials);
    LC_CUDA(ctx->scratch.ensure(words * 8));
    LC_CUDA(ctx->d.ensure(8));
    int launches = 0;
    LC_CUDA(lc::launch_random_candidates(id, static_cast<uint32_t>(fixed_r3), seed, trials, d_out, n,
                                         ctx->d.as<uint64_t>(), ctx->scratch.as<uint64_t>(), words, st,
                                         &launches));
    g_launches += launches;
    uint64_t got = 0;
    LC_CUDA(cudaMemcpyAsync(&got, ctx->d.p, 8, cudaMemcpyDeviceToHost, st));
    LC_CUDA(cudaStreamSynchronize(st));
    if (got >= n) return LC_OK;
    trials *= 2;
  }
  return fail(LC_ERR_ARG, "too few special nodes in the trial stream (wrong fixed R3?)");
}

int lc_random_candidates(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, uint64_t seed, uint64_t n,
                         uint64_t* out, uint64_t* trials_used) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (n == 0) {
    if (trials_used) *trials_used = 0;
    return LC_OK;
  }
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->b.ensure(n * 8));
  int rc = lc_random_candidates_device(ctx, spec, fixed_r3, seed, n, ctx->b.as<uint64_t>(), ctx->stream);
  if (rc) return rc;
  LC_CUDA(cudaMemcpyAsync(out, ctx->b.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  if (trials_used) *trials_used = 0;  // not tracked (the host restatement recomputes it)
  return LC_OK;
}

// ------------------------------------------------------------------------ prune (K3)

int lc_prune_device(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, int32_t mode, uint64_t limit,
                    const uint64_t* d_cands, uint64_t n, uint8_t* d_removed, uint64_t* d_work, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  if (mode != 0 && mode != 1) return fail(LC_ERR_ARG, "mode must be 0 (dfs) or 1 (bfs)");
  if (limit < 1) return fail(LC_ERR_ARG, "limit must be >= 1");
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->pq.ensure(8));
  LC_CUDA(cudaMemsetAsync(ctx->pq.p, 0, 8, st));
#ifndef LC_PRUNE_SPILL
#define LC_PRUNE_SPILL 512
#endif
  // overflow entries per lane behind the shared-memory ring; LFSR_PRUNE_SPILL overrides it
  // (testing: small values exercise the drop-and-climb fallback)
  uint32_t spill_cap = LC_PRUNE_SPILL;
  if (const char* env = getenv("LFSR_PRUNE_SPILL")) spill_cap = static_cast<uint32_t>(strtoul(env, nullptr, 10));
  int prune3_blocks = 0;
  const char* v1 = getenv("LFSR_PRUNE_V1");  // A/B: the round-1 kernel (64-bit node, no register cache)
  if (v1 && v1[0] == '1' && id != lc::SpecId::CUSTOM) {
    const int ring = lc::prune_ring_for(n);
    const int blocks = lc::prune_blocks_per_sm(id, ring) * ctx->sms;
    if (spill_cap) LC_CUDA(ctx->spill.ensure(lc::prune_spill_bytes(blocks, spill_cap)));
    LC_CUDA(lc::launch_prune(id, static_cast<uint32_t>(fixed_r3), mode, limit, d_cands, n, d_removed, d_work,
                             ctx->pq.as<unsigned long long>(), spill_cap ? ctx->spill.p : nullptr, spill_cap, ring,
                             blocks, st));
  } else if (limit <= lc::prune3_max_limit() && !(v1 && v1[0] == '2') &&
             [&] {  // the uniform-step kernel, if its stacks fit in device memory
               // (LFSR_PRUNE_V1=2 selects the v2 kernel for A/B).  A stack holds at most
               // `limit` entries in either mode (DFS: ancestors at distinct depths <=
               // limit; BFS: the traversal stops past `limit` nodes); the grid is capped
               // by the batch so small batches do not allocate every lane's stack.
               const uint64_t lanes_max = (n + 31) / 32 * 32;
               int blocks = lc::prune3_blocks_per_sm(id) * ctx->sms;
               const uint64_t need_blocks = (lanes_max + lc::prune3_threads() - 1) / lc::prune3_threads();
               if (static_cast<uint64_t>(blocks) > need_blocks) blocks = static_cast<int>(need_blocks);
               if (ctx->spill.ensure(lc::prune3_spill_bytes(blocks, static_cast<uint32_t>(limit))) != cudaSuccess) {
                 cudaGetLastError();  // out of memory: fall through to v2 (bounded spill rings)
                 return false;
               }
               prune3_blocks = blocks;
               return true;
             }()) {
    LC_CUDA(lc::launch_prune3(id, static_cast<uint32_t>(fixed_r3), mode, static_cast<uint32_t>(limit), d_cands, n,
                              d_removed, d_work, ctx->pq.as<unsigned long long>(), ctx->spill.p, prune3_blocks, st));
  } else {
    const int blocks = lc::prune2_blocks_per_sm(id, mode) * ctx->sms;
    if (spill_cap) LC_CUDA(ctx->spill.ensure(lc::prune2_spill_bytes(blocks, spill_cap)));
    LC_CUDA(lc::launch_prune2(id, static_cast<uint32_t>(fixed_r3), mode, limit, d_cands, n, d_removed, d_work,
                              ctx->pq.as<unsigned long long>(), spill_cap ? ctx->spill.p : nullptr, spill_cap, blocks,
                              st));
  }
  g_launches += 1;
  return LC_OK;
}

int lc_prune(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, int32_t mode, uint64_t limit,
             const uint64_t* cands, uint64_t n, uint8_t* removed, uint64_t* work) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->a.ensure(n * 8));
  LC_CUDA(ctx->b.ensure(n));
  LC_CUDA(ctx->c.ensure(n * 8));
  LC_CUDA(cudaMemcpyAsync(ctx->a.p, cands, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  int rc = lc_prune_device(ctx, spec, fixed_r3, mode, limit, ctx->a.as<uint64_t>(), n, ctx->b.as<uint8_t>(),
                           ctx->c.as<uint64_t>(), ctx->stream);
  if (rc) return rc;
  LC_CUDA(cudaMemcpyAsync(removed, ctx->b.p, n, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaMemcpyAsync(work, ctx->c.p, n * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

// ------------------------------------------------------- batched segment probes

int lc_probe_segments(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, const uint64_t* roots, uint64_t k,
                      int64_t depth_cap, int64_t node_cap, uint64_t* depth, uint64_t* nodes, uint8_t* censored,
                      uint64_t* level_counts, uint32_t levels_cap) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  if (k == 0) return LC_OK;
  if (!roots || !depth || !nodes || !censored || (levels_cap && !level_counts)) return fail(LC_ERR_ARG, "null buffer");
  if (k >= (1ull << 32)) return fail(LC_ERR_ARG, "too many roots");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = ctx->stream;
  Ordered ord_(ctx, st);
  const uint32_t kk = static_cast<uint32_t>(k);
  // per-root state, counters, level counts
  struct Ctl {
    unsigned long long cnt[2], live[2], done;
    unsigned int overflow;
  };
  const size_t per_root = 8 + 8 + 8 + 1;  // depth, nodes, lvl, status
  LC_CUDA(ctx->d.ensure(k * per_root + 512 + static_cast<size_t>(levels_cap) * 8 + 64));
  uint8_t* p = ctx->d.as<uint8_t>();
  uint64_t* d_depth = reinterpret_cast<uint64_t*>(p);
  uint64_t* d_nodes = d_depth + k;
  unsigned long long* d_lvl = reinterpret_cast<unsigned long long*>(d_nodes + k);
  Ctl* ctl = reinterpret_cast<Ctl*>(d_lvl + k);
  unsigned long long* d_levels = reinterpret_cast<unsigned long long*>(ctl + 1);
  uint8_t* d_status = reinterpret_cast<uint8_t*>(d_levels + levels_cap);
  // frontier buffers (node, owner) x 2
  unsigned long long cap = std::max<unsigned long long>(4ull * k, 1ull << 20);
  if (const char* env = getenv("LFSR_PROBE_CAP"))  // testing: a tiny frontier forces the grow-and-redo path
    cap = std::max<unsigned long long>(strtoull(env, nullptr, 10), k);  // (the roots always fit)
  struct Pair {  // frees its buffers on every exit path
    DevBuf b[2];
    ~Pair() {
      b[0].release();
      b[1].release();
    }
  } fp;
  DevBuf* fb = fp.b;
  auto alloc = [&](DevBuf& b, unsigned long long c) { return b.ensure(c * 12); };
  auto nodes_of = [&](DevBuf& b) { return b.as<uint64_t>(); };
  auto owners_of = [&](DevBuf& b, unsigned long long c) { return reinterpret_cast<uint32_t*>(b.as<uint64_t>() + c); };
  LC_CUDA(alloc(fb[0], cap));
  LC_CUDA(alloc(fb[1], cap));
  {  // level 0: the roots
    std::vector<uint32_t> own(k);
    for (uint64_t i = 0; i < k; ++i) own[i] = static_cast<uint32_t>(i);
    LC_CUDA(cudaMemcpyAsync(nodes_of(fb[0]), roots, k * 8, cudaMemcpyHostToDevice, st));
    LC_CUDA(cudaMemcpyAsync(owners_of(fb[0], cap), own.data(), k * 4, cudaMemcpyHostToDevice, st));
    Ctl h{};
    h.cnt[0] = k;
    LC_CUDA(cudaMemcpyAsync(ctl, &h, sizeof h, cudaMemcpyHostToDevice, st));
    LC_CUDA(cudaMemsetAsync(d_depth, 0, k * 8, st));
    std::vector<uint64_t> ones(k, 1);
    LC_CUDA(cudaMemcpyAsync(d_nodes, ones.data(), k * 8, cudaMemcpyHostToDevice, st));
    LC_CUDA(cudaMemsetAsync(d_lvl, 0, k * 8, st));
    LC_CUDA(cudaMemsetAsync(d_status, 0, k, st));
    if (levels_cap) LC_CUDA(cudaMemsetAsync(d_levels, 0, static_cast<size_t>(levels_cap) * 8, st));
    LC_CUDA(cudaStreamSynchronize(st));  // (host vectors go out of scope)
  }
  const int blocks = ctx->sms * 8;
  uint64_t level = 0;
  constexpr uint64_t kCheck = 16;  // levels between looks at the live count
  for (;;) {
    if (depth_cap >= 0 && level >= static_cast<uint64_t>(depth_cap)) {  // pipeline.py:280-281
      LC_CUDA(lc::launch_probe_censor(kk, d_status, st));
      g_launches += 1;
      break;
    }
    const int a = static_cast<int>(level & 1), b = a ^ 1;
    LC_CUDA(lc::launch_probe_expand(id, static_cast<uint32_t>(fixed_r3), nodes_of(fb[a]), owners_of(fb[a], cap),
                                    &ctl->cnt[a], d_status, nodes_of(fb[b]), owners_of(fb[b], cap), &ctl->cnt[b], cap,
                                    d_lvl, &ctl->overflow, blocks, st));
    LC_CUDA(lc::launch_probe_finalize(kk, static_cast<uint32_t>(level), d_lvl, d_status, d_depth, d_nodes, d_levels,
                                      levels_cap, node_cap, &ctl->overflow, &ctl->live[a], &ctl->done, &ctl->cnt[a],
                                      &ctl->live[b], st));
    g_launches += 2;
    ++level;
    if (level % kCheck != 0 && !(depth_cap >= 0 && level >= static_cast<uint64_t>(depth_cap))) continue;
    Ctl h{};
    LC_CUDA(cudaMemcpyAsync(&h, ctl, sizeof h, cudaMemcpyDeviceToHost, st));
    LC_CUDA(cudaStreamSynchronize(st));
    if (h.overflow) {  // level h.done did not fit: grow both buffers, keep its frontier, redo
      const uint64_t redo = h.done;
      const int ra = static_cast<int>(redo & 1), rb = ra ^ 1;
      const unsigned long long need = h.cnt[rb];  // the attempted next-level size
      const unsigned long long ncap = std::max<unsigned long long>(2 * cap, need + (need >> 2));
      Pair np;
      DevBuf* nb = np.b;
      LC_CUDA(alloc(nb[0], ncap));
      LC_CUDA(alloc(nb[1], ncap));
      const unsigned long long cur = h.cnt[ra];
      LC_CUDA(cudaMemcpyAsync(nodes_of(nb[ra]), nodes_of(fb[ra]), cur * 8, cudaMemcpyDeviceToDevice, st));
      LC_CUDA(cudaMemcpyAsync(owners_of(nb[ra], ncap), owners_of(fb[ra], cap), cur * 4, cudaMemcpyDeviceToDevice,
                              st));
      LC_CUDA(cudaStreamSynchronize(st));
      std::swap(fb[0], nb[0]);
      std::swap(fb[1], nb[1]);
      cap = ncap;
      h.overflow = 0;
      h.cnt[rb] = 0;
      LC_CUDA(cudaMemcpyAsync(ctl, &h, sizeof h, cudaMemcpyHostToDevice, st));
      LC_CUDA(cudaMemsetAsync(d_lvl, 0, k * 8, st));
      LC_CUDA(cudaStreamSynchronize(st));
      level = redo;
      continue;
    }
    if (h.live[static_cast<int>((level - 1) & 1)] == 0) break;
  }
  LC_CUDA(cudaMemcpyAsync(depth, d_depth, k * 8, cudaMemcpyDeviceToHost, st));
  LC_CUDA(cudaMemcpyAsync(nodes, d_nodes, k * 8, cudaMemcpyDeviceToHost, st));
  LC_CUDA(cudaMemcpyAsync(censored, d_status, k, cudaMemcpyDeviceToHost, st));
  if (levels_cap) LC_CUDA(cudaMemcpyAsync(level_counts, d_levels, static_cast<size_t>(levels_cap) * 8,
                                          cudaMemcpyDeviceToHost, st));
  LC_CUDA(cudaStreamSynchronize(st));
  for (uint64_t i = 0; i < k; ++i) censored[i] = censored[i] == 2 ? 1 : 0;
  if (levels_cap) level_counts[0] = k;
  return LC_OK;
}

// ---------------------------------------------------------------- closure check

int lc_first_missing(lc_ctx* ctx, const uint64_t* sorted_set, uint64_t m, const uint64_t* queries, uint64_t n,
                     uint64_t* first_missing) {
  if (!ctx || !first_missing) return fail(LC_ERR_ARG, "null argument");
  *first_missing = n;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  LC_CUDA(ctx->a.ensure(std::max<uint64_t>(m, 1) * 8));
  LC_CUDA(ctx->b.ensure(n * 8));
  LC_CUDA(ctx->d.ensure(8));
  if (m) LC_CUDA(cudaMemcpyAsync(ctx->a.p, sorted_set, m * 8, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(cudaMemcpyAsync(ctx->b.p, queries, n * 8, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(cudaMemcpyAsync(ctx->d.p, &n, 8, cudaMemcpyHostToDevice, ctx->stream));
  LC_CUDA(lc::launch_first_missing(ctx->a.as<uint64_t>(), m, ctx->b.as<uint64_t>(), n,
                                   ctx->d.as<unsigned long long>(), ctx->stream));
  g_launches += 1;
  LC_CUDA(cudaMemcpyAsync(first_missing, ctx->d.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

// ------------------------------------------------- steps 4-5: sort, leaf cutting, cycles

static int reduce_error(unsigned int err) {
  switch (err) {
    case 1: return fail(LC_ERR_UNSORTED, "edge records are not sorted by unique source");
    case 2: return fail(LC_ERR_NOT_CLOSED, "a removed leaf's destination has no surviving record; input was not closed");
    case 3: return fail(LC_ERR_NOT_PERMUTATION, "a destination is not a source");
    case 4: return fail(LC_ERR_NOT_PERMUTATION, "destinations are not a permutation of sources");
    default: return LC_OK;
  }
}

// An empty edge list: one pass that removes nothing, as the reference logs it
// (reduce.py:189-223 runs cut_leaves_pass once before testing for the fixpoint).
static int empty_cut(uint64_t* pass_stats, uint32_t max_stats, uint32_t* n_passes) {
  *n_passes = 1;
  if (max_stats && pass_stats) pass_stats[0] = pass_stats[1] = pass_stats[2] = 0;
  return LC_OK;
}

int lc_sort_edges(lc_ctx* ctx, uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist, uint64_t* subtree_size,
                  uint64_t* subtree_depth) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (n < 2) return LC_OK;
  if (!src || !dst || !dist) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  const size_t nb = n * 8;
  uint64_t* host[5] = {src, dst, dist, subtree_size, subtree_depth};
  DevBuf* bufs[5] = {&ctx->a, &ctx->b, &ctx->c, &ctx->d, &ctx->stats};
  uint64_t* dev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  for (int k = 0; k < 5; ++k) {
    if (!host[k]) continue;
    LC_CUDA(bufs[k]->ensure(nb));
    dev[k] = bufs[k]->as<uint64_t>();
    LC_CUDA(cudaMemcpyAsync(dev[k], host[k], nb, cudaMemcpyHostToDevice, ctx->stream));
  }
  LC_CUDA(ctx->scratch.ensure(lc::sort_scratch_bytes(n)));
  int launches = 0;
  LC_CUDA(lc::sort_records_device(n, dev, 5, ctx->scratch.p, ctx->scratch.bytes, ctx->stream, &launches));
  g_launches += launches;
  for (int k = 0; k < 5; ++k)
    if (host[k]) LC_CUDA(cudaMemcpyAsync(host[k], dev[k], nb, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

int lc_sort_edges_device(lc_ctx* ctx, uint64_t n, const uint64_t* const* d_in, uint64_t* const* d_out,
                         void* stream) {
  if (!ctx || !d_in || !d_out) return fail(LC_ERR_ARG, "null argument");
  if (n >= (1ull << 32)) return fail(LC_ERR_ARG, "at most 2^32 - 1 records per sort");
  if (n == 0) return LC_OK;
  if (!d_in[0] || !d_in[1] || !d_in[2] || !d_out[0] || !d_out[1] || !d_out[2]) return fail(LC_ERR_ARG, "null buffer");
  for (int k = 0; k < 5; ++k)
    if ((d_in[k] == nullptr) != (d_out[k] == nullptr)) return fail(LC_ERR_ARG, "column %d: input and output must both be set", k);
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->scratch.ensure(lc::radix_sort_scratch_bytes(n)));
  int launches = 0;
  LC_CUDA(lc::radix_sort_records(n, d_in, d_out, 5, ctx->scratch.p, ctx->scratch.bytes, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_pack_records_device(lc_ctx* ctx, uint64_t n, const uint64_t* d_src, const uint64_t* d_dst,
                           const uint64_t* d_dist, const uint64_t* d_subtree_size, const uint64_t* d_subtree_depth,
                           uint64_t* d_out, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (n && (!d_src || !d_dst || !d_dist || !d_out)) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  int launches = 0;
  LC_CUDA(lc::pack_records_device(n, d_src, d_dst, d_dist, d_subtree_size, d_subtree_depth, d_out, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_cut_leaves(lc_ctx* ctx, uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist, uint64_t* subtree_size,
                  uint64_t* subtree_depth, uint32_t max_passes, uint64_t* pass_stats, uint32_t max_stats,
                  uint32_t* n_passes, uint64_t* n_out) {
  if (!ctx || !n_passes || !n_out) return fail(LC_ERR_ARG, "null argument");
  *n_passes = 0;
  *n_out = n;
  if (n == 0) return empty_cut(pass_stats, max_stats, n_passes);
  if (!src || !dst || !dist || !subtree_size || !subtree_depth) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  const size_t nb = n * 8;
  DevBuf* cols[5] = {&ctx->a, &ctx->b, &ctx->c, &ctx->d, &ctx->stats};
  uint64_t* host[5] = {src, dst, dist, subtree_size, subtree_depth};
  for (int k = 0; k < 5; ++k) {
    LC_CUDA(cols[k]->ensure(nb));
    LC_CUDA(cudaMemcpyAsync(cols[k]->p, host[k], nb, cudaMemcpyHostToDevice, ctx->stream));
  }
  LC_CUDA(ctx->scratch.ensure(lc::reduce_scratch_bytes(n, max_stats)));
  int launches = 0;
  unsigned int err = 0;
  LC_CUDA(lc::cut_leaves_device(n, ctx->a.as<uint64_t>(), ctx->b.as<uint64_t>(), ctx->c.as<uint64_t>(),
                                ctx->d.as<uint64_t>(), ctx->stats.as<uint64_t>(), max_passes, pass_stats, max_stats,
                                n_passes, n_out, &err, ctx->scratch.p, ctx->stream, &launches));
  g_launches += launches;
  if (err) return reduce_error(err);
  for (int k = 0; k < 5; ++k)
    if (*n_out) LC_CUDA(cudaMemcpyAsync(host[k], cols[k]->p, *n_out * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

int lc_cut_leaves_device(lc_ctx* ctx, uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist,
                         uint64_t* subtree_size, uint64_t* subtree_depth, uint32_t max_passes, uint64_t* pass_stats,
                         uint32_t max_stats, uint32_t* n_passes, uint64_t* n_out, void* stream) {
  if (!ctx || !n_passes || !n_out) return fail(LC_ERR_ARG, "null argument");
  *n_passes = 0;
  *n_out = n;
  if (max_stats && !pass_stats) return fail(LC_ERR_ARG, "null pass_stats");
  if (n == 0) return empty_cut(pass_stats, max_stats, n_passes);
  if (!src || !dst || !dist || !subtree_size || !subtree_depth) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  // The passes are replayed from a CUDA graph, which cannot be captured on the legacy
  // default stream: wait for the caller's stream, then run on the context's own stream
  // (the call is synchronous, so the caller's later work sees the results).
  LC_CUDA(cudaStreamSynchronize(stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy));
  LC_CUDA(ctx->scratch.ensure(lc::reduce_scratch_bytes(n, max_stats)));
  int launches = 0;
  unsigned int err = 0;
  LC_CUDA(lc::cut_leaves_device(n, src, dst, dist, subtree_size, subtree_depth, max_passes, pass_stats, max_stats,
                                n_passes, n_out, &err, ctx->scratch.p, ctx->stream, &launches));
  g_launches += launches;
  LC_CUDA(cudaStreamSynchronize(ctx->stream));  // the compaction's last copies are still queued
  return err ? reduce_error(err) : LC_OK;
}

}  // extern "C"

struct lc_cut_shard {
  lc_ctx* ctx = nullptr;
  cudaStream_t stream = nullptr;
  void* mem = nullptr;
  lc::ShardState st{};
};

extern "C" {

int lc_cut_shard_create(lc_ctx* ctx, uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist,
                        uint64_t* subtree_size, uint64_t* subtree_depth, uint32_t n_ranks,
                        const uint64_t* rank_first, const uint64_t* rank_count, void* stream, lc_cut_shard** out,
                        uint64_t* size_sum) {
  if (!ctx || !out || !size_sum || !rank_first || !rank_count) return fail(LC_ERR_ARG, "null argument");
  *out = nullptr;
  if (n_ranks == 0 || n_ranks > lc::kMaxShardRanks)
    return fail(LC_ERR_ARG, "n_ranks must be in [1, %u]", lc::kMaxShardRanks);
  if (n && (!src || !dst || !dist || !subtree_size || !subtree_depth)) return fail(LC_ERR_ARG, "null buffer");
  // shard ranges must ascend (non-empty ranks only; the driver checks the last/first pairs)
  uint64_t prev = 0;
  bool any = false;
  for (uint32_t r = 0; r < n_ranks; ++r) {
    if (!rank_count[r]) continue;
    if (any && rank_first[r] <= prev) return fail(LC_ERR_UNSORTED, "shard ranges do not ascend with rank");
    prev = rank_first[r];
    any = true;
  }
  LC_CUDA(cudaSetDevice(ctx->device));
  lc_cut_shard* h = new lc_cut_shard;
  h->ctx = ctx;
  h->stream = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  cudaError_t e = cudaMalloc(&h->mem, lc::shard_scratch_bytes(n, n_ranks));
  if (e != cudaSuccess) {
    delete h;
    return fail(LC_ERR_CUDA, "shard scratch: %s", cudaGetErrorString(e));
  }
  uint64_t* cols[5] = {src, dst, dist, subtree_size, subtree_depth};
  unsigned int err = 0;
  int launches = 0;
  e = lc::shard_init(&h->st, h->mem, n, cols, n_ranks, rank_first, rank_count, size_sum, &err, h->stream, &launches);
  g_launches += launches;
  if (e != cudaSuccess || err) {
    cudaFree(h->mem);
    delete h;
    if (e != cudaSuccess) return fail(LC_ERR_CUDA, "shard init: %s", cudaGetErrorString(e));
    return reduce_error(err);
  }
  *out = h;
  return LC_OK;
}

int lc_cut_shard_emit(lc_cut_shard* h, int phase, uint64_t* send, uint64_t* counts, uint64_t* info) {
  if (!h || !counts || !info || (h->st.n && !send)) return fail(LC_ERR_ARG, "null argument");
  if (phase != 0 && phase != 1) return fail(LC_ERR_ARG, "phase must be 0 or 1");
  LC_CUDA(cudaSetDevice(h->ctx->device));
  int launches = 0;
  LC_CUDA(lc::shard_emit(&h->st, phase, send, counts, info, h->stream, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_cut_shard_apply(lc_cut_shard* h, int phase, const uint64_t* recv, uint64_t m) {
  if (!h || (m && !recv)) return fail(LC_ERR_ARG, "null argument");
  if (phase != 0 && phase != 1) return fail(LC_ERR_ARG, "phase must be 0 or 1");
  LC_CUDA(cudaSetDevice(h->ctx->device));
  int launches = 0;
  LC_CUDA(lc::shard_apply(&h->st, phase, recv, m, h->stream, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_cut_shard_finish(lc_cut_shard* h, uint64_t* n_out) {
  if (!h || !n_out) return fail(LC_ERR_ARG, "null argument");
  LC_CUDA(cudaSetDevice(h->ctx->device));
  int launches = 0;
  unsigned int err = 0;
  LC_CUDA(lc::shard_finish(&h->st, n_out, &err, h->stream, &launches));
  g_launches += launches;
  return err ? reduce_error(err) : LC_OK;
}

int lc_cut_shard_destroy(lc_cut_shard* h) {
  if (!h) return LC_OK;
  cudaSetDevice(h->ctx->device);
  cudaStreamSynchronize(h->stream);
  if (h->mem) cudaFree(h->mem);
  delete h;
  return LC_OK;
}

// ------------------------------------------------ exhaustive mini-cipher analysis

static uint64_t valid_states(lc::SpecId id) {
  switch (id) {
    case lc::SpecId::A51: return ((1ull << 19) - 1) * ((1ull << 22) - 1) * ((1ull << 23) - 1);
    case lc::SpecId::MINI567: return 31ull * 63ull * 127ull;
    case lc::SpecId::MINI789: return 127ull * 255ull * 511ull;
    default: return 0;
  }
}

int lc_bf_build_device(lc_ctx* ctx, const lc_spec* spec, uint64_t fixed_r3, int clock_all, uint64_t n,
                       int64_t* d_succ, int32_t* d_indeg, uint8_t* d_is_cand, int64_t* d_cycle_of, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if ((rc = check_fixed(id, fixed_r3))) return rc;
  if (id == lc::SpecId::CUSTOM) return fail(LC_ERR_UNSUPPORTED, "the exhaustive analysis is built for the minis only");
  if (n != valid_states(id)) return fail(LC_ERR_ARG, "n must be the spec's valid state count");
  if (n > (1ull << 31)) return fail(LC_ERR_ARG, "instance too large for exhaustive analysis");
  if (!d_succ || !d_indeg || !d_is_cand || !d_cycle_of) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->scratch.ensure(n * 8));
  int launches = 0;
  LC_CUDA(lc::bf_build(id, n, clock_all, static_cast<uint32_t>(fixed_r3), d_succ, d_indeg, d_is_cand, d_cycle_of,
                       ctx->scratch.as<int64_t>(), st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_edges_device(lc_ctx* ctx, uint64_t n, const int64_t* d_succ, const uint8_t* d_is_cand,
                       const int64_t* d_cand, uint64_t m, int64_t* d_dst, int64_t* d_dist, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (m && (!d_succ || !d_is_cand || !d_cand || !d_dst || !d_dist)) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  int launches = 0;
  LC_CUDA(lc::bf_edges(n, d_succ, d_is_cand, d_cand, m, d_dst, d_dist, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_segments_device(lc_ctx* ctx, uint64_t n, const int64_t* d_succ, const int32_t* d_indeg,
                          const uint8_t* d_is_cand, const int64_t* d_cand, uint64_t ncand, int64_t* d_root,
                          int32_t* d_depth, uint64_t* level_counts, uint32_t level_cap, uint32_t* n_levels,
                          void* stream) {
  if (!ctx || !n_levels || (level_cap && !level_counts)) return fail(LC_ERR_ARG, "null argument");
  if (!d_succ || !d_indeg || !d_is_cand || !d_root || !d_depth || (ncand && !d_cand))
    return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  const size_t bytes = lc::bf_segments_scratch(n);
  LC_CUDA(ctx->scratch.ensure(bytes));
  int launches = 0;
  LC_CUDA(lc::bf_segments(n, d_succ, d_indeg, d_is_cand, d_cand, ncand, d_root, d_depth, level_counts, level_cap,
                          n_levels, ctx->scratch.p, ctx->scratch.bytes, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_candidates_device(lc_ctx* ctx, uint64_t n, const uint8_t* d_is_cand, int64_t* d_cand, uint64_t* m_out,
                            void* stream) {
  if (!ctx || !m_out) return fail(LC_ERR_ARG, "null argument");
  *m_out = 0;
  if (n == 0) return LC_OK;
  if (!d_is_cand || !d_cand) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->scratch.ensure(lc::bf_candidates_scratch(n)));
  int launches = 0;
  LC_CUDA(lc::bf_candidates(n, d_is_cand, d_cand, m_out, ctx->scratch.p, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_summary_device(lc_ctx* ctx, uint64_t n, const int32_t* d_indeg, const int64_t* d_root,
                         const int32_t* d_depth, uint64_t m, uint64_t* d_pred_hist, int64_t* d_seg_depth,
                         int64_t* d_seg_size, void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (!d_pred_hist || (n && (!d_indeg || !d_root || !d_depth)) || (m && (!d_seg_depth || !d_seg_size)))
    return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  int launches = 0;
  LC_CUDA(lc::bf_summary(n, d_indeg, d_root, d_depth, m, d_pred_hist, d_seg_depth, d_seg_size, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_cycles_device(lc_ctx* ctx, const lc_spec* spec, uint64_t n, const int64_t* d_succ, const int64_t* d_cycle_of,
                        const uint8_t* d_is_cand, int64_t* d_order, int64_t* d_offset, int64_t* d_length,
                        int64_t* d_leader, int64_t* d_cand_on, int64_t* d_comp, uint64_t* n_on, uint64_t* n_cycles,
                        void* stream) {
  if (!ctx || !n_on || !n_cycles) return fail(LC_ERR_ARG, "null argument");
  lc::SpecId id;
  int rc = check_spec(spec, &id);
  if (rc) return rc;
  if (n == 0 || n != valid_states(id)) return fail(LC_ERR_ARG, "n must be the spec's valid state count");
  if (!d_succ || !d_cycle_of || !d_is_cand || !d_order || !d_offset || !d_length || !d_leader || !d_cand_on ||
      !d_comp)
    return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->scratch.ensure(lc::bf_cycles_scratch(n)));
  const uint64_t m2 = (1ull << spec->lengths[1]) - 1, m3 = (1ull << spec->lengths[2]) - 1;
  const int o2 = spec->lengths[0], o3 = spec->lengths[0] + spec->lengths[1];
  int launches = 0;
  LC_CUDA(lc::bf_cycles(n, d_succ, d_cycle_of, d_is_cand, m2, m3, o2, o3, d_order, d_offset, d_length, d_leader,
                        d_cand_on, d_comp, n_on, n_cycles, ctx->scratch.p, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_bf_cycle_order_device(lc_ctx* ctx, uint64_t m, const int64_t* d_cs, int64_t* d_start, int64_t* d_steps,
                             void* stream) {
  if (!ctx) return fail(LC_ERR_ARG, "null context");
  if (m && (!d_cs || !d_start || !d_steps)) return fail(LC_ERR_ARG, "null buffer");
  LC_CUDA(cudaSetDevice(ctx->device));
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : cudaStreamLegacy;
  Ordered ord_(ctx, st);
  LC_CUDA(ctx->scratch.ensure(std::max<uint64_t>(m, 1) * 8 * 3));
  int64_t* t = ctx->scratch.as<int64_t>();
  int launches = 0;
  LC_CUDA(lc::bf_cycle_order(m, d_cs, d_start, d_steps, t, t + m, t + 2 * m, st, &launches));
  g_launches += launches;
  return LC_OK;
}

int lc_count_cycles(lc_ctx* ctx, uint64_t n, const uint64_t* src, const uint64_t* dst, const uint64_t* dist,
                    const uint64_t* subtree_size, uint64_t* leader, uint64_t* hop_count, uint64_t* clock_length,
                    uint64_t* tree_size, uint64_t* n_cycles) {
  if (!ctx || !n_cycles) return fail(LC_ERR_ARG, "null argument");
  *n_cycles = 0;
  if (n == 0) return LC_OK;
  LC_CUDA(cudaSetDevice(ctx->device));
  Ordered ord_(ctx, ctx->stream);
  const size_t nb = n * 8;
  DevBuf* in[4] = {&ctx->a, &ctx->b, &ctx->c, &ctx->d};
  const uint64_t* host[4] = {src, dst, dist, subtree_size};
  for (int k = 0; k < 4; ++k) {
    LC_CUDA(in[k]->ensure(nb));
    LC_CUDA(cudaMemcpyAsync(in[k]->p, host[k], nb, cudaMemcpyHostToDevice, ctx->stream));
  }
  LC_CUDA(ctx->stats.ensure(4 * nb));
  uint64_t* out = ctx->stats.as<uint64_t>();
  LC_CUDA(ctx->scratch.ensure(lc::cycles_scratch_bytes(n)));
  int launches = 0;
  unsigned int err = 0;
  LC_CUDA(lc::count_cycles_device(n, ctx->a.as<uint64_t>(), ctx->b.as<uint64_t>(), ctx->c.as<uint64_t>(),
                                  ctx->d.as<uint64_t>(), out, out + n, out + 2 * n, out + 3 * n, n_cycles, &err,
                                  ctx->scratch.p, ctx->stream, &launches));
  g_launches += launches;
  if (err == 1) return fail(LC_ERR_NOT_PERMUTATION, "duplicate or unsorted source");
  if (err) return reduce_error(err);
  const uint64_t m = *n_cycles;
  uint64_t* dsts[4] = {leader, hop_count, clock_length, tree_size};
  for (int k = 0; k < 4; ++k)
    if (m) LC_CUDA(cudaMemcpyAsync(dsts[k], out + k * n, m * 8, cudaMemcpyDeviceToHost, ctx->stream));
  LC_CUDA(cudaStreamSynchronize(ctx->stream));
  return LC_OK;
}

}  // extern "C"
