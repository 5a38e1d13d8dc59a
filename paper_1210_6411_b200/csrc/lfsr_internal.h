// Host/device shared declarations for the lfsr_b200 kernels (not part of the C ABI).
#pragma once

#ifndef __CUDACC_RTC__  // (csrc/jit.cu compiles the kernels with NVRTC: device parts only)
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#endif

// Bounds / invariant checks of the checked build (-DLC_CHECKS=1, __graft_entry__.build()
// writes it to _lib/checked/; tests/test_gpu_checked.py runs every kernel mode on it): a
// failed check prints its site and traps, so the call fails with a CUDA error.  Compiled
// out of the product library.
#ifndef LC_CHECKS
#define LC_CHECKS 0
#endif
#if LC_CHECKS
#define LC_CHECK(c)                                                                \
  do {                                                                             \
    if (!(c)) {                                                                    \
      printf("LC_CHECK failed at %s:%d: %s\n", __FILE__, __LINE__, #c);            \
      __trap();                                                                    \
    }                                                                              \
  } while (0)
#else
#define LC_CHECK(c) \
  do {              \
  } while (0)
#endif

#include "../../include/lfsr_b200.h"

namespace lc {

// CUSTOM: a valid cipher spec without a precompiled kernel; its kernels are compiled for
// it at first use (csrc/jit.cu) and the calling thread's current custom spec selects them.
enum class SpecId { A51 = 0, MINI567 = 1, MINI789 = 2, CUSTOM = 3, UNSUPPORTED = -1 };

constexpr int kWalkThreads = 128;
constexpr uint64_t kInf = ~0ull;

// Per-lane bookkeeping of the chain walk (global scratch, touched only on events).
struct LaneMeta {
  uint64_t walk;       // index of the start this lane is walking
  uint64_t leg_start;  // warp clock at which the current leg began
  uint64_t arm_at;     // warp clock from which the lane may report a special node
  uint64_t deadline;   // warp clock of the cap audit
  uint32_t legs_done;
  uint32_t pad;        // 1: the cap audit excused this leg once (inside a fixed-R3 run)
};

// A parked lane (lane mode): state and leg bookkeeping relative to the parking clock, so
// a later launch can resume it in any lane of any warp (csrc/walk.cu, "parking").
struct ResumeRec {
  uint64_t state;
  uint64_t walk;
  uint64_t elapsed;   // clocks since the leg started
  uint64_t arm_rel;   // clocks until the lane may report (0: armed)
  uint64_t dead_rel;  // clocks until the cap audit (kInf: none)
  uint32_t legs_done;
  uint32_t pad;       // LaneMeta::pad
};

struct WalkParams {
  const uint64_t* starts;
  uint64_t n;
  uint64_t* dst;  // [n][legs]
  uint64_t* dist;
  uint64_t stride;
  uint64_t cap1;  // max_clocks + 1, saturated
  uint64_t hist_lo;
  uint32_t hist_shift;
  uint32_t hist_bins;
  uint32_t legs;
  uint32_t fixed_r3;
  uint32_t refill_min;  // lane mode: refill once this many of the warp's 1024 lanes are idle
  uint32_t chunk;       // starts per queue item: 1024 (whole-warp refill) or 1 (lane refill)
  uint32_t nq;          // queues: one per SM sub-partition, or 1
  uint32_t pad;
  unsigned long long* queues;  // nq counters, 16 words apart
  const uint16_t* smsp_map;    // %smid -> dense SM index (nq > 1)
  unsigned int* exhausted;     // set once every queue is empty
  unsigned long long* stats;   // LC_ST_* block
  LaneMeta* meta;              // [threads][32]
  const uint32_t* mode_word;   // auto mode: 1 = whole-warp refill, 0 = lane refill (else null)
  const ResumeRec* resume;     // lane mode: items are parked lanes instead of starts
  ResumeRec* pool;             // parking destination (null: never park)
  unsigned long long* pool_count;
  uint32_t park_below;         // park a drained warp once fewer lanes than this are live
  uint32_t pad2;
  const uint32_t* need3;       // [2^l3] R3 clocks from each R3 value to fixed_r3 (null: none)
  uint32_t run_if_mode;        // ~0: always run; else run only if *mode_word equals it
  uint32_t pad3;
  const unsigned long long* n_dev;  // resume round queued without a host sync: item count on the device (else null)
  uint64_t park_min;                // park only while the round has more than this many items
  uint64_t pool_cap;                // ResumeRec slots in `pool` (a warp that does not fit keeps walking)
  uint64_t window;                  // R3's period through F (custom specs; built-ins use Spec::WINDOW)
};

#ifndef __CUDACC_RTC__
// Launchers (defined in the .cu files); all enqueue on `stream`.
// rearm: the variant that bounds each lane's next special node by R3's distance to F
// (WalkParams::need3) instead of checking every step once armed.
cudaError_t launch_walk(SpecId id, bool static_f, bool rearm, const WalkParams& p, int blocks,
                        cudaStream_t stream);
int walk_blocks_per_sm(SpecId id, bool static_f);
cudaError_t launch_init_stats(uint64_t* stats, uint64_t hist_lo, uint32_t hist_shift, uint32_t hist_bins,
                              unsigned long long* queues, uint32_t nq, unsigned int* exhausted,
                              cudaStream_t stream);
cudaError_t probe_smids(int sms, unsigned int* d_flags, cudaStream_t stream);
// mode_word <- 1 iff every start is a special-node-like start (fixed R3, R3 clocked at
// once): near-constant chain lengths, so whole-warp refill loses nothing.
cudaError_t launch_mode_probe(SpecId id, const uint64_t* starts, uint64_t n, uint32_t F, uint32_t* mode_word,
                              cudaStream_t stream);

cudaError_t launch_is_candidate(SpecId id, const uint64_t* xs, uint64_t n, uint32_t F, uint8_t* out,
                                cudaStream_t stream);
cudaError_t launch_predecessors(SpecId id, const uint64_t* xs, uint64_t n, uint64_t* out,
                                uint8_t* count, cudaStream_t stream);
cudaError_t launch_clock(SpecId id, const uint64_t* xs, uint64_t n, uint64_t t, uint64_t* out,
                         cudaStream_t stream);

// Step-1 enumeration of R2 rows [r2_lo, r2_hi) (closed-form streaming writer).
cudaError_t launch_enumerate(SpecId id, uint32_t F, uint64_t r2_lo, uint64_t r2_hi, uint64_t* out,
                             uint64_t cap, uint64_t* d_count, cudaStream_t stream, int* launches);
// K0 seeded start set: ordered compaction (tile counts, scan, ballot writes); scratch
// must hold random_scratch_words(trials) u64.
cudaError_t launch_random_candidates(SpecId id, uint32_t F, uint64_t seed, uint64_t trials,
                                     uint64_t* out, uint64_t cap, uint64_t* d_count,
                                     uint64_t* scratch, uint64_t scratch_words,
                                     cudaStream_t stream, int* launches);
uint64_t random_scratch_words(uint64_t trials);

// spill: per-lane global overflow stacks behind the shared-memory ring (spill_cap
// entries per lane, prune_spill_bytes(blocks, spill_cap) bytes; null: none).
uint64_t prune_spill_bytes(int blocks, uint32_t cap);
cudaError_t launch_prune(SpecId id, uint32_t F, int mode, uint64_t limit, const uint64_t* cands,
                         uint64_t n, uint8_t* removed, uint64_t* work, unsigned long long* queue,
                         void* spill, uint32_t spill_cap, int ring, int blocks, cudaStream_t stream);
// Ring depth (entries per lane in shared memory) for a batch of n candidates: the deep
// ring below 2^24 (tail-bound), the wide-occupancy one above (LFSR_PRUNE_RING forces 20/32).
int prune_ring_for(uint64_t n);
int prune_blocks_per_sm(SpecId id, int ring);

// K3 v2 (csrc/prune.cu): 32-bit node registers, register-cached pending entries; same
// results as launch_prune.  mode 0 = dfs, 1 = bfs.
int prune2_blocks_per_sm(SpecId id, int mode);
uint64_t prune2_spill_bytes(int blocks, uint32_t cap);
cudaError_t launch_prune2(SpecId id, uint32_t F, int mode, uint64_t limit, const uint64_t* cands, uint64_t n,
                          uint8_t* removed, uint64_t* work, unsigned long long* queue, void* spill,
                          uint32_t spill_cap, int blocks, cudaStream_t stream);

// K3 v3 (csrc/prune.cu): one uniform step per expansion, a per-lane stack that never
// drops entries (spill: prune3_spill_bytes(blocks, limit) bytes); for limit <=
// prune3_max_limit().  Same results as launch_prune2; mode 0 = dfs, 1 = bfs.
int prune3_blocks_per_sm(SpecId id);
int prune3_threads();
uint32_t prune3_max_limit();
uint64_t prune3_spill_bytes(int blocks, uint32_t limit);
cudaError_t launch_prune3(SpecId id, uint32_t F, int mode, uint32_t limit, const uint64_t* cands, uint64_t n,
                          uint8_t* removed, uint64_t* work, unsigned long long* queue, void* spill, int blocks,
                          cudaStream_t stream);

// Batched segment probes (prune.cu; pipeline.probe_segment): one expand launch and one
// finalize launch per level, driven by lc_probe_segments.
cudaError_t launch_probe_expand(SpecId id, uint32_t F, const uint64_t* fnode, const uint32_t* fowner,
                                const unsigned long long* cur_count, const uint8_t* status, uint64_t* nnode,
                                uint32_t* nowner, unsigned long long* next_count, unsigned long long cap,
                                unsigned long long* lvl, unsigned int* overflow, int blocks, cudaStream_t st);
cudaError_t launch_probe_finalize(uint32_t k, uint32_t level, unsigned long long* lvl, uint8_t* status,
                                  uint64_t* depth, uint64_t* nodes, unsigned long long* level_counts,
                                  uint32_t levels_cap, int64_t node_cap, const unsigned int* overflow,
                                  unsigned long long* live, unsigned long long* done_count,
                                  unsigned long long* cnt_reset, unsigned long long* live_reset, cudaStream_t st);
cudaError_t launch_probe_censor(uint32_t k, uint8_t* status, cudaStream_t st);

cudaError_t measure_lop3_peak(int sms, double* ops_per_s, double* sm_mhz);

// Steps 4-5 (reduce.cu).  err_out: 0 ok, 1 unsorted sources, 2 not closed,
// 3 destination not a source, 4 not a permutation.
size_t reduce_scratch_bytes(uint64_t n, uint32_t max_stats);
cudaError_t cut_leaves_device(uint64_t n, uint64_t* src, uint64_t* dst, uint64_t* dist, uint64_t* size,
                              uint64_t* depth, uint32_t max_passes, uint64_t* pass_stats, uint32_t max_stats,
                              uint32_t* n_passes, uint64_t* n_out, unsigned int* err_out, void* scratch,
                              cudaStream_t st, int* launches);

// Leaf-cutting control block in device memory (frontier sizes and pass counters, so
// passes can be replayed from a CUDA graph).
struct CutCtl {
  unsigned long long cnt[2];   // frontier sizes; pass parity w consumes cnt[w], fills cnt[w^1]
  unsigned long long alive;    // records alive before the current pass
  unsigned long long sum;      // subtree-size sum over the alive records
  unsigned long long pass;     // passes completed
  unsigned long long done_at;  // first pass that removed nothing (0: not yet)
};

// One rank's shard of a sharded leaf cut (multi-GPU step 4): contiguous source range,
// caller-owned device columns, in-degrees, alive flags and two frontiers in scratch.
struct ShardState {
  uint64_t n;
  uint64_t* cols[5];  // source, destination, distance, subtree_size, subtree_depth
  uint32_t n_ranks, nb;
  uint64_t* bounds;   // [nb] first source per non-empty rank (bounds[0] = 0)
  uint32_t* brank;    // [nb] rank of each bound
  unsigned long long *ocount, *ocursor;
  unsigned int* err;
  CutCtl* ctl;
  uint64_t* tiles;
  unsigned int* indeg;
  uint8_t* alive;
  uint64_t* f[2];
  int w;
  bool started;
};
size_t shard_scratch_bytes(uint64_t n, uint32_t n_ranks);
cudaError_t shard_init(ShardState* sh, void* scratch, uint64_t n, uint64_t* const cols[5], uint32_t n_ranks,
                       const uint64_t* rank_first, const uint64_t* rank_count, uint64_t* size_sum,
                       unsigned int* err_out, cudaStream_t st, int* launches);
cudaError_t shard_emit(ShardState* sh, int phase, uint64_t* send, uint64_t* counts, uint64_t* info,
                       cudaStream_t st, int* launches);
cudaError_t shard_apply(ShardState* sh, int phase, const uint64_t* msgs, uint64_t m, cudaStream_t st,
                        int* launches);
cudaError_t shard_finish(ShardState* sh, uint64_t* n_out, unsigned int* err_out, cudaStream_t st, int* launches);
constexpr uint32_t kMaxShardRanks = 1024;

// Exhaustive mini-cipher analysis (bruteforce.cu; oracle.brute_force_analysis).
cudaError_t bf_build(SpecId id, uint64_t n, int clock_all, uint32_t F, int64_t* succ, int32_t* indeg,
                     uint8_t* is_cand, int64_t* g, int64_t* tmp, cudaStream_t st, int* launches);
cudaError_t bf_edges(uint64_t n, const int64_t* succ, const uint8_t* is_cand, const int64_t* cand, uint64_t m,
                     int64_t* dst, int64_t* dist, cudaStream_t st, int* launches);
size_t bf_segments_scratch(uint64_t n);
cudaError_t bf_segments(uint64_t n, const int64_t* succ, const int32_t* indeg, const uint8_t* is_cand,
                        const int64_t* cand, uint64_t ncand, int64_t* root, int32_t* depth, uint64_t* level_counts,
                        uint32_t level_cap, uint32_t* n_levels, void* scratch, size_t scratch_bytes, cudaStream_t st,
                        int* launches);
cudaError_t bf_cycle_order(uint64_t m, const int64_t* cs, int64_t* lab, int64_t* steps, int64_t* t0, int64_t* t1,
                           int64_t* t2, cudaStream_t st, int* launches);
size_t bf_candidates_scratch(uint64_t n);
cudaError_t bf_candidates(uint64_t n, const uint8_t* is_cand, int64_t* cand, uint64_t* m_out, void* scratch,
                          cudaStream_t st, int* launches);
cudaError_t bf_summary(uint64_t n, const int32_t* indeg, const int64_t* root, const int32_t* depth, uint64_t m,
                       uint64_t* pred_hist, int64_t* seg_depth, int64_t* seg_size, cudaStream_t st, int* launches);
size_t bf_cycles_scratch(uint64_t n);
cudaError_t bf_cycles(uint64_t n, const int64_t* succ, const int64_t* g, const uint8_t* is_cand, uint64_t m2,
                      uint64_t m3, int o2, int o3, int64_t* order, int64_t* offset, int64_t* length, int64_t* leader,
                      int64_t* cand_on, int64_t* comp, uint64_t* n_on, uint64_t* n_cycles, void* scratch,
                      cudaStream_t st, int* launches);

size_t cycles_scratch_bytes(uint64_t n);
cudaError_t count_cycles_device(uint64_t n, const uint64_t* src, const uint64_t* dst, const uint64_t* dist,
                                const uint64_t* size, uint64_t* leader, uint64_t* hops_out, uint64_t* clocks_out,
                                uint64_t* tree_out, uint64_t* n_cycles, unsigned int* err_out, void* scratch,
                                cudaStream_t st, int* launches);
cudaError_t pack_records_device(uint64_t n, const uint64_t* src, const uint64_t* dst, const uint64_t* dist,
                                const uint64_t* size, const uint64_t* depth, uint64_t* out, cudaStream_t st,
                                int* launches);
size_t sort_scratch_bytes(uint64_t n);
// In-house LSD radix sort (csrc/sort.cu): cols_in[0] = keys; out of place; n < 2^32.
size_t radix_sort_scratch_bytes(uint64_t n);
cudaError_t radix_sort_records(uint64_t n, const uint64_t* const* cols_in, uint64_t* const* cols_out, int ncols,
                               void* scratch, size_t scratch_bytes, cudaStream_t st, int* launches);
cudaError_t sort_records_device(uint64_t n, uint64_t* const* cols, int ncols, void* scratch, size_t scratch_bytes,
                                cudaStream_t st, int* launches);

cudaError_t launch_first_missing(const uint64_t* set, uint64_t m, const uint64_t* q, uint64_t n,
                                 unsigned long long* first, cudaStream_t stream);

#endif  // !__CUDACC_RTC__

}  // namespace lc
