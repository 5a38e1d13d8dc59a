/*
 * lfsr_b200 -- C ABI of the B200-native A5/1 state-graph kernels (arXiv 1210.6411,
 * steps 1-3).  Plain pointers and sizes only; no torch types cross this boundary.
 *
 * The reference (`lfsrcycles`, /root/reference/pkg/src/lfsrcycles) is pure Python and
 * has no FFI of its own; each entry point below replaces one reference function (the
 * "operator API" of SURVEY.md §8(b)) and says which.  INTEGRATION.md shows the ctypes
 * binding the Python package uses (paper_1210_6411_b200/_native.py).
 *
 * Conventions
 *  - States are packed u64 exactly as cipher.py:90-131 (R1 low bits, R3 high bits).
 *  - Functions without a `_device` suffix take HOST buffers, are synchronous, and do
 *    the host<->device copies themselves.  `_device` variants take device pointers and
 *    a cudaStream_t (passed as void*), enqueue work and return without synchronising.
 *  - Return 0 on success or a negative LC_ERR_* code; lc_last_error() (thread-local)
 *    holds the message.  No C++ exception crosses the ABI.
 *  - A context owns scratch buffers (walk pools, queues, staging).  Calls on one context
 *    are ordered on the device: each call's stream first waits for the previous call's
 *    work (an event the context records), so `_device` calls on different streams may
 *    share a context safely; they then run one after another, not concurrently.
 *  - The three built-in ciphers (A5/1, mini567, mini789 -- cipher.py:173-194) have
 *    precompiled kernels; any other valid spec (registers of at most 32 bits) gets the
 *    same kernels compiled for it at first use (NVRTC, csrc/jit.cu).  Specs the kernels
 *    cannot hold return LC_ERR_UNSUPPORTED (there is no CPU path).
 */
#ifndef LFSR_B200_H
#define LFSR_B200_H

#ifndef __CUDACC_RTC__
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define LC_ABI_VERSION 1

#define LC_OK 0
#define LC_ERR_ARG (-1)          /* ValueError in the reference (bitslice.py:269-272, ...) */
#define LC_ERR_CUDA (-2)         /* CUDA runtime failure */
#define LC_ERR_UNSUPPORTED (-3)  /* spec the kernels cannot hold (or NVRTC unavailable) */
#define LC_ERR_CAP (-4)          /* StrideError: walk cap exceeded (bitslice.py:316-322) */
#define LC_ERR_INVALID_STATE (-5)/* a start has a zero register; the reference
                                    walks it to the cap and raises StrideError */
#define LC_ERR_OVERFLOW (-6)     /* output capacity too small */
#define LC_ERR_UNSORTED (-7)     /* edge records not sorted by unique source (records.py:3-5) */
#define LC_ERR_NOT_CLOSED (-8)   /* a removed leaf's destination has no record (reduce.py:182-184) */
#define LC_ERR_NOT_PERMUTATION (-9) /* count_cycles input is not a permutation (reduce.py:226-246) */

/* Cipher instance (cipher.py:57-170 CipherSpec): register lengths, feedback tap masks
 * (bit i set = tap at register bit i) and clock tap positions. */
typedef struct {
    int32_t lengths[3];
    uint64_t tap_masks[3];
    int32_t clock_taps[3];
} lc_spec;

/* Layout of the u64 statistics block every walk accumulates into (device or host).
 * All counters are integers (bit-exact, order independent) and are summed / min-ed /
 * max-ed across ranks by the distributed driver (NCCL all-reduce). */
enum {
    LC_ST_EDGES = 0,        /* walks (legs) completed                          (sum) */
    LC_ST_TRANSITIONS = 1,  /* sum of dist = A5/1 transitions walked           (sum) */
    LC_ST_MIN = 2,          /* min dist                                         (min) */
    LC_ST_MAX = 3,          /* max dist                                         (max) */
    LC_ST_SQ_LO = 4,        /* sum (dist - hist_lo)^2, low 64 bits              (u128 sum) */
    LC_ST_SQ_HI = 5,        /*                         high 64 bits                      */
    LC_ST_ERROR = 6,        /* 0 or -LC_ERR_* of the first error                        */
    LC_ST_ERROR_INDEX = 7,  /* smallest start index that raised (min)                   */
    LC_ST_HIST_LO = 8,      /* histogram: bin b counts dist in [lo + b<<shift, ...)      */
    LC_ST_HIST_SHIFT = 9,
    LC_ST_HIST_BINS = 10,   /* number of interior bins; +2 under/overflow bins          */
    LC_ST_LAUNCHES = 11,    /* kernels launched by the call (host-side count)           */
    LC_ST_HEADER = 16       /* histogram starts here: [under, bins..., over]            */
};

typedef struct lc_ctx lc_ctx;

int lc_abi_version(void);
const char *lc_last_error(void);
int lc_device_count(int *count);
/* Compile every kernel for a (custom) spec with NVRTC and discard the result: no device
 * needed.  LC_ERR_UNSUPPORTED with the compiler log in lc_last_error() on failure.  (The
 * kernels are compiled and loaded at the spec's first use anyway; this is the check.) */
int lc_spec_compile_check(const lc_spec *spec);

/* One context per (device, host thread).  Owns scratch buffers and a stream. */
int lc_ctx_create(int device, lc_ctx **out);
int lc_ctx_destroy(lc_ctx *ctx);
int lc_ctx_sm_count(lc_ctx *ctx, int *sms);
int lc_ctx_synchronize(lc_ctx *ctx);

/* Pinned host memory for the end-to-end (host-buffer) path. */
int lc_host_alloc(uint64_t bytes, void **out);
int lc_host_free(void *p);

/* Roofline denominator (no reference counterpart): measured sustained 32-bit LOP3
 * results/s of the whole device and the SM clock seen meanwhile (MHz). */
int lc_lop3_peak(lc_ctx *ctx, double *lop3_per_s, double *sm_mhz);

/* Kernel launches made by this thread's lc_* calls since the last reset. */
uint64_t lc_launch_count(void);
void lc_launch_count_reset(void);

/* ---------------------------------------------------------------- step 3: walks */

/* Replaces bitslice._run_walks (bitslice.py:259-323), i.e. forward_to_candidate
 * (bitslice.py:326-342, legs = 1) and candidate_hops (bitslice.py:345-354, stride = 1,
 * legs >= 1).  For every start, `legs` consecutive candidate hops; hop 1 is the first
 * candidate at clock >= max(stride, 1).  dest/dist are [n][legs] row-major.
 * max_clocks: the reference cap (bitslice.py:273-274); StrideError semantics in
 * DESIGN.md §"Cap".  refill: 0 = auto (single-hop walks from all special-node-like
 * starts refill whole warps, decided on the device; otherwise per lane), 1 = refill a
 * lane as soon as it finishes, 1024 = refill a warp only when all 1024 lanes are idle.
 * hist_lo/hist_shift/hist_bins configure the chain-length histogram in `stats`
 * (LC_ST_HEADER + hist_bins + 2 words). */
int lc_walk(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, const uint64_t *starts,
            uint64_t n, uint64_t stride, uint64_t max_clocks, uint32_t legs, uint32_t refill,
            uint64_t *dest, uint64_t *dist, uint64_t hist_lo, uint32_t hist_shift,
            uint32_t hist_bins, uint64_t *stats);
/* lc_walk on device buffers, enqueued on `stream` and returning without a sync.  Lane-mode
 * walks with more starts than one wave of the GPU's warp schedulers holds queue up to
 * four launches: warps drained below half occupancy park their lanes and the next launch
 * resumes them packed (item count read on the device).  Results are identical to one
 * launch; the environment variable LFSR_WALK_NO_PARK forces one launch (A/B testing). */
int lc_walk_device(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3,
                   const uint64_t *d_starts, uint64_t n, uint64_t stride, uint64_t max_clocks,
                   uint32_t legs, uint32_t refill, uint64_t *d_dest, uint64_t *d_dist,
                   uint64_t hist_lo, uint32_t hist_shift, uint32_t hist_bins,
                   uint64_t *d_stats, void *stream);

/* Replaces bitslice.clock_sliced (bitslice.py:223-228): every state advanced t clocks. */
int lc_clock(lc_ctx *ctx, const lc_spec *spec, const uint64_t *xs, uint64_t n, uint64_t t,
             uint64_t *out);

/* ------------------------------------------------------- steps 1-2: predicate, prune */

/* Replaces is_candidate (cipher.py:420-428) over a batch: out[i] = 1 iff xs[i] is a
 * special node (R3 == fixed, R3 leaves fixed on the next clock, has a predecessor). */
int lc_is_candidate(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, const uint64_t *xs,
                    uint64_t n, uint8_t *out);

/* Replaces predecessors (cipher.py:342-369) over a batch: out is [n][4] in the
 * reference's LUT pattern order, count[i] in 0..4 (the leaf filter is count == 0). */
int lc_predecessors(lc_ctx *ctx, const lc_spec *spec, const uint64_t *xs, uint64_t n,
                    uint64_t *out, uint8_t *count);

/* Replaces enumerate_candidates (pipeline.py:104-118) restricted to R2 rows
 * [r2_lo, r2_hi): every candidate, ascending.  Writes min(count, cap) states and
 * sets *count; returns LC_ERR_OVERFLOW if count > cap. */
int lc_enumerate(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, uint64_t r2_lo,
                 uint64_t r2_hi, uint64_t *out, uint64_t cap, uint64_t *count);
int lc_enumerate_device(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, uint64_t r2_lo,
                        uint64_t r2_hi, uint64_t *d_out, uint64_t cap, uint64_t *d_count,
                        void *stream);

/* Replaces the per-candidate decision of prune_shallow_segments (pipeline.py:163-222):
 * mode 0 = dfs (_dfs_is_shallow, depth limit), 1 = bfs (_bfs_is_small, node limit).
 * removed[i] = 1 iff cands[i] roots a shallow segment; work[i] = the reference's
 * per-candidate `expanded` counter (LIFO order replicated). */
int lc_prune(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, int32_t mode, uint64_t limit,
             const uint64_t *cands, uint64_t n, uint8_t *removed, uint64_t *work);
int lc_prune_device(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, int32_t mode,
                    uint64_t limit, const uint64_t *d_cands, uint64_t n, uint8_t *d_removed,
                    uint64_t *d_work, void *stream);

/* Seeded synthetic start set (K0): the first n special nodes of the
 * counter-based stream trial i -> (r1, r2) = split(splitmix64(seed + i*golden)), in trial
 * order.  *trials_used = trials consumed.  Host and device variants. */
/* Replaces probe_segment (pipeline.py:262-298) for k roots at once: each root's reverse
 * level-order sweep through its segment (predecessors that are not special nodes), as
 * (deepest level reached, nodes seen, censored).  depth_cap / node_cap < 0: no cap.
 * level_counts[l] (levels_cap entries, host) = nodes at depth l summed over the roots
 * (index 0 = the roots).  Device-resident: one expand and one finalize launch per level,
 * the host looking at the live count every 16 levels.  Synchronous. */
int lc_probe_segments(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, const uint64_t *roots, uint64_t k,
                      int64_t depth_cap, int64_t node_cap, uint64_t *depth, uint64_t *nodes, uint8_t *censored,
                      uint64_t *level_counts, uint32_t levels_cap);
int lc_random_candidates(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, uint64_t seed,
                         uint64_t n, uint64_t *out, uint64_t *trials_used);
int lc_random_candidates_device(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3,
                                uint64_t seed, uint64_t n, uint64_t *d_out, void *stream);

/* The reference's own seeded sampler, host-side (no context, no device): the first n
 * results of `random_candidate(random.Random(seed), spec, params, table)` called n times on
 * one generator (pipeline.py:301-310), bit-identical to CPython's MT19937 / randrange
 * stream.  Config 1 is seed 0 x 2^16, config 2 seed 0 x 2^24.
 * *draws_used = (r1, r2) pairs drawn.  Registers of more than 32 bits: LC_ERR_UNSUPPORTED. */
int lc_reference_candidates(const lc_spec *spec, uint64_t fixed_r3, uint64_t seed, uint64_t n,
                            uint64_t *out, uint64_t *draws_used);
/* `count` independent streams, stream i = lc_reference_candidates(seeds[i], n_each) into
 * out[i*n_each ...], on up to `threads` host threads (per-shard seeds of the multi-GPU
 * bench). */
int lc_reference_candidates_multi(const lc_spec *spec, uint64_t fixed_r3, const uint64_t *seeds,
                                  uint32_t count, uint64_t n_each, uint64_t *out, uint32_t threads);

/* Closure check of build_skeleton_edges (pipeline.py:251-255): first i with
 * queries[i] not in the ascending array `sorted_set`, or n if all are members. */
int lc_first_missing(lc_ctx *ctx, const uint64_t *sorted_set, uint64_t m, const uint64_t *queries,
                     uint64_t n, uint64_t *first_missing);

/* ------------------------------------------- steps 4-5: edge output, leaf cutting, cycles */

/* Edge-output stage: sort skeleton edge records ascending by source, in place (host
 * buffers; subtree_size / subtree_depth may be NULL).  Produces the order write_edges
 * and step 4 require (records.py:3-5, reduce.py:3-4). */
int lc_sort_edges(lc_ctx *ctx, uint64_t n, uint64_t *src, uint64_t *dst, uint64_t *dist,
                  uint64_t *subtree_size, uint64_t *subtree_depth);
/* Device form, out of place: d_in[0..4] = (source, destination, distance, subtree_size,
 * subtree_depth) columns (sizes / depths may be NULL), d_out[0..4] receive them sorted by
 * source (stable: equal sources keep their input order).  The output columns must not
 * alias the inputs; n < 2^32.  Enqueued on `stream` without a host synchronisation
 * (in-house LSD radix sort, csrc/sort.cu). */
int lc_sort_edges_device(lc_ctx *ctx, uint64_t n, const uint64_t *const *d_in, uint64_t *const *d_out,
                         void *stream);

/* Edge-output writer: 40-byte little-endian '<5Q' records (records.py:24-36) from
 * device columns, d_out = 5 * n u64 words (subtree_size / subtree_depth may be NULL:
 * zero).  Enqueued on `stream`. */
int lc_pack_records_device(lc_ctx *ctx, uint64_t n, const uint64_t *d_src, const uint64_t *d_dst,
                           const uint64_t *d_dist, const uint64_t *d_subtree_size,
                           const uint64_t *d_subtree_depth, uint64_t *d_out, void *stream);

/* Replaces reduce.cut_leaves_pass (reduce.py:118-186; max_passes = 1) and
 * cut_leaves_to_fixpoint (reduce.py:189-223; max_passes = 0) on records held in host
 * buffers (SoA, sorted by unique source), in place: the first *n_out records are the
 * survivors in source order with folded subtree sizes/depths.  pass_stats receives
 * (leaves_removed, inner_nodes, out_size_sum) per pass, up to max_stats passes. */
int lc_cut_leaves(lc_ctx *ctx, uint64_t n, uint64_t *src, uint64_t *dst, uint64_t *dist,
                  uint64_t *subtree_size, uint64_t *subtree_depth, uint32_t max_passes,
                  uint64_t *pass_stats, uint32_t max_stats, uint32_t *n_passes, uint64_t *n_out);

/* lc_cut_leaves on device-resident columns (synchronous on `stream`; NULL = legacy
 * default stream).  pass_stats is a host array. */
int lc_cut_leaves_device(lc_ctx *ctx, uint64_t n, uint64_t *d_src, uint64_t *d_dst, uint64_t *d_dist,
                         uint64_t *d_subtree_size, uint64_t *d_subtree_depth, uint32_t max_passes,
                         uint64_t *pass_stats, uint32_t max_stats, uint32_t *n_passes, uint64_t *n_out,
                         void *stream);

/* Sharded leaf cutting: the multi-GPU form of cut_leaves_pass / cut_leaves_to_fixpoint
 * (reduce.py:118-223).  Rank r of n_ranks holds the records whose sources fall in its
 * contiguous range (rank_first[r] = its first source, rank_count[r] = its record count;
 * ranges ascend with r) in device columns it owns.  The host driver alternates
 *   emit(phase) -> exchange messages by owner rank (all-to-all) -> apply(phase)
 * once with phase 0 (in-degree counting) and then once per pass with phase 1 (fold the
 * pass's leaves into their destinations).  A message is 3 u64 words (destination,
 * size + 1, depth + 1); emit writes them to `d_send` (capacity 3 * n words) grouped by
 * owner rank and returns the per-rank counts in counts[n_ranks] and, in info[2], the
 * records emitted (phase 1: this pass's local leaves) and the shard's error word
 * (2: a destination has no record -- input not closed).  finish compacts the survivors
 * in place (*n_out of them, source order).  All calls are synchronous on `stream`. */
typedef struct lc_cut_shard lc_cut_shard;
int lc_cut_shard_create(lc_ctx *ctx, uint64_t n, uint64_t *d_src, uint64_t *d_dst, uint64_t *d_dist,
                        uint64_t *d_subtree_size, uint64_t *d_subtree_depth, uint32_t n_ranks,
                        const uint64_t *rank_first, const uint64_t *rank_count, void *stream,
                        lc_cut_shard **out, uint64_t *size_sum);
int lc_cut_shard_emit(lc_cut_shard *shard, int phase, uint64_t *d_send, uint64_t *counts, uint64_t *info);
int lc_cut_shard_apply(lc_cut_shard *shard, int phase, const uint64_t *d_recv, uint64_t n_messages);
int lc_cut_shard_finish(lc_cut_shard *shard, uint64_t *n_out);
int lc_cut_shard_destroy(lc_cut_shard *shard);

/* Replaces reduce.count_cycles (reduce.py:226-266): cycles of a permutation, sorted by
 * leader (smallest source on the cycle): hop count, clock length (sum of distances),
 * aggregate tree size (sum of subtree sizes).  Output arrays hold up to n entries. */
int lc_count_cycles(lc_ctx *ctx, uint64_t n, const uint64_t *src, const uint64_t *dst,
                    const uint64_t *dist, const uint64_t *subtree_size, uint64_t *leader,
                    uint64_t *hop_count, uint64_t *clock_length, uint64_t *tree_size,
                    uint64_t *n_cycles);

/* ------------------------- exhaustive mini-cipher analysis (oracle.py:141-283) */

/* The building blocks of the reference's ground-truth oracle brute_force_analysis, on
 * the GPU (device buffers, rank-encoded states as oracle.py:55-63).  n must be the spec's
 * valid state count (< 2^31).  build: successor ranks (majority rule, or every register
 * clocked when clock_all), in-degrees, candidate flags (R3 == F, successor's R3 != F,
 * in-degree > 0) and cycle_of[i] = f^(2^k)(i), an on-cycle state of i's component. */
int lc_bf_build_device(lc_ctx *ctx, const lc_spec *spec, uint64_t fixed_r3, int clock_all, uint64_t n,
                       int64_t *d_succ, int32_t *d_indeg, uint8_t *d_is_cand, int64_t *d_cycle_of,
                       void *stream);
/* Candidate-graph edges: each of the m candidate ranks walked through the successor map
 * to the first candidate (dst rank, distance). */
int lc_bf_edges_device(lc_ctx *ctx, uint64_t n, const int64_t *d_succ, const uint8_t *d_is_cand,
                       const int64_t *d_cand, uint64_t m, int64_t *d_dst, int64_t *d_dist, void *stream);
/* Segment sweep from the ascending candidate ranks: root[i] = index of i's candidate
 * (or -1), depth[i]; level_counts[l] = states at depth l (host array, level_cap entries;
 * *n_levels = levels found).  Synchronous. */
int lc_bf_segments_device(lc_ctx *ctx, uint64_t n, const int64_t *d_succ, const int32_t *d_indeg,
                          const uint8_t *d_is_cand, const int64_t *d_cand, uint64_t ncand, int64_t *d_root,
                          int32_t *d_depth, uint64_t *level_counts, uint32_t level_cap, uint32_t *n_levels,
                          void *stream);
/* The candidate ranks, ascending (ordered compaction of is_cand); *m_out = their count.
 * Synchronous. */
int lc_bf_candidates_device(lc_ctx *ctx, uint64_t n, const uint8_t *d_is_cand, int64_t *d_cand,
                            uint64_t *m_out, void *stream);
/* pred_hist[k] (5 entries, device) = states with k predecessors; per candidate index j <
 * m: seg_depth[j] = deepest level of its segment, seg_size[j] = its states (from the
 * segment sweep's root / depth). */
int lc_bf_summary_device(lc_ctx *ctx, uint64_t n, const int32_t *d_indeg, const int64_t *d_root,
                         const int32_t *d_depth, uint64_t m, uint64_t *d_pred_hist, int64_t *d_seg_depth,
                         int64_t *d_seg_size, void *stream);
/* The cycles of the functional graph (oracle.py:168-186, 254-283), from the successor map
 * and cycle_of (lc_bf_build_device).  Cycles are numbered by their smallest on-cycle rank
 * (ascending); cycle c's on-cycle ranks in walk order from that rank are
 * order[offset[c] .. offset[c] + length[c]); leader[c] = its smallest packed state,
 * cand_on[c] = candidates on it, comp[c] = states of its component.  Every output holds
 * n entries (only *n_on, resp. *n_cycles, are written).  Synchronous. */
int lc_bf_cycles_device(lc_ctx *ctx, const lc_spec *spec, uint64_t n, const int64_t *d_succ,
                        const int64_t *d_cycle_of, const uint8_t *d_is_cand, int64_t *d_order, int64_t *d_offset,
                        int64_t *d_length, int64_t *d_leader, int64_t *d_cand_on, int64_t *d_comp,
                        uint64_t *n_on, uint64_t *n_cycles, void *stream);
/* Cycles of a permutation of m compact indices (cs[i] = successor's index; indices in
 * ascending state order): start[i] = smallest index on i's cycle, steps[i] = steps from
 * i forward to it. */
int lc_bf_cycle_order_device(lc_ctx *ctx, uint64_t m, const int64_t *d_cs, int64_t *d_start,
                             int64_t *d_steps, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* LFSR_B200_H */
