"""Steps 1-3 orchestration: drop-in for ``lfsrcycles.pipeline`` (reference
``pkg/src/lfsrcycles/pipeline.py``).

* ``enumerate_candidates`` -- step 1 on the GPU (K2 closed-form writer), ascending.
* ``prune_shallow_segments`` -- step 2 on the GPU (K3 reverse DFS with a pending-branch ring); the
  survivor list, ``removed`` and the order-dependent ``expanded`` counter match the
  reference exactly.
* ``build_skeleton_edges`` -- step 3: the GPU chain walk plus a GPU closure check.
* ``probe_segment`` / ``auto_depth_limit`` -- level-order segment sweeps, one batched GPU
  predecessor/predicate pass per level.
* ``random_candidate`` -- the reference's seeded scalar sampler (same stream of states
  for the same ``random.Random``); ``random_candidates_gpu`` is the counter-based K0
  generator used for large synthetic start sets.
"""

from __future__ import annotations

import ctypes as C
import os
import random
from dataclasses import dataclass
from typing import Iterable, Iterator

import numpy as np

from . import _batch
from . import _native as N
from .bitslice import forward_to_candidate
from .cipher import (CandidateParams, CipherSpec, PredecessorTable, is_candidate,  # noqa: F401  (names the
                     predecessors, shared_table, unrank_state)  # reference's module also exposes)
from .records import EdgeRecord

__all__ = [
    "PruneConfig", "PruneStats", "PruneSoundnessError", "enumerate_candidates",
    "enumerate_candidates_array", "prune_shallow_segments", "build_skeleton_edges",
    "probe_segment", "probe_segments", "auto_depth_limit", "random_candidate",
    "random_candidates_gpu", "reference_candidates", "reference_candidate_streams",
]

_PRUNE_CHUNK_GPU = 1 << 25  # candidates per kernel launch: large, so the tail of the longest traversals amortises
_ENUM_ROWS_PER_CALL = 1 << 12


class PruneSoundnessError(RuntimeError):
    """A surviving node's forward walk hit a pruned candidate (pipeline.py:45-47)."""


@dataclass(frozen=True)
class PruneConfig:
    """Bounded reverse traversal settings (pipeline.py:50-84).  ``workers`` (the
    reference's process-pool size) is the number of GPUs the prune may spread over."""

    mode: str = "dfs"
    depth_limit: int | None = None
    node_limit: int | None = None
    workers: int = 1

    def validate(self, spec: CipherSpec) -> None:
        bound = (1 << spec.lengths[2]) - 1
        if self.mode == "dfs":
            if not self.depth_limit or self.depth_limit < 1:
                raise ValueError("dfs mode needs a positive depth_limit")
            if self.depth_limit >= bound:
                raise ValueError(f"depth_limit {self.depth_limit} must stay below the minimum "
                                 f"candidate spacing {bound}")
        elif self.mode == "bfs":
            if not self.node_limit or self.node_limit < 1:
                raise ValueError("bfs mode needs a positive node_limit")
            if self.node_limit >= bound:
                raise ValueError(f"node_limit {self.node_limit} must stay below the minimum "
                                 f"candidate spacing {bound}")
        else:
            raise ValueError(f"unknown prune mode {self.mode!r}")
        if self.workers < 1:
            raise ValueError("workers must be >= 1")


@dataclass
class PruneStats:
    mode: str
    limit: int
    total: int = 0
    removed: int = 0
    expanded: int = 0

    @property
    def surviving(self) -> int:
        return self.total - self.removed

    @property
    def removed_fraction(self) -> float:
        return self.removed / self.total if self.total else 0.0


# ----------------------------------------------------------------------- step 1


def enumerate_candidates_array(spec: CipherSpec, params: CandidateParams, r2_lo: int = 1,
                               r2_hi: int | None = None) -> np.ndarray:
    """Special nodes with R2 in [r2_lo, r2_hi) (default: all), ascending, as uint64."""
    if r2_hi is None:
        r2_hi = spec.reg_masks[1] + 1
    parts = [_batch.enumerate_rows(spec, params, lo, min(r2_hi, lo + _ENUM_ROWS_PER_CALL))
             for lo in range(r2_lo, r2_hi, _ENUM_ROWS_PER_CALL)]
    return np.concatenate(parts) if parts else np.zeros(0, dtype=np.uint64)


def enumerate_candidates(spec: CipherSpec, params: CandidateParams,
                         table: PredecessorTable | None = None) -> Iterator[int]:
    """All candidates in ascending packed order (pipeline.py:104-118), produced on the
    GPU a block of R2 rows at a time."""
    r2_hi = spec.reg_masks[1] + 1
    for lo in range(1, r2_hi, _ENUM_ROWS_PER_CALL):
        rows = _batch.enumerate_rows(spec, params, lo, min(r2_hi, lo + _ENUM_ROWS_PER_CALL))
        yield from rows.tolist()


# ----------------------------------------------------------------------- step 2


def prune_shallow_segments(candidates: Iterable[int], config: PruneConfig, spec: CipherSpec,
                           params: CandidateParams,
                           table: PredecessorTable | None = None, *, devices: list | None = None) -> tuple:
    """Drop candidates rooting shallow segments; survivors keep input order
    (pipeline.py:192-222).  ``config.workers`` (the reference's process-pool size) spreads
    contiguous chunks over up to that many GPUs of this process (or over ``devices``)."""
    config.validate(spec)
    limit = config.depth_limit if config.mode == "dfs" else config.node_limit
    stats = PruneStats(mode=config.mode, limit=limit)
    cands = np.asarray(candidates if isinstance(candidates, np.ndarray) else list(candidates),
                       dtype=np.uint64)
    if devices is None:
        devices = list(range(max(1, min(int(config.workers), N.device_count()))))
    chunks = [cands[lo: lo + _PRUNE_CHUNK_GPU] for lo in range(0, cands.size, _PRUNE_CHUNK_GPU)]
    if len(devices) > 1 and len(chunks) == 1 and cands.size >= 2 * len(devices):
        chunks = np.array_split(cands, len(devices))

    def run(i):
        return _batch.prune(chunks[i], spec, params, config.mode, limit, device=devices[i % len(devices)])

    if len(devices) > 1 and len(chunks) > 1:
        from concurrent.futures import ThreadPoolExecutor

        with ThreadPoolExecutor(len(devices)) as ex:  # one thread (and context) per device
            results = list(ex.map(run, range(len(chunks))))
    else:
        results = [run(i) for i in range(len(chunks))]
    survivors = []
    for chunk, (removed, work) in zip(chunks, results):
        survivors.append(chunk[~removed])
        stats.total += chunk.size
        stats.removed += int(removed.sum())
        stats.expanded += int(work.sum())
    out = np.concatenate(survivors) if survivors else np.zeros(0, dtype=np.uint64)
    return out.tolist(), stats


# ----------------------------------------------------------------------- step 3


def _edges_chunk(args) -> list:
    """The reference's pickled unit of step-3 work (pipeline.py:225-228)."""
    chunk, params, spec, table, stride = args
    walked = forward_to_candidate(chunk, params, spec, table, stride=stride)
    return [(src, dest, dist) for src, (dest, dist) in zip(chunk, walked)]


def _walk_sharded(sk: np.ndarray, params, spec, stride: int, devices: list):
    """Contiguous shards walked concurrently, one host thread (and native context) per
    device; results in input order."""
    from concurrent.futures import ThreadPoolExecutor

    shards = np.array_split(sk, len(devices))

    def run(i):
        return _batch.walk(shards[i], params, spec, stride=stride, legs=1, device=devices[i])

    with ThreadPoolExecutor(len(devices)) as ex:  # ctypes releases the GIL in lc_walk
        parts = list(ex.map(run, range(len(devices))))
    return (np.concatenate([r.dst[:, 0] for r in parts]), np.concatenate([r.dist[:, 0] for r in parts]))


def build_skeleton_edges(skeleton: list, params: CandidateParams, spec: CipherSpec,
                         table: PredecessorTable | None = None, stride: int = 1,
                         workers: int = 1, *, devices: list | None = None) -> list:
    """One weighted edge per skeleton node (pipeline.py:231-256); every destination
    must be in the skeleton, else PruneSoundnessError.  ``workers`` (the reference's
    process-pool size, pipeline.py:244-249) spreads contiguous shards over up to that
    many GPUs of this process (or over ``devices``); the order is the input order."""
    sk = np.asarray(skeleton if isinstance(skeleton, np.ndarray) else list(skeleton), dtype=np.uint64)
    if sk.size == 0:
        raise ValueError("skeleton is empty")
    if devices is None:
        devices = list(range(max(1, min(int(workers), N.device_count()))))
    if len(devices) > 1:
        dst, dist = _walk_sharded(sk, params, spec, stride, devices)
    else:
        res = _batch.walk(sk, params, spec, stride=stride, legs=1, device=devices[0])
        dst, dist = res.dst[:, 0], res.dist[:, 0]
    bad = _batch.first_missing(np.unique(sk), dst)
    if bad < sk.size:
        raise PruneSoundnessError(
            f"walk from {int(sk[bad]):#x} reached pruned candidate {int(dst[bad]):#x}; "
            "prune limit exceeded the minimum candidate spacing")
    return [EdgeRecord(s, d, w, 0, 0) for s, d, w in zip(sk.tolist(), dst.tolist(), dist.tolist())]


# ----------------------------------------------------------------------- probing


def probe_segments(roots, spec: CipherSpec, params: CandidateParams, *, depth_cap: int | None = None,
                   node_cap: int | None = None, level_counts: list | None = None):
    """Batched probe_segment (pipeline.py:262-298): per root (depth, nodes, censored)
    arrays.  The sweeps run device-resident (lc_probe_segments: one expand and one
    finalize launch per level for all roots); ``level_counts`` accumulates nodes per
    depth level summed over the roots (index 0 counts the roots)."""
    roots = np.ascontiguousarray(np.asarray(roots, dtype=np.uint64).reshape(-1))
    k = roots.size
    depth = np.zeros(k, dtype=np.uint64)
    nodes = np.ones(k, dtype=np.uint64)
    censored = np.zeros(k, dtype=np.uint8)
    if k == 0:
        return depth.astype(np.int64), nodes.astype(np.int64), censored.astype(bool)
    cap_levels = (int(depth_cap) + 1) if depth_cap is not None else 1 << 20
    cap_levels = max(1, min(cap_levels, 1 << 24))
    levels = np.zeros(cap_levels, dtype=np.uint64)
    ctx = N.context()
    N.check(N.lib.lc_probe_segments(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3, N.u64p(roots), k,
                                    -1 if depth_cap is None else int(depth_cap),
                                    -1 if node_cap is None else int(node_cap), N.u64p(depth), N.u64p(nodes),
                                    censored.ctypes.data_as(C.POINTER(C.c_uint8)), N.u64p(levels), cap_levels))
    depth = depth.astype(np.int64)
    if level_counts is not None:
        top = int(depth.max()) + 1
        if top > cap_levels:
            raise ValueError("segment deeper than the level-count buffer (pass a depth_cap)")
        while len(level_counts) < top:
            level_counts.append(0)
        for lv in range(top):
            level_counts[lv] += int(levels[lv])
    return depth, nodes.astype(np.int64), censored.astype(bool)


def probe_segment(root: int, spec: CipherSpec, params: CandidateParams,
                  table: PredecessorTable | None = None, *, depth_cap: int | None = None,
                  node_cap: int | None = None, level_counts: list | None = None) -> tuple:
    """Reverse level-order sweep of one segment (pipeline.py:262-298):
    (deepest level, nodes seen, censored)."""
    d, n, c = probe_segments([root], spec, params, depth_cap=depth_cap, node_cap=node_cap,
                             level_counts=level_counts)
    return int(d[0]), int(n[0]), bool(c[0])


def random_candidate(rng: random.Random, spec: CipherSpec, params: CandidateParams,
                     table: PredecessorTable | None = None) -> int:
    """Uniform candidate by rejection over the fixed-R3 plane (pipeline.py:301-310);
    consumes ``rng`` exactly like the reference, so seeds give the same states."""
    m1, m2, _ = spec.reg_masks
    o2 = spec.offsets[1]
    table = table or shared_table()
    while True:
        x = rng.randrange(1, m1 + 1) | (rng.randrange(1, m2 + 1) << o2) | params.packed_r3
        if is_candidate(x, params, spec, table):
            return x


def reference_candidates(spec: CipherSpec, params: CandidateParams, seed: int, n: int) -> np.ndarray:
    """``[random_candidate(rng, spec, params) for _ in range(n)]`` with
    ``rng = random.Random(seed)`` (pipeline.py:301-310), as a u64 array: the same states
    in the same order, from a native restatement of CPython's MT19937 / ``randrange``
    stream (``csrc/sampler.cu``; ~50 M states/s instead of ~65 k/s).  Configs 1 and 2 are
    ``seed=0`` with n = 2^16 and 2^24."""
    if seed < 0 or seed >= 1 << 64:
        raise ValueError("seed must be a non-negative 64-bit integer")
    out = np.empty(int(n), dtype=np.uint64)
    N.check(N.lib.lc_reference_candidates(C.byref(N.spec_struct(spec)), params.fixed_r3, int(seed), int(n),
                                          N.u64p(out), None))
    return out


def reference_candidate_streams(spec: CipherSpec, params: CandidateParams, seeds, n_each: int,
                                threads: int | None = None) -> np.ndarray:
    """``reference_candidates`` for several seeds at once (one host thread per stream, up
    to ``threads``): row i of the result is ``reference_candidates(..., seeds[i], n_each)``."""
    seeds = np.ascontiguousarray(np.asarray(seeds, dtype=np.uint64))
    out = np.empty((seeds.size, int(n_each)), dtype=np.uint64)
    threads = threads or len(os.sched_getaffinity(0))
    N.check(N.lib.lc_reference_candidates_multi(C.byref(N.spec_struct(spec)), params.fixed_r3, N.u64p(seeds),
                                                seeds.size, int(n_each), N.u64p(out), int(threads)))
    return out


def random_candidates_gpu(spec: CipherSpec, params: CandidateParams, seed: int, n: int) -> np.ndarray:
    """K0 seeded synthetic start set: the first n candidates of the counter-based trial
    stream, generated and filtered on the GPU."""
    return _batch.random_candidates(spec, params, seed, n)


def auto_depth_limit(spec: CipherSpec, params: CandidateParams, table: PredecessorTable | None = None, *,
                     sample: int = 256, seed: int = 0) -> int:
    """75th-percentile sampled segment depth, clamped under the spacing bound
    (pipeline.py:313-333)."""
    bound = (1 << spec.lengths[2]) - 2
    rng = random.Random(seed)
    roots = [random_candidate(rng, spec, params, table) for _ in range(sample)]
    depths, _, _ = probe_segments(roots, spec, params, depth_cap=bound, node_cap=200_000)
    depths = sorted(int(d) for d in depths)
    return max(4, min(depths[(3 * len(depths)) // 4], bound))
