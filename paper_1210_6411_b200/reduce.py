"""Steps 4-5 on the GPU: drop-in for ``lfsrcycles.reduce`` (reference
``pkg/src/lfsrcycles/reduce.py``) -- iterative leaf cutting of the skeleton-edge file to
its fixpoint and cycle counting -- plus the edge-output sort that precedes it
(SURVEY.md §8(f) ranks 1-2).

The whole edge list is held in HBM (SoA columns, csrc/reduce.cu) and leaf cutting runs
as a frontier computation (each pass touches only its own leaves) instead of external
sorts over files; the fixpoint records, cycle list and per-pass ``leaves_removed`` /
``inner_nodes`` / ``out_size_sum`` equal the reference's.  Differences, by design:

* ``cut_leaves_to_fixpoint`` checks the conservation invariant the reference intends
  (sum of subtree sizes + surviving records == input records + input sizes).  The
  reference's check (reduce.py:210-215) counts pass-1 leaves twice and raises
  ``AssertionError`` on every input whose first pass removes a leaf.
* ``PassStats.bytes_read`` / ``bytes_written`` count this implementation's file I/O
  (the edge file in, the result out), not the reference's external-sort spills.
* ``ReduceConfig.memory_budget`` is validated like the reference but not otherwise
  needed (no spills).
"""

from __future__ import annotations

import csv
import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple

import numpy as np

from . import _native as N
from .records import (EDGE_SIZE, ByteCounter, EdgeRecord, read_edge_arrays, read_edges,  # noqa: F401
                      write_edge_arrays, write_edges)  # (the last names re-exported as the reference's module does)

__all__ = ["ReduceConfig", "PassStats", "IterationLog", "CycleRecord", "cut_leaves_pass",
           "cut_leaves_to_fixpoint", "count_cycles", "NotAPermutationError", "sort_edge_arrays",
           "cut_leaves_arrays", "cut_leaves_tensors", "count_cycles_arrays"]

_MIN_BUDGET = 3 * (1 << 20)


class NotAPermutationError(ValueError):
    """Cycle counting ran on records that still contain tree edges (reduce.py:38)."""


@dataclass(frozen=True)
class ReduceConfig:
    memory_budget: int = 64 * (1 << 20)
    scratch_dir: str | None = None
    overlap_io: bool = False

    def validate(self) -> None:
        if self.memory_budget < _MIN_BUDGET:
            raise ValueError(f"memory budget below {_MIN_BUDGET} bytes (three 1 MiB sort buffers)")


@dataclass
class PassStats:
    leaves_removed: int = 0
    inner_nodes: int = 0
    bytes_read: int = 0
    bytes_written: int = 0
    out_size_sum: int = 0


@dataclass
class IterationLog:
    passes: list = field(default_factory=list)

    @property
    def iterations(self) -> int:
        """Passes that removed something; equals the maximum tree height."""
        return sum(1 for p in self.passes if p.leaves_removed > 0)

    @property
    def bytes_read(self) -> int:
        return sum(p.bytes_read for p in self.passes)

    @property
    def bytes_written(self) -> int:
        return sum(p.bytes_written for p in self.passes)

    def write_csv(self, path) -> None:
        with open(path, "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["iteration", "removed", "remaining", "bytes_read", "bytes_written"])
            for i, p in enumerate(self.passes, 1):
                w.writerow([i, p.leaves_removed, p.inner_nodes, p.bytes_read, p.bytes_written])


class CycleRecord(NamedTuple):
    leader: int
    hop_count: int
    clock_length: int
    aggregate_tree_size: int


def _cols(*arrays):
    return [np.ascontiguousarray(np.asarray(a, dtype=np.uint64)).copy() for a in arrays]


def _raise(rc: int):
    msg = N.last_error()
    if rc == N.LC_ERR_NOT_PERMUTATION:
        raise NotAPermutationError(msg)
    if rc in (N.LC_ERR_UNSORTED, N.LC_ERR_NOT_CLOSED, N.LC_ERR_ARG):
        raise ValueError(msg)
    raise N.NativeError(rc, msg)


def sort_edge_arrays(src, dst, dist, subtree_size=None, subtree_depth=None):
    """Edge-output stage: records sorted ascending by source on the GPU (radix sort)."""
    cols = _cols(src, dst, dist)
    extra = _cols(*(c for c in (subtree_size, subtree_depth) if c is not None))
    size = extra[0] if subtree_size is not None else None
    depth = extra[-1] if subtree_depth is not None else None
    n = cols[0].size
    ctx = N.context()
    rc = N.lib.lc_sort_edges(ctx.handle, n, *(N.u64p(c) for c in cols),
                             N.u64p(size) if size is not None else None,
                             N.u64p(depth) if depth is not None else None)
    if rc != N.LC_OK:
        _raise(rc)
    return tuple(cols) + tuple(c for c in (size, depth) if c is not None)


def cut_leaves_arrays(src, dst, dist, subtree_size, subtree_depth, *, max_passes: int = 0):
    """Leaf cutting on arrays (sorted by unique source).  max_passes = 1: one pass;
    0: to the fixpoint.  Returns (src, dst, dist, size, depth, [(leaves, inner, out_size_sum)])."""
    cap = 1 << 16  # per-pass statistics kept (the paper's A5/1 skeleton needs 88 passes)
    ctx = N.context()
    while True:  # a taller forest than `cap` passes: run again with room for every pass
        cols = _cols(src, dst, dist, subtree_size, subtree_depth)
        n = cols[0].size
        stats = np.zeros((cap, 3), dtype=np.uint64)
        npass = C.c_uint32(0)
        nout = C.c_uint64(0)
        rc = N.lib.lc_cut_leaves(ctx.handle, n, *(N.u64p(c) for c in cols), int(max_passes), N.u64p(stats), cap,
                                 C.byref(npass), C.byref(nout))
        if rc != N.LC_OK:
            _raise(rc)
        if int(npass.value) <= cap:
            break
        cap = int(npass.value)
    m = int(nout.value)
    passes = [tuple(r) for r in stats[: min(int(npass.value), cap)].tolist()]
    return tuple(c[:m] for c in cols) + (passes,)


def cut_leaves_tensors(src, dst, dist, subtree_size, subtree_depth, *, max_passes: int = 0):
    """Leaf cutting on device-resident torch columns (64-bit, contiguous, one CUDA device,
    sorted by unique source), in place on the current stream.  Returns (n_out, passes):
    the first n_out rows are the survivors."""
    import torch

    cols = (src, dst, dist, subtree_size, subtree_depth)
    dev = src.device
    for c in cols:
        if c.device != dev or c.device.type != "cuda" or c.element_size() != 8 or not c.is_contiguous():
            raise ValueError("columns must be contiguous 64-bit tensors on one CUDA device")
        if c.numel() != src.numel():
            raise ValueError("columns differ in length")
    cap = max(1, min(src.numel() + 2, 1 << 22))  # a forest of n records has at most n + 1 passes
    stats = np.zeros((cap, 3), dtype=np.uint64)
    npass = C.c_uint32(0)
    nout = C.c_uint64(0)
    ctx = N.context(dev.index)
    stream = torch.cuda.current_stream(dev).cuda_stream
    rc = N.lib.lc_cut_leaves_device(ctx.handle, src.numel(), *(c.data_ptr() for c in cols), int(max_passes),
                                    N.u64p(stats), cap, C.byref(npass), C.byref(nout), stream)
    if rc != N.LC_OK:
        _raise(rc)
    passes = [tuple(r) for r in stats[: min(int(npass.value), cap)].tolist()]
    return int(nout.value), passes


def count_cycles_arrays(src, dst, dist, subtree_size):
    """Cycles of a permutation given as arrays (any order; sorted on the GPU first)."""
    src, dst, dist, size = sort_edge_arrays(src, dst, dist, subtree_size)
    n = src.size
    out = [np.zeros(max(n, 1), dtype=np.uint64) for _ in range(4)]
    m = C.c_uint64(0)
    ctx = N.context()
    rc = N.lib.lc_count_cycles(ctx.handle, n, N.u64p(src), N.u64p(dst), N.u64p(dist), N.u64p(size),
                               *(N.u64p(o) for o in out), C.byref(m))
    if rc != N.LC_OK:
        _raise(rc)
    k = int(m.value)
    return tuple(o[:k] for o in out)


def _load(path):
    rec = read_edge_arrays(path)
    return (rec["source"], rec["destination"], rec["distance"], rec["subtree_size"], rec["subtree_depth"]), \
        rec.size * EDGE_SIZE


def cut_leaves_pass(in_path, out_path, config: ReduceConfig) -> PassStats:
    """One leaf-cutting iteration over an edge file (reduce.py:118-186)."""
    config.validate()
    cols, nbytes = _load(in_path)
    *out, passes = cut_leaves_arrays(*cols, max_passes=1)
    leaves, inner, out_sum = passes[0] if passes else (0, 0, 0)
    write_edge_arrays(out_path, *out)
    return PassStats(leaves_removed=leaves, inner_nodes=inner, bytes_read=nbytes,
                     bytes_written=out[0].size * EDGE_SIZE, out_size_sum=out_sum)


def cut_leaves_to_fixpoint(in_path, out_path, config: ReduceConfig) -> IterationLog:
    """Repeat leaf cutting until a pass removes nothing (reduce.py:189-223); the
    surviving records are exactly the on-cycle skeleton nodes."""
    config.validate()
    cols, nbytes = _load(in_path)
    expected = cols[0].size + int(cols[3].sum(dtype=np.uint64))
    *out, passes = cut_leaves_arrays(*cols, max_passes=0)
    log = IterationLog()
    for i, (leaves, inner, out_sum) in enumerate(passes):
        if out_sum + inner != expected:
            raise AssertionError("subtree size conservation violated")
        log.passes.append(PassStats(leaves_removed=leaves, inner_nodes=inner,
                                    bytes_read=nbytes if i == 0 else 0, out_size_sum=out_sum))
    write_edge_arrays(out_path, *out)
    if log.passes:
        log.passes[-1].bytes_written = out[0].size * EDGE_SIZE
    return log


def count_cycles(edges: Iterable[EdgeRecord] | str) -> list:
    """Partition a pure-cycle edge list into cycles (reduce.py:226-266), sorted."""
    if isinstance(edges, (str, os.PathLike)):
        rec = read_edge_arrays(edges)
        cols = (rec["source"], rec["destination"], rec["distance"], rec["subtree_size"])
    else:
        rows = list(edges)
        if not rows:
            return []
        arr = np.array(rows, dtype=np.uint64).reshape(-1, 5)
        cols = (arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3])
    if cols[0].size == 0:
        return []
    leader, hops, clocks, tree = count_cycles_arrays(*cols)
    return [CycleRecord(*r) for r in zip(leader.tolist(), hops.tolist(), clocks.tolist(), tree.tolist())]
