"""Multi-GPU leaf cutting (step 4): the reference's
``cut_leaves_pass`` / ``cut_leaves_to_fixpoint`` (reduce.py:118-223) over an edge list
partitioned across ranks, one process per GPU.

The records (sorted by unique source, records.py:3-5) are split into contiguous source
ranges, rank r holding the r-th range in its own HBM.  Unlike the walk, this step has a
real exchange: a record's destination can live on any rank.  Leaf cutting is run as a
frontier computation (csrc/reduce.cu): a record is a leaf of pass p iff its in-degree
among the records alive after pass p-1 is zero, so

* phase 0 -- every record sends one message to its destination's owner, which counts
  in-degrees;
* pass p -- every rank turns its current leaves into messages (destination, size + 1,
  depth + 1), the messages are exchanged by owner with one all-to-all, and each owner
  folds them into its records (atomic sum / max) and collects the records whose
  in-degree drops to zero: the leaves of pass p+1.

Per pass the host makes one all-gather of the per-owner message counts (it sizes the
all-to-all and carries the pass's global leaf count and error flags) and one
all-to-all of the messages -- NCCL over NVLink between GPUs, gloo in the CPU tests.
Pass statistics follow from the counts alone: inner_nodes = alive - leaves, and the
survivors' subtree-size sum grows by exactly the leaves removed.  The survivors end up
compacted in place on each rank (source order), so the concatenation over ranks is the
reference's output file.

The tail.  A frontier never grows, and random mappings spend thousands of passes on a
few leaves each, where the two collectives per pass are the whole cost.  Once a pass
removes at most ``TAIL_LEAVES`` records and at most ``TAIL_ALIVE`` are still alive,
every rank compacts its alive records (``lc_cut_shard_finish``), the alive records of
all ranks are all-gathered (they form a closed graph: a survivor's destination
survives), and every rank runs the single-GPU cut to the fixpoint on that copy
(``reduce.cut_leaves_tensors``, deterministic: atomic sums and maxima) and keeps the
survivors in its own source range.  Its pass statistics continue the global ones (its
alive count and size sum are the global ones).  One all-gather instead of two
collectives per remaining pass.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _native as N

__all__ = ["NativeShard", "cut_leaves_sharded", "shard_bounds"]

_U64 = (1 << 64) - 1
TAIL_LEAVES = 1 << 16
TAIL_ALIVE = 1 << 23


class NativeShard:
    """One rank's shard on its GPU (lc_cut_shard_* in include/lfsr_b200.h).  ``cols`` are
    contiguous 64-bit torch CUDA tensors (source, destination, distance, subtree_size,
    subtree_depth), updated in place."""

    def __init__(self, cols, n_ranks: int, rank_first, rank_count):
        import torch

        self.torch = torch
        self.cols = cols
        dev = cols[0].device
        for c in cols:
            if c.device != dev or dev.type != "cuda" or c.element_size() != 8 or not c.is_contiguous():
                raise ValueError("columns must be contiguous 64-bit tensors on one CUDA device")
        self.n = cols[0].numel()
        self.n_ranks = int(n_ranks)
        self.device = dev
        self.send = torch.empty((max(self.n, 1), 3), dtype=torch.int64, device=dev)
        first = np.ascontiguousarray(rank_first, dtype=np.uint64)
        count = np.ascontiguousarray(rank_count, dtype=np.uint64)
        ctx = N.context(dev.index)
        stream = torch.cuda.current_stream(dev).cuda_stream
        h = C.c_void_p()
        s = np.zeros(1, dtype=np.uint64)
        N.check(N.lib.lc_cut_shard_create(ctx.handle, self.n, *(c.data_ptr() for c in cols), self.n_ranks,
                                          N.u64p(first), N.u64p(count), stream, C.byref(h), N.u64p(s)))
        self.handle = h
        self.size_sum = int(s[0])
        self._counts = np.zeros(self.n_ranks, dtype=np.uint64)
        self._info = np.zeros(2, dtype=np.uint64)
        self.gathers_tail = True  # the driver may finish the cut on gathered records

    def emit(self, phase: int):
        """-> (messages [m, 3] grouped by owner, per-owner counts, records emitted, error word)."""
        rc = N.lib.lc_cut_shard_emit(self.handle, int(phase), self.send.data_ptr(), N.u64p(self._counts),
                                     N.u64p(self._info))
        N.check(rc)
        counts = self._counts.astype(np.int64)
        return self.send[: int(counts.sum())], counts, int(self._info[0]), int(self._info[1])

    def apply(self, phase: int, recv) -> None:
        if recv.device != self.device or not recv.is_contiguous():
            recv = recv.to(self.device).contiguous()
        N.check(N.lib.lc_cut_shard_apply(self.handle, int(phase), recv.data_ptr() if recv.numel() else None,
                                         recv.shape[0]))

    def finish(self):
        """-> (survivors, error code: 0 or N.LC_ERR_NOT_CLOSED)."""
        out = np.zeros(1, dtype=np.uint64)
        rc = N.lib.lc_cut_shard_finish(self.handle, N.u64p(out))
        if rc == N.LC_ERR_NOT_CLOSED:
            return self.n, rc
        N.check(rc)
        return int(out[0]), 0

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib.lc_cut_shard_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Exchange:
    """torch.distributed plumbing: all-gather of small int64 vectors and the per-pass
    all-to-all of [m, 3] int64 message tensors (staged through host memory when the
    backend cannot move device tensors, i.e. gloo)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.torch, self.dist, self.group = torch, dist, group
        # with a process group (even of one rank) every exchange is a real collective;
        # without one the exchanges are identities
        self.solo = not (dist.is_available() and dist.is_initialized())
        if not self.solo:
            self.world = dist.get_world_size(group)
            self.rank = dist.get_rank(group)
            self.nccl = dist.get_backend(group) == "nccl"
        else:
            self.world, self.rank, self.nccl = 1, 0, False

    def allgather(self, vec) -> np.ndarray:
        v = np.asarray(vec, dtype=np.int64)
        if self.solo:
            return v[None, :].copy()
        torch = self.torch
        dev = torch.device("cuda", torch.cuda.current_device()) if self.nccl else torch.device("cpu")
        t = torch.from_numpy(v).to(dev)
        out = [torch.empty_like(t) for _ in range(self.world)]
        self.dist.all_gather(out, t, group=self.group)
        return np.stack([o.cpu().numpy() for o in out])

    def alltoallv(self, send, send_counts, recv_counts):
        if self.solo:
            return send
        torch = self.torch
        staged = send.is_cuda and not self.nccl
        src = send.cpu() if staged else send
        recv = torch.empty((int(np.sum(recv_counts)), 3), dtype=torch.int64, device=src.device)
        self.dist.all_to_all_single(recv, src.contiguous(), [int(c) for c in recv_counts],
                                    [int(c) for c in send_counts], group=self.group)
        return recv.to(send.device) if staged else recv

    def allgather_rows(self, rows, counts):
        """Every rank's [counts[r], k] int64 rows, concatenated in rank order."""
        if self.solo:
            return rows
        torch = self.torch
        staged = rows.is_cuda and not self.nccl
        src = rows.cpu() if staged else rows
        width, top = src.shape[1], int(max(counts))
        pad = torch.zeros((top, width), dtype=torch.int64, device=src.device)
        pad[: src.shape[0]] = src
        out = [torch.empty_like(pad) for _ in range(self.world)]
        self.dist.all_gather(out, pad, group=self.group)
        cat = torch.cat([o[: int(c)] for o, c in zip(out, counts)])
        return cat.to(rows.device) if staged else cat


def _u64(x) -> int:
    return int(x) & _U64


def shard_bounds(first_last_count: np.ndarray):
    """Check that the ranks' source ranges ascend (non-empty ranks only) and return
    (rank_first, rank_count) as uint64 arrays."""
    first = np.array([_u64(r[0]) for r in first_last_count], dtype=np.uint64)
    last = [_u64(r[1]) for r in first_last_count]
    count = np.array([int(r[2]) for r in first_last_count], dtype=np.uint64)
    prev = None
    for r in range(len(count)):
        if count[r] == 0:
            continue
        if prev is not None and int(first[r]) <= prev:
            raise ValueError("edge records are not sorted by unique source across ranks")
        prev = last[r]
    return first, count


def _signed(v: int) -> int:
    v &= _U64
    return v - (1 << 64) if v >> 63 else v


def cut_leaves_sharded(src, dst, dist, subtree_size, subtree_depth, *, max_passes: int = 0, group=None,
                       shard_factory=None):
    """Leaf cutting of this rank's shard of a globally source-sorted edge list, in place.

    Collective over ``group`` (every rank calls it with its own contiguous source range;
    works without an initialised process group as a single shard).  ``max_passes`` 1 is
    ``cut_leaves_pass``, 0 runs to the fixpoint.  Returns (n_out, passes): this rank's
    survivors are the first n_out rows; ``passes`` is the global
    [(leaves_removed, inner_nodes, out_size_sum)] per pass, identical on every rank and
    equal to the single-GPU / reference statistics.  Raises ValueError (on every rank)
    if the input is not sorted or a removed leaf's destination has no record.
    """
    ex = _Exchange(group)
    cols = (src, dst, dist, subtree_size, subtree_depth)
    n = int(src.shape[0])
    ends = (_signed(int(src[0])), _signed(int(src[-1]))) if n else (0, 0)
    table = ex.allgather([ends[0], ends[1], n])
    first, count = shard_bounds(table)
    factory = shard_factory or NativeShard
    shard, failure = None, None
    try:
        shard = factory(cols, ex.world, first, count)
    except (ValueError, N.NativeError) as e:  # e.g. unsorted within a shard
        failure = e
    if ex.allgather([failure is not None]).any():  # fail on every rank, not just one
        if shard is not None:
            shard.close()
        raise ValueError(f"sharded leaf cutting: {failure or 'another rank rejected its shard'}")
    try:
        return _drive(ex, shard, cols, int(count.sum()), max_passes)
    finally:
        shard.close()


def _drive(ex, shard, cols, total: int, max_passes: int):
    W = ex.world
    # phase 0: in-degrees
    send, counts, _, err = shard.emit(0)
    mat = ex.allgather(list(counts) + [err, shard.size_sum])
    if mat[:, W].any():
        raise ValueError("edge records are not sorted by unique source")
    s = sum(_u64(v) for v in mat[:, W + 1]) & _U64
    shard.apply(0, ex.alltoallv(send, counts, mat[:, ex.rank]))
    alive = total
    passes = []
    p = 0
    while True:
        p += 1
        send, counts, leaves, err = shard.emit(1)
        mat = ex.allgather(list(counts) + [leaves, err])
        if mat[:, W + 1].any():  # a fold of the previous pass found no record
            raise ValueError("a removed leaf's destination has no surviving record; input was not closed")
        shard.apply(1, ex.alltoallv(send, counts, mat[:, ex.rank]))
        removed = int(mat[:, W].sum())
        passes.append((removed, alive - removed, (s + removed) & _U64))
        alive -= removed
        s = (s + removed) & _U64
        if removed == 0 or (max_passes and p >= max_passes):
            break
        if (not max_passes and getattr(shard, "gathers_tail", False) and removed <= TAIL_LEAVES
                and 0 < alive <= TAIL_ALIVE and os.environ.get("LFSR_SHARD_TAIL", "1") != "0"):
            return _gathered_tail(ex, shard, cols, passes, alive)
    n_out, rc = shard.finish()
    flags = ex.allgather([rc])
    if flags.any():
        raise ValueError("a removed leaf's destination has no surviving record; input was not closed")
    return n_out, passes


def _gathered_tail(ex, shard, cols, passes, alive: int):
    """Finish the cut on the all-gathered alive records (module docstring, "The tail")."""
    import torch

    from .reduce import cut_leaves_tensors

    n_loc, rc = shard.finish()  # this rank's alive records, compacted to the front in source order
    mat = ex.allgather([rc, n_loc])
    if mat[:, 0].any():
        raise ValueError("a removed leaf's destination has no surviving record; input was not closed")
    counts = mat[:, 1]
    if int(counts.sum()) != alive:
        raise RuntimeError(f"sharded leaf cutting: {int(counts.sum())} alive records gathered, {alive} expected")
    rows = ex.allgather_rows(torch.stack([c[:n_loc] for c in cols], 1), counts)
    g = [rows[:, k].contiguous() for k in range(5)]
    try:
        n_fix, tail = cut_leaves_tensors(*g)
    except ValueError as e:  # every rank runs the same cut: all of them raise
        raise ValueError(f"a removed leaf's destination has no surviving record; input was not closed ({e})") from e
    passes.extend(tail)
    # the gathered survivors stay in source order: this rank's are the run between its own
    # first and last alive source (located on the host: the fixpoint set is small)
    if not n_loc or not n_fix:
        return 0, passes
    surv = g[0][:n_fix].cpu().numpy().view(np.uint64)
    ends = cols[0][[0, n_loc - 1]].cpu().numpy().view(np.uint64)
    a = int(np.searchsorted(surv, ends[0], side="left"))
    b = int(np.searchsorted(surv, ends[1], side="right"))
    for k in range(5):
        cols[k][: b - a] = g[k][a:b]
    return b - a, passes
