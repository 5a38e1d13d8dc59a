"""Test-only numpy stand-in for one rank's NativeShard (the lc_cut_shard_* contract in
include/lfsr_b200.h), so the multi-rank driver in sharded_reduce.py can run under gloo in
this GPU-less container.  It is never used by the package."""

from __future__ import annotations

import numpy as np
import torch

LC_ERR_NOT_CLOSED = -8


class NumpyShard:
    gathers_tail = False  # NumpyShardTail: let the driver finish on the gathered records

    def __init__(self, cols, n_ranks, rank_first, rank_count):
        self.cols = [c.numpy().view(np.uint64) for c in cols]  # shares memory with the tensors
        self.src, self.dst, _, self.size, self.depth = self.cols
        self.n = self.src.size
        if self.n > 1 and not (self.src[1:] > self.src[:-1]).all():
            raise ValueError("edge records are not sorted by unique source")
        self.n_ranks = n_ranks
        ranks = [r for r in range(n_ranks) if rank_count[r]] or [0]
        self.bounds = np.array([0] + [int(rank_first[r]) for r in ranks[1:]], dtype=np.uint64)
        self.brank = np.array(ranks, dtype=np.int64)
        self.indeg = np.zeros(self.n, dtype=np.int64)
        self.alive = np.ones(self.n, dtype=bool)
        self.frontier = None
        self.err = 0
        self.size_sum = int(self.size.sum(dtype=np.uint64))

    def _owner(self, v):
        return self.brank[np.searchsorted(self.bounds, v, side="right") - 1]

    def emit(self, phase):
        if phase and self.frontier is None:
            self.frontier = np.nonzero(self.indeg == 0)[0]
        items = np.arange(self.n) if phase == 0 else self.frontier
        d = self.dst[items]
        o = self._owner(d)
        msgs = np.zeros((items.size, 3), dtype=np.uint64)
        msgs[:, 0] = d
        if phase:
            msgs[:, 1] = self.size[items] + np.uint64(1)
            msgs[:, 2] = self.depth[items] + np.uint64(1)
            self.alive[items] = False
        order = np.argsort(o, kind="stable")
        counts = np.bincount(o, minlength=self.n_ranks).astype(np.int64)
        return torch.from_numpy(msgs[order].view(np.int64)), counts, int(items.size), self.err

    def apply(self, phase, recv):
        m = recv.numpy().view(np.uint64).reshape(-1, 3)
        v = m[:, 0]
        j = np.searchsorted(self.src, v)
        jc = np.minimum(j, max(self.n - 1, 0))
        found = (j < self.n) & (self.src[jc] == v) if self.n else np.zeros(v.size, dtype=bool)
        jj = j[found]
        if phase == 0:
            np.add.at(self.indeg, jj, 1)
            return
        if not found.all():
            self.err = 2
        np.add.at(self.size, jj, m[found, 1])
        np.maximum.at(self.depth, jj, m[found, 2])
        np.subtract.at(self.indeg, jj, 1)
        touched = np.unique(jj)
        self.frontier = touched[self.indeg[touched] == 0]

    def finish(self):
        if self.err:
            return self.n, LC_ERR_NOT_CLOSED
        k = int(self.alive.sum())
        for c in self.cols:
            c[:k] = c[self.alive]
        return k, 0

    def close(self):
        pass


class NumpyShardTail(NumpyShard):
    gathers_tail = True


def numpy_cut_leaves_tensors(src, dst, dist, subtree_size, subtree_depth, *, max_passes=0):
    """Stand-in for reduce.cut_leaves_tensors on CPU tensors (the reduce oracle, in place)."""
    from oracle import reduce_np

    cols = [t.numpy().view(np.uint64) for t in (src, dst, dist, subtree_size, subtree_depth)]
    res = reduce_np.cut_leaves(*cols, max_passes=max_passes)
    n = res[0].size
    for c, r in zip(cols, res[:5]):
        c[:n] = r
    return n, [tuple(int(v) for v in p) for p in res[5]]
