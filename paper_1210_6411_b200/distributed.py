"""Multi-GPU sharding of the chain walk.

Walks are independent, so start indices are split into contiguous equal shards, one per
rank (one process per GPU).  There is no collective on the data path: each rank walks
its shard and keeps its edges.  The only exchange is one all-reduce of the integer
statistics block (edge count, transitions, min/max, exact sum of squares, chain-length
histogram) -- NCCL over NVLink on GPUs, gloo in the CPU tests.  Results are identical
to a single-rank run over the concatenated shards.
"""

from __future__ import annotations

import numpy as np

from . import _native as N

__all__ = ["shard_range", "combine_stats", "allreduce_stats", "stats_summary"]

_MASK32 = (1 << 32) - 1


def shard_range(n: int, rank: int, world: int) -> tuple:
    """Contiguous shard [lo, hi) of n items for rank r of world ranks (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def _limbs(stats: np.ndarray) -> np.ndarray:
    """u128 sum of squares -> four 32-bit limbs (summable across < 2^31 ranks)."""
    lo, hi = int(stats[N.ST_SQ_LO]), int(stats[N.ST_SQ_HI])
    v = (hi << 64) | lo
    return np.array([(v >> (32 * i)) & _MASK32 for i in range(4)], dtype=np.int64)


def _from_limbs(limbs) -> tuple:
    v = sum(int(x) << (32 * i) for i, x in enumerate(limbs))
    return v & ((1 << 64) - 1), (v >> 64) & ((1 << 64) - 1)


_NO_ERROR = (1 << 64) - 1


def _error_key(stats: np.ndarray, offset: int) -> int:
    """(global start index, error code) of a block as one orderable key: the smallest
    key over the shards is the first failing start and its own code (the code and the
    index are never taken from different shards)."""
    code = int(stats[N.ST_ERROR])
    if not code:
        return _NO_ERROR
    return ((int(stats[N.ST_ERROR_INDEX]) + int(offset)) << 8) | (code & 0xFF)


def _apply_error_key(out: np.ndarray, key: int) -> None:
    if key == _NO_ERROR:
        out[N.ST_ERROR], out[N.ST_ERROR_INDEX] = 0, np.uint64(_NO_ERROR)
    else:
        out[N.ST_ERROR], out[N.ST_ERROR_INDEX] = key & 0xFF, key >> 8


def combine_stats(blocks, offsets=None) -> np.ndarray:
    """Host reduction of per-shard statistics blocks (same rule as allreduce_stats).
    offsets[i] = global index of shard i's first start (its ST_ERROR_INDEX is local)."""
    blocks = [np.asarray(b, dtype=np.uint64) for b in blocks]
    offsets = [0] * len(blocks) if offsets is None else list(offsets)
    out = blocks[0].copy()
    key = _error_key(blocks[0], offsets[0])
    for b, o in zip(blocks[1:], offsets[1:]):
        for i in (N.ST_EDGES, N.ST_TRANSITIONS):
            out[i] = np.uint64((int(out[i]) + int(b[i])) & ((1 << 64) - 1))
        out[N.ST_MIN] = min(out[N.ST_MIN], b[N.ST_MIN])
        out[N.ST_MAX] = max(out[N.ST_MAX], b[N.ST_MAX])
        key = min(key, _error_key(b, o))
        out[N.ST_HEADER:] += b[N.ST_HEADER:]
    _apply_error_key(out, key)
    limbs = sum(_limbs(b) for b in blocks)
    out[N.ST_SQ_LO], out[N.ST_SQ_HI] = _from_limbs(limbs)
    return out


def allreduce_stats(stats: np.ndarray, group=None, offset: int = 0) -> np.ndarray:
    """All-reduce one rank's statistics block with torch.distributed (NCCL on CUDA
    tensors when the default backend is NCCL, gloo otherwise).  ``offset`` = global
    index of this rank's first start (ST_ERROR_INDEX is shard-local).  Returns the global
    block on every rank."""
    import torch
    import torch.distributed as dist

    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    s = np.asarray(stats, dtype=np.uint64)
    # sums: counters, histogram, u128 limbs (as int64; values < 2^63 per rank)
    sums = np.concatenate([s[[N.ST_EDGES, N.ST_TRANSITIONS]].astype(np.int64), _limbs(s),
                           s[N.ST_HEADER:].astype(np.int64)])
    t_sum = torch.from_numpy(sums).to(dev)
    dist.all_reduce(t_sum, op=dist.ReduceOp.SUM, group=group)
    # min / max (unsigned values mapped to order-preserving int64)
    flip = np.uint64(1 << 63)
    key = np.array([_error_key(s, offset)], dtype=np.uint64)
    mins = (np.concatenate([s[[N.ST_MIN]], key]) ^ flip).view(np.int64)
    maxs = (s[[N.ST_MAX]] ^ flip).view(np.int64)
    t_min = torch.from_numpy(mins.copy()).to(dev)
    t_max = torch.from_numpy(maxs.copy()).to(dev)
    dist.all_reduce(t_min, op=dist.ReduceOp.MIN, group=group)
    dist.all_reduce(t_max, op=dist.ReduceOp.MAX, group=group)
    sums = t_sum.cpu().numpy()
    out = s.copy()
    out[N.ST_EDGES], out[N.ST_TRANSITIONS] = sums[0], sums[1]
    out[N.ST_SQ_LO], out[N.ST_SQ_HI] = _from_limbs(sums[2:6])
    out[N.ST_HEADER:] = sums[6:].astype(np.uint64)
    mn = t_min.cpu().numpy().view(np.uint64) ^ flip
    mx = t_max.cpu().numpy().view(np.uint64) ^ flip
    out[N.ST_MIN] = mn[0]
    _apply_error_key(out, int(mn[1]))
    out[N.ST_MAX] = mx[0]
    return out


def stats_summary(stats: np.ndarray) -> dict:
    """Edges, transitions, mean, standard deviation and range from a statistics block."""
    s = np.asarray(stats, dtype=np.uint64)
    e = int(s[N.ST_EDGES])
    tr = int(s[N.ST_TRANSITIONS])
    lo = int(s[N.ST_HIST_LO])
    sq = (int(s[N.ST_SQ_HI]) << 64) | int(s[N.ST_SQ_LO])
    out = {"edges": e, "transitions": tr}
    if e:
        mean = tr / e
        # sum (d - lo)^2 = sum (d - mean)^2 + e (mean - lo)^2
        var = max(0.0, sq / e - (mean - lo) ** 2)
        out.update(mean=mean, sd=var ** 0.5, min=int(s[N.ST_MIN]), max=int(s[N.ST_MAX]))
    return out
