"""World-size-2 gloo run of the multi-rank path on CPU: contiguous shards, per-rank
walks (computed by the C oracle here -- no GPU in this container), one all-reduce of the
statistics block.  The reduced block must equal the single-rank block and the
concatenated shard edges must equal the unsharded walk."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import golden_npz


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stats_block(dist, lo, bins):
    from paper_1210_6411_b200 import _native as N

    s = np.zeros(N.ST_HEADER + bins + 2, dtype=np.uint64)
    s[N.ST_MIN] = np.uint64((1 << 64) - 1)
    s[N.ST_ERROR_INDEX] = np.uint64((1 << 64) - 1)
    s[N.ST_HIST_LO] = lo
    s[N.ST_HIST_BINS] = bins
    if dist.size:
        s[N.ST_EDGES] = dist.size
        s[N.ST_TRANSITIONS] = int(dist.sum())
        s[N.ST_MIN], s[N.ST_MAX] = dist.min(), dist.max()
        sq = sum((int(x) - lo) ** 2 for x in dist)
        s[N.ST_SQ_LO], s[N.ST_SQ_HI] = sq & ((1 << 64) - 1), sq >> 64
        b = np.clip(dist.astype(np.int64) - lo, -1, bins) + 1
        s[N.ST_HEADER:] = np.bincount(b, minlength=bins + 2)
    return s


def _worker(rank, world, port, out):
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1210_6411_b200  # noqa: F401
        from oracle import port as oport
        from paper_1210_6411_b200.cipher import MINI789
        from paper_1210_6411_b200.distributed import allreduce_stats, shard_range

        g = golden_npz("edges_mini789")
        lo, hi = shard_range(g["src"].size, rank, world)
        d, w = oport.walk(MINI789, 0xAA, g["src"][lo:hi])
        local = _stats_block(w[:, 0], 600, 200)
        glob = allreduce_stats(local)
        out[rank] = (lo, hi, d[:, 0].tolist(), w[:, 0].tolist(), glob.tolist())
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_matches_single_rank():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    g = golden_npz("edges_mini789")
    spans = [out[r][:2] for r in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == g["src"].size
    dst = sum((out[r][2] for r in range(world)), [])
    dist_ = sum((out[r][3] for r in range(world)), [])
    assert dst == g["dst"].tolist() and dist_ == g["dist"].tolist()
    whole = _stats_block(g["dist"], 600, 200)
    for r in range(world):
        assert out[r][4] == whole.tolist()
