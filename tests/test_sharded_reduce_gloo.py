"""Multi-rank leaf cutting (sharded_reduce.py) under gloo on CPU: world sizes 2 and 3,
contiguous source-range shards (one empty), the per-pass all-gather / all-to-all
protocol of the multi-GPU path.  Per-rank shard kernels are replaced by the test-only
numpy stand-in (tests/_shard_np.py), with and without the gathered tail (whose
single-GPU cut is the reduce oracle here); the GPU form of the same driver runs in
tests/test_gpu_sharded_reduce.py.  Results must equal the reduce oracle (pinned to the
reference's cut_leaves_pass, tests/test_oracle.py)."""

from __future__ import annotations

import os
import socket

import numpy as np
import torch.multiprocessing as mp

from conftest import golden_npz


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _random_mapping(n, seed):
    rng = np.random.default_rng(seed)
    src = np.unique(rng.integers(1, 1 << 62, size=n, dtype=np.int64)).astype(np.uint64)
    dst = src[rng.integers(0, src.size, size=src.size)]
    dist = rng.integers(1, 1000, size=src.size).astype(np.uint64)
    size = rng.integers(0, 5, size=src.size).astype(np.uint64)
    depth = rng.integers(0, 3, size=src.size).astype(np.uint64)
    return src, dst, dist, size, depth


def _cases():
    g = golden_npz("edges_mini789")
    z = np.zeros(g["src"].size, dtype=np.uint64)
    mini = (g["src"].astype(np.uint64), g["dst"].astype(np.uint64), g["dist"].astype(np.uint64), z, z)
    rm = _random_mapping(5000, 7)
    broken = tuple(c[np.arange(c.size) % 97 != 5] for c in rm)  # drop records: not closed
    return {"mini789": (mini, 0, None), "mini789_one": (mini, 1, None), "random": (rm, 0, None),
            "random_empty_rank": (rm, 0, "empty1"), "broken": (broken, 0, None)}


def _split(n, rank, world, mode):
    from paper_1210_6411_b200.distributed import shard_range

    if mode != "empty1":
        return shard_range(n, rank, world)
    cut = n if world == 2 else n // 2  # rank 1 holds nothing
    if rank < 2:
        return (0, cut) if rank == 0 else (cut, cut)
    lo, hi = shard_range(n - cut, rank - 2, world - 2)
    return cut + lo, cut + hi


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from _shard_np import NumpyShard, NumpyShardTail, numpy_cut_leaves_tensors
        from paper_1210_6411_b200 import reduce as R
        from paper_1210_6411_b200.sharded_reduce import cut_leaves_sharded

        R.cut_leaves_tensors = numpy_cut_leaves_tensors  # the gathered tail's single-GPU cut, on CPU
        for tail, factory in ((False, NumpyShard), (True, NumpyShardTail)):
            for name, (cols, max_passes, mode) in _cases().items():
                n = cols[0].size
                lo, hi = _split(n, rank, world, mode)
                t = [torch.from_numpy(c[lo:hi].copy().view(np.int64)) for c in cols]
                try:
                    n_out, passes = cut_leaves_sharded(*t, max_passes=max_passes, shard_factory=factory)
                    rows = np.stack([c[:n_out].numpy().view(np.uint64) for c in t], 1).tolist()
                    out[(name, tail, rank)] = ("ok", rows, passes)
                except ValueError as e:
                    out[(name, tail, rank)] = ("ValueError", str(e), None)
    finally:
        dist.destroy_process_group()


def _run(world):
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    return dict(out)


def _check(out, world):
    from oracle import reduce_np

    for (name, (cols, max_passes, _)), tail in ((c, t) for c in _cases().items() for t in (False, True)):
        res = [out[(name, tail, r)] for r in range(world)]
        if name == "broken":
            assert all(r[0] == "ValueError" for r in res), res
            continue
        assert all(r[0] == "ok" for r in res), res
        want = reduce_np.cut_leaves(*cols, max_passes=max_passes)
        rows = sum((r[1] for r in res), [])
        assert rows == np.stack(want[:5], 1).tolist(), name
        for r in res:
            assert [tuple(p) for p in r[2]] == [tuple(int(v) for v in p) for p in want[5]], name


def test_sharded_leaf_cut_two_ranks():
    _check(_run(2), 2)


def test_sharded_leaf_cut_three_ranks():
    _check(_run(3), 3)
