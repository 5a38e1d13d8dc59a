"""GPU leaf cutting through the device-pointer ABI (lc_cut_leaves_device) and the sharded
multi-rank driver (lc_cut_shard_*, sharded_reduce.py): one shard on one GPU, and two
gloo ranks sharing cuda:0 (messages staged through host memory; the kernels of the two
ranks never wait on each other).  Everything must equal the reduce oracle, which is
pinned to the reference's cut_leaves_pass (tests/test_oracle.py)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import golden_npz

pytestmark = pytest.mark.gpu


def _random_mapping(n, seed):
    rng = np.random.default_rng(seed)
    src = np.unique(rng.integers(1, 1 << 62, size=n, dtype=np.int64)).astype(np.uint64)
    dst = src[rng.integers(0, src.size, size=src.size)]
    dist = rng.integers(1, 1000, size=src.size).astype(np.uint64)
    size = rng.integers(0, 5, size=src.size).astype(np.uint64)
    depth = rng.integers(0, 3, size=src.size).astype(np.uint64)
    return src, dst, dist, size, depth


def _mini789():
    g = golden_npz("edges_mini789")
    z = np.zeros(g["src"].size, dtype=np.uint64)
    return g["src"].astype(np.uint64), g["dst"].astype(np.uint64), g["dist"].astype(np.uint64), z, z


def _tensors(cols, lo=0, hi=None):
    import torch

    return [torch.from_numpy(c[lo:hi].copy().view(np.int64)).cuda() for c in cols]


def _rows(t, n_out):
    return np.stack([c[:n_out].cpu().numpy().view(np.uint64) for c in t], 1).tolist()


@pytest.mark.parametrize("case", ["mini789", "random", "random_big"])
@pytest.mark.parametrize("max_passes", [0, 1, 3])
def test_cut_leaves_tensors_matches_oracle(gpu, case, max_passes):
    from oracle import reduce_np
    from paper_1210_6411_b200.reduce import cut_leaves_tensors

    cols = {"mini789": _mini789, "random": lambda: _random_mapping(5000, 7),
            "random_big": lambda: _random_mapping(1 << 18, 11)}[case]()
    want = reduce_np.cut_leaves(*cols, max_passes=max_passes)
    t = _tensors(cols)
    n_out, passes = cut_leaves_tensors(*t, max_passes=max_passes)
    assert passes == [tuple(int(v) for v in p) for p in want[5]]
    assert _rows(t, n_out) == np.stack(want[:5], 1).tolist()


def test_sharded_single_rank_matches_oracle(gpu):
    from oracle import reduce_np
    from paper_1210_6411_b200.sharded_reduce import cut_leaves_sharded

    for cols in (_mini789(), _random_mapping(1 << 16, 3)):
        for max_passes in (0, 1):
            want = reduce_np.cut_leaves(*cols, max_passes=max_passes)
            t = _tensors(cols)
            n_out, passes = cut_leaves_sharded(*t, max_passes=max_passes)
            assert passes == [tuple(int(v) for v in p) for p in want[5]]
            assert _rows(t, n_out) == np.stack(want[:5], 1).tolist()
    broken = tuple(c[np.arange(c.size) % 97 != 5] for c in _random_mapping(5000, 7))
    with pytest.raises(ValueError):
        cut_leaves_sharded(*_tensors(broken))
    rm = _random_mapping(100, 1)
    unsorted = tuple(c[::-1].copy() for c in rm)
    with pytest.raises(ValueError):
        cut_leaves_sharded(*_tensors(unsorted))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _two_rank_cases():
    # the 2^18 mapping's first pass removes more than TAIL_LEAVES: the gathered tail starts later
    return {"mini789": _mini789(), "random": _random_mapping(1 << 16, 5), "random_2p18": _random_mapping(1 << 18, 9)}


def _worker(rank, world, port, out, backend="gloo", tail="1"):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), LFSR_SHARD_TAIL=tail)
    if backend == "nccl":
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    else:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1210_6411_b200.distributed import shard_range
        from paper_1210_6411_b200.sharded_reduce import cut_leaves_sharded

        cases = _two_rank_cases()
        for name, cols in cases.items():
            lo, hi = shard_range(cols[0].size, rank, world)
            t = _tensors(cols, lo, hi)
            n_out, passes = cut_leaves_sharded(*t)
            out[(name, rank)] = (_rows(t, n_out), passes)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tail", ["1", "0"], ids=["gathered_tail", "per_pass_only"])
def test_sharded_two_ranks_on_one_gpu(gpu, tail):
    """Two gloo ranks (sharing this box's one GPU): with the gathered tail (the default:
    after the first pass here) and with every pass exchanged."""
    import torch.multiprocessing as mp
    from oracle import reduce_np

    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out, "gloo", tail), nprocs=world, join=True)
    for name, cols in _two_rank_cases().items():
        want = reduce_np.cut_leaves(*cols)
        rows = sum((out[(name, r)][0] for r in range(world)), [])
        assert rows == np.stack(want[:5], 1).tolist(), name
        for r in range(world):
            assert out[(name, r)][1] == [tuple(int(v) for v in p) for p in want[5]], name


def test_sharded_one_rank_over_nccl(gpu):
    """The per-pass all-gather and all-to-all through a real NCCL communicator (one rank:
    this box has one GPU; a multi-GPU node runs the same calls with N ranks)."""
    import torch.multiprocessing as mp
    from oracle import reduce_np

    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(1, _free_port(), out, "nccl"), nprocs=1, join=True)
    for name, cols in _two_rank_cases().items():
        want = reduce_np.cut_leaves(*cols)
        assert out[(name, 0)][0] == np.stack(want[:5], 1).tolist(), name
        assert out[(name, 0)][1] == [tuple(int(v) for v in p) for p in want[5]], name


def _shaped(kind, n, seed):
    """Edge lists with extreme shapes: a long chain into a 3-cycle, a star into a
    self-loop, pure cycles, and a binary tree hanging off a 2-cycle."""
    rng = np.random.default_rng(seed)
    src = np.unique(rng.integers(1, 1 << 62, size=n, dtype=np.int64)).astype(np.uint64)
    rng.shuffle(src)
    m = src.size
    if kind == "chain":
        nxt = np.arange(1, m + 1) % m
        nxt[m - 1] = m - 3
    elif kind == "star":
        nxt = np.zeros(m, dtype=np.int64)
    elif kind == "cycles":
        nxt = np.arange(1, m + 1) % m
        nxt[m // 2 - 1] = 0
        nxt[m - 1] = m // 2
    else:  # tree
        nxt = (np.arange(m) - 1) // 2
        nxt[0] = 1
        nxt[1] = 0
    dst = src[nxt]
    dist = rng.integers(1, 100, size=m).astype(np.uint64)
    z = np.zeros(m, dtype=np.uint64)
    order = np.argsort(src)
    return src[order], dst[order], dist[order], z, z


@pytest.mark.parametrize("kind", ["chain", "star", "cycles", "tree"])
def test_cut_leaves_extreme_shapes(gpu, kind):
    from oracle import reduce_np
    from paper_1210_6411_b200.reduce import cut_leaves_tensors
    from paper_1210_6411_b200.sharded_reduce import cut_leaves_sharded

    cols = _shaped(kind, 20000, 3)
    want = reduce_np.cut_leaves(*cols)
    for fn in (cut_leaves_tensors, cut_leaves_sharded):
        t = _tensors(cols)
        n_out, passes = fn(*t)
        assert passes == [tuple(int(v) for v in p) for p in want[5]], (kind, fn.__name__)
        assert _rows(t, n_out) == np.stack(want[:5], 1).tolist(), (kind, fn.__name__)


def test_cut_leaves_arrays_tall_chain_keeps_every_pass(gpu, lc):
    """A 70,000-record chain into a 3-cycle needs 69,998 passes -- more than the first
    statistics buffer -- and every pass is reported (closed forms: pass i removes one
    leaf, leaves m - i inner records, and the survivors' size sum is i)."""
    cols = _shaped("chain", 70000, 8)
    m = cols[0].size
    out = lc.cut_leaves_arrays(*cols)
    passes = out[5]
    assert len(passes) == m - 3 + 1
    assert passes[:-1] == [(1, m - i, i) for i in range(1, m - 2)]
    assert passes[-1] == (0, 3, m - 3)
    assert out[0].size == 3 and int(out[3].sum()) == m - 3
