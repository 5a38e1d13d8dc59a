"""The in-house edge-output radix sort (csrc/sort.cu): records
ascending by source (records.py:3-5, reduce.py:3-4), stable like numpy's argsort(kind=
"stable"), through the host API (reduce.sort_edge_arrays -> lc_sort_edges) and the
asynchronous device API (lc_sort_edges_device).  Key shapes: full 64-bit random, A5/1
skeleton sources (constant R3 bytes -> skipped passes), already ascending (no pass runs),
heavy duplicates, descending, tile-boundary sizes; from 2^16 records the MSD route (bit
windows + per-group shared-memory sorts) with its LSD fallback for oversized groups."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _keys(kind, n, rng):
    if kind == "random64":
        return rng.integers(0, np.iinfo(np.uint64).max, size=n, dtype=np.uint64, endpoint=True)
    if kind == "a51":  # special nodes: R3 = 0x2AAA00 in bits 41..63, R1/R2 random
        r1 = rng.integers(1, 1 << 19, size=n, dtype=np.uint64)
        r2 = rng.integers(1, 1 << 22, size=n, dtype=np.uint64)
        return r1 | (r2 << np.uint64(19)) | (np.uint64(0x2AAA00) << np.uint64(41))
    if kind == "sorted":
        return np.sort(rng.integers(0, 1 << 50, size=n, dtype=np.uint64))
    if kind == "descending":
        return np.sort(rng.integers(0, 1 << 40, size=n, dtype=np.uint64))[::-1].copy()
    if kind == "dups":
        return rng.integers(0, 37, size=n, dtype=np.uint64) << np.uint64(23)
    if kind == "constant":
        return np.full(n, 0x1234_5678_9ABC_DEF0, dtype=np.uint64)
    if kind == "clustered":  # few distinct high parts, random low bits: groups too big for the
        # MSD route's per-group shared-memory sort -> the device falls back to the LSD passes
        return (rng.integers(0, 37, size=n, dtype=np.uint64) << np.uint64(40)) | \
            rng.integers(0, 1 << 30, size=n, dtype=np.uint64)
    raise ValueError(kind)


@pytest.mark.parametrize("route", ["auto", "lsd"])
@pytest.mark.parametrize("kind", ["random64", "a51", "sorted", "descending", "dups", "constant", "clustered"])
@pytest.mark.parametrize("n", [1, 2, 4095, 4096, 4097, 65_537, 300_001])
def test_host_sort_is_stable_argsort(gpu, lc, kind, n, route, monkeypatch):
    if route == "lsd":
        if n < 65_537:
            pytest.skip("below 2^16 records the LSD route is the only one")
        monkeypatch.setenv("LFSR_SORT_LSD", "1")  # the LSD route at sizes that default to MSD
    rng = np.random.default_rng(n * 7 + len(kind))
    src = _keys(kind, n, rng)
    dst = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
    dist = np.arange(n, dtype=np.uint64)
    size = rng.integers(0, 1000, size=n, dtype=np.uint64)
    depth = rng.integers(0, 100, size=n, dtype=np.uint64)
    s, d, w, z, h = lc.sort_edge_arrays(src, dst, dist, size, depth)
    order = np.argsort(src, kind="stable")
    assert (s == src[order]).all() and (d == dst[order]).all() and (w == dist[order]).all()
    assert (z == size[order]).all() and (h == depth[order]).all()


def test_device_sort_out_of_place(gpu, lc):
    import torch

    from paper_1210_6411_b200 import _native as N

    ctx = N.context()
    dev = torch.device("cuda", ctx.device)
    rng = np.random.default_rng(3)
    n = (1 << 22) + 12345
    cols = [_keys("a51", n, rng), rng.integers(0, 1 << 62, size=n, dtype=np.uint64),
            np.arange(n, dtype=np.uint64)]
    d_in = [torch.from_numpy(c.view(np.int64)).to(dev) for c in cols]
    d_out = [torch.empty_like(t) for t in d_in]
    pin = (C.c_void_p * 5)(*[t.data_ptr() for t in d_in], None, None)
    pout = (C.c_void_p * 5)(*[t.data_ptr() for t in d_out], None, None)
    st = torch.cuda.Stream(dev)
    torch.cuda.synchronize()
    N.check(N.lib.lc_sort_edges_device(ctx.handle, n, pin, pout, C.c_void_p(st.cuda_stream)))
    torch.cuda.synchronize()
    order = np.argsort(cols[0], kind="stable")
    for c, o in zip(cols, d_out):
        assert (o.cpu().numpy().view(np.uint64) == c[order]).all()
    for c, i in zip(cols, d_in):  # inputs untouched
        assert (i.cpu().numpy().view(np.uint64) == c).all()
    # argument checks
    bad = (C.c_void_p * 5)(*[t.data_ptr() for t in d_out], d_out[0].data_ptr(), None)
    with pytest.raises(N.NativeError):
        N.check(N.lib.lc_sort_edges_device(ctx.handle, n, pin, bad, None))


def test_device_sort_unaligned_columns(gpu, lc):
    """Key columns 8 bytes past a 16-byte boundary (a view one element into a buffer):
    the window histogram and the group-bounds kernel take their one-key-per-load paths."""
    import torch

    from paper_1210_6411_b200 import _native as N

    ctx = N.context()
    dev = torch.device("cuda", ctx.device)
    rng = np.random.default_rng(5)
    n = (1 << 18) + 3
    cols = [_keys("a51", n, rng), rng.integers(0, 1 << 62, size=n, dtype=np.uint64), np.arange(n, dtype=np.uint64)]
    bufs_in = [torch.empty(n + 1, dtype=torch.int64, device=dev) for _ in cols]
    bufs_out = [torch.empty(n + 1, dtype=torch.int64, device=dev) for _ in cols]
    d_in = [b[1:] for b in bufs_in]
    d_out = [b[1:] for b in bufs_out]
    for t, c in zip(d_in, cols):
        t.copy_(torch.from_numpy(c.view(np.int64)))
    assert all(t.data_ptr() % 16 == 8 for t in d_in + d_out)
    pin = (C.c_void_p * 5)(*[t.data_ptr() for t in d_in], None, None)
    pout = (C.c_void_p * 5)(*[t.data_ptr() for t in d_out], None, None)
    torch.cuda.synchronize()
    N.check(N.lib.lc_sort_edges_device(ctx.handle, n, pin, pout, None))
    torch.cuda.synchronize()
    order = np.argsort(cols[0], kind="stable")
    for c, o in zip(cols, d_out):
        assert (o.cpu().numpy().view(np.uint64) == c[order]).all()
