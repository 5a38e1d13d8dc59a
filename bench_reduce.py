"""Steps 4-5 throughput: edge sort, leaf cutting to the
fixpoint and cycle counting on a synthetic skeleton held in HBM.

    python bench_reduce.py [--log2 26]

The synthetic skeleton is a seeded random mapping on 2^k sources (each source's
destination drawn uniformly among the sources), the graph model the paper compares A5/1
against (§6).  Records go through the public host-buffer C ABI calls
(lc_sort_edges, lc_cut_leaves, lc_count_cycles); wall-clock times include the
host<->device copies.  The leaf cut is also timed device-resident (lc_cut_leaves_device,
CUDA events) and through the sharded multi-GPU driver run as one rank.  Parity: a 2^20 instance is checked against oracle/reduce_np.py.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2", type=int, default=26)
    args = ap.parse_args()
    import paper_1210_6411_b200 as lc
    from oracle import reduce_np

    def instance(k, seed):
        rng = np.random.default_rng(seed)
        n = 1 << k
        src = np.unique(rng.integers(0, 1 << 62, size=n + n // 64, dtype=np.uint64))[:n]
        rng.shuffle(src)  # unsorted input: the edge-output sort has real work
        dst = src[rng.integers(0, n, size=n)]
        dist = rng.integers(11_000_000, 11_400_000, size=n, dtype=np.uint64)
        return src, dst, dist

    # parity on 2^20
    s, d, w = instance(20, 1)
    s, d, w = lc.sort_edge_arrays(s, d, w)
    z = np.zeros(s.size, dtype=np.uint64)
    got = lc.cut_leaves_arrays(s, d, w, z, z)
    want = reduce_np.cut_leaves(s, d, w, z, z)
    parity = got[5] == want[5] and all((a == b).all() for a, b in zip(got[:5], want[:5]))
    cyc = lc.count_cycles_arrays(*got[:4])
    parity = parity and [tuple(r) for r in zip(*(c.tolist() for c in cyc))] == reduce_np.count_cycles(*want[:4])

    src, dst, dist = instance(args.log2, 2)
    n = src.size
    lc.sort_edge_arrays(src[:1024], dst[:1024], dist[:1024])  # warm-up
    t0 = time.perf_counter()
    s, d, w = lc.sort_edge_arrays(src, dst, dist)
    t_sort = time.perf_counter() - t0
    z = np.zeros(n, dtype=np.uint64)
    t0 = time.perf_counter()
    fs, fd, fw, fz, fdep, passes = lc.cut_leaves_arrays(s, d, w, z, z)
    t_cut = time.perf_counter() - t0
    t0 = time.perf_counter()
    cyc = lc.count_cycles_arrays(fs, fd, fw, fz)
    t_cyc = time.perf_counter() - t0

    # device-resident leaf cutting (lc_cut_leaves_device), timed with CUDA events, and the
    # sharded driver (lc_cut_shard_*) as a single rank
    import torch
    from paper_1210_6411_b200.reduce import cut_leaves_tensors
    from paper_1210_6411_b200.sharded_reduce import cut_leaves_sharded

    def dev_cols():
        return [torch.from_numpy(c.view(np.int64)).cuda() for c in (s, d, w, z, z)]

    timings = {}
    for name, fn in (("device", cut_leaves_tensors), ("sharded_1rank", cut_leaves_sharded)):
        fn(*dev_cols())  # warm-up: first-use kernel loading and graph setup stay out of the timing
        cols = dev_cols()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n_out, p2 = fn(*cols)
        e1.record()
        torch.cuda.synchronize()
        ok = n_out == fs.size and p2 == passes and (cols[3][:n_out].cpu().numpy().view(np.uint64) == fz).all()
        timings[name] = (e0.elapsed_time(e1) / 1e3, bool(ok))
        del cols
    line = {
        "metric": "steps 4-5: sort + leaf cutting to fixpoint + cycle counting (records/s)",
        "config": {"workload": f"seeded random mapping on 2^{args.log2} sources, 40-byte edge records",
                   "path": "host-buffer C ABI (copies included)"},
        "records": n, "sort_s": t_sort, "sort_records_per_s": n / t_sort,
        "cut_s": t_cut, "passes": len(passes), "cut_records_per_s": n / t_cut,
        "cut_device_s": timings["device"][0], "cut_device_records_per_s": n / timings["device"][0],
        "cut_device_matches": timings["device"][1],
        "cut_sharded_1rank_s": timings["sharded_1rank"][0],
        "cut_sharded_1rank_matches": timings["sharded_1rank"][1],
        "fixpoint_records": int(fs.size), "cycles": int(cyc[0].size), "cycles_s": t_cyc,
        "parity_2p20_vs_restatement": bool(parity),
    }
    print(json.dumps(line), flush=True)


def measure_next(sort_log2: int = 26, cut_log2: int = 24) -> dict:
    """The §8(f) rows for the default bench line (bench.py): the edge-output sort of a
    device-resident 5-column record set (A5/1 skeleton sources) with its HBM roofline,
    and device-resident leaf cutting to the fixpoint on a seeded random mapping; parity of
    sort + cut + cycle count against oracle/reduce_np.py on a 2^20 instance."""
    import ctypes as C

    import torch

    import paper_1210_6411_b200 as lc
    from oracle import reduce_np
    from paper_1210_6411_b200 import _native as N
    from paper_1210_6411_b200.reduce import cut_leaves_tensors

    def instance(k, seed):
        rng = np.random.default_rng(seed)
        n = 1 << k
        src = np.unique(rng.integers(0, 1 << 62, size=n + n // 64, dtype=np.uint64))[:n]
        rng.shuffle(src)
        dst = src[rng.integers(0, n, size=n)]
        dist = rng.integers(11_000_000, 11_400_000, size=n, dtype=np.uint64)
        return src, dst, dist

    s, d, w = instance(20, 1)
    s, d, w = lc.sort_edge_arrays(s, d, w)
    z = np.zeros(s.size, dtype=np.uint64)
    got = lc.cut_leaves_arrays(s, d, w, z, z)
    want = reduce_np.cut_leaves(s, d, w, z, z)
    parity = got[5] == want[5] and all((a == b).all() for a, b in zip(got[:5], want[:5]))
    cyc = lc.count_cycles_arrays(*got[:4])
    parity = bool(parity and [tuple(r) for r in zip(*(c.tolist() for c in cyc))] == reduce_np.count_cycles(*want[:4]))

    dev = torch.device("cuda", torch.cuda.current_device())
    ctx = N.context(dev.index)
    st = torch.cuda.current_stream(dev)
    n = 1 << sort_log2
    g = torch.Generator(device=dev)
    g.manual_seed(sort_log2)
    r1 = torch.randint(1, 1 << 19, (n,), device=dev, generator=g)
    r2 = torch.randint(1, 1 << 22, (n,), device=dev, generator=g)
    cols = [r1 | (r2 << 19) | (0x2AAA00 << 41), torch.randint(0, 1 << 62, (n,), device=dev, generator=g),
            torch.arange(n, device=dev), torch.zeros(n, dtype=torch.int64, device=dev),
            torch.zeros(n, dtype=torch.int64, device=dev)]
    del r1, r2
    outs = [torch.empty_like(c) for c in cols]
    pin = (C.c_void_p * 5)(*[c.data_ptr() for c in cols])
    pout = (C.c_void_p * 5)(*[c.data_ptr() for c in outs])

    def run():
        N.check(N.lib.lc_sort_edges_device(ctx.handle, n, pin, pout, C.c_void_p(st.cuda_stream)))

    run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    run()
    e1.record(st)
    torch.cuda.synchronize()
    sort_s = e0.elapsed_time(e1) / 1e3
    ascending = bool((outs[0][1:] >= outs[0][:-1]).all().item())
    # stable: rows (the arange column) ascend within equal sources
    eq = outs[0][1:] == outs[0][:-1]
    stable = bool(((outs[2][1:] > outs[2][:-1]) | ~eq).all().item())
    W = min(max((n - 1).bit_length() - 10, 8), 22)
    alg = n * (72 + 8 + 20 + 24 * ((W + 7) // 8 - 1) + 8 + 84)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm = float(peaks.get("hbm_gbs", 0.0)) * 1e9 or None
    del cols, outs
    torch.cuda.empty_cache()

    src, dst, dist = instance(cut_log2, 2)
    src, dst, dist = lc.sort_edge_arrays(src, dst, dist)
    zc = np.zeros(src.size, dtype=np.uint64)
    tens = [torch.from_numpy(c.view(np.int64)).to(dev) for c in (src, dst, dist, zc, zc)]
    cut_leaves_tensors(*[t.clone() for t in tens])  # warm-up: context scratch, graph, attributes
    torch.cuda.synchronize()
    e0.record(st)
    n_out, passes = cut_leaves_tensors(*tens)
    e1.record(st)
    torch.cuda.synchronize()
    cut_s = e0.elapsed_time(e1) / 1e3
    del tens
    return {
        "edge_sort": {"workload": f"2^{sort_log2} device-resident 5-column records, A5/1 skeleton-like sources",
                      "records": n, "seconds": sort_s, "records_per_s": n / sort_s,
                      "route": f"msd (window {W} bits)", "ascending": ascending, "stable": stable,
                      "roofline": {"bound": "hbm", "achieved": alg / sort_s / 1e9,
                                   "peak": hbm / 1e9 if hbm else None, "unit": "GB/s",
                                   "frac": alg / sort_s / hbm if hbm else None,
                                   "algorithmic_bytes_per_record": alg / n,
                                   "peak_source": "MEASURED_PEAKS.json hbm_gbs"}},
        "leaf_cut": {"workload": f"seeded random mapping on 2^{cut_log2} sources, device-resident",
                     "records": int(src.size), "seconds": cut_s, "records_per_s": src.size / cut_s,
                     "passes": len(passes), "fixpoint_records": int(n_out)},
        "parity_2p20_sort_cut_cycles_vs_restatement": parity,
    }


if __name__ == "__main__":
    main()
