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


if __name__ == "__main__":
    main()
