"""K3 (step-2 prune) kernel A/B on the config-3 slice, one B200: the default kernel (v3,
the uniform-step DFS/BFS of csrc/prune.cu) against v2 (LFSR_PRUNE_V1=2), on the same box,
on prefixes of the 2^32-state slice's candidates (K2 enumeration order) -- or the whole
slice with --log2 full.  Each line: seconds per kernel, expansions/s, and whether the two
kernels' per-candidate results (removed flag, `expanded` counter) are identical, compared
element by element on the device.

    python bench_prune_ab.py [--log2 24,26,28|full] [--mode dfs|bfs] [--limit 3000]

Numbers recorded in profiles/r02_prune3_ab.txt and profiles/r02_prune3_full_slice_identity.json.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2", default="24,26,28")
    ap.add_argument("--mode", default="dfs", choices=["dfs", "bfs"])
    ap.add_argument("--limit", type=int, default=3000)
    args = ap.parse_args()

    import torch

    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ctx = N.context(0)
    spec = lc.A51
    params = lc.CandidateParams.from_spec(spec, 0x2AAA00)
    sspec = N.spec_struct(spec)
    rows = 1 << 13  # R2 rows of the slice (configs[2])
    cap = rows * spec.reg_masks[0] // 2 + (1 << 20)
    out = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    N.check(N.lib.lc_enumerate_device(ctx.handle, C.byref(sspec), params.fixed_r3, 0x2AAA, 0x2AAA + rows,
                                      C.c_void_p(out.data_ptr()), cap, C.c_void_p(count.data_ptr()),
                                      C.c_void_p(stream.cuda_stream)))
    torch.cuda.synchronize()
    ncand = int(count.item())
    mode = 0 if args.mode == "dfs" else 1
    sizes = [None if s == "full" else int(s) for s in args.log2.split(",")]
    for lg in sizes:
        n = ncand if lg is None else min(1 << lg, ncand)
        cands = out[:n]
        res = {}
        for name, env in (("v3", ""), ("v2", "2")):
            os.environ["LFSR_PRUNE_V1"] = env
            removed = torch.empty(n, dtype=torch.uint8, device=dev)
            work = torch.empty(n, dtype=torch.int64, device=dev)

            def go():
                N.check(N.lib.lc_prune_device(ctx.handle, C.byref(sspec), params.fixed_r3, mode, args.limit,
                                              C.c_void_p(cands.data_ptr()), n, C.c_void_p(removed.data_ptr()),
                                              C.c_void_p(work.data_ptr()), C.c_void_p(stream.cuda_stream)))

            if lg is not None:  # warm-up (the whole-slice run is its own warm-up-free measurement)
                go()
                torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            go()
            e1.record(stream)
            torch.cuda.synchronize()
            res[name] = (e0.elapsed_time(e1) / 1e3, removed, work)
        os.environ.pop("LFSR_PRUNE_V1", None)
        expanded = int(res["v3"][2].sum().item())
        print(json.dumps({
            "candidates": n, "log2": lg if lg is not None else "full slice", "mode": args.mode, "limit": args.limit,
            "v3_s": res["v3"][0], "v2_s": res["v2"][0], "speedup": res["v2"][0] / res["v3"][0],
            "v3_expansions_per_s": expanded / res["v3"][0], "v2_expansions_per_s": expanded / res["v2"][0],
            "expanded": expanded, "survivors": int((res["v3"][1] == 0).sum().item()),
            "removed_identical": bool(torch.equal(res["v3"][1], res["v2"][1])),
            "expanded_identical": bool(torch.equal(res["v3"][2], res["v2"][2]))}), flush=True)


if __name__ == "__main__":
    main()
