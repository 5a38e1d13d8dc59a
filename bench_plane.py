"""Steps 1-3 over consecutive 2^32-state slices of the fixed-R3 plane, one B200: the
whole skeleton construction of the paper (every special node has R3 = F, so the plane's
(2^19-1)(2^22-1) states hold all 2^40.8 candidates; 512 slices of 8192 R2 rows cover it)
measured on a run of slices and projected to the plane.

    python bench_plane.py [--slices 4] [--first-row 0x2AAA] [--depth 3000]

Per slice: K2 enumerates the slice's candidates into HBM, K3 prunes all of them (DFS,
`depth`, one launch), the survivors are compacted and K1 walks every one to its next
special node at the paper's stride.  One JSON line: per-slice counts and times, totals,
and the projection to all 512 slices on one and on eight GPUs (slices are independent).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ROWS = 1 << 13  # R2 rows per slice: 8192 x (2^19 - 1) states ~ 2^32


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slices", type=int, default=4)
    ap.add_argument("--first-row", type=lambda v: int(v, 0), default=0x2AAA)
    ap.add_argument("--depth", type=int, default=3000)
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
    m2 = spec.reg_masks[1]
    cap = ROWS * spec.reg_masks[0] // 2 + (1 << 20)
    cands = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)
    removed = torch.empty(cap, dtype=torch.uint8, device=dev)
    work = torch.empty(cap, dtype=torch.int64, device=dev)
    words = N.ST_HEADER + 2
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    per = []
    t_wall = time.perf_counter()
    for s in range(args.slices):
        lo = args.first_row + s * ROWS
        hi = min(lo + ROWS, m2 + 1)
        if lo >= hi:
            break
        ev[0].record(stream)
        N.check(N.lib.lc_enumerate_device(ctx.handle, C.byref(sspec), params.fixed_r3, lo, hi,
                                          C.c_void_p(cands.data_ptr()), cap, C.c_void_p(count.data_ptr()),
                                          C.c_void_p(stream.cuda_stream)))
        ev[1].record(stream)
        torch.cuda.synchronize()
        n = int(count.item())
        ev[2].record(stream)
        N.check(N.lib.lc_prune_device(ctx.handle, C.byref(sspec), params.fixed_r3, 0, args.depth,
                                      C.c_void_p(cands.data_ptr()), n, C.c_void_p(removed.data_ptr()),
                                      C.c_void_p(work.data_ptr()), C.c_void_p(stream.cuda_stream)))
        ev[3].record(stream)
        surv = cands[:n][removed[:n] == 0]
        ns = surv.numel()
        expanded = int(work[:n].sum().item())
        dst = torch.empty(ns, dtype=torch.int64, device=dev)
        dist = torch.empty(ns, dtype=torch.int64, device=dev)
        st = torch.zeros(words, dtype=torch.int64, device=dev)
        ev[4].record(stream)
        N.check(N.lib.lc_walk_device(ctx.handle, C.byref(sspec), params.fixed_r3, C.c_void_p(surv.data_ptr()), ns,
                                     lc.DEFAULT_STRIDE_A51, 16 * int(4 * ((1 << 23) - 1) / 3) + 64, 1, 0,
                                     C.c_void_p(dst.data_ptr()), C.c_void_p(dist.data_ptr()), 0, 0, 0,
                                     C.c_void_p(st.data_ptr()), C.c_void_p(stream.cuda_stream)))
        ev[5].record(stream)
        torch.cuda.synchronize()
        stats = st.cpu().numpy().view(np.uint64)
        if int(stats[N.ST_ERROR]):
            raise SystemExit(f"walk error {int(stats[N.ST_ERROR])} in slice {s}")
        special = bool(lc.is_candidate(dst[: 1 << 14].cpu().numpy().view(np.uint64), params, spec).all())
        rec = {"r2_rows": [lo, hi], "candidates": n, "survivors": ns, "expanded": expanded,
               "k2_s": ev[0].elapsed_time(ev[1]) / 1e3, "k3_s": ev[2].elapsed_time(ev[3]) / 1e3,
               "k1_s": ev[4].elapsed_time(ev[5]) / 1e3, "transitions": int(stats[N.ST_TRANSITIONS]),
               "destinations_are_special_nodes": special}
        rec["steps_1_to_3_s"] = rec["k2_s"] + rec["k3_s"] + rec["k1_s"]
        per.append(rec)
        print(json.dumps({"slice": s, **rec}), file=sys.stderr, flush=True)
        del surv, dst, dist
    total = {k: sum(r[k] for r in per) for k in ("candidates", "survivors", "expanded", "k2_s", "k3_s", "k1_s",
                                                  "transitions", "steps_1_to_3_s")}
    slices_in_plane = -(-m2 // ROWS)
    per_slice = total["steps_1_to_3_s"] / len(per)
    line = {"metric": "steps 1-3 over slices of the fixed-R3 plane (special-node enumeration, prune, walk)",
            "config": {"workload": f"{len(per)} consecutive 8192-row slices of R3 = 0x2AAA00 from R2 row "
                                   f"{args.first_row:#x}", "depth_limit": args.depth,
                       "stride": lc.DEFAULT_STRIDE_A51},
            "gpu": torch.cuda.get_device_name(0), "slices": per, "total": total,
            "survivor_fraction": total["survivors"] / total["candidates"],
            "expansions_per_s": total["expanded"] / total["k3_s"],
            "transitions_per_s": total["transitions"] / total["k1_s"],
            "wall_s": time.perf_counter() - t_wall,
            "projection": {"slices_in_plane": slices_in_plane,
                           "hours_one_gpu": per_slice * slices_in_plane / 3600,
                           "hours_eight_gpus": per_slice * slices_in_plane / 3600 / 8,
                           "basis": "mean steps 1-3 time of the measured slices x slices in the plane "
                                    "(slices are independent; the paper: step 2 12 h on 2048 cores, step 3 "
                                    "9 d 3 h on 5 GPUs, PAPER.md:418-426, 486)"}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
