"""Steps 1-2 feeding the walk (BASELINE.json configs[2]): special-node enumeration with
the leaf/predecessor filter over a 2^32-state slice of the fixed-R3 plane (K2), the
step-2 prune of the resulting candidates (K3), and a walk of the survivors (K1).

    python bench_steps12.py [--rows-log2 13] [--prune-log2 20] [--depth 3000] [--full]

Prints one JSON line.  --full runs steps 1-3 over the whole slice: every candidate is
pruned (one launch; --prune-chunk-log2 splits it) and every survivor is walked to its next special node.  Parity:
the first 4 R2 rows of the slice and a 65536-candidate sample of the prune are compared
with the C oracle on the host.
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

R2_0 = 0x2AAA  # first R2 row of the slice


def k3_roofline(expansions_per_s: float, lop3_peak: float, sm_mhz: float) -> dict:
    """K3 is bound by instruction issue on the integer ALU pipe (no tensor or HBM work:
    its stack traffic stays mostly in L2).  achieved = the live expansions/s times the
    ALU-pipe warp instructions per expansion that ncu counted for this kernel
    (profiles/r02_prune3_metrics.json); peak = the ALU pipe's warp-instruction rate,
    i.e. the LOP3 issue peak measured in this process (lc_lop3_peak: one 32-lane ALU
    instruction per 2 cycles per SM sub-partition) / 32 -- so frac is the ALU pipe's
    busy fraction.  simt_efficiency says how much of that issue carries live lanes."""
    path = os.path.join(ROOT, "profiles", "r02_prune3_metrics.json")
    try:
        with open(path) as f:
            met = json.load(f)
    except OSError:
        return {"bound": "issue (integer ALU pipe)", "achieved": None, "peak": None, "frac": None,
                "note": "profiles/r02_prune3_metrics.json missing"}
    alu = float(met["alu_warp_inst_per_expansion"])
    achieved = expansions_per_s * alu
    peak = lop3_peak / 32.0
    return {"bound": "issue (integer ALU pipe)", "achieved": achieved / 1e9, "peak": peak / 1e9,
            "unit": "G ALU warp-instructions/s", "frac": achieved / peak,
            "peak_source": f"lc_lop3_peak measured in this run / 32 lanes ({sm_mhz:.0f} MHz)",
            "alu_warp_inst_per_expansion": alu,
            "simt_efficiency": met["simt_efficiency"], "warp_inst_per_expansion": met["warp_inst_per_expansion"],
            "traffic": None,
            "traffic_note": "no HBM-bound work: ncu DRAM bytes at 2^26 = "
                            f"{(met['dram__bytes_read.sum'] + met['dram__bytes_write.sum']) / met['expansions']:.2f} B "
                            "per expansion (the write-through stack, mostly absorbed by L2)",
            "ncu": {k: met[k] for k in ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
                                         "smsp__issue_active.avg.pct_of_peak_sustained_active",
                                         "sm__warps_active.avg.pct_of_peak_sustained_active")},
            "source": "profiles/r02_prune3_metrics.json"}


def measure(ctx, stream, *, rows_log2: int = 13, prune_log2: int = 26, depth: int = 3000, walk_log2: int = 14,
            cpu_sample: int = 1 << 14, keep=None, lop3_peak=None) -> dict:
    """Config 3 on one GPU: K2 over 2^rows_log2 R2 rows (the 2^32-state slice by default),
    K3 (DFS, `depth`) on the first 2^prune_log2 candidates, K1 on a prefix of the
    survivors; each with parity against the C restatement on a sample and a CPU baseline.
    `keep` (dict) receives the device tensors for --full."""
    import torch

    import paper_1210_6411_b200 as lc
    from oracle import port
    from paper_1210_6411_b200 import _native as N

    dev = torch.device("cuda", ctx.device)
    spec = lc.A51
    params = lc.CandidateParams.from_spec(spec, 0x2AAA00)
    sspec = N.spec_struct(spec)
    rows = 1 << rows_log2
    states = rows * spec.reg_masks[0]
    cap = states // 2 + (1 << 20)
    cores = len(os.sched_getaffinity(0))
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    hbm_peak = float(peaks.get("hbm_gbs", 0.0)) * 1e9 or None

    out = torch.empty(cap, dtype=torch.int64, device=dev)
    count = torch.zeros(1, dtype=torch.int64, device=dev)

    def enumerate_slice():
        N.check(N.lib.lc_enumerate_device(ctx.handle, C.byref(sspec), params.fixed_r3, R2_0, R2_0 + rows,
                                          C.c_void_p(out.data_ptr()), cap, C.c_void_p(count.data_ptr()),
                                          C.c_void_p(stream.cuda_stream)))

    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # the write-stream roof of this GPU: a plain fill of the same output bytes
    n_fill = states // 2
    out[:n_fill].fill_(1)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(3):
        out[:n_fill].fill_(1)
    e1.record(stream)
    torch.cuda.synchronize()
    write_peak = n_fill * 8 * 3 / (e0.elapsed_time(e1) / 1e3)

    enumerate_slice()  # warm-up
    torch.cuda.synchronize()
    reps = 3
    e0.record(stream)
    for _ in range(reps):
        enumerate_slice()
    e1.record(stream)
    torch.cuda.synchronize()
    k2_s = e0.elapsed_time(e1) / 1e3 / reps
    ncand = int(count.item())

    # parity: first 4 rows vs the C restatement (host), which is also K2's CPU baseline
    os.environ["OMP_NUM_THREADS"] = str(cores)
    t0 = time.perf_counter()
    want = port.enumerate_rows(spec, 0x2AAA00, R2_0, R2_0 + 4)
    k2_cpu_s = time.perf_counter() - t0
    got = out[: want.size].cpu().numpy().view(np.uint64)
    k2_parity = bool((got == want).all())
    # size-independent checks over the whole slice: ascending, count = closed form
    head = out[:ncand]
    ascending = bool((head[1:] > head[:-1]).all().item()) if ncand > 1 else True
    k2_bytes = ncand * 8
    k2 = {"states": states, "candidates": ncand, "seconds": k2_s, "states_per_s": states / k2_s,
          "candidates_per_s": ncand / k2_s,
          "roofline": {"bound": "hbm", "achieved": k2_bytes / k2_s / 1e9,
                       "peak": hbm_peak / 1e9 if hbm_peak else None, "unit": "GB/s",
                       "frac": k2_bytes / k2_s / hbm_peak if hbm_peak else None,
                       "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy: read + write bytes)",
                       "write_stream_gbs_measured": write_peak / 1e9,
                       "frac_of_write_stream": k2_bytes / k2_s / write_peak,
                       "algorithmic": "8 B written per candidate (a pure write stream)"},
          "parity_first_4_rows_vs_oracle": k2_parity, "ascending": ascending,
          "cpu_baseline": {"value": 4 * spec.reg_masks[0] / k2_cpu_s, "unit": "states/s", "cores": 1,
                           "kind": "port", "sample": f"4 R2 rows ({4 * spec.reg_masks[0]} states), "
                                                     "orc_enumerate (pipeline.py:104-118 restated)"}}

    # ---- K3: prune a prefix of the enumerated candidates (DFS, depth limit)
    npr = min(1 << prune_log2, ncand)
    cands = out[:npr].clone()
    if keep is not None:
        keep["cands_all"] = out[:ncand]
    else:
        del out
    removed = torch.empty(npr, dtype=torch.uint8, device=dev)
    work = torch.empty(npr, dtype=torch.int64, device=dev)

    def prune():
        N.check(N.lib.lc_prune_device(ctx.handle, C.byref(sspec), params.fixed_r3, 0, depth,
                                      C.c_void_p(cands.data_ptr()), npr, C.c_void_p(removed.data_ptr()),
                                      C.c_void_p(work.data_ptr()), C.c_void_p(stream.cuda_stream)))

    # warm-up on a 2^20 prefix (same grid and stack allocation as the timed launch)
    npr_full = npr
    npr = min(npr_full, 1 << 20)
    prune()
    npr = npr_full
    torch.cuda.synchronize()
    e0.record(stream)
    prune()
    e1.record(stream)
    torch.cuda.synchronize()
    k3_s = e0.elapsed_time(e1) / 1e3
    expanded = int(work.sum().item())
    nremoved = int(removed.sum().item())
    # parity on an evenly spaced sample (the C restatement on the host cores)
    idx = np.linspace(0, npr - 1, min(cpu_sample, npr)).astype(np.int64)
    sample = cands.cpu().numpy().view(np.uint64)[idx]
    t0 = time.perf_counter()
    o_removed, o_work = port.prune(spec, 0x2AAA00, "dfs", depth, sample)
    cpu_s = time.perf_counter() - t0
    k3_parity = bool((o_removed == removed.cpu().numpy()[idx]).all() and
                     (o_work == work.cpu().numpy().view(np.uint64)[idx]).all())
    if lop3_peak is None:
        lop3_peak = N.lop3_peak(ctx.device)
    k3 = {"candidates": npr, "depth_limit": depth, "removed": nremoved, "removed_fraction": nremoved / npr,
          "expanded": expanded, "seconds": k3_s, "candidates_per_s": npr / k3_s,
          "expansions_per_s": expanded / k3_s,
          "roofline": k3_roofline(expanded / k3_s, lop3_peak[0], lop3_peak[1]),
          "kernel": "prune3_kernel (K3 v3, csrc/prune.cu)",
          "parity_sample_vs_oracle": k3_parity,
          "parity_sample": int(idx.size),
          "cpu_baseline": {"value": float(o_work.sum()) / cpu_s, "unit": "expansions/s", "cores": cores,
                           "kind": "port", "sample": f"{idx.size} evenly spaced candidates of the {npr} "
                                                     f"({cpu_s:.2f} s), orc_prune (pipeline.py:121-178 restated)"}}

    # ---- K1: walk (a prefix of) the survivors to their next special node
    surv = cands[removed == 0]
    nw = min(1 << walk_log2, surv.numel())
    res = lc.walk_arrays(surv[:nw].cpu().numpy().view(np.uint64), params, spec, stride=lc.DEFAULT_STRIDE_A51)
    if keep is not None:
        keep.update(out=keep["cands_all"], ncand=ncand)
    return {"workload": f"configs[2]: R3 = 0x2AAA00, R2 in [{R2_0:#x}, {R2_0 + rows:#x}), all R1 ({states} states)",
            "k2_enumerate": k2, "k3_prune": k3,
            "k1_walk_survivors": {"walks": nw, "edges": res.edges, "transitions": res.transitions}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rows-log2", type=int, default=13)   # 2^13 rows x (2^19-1) = 2^32 states
    ap.add_argument("--prune-log2", type=int, default=26)
    ap.add_argument("--depth", type=int, default=3000)     # the paper's DFS depth
    ap.add_argument("--walk-log2", type=int, default=14)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--prune-chunk-log2", type=int, default=31)  # --full: candidates per prune launch
    ap.add_argument("--skip-walk", action="store_true")  # --full: prune only (A/B of K3 variants)
    ap.add_argument("--cpu-sample", type=int, default=1 << 16)
    args = ap.parse_args()

    import torch

    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N

    stream = torch.cuda.Stream(torch.device("cuda", 0))
    torch.cuda.set_stream(stream)
    ctx = N.context(0)
    keep = {} if args.full else None
    line = {"metric": "steps 1-2 feeding the walk (special-node enumeration + leaf/predecessor filter, prune)"}
    line.update(measure(ctx, stream, rows_log2=args.rows_log2, prune_log2=args.prune_log2, depth=args.depth,
                        walk_log2=args.walk_log2, cpu_sample=args.cpu_sample, keep=keep))
    line["gpu"] = torch.cuda.get_device_name(0)
    if args.full:
        params = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
        line["full_slice_steps_1_to_3"] = full_slice(args, ctx, N.spec_struct(lc.A51), params,
                                                     keep["out"][:keep["ncand"]], stream, torch, N, lc)
    print(json.dumps(line), flush=True)


def full_slice(args, ctx, sspec, params, cands, stream, torch, N, lc):
    """Steps 1-3 over the whole slice: prune every candidate (one lc_prune_device launch
    per 2^prune_chunk_log2 candidates -- by default the whole slice at once, so the
    heavy-tailed traversals leave one tail, not one per chunk), compact the survivors,
    walk them all (one lc_walk_device call)."""
    dev = cands.device
    n = cands.numel()
    chunk = min(n, 1 << args.prune_chunk_log2)
    removed = torch.empty(chunk, dtype=torch.uint8, device=dev)
    work = torch.empty(chunk, dtype=torch.int64, device=dev)
    keep = []
    expanded = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for lo in range(0, n, chunk):
        m = min(chunk, n - lo)
        N.check(N.lib.lc_prune_device(ctx.handle, C.byref(sspec), params.fixed_r3, 0, args.depth,
                                      C.c_void_p(cands[lo:].data_ptr()), m, C.c_void_p(removed.data_ptr()),
                                      C.c_void_p(work.data_ptr()), C.c_void_p(stream.cuda_stream)))
        keep.append(cands[lo:lo + m][removed[:m] == 0])
        expanded += int(work[:m].sum().item())
    e1.record(stream)
    torch.cuda.synchronize()
    prune_s = e0.elapsed_time(e1) / 1e3
    surv = torch.cat(keep)
    ns = surv.numel()
    if args.skip_walk:
        return {"candidates": n, "prune_depth": args.depth, "survivors": ns, "expanded": expanded,
                "prune_s": prune_s, "expansions_per_s": expanded / prune_s, "prune_launch_candidates": chunk}
    dst = torch.empty(ns, dtype=torch.int64, device=dev)
    dist = torch.empty(ns, dtype=torch.int64, device=dev)
    words = N.ST_HEADER + 2
    st = torch.zeros(words, dtype=torch.int64, device=dev)
    e0.record(stream)
    N.check(N.lib.lc_walk_device(ctx.handle, C.byref(sspec), params.fixed_r3, C.c_void_p(surv.data_ptr()), ns,
                                 lc.DEFAULT_STRIDE_A51, 16 * int(4 * ((1 << 23) - 1) / 3) + 64, 1, 0,
                                 C.c_void_p(dst.data_ptr()), C.c_void_p(dist.data_ptr()), 0, 0, 0,
                                 C.c_void_p(st.data_ptr()), C.c_void_p(stream.cuda_stream)))
    e1.record(stream)
    torch.cuda.synchronize()
    walk_s = e0.elapsed_time(e1) / 1e3
    stats = st.cpu().numpy().view(np.uint64)
    if int(stats[N.ST_ERROR]):
        raise SystemExit(f"walk error {int(stats[N.ST_ERROR])}")
    tr = int(stats[N.ST_TRANSITIONS])
    # every survivor's destination is a special node (K2/K3's set is closed under the walk
    # only for the whole plane; here the check is the predicate itself)
    ok = bool(lc.is_candidate(dst[: 1 << 16].cpu().numpy().view(np.uint64), params, lc.A51).all())
    return {"candidates": n, "prune_depth": args.depth, "survivors": ns, "survivor_fraction": ns / n,
            "expanded": expanded, "prune_s": prune_s, "expansions_per_s": expanded / prune_s,
            "walks": ns, "transitions": tr, "walk_s": walk_s, "transitions_per_s": tr / walk_s,
            "min_dist": int(stats[N.ST_MIN]), "max_dist": int(stats[N.ST_MAX]),
            "destinations_are_special_nodes": ok,
            "prune_launch_candidates": chunk, "steps_1_to_3_s": prune_s + walk_s}


if __name__ == "__main__":
    main()
