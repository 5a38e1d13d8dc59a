"""Benchmark of the step-3 chain walk (BASELINE.json metric: A5/1 transitions/s and
weighted edges/s) on 1..8 B200s, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[1]): per GPU a set of 2^24 special A5/1 start nodes from
the seeded K0 generator; a step walks one batch of 2^22 of them to their next special
node (stride 11,170,000, as the reference's benchmark and the paper), cycling through
the 4 batches.  Weak scaling: rank r walks its own contiguous 2^24-start shard of one
global K0 stream.  Timing: CUDA events on the launching stream, barrier + synchronize on
both sides, max over ranks; L2 is flushed (256 MiB write) before every step.  One NCCL
all-reduce after the timed region gathers the chain-length histogram and edge counts.
`--total-log2 30 --steps 256/N` is configs[3] (2^30 starts split over N ranks, strong
scaling).

`--impl reference` times the reference algorithm on the host cores instead (the C
restatement in oracle/, since the Python reference cannot travel to the GPU box).
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "A5/1 transitions/s & weighted edges/s (step-3 chain walk), 1/2/4/8 B200"
PAPER_GTX580 = 9_800 * 11_170_000  # PAPER.md:478-479, transitions/s on one GTX 580
LOP3_PER_TRANSITION = 72 / 32      # algorithmic LOP3 per A5/1 transition
SEED = 1210_6411
STRIDE = 11_170_000
CAP = 178_957_008  # the reference's default walk cap for A5/1 (bitslice.py:273-274)
PAPER_SCALE_TRANSITIONS = int(2 ** 33.6 * 11_184_857)  # ~1.46e17
# DRAM bytes per walk of the walk kernel: dram__bytes_read.sum + dram__bytes_write.sum of
# one ncu capture (profiles/r01_walk_a51_metrics.json, a 2^20-walk launch) / walks
TRAFFIC_BYTES_PER_WALK = (9.564160e6 + 47.801344e6) / (1 << 20)


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def cpu_walk_sample(starts: np.ndarray, cores: int):
    """The reference algorithm on the host cores (oracle port, OpenMP, 256-lane waves
    like the reference's _edges_chunk chunks).  Returns (transitions/s, edges/s, s, dst, dist)."""
    from oracle import port
    from paper_1210_6411_b200.cipher import A51

    os.environ["OMP_NUM_THREADS"] = str(cores)
    t0 = time.perf_counter()
    dst, dist = port.walk(A51, 0x2AAA00, starts, stride=STRIDE, width=256)
    el = time.perf_counter() - t0
    return float(dist.sum()) / el, starts.size / el, el, dst[:, 0], dist[:, 0]


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = f"/tmp/lfsr_clocks_{os.getpid()}.csv"

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            self.proc.wait()

    def summary(self) -> dict:
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except OSError:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in rows if len(r) >= 9 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) >= 9 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4) if r[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def reference_arm(args, rank: int) -> None:
    """--impl reference: the reference algorithm (oracle port) on all host cores, same
    workload/metric; rank 0 only."""
    if rank != 0:
        return
    import paper_1210_6411_b200 as lc  # noqa: F401  (only for the K0 restatement's spec)
    from oracle import k0
    from paper_1210_6411_b200.cipher import A51

    cores = host_cores()
    per_step = cores * 256
    starts = k0.random_candidates(A51, 0x2AAA00, SEED, per_step * min(args.steps, 2))
    for _ in range(args.warmup):
        cpu_walk_sample(starts[:per_step], cores)
    tr = ed = el = 0.0
    for k in range(args.steps):
        s = starts[(k % 2) * per_step:(k % 2 + 1) * per_step]
        t, e, dt, _, dist = cpu_walk_sample(s, cores)
        tr += float(dist.sum())
        ed += s.size
        el += dt
    value = tr / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "transitions/s",
        "edges_per_s": ed / el, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": value / PAPER_GTX580, "dtype": "u64 (64-lane bitsliced words)",
        "data": "synthetic (K0 seeded special nodes, first host-sized sample)",
        "config": {"workload": f"A5/1 step-3 walk, stride {STRIDE}, {per_step} K0 starts per step "
                               f"(a bounded sample of the 2^24-start workload)", "parallelism": f"{cores} host threads"},
        "cpu_baseline": {"value": value, "unit": "transitions/s", "cores": cores, "kind": "port",
                         "sample": f"{per_step} starts per step x {args.steps} steps (256-lane waves)"},
        "e2e": {"value": value, "unit": "transitions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch-log2", type=int, default=22)
    ap.add_argument("--workload-log2", type=int, default=24)
    ap.add_argument("--total-log2", type=int, default=0,
                    help="strong scaling (configs[3]): 2^k starts in total, split over the ranks")
    ap.add_argument("--refill", type=int, default=0)
    ap.add_argument("--starts", default="k0", choices=["k0", "random"],
                    help="k0: special nodes (the metric's workload); random: uniform valid states")
    ap.add_argument("--legs", type=int, default=1)
    ap.add_argument("--stride", type=int, default=STRIDE)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        reference_arm(args, rank)
        return

    import torch
    import torch.distributed as dist

    # LFSR_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 with gloo, to exercise the
    # multi-rank path on a one-GPU box (the walks are independent; the only collectives
    # are the barriers and the statistics all-reduce outside the timed region)
    share = os.environ.get("LFSR_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N
    from paper_1210_6411_b200.distributed import allreduce_stats, stats_summary

    lc.set_device(local)
    spec = lc.A51
    params = lc.CandidateParams.from_spec(spec, 0x2AAA00)
    ctx = N.context(local)
    sspec = N.spec_struct(spec)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)  # explicit stream: kernels and events share it
    torch.cuda.set_stream(stream)

    if args.total_log2:  # configs[3]: a fixed total split over the ranks
        args.workload_log2 = args.total_log2 - (world.bit_length() - 1)
        if 1 << args.total_log2 != world << args.workload_log2:
            raise SystemExit("--total-log2 needs a power-of-two world size")
    per_gpu = 1 << args.workload_log2
    batch = 1 << args.batch_log2
    nbatches = max(1, per_gpu // batch)
    hist_lo, hist_shift, hist_bins = 11_184_809 - (1 << 15), 0, 1 << 16
    words = N.ST_HEADER + hist_bins + 2

    if args.starts == "k0":
        # this rank's contiguous shard of one global K0 stream, resident in HBM
        allstarts = torch.empty((rank + 1) * per_gpu, dtype=torch.int64, device=dev)
        N.check(N.lib.lc_random_candidates_device(ctx.handle, C.byref(sspec), params.fixed_r3, SEED,
                                                  allstarts.numel(), C.c_void_p(allstarts.data_ptr()),
                                                  C.c_void_p(stream.cuda_stream)))
        starts = allstarts[rank * per_gpu:].clone()
        del allstarts
    else:
        rng = np.random.default_rng(SEED + rank)
        regs = [rng.integers(1, m + 1, size=per_gpu, dtype=np.uint64) for m in spec.reg_masks]
        host = regs[0] | (regs[1] << np.uint64(19)) | (regs[2] << np.uint64(41))
        starts = torch.from_numpy(host.view(np.int64)).to(dev)
    STRIDE_, LEGS = args.stride, args.legs
    dst = torch.empty(batch * LEGS, dtype=torch.int64, device=dev)
    dist_ = torch.empty(batch * LEGS, dtype=torch.int64, device=dev)
    stats = torch.zeros((max(args.steps, 1), words), dtype=torch.int64, device=dev)
    wstats = torch.zeros(words, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def walk(b: int, out_stats) -> None:
        s = starts[b * batch:(b + 1) * batch]
        N.check(N.lib.lc_walk_device(ctx.handle, C.byref(sspec), params.fixed_r3, C.c_void_p(s.data_ptr()),
                                     s.numel(), STRIDE_, CAP, LEGS,
                                     args.refill, C.c_void_p(dst.data_ptr()), C.c_void_p(dist_.data_ptr()),
                                     hist_lo, hist_shift, hist_bins, C.c_void_p(out_stats.data_ptr()),
                                     C.c_void_p(stream.cuda_stream)))

    # roofline denominator: measured LOP3 issue rate of this GPU
    lop3_peak, peak_mhz = N.lop3_peak(local)

    for w in range(args.warmup):
        flush.zero_()
        walk(w % nbatches, wstats)
    torch.cuda.synchronize()

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    e_all0, e_all1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    N.launch_count_reset()
    with ClockSampler(local) as clocks:
        e_all0.record(stream)
        for k in range(args.steps):
            flush.zero_()
            ev[k][0].record(stream)
            walk(k % nbatches, stats[k])
            ev[k][1].record(stream)
        e_all1.record(stream)
        torch.cuda.synchronize()
    launches = N.launch_count()
    if world > 1:
        dist.barrier()
    elapsed = e_all0.elapsed_time(e_all1) / 1e3
    kernel_s = [a.elapsed_time(b) / 1e3 for a, b in ev]

    # per-rank totals -> one NCCL all-reduce of the statistics block
    from paper_1210_6411_b200.distributed import combine_stats

    local_stats = combine_stats([stats[k].cpu().numpy().view(np.uint64) for k in range(args.steps)])
    if int(local_stats[N.ST_ERROR]):
        raise SystemExit(f"walk error {int(local_stats[N.ST_ERROR])}")
    glob = allreduce_stats(local_stats) if world > 1 else local_stats
    t_max = elapsed
    if world > 1:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    summ = stats_summary(glob)
    value = summ["transitions"] / t_max
    edges_per_s = summ["edges"] / t_max

    # roofline of the dominant kernel (walk): algorithmic LOP3 per launch / launch time
    local_summ = stats_summary(local_stats)
    per_launch_tr = local_summ["transitions"] / args.steps
    achieved = per_launch_tr * LOP3_PER_TRANSITION / (sum(kernel_s) / len(kernel_s))

    # e2e: the public host-buffer C ABI call (lc_walk), pinned host memory, copies inside
    e2e = None
    if not args.no_e2e:
        hp = [C.c_void_p() for _ in range(4)]
        sizes = (batch, batch * LEGS, batch * LEGS, words)
        for p, n in zip(hp, sizes):
            N.check(N.lib.lc_host_alloc(n * 8, C.byref(p)))
        h_starts, h_dst, h_dist, h_stats = (np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(n,))
                                            for p, n in zip(hp, sizes))
        e2e_tr = 0
        e2e_el = 0.0
        if world > 1:
            dist.barrier()
        for k in range(args.steps):
            b = k % nbatches
            h_starts[:] = starts[b * batch:(b + 1) * batch].cpu().numpy().view(np.uint64)
            t0 = time.perf_counter()
            N.check(N.lib.lc_walk(ctx.handle, C.byref(sspec), params.fixed_r3, N.u64p(h_starts), batch, STRIDE_,
                                  CAP, LEGS, args.refill, N.u64p(h_dst), N.u64p(h_dist), hist_lo,
                                  hist_shift, hist_bins, N.u64p(h_stats)))
            e2e_el += time.perf_counter() - t0
            e2e_tr += int(h_stats[N.ST_TRANSITIONS])
        if world > 1:
            t = torch.tensor([e2e_el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_el = float(t.item())
            tt = torch.tensor([e2e_tr], dtype=torch.int64, device=dev)
            dist.all_reduce(tt)
            e2e_tr = int(tt.item())
        e2e = {"value": e2e_tr / e2e_el, "unit": "transitions/s", "h2d_bytes_per_step": batch * 8,
               "d2h_bytes_per_step": batch * LEGS * 16 + words * 8,
               "note": "lc_walk host-buffer C ABI call from pinned memory, wall clock"}
        for p in hp:
            N.lib.lc_host_free(p)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        sample = starts[: cores * 256].cpu().numpy().view(np.uint64)
        cpu_tr, cpu_ed, cpu_s, cdst, cdist = cpu_walk_sample(sample, cores)
        # the sample doubles as a parity check of the GPU walk on the same starts
        res = lc.walk_arrays(sample, params, spec, stride=STRIDE)
        parity = bool((res.dst[:, 0] == cdst).all() and (res.dist[:, 0] == cdist).all())
        cpu = {"value": cpu_tr, "unit": "transitions/s", "cores": cores, "kind": "port",
               "sample": f"first {sample.size} starts of the workload ({cpu_s:.1f} s), 256-lane waves",
               "edges_per_s": cpu_ed, "matches_gpu": parity}

    if rank == 0:
        clk = clocks.summary()
        sms = ctx.sm_count
        line = {
            "metric": METRIC, "value": value, "unit": "transitions/s", "edges_per_s": edges_per_s,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / args.steps, "higher_is_better": True,
            "scaling": "strong" if args.total_log2 else "weak",
            "vs_baseline": value / PAPER_GTX580,
            "vs_baseline_ref": "paper GTX 580 bitsliced walk, 9,800 nodes/s x 11.17e6 clocks (PAPER.md:478-479)",
            "dtype": "u32 (bitsliced words, 32 lanes)",
            "data": "synthetic (" + ("K0 seeded special A5/1 nodes" if args.starts == "k0"
                                     else "seeded uniform random valid A5/1 states") + ")",
            "config": {"workload": (f"configs[3]: 2^{args.total_log2} in total, " if args.total_log2 else "configs[1]: ")
                                   + f"2^{args.workload_log2} "
                                   f"{'special A5/1 start nodes' if args.starts == 'k0' else 'uniform random A5/1 states'}"
                                   f" per GPU, walked {LEGS} hop(s) to the next special node, stride {STRIDE_}; "
                                   f"one step = one batch of 2^{args.batch_log2}", "starts_per_step_per_gpu": batch,
                       "parallelism": f"dp{world} (independent start shards, stats all-reduce only)",
                       "l2": "flushed (256 MiB write) before every step", "refill": args.refill or "auto"},
            "gpu_launches": launches,
            "walk_stats": {k: summ[k] for k in ("edges", "transitions", "mean", "sd", "min", "max") if k in summ},
            "roofline": {"bound": "int-alu (LOP3 issue)", "achieved": achieved / 1e12, "peak": lop3_peak / 1e12,
                         "unit": "TLOP3/s", "frac": achieved / lop3_peak,
                         "traffic": TRAFFIC_BYTES_PER_WALK * batch,
                         "traffic_note": "DRAM bytes per launch: ncu dram__bytes_read+write per walk "
                                         "(profiles/r01_walk_a51_metrics.json) x walks per launch; "
                                         "algorithmic 24 B/walk (8 in, 16 out)",
                         "algorithmic": "2.25 LOP3 per transition (72 per 32-lane step)",
                         "kernel_ms_per_launch": 1e3 * sum(kernel_s) / len(kernel_s),
                         "peak_source": f"measured lop3 microbenchmark ({peak_mhz:.0f} MHz), "
                                        f"spec {sms}x64x{(clk.get('sm_max_mhz') or 1965):.0f} MHz = "
                                        f"{sms * 64 * (clk.get('sm_max_mhz') or 1965) * 1e6 / 1e12:.2f} T/s"},
            "clocks": clk,
            # configs[4]: paper-scale step 3 (~2^33.6 skeleton nodes x 11,184,857 clocks,
            # PAPER.md:490, :672) at this run's per-GPU rate on 8 GPUs
            "projection": {"paper_scale_transitions": PAPER_SCALE_TRANSITIONS,
                           "hours_on_8_gpus": PAPER_SCALE_TRANSITIONS / (8 * value / world) / 3600,
                           "paper": "9 d 3 h on 5x Tesla C1060; 4 d 8 h projected on 5x GTX 580 (PAPER.md:486-487)"},
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
