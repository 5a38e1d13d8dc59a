"""Benchmark of the step-3 chain walk (BASELINE.json metric: A5/1 transitions/s and
weighted edges/s) on 1..8 B200s, one process per GPU.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N ...

Workload (BASELINE.json configs[1]): per GPU 2^24 special A5/1
start nodes drawn by the reference's own sampler, `random_candidate(random.Random(seed),
A51, 0x2AAA00)` x 2^24 (pipeline.py:301-310; csrc/sampler.cu reproduces CPython's
stream), rank r using seed r -- so rank 0's set is config 2 and its first 2^16 starts are
config 1.  A step walks one batch of 2^22 of them to their next special node (stride
11,170,000, as the reference's benchmark and the paper), cycling through the 4 batches.
Weak scaling: every rank walks its own 2^24-start stream.  `--total-log2 30` is
configs[3] (2^30 starts = 64 streams of 2^24, seeds 0..63, split over the ranks; strong
scaling).  Timing: CUDA events on the launching stream, barrier + synchronize on both
sides, max over ranks; L2 is flushed (256 MiB write) before every step.  One NCCL
all-reduce after the timed region gathers the chain-length histogram and edge counts.

Parity (outside the timed region, in the JSON line): every batch's (dst, dist) is hashed
and compared with tests/golden/a51_c2_digests.json (the pinned restatement over the
reference's own 2^24 starts), and the first 2^16 rows with the reference's own config-1
run (tests/golden/a51_c1_65536.json).

`--impl reference` times the reference algorithm on the host cores instead (the C
restatement in oracle/, since the Python reference cannot travel to the GPU box); it
does not import the product package.
"""

from __future__ import annotations

import argparse
import ctypes as C
import hashlib
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
F = 0x2AAA00
STRIDE = 11_170_000
CAP = 178_957_008  # the reference's default walk cap for A5/1 (bitslice.py:273-274)
STREAM = 1 << 24   # starts per seeded stream (config 2)
GOLDEN_BATCH = 1 << 22
PAPER_SCALE_TRANSITIONS = int(2 ** 33.6 * 11_184_857)  # ~1.46e17
GOLDEN = os.path.join(ROOT, "tests", "golden")
PROFILES = os.path.join(ROOT, "profiles")


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def workload(args, world: int) -> dict:
    """`config` of the JSON line -- identical in both arms for the same flags."""
    total = (1 << args.total_log2) if args.total_log2 else world << args.workload_log2
    per_gpu = total // world
    if args.starts == "ref":
        src = ("special A5/1 start nodes from the reference sampler random_candidate(random.Random(seed), "
               "A51, 0x2AAA00) (pipeline.py:301-310), one seed per 2^24-start stream")
    elif args.starts == "k0":
        src = "special A5/1 start nodes from the K0 counter-based generator"
    else:
        src = "uniform random valid A5/1 states"
    head = f"configs[3]: 2^{args.total_log2} starts in total" if args.total_log2 else \
        f"configs[1]: 2^{args.workload_log2} starts per GPU"
    return {"workload": f"{head}, {src}, walked {args.legs} hop(s) to the next special node, stride {args.stride}",
            "starts_per_gpu": per_gpu, "stride": args.stride, "legs": args.legs,
            "parallelism": f"dp{world} (independent start shards, statistics all-reduce only)",
            "l2": "flushed (256 MiB write) before every timed GPU step"}


def stream_seeds(args, rank: int, world: int) -> list:
    """Seeds of the 2^24-start streams this rank walks (rank 0 of a weak-scaling run and
    the first shard of a strong-scaling run hold seed 0 = config 2)."""
    total = (1 << args.total_log2) if args.total_log2 else world << args.workload_log2
    per_gpu = total // world
    per = max(1, per_gpu // STREAM)
    return [rank * per + i for i in range(per)]


def cpu_walk_sample(starts: np.ndarray, cores: int):
    """The reference algorithm on the host cores (the C restatement, OpenMP, 256-lane
    waves like the reference's _edges_chunk chunks).  Returns (transitions/s, edges/s, s,
    dst, dist).  Imports nothing from the product package."""
    from oracle import port

    os.environ["OMP_NUM_THREADS"] = str(cores)
    t0 = time.perf_counter()
    dst, dist = port.walk(port.A51, F, starts, stride=STRIDE, width=256)
    el = time.perf_counter() - t0
    return float(dist.sum()) / el, starts.size / el, el, dst[:, 0], dist[:, 0]


def batch_digest(dst: np.ndarray, dist: np.ndarray) -> str:
    """oracle/gen_golden.py batch_digest: sha256(dst <u8 || dist <u8), input order."""
    h = hashlib.sha256(np.ascontiguousarray(dst, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(dist, dtype="<u8").tobytes())
    return h.hexdigest()


def u64_digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<u8").tobytes()).hexdigest()


def load_json(path: str):
    try:
        with open(path) as f:
            return json.load(f)
    except OSError:
        return None


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


def reference_arm(args, rank: int, world: int) -> None:
    """--impl reference: the reference algorithm (the C restatement, oracle/port) on all
    host cores, on bounded samples of the same workload; rank 0 only.  The starts are the
    same reference-sampler stream (Python's own random.Random, restated predicate), so
    this arm loads nothing but oracle/_build/liboracle.so."""
    if rank != 0:
        return
    from oracle import port

    cores = host_cores()
    per_step = cores * 256
    starts = port.random_candidates(port.A51, F, 0, per_step * min(max(args.steps, 1), 2))
    for w in range(args.warmup):
        cpu_walk_sample(starts[(w % 2) * per_step:(w % 2 + 1) * per_step], cores)
    tr = ed = el = 0.0
    for k in range(args.steps):
        s = starts[(k % 2) * per_step:(k % 2 + 1) * per_step]
        _, _, dt, _, dist = cpu_walk_sample(s, cores)
        tr += float(dist.sum())
        ed += s.size
        el += dt
    value = tr / el
    sample = (f"{per_step} starts per step (the first {min(args.steps, 2) * per_step} of the seed-0 stream, "
              f"alternating), 256-lane waves, {cores} threads")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "transitions/s",
        "edges_per_s": ed / el, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * el / max(args.steps, 1), "higher_is_better": True,
        "scaling": "strong" if args.total_log2 else "weak",
        "vs_baseline": None, "dtype": "u64 (64-lane bitsliced words)",
        "data": "synthetic (seeded special A5/1 nodes)",
        "config": workload(args, world),
        "sample": sample,
        "cpu_baseline": {"value": value, "unit": "transitions/s", "cores": cores, "kind": "port", "sample": sample},
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
    ap.add_argument("--starts", default="ref", choices=["ref", "k0", "random"],
                    help="ref: the reference sampler (the metric's workload); k0: the K0 generator; "
                         "random: uniform valid states")
    ap.add_argument("--legs", type=int, default=1)
    ap.add_argument("--stride", type=int, default=STRIDE)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-steps12", action="store_true")
    ap.add_argument("--no-next", action="store_true")  # skip the §8(f) sort / leaf-cut object
    args = ap.parse_args()
    args.warmup = max(args.warmup, 0)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.total_log2:
        if (1 << args.total_log2) % world or world & (world - 1):
            raise SystemExit("--total-log2 needs a power-of-two world size")
        args.workload_log2 = args.total_log2 - (world.bit_length() - 1)

    if args.impl == "reference":
        reference_arm(args, rank, world)
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
    nccl = None
    # LFSR_BENCH_NCCL=1 (testing only): a one-rank NCCL communicator under torchrun, so the
    # NCCL data plane (statistics all-reduce, max-over-ranks timing) runs on a one-GPU box
    force_nccl = os.environ.get("LFSR_BENCH_NCCL") == "1" and "RANK" in os.environ
    if world > 1 or force_nccl:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
            nccl = {"world_size": dist.get_world_size(), "backend": dist.get_backend(),
                    "nccl_version": ".".join(map(str, torch.cuda.nccl.version()))}
            if rank == 0:
                print(f"[bench] NCCL communicator: {nccl['world_size']} ranks, NCCL {nccl['nccl_version']}",
                      file=sys.stderr, flush=True)

    multi = world > 1 or nccl is not None  # collectives run (a one-rank NCCL communicator too)

    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N
    from paper_1210_6411_b200.distributed import allreduce_stats, combine_stats, stats_summary

    lc.set_device(local)
    spec = lc.A51
    params = lc.CandidateParams.from_spec(spec, F)
    ctx = N.context(local)
    sspec = N.spec_struct(spec)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)  # explicit stream: kernels and events share it
    torch.cuda.set_stream(stream)

    per_gpu = 1 << args.workload_log2
    batch = min(1 << args.batch_log2, per_gpu)
    nbatches = max(1, per_gpu // batch)
    hist_lo, hist_shift, hist_bins = 11_184_809 - (1 << 15), 0, 1 << 16
    words = N.ST_HEADER + hist_bins + 2
    seeds = stream_seeds(args, rank, world)

    t_setup = time.perf_counter()
    if args.starts == "ref":
        # this rank's streams of the reference sampler, generated on the host cores (one
        # thread per stream) and kept resident in HBM
        host = lc.pipeline.reference_candidate_streams(spec, params, seeds, min(per_gpu, STREAM)).reshape(-1)
        starts = torch.from_numpy(host.view(np.int64)).to(dev)
    elif args.starts == "k0":
        starts = torch.empty(per_gpu, dtype=torch.int64, device=dev)
        N.check(N.lib.lc_random_candidates_device(ctx.handle, C.byref(sspec), params.fixed_r3, 1210_6411 + rank,
                                                  per_gpu, C.c_void_p(starts.data_ptr()),
                                                  C.c_void_p(stream.cuda_stream)))
    else:
        rng = np.random.default_rng(1210_6411 + rank)
        regs = [rng.integers(1, m + 1, size=per_gpu, dtype=np.uint64) for m in spec.reg_masks]
        host = regs[0] | (regs[1] << np.uint64(19)) | (regs[2] << np.uint64(41))
        starts = torch.from_numpy(host.view(np.int64)).to(dev)
    setup_s = time.perf_counter() - t_setup
    STRIDE_, LEGS = args.stride, args.legs
    # outputs of the whole per-GPU workload stay resident (each batch writes its slice), so
    # every batch can be checked after the timed region
    dst = torch.empty(per_gpu * LEGS, dtype=torch.int64, device=dev)
    dist_ = torch.empty(per_gpu * LEGS, dtype=torch.int64, device=dev)
    stats = torch.zeros((max(args.steps, 1), words), dtype=torch.int64, device=dev)
    wstats = torch.zeros(words, dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    def walk(b: int, out_stats) -> None:
        s = starts[b * batch:(b + 1) * batch]
        o = b * batch * LEGS
        N.check(N.lib.lc_walk_device(ctx.handle, C.byref(sspec), params.fixed_r3, C.c_void_p(s.data_ptr()),
                                     s.numel(), STRIDE_, CAP, LEGS, args.refill,
                                     C.c_void_p(dst[o:].data_ptr()), C.c_void_p(dist_[o:].data_ptr()),
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
    if multi:
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
    if multi:
        dist.barrier()
    elapsed = e_all0.elapsed_time(e_all1) / 1e3
    kernel_s = [a.elapsed_time(b) / 1e3 for a, b in ev]

    # per-rank totals -> one NCCL all-reduce of the statistics block
    local_stats = combine_stats([stats[k].cpu().numpy().view(np.uint64) for k in range(args.steps)])
    if int(local_stats[N.ST_ERROR]):
        raise SystemExit(f"walk error {int(local_stats[N.ST_ERROR])}")
    glob = allreduce_stats(local_stats, offset=rank * per_gpu) if multi else local_stats
    t_max = elapsed
    if multi:
        t = torch.tensor([elapsed], dtype=torch.float64, device=dev if nccl else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_max = float(t.item())
    summ = stats_summary(glob)
    value = summ["transitions"] / t_max
    edges_per_s = summ["edges"] / t_max

    # roofline of the dominant kernel (walk): algorithmic LOP3 per launch / launch time
    local_summ = stats_summary(local_stats)
    per_launch_tr = local_summ["transitions"] / max(args.steps, 1)
    achieved = per_launch_tr * LOP3_PER_TRANSITION / (sum(kernel_s) / len(kernel_s))

    # ---- parity (untimed): batches of this rank's first 2^24-start stream that the timed
    # steps did not reach are walked now, then that stream is hashed; rank 0's seed-0
    # stream (config 2) has committed digests
    checked = min(per_gpu, STREAM)
    for b in range(min(args.steps, nbatches), min(nbatches, max(1, checked // batch))):
        walk(b, wstats)
    torch.cuda.synchronize()
    parity = None
    if args.starts == "ref" and LEGS == 1 and STRIDE_ == STRIDE:
        h_dst = dst[:checked].cpu().numpy().view(np.uint64)
        h_dist = dist_[:checked].cpu().numpy().view(np.uint64)
        parity = {"edge_digest": batch_digest(h_dst, h_dist), "walks_hashed": int(h_dst.size)}
        if seeds[0] == 0 and per_gpu >= STREAM:
            c1 = load_json(os.path.join(GOLDEN, "a51_c1_65536.json"))
            c2 = load_json(os.path.join(GOLDEN, "a51_c2_digests.json"))
            if c1:
                parity["c1_reference_digest"] = bool(u64_digest(h_dst[:1 << 16]) == c1["dst_digest"] and
                                                     u64_digest(h_dist[:1 << 16]) == c1["dist_digest"])
            if c2:
                parity["c2_starts_digest"] = bool(u64_digest(host[:STREAM]) == c2["starts_digest"]) \
                    if args.starts == "ref" else None
                parity["c2_batches"] = [bool(batch_digest(h_dst[g["index"] * GOLDEN_BATCH:(g["index"] + 1) * GOLDEN_BATCH],
                                                          h_dist[g["index"] * GOLDEN_BATCH:(g["index"] + 1) * GOLDEN_BATCH])
                                             == g["digest"]) for g in c2["batches"]]
                parity["c2_set"] = bool(u64_digest(h_dst[:STREAM]) == c2["dst_digest"] and
                                        u64_digest(h_dist[:STREAM]) == c2["dist_digest"])
            else:
                parity["c2_batches"] = "tests/golden/a51_c2_digests.json missing"
            parity["golden"] = ("c1: the reference's own _edges_chunk run (tests/golden/a51_c1_65536.json); "
                                "c2: oracle/walk512.c over the reference's 2^24 starts, pinned on c1 "
                                "(tests/golden/a51_c2_digests.json)")
        del h_dst, h_dist

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
        e2e_match = []
        d_all = dst.view(torch.int64)
        if multi:
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
            if k < nbatches:  # the host-buffer results equal the device path's, batch by batch
                o = b * batch * LEGS
                e2e_match.append(bool((h_dst == d_all[o:o + batch * LEGS].cpu().numpy().view(np.uint64)).all()))
        if multi:
            t = torch.tensor([e2e_el], dtype=torch.float64, device=dev if nccl else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_el = float(t.item())
            tt = torch.tensor([e2e_tr], dtype=torch.int64, device=dev if nccl else "cpu")
            dist.all_reduce(tt)
            e2e_tr = int(tt.item())
        e2e = {"value": e2e_tr / e2e_el, "unit": "transitions/s", "h2d_bytes_per_step": batch * 8,
               "d2h_bytes_per_step": batch * LEGS * 16 + words * 8,
               "note": "lc_walk host-buffer C ABI call from pinned memory, wall clock",
               "dst_equal_to_device_path": all(e2e_match) if e2e_match else None}
        for p in hp:
            N.lib.lc_host_free(p)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cores = host_cores()
        sample = starts[: cores * 256 * 3].cpu().numpy().view(np.uint64)
        cpu_tr, cpu_ed, cpu_s, cdst, cdist = cpu_walk_sample(sample, cores)
        # the sample doubles as a parity check of the GPU walk on the same starts
        gd = dst[: sample.size * LEGS].cpu().numpy().view(np.uint64)[::LEGS]
        gw = dist_[: sample.size * LEGS].cpu().numpy().view(np.uint64)[::LEGS]
        cpu = {"value": cpu_tr, "unit": "transitions/s", "cores": cores, "kind": "port",
               "sample": f"first {sample.size} starts of the workload ({cpu_s:.1f} s), 256-lane waves, "
                         f"C restatement of bitslice._run_walks (oracle/lfsr_oracle.c)",
               "edges_per_s": cpu_ed, "matches_gpu": bool((gd == cdst).all() and (gw == cdist).all())}

    steps12 = None
    if rank == 0 and world == 1 and not args.no_steps12:
        import bench_steps12

        torch.cuda.empty_cache()
        steps12 = bench_steps12.measure(ctx, stream, prune_log2=27, cpu_sample=1 << 16,
                                        lop3_peak=(lop3_peak, peak_mhz))
    next_rows = None
    if rank == 0 and world == 1 and not args.no_next:
        import bench_reduce

        torch.cuda.empty_cache()
        next_rows = bench_reduce.measure_next()

    if rank == 0:
        clk = clocks.summary()
        sms = ctx.sm_count
        f_mhz = clk.get("sm_max_mhz") or 1965.0
        spec128 = sms * 128 * f_mhz * 1e6
        ncu = load_json(os.path.join(PROFILES, "r01_walk_a51_metrics.json")) or {}

        def ncu_pct(key):
            v = ncu.get(key, {}).get("value")
            return float(v) if v is not None else None

        line = {
            "metric": METRIC, "value": value, "unit": "transitions/s", "edges_per_s": edges_per_s,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * t_max / max(args.steps, 1), "higher_is_better": True,
            "scaling": "strong" if args.total_log2 else "weak",
            "vs_baseline": value / PAPER_GTX580,
            "vs_baseline_ref": "paper GTX 580 bitsliced walk, 9,800 nodes/s x 11.17e6 clocks (PAPER.md:478-479)",
            "dtype": "u32 (bitsliced words, 32 lanes)",
            "data": "synthetic (" + {"ref": "reference-sampler special A5/1 nodes", "k0": "K0 seeded special A5/1 nodes",
                                     "random": "seeded uniform random valid A5/1 states"}[args.starts] + ")",
            "config": workload(args, world),
            "starts_per_step_per_gpu": batch, "refill": args.refill or "auto",
            "seeds_rank0": seeds[:4] + (["..."] if len(seeds) > 4 else []),
            "setup_s": setup_s,
            "gpu_launches": launches,
            "walk_stats": {k: summ[k] for k in ("edges", "transitions", "mean", "sd", "min", "max") if k in summ},
            "parity": parity,
            "roofline": {"bound": "int-alu (LOP3 issue)", "achieved": achieved / 1e12, "peak": lop3_peak / 1e12,
                         "unit": "TLOP3/s", "frac": achieved / lop3_peak,
                         "peak_source": f"measured: lc_lop3_peak microbenchmark on this GPU = {sms} SMs x 64 LOP3/clk "
                                        f"x {peak_mhz:.0f} MHz (the ALU pipe issues one 32-lane LOP3 every 2 "
                                        f"cycles per SM sub-partition)",
                         "peak_spec_128": spec128 / 1e12, "frac_spec_128": achieved / spec128,
                         "peak_spec_128_source": f"spec-style SMs x 128 lanes x clock = {sms} x 128 x {f_mhz:.0f} MHz "
                                                 "(not reachable by LOP3: see peak_source)",
                         "traffic": None,
                         "traffic_note": "ncu dram__bytes_read+write of a 2^20-walk launch = 55 B/walk "
                                         "(profiles/r01_walk_a51_metrics.json) vs 24 B algorithmic (8 in, 16 out); "
                                         "~5e-6 B per transition, irrelevant to an ALU-bound kernel",
                         "algorithmic": "2.25 LOP3 per transition (72 per 32-lane step)",
                         "kernel_ms_per_launch": 1e3 * sum(kernel_s) / len(kernel_s),
                         "ncu": {"sm__pipe_alu_cycles_active_pct_active":
                                 ncu_pct("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                                 "smsp__issue_active_pct_active":
                                 ncu_pct("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                                 "registers_per_thread": ncu_pct("launch__registers_per_thread"),
                                 "source": "profiles/r01_walk_a51_metrics.json"}},
            "clocks": clk,
            # configs[4]: paper-scale step 3 (~2^33.6 skeleton nodes x 11,184,857 clocks,
            # PAPER.md:490, :672) at this run's per-GPU rate on 8 GPUs
            "projection": {"paper_scale_transitions": PAPER_SCALE_TRANSITIONS,
                           "hours_on_8_gpus": PAPER_SCALE_TRANSITIONS / (8 * value / world) / 3600,
                           "basis": "this run's per-GPU rate x 8 (independent shards, no data-path collective)",
                           "paper": "9 d 3 h on 5x Tesla C1060; 4 d 8 h projected on 5x GTX 580 (PAPER.md:486-487)"},
            "nccl": nccl,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "steps12": steps12,
            "next_rows": next_rows,
        }
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
