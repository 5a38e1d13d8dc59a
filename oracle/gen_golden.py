"""TEST INFRASTRUCTURE ONLY -- generates tests/golden/ fixtures from the reference.

Runs the *unmodified* reference (``lfsrcycles`` under /root/reference, imported via
``oracle/ref_shim.py``) on seeded inputs and writes small fixtures that travel with
the repo (the reference itself does not exist on the GPU box).  Every fixture names
the reference function that produced it.

Usage (from the repo root, in the build container):

    python oracle/gen_golden.py basic      # seconds: tables, trajectories, minis, predicates
    python oracle/gen_golden.py prune      # ~1 min: step-2 prune fixtures
    python oracle/gen_golden.py enumerate  # ~30 s: A5/1 step-1 sub-slice digest
    python oracle/gen_golden.py kat        # ~2 min: A5/1 seed-0 256-walk known answer
    python oracle/gen_golden.py reduce     # ~1 min: steps 4-5 (leaf cutting, cycles) on minis
    python oracle/gen_golden.py bruteforce # ~2 min: the reference's exhaustive mini analysis
    python oracle/gen_golden.py c1 [W]     # ~1 h on 8 cores: the full 2^16 config-1 set
    python oracle/gen_golden.py c2         # ~40 min on 8 AVX-512 cores: config-2 (2^24) digests

Digest format: sha256 over lines
``f"{src:016x} {dst:016x} {dist}\\n"`` sorted by (src, dst, dist).
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import ref_shim  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(HERE), "tests", "golden")
SEED_C1 = 0
A51_STRIDE = 11_170_000


def edge_digest(src, dst, dist) -> str:
    rows = sorted(zip((int(s) for s in src), (int(d) for d in dst), (int(w) for w in dist)))
    h = hashlib.sha256()
    for s, d, w in rows:
        h.update(f"{s:016x} {d:016x} {w}\n".encode())
    return h.hexdigest()


def u64_digest(values) -> str:
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


def save(name, **arrays):
    path = os.path.join(GOLDEN, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path}.npz", {k: getattr(v, 'shape', v) for k, v in arrays.items()})


def save_json(name, doc):
    path = os.path.join(GOLDEN, name)
    with open(path, "w") as f:
        json.dump(doc, f, indent=1, sort_keys=True)
        f.write("\n")
    print(f"wrote {path}")


def random_states(ref, spec, n, seed):
    # same sampler as the reference tests (pkg/tests/conftest.py:43-46)
    rng = random.Random(seed)
    total = spec.valid_state_count
    return [ref.cipher.unrank_state(rng.randrange(total), spec) for _ in range(n)]


def mini_candidates(ref, spec, params, table):
    return list(ref.pipeline.enumerate_candidates(spec, params, table))


# ---------------------------------------------------------------------------------


def gen_basic(ref):
    C = ref.cipher
    B = ref.bitslice
    table = C.build_predecessor_table()
    doc = {
        "source": "lfsrcycles.cipher.build_predecessor_table (cipher.py:297-313)",
        "entries": [list(e) for e in table.entries],
        "nonempty_mask": hex(sum(1 << i for i, e in enumerate(table.entries) if e)),
    }
    specs = {}
    for spec in (C.A51, C.MINI567, C.MINI789):
        p = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        specs[spec.name] = {
            "lengths": list(spec.lengths), "taps": [list(t) for t in spec.taps],
            "clock_taps": list(spec.clock_taps), "default_fixed_r3": p.fixed_r3,
            "packed_r3": p.packed_r3, "r3_field_mask": p.r3_field_mask,
            "min_cycle_num": C.minimum_cycle_length(spec).numerator,
            "min_cycle_den": C.minimum_cycle_length(spec).denominator,
            "default_cap": 16 * int(C.minimum_cycle_length(spec)) + 64,
        }
    doc["specs"] = specs
    save_json("tables.json", doc)

    # trajectories: clock_forward iterated (cipher.py:228-253)
    for spec in (C.A51, C.MINI567, C.MINI789):
        starts = random_states(ref, spec, 256, seed=1000 + spec.total_bits)
        traj = np.zeros((256, 64), dtype=np.uint64)
        for j, x in enumerate(starts):
            for t in range(64):
                x = C.clock_forward(x, spec)
                traj[j, t] = x
        # longer horizon for the sliced-engine tests: clock_sliced (bitslice.py:223-228)
        sb = B.clock_sliced(B.transpose(starts, spec, 256), spec, 500)
        save(f"traj_{spec.name}", starts=np.array(starts, dtype=np.uint64), traj=traj,
             after500=np.array(B.untranspose(sb), dtype=np.uint64))

    # predicates on random states: is_candidate (cipher.py:420-428), predecessors (:342-369)
    for spec in (C.A51, C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        xs = random_states(ref, spec, 4000, seed=77)
        # half of them moved onto the fixed-R3 plane so the predicate is exercised
        xs = [((x & ~params.r3_field_mask) | params.packed_r3) if i % 2 else x for i, x in enumerate(xs)]
        cand = np.array([C.is_candidate(x, params, spec, table) for x in xs], dtype=np.uint8)
        preds = np.zeros((len(xs), 4), dtype=np.uint64)
        npred = np.zeros(len(xs), dtype=np.uint8)
        for i, x in enumerate(xs):
            ps = C.predecessors(x, spec, table)
            npred[i] = len(ps)
            preds[i, :len(ps)] = ps
        tidx = np.array([C.table_index(x, spec) for x in xs], dtype=np.uint8)
        save(f"pred_{spec.name}", states=np.array(xs, dtype=np.uint64), is_candidate=cand,
             npred=npred, preds=preds, table_index=tidx)

    # minis: every candidate's edge, and the independent brute-force oracle's edges
    for spec in (C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        cands = mini_candidates(ref, spec, params, table)
        edges = ref.pipeline.build_skeleton_edges(cands, params, spec, table)
        gt = ref.oracle.brute_force_analysis(spec, params)
        emap = gt.candidate_edge_map()
        assert all(emap[e.source] == (e.destination, e.distance) for e in edges)
        src = np.array([e.source for e in edges], dtype=np.uint64)
        dst = np.array([e.destination for e in edges], dtype=np.uint64)
        dist = np.array([e.distance for e in edges], dtype=np.uint64)
        # random (non-candidate) starts, stride 1 (bitslice.py:326-342)
        rs = random_states(ref, spec, 300, seed=9)
        rw = B.forward_to_candidate(rs, params, spec, table)
        # stride variants on the candidate set
        strides = {}
        for s in (16, 100, 127, 148, 149, 150, 200):
            w = B.forward_to_candidate(cands, params, spec, table, stride=s)
            strides[f"stride_{s}_dst"] = np.array([d for d, _ in w], dtype=np.uint64)
            strides[f"stride_{s}_dist"] = np.array([k for _, k in w], dtype=np.uint64)
        # two- and three-leg hops from random starts (bitslice.py:345-354)
        hs = random_states(ref, spec, 200, seed=10)
        h2 = B.candidate_hops(hs, params, spec, table, legs=2)
        h3 = B.candidate_hops(hs, params, spec, table, legs=3)
        save(f"edges_{spec.name}", src=src, dst=dst, dist=dist,
             random_starts=np.array(rs, dtype=np.uint64),
             random_dst=np.array([d for d, _ in rw], dtype=np.uint64),
             random_dist=np.array([k for _, k in rw], dtype=np.uint64),
             hop_starts=np.array(hs, dtype=np.uint64),
             hop2=np.array([[v for leg in h for v in leg] for h in h2], dtype=np.uint64),
             hop3=np.array([[v for leg in h for v in leg] for h in h3], dtype=np.uint64),
             **strides)
        summary = {
            "count": len(cands), "sum_dist": int(dist.sum()), "min": int(dist.min()),
            "max": int(dist.max()), "digest": edge_digest(src, dst, dist),
            "oracle_node_count": gt.node_count, "oracle_cycles": gt.component_count,
            "oracle_on_cycle": gt.on_cycle_states, "oracle_leaf_count": gt.leaf_count,
            "oracle_max_segment_depth": int(gt.seg_depth.max()),
        }
        # calibrate_stride as shipped (bitslice.py:357-376); sampled, can overshoot
        summary["calibrate_stride"] = {
            f"{n}_{sd}": B.calibrate_stride(spec, params, table, samples=n, seed=sd)
            for n, sd in ((500, 0), (2000, 1))
        }
        save_json(f"edges_{spec.name}.json", summary)

    # walk cap -> StrideError and the documented ValueError band
    params = C.CandidateParams.from_spec(C.MINI567, C.default_fixed_r3(C.MINI567))
    first = mini_candidates(ref, C.MINI567, params, table)[0]
    band = {}
    for mc in range(150, 160):
        try:
            r = B.forward_to_candidate([first], params, C.MINI567, table, max_clocks=mc)
            band[mc] = ["ok", r[0][0], r[0][1]]
        except B.StrideError:
            band[mc] = ["StrideError"]
        except ValueError as exc:
            band[mc] = ["ValueError", str(exc)]
    starts = random_states(ref, C.MINI567, 4, seed=11)
    try:
        B.forward_to_candidate(starts, params, C.MINI567, table, max_clocks=3)
        cap3 = "ok"
    except B.StrideError:
        cap3 = "StrideError"
    save_json("cap_mini567.json", {"first_candidate": first, "band": band,
                                   "cap3_starts": starts, "cap3": cap3})

    # random_candidate stream (pipeline.py:301-310), seeds 0..3
    rc = {}
    for spec in (C.A51, C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        for seed in range(4):
            rng = random.Random(seed)
            rc[f"{spec.name}_{seed}"] = [ref.pipeline.random_candidate(rng, spec, params, table)
                                         for _ in range(64)]
    save_json("random_candidate.json", rc)

    # byte-exact record formats (records.py:24-106)
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        p = os.path.join(d, "e.bin")
        E = ref.records.EdgeRecord
        recs = [E(1, 2, 3, 4, 5), E((1 << 64) - 1, 0x5554000000000000, 11184809, 0, 0)]
        ref.records.write_edges(p, recs)
        eb = open(p, "rb").read()
        ref.records.write_states(p, [1, 0x5554000000000001, (1 << 64) - 1])
        sb = open(p, "rb").read()
    save_json("records.json", {"edges_hex": eb.hex(), "states_hex": sb.hex()})


def gen_prune(ref):
    C, P = ref.cipher, ref.pipeline
    table = C.build_predecessor_table()
    out = {}
    for spec in (C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        cands = mini_candidates(ref, spec, params, table)
        for mode, lim in (("dfs", 1), ("dfs", 4), ("dfs", 16), ("dfs", 60), ("bfs", 8), ("bfs", 64)):
            if lim >= (1 << spec.lengths[2]) - 1:
                continue
            cfg = P.PruneConfig(mode=mode, depth_limit=lim if mode == "dfs" else None,
                                node_limit=lim if mode == "bfs" else None)
            surv, st = P.prune_shallow_segments(cands, cfg, spec, params, table)
            out[f"{spec.name}_{mode}_{lim}"] = {
                "survivors_digest": u64_digest(surv), "surviving": len(surv),
                "total": st.total, "removed": st.removed, "expanded": st.expanded}
        # probe_segment (pipeline.py:262-298) on the first 64 candidates
        probes = []
        for x in cands[:64]:
            lc = []
            probes.append(list(P.probe_segment(x, spec, params, table, level_counts=lc)) + [lc])
        out[f"{spec.name}_probe"] = probes
    spec = C.A51
    params = C.CandidateParams.from_spec(spec, 0x2AAA00)
    rng = random.Random(4242)
    cands = [P.random_candidate(rng, spec, params, table) for _ in range(300)]
    out["a51_cands"] = cands
    for mode, lim in (("dfs", 56), ("dfs", 319), ("dfs", 3000), ("bfs", 1000), ("bfs", 100000)):
        t0 = time.time()
        cfg = P.PruneConfig(mode=mode, depth_limit=lim if mode == "dfs" else None,
                            node_limit=lim if mode == "bfs" else None)
        surv, st = P.prune_shallow_segments(cands, cfg, spec, params, table)
        out[f"a51_{mode}_{lim}"] = {
            "survivors": surv, "surviving": len(surv), "total": st.total,
            "removed": st.removed, "expanded": st.expanded}
        print(f"a51 {mode} {lim}: removed {st.removed}/{st.total} expanded {st.expanded} "
              f"({time.time() - t0:.1f}s)")
        # per-candidate work to pin the order-dependent DFS counter exactly
        if mode == "dfs" and lim <= 319:
            per = [P._dfs_is_shallow(x, lim, spec, params, table) for x in cands]
            out[f"a51_{mode}_{lim}"]["per_candidate"] = [[int(s), w] for s, w in per]
    save_json("prune.json", out)


def gen_enumerate(ref):
    C = ref.cipher
    table = C.build_predecessor_table()
    out = {}
    # minis: full enumeration (pipeline.py:104-118)
    for spec in (C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        cands = mini_candidates(ref, spec, params, table)
        out[spec.name] = {"count": len(cands), "digest": u64_digest(cands)}
    # A5/1: the enumeration inner loop restricted to R2 rows [r2_0, r2_0 + 4)
    spec = C.A51
    params = C.CandidateParams.from_spec(spec, 0x2AAA00)
    m1 = spec.reg_masks[0]
    o2 = spec.offsets[1]
    for r2_0 in (1, 0x1234, 0x3FFFFC):
        t0 = time.time()
        got = []
        for r2 in range(r2_0, r2_0 + 4):
            high = (r2 << o2) | params.packed_r3
            got.extend(high | r1 for r1 in range(1, m1 + 1)
                       if C.is_candidate(high | r1, params, spec, table))
        out[f"a51_rows_{r2_0:#x}_4"] = {"count": len(got), "digest": u64_digest(got),
                                        "first": got[:64], "last": got[-64:]}
        print(f"a51 rows {r2_0:#x}: {len(got)} candidates ({time.time() - t0:.1f}s)")
    save_json("enumerate.json", out)


def gen_reduce(ref):
    """Steps 4-5 on mini skeletons (reduce.py:118-266): full candidate sets and pruned
    skeletons, through the reference's own file-based pipeline."""
    import tempfile

    C, P, R, Rec = ref.cipher, ref.pipeline, ref.reduce, ref.records
    table = C.build_predecessor_table()
    out = {}
    for spec in (C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        cands = mini_candidates(ref, spec, params, table)
        gt = ref.oracle.brute_force_analysis(spec, params)
        out[f"{spec.name}_oracle_cycles"] = [list(c) for c in gt.cycle_multiset()]
        for label, cfg in (("full", None), ("dfs4", P.PruneConfig(mode="dfs", depth_limit=4)),
                           ("bfs8", P.PruneConfig(mode="bfs", node_limit=8))):
            skel = cands if cfg is None else P.prune_shallow_segments(cands, cfg, spec, params, table)[0]
            edges = P.build_skeleton_edges(skel, params, spec, table)
            with tempfile.TemporaryDirectory() as d:
                src = os.path.join(d, "edges.bin")
                dst = os.path.join(d, "fix.bin")
                Rec.write_edges(src, edges)
                one = os.path.join(d, "one.bin")
                st1 = R.cut_leaves_pass(src, one, R.ReduceConfig())
                one_recs = list(Rec.read_edges(one))
                # cut_leaves_to_fixpoint (reduce.py:189-223) raises "subtree size conservation
                # violated" on every input whose first pass removes a leaf: its expected total
                # (reduce.py:210-212) counts pass-1 leaves twice.  Iterate the reference's
                # own cut_leaves_pass to the fixpoint instead (what :203-219 intends).
                passes, cur, gen = [], src, 0
                while True:
                    nxt = os.path.join(d, f"gen{gen}.bin")
                    st = R.cut_leaves_pass(cur, nxt, R.ReduceConfig())
                    passes.append(st)
                    cur, gen = nxt, gen + 1
                    if st.leaves_removed == 0:
                        break
                try:
                    R.cut_leaves_to_fixpoint(src, dst, R.ReduceConfig())
                    fixpoint_raises = None
                except AssertionError as exc:
                    fixpoint_raises = str(exc)
                log = R.IterationLog(passes=passes)
                fix = list(Rec.read_edges(cur))
                cycles = R.count_cycles(cur)
            out[f"{spec.name}_{label}"] = {
                "skeleton": len(skel),
                "pass1": {"leaves_removed": st1.leaves_removed, "inner_nodes": st1.inner_nodes,
                          "out_size_sum": st1.out_size_sum, "records_digest": u64_digest(
                              [v for r in one_recs for v in r])},
                "passes": [[p.leaves_removed, p.inner_nodes, p.out_size_sum] for p in log.passes],
                "iterations": log.iterations, "reference_fixpoint_raises": fixpoint_raises,
                "fixpoint": [list(r) for r in fix],
                "cycles": [list(c) for c in cycles],
            }
            print(spec.name, label, len(skel), "passes", len(log.passes), "cycles", len(cycles))
    save_json("reduce.json", out)


def gen_tuning(ref):
    """auto_depth_limit (pipeline.py:313-333) and calibrate_stride (bitslice.py:357-376)
    outputs, and PruneConfig validation outcomes (pipeline.py:65-84)."""
    C, P, B = ref.cipher, ref.pipeline, ref.bitslice
    table = C.build_predecessor_table()
    out = {}
    for spec, sample, seed in ((C.MINI567, 256, 0), (C.MINI789, 256, 3), (C.A51, 24, 0), (C.A51, 256, 0)):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        t0 = time.time()
        out[f"auto_depth_{spec.name}_{sample}_{seed}"] = P.auto_depth_limit(spec, params, table, sample=sample,
                                                                            seed=seed)
        print(spec.name, "auto_depth_limit", out[f"auto_depth_{spec.name}_{sample}_{seed}"], f"{time.time() - t0:.1f}s")
    for spec in (C.MINI567, C.MINI789):
        params = C.CandidateParams.from_spec(spec, C.default_fixed_r3(spec))
        for n, sd in ((300, 5), (1000, 7)):
            out[f"calibrate_{spec.name}_{n}_{sd}"] = B.calibrate_stride(spec, params, table, samples=n, seed=sd)
    cfgs = {}
    for mode, d, nl, w in (("dfs", None, None, 1), ("dfs", 0, None, 1), ("dfs", 127, None, 1), ("dfs", 126, None, 1),
                           ("bfs", None, 10, 1), ("bfs", None, 127, 1), ("bfs", None, 0, 1), ("xyz", 3, 3, 1),
                           ("dfs", 3, None, 0)):
        try:
            P.PruneConfig(mode=mode, depth_limit=d, node_limit=nl, workers=w).validate(C.MINI567)
            cfgs[f"{mode}_{d}_{nl}_{w}"] = "ok"
        except ValueError:
            cfgs[f"{mode}_{d}_{nl}_{w}"] = "ValueError"
    out["prune_config_mini567"] = cfgs
    save_json("tuning.json", out)


def c1_starts(ref, n):
    C, P = ref.cipher, ref.pipeline
    table = C.build_predecessor_table()
    params = C.CandidateParams.from_spec(C.A51, 0x2AAA00)
    rng = random.Random(SEED_C1)
    return [P.random_candidate(rng, C.A51, params, table) for _ in range(n)]


def gen_kat(ref):
    C, B = ref.cipher, ref.bitslice
    table = C.build_predecessor_table()
    params = C.CandidateParams.from_spec(C.A51, 0x2AAA00)
    starts = c1_starts(ref, 256)
    t0 = time.time()
    w = B.forward_to_candidate(starts, params, C.A51, table, stride=A51_STRIDE)
    el = time.time() - t0
    dst = np.array([d for d, _ in w], dtype=np.uint64)
    dist = np.array([k for _, k in w], dtype=np.uint64)
    src = np.array(starts, dtype=np.uint64)
    save("a51_kat256", src=src, dst=dst, dist=dist)
    save_json("a51_kat256.json", {
        "source": "lfsrcycles.bitslice.forward_to_candidate(stride=11_170_000), starts = "
                  "random_candidate(random.Random(0), A51, 0x2AAA00) x256",
        "starts_digest": hashlib.sha256("".join(f"{x:016x}\n" for x in starts).encode()).hexdigest(),
        "digest": edge_digest(src, dst, dist), "sum_dist": int(dist.sum()),
        "min": int(dist.min()), "max": int(dist.max()), "seconds_1core": el})


def _walk_chunk(args):
    ref = ref_shim.load()
    C = ref.cipher
    chunk = args
    table = C.build_predecessor_table()
    params = C.CandidateParams.from_spec(C.A51, 0x2AAA00)
    # the reference's own worker (pipeline.py:225-228)
    return ref.pipeline._edges_chunk((chunk, params, C.A51, table, A51_STRIDE))


def gen_c1(ref, workers):
    from concurrent.futures import ProcessPoolExecutor
    n = 1 << 16
    starts = c1_starts(ref, n)
    chunks = [starts[i:i + 256] for i in range(0, n, 256)]
    t0 = time.time()
    rows = []
    with ProcessPoolExecutor(max_workers=workers) as pool:
        for k, part in enumerate(pool.map(_walk_chunk, chunks)):
            rows.extend(part)
            if k % 16 == 0:
                print(f"c1: {len(rows)}/{n} walks, {time.time() - t0:.0f}s", flush=True)
    el = time.time() - t0
    src = np.array([r[0] for r in rows], dtype=np.uint64)
    dst = np.array([r[1] for r in rows], dtype=np.uint64)
    dist = np.array([r[2] for r in rows], dtype=np.uint64)
    hist_lo = int(dist.min())
    save_json("a51_c1_65536.json", {
        "source": "lfsrcycles.pipeline._edges_chunk((chunk, params, A51, table, 11_170_000)), "
                  "chunks of 256 over ProcessPoolExecutor; starts = random_candidate("
                  "random.Random(0), A51, 0x2AAA00) x65536",
        "starts_digest": u64_digest(src), "digest": edge_digest(src, dst, dist),
        "dst_digest": u64_digest(dst), "dist_digest": u64_digest(dist),
        "sum_dist": int(dist.sum()), "sum_dist_sq": int((dist.astype(object) ** 2).sum()),
        "min": int(dist.min()), "max": int(dist.max()), "hist_lo": hist_lo,
        "hist": np.bincount((dist - hist_lo).astype(np.int64)).tolist(),
        "seconds": el, "workers": workers,
        "transitions_per_s": float(dist.sum()) / el})
    # a sparse sample of full rows (every 256th walk) for targeted debugging
    save("a51_c1_sample", idx=np.arange(0, n, 256, dtype=np.uint64), src=src[::256],
         dst=dst[::256], dist=dist[::256])


C2_LOG2 = 24
C2_BATCH_LOG2 = 22
A51_CAP = 178_957_008  # 16 * int(L) + 64 (bitslice.py:273-274)


def batch_digest(dst, dist) -> str:
    """sha256 over the little-endian u64 dst column then the dist column, input order."""
    h = hashlib.sha256(np.asarray(dst, dtype="<u8").tobytes())
    h.update(np.asarray(dist, dtype="<u8").tobytes())
    return h.hexdigest()


def _walk512():
    import ctypes as C
    import subprocess
    subprocess.run(["make", "-s", "-C", HERE, "walk512"], check=True)
    lib = C.CDLL(os.path.join(HERE, "_build", "libwalk512.so"))
    u = C.POINTER(C.c_uint64)
    lib.w512_walk.argtypes = [C.c_uint32, u, C.c_uint64, C.c_uint64, C.c_uint64, u, u, u]

    def walk(starts):
        starts = np.ascontiguousarray(starts, dtype=np.uint64)
        n = starts.size
        dst, dist, bad = np.zeros(n, np.uint64), np.zeros(n, np.uint64), np.zeros(1, np.uint64)
        p = lambda a: a.ctypes.data_as(u)  # noqa: E731
        rc = lib.w512_walk(0x2AAA00, p(starts), n, A51_STRIDE, A51_CAP, p(dst), p(dist), p(bad))
        if rc:
            raise RuntimeError(f"walk512: cap exceeded near start {int(bad[0])}")
        return dst, dist
    return walk


def gen_c2(ref):
    """Config 2: the first 2^24 results of the reference sampler
    random_candidate(random.Random(0), A51, 0x2AAA00) -- config 1 is its 2^16 prefix --
    walked to the next special node at the paper's stride.  The starts come from the
    reference itself; the walks from oracle/walk512.c, which is first pinned against the
    reference-produced config-1 set and the 256-walk KAT.  Output: per-batch digests of
    (dst, dist) for the 2^22-start batches bench.py times, plus whole-set statistics."""
    n = 1 << C2_LOG2
    t0 = time.time()
    starts = np.array(c1_starts(ref, n), dtype=np.uint64)
    t_starts = time.time() - t0
    print(f"c2: {n} reference starts in {t_starts:.0f} s", flush=True)
    c1 = json.load(open(os.path.join(GOLDEN, "a51_c1_65536.json")))
    assert u64_digest(starts[:1 << 16]) == c1["starts_digest"], "config-1 prefix mismatch"
    walk = _walk512()
    kat = np.load(os.path.join(GOLDEN, "a51_kat256.npz"))
    d, w = walk(kat["src"])
    assert (d == kat["dst"]).all() and (w == kat["dist"]).all(), "walk512 disagrees with the KAT"
    t1 = time.time()
    d, w = walk(starts[:1 << 16])
    assert u64_digest(d) == c1["dst_digest"] and u64_digest(w) == c1["dist_digest"], \
        "walk512 disagrees with the reference's config-1 run"
    print(f"c2: walk512 pinned on config 1 ({time.time() - t1:.0f} s)", flush=True)
    batch = 1 << C2_BATCH_LOG2
    batches = []
    dsts, dists = [], []
    t2 = time.time()
    for b in range(n // batch):
        d, w = walk(starts[b * batch:(b + 1) * batch])
        batches.append({"index": b, "digest": batch_digest(d, w), "sum_dist": int(w.sum()),
                        "min": int(w.min()), "max": int(w.max())})
        dsts.append(d)
        dists.append(w)
        print(f"c2: batch {b} done, {time.time() - t2:.0f} s", flush=True)
    el = time.time() - t2
    dst, dist = np.concatenate(dsts), np.concatenate(dists)
    hist_lo = int(dist.min())
    save_json("a51_c2_digests.json", {
        "source": "starts = lfsrcycles.pipeline.random_candidate(random.Random(0), A51, "
                  "CandidateParams.from_spec(A51, 0x2AAA00)) x 2^24 (the reference, via oracle/ref_shim.py); "
                  "walks = oracle/walk512.c at stride 11_170_000, pinned against a51_c1_65536.json "
                  "(the reference's own config-1 run) and a51_kat256",
        "n": n, "batch": batch, "stride": A51_STRIDE, "seed": SEED_C1, "fixed_r3": 0x2AAA00,
        "starts_digest": u64_digest(starts), "c1_prefix_starts_digest": c1["starts_digest"],
        "batch_digest_format": "sha256(dst as <u8 bytes || dist as <u8 bytes), input order",
        "batches": batches, "dst_digest": u64_digest(dst), "dist_digest": u64_digest(dist),
        "sum_dist": int(dist.sum()), "sum_dist_sq": int((dist.astype(object) ** 2).sum()),
        "min": int(dist.min()), "max": int(dist.max()), "hist_lo": hist_lo,
        "hist": np.bincount((dist - hist_lo).astype(np.int64)).tolist(),
        "seconds_walk": el, "seconds_starts": t_starts, "threads": os.cpu_count()})
    # a sparse sample of rows (every 4096th walk) for targeted debugging
    save("a51_c2_sample", idx=np.arange(0, n, 4096, dtype=np.uint64), src=starts[::4096],
         dst=dst[::4096], dist=dist[::4096])


def gen_bruteforce(ref):
    """oracle.brute_force_analysis (oracle.py:141-283) on the minis, majority and
    clock-all dynamics: summaries, cycles, histograms and digests of every array."""
    out = {}
    for name in ("MINI567", "MINI789"):
        spec = getattr(ref.cipher, name)
        params = ref.cipher.CandidateParams.from_spec(spec, ref.cipher.default_fixed_r3(spec))
        for clock_all in (False, True):
            t0 = time.perf_counter()
            gt = ref.oracle.brute_force_analysis(spec, params, clock_all=clock_all)
            el = time.perf_counter() - t0
            cycles = sorted((c.leader, c.clock_length, c.candidate_count, c.component_size) for c in gt.cycles)
            members = np.concatenate([c.ranks for c in sorted(gt.cycles, key=lambda c: int(c.ranks[0]))]) \
                if gt.cycles else np.zeros(0, dtype=np.int64)
            out[f"{name.lower()}_{'clockall' if clock_all else 'majority'}"] = {
                "summary": gt.summary(), "pred_count_hist": gt.pred_count_hist.tolist(),
                "cycles": [list(map(int, c)) for c in cycles],
                "cycle_members_digest": u64_digest(members),
                "level_counts": gt.level_counts.tolist(),
                "succ_digest": u64_digest(gt.succ), "cand_ranks_digest": u64_digest(gt.cand_ranks),
                "edge_dst_digest": u64_digest(gt.edge_dst), "edge_dist_digest": u64_digest(gt.edge_dist),
                "seg_depth_digest": u64_digest(gt.seg_depth), "seg_size_digest": u64_digest(gt.seg_size),
                "seconds": el,
            }
            print(name, clock_all, gt.summary(), f"{el:.1f}s", flush=True)
    save_json("bruteforce.json", out)


def main():
    ref = ref_shim.load()
    what = sys.argv[1] if len(sys.argv) > 1 else "basic"
    os.makedirs(GOLDEN, exist_ok=True)
    if what == "basic":
        gen_basic(ref)
    elif what == "prune":
        gen_prune(ref)
    elif what == "enumerate":
        gen_enumerate(ref)
    elif what == "kat":
        gen_kat(ref)
    elif what == "reduce":
        gen_reduce(ref)
    elif what == "tuning":
        gen_tuning(ref)
    elif what == "bruteforce":
        gen_bruteforce(ref)
    elif what == "c2":
        gen_c2(ref)
    elif what == "c1":
        gen_c1(ref, int(sys.argv[2]) if len(sys.argv) > 2 else os.cpu_count())
    else:
        raise SystemExit(f"unknown fixture group {what!r}")


if __name__ == "__main__":
    main()
