"""GPU parity of the step-1/2 kernels and batch predicates against the reference's
golden vectors: is_candidate / predecessors (cipher.py:342-428), clock_sliced
(bitslice.py:223-228), enumerate_candidates (pipeline.py:104-118), prune_shallow_segments
(pipeline.py:192-222), build_skeleton_edges (pipeline.py:231-256), probe_segment, K0."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, golden_npz, has_golden

pytestmark = pytest.mark.gpu


def u64_digest(values):
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["a51", "mini567", "mini789"])
def test_batch_predicate_and_predecessors(gpu, lc, specs, params, name):
    g = golden_npz(f"pred_{name}")
    got = lc.is_candidate(g["states"], params[name], specs[name])
    assert (got == g["is_candidate"].astype(bool)).all()
    preds, cnt = lc.predecessors(g["states"], specs[name])
    assert (cnt == g["npred"]).all()
    assert (preds == g["preds"]).all()


@pytest.mark.parametrize("name", ["a51", "mini567", "mini789"])
def test_clock_sliced_matches_reference(gpu, lc, specs, name):
    from paper_1210_6411_b200 import _batch

    g = golden_npz(f"traj_{name}")
    assert (_batch.clock(g["starts"], specs[name], 1) == g["traj"][:, 0]).all()
    assert (_batch.clock(g["starts"], specs[name], 64) == g["traj"][:, 63]).all()
    sb = lc.transpose(g["starts"].tolist(), specs[name], 256)
    out = lc.clock_sliced(sb, specs[name], 500)
    assert lc.untranspose(out) == g["after500"].tolist()


@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_enumerate_minis(gpu, lc, specs, params, name):
    meta = golden_json("enumerate.json")[name]
    got = list(lc.enumerate_candidates(specs[name], params[name]))
    assert len(got) == meta["count"]
    assert u64_digest(got) == meta["digest"]


@pytest.mark.parametrize("r2_0", [0x1, 0x1234, 0x3FFFFC])
def test_enumerate_a51_rows(gpu, lc, specs, params, r2_0):
    meta = golden_json("enumerate.json")[f"a51_rows_{r2_0:#x}_4"]
    got = lc.enumerate_candidates_array(specs["a51"], params["a51"], r2_0, r2_0 + 4)
    assert got.size == meta["count"]
    assert got[:64].tolist() == meta["first"] and got[-64:].tolist() == meta["last"]
    assert u64_digest(got) == meta["digest"]


@pytest.mark.skipif(not has_golden("prune.json"), reason="prune fixture not generated")
@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_prune_minis(gpu, lc, specs, params, name):
    fx = golden_json("prune.json")
    cands = list(lc.enumerate_candidates(specs[name], params[name]))
    for key, want in fx.items():
        if not key.startswith(name + "_") or key.endswith("_probe"):
            continue
        _, mode, lim = key.split("_")
        cfg = lc.PruneConfig(mode=mode, depth_limit=int(lim) if mode == "dfs" else None,
                             node_limit=int(lim) if mode == "bfs" else None)
        surv, st = lc.prune_shallow_segments(cands, cfg, specs[name], params[name])
        assert u64_digest(surv) == want["survivors_digest"], key
        assert (st.total, st.removed, st.expanded) == (want["total"], want["removed"], want["expanded"]), key


@pytest.mark.skipif(not has_golden("prune.json"), reason="prune fixture not generated")
def test_prune_a51_sample(gpu, lc, specs, params):
    fx = golden_json("prune.json")
    cands = fx["a51_cands"]
    for key, want in fx.items():
        if not key.startswith("a51_") or key == "a51_cands":
            continue
        _, mode, lim = key.split("_")
        cfg = lc.PruneConfig(mode=mode, depth_limit=int(lim) if mode == "dfs" else None,
                             node_limit=int(lim) if mode == "bfs" else None)
        surv, st = lc.prune_shallow_segments(cands, cfg, specs["a51"], params["a51"])
        assert surv == want["survivors"], key
        assert (st.total, st.removed, st.expanded) == (want["total"], want["removed"], want["expanded"]), key
        if "per_candidate" in want:
            from paper_1210_6411_b200 import _batch

            removed, work = _batch.prune(cands, specs["a51"], params["a51"], mode, int(lim))
            assert [[int(r), int(w)] for r, w in zip(removed, work)] == want["per_candidate"]


@pytest.mark.skipif(not has_golden("prune.json"), reason="prune fixture not generated")
@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_probe_segment_minis(gpu, lc, specs, params, name):
    probes = golden_json("prune.json")[f"{name}_probe"]
    cands = list(lc.enumerate_candidates(specs[name], params[name]))[:64]
    for x, (depth, nodes, cens, levels) in zip(cands, probes):
        lc_ = []
        got = lc.probe_segment(x, specs[name], params[name], level_counts=lc_)
        assert got == (depth, nodes, cens)
        assert lc_ == levels


@pytest.mark.parametrize("frontier", [None, "64"])
def test_probe_segments_batched_match_oracle(gpu, lc, specs, params, frontier, monkeypatch):
    """Batched device-resident probes (lc_probe_segments) equal the C restatement root by
    root -- depth, nodes, censoring, and the level counts summed over the roots -- with and
    without caps; LFSR_PROBE_CAP=64 starts the frontier buffers tiny, so every few levels
    overflow and are grown and redone."""
    from oracle import port

    if frontier:
        monkeypatch.setenv("LFSR_PROBE_CAP", frontier)
    for name, n_roots, caps in (("mini567", 200, [(None, None), (5, None), (None, 40)]),
                                ("mini789", 300, [(None, None), (12, 500)]),
                                ("a51", 256, [(3000, 200000), (400, None)])):
        roots = lc.random_candidates_gpu(specs[name], params[name], seed=31, n=n_roots)
        for depth_cap, node_cap in caps:
            levels = []
            d, nn, c = lc.pipeline.probe_segments(roots, specs[name], params[name], depth_cap=depth_cap,
                                                  node_cap=node_cap, level_counts=levels)
            want_levels = []
            for i, x in enumerate(roots):
                wd, wn, wc, wl = port.probe_segment(specs[name], params[name].fixed_r3, int(x), depth_cap, node_cap,
                                                    levels=8192)
                assert (int(d[i]), int(nn[i]), bool(c[i])) == (wd, wn, wc), (name, depth_cap, node_cap, i)
                want_levels += [0] * (len(wl) - len(want_levels))
                for lv, v in enumerate(wl):
                    want_levels[lv] += int(v)
            assert levels == want_levels, (name, depth_cap, node_cap)


@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_build_skeleton_edges_closed_set(gpu, lc, specs, params, name):
    g = golden_npz(f"edges_{name}")
    edges = lc.build_skeleton_edges(g["src"].tolist(), params[name], specs[name])
    assert [e.destination for e in edges] == g["dst"].tolist()
    assert [e.distance for e in edges] == g["dist"].tolist()
    assert all(e.subtree_size == 0 and e.subtree_depth == 0 for e in edges)


def test_build_skeleton_edges_detects_unsound_prune(gpu, lc, specs, params):
    g = golden_npz("edges_mini567")
    with pytest.raises(lc.PruneSoundnessError):
        lc.build_skeleton_edges(g["src"][:100].tolist(), params["mini567"], specs["mini567"])
    with pytest.raises(ValueError):
        lc.build_skeleton_edges([], params["mini567"], specs["mini567"])


@pytest.mark.parametrize("name", ["a51", "mini789"])
def test_k0_matches_numpy_restatement(gpu, lc, specs, params, name):
    from oracle import k0

    got = lc.random_candidates_gpu(specs[name], params[name], seed=12345, n=5000)
    want = k0.random_candidates(specs[name], params[name].fixed_r3, 12345, 5000)
    assert (got == want).all()
    assert lc.is_candidate(got, params[name], specs[name]).all()


def test_tuning_functions_match_reference(gpu, lc, specs, params):
    """auto_depth_limit (pipeline.py:313-333, GPU batched segment probes) and
    calibrate_stride (bitslice.py:357-376, GPU two-hop walks) return the reference's values."""
    fx = golden_json("tuning.json")
    for key, want in fx.items():
        if key.startswith("auto_depth_"):
            _, _, name, sample, seed = key.split("_")
            got = lc.auto_depth_limit(specs[name], params[name], sample=int(sample), seed=int(seed))
            assert got == want, key
        elif key.startswith("calibrate_"):
            _, name, n, seed = key.split("_")
            assert lc.calibrate_stride(specs[name], params[name], samples=int(n), seed=int(seed)) == want, key
    # the reference's sampled stride for mini567 (149 / 150, unsafe > 148)
    meta = golden_json("edges_mini567.json")["calibrate_stride"]
    assert lc.calibrate_stride(specs["mini567"], params["mini567"], samples=500, seed=0) == meta["500_0"]
    assert lc.calibrate_stride(specs["mini567"], params["mini567"], samples=2000, seed=1) == meta["2000_1"]
    assert lc.calibrate_stride(specs["a51"], params["a51"]) == lc.DEFAULT_STRIDE_A51


def test_edges_chunk_worker(gpu, lc, specs, params):
    from paper_1210_6411_b200.pipeline import _edges_chunk

    g = golden_npz("edges_mini789")
    rows = _edges_chunk((g["src"][:500].tolist(), params["mini789"], specs["mini789"], None, 1))
    assert rows == list(zip(g["src"][:500].tolist(), g["dst"][:500].tolist(), g["dist"][:500].tolist()))


def test_build_skeleton_edges_sharded_devices(gpu, lc, specs, params):
    """workers > 1: contiguous shards walked concurrently, one host thread and native
    context per device (here twice the one GPU), results in input order."""
    g = golden_npz("edges_mini789")
    for devices in ([0, 0], [0, 0, 0]):
        edges = lc.build_skeleton_edges(g["src"].tolist(), params["mini789"], specs["mini789"], devices=devices)
        assert [e.destination for e in edges] == g["dst"].tolist()
        assert [e.distance for e in edges] == g["dist"].tolist()
    edges = lc.build_skeleton_edges(g["src"].tolist(), params["mini789"], specs["mini789"], workers=8)
    assert [e.distance for e in edges] == g["dist"].tolist()


def test_prune_sharded_devices(gpu, lc, specs, params):
    """config.workers / devices > 1: chunks pruned concurrently, survivors in input order,
    statistics summed -- equal to the single-device result and the reference's."""
    fx = golden_json("prune.json")
    cands = fx["a51_cands"]
    key = next(k for k in fx if k.startswith("a51_dfs_"))
    want = fx[key]
    cfg = lc.PruneConfig(mode="dfs", depth_limit=int(key.split("_")[2]))
    for devices in ([0, 0], [0, 0, 0]):
        surv, st = lc.prune_shallow_segments(cands, cfg, specs["a51"], params["a51"], devices=devices)
        assert surv == want["survivors"]
        assert (st.total, st.removed, st.expanded) == (want["total"], want["removed"], want["expanded"])


def test_prune_deep_limit_matches_oracle(gpu, lc, specs, params):
    """Depth limits beyond the ring's 12-bit depth field (>= 4096) take the stackless-climb
    fallback for the deep part of a traversal; results and the LIFO `expanded` counter
    still equal the C restatement (oracle/lfsr_oracle.c, pinned to the reference)."""
    from oracle import port
    from paper_1210_6411_b200 import _batch

    cands = lc.random_candidates_gpu(specs["a51"], params["a51"], seed=77, n=512)
    for limit in (4095, 4097, 6000):
        removed, work = _batch.prune(cands, specs["a51"], params["a51"], "dfs", limit)
        o_removed, o_work = port.prune(specs["a51"], 0x2AAA00, "dfs", limit, cands)
        assert (removed == np.asarray(o_removed).astype(bool)).all(), limit
        assert (work == np.asarray(o_work)).all(), limit


@pytest.mark.parametrize("spill,ring", [("0", "32"), ("1", "32"), ("3", "32"), ("0", "20"), ("3", "20"),
                                       ("512", "20")])
def test_prune_small_spill_matches_reference(gpu, lc, specs, params, spill, ring):
    """Tiny (or no) global spill behind the shared-memory ring (32 entries, or the
    20-entry variant launched for batches of 2^24 and more) forces the drop-oldest +
    stackless-climb fallback on deep traversals; survivors and the per-candidate LIFO
    `expanded` counters must still equal the reference's (prune.json) and the C
    restatement.  The kernel reads LFSR_PRUNE_SPILL / LFSR_PRUNE_RING at launch, so it
    runs in a child process."""
    import json
    import os
    import subprocess
    import sys

    code = r'''
import json, numpy as np, sys
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1210_6411_b200 as lc
from paper_1210_6411_b200 import _batch
from conftest import golden_json
from oracle import port
fx = golden_json("prune.json")
cands = fx["a51_cands"]
p = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
ok = True
for key, want in fx.items():
    if not key.startswith("a51_") or key == "a51_cands":
        continue
    _, mode, lim = key.split("_")
    removed, work = _batch.prune(cands, lc.A51, p, mode, int(lim))
    surv = [c for c, r in zip(cands, removed) if not r]
    ok = ok and surv == want["survivors"] and int(work.sum()) == want["expanded"]
extra = lc.random_candidates_gpu(lc.A51, p, seed=5, n=256)
removed, work = _batch.prune(extra, lc.A51, p, "dfs", 6000)
o_removed, o_work = port.prune(lc.A51, 0x2AAA00, "dfs", 6000, extra)
ok = ok and (removed == np.asarray(o_removed).astype(bool)).all() and (work == np.asarray(o_work)).all()
print(json.dumps({"ok": bool(ok)}))
'''
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, LFSR_PRUNE_SPILL=spill, LFSR_PRUNE_RING=ring, LFSR_PRUNE_V1="2")  # v2's fallback
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    assert json.loads(r.stdout.strip().splitlines()[-1])["ok"]


def test_enumerate_overflow_returns_prefix(gpu, lc, specs, params):
    """lc_enumerate with too small a buffer: LC_ERR_OVERFLOW, the full count, and the
    ascending prefix that fits (the writer's cap check on its 16-byte pair stores)."""
    import ctypes as C

    from paper_1210_6411_b200 import _native as N

    full = lc.enumerate_candidates_array(specs["a51"], params["a51"], 0x1234, 0x1236)
    ctx = N.context()
    for cap in (1, 2, 3, 1000, 1001, full.size - 1):
        out = np.zeros(cap, dtype=np.uint64)
        count = C.c_uint64(0)
        rc = N.lib.lc_enumerate(ctx.handle, C.byref(N.spec_struct(specs["a51"])), params["a51"].fixed_r3, 0x1234,
                                0x1236, N.u64p(out), cap, C.byref(count))
        assert rc == N.LC_ERR_OVERFLOW and count.value == full.size
        assert (out == full[:cap]).all(), cap


@pytest.mark.parametrize("kernel", ["v3", "v2", "v1"])
def test_prune_random_configs_match_restatement(gpu, lc, specs, params, kernel, monkeypatch):
    """Seeded random (cipher, mode, limit, candidate subset) configurations: removed flags
    and per-candidate `expanded` counters equal the C restatement's (pinned to the
    reference by prune.json) -- including limits around v2's 12-bit depth field and v3's
    4096 cut-over, and node limits that cut traversals mid-way -- for each kernel (the
    launch reads LFSR_PRUNE_V1: unset = v3 for DFS up to 4096, 2 = v2, 1 = round 1)."""
    import random

    if kernel != "v3":
        monkeypatch.setenv("LFSR_PRUNE_V1", kernel[1])
    from oracle import port
    from paper_1210_6411_b200 import _batch

    rng = random.Random(20261018)
    pools = {name: lc.random_candidates_gpu(specs[name], params[name], seed=9, n=4096)
             for name in ("a51", "mini567", "mini789")}
    for _ in range(12):
        name = rng.choice(["a51", "a51", "mini567", "mini789"])
        mode = rng.choice(["dfs", "bfs"])
        limit = rng.choice([1, 2, 7, 50, 300, 3000, 4095, 4096, 4097, 20000]) if mode == "dfs" else \
            rng.choice([1, 2, 10, 500, 5000, 100000])
        pool = pools[name]
        cands = pool[np.array(sorted(rng.sample(range(pool.size), 1024)))]
        removed, work = _batch.prune(cands, specs[name], params[name], mode, limit)
        o_removed, o_work = port.prune(specs[name], params[name].fixed_r3, mode, limit, cands)
        assert (removed == np.asarray(o_removed).astype(bool)).all(), (name, mode, limit)
        assert (work == np.asarray(o_work)).all(), (name, mode, limit)


@pytest.mark.parametrize("fixed_r3", [0x7FFC00, 0x123C00, 0x2AA800, 0x2A8000])
@pytest.mark.parametrize("kernel", ["v3", "v2"])
def test_prune_other_fixed_r3_matches_oracle(gpu, lc, specs, fixed_r3, kernel, monkeypatch):
    """Fixed-R3 planes other than the paper's 0x2AAA00, one per (clock bit, bit above) class
    that has candidates (c3 = 1, n3 = 0 planes have none; the prune kernels take F at run
    time: the special-child test depends on it): candidates of the plane, DFS and BFS,
    against the C restatement."""
    from oracle import port
    from paper_1210_6411_b200 import _batch

    if kernel == "v2":
        monkeypatch.setenv("LFSR_PRUNE_V1", "2")
    p = lc.CandidateParams.from_spec(specs["a51"], fixed_r3)
    cands = lc.enumerate_candidates_array(specs["a51"], p, 0x2AAA, 0x2AAB)[:3000]
    assert cands.size and (cands == port.enumerate_rows(specs["a51"], fixed_r3, 0x2AAA, 0x2AAB)[:3000]).all()
    for mode, limit in (("dfs", 3000), ("dfs", 40), ("bfs", 700)):
        removed, work = _batch.prune(cands, specs["a51"], p, mode, limit)
        o_removed, o_work = port.prune(specs["a51"], fixed_r3, mode, limit, cands)
        assert (removed == np.asarray(o_removed).astype(bool)).all(), (mode, limit)
        assert (work == np.asarray(o_work)).all(), (mode, limit)
