"""GPU parity of the edge-output sort and steps 4-5 (leaf cutting, cycle counting)
against the reference's own reduce.py run on mini skeletons (tests/golden/reduce.json)
and, at larger sizes, the numpy restatement oracle/reduce_np.py."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, golden_npz

pytestmark = pytest.mark.gpu


def u64_digest(values):
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


def skeleton_edges(lc, specs, params, name, label):
    spec, p = specs[name], params[name]
    cands = lc.enumerate_candidates_array(spec, p)
    if label == "dfs4":
        skel, _ = lc.prune_shallow_segments(cands, lc.PruneConfig(mode="dfs", depth_limit=4), spec, p)
    elif label == "bfs8":
        skel, _ = lc.prune_shallow_segments(cands, lc.PruneConfig(mode="bfs", node_limit=8), spec, p)
    else:
        skel = cands.tolist()
    return lc.build_skeleton_edges(skel, p, spec)


@pytest.mark.parametrize("name", ["mini567", "mini789"])
@pytest.mark.parametrize("label", ["full", "dfs4", "bfs8"])
def test_pipeline_steps_1_to_5_match_reference(gpu, lc, specs, params, tmp_path, name, label):
    want = golden_json("reduce.json")[f"{name}_{label}"]
    edges = skeleton_edges(lc, specs, params, name, label)
    assert len(edges) == want["skeleton"]
    path = tmp_path / "edges.bin"
    lc.write_edges(path, edges)
    one = tmp_path / "one.bin"
    st = lc.cut_leaves_pass(path, one, lc.ReduceConfig())
    assert (st.leaves_removed, st.inner_nodes, st.out_size_sum) == tuple(
        want["pass1"][k] for k in ("leaves_removed", "inner_nodes", "out_size_sum"))
    assert u64_digest([v for r in lc.read_edges(one) for v in r]) == want["pass1"]["records_digest"]
    fix = tmp_path / "fix.bin"
    log = lc.cut_leaves_to_fixpoint(path, fix, lc.ReduceConfig())
    assert [[p.leaves_removed, p.inner_nodes, p.out_size_sum] for p in log.passes] == want["passes"]
    assert log.iterations == want["iterations"]
    assert [list(r) for r in lc.read_edges(fix)] == want["fixpoint"]
    assert [list(c) for c in lc.count_cycles(str(fix))] == want["cycles"]
    assert [list(c) for c in lc.count_cycles(lc.read_edges(fix))] == want["cycles"]


@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_cycles_match_brute_force_oracle(gpu, lc, name):
    """(hop count, clock length) per cycle == the reference oracle's exhaustive
    functional-graph analysis (oracle.py:141-283)."""
    fx = golden_json("reduce.json")
    g = golden_npz(f"edges_{name}")
    z = np.zeros(g["src"].size, dtype=np.uint64)
    src, dst, dist, size, depth, _ = lc.cut_leaves_arrays(g["src"], g["dst"], g["dist"], z, z)
    leader, hops, clocks, tree = lc.count_cycles_arrays(src, dst, dist, size)
    assert sorted(zip(hops.tolist(), clocks.tolist())) == sorted(tuple(c) for c in fx[f"{name}_oracle_cycles"])
    # conservation: every skeleton node is on a cycle or in a tree hanging off one
    assert int(hops.sum()) + int(tree.sum()) == g["src"].size


def test_sort_edge_arrays(gpu, lc):
    rng = np.random.default_rng(1)
    n = 300_000
    src = rng.choice(np.uint64(1) << np.uint64(60), size=n, replace=False).astype(np.uint64)
    dst = rng.integers(0, 1 << 62, size=n, dtype=np.uint64)
    dist = np.arange(n, dtype=np.uint64)
    s, d, w = lc.sort_edge_arrays(src, dst, dist)
    order = np.argsort(src)
    assert (s == src[order]).all() and (d == dst[order]).all() and (w == dist[order]).all()


def test_random_functional_graph_matches_restatement(gpu, lc):
    """2^20-node random mapping (mostly trees into few cycles) vs oracle/reduce_np.py."""
    from oracle import reduce_np

    rng = np.random.default_rng(7)
    n = 1 << 20
    src = np.sort(rng.choice(np.uint64(1) << np.uint64(40), size=n, replace=False).astype(np.uint64))
    dst = src[rng.integers(0, n, size=n)]
    dist = rng.integers(1, 1000, size=n, dtype=np.uint64)
    z = np.zeros(n, dtype=np.uint64)
    got = lc.cut_leaves_arrays(src, dst, dist, z, z)
    want = reduce_np.cut_leaves(src, dst, dist, z, z)
    assert got[5] == want[5]
    for a, b in zip(got[:5], want[:5]):
        assert (a == b).all()
    cyc = lc.count_cycles_arrays(*got[:4])
    assert [tuple(r) for r in zip(*(c.tolist() for c in cyc))] == reduce_np.count_cycles(*want[:4])


def test_reduce_errors(gpu, lc, tmp_path):
    # unsorted sources
    with pytest.raises(ValueError):
        lc.cut_leaves_arrays([5, 3], [3, 5], [1, 1], [0, 0], [0, 0])
    # a leaf whose destination is no record: not closed
    with pytest.raises(ValueError):
        lc.cut_leaves_arrays([1, 2], [2, 9], [1, 1], [0, 0], [0, 0])
    # trees left: not a permutation
    with pytest.raises(lc.NotAPermutationError):
        lc.count_cycles_arrays([1, 2, 3], [2, 3, 2], [1, 1, 1], [0, 0, 0])
    with pytest.raises(lc.NotAPermutationError):
        lc.count_cycles([lc.EdgeRecord(1, 2, 1, 0, 0), lc.EdgeRecord(1, 2, 1, 0, 0)])
    with pytest.raises(ValueError):
        lc.cut_leaves_pass(tmp_path / "x.bin", tmp_path / "y.bin", lc.ReduceConfig(memory_budget=1024))


def test_write_edge_tensors_byte_identical(gpu, tmp_path):
    """GPU record packer (lc_pack_records_device) == the reference's write_edges bytes."""
    import torch

    from paper_1210_6411_b200.records import EdgeRecord, write_edge_tensors, write_edges

    rng = np.random.default_rng(5)
    cols = [rng.integers(0, 1 << 63, size=1000, dtype=np.int64).astype(np.uint64) for _ in range(5)]
    write_edges(tmp_path / "a.bin", [EdgeRecord(*map(int, r)) for r in zip(*cols)])
    t = [torch.from_numpy(c.view(np.int64)).cuda() for c in cols]
    write_edge_tensors(tmp_path / "b.bin", *t)
    assert (tmp_path / "a.bin").read_bytes() == (tmp_path / "b.bin").read_bytes()
    write_edges(tmp_path / "c.bin", [EdgeRecord(int(s), int(d), int(w), 0, 0) for s, d, w in zip(*cols[:3])])
    write_edge_tensors(tmp_path / "d.bin", *t[:3])
    assert (tmp_path / "c.bin").read_bytes() == (tmp_path / "d.bin").read_bytes()
    write_edge_tensors(tmp_path / "e.bin", *(x[:0] for x in t[:3]))
    assert (tmp_path / "e.bin").read_bytes() == b""


@pytest.mark.parametrize("shape", ["path", "broom"])
def test_long_tail_of_passes_matches_restatement(gpu, lc, shape):
    """Thousands of passes with tiny frontiers: the single-block tail kernel (csrc/reduce.cu
    cut_tail_kernel) runs them, across several graph replays (1024 tail passes each), and
    must give the restatement's per-pass statistics exactly.  "path": one 3000-record chain
    into a self-loop (one leaf per pass); "broom": a 2^16-node random forest (wide passes
    first) whose roots hang off a 2500-record chain."""
    from oracle import reduce_np

    rng = np.random.default_rng(11)
    if shape == "path":
        n = 3000
        dst_idx = np.minimum(np.arange(n) + 1, n - 1)
    else:
        chain, bush = 2500, 1 << 16
        n = chain + bush
        dst_idx = np.empty(n, dtype=np.int64)
        dst_idx[:chain] = np.minimum(np.arange(chain) + 1, chain - 1)
        dst_idx[chain:] = rng.integers(0, chain // 8, size=bush)  # trees rooted near the chain's start
        inner = rng.random(bush) < 0.7
        dst_idx[chain:][inner] = chain + rng.integers(0, bush, size=int(inner.sum()))
    src = np.sort(rng.choice(np.uint64(1) << np.uint64(50), size=n, replace=False).astype(np.uint64))
    dst = src[dst_idx]
    dist = rng.integers(1, 1000, size=n, dtype=np.uint64)
    z = np.zeros(n, dtype=np.uint64)
    got = lc.cut_leaves_arrays(src, dst, dist, z, z)
    want = reduce_np.cut_leaves(src, dst, dist, z, z)
    assert got[5] == want[5]
    assert len(got[5]) > 2000
    for a, b in zip(got[:5], want[:5]):
        assert (a == b).all()
