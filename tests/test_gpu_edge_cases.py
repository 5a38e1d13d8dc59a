"""Empty and minimal inputs through the public API, against the reference's behaviour on
the same inputs (recorded here from runs of the reference in the build container):
empty edge files (one pass that removes nothing), a single self-loop record, empty
candidate lists, empty walks and empty sliced batches."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_empty_and_self_loop_reduce(gpu, lc, tmp_path):
    from paper_1210_6411_b200 import reduce as R
    from paper_1210_6411_b200.records import EdgeRecord, read_edges, write_edges

    cfg = R.ReduceConfig()
    p, q = tmp_path / "e.bin", tmp_path / "o.bin"
    write_edges(p, [])
    st = R.cut_leaves_pass(p, q, cfg)
    assert (st.leaves_removed, st.inner_nodes, st.out_size_sum) == (0, 0, 0)
    log = R.cut_leaves_to_fixpoint(p, q, cfg)
    assert [(s.leaves_removed, s.inner_nodes, s.out_size_sum) for s in log.passes] == [(0, 0, 0)]
    assert log.iterations == 0 and list(read_edges(q)) == []
    assert R.count_cycles([]) == [] and R.count_cycles(str(q)) == []
    write_edges(p, [EdgeRecord(5, 5, 7, 0, 0)])
    log = R.cut_leaves_to_fixpoint(p, q, cfg)
    assert [(s.leaves_removed, s.inner_nodes, s.out_size_sum) for s in log.passes] == [(0, 1, 0)]
    assert list(read_edges(q)) == [EdgeRecord(5, 5, 7, 0, 0)]
    assert R.count_cycles(list(read_edges(q))) == [R.CycleRecord(5, 1, 7, 0)]


def test_empty_candidate_lists(gpu, lc, specs, params):
    spec, prm = specs["mini567"], params["mini567"]
    surv, st = lc.prune_shallow_segments([], lc.PruneConfig(depth_limit=10), spec, prm)
    assert surv == [] and (st.mode, st.limit, st.total, st.removed, st.expanded) == ("dfs", 10, 0, 0, 0)
    assert lc.forward_to_candidate([], prm, spec) == []
    from paper_1210_6411_b200.bitslice import candidate_hops

    assert candidate_hops([], prm, spec) == []
    sb = lc.transpose([], spec, 64)
    filler = spec.pack(1, 1, 1)  # every lane of an empty batch is a filler (bitslice.py:46, :71-77)
    assert sb.words == [(1 << 64) - 1 if (filler >> i) & 1 else 0 for i in range(spec.total_bits)]
    assert sb.lane_count == 0 and lc.untranspose(lc.clock_sliced(sb, spec, 5)) == []
    empty = np.zeros(0, dtype=np.uint64)
    assert lc.is_candidate(empty, prm, spec).size == 0
    assert lc.enumerate_candidates_array(spec, prm, 5, 5).size == 0


def test_cut_leaves_arrays_empty(gpu, lc):
    z = np.zeros(0, dtype=np.uint64)
    out = lc.cut_leaves_arrays(z, z, z, z, z)
    assert out[5] == [(0, 0, 0)] and all(c.size == 0 for c in out[:5])
    out = lc.cut_leaves_arrays(z, z, z, z, z, max_passes=1)
    assert out[5] == [(0, 0, 0)]


def test_minimal_walk_sort_and_generator_inputs(gpu, lc, specs, params):
    from paper_1210_6411_b200 import _batch

    prm, spec = params["a51"], specs["a51"]
    assert lc.random_candidates_gpu(spec, prm, seed=1, n=0).size == 0
    one = lc.random_candidates_gpu(spec, prm, seed=1, n=1)
    assert one.size == 1 and bool(lc.is_candidate(one, prm, spec)[0])
    res = lc.walk_arrays(np.zeros(0, dtype=np.uint64), prm, spec)
    assert res.dst.shape == (0, 1) and res.edges == 0
    mini, mprm = specs["mini567"], params["mini567"]
    start = np.array([lc.random_candidate(__import__("random").Random(3), mini, mprm)], dtype=np.uint64)
    res = lc.walk_arrays(start, mprm, mini, legs=3)
    hops = lc.candidate_hops(start.tolist(), mprm, mini, legs=3)[0]
    assert [(int(d), int(w)) for d, w in zip(res.dst[0], res.dist[0])] == hops
    z = np.zeros(0, dtype=np.uint64)
    assert all(c.size == 0 for c in lc.sort_edge_arrays(z, z, z))
    s1 = lc.sort_edge_arrays(np.array([7], dtype=np.uint64), np.array([7], dtype=np.uint64),
                             np.array([1], dtype=np.uint64))
    assert [int(c[0]) for c in s1] == [7, 7, 1]
    assert _batch.first_missing(np.zeros(0, dtype=np.uint64), np.array([5], dtype=np.uint64)) == 0
    assert _batch.first_missing(np.array([5], dtype=np.uint64), np.zeros(0, dtype=np.uint64)) == 0


@pytest.mark.parametrize("kernel", ["v3", "v2"])
def test_prune_partial_warps_match_oracle(gpu, lc, specs, params, kernel, monkeypatch):
    """Batches smaller than a warp, a warp plus one, and one lane short of a block: the
    prune's per-lane candidate tickets, the drained-queue exit and (v3) the grid sized to
    the batch, in both modes; results equal the C restatement."""
    from oracle import port
    from paper_1210_6411_b200 import _batch

    if kernel == "v2":
        monkeypatch.setenv("LFSR_PRUNE_V1", "2")
    for name in ("a51", "mini789"):
        pool = lc.random_candidates_gpu(specs[name], params[name], seed=123, n=300)
        for n in (1, 2, 31, 33, 127, 129, 300):
            cands = pool[:n]
            for mode, limit in (("dfs", 3000 if name == "a51" else 60), ("bfs", 500)):
                removed, work = _batch.prune(cands, specs[name], params[name], mode, limit)
                o_removed, o_work = port.prune(specs[name], params[name].fixed_r3, mode, limit, cands)
                assert (removed == np.asarray(o_removed).astype(bool)).all(), (name, n, mode)
                assert (work == np.asarray(o_work)).all(), (name, n, mode)


def test_probe_segments_tiny_batches(gpu, lc, specs, params):
    """Zero and one root through the device-resident probe, with and without caps."""
    from oracle import port

    d, nn, c = lc.pipeline.probe_segments([], specs["mini567"], params["mini567"])
    assert d.size == 0 and nn.size == 0 and c.size == 0
    root = int(lc.random_candidates_gpu(specs["a51"], params["a51"], seed=4, n=1)[0])
    for depth_cap, node_cap in ((None, None), (3, None), (None, 10)):
        lv = []
        got = lc.probe_segment(root, specs["a51"], params["a51"], depth_cap=depth_cap, node_cap=node_cap,
                               level_counts=lv)
        wd, wn, wc, wl = port.probe_segment(specs["a51"], 0x2AAA00, root, depth_cap, node_cap)
        assert got == (wd, wn, wc) and lv == [int(v) for v in wl]
