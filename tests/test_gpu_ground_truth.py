"""The GPU exhaustive analysis (ground_truth.brute_force_analysis, csrc/bruteforce.cu)
against the reference's own oracle.brute_force_analysis (oracle.py:141-283) on both
minis, majority and clock-all dynamics: summaries, cycles, histograms, level counts and
digests of every array (tests/golden/bruteforce.json, oracle/gen_golden.py bruteforce).
It is also an independent check of steps 1-5: its candidate edges equal the walk's."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, golden_npz

pytestmark = pytest.mark.gpu


def u64_digest(values):
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


@pytest.mark.parametrize("name", ["mini567", "mini789"])
@pytest.mark.parametrize("clock_all", [False, True])
def test_brute_force_matches_reference(gpu, lc, specs, params, name, clock_all):
    from paper_1210_6411_b200.ground_truth import brute_force_analysis

    want = golden_json("bruteforce.json")[f"{name}_{'clockall' if clock_all else 'majority'}"]
    gt = brute_force_analysis(specs[name], params[name], clock_all=clock_all)
    got = gt.summary()
    for k, v in want["summary"].items():
        assert got[k] == pytest.approx(v, rel=1e-12), k
    assert gt.pred_count_hist.tolist() == want["pred_count_hist"]
    assert sorted([c.leader, c.clock_length, c.candidate_count, c.component_size] for c in gt.cycles) == want["cycles"]
    members = np.concatenate([c.ranks for c in sorted(gt.cycles, key=lambda c: int(c.ranks[0]))])
    assert u64_digest(members) == want["cycle_members_digest"]
    assert gt.level_counts.tolist() == want["level_counts"]
    for key, arr in (("succ", gt.succ), ("cand_ranks", gt.cand_ranks), ("edge_dst", gt.edge_dst),
                     ("edge_dist", gt.edge_dist), ("seg_depth", gt.seg_depth), ("seg_size", gt.seg_size)):
        assert u64_digest(arr) == want[f"{key}_digest"], key


@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_brute_force_edges_equal_the_walk(gpu, lc, specs, params, name):
    """Two independent GPU paths: successor-map walking vs the bitsliced walk kernel."""
    from paper_1210_6411_b200.ground_truth import brute_force_analysis

    gt = brute_force_analysis(specs[name], params[name])
    g = golden_npz(f"edges_{name}")
    emap = gt.candidate_edge_map()
    assert sorted(emap) == sorted(g["src"].tolist())
    assert [emap[int(s)] for s in g["src"]] == list(zip(g["dst"].tolist(), g["dist"].tolist()))
    assert gt.cycle_multiset() == sorted(gt.cycle_multiset())
