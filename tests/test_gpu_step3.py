"""The resumable step-3 driver on the GPU: config 1 (the reference sampler's 2^16 seed-0
special nodes) walked in four chunks to edge files, rerun as a no-op, merged -- and the
merged file's records equal the reference's own config-1 output (its digest in
tests/golden/a51_c1_65536.json)."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, has_golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_golden("a51_c1_65536.json"), reason="C1 fixture not generated")]


def test_config1_through_edge_files(gpu, lc, specs, params, tmp_path):
    from paper_1210_6411_b200 import pipeline as P
    from paper_1210_6411_b200 import records, step3

    want = golden_json("a51_c1_65536.json")
    starts = P.reference_candidates(specs["a51"], params["a51"], 0, 1 << 16)
    out = str(tmp_path / "c1")
    recs = step3.walk_to_edge_files(starts, out, specs["a51"], params["a51"], stride=lc.DEFAULT_STRIDE_A51,
                                    chunk=1 << 14)
    assert len(recs) == 4 and sum(r.edges for r in recs) == 1 << 16
    assert sum(r.transitions for r in recs) == want["sum_dist"]
    assert step3.walk_to_edge_files(starts, out, specs["a51"], params["a51"], stride=lc.DEFAULT_STRIDE_A51,
                                    chunk=1 << 14) == recs
    assert step3.merge_edge_files(out, str(tmp_path / "c1.bin")) == 1 << 16
    rec = records.read_edge_arrays(str(tmp_path / "c1.bin"))
    assert (rec["source"] == starts).all()
    assert hashlib.sha256(rec["destination"].astype("<u8").tobytes()).hexdigest() == want["dst_digest"]
    assert hashlib.sha256(rec["distance"].astype("<u8").tobytes()).hexdigest() == want["dist_digest"]
    assert (rec["subtree_size"] == 0).all() and (rec["subtree_depth"] == 0).all()
