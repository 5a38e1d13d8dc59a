"""Config 1 at full size against the reference itself: the 2^16 seed-0 special nodes of
the reference sampler (pipeline.random_candidate with random.Random(0)), walked with the
reference benchmark's stride 11,170,000.  tests/golden/a51_c1_65536.json holds the
digest of the reference's own output (pipeline._edges_chunk over the same starts,
oracle/gen_golden.py c1, about an hour on 6 cores).  Bit-exact."""

from __future__ import annotations

import hashlib
import random

import numpy as np
import pytest

from conftest import golden_json, has_golden

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not has_golden("a51_c1_65536.json"), reason="C1 fixture not generated")]


def edge_digest(src, dst, dist):
    rows = sorted(zip((int(s) for s in src), (int(d) for d in dst), (int(w) for w in dist)))
    h = hashlib.sha256()
    for s, d, w in rows:
        h.update(f"{s:016x} {d:016x} {w}\n".encode())
    return h.hexdigest()


def test_config1_full_set_matches_reference(gpu, lc, specs, params):
    want = golden_json("a51_c1_65536.json")
    rng = random.Random(0)
    starts = np.array([lc.random_candidate(rng, specs["a51"], params["a51"]) for _ in range(1 << 16)],
                      dtype=np.uint64)
    assert hashlib.sha256(starts.astype("<u8").tobytes()).hexdigest() == want["starts_digest"]
    res = lc.walk_arrays(starts, params["a51"], specs["a51"], stride=lc.DEFAULT_STRIDE_A51,
                         histogram=(want["hist_lo"], 0, len(want["hist"])))
    dst, dist = res.dst[:, 0], res.dist[:, 0]
    assert hashlib.sha256(dst.astype("<u8").tobytes()).hexdigest() == want["dst_digest"]
    assert hashlib.sha256(dist.astype("<u8").tobytes()).hexdigest() == want["dist_digest"]
    assert edge_digest(starts, dst, dist) == want["digest"]
    assert res.transitions == want["sum_dist"]
    assert int(res.stats[2]) == want["min"] and int(res.stats[3]) == want["max"]
    # the GPU histogram block equals the reference's chain-length histogram
    hist = res.histogram[1:-1].astype(np.int64)
    assert hist[: len(want["hist"])].tolist() == want["hist"]
