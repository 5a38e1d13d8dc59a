"""Config 2 parity, the whole set: the reference sampler's first 2^24 starts
(random_candidate(random.Random(0), A51, 0x2AAA00), pipeline.py:301-310 -- config 1 is
their 2^16 prefix) walked on the GPU at the paper's stride, compared batch by batch with
the committed digests (tests/golden/a51_c2_digests.json: oracle/walk512.c over the
reference's own starts, pinned on the reference's config-1 run).  About 25 s of GPU time.

The opt-in variant (LFSR_SLOW=1) re-walks a prefix with the reference-structured C
restatement (oracle/lfsr_oracle.c) on the host cores, as a second, independent check."""

from __future__ import annotations

import hashlib
import os
import time

import numpy as np
import pytest

from conftest import golden_json

pytestmark = pytest.mark.gpu

STRIDE = 11_170_000


def _digest(dst, dist):
    h = hashlib.sha256(np.ascontiguousarray(dst, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(dist, dtype="<u8").tobytes())
    return h.hexdigest()


def test_config2_full_set_matches_committed_digests(gpu, lc, specs, params):
    from paper_1210_6411_b200 import pipeline as P

    c2 = golden_json("a51_c2_digests.json")
    starts = P.reference_candidates(specs["a51"], params["a51"], 0, c2["n"])
    assert hashlib.sha256(starts.astype("<u8").tobytes()).hexdigest() == c2["starts_digest"]
    batch = c2["batch"]
    total = 0
    for g in c2["batches"]:
        b = g["index"]
        res = lc.walk_arrays(starts[b * batch:(b + 1) * batch], params["a51"], specs["a51"], stride=STRIDE)
        assert _digest(res.dst[:, 0], res.dist[:, 0]) == g["digest"], f"batch {b}"
        assert int(res.dist.sum()) == g["sum_dist"]
        total += int(res.dist.sum())
    assert total == c2["sum_dist"]


@pytest.mark.slow
@pytest.mark.skipif(os.environ.get("LFSR_SLOW") != "1", reason="opt-in: LFSR_SLOW=1")
def test_config2_prefix_matches_restatement(gpu, lc, specs, params):
    from oracle import port
    from paper_1210_6411_b200 import pipeline as P

    n = 1 << int(os.environ.get("LFSR_C2_LOG2", "18"))
    starts = P.reference_candidates(specs["a51"], params["a51"], 0, n)
    t0 = time.perf_counter()
    res = lc.walk_arrays(starts, params["a51"], specs["a51"], stride=STRIDE)
    gpu_s = time.perf_counter() - t0
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    t0 = time.perf_counter()
    dst, dist = port.walk(specs["a51"], 0x2AAA00, starts, stride=STRIDE, width=256)
    cpu_s = time.perf_counter() - t0
    assert (res.dst[:, 0] == dst[:, 0]).all() and (res.dist[:, 0] == dist[:, 0]).all()
    assert lc.is_candidate(res.dst[:, 0], params["a51"], specs["a51"]).all()
    print(f"\nconfig-2 prefix: {n} walks bit-exact; GPU {gpu_s:.2f} s, C restatement {cpu_s:.1f} s "
          f"on {os.environ['OMP_NUM_THREADS']} cores; transitions {int(dist.sum())}")
