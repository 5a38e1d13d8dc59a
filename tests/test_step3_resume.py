"""The resumable step-3 driver (paper_1210_6411_b200/step3.py) on CPU: chunking, rank
shares, manifest lines, idempotent reruns, recovery from a lost or corrupted chunk file,
configuration mismatches and the merged edge file -- with the GPU walk replaced by a
deterministic stand-in (the GPU path itself is tests/test_gpu_step3.py)."""

from __future__ import annotations

import numpy as np
import pytest


class _FakeWalk:
    def __init__(self):
        self.calls = []

    def __call__(self, starts, params, spec, *, stride=1, max_clocks=None):
        self.calls.append((int(starts[0]), starts.size))
        dst = (starts ^ np.uint64(0x5A5A)).reshape(-1, 1)
        dist = (starts % np.uint64(977) + np.uint64(stride)).reshape(-1, 1)

        class R:
            pass

        r = R()
        r.dst, r.dist = dst, dist
        r.edges, r.transitions = int(starts.size), int(dist.sum())
        return r


@pytest.fixture()
def fake(monkeypatch):
    from paper_1210_6411_b200 import step3

    f = _FakeWalk()
    monkeypatch.setattr(step3, "walk_arrays", f)
    return f


def _expected(states, stride):
    from paper_1210_6411_b200 import records

    rec = np.zeros(states.size, dtype=records.EDGE_DTYPE)
    rec["source"], rec["destination"] = states, states ^ np.uint64(0x5A5A)
    rec["distance"] = states % np.uint64(977) + np.uint64(stride)
    return rec.tobytes()


def test_chunks_resume_and_merge(tmp_path, fake):
    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import step3

    states = np.sort(np.random.default_rng(1).integers(1, 1 << 60, size=1000, dtype=np.uint64))
    p = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
    out = str(tmp_path / "run")
    recs = step3.walk_to_edge_files(states, out, lc.A51, p, stride=7, chunk=128)
    assert [r.lo for r in recs] == list(range(0, 1000, 128)) and recs[-1].hi == 1000
    assert len(fake.calls) == 8
    # a finished run is a no-op
    again = step3.walk_to_edge_files(states, out, lc.A51, p, stride=7, chunk=128)
    assert again == recs and len(fake.calls) == 8
    # a lost and a corrupted chunk are walked again, nothing else
    (tmp_path / "run" / recs[2].file).unlink()
    with open(tmp_path / "run" / recs[5].file, "r+b") as f:
        f.seek(17)
        f.write(b"\xff")
    step3.walk_to_edge_files(states, out, lc.A51, p, stride=7, chunk=128)
    assert sorted(c[0] for c in fake.calls[8:]) == sorted([int(states[256]), int(states[640])])
    n = step3.merge_edge_files(out, str(tmp_path / "all.bin"))
    assert n == 1000 and (tmp_path / "all.bin").read_bytes() == _expected(states, 7)
    # another configuration in the same directory is refused
    with pytest.raises(ValueError):
        step3.walk_to_edge_files(states, out, lc.A51, p, stride=8, chunk=128)


def test_rank_shares_cover_the_set(tmp_path, fake):
    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import step3

    states = np.arange(1, 1001, dtype=np.uint64)
    p = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
    out = str(tmp_path / "run")
    shares = [step3.walk_to_edge_files(states, out, lc.A51, p, stride=3, chunk=100, rank=r, world=3)
              for r in range(3)]
    assert sum(len(s) for s in shares) == 10
    assert [r.lo for s in shares for r in s] == list(range(0, 1000, 100))
    assert step3.merge_edge_files(out, str(tmp_path / "all.bin"), ranks=3) == 1000
    assert (tmp_path / "all.bin").read_bytes() == _expected(states, 3)
    with pytest.raises(ValueError):  # rank 2's chunks (the tail) not merged in
        step3.merge_edge_files(out, str(tmp_path / "part.bin"), ranks=2)


def test_torn_manifest_line_is_ignored(tmp_path, fake):
    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import step3

    states = np.arange(1, 301, dtype=np.uint64)
    p = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
    out = tmp_path / "run"
    step3.walk_to_edge_files(states, str(out), lc.A51, p, stride=1, chunk=100)
    with open(out / "manifest.rank0.jsonl", "a") as f:
        f.write('{"kind": "chunk", "chu')  # a crash mid-append
    calls = len(fake.calls)
    step3.walk_to_edge_files(states, str(out), lc.A51, p, stride=1, chunk=100)
    assert len(fake.calls) == calls
