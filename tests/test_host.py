"""Host-side logic (CPU): the reference-shaped value types and scalar helpers, record
formats, sliced-batch format, and the C ABI surface (library loads, every symbol that
include/lfsr_b200.h declares is exported -- no compute calls without a GPU)."""

from __future__ import annotations

import ctypes
import os
import random
import re
from fractions import Fraction

import numpy as np
import pytest

from conftest import ROOT, golden_json, golden_npz, random_states


def test_header_symbols_are_exported():
    from paper_1210_6411_b200 import _native

    header = open(os.path.join(ROOT, "include", "lfsr_b200.h")).read()
    declared = set(re.findall(r"^\s*(?:int|const char \*|uint64_t|void)\s*\*?\s*(lc_\w+)\(", header, re.M))
    assert len(declared) >= 20
    lib = ctypes.CDLL(_native.LIB_PATH)
    for name in declared:
        assert hasattr(lib, name), name
    assert declared == set(_native.EXPORTED)
    assert lib.lc_abi_version() == 1


def test_library_is_sm100a_cuda():
    """The shipped .so carries sm_100a SASS (cuobjdump is in the image)."""
    import shutil
    import subprocess

    from paper_1210_6411_b200 import _native

    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", _native.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_builtin_layout(lc):
    assert lc.A51.offsets == (0, 19, 41) and lc.A51.total_bits == 64
    assert lc.MINI567.valid_state_count == 31 * 63 * 127
    for s in (lc.A51, lc.MINI567, lc.MINI789):
        assert lc.CipherSpec.from_json(s.to_json()) == s


def test_spec_validation(lc):
    with pytest.raises(ValueError):
        lc.CipherSpec("bad", (7, 6, 5), ((5, 6), (4, 5), (1, 4)), (2, 2, 2))
    with pytest.raises(ValueError):
        lc.CipherSpec("bad", (5, 6, 7), ((1, 3), (4, 5), (5, 6)), (2, 2, 3))
    with pytest.raises(ValueError):
        lc.CipherSpec("bad", (5, 6, 7), ((1, 4), (4, 5), (5, 6)), (4, 2, 3))
    with pytest.raises(KeyError):
        lc.builtin_spec("nope")
    with pytest.raises(ValueError):
        lc.CandidateParams.from_spec(lc.A51, 0)
    with pytest.raises(ValueError):
        lc.CandidateParams.from_spec(lc.MINI567, 1 << 7)


def test_register_periods(lc):
    for s in (lc.MINI567, lc.MINI789):
        for k, n in enumerate(s.lengths):
            assert s.register_period(k) == 2 ** n - 1


def test_predecessor_table_matches_reference(lc):
    t = golden_json("tables.json")
    tab = lc.build_predecessor_table()
    assert [list(e) for e in tab.entries] == t["entries"]
    assert tab.empty_count == 24 and tab.total_patterns == 64
    assert hex(tab.nonempty_mask) == t["nonempty_mask"]
    assert lc.shared_table() is lc.shared_table()


@pytest.mark.parametrize("name", ["a51", "mini567", "mini789"])
def test_scalar_helpers_match_reference(lc, specs, params, name):
    g = golden_npz(f"traj_{name}")
    spec = specs[name]
    for j in range(0, 256, 17):
        x = int(g["starts"][j])
        for t in range(8):
            x = lc.clock_forward(x, spec)
            assert x == int(g["traj"][j, t])
    p = golden_npz(f"pred_{name}")
    for i in range(0, 4000, 13):
        x = int(p["states"][i])
        assert lc.table_index(x, spec) == int(p["table_index"][i])
        ps = lc.predecessors(x, spec)
        assert ps == [int(v) for v in p["preds"][i][: int(p["npred"][i])]]
        assert lc.is_candidate(x, params[name], spec) == bool(p["is_candidate"][i])


def test_majority_and_registers(lc):
    assert lc.majority_clock_mask(0, 0, 0) == 0b111
    assert lc.majority_clock_mask(1, 1, 0) == 0b011
    assert lc.majority_clock_mask(0, 1, 1) == 0b110
    x = lc.A51.pack(1, 1, 1)
    assert lc.A51.unpack(lc.clock_forward(x, lc.A51)) == (2, 2, 2)
    rng = random.Random(2)
    for s in (lc.A51, lc.MINI567):
        for k in range(3):
            n, tm = s.lengths[k], s.tap_masks[k]
            for _ in range(200):
                r = rng.randrange(1, 1 << n)
                assert lc.unstep_register(lc.step_register(r, n, tm), n, tm) == r
    for _ in range(1000):
        v = rng.getrandbits(64)
        assert lc.parity_fold(v) == bin(v).count("1") & 1


def test_closed_forms(lc):
    assert lc.minimum_cycle_length(lc.A51) == Fraction(33554428, 3)
    assert lc.expected_chain_count(lc.A51, 0) == (2**19 - 1) * (2**22 - 1) - 2**18 * 2**21
    assert lc.default_fixed_r3(lc.A51) == 0x2AAA00
    assert lc.default_fixed_r3(lc.MINI567) == 0x22 and lc.default_fixed_r3(lc.MINI789) == 0xAA
    for x in random_states(lc.A51, 200, seed=11):
        assert lc.unrank_state(lc.rank_state(x, lc.A51), lc.A51) == x


def test_random_candidate_stream_matches_reference(lc, specs, params):
    rc = golden_json("random_candidate.json")
    for name in ("a51", "mini567", "mini789"):
        for seed in range(4):
            rng = random.Random(seed)
            got = [lc.random_candidate(rng, specs[name], params[name]) for _ in range(64)]
            assert got == rc[f"{name}_{seed}"]


def test_kat_starts_are_reference_sampler_prefix(lc, specs, params):
    g = golden_npz("a51_kat256")
    rng = random.Random(0)
    got = [lc.random_candidate(rng, specs["a51"], params["a51"]) for _ in range(256)]
    assert got == g["src"].tolist()


def test_native_reference_sampler_matches_python_random(lc, specs, params):
    """csrc/sampler.cu (host code) restates CPython's MT19937 + randrange stream and the
    reference's random_candidate rejection (pipeline.py:301-310): the same states, in the
    same order, as the Python sampler on a random.Random of the same seed."""
    from paper_1210_6411_b200 import pipeline as P

    rc = golden_json("random_candidate.json")  # produced by the reference itself
    for name in ("a51", "mini567", "mini789"):
        for seed in range(4):
            got = P.reference_candidates(specs[name], params[name], seed, 64)
            assert got.tolist() == rc[f"{name}_{seed}"]
        for seed in (5, 2**32 - 1, 2**32, 2**40 + 7, 2**64 - 1):  # one- and two-word MT keys
            rng = random.Random(seed)
            want = [lc.random_candidate(rng, specs[name], params[name]) for _ in range(500)]
            assert P.reference_candidates(specs[name], params[name], seed, 500).tolist() == want
    # a non-default fixed R3 value (different predicate table)
    p2 = lc.CandidateParams.from_spec(specs["a51"], 0x1234)
    rng = random.Random(9)
    want = [lc.random_candidate(rng, specs["a51"], p2) for _ in range(500)]
    assert P.reference_candidates(specs["a51"], p2, 9, 500).tolist() == want
    multi = P.reference_candidate_streams(specs["mini789"], params["mini789"], [3, 0, 7], 200, threads=2)
    for row, seed in zip(multi, (3, 0, 7)):
        assert (row == P.reference_candidates(specs["mini789"], params["mini789"], seed, 200)).all()


def test_config1_and_config2_starts_from_native_sampler(lc, specs, params):
    """Config 1 = the first 2^16 reference-sampler starts of random.Random(0); config 2
    = the first 2^24 (digests of the reference's own output, tests/golden)."""
    import hashlib

    from paper_1210_6411_b200 import pipeline as P

    c1 = golden_json("a51_c1_65536.json")
    starts = P.reference_candidates(specs["a51"], params["a51"], 0, 1 << 24)
    assert hashlib.sha256(starts[:1 << 16].astype("<u8").tobytes()).hexdigest() == c1["starts_digest"]
    path = os.path.join(ROOT, "tests", "golden", "a51_c2_digests.json")
    if os.path.exists(path):
        c2 = golden_json("a51_c2_digests.json")
        assert hashlib.sha256(starts.astype("<u8").tobytes()).hexdigest() == c2["starts_digest"]


def test_records_byte_exact(lc, tmp_path):
    fx = golden_json("records.json")
    recs = [lc.EdgeRecord(1, 2, 3, 4, 5), lc.EdgeRecord((1 << 64) - 1, 0x5554000000000000, 11184809, 0, 0)]
    p = tmp_path / "e.bin"
    assert lc.write_edges(p, recs) == 2
    assert p.read_bytes().hex() == fx["edges_hex"]
    assert list(lc.read_edges(p)) == recs
    q = tmp_path / "e2.bin"
    lc.write_edge_arrays(q, [r.source for r in recs], [r.destination for r in recs],
                         [r.distance for r in recs], [r.subtree_size for r in recs],
                         [r.subtree_depth for r in recs])
    assert q.read_bytes() == p.read_bytes()
    arr = lc.read_edge_arrays(q)
    assert arr["distance"].tolist() == [3, 11184809]
    s = tmp_path / "s.bin"
    lc.write_states(s, [1, 0x5554000000000001, (1 << 64) - 1])
    assert s.read_bytes().hex() == fx["states_hex"]
    assert list(lc.read_states(s)) == [1, 0x5554000000000001, (1 << 64) - 1]
    c = lc.ByteCounter()
    list(lc.read_edges(p, c))
    assert c.read == 80


def test_transpose_roundtrip_and_fillers(lc):
    rng = random.Random(1)
    for _ in range(50):
        n = rng.randrange(1, 65)
        batch = random_states(lc.A51, n, seed=rng.randrange(1 << 30))
        sb = lc.transpose(batch, lc.A51, 64)
        assert sb.lane_count == n and sb.nbits == 64
        assert lc.untranspose(sb) == batch
    x = random_states(lc.A51, 1, seed=4)[0]
    sb = lc.transpose([x] * 64, lc.A51, 64)
    for i, w in enumerate(sb.words):
        assert w in (0, (1 << 64) - 1) and (w != 0) == bool((x >> i) & 1)
    # the reference's filler lanes are state (1,1,1): word 0 of a 3-lane MINI567 batch
    sb = lc.transpose([1 << j for j in range(3)], lc.MINI567, 64)
    assert sb.words[0] == (((1 << 64) - 1) & ~0b111) | 0b001
    with pytest.raises(ValueError):
        lc.transpose(random_states(lc.A51, 65, seed=0), lc.A51, 64)


def test_shard_ranges_cover_exactly():
    from paper_1210_6411_b200.distributed import shard_range

    for n in (0, 1, 7, 1000, 1 << 20):
        for world in (1, 2, 3, 4, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [hi - lo for lo, hi in spans]
            assert max(sizes) - min(sizes) <= 1


def test_stats_combine_and_summary():
    from paper_1210_6411_b200 import _native as N
    from paper_1210_6411_b200.distributed import combine_stats, stats_summary

    rng = np.random.default_rng(0)
    d = rng.integers(11_180_000, 11_190_000, size=1000).astype(np.uint64)
    lo = 11_184_809 - 32768

    def block(v):
        s = np.zeros(N.ST_HEADER + 66, dtype=np.uint64)
        s[N.ST_EDGES] = v.size
        s[N.ST_TRANSITIONS] = int(v.sum())
        s[N.ST_MIN], s[N.ST_MAX] = v.min(), v.max()
        sq = sum((int(x) - lo) ** 2 for x in v)
        s[N.ST_SQ_LO], s[N.ST_SQ_HI] = sq & ((1 << 64) - 1), sq >> 64
        s[N.ST_ERROR_INDEX] = np.uint64((1 << 64) - 1)
        s[N.ST_HIST_LO] = lo
        s[N.ST_HEADER + 1:N.ST_HEADER + 65] = np.bincount(((v - lo) >> 10).astype(np.int64), minlength=64)[:64]
        return s

    whole = block(d)
    parts = combine_stats([block(d[:300]), block(d[300:700]), block(d[700:])])
    assert (parts == whole).all()
    summ = stats_summary(whole)
    assert summ["edges"] == 1000 and abs(summ["mean"] - d.mean()) < 1e-6
    assert abs(summ["sd"] - d.astype(np.float64).std()) < 1e-3


def test_error_code_and_index_reduce_as_a_pair():
    """A failing shard's (code, global index) travel together: the merged block reports
    the first failing start over all shards and that start's own code."""
    from paper_1210_6411_b200 import _native as N
    from paper_1210_6411_b200.distributed import combine_stats

    def block(code=0, index=(1 << 64) - 1):
        s = np.zeros(N.ST_HEADER + 2, dtype=np.uint64)
        s[N.ST_MIN] = np.uint64((1 << 64) - 1)
        s[N.ST_ERROR] = code
        s[N.ST_ERROR_INDEX] = np.uint64(index)
        return s

    ok = combine_stats([block(), block()], offsets=[0, 100])
    assert ok[N.ST_ERROR] == 0 and ok[N.ST_ERROR_INDEX] == np.uint64((1 << 64) - 1)
    # shard 0 fails late with code 5, shard 1 fails early (local index 3 = global 103)
    # with code 4; shard 2 fails at global 250 with code 4
    m = combine_stats([block(5, 90), block(4, 3), block(4, 50)], offsets=[0, 100, 200])
    assert int(m[N.ST_ERROR]) == 5 and int(m[N.ST_ERROR_INDEX]) == 90
    m = combine_stats([block(), block(4, 3), block(5, 1)], offsets=[0, 100, 200])
    assert int(m[N.ST_ERROR]) == 4 and int(m[N.ST_ERROR_INDEX]) == 103


def test_prune_config_validation_matches_reference(lc):
    fx = golden_json("tuning.json")["prune_config_mini567"]
    for key, want in fx.items():
        mode, d, nl, w = key.split("_")
        cfg = lc.PruneConfig(mode=mode, depth_limit=None if d == "None" else int(d),
                             node_limit=None if nl == "None" else int(nl), workers=int(w))
        try:
            cfg.validate(lc.MINI567)
            got = "ok"
        except ValueError:
            got = "ValueError"
        assert got == want, key


def test_package_exports_reference_namespace():
    """Every name the reference package exports (pkg/src/lfsrcycles/__init__.py:3-32)."""
    import paper_1210_6411_b200 as pkg

    names = ("A51 MINI567 MINI789 CandidateParams CipherSpec PredecessorTable build_predecessor_table "
             "builtin_spec clock_forward default_fixed_r3 expected_chain_count expected_chain_length "
             "is_candidate majority_clock_mask minimum_cycle_length predecessors SlicedBatch calibrate_stride "
             "clock_sliced forward_to_candidate transpose untranspose PruneConfig build_skeleton_edges "
             "enumerate_candidates prune_shallow_segments EdgeRecord CycleRecord ReduceConfig count_cycles "
             "cut_leaves_pass cut_leaves_to_fixpoint GroundTruth brute_force_analysis AnalysisReport "
             "ExpectationTable SampleStats deviation_report random_mapping_expectations "
             "sample_segment_distances sample_segment_shapes").split()
    assert [n for n in names if not hasattr(pkg, n)] == []
    # the reference's submodules exist under the same names (lfsrcycles.<module>)
    import importlib

    for mod, attrs in {"cipher": ("A51", "predecessors"), "bitslice": ("forward_to_candidate",),
                       "pipeline": ("prune_shallow_segments", "random_candidate"), "records": ("write_edges",),
                       "reduce": ("cut_leaves_to_fixpoint",), "oracle": ("brute_force_analysis", "GroundTruth"),
                       "stats": ("sample_segment_distances",)}.items():
        m = importlib.import_module(f"paper_1210_6411_b200.{mod}")
        assert all(hasattr(m, a) for a in attrs), mod


def test_missing_library_fails_loudly(tmp_path):
    """No CPU fallback: without the CUDA library the package import raises ImportError."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, LFSR_LIB=str(tmp_path / "missing.so"))
    code = "import paper_1210_6411_b200"
    r = subprocess.run([sys.executable, "-c", code], cwd=os.path.dirname(os.path.dirname(__file__)), env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "no CPU fallback" in r.stderr.replace("There is no", "no")


def test_build_entry_does_not_need_the_library(tmp_path):
    """__graft_entry__.build() must work on a fresh checkout: loading the build script may
    not import the package (whose __init__ refuses to load without the library)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import importlib.util, os, sys; sys.path.insert(0, '.'); import __graft_entry__; "
            "assert 'paper_1210_6411_b200' not in sys.modules; "
            "spec = importlib.util.spec_from_file_location('b', os.path.join('paper_1210_6411_b200', 'build.py')); "
            "m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m); "
            "assert 'paper_1210_6411_b200' not in sys.modules; print('ok')")
    env = dict(os.environ, LFSR_LIB=str(tmp_path / "missing.so"))
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True)
    assert r.returncode == 0 and r.stdout.strip() == "ok", r.stderr
