"""Pins the C oracle (oracle/lfsr_oracle.c) to the reference: every fixture here was
produced by the unmodified reference (oracle/gen_golden.py).  CPU only."""

from __future__ import annotations

import hashlib

import numpy as np
import pytest

from conftest import golden_json, golden_npz, has_golden

from oracle import port


def edge_digest(src, dst, dist):
    rows = sorted(zip((int(s) for s in src), (int(d) for d in dst), (int(w) for w in dist)))
    h = hashlib.sha256()
    for s, d, w in rows:
        h.update(f"{s:016x} {d:016x} {w}\n".encode())
    return h.hexdigest()


def u64_digest(values):
    return hashlib.sha256(np.asarray(values, dtype="<u8").tobytes()).hexdigest()


def test_table_matches_reference():
    t = golden_json("tables.json")
    assert [list(e) for e in port.table_entries()] == t["entries"]
    assert t["nonempty_mask"] == "0xb5bf5d0db0bafdad"


@pytest.mark.parametrize("name", ["a51", "mini567", "mini789"])
def test_trajectories(specs, name):
    g = golden_npz(f"traj_{name}")
    assert (port.clock_n(specs[name], g["starts"], 1) == g["traj"][:, 0]).all()
    assert (port.clock_n(specs[name], g["starts"], 64) == g["traj"][:, 63]).all()
    assert (port.clock_sliced(specs[name], g["starts"], 500) == g["after500"]).all()


@pytest.mark.parametrize("name", ["a51", "mini567", "mini789"])
def test_predicate_and_predecessors(specs, params, name):
    g = golden_npz(f"pred_{name}")
    F = params[name].fixed_r3
    for i in range(0, g["states"].size, 3):
        x = int(g["states"][i])
        ps = port.predecessors(specs[name], x)
        assert len(ps) == g["npred"][i]
        assert ps == [int(v) for v in g["preds"][i][: len(ps)]]
        assert port.is_candidate(specs[name], F, x) == bool(g["is_candidate"][i])
        assert port.table_index(specs[name], x) == g["table_index"][i]


@pytest.mark.parametrize("name", ["mini567", "mini789"])
def test_mini_edges_and_strides(specs, params, name):
    spec, F = specs[name], params[name].fixed_r3
    g = golden_npz(f"edges_{name}")
    meta = golden_json(f"edges_{name}.json")
    cands = port.enumerate_rows(spec, F, 1, 1 << spec.lengths[1])
    assert (cands == g["src"]).all()
    d, w = port.walk(spec, F, cands)
    assert edge_digest(cands, d[:, 0], w[:, 0]) == meta["digest"]
    d, w = port.walk(spec, F, g["random_starts"])
    assert (d[:, 0] == g["random_dst"]).all() and (w[:, 0] == g["random_dist"]).all()
    for s in (16, 100, 127, 148, 149, 150, 200):
        d, w = port.walk(spec, F, cands, stride=s)
        assert (d[:, 0] == g[f"stride_{s}_dst"]).all() and (w[:, 0] == g[f"stride_{s}_dist"]).all()
    d, w = port.walk(spec, F, g["hop_starts"], legs=2)
    assert (np.stack([d[:, 0], w[:, 0], d[:, 1], w[:, 1]], 1) == g["hop2"]).all()


def test_cap_band_reproduces_reference_quirks(specs, params):
    cap = golden_json("cap_mini567.json")
    for mc, outcome in cap["band"].items():
        try:
            d, w = port.walk(specs["mini567"], 0x22, [cap["first_candidate"]], max_clocks=int(mc))
            got = ["ok", int(d[0, 0]), int(w[0, 0])]
        except port.OracleStrideError:
            got = ["StrideError"]
        except port.OracleValueError:
            got = ["ValueError"]
        assert got == outcome[: len(got)]
    with pytest.raises(port.OracleStrideError):
        port.walk(specs["mini567"], 0x22, cap["cap3_starts"], max_clocks=3)


def test_a51_kat(specs, params):
    g = golden_npz("a51_kat256")
    meta = golden_json("a51_kat256.json")
    d, w = port.walk(specs["a51"], 0x2AAA00, g["src"], stride=11_170_000)
    assert (d[:, 0] == g["dst"]).all() and (w[:, 0] == g["dist"]).all()
    assert edge_digest(g["src"], d[:, 0], w[:, 0]) == meta["digest"]


def test_enumerate_rows_a51():
    meta = golden_json("enumerate.json")
    import paper_1210_6411_b200 as lc

    got = port.enumerate_rows(lc.A51, 0x2AAA00, 0x1234, 0x1234 + 4)
    want = meta["a51_rows_0x1234_4"]
    assert got.size == want["count"] and u64_digest(got) == want["digest"]


@pytest.mark.skipif(not has_golden("prune.json"), reason="prune fixture not generated")
def test_prune_matches_reference(specs, params):
    fx = golden_json("prune.json")
    cands = np.array(fx["a51_cands"], dtype=np.uint64)
    for key in ("a51_dfs_56", "a51_dfs_319", "a51_bfs_1000"):
        _, mode, lim = key.split("_")
        removed, work = port.prune(specs["a51"], 0x2AAA00, mode, int(lim), cands)
        want = fx[key]
        assert cands[removed == 0].tolist() == want["survivors"]
        assert int(work.sum()) == want["expanded"]
    for name in ("mini567", "mini789"):
        spec, F = specs[name], params[name].fixed_r3
        mc = port.enumerate_rows(spec, F, 1, 1 << spec.lengths[1])
        for key, want in fx.items():
            if key.startswith(name + "_") and not key.endswith("probe"):
                _, mode, lim = key.split("_")
                removed, work = port.prune(spec, F, mode, int(lim), mc)
                assert u64_digest(mc[removed == 0]) == want["survivors_digest"]
                assert int(work.sum()) == want["expanded"]


@pytest.mark.skipif(not has_golden("a51_c1_65536.json"), reason="C1 fixture not generated")
def test_c1_sample_rows(specs):
    """Spot rows of the full 2^16 config-1 reference run (every 256th walk)."""
    g = golden_npz("a51_c1_sample")
    d, w = port.walk(specs["a51"], 0x2AAA00, g["src"], stride=11_170_000)
    assert (d[:, 0] == g["dst"]).all() and (w[:, 0] == g["dist"]).all()


@pytest.mark.skipif(not has_golden("reduce.json"), reason="reduce fixture not generated")
def test_reduce_restatement_matches_reference(specs):
    """oracle/reduce_np.py vs the reference's cut_leaves_pass iterated to the fixpoint
    and count_cycles, on the full mini candidate sets."""
    from oracle import reduce_np

    fx = golden_json("reduce.json")
    for name in ("mini567", "mini789"):
        g = golden_npz(f"edges_{name}")
        z = np.zeros(g["src"].size, dtype=np.uint64)
        want = fx[f"{name}_full"]
        out = reduce_np.cut_leaves(g["src"], g["dst"], g["dist"], z, z)
        assert [list(p) for p in out[5]] == want["passes"]
        fix = np.stack(out[:5], 1).tolist()
        assert fix == want["fixpoint"]
        assert [list(c) for c in reduce_np.count_cycles(*out[:4])] == want["cycles"]
        one = reduce_np.cut_leaves(g["src"], g["dst"], g["dist"], z, z, max_passes=1)
        assert list(one[5][0]) == [want["pass1"][k] for k in ("leaves_removed", "inner_nodes", "out_size_sum")]
        assert u64_digest(np.stack(one[:5], 1).reshape(-1)) == want["pass1"]["records_digest"]


def _avx512():
    try:
        return "avx512f" in open("/proc/cpuinfo").read()
    except OSError:
        return False


@pytest.mark.skipif(not _avx512(), reason="oracle/walk512.c needs AVX-512 (build container only)")
def test_walk512_pinned_on_the_reference_config1_run():
    """oracle/walk512.c (the generator of the config-2 digests) reproduces the reference's
    own config-1 run (65,536 walks, _edges_chunk over a process pool) and the 256-walk KAT
    before its 2^24-walk output is trusted (tests/golden/a51_c2_digests.json)."""
    import ctypes as C
    import hashlib
    import os
    import subprocess

    from conftest import ROOT

    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "walk512"], check=True)
    lib = C.CDLL(os.path.join(odir, "_build", "libwalk512.so"))
    u = C.POINTER(C.c_uint64)
    lib.w512_walk.argtypes = [C.c_uint32, u, C.c_uint64, C.c_uint64, C.c_uint64, u, u, u]

    def walk(starts):
        starts = np.ascontiguousarray(starts, dtype=np.uint64)
        dst, dist, bad = (np.zeros(starts.size, np.uint64) for _ in range(3))
        p = lambda a: a.ctypes.data_as(u)  # noqa: E731
        assert lib.w512_walk(0x2AAA00, p(starts), starts.size, 11_170_000, 178_957_008, p(dst), p(dist), p(bad)) == 0
        return dst, dist

    kat = golden_npz("a51_kat256")
    d, w = walk(kat["src"])
    assert (d == kat["dst"]).all() and (w == kat["dist"]).all()
    c1 = golden_json("a51_c1_65536.json")
    c2 = golden_json("a51_c2_digests.json")
    sample = golden_npz("a51_c1_sample")
    from paper_1210_6411_b200 import A51, CandidateParams
    from paper_1210_6411_b200.pipeline import reference_candidates

    starts = reference_candidates(A51, CandidateParams.from_spec(A51, 0x2AAA00), 0, 1 << 16)
    assert (starts[sample["idx"].astype(np.int64)] == sample["src"]).all()
    d, w = walk(starts)
    assert hashlib.sha256(d.astype("<u8").tobytes()).hexdigest() == c1["dst_digest"]
    assert hashlib.sha256(w.astype("<u8").tobytes()).hexdigest() == c1["dist_digest"]
    # the committed config-2 batches: batch 0's first 2^16 rows are config 1
    assert c2["c1_prefix_starts_digest"] == c1["starts_digest"] and c2["n"] == 1 << 24
    assert sum(b["sum_dist"] for b in c2["batches"]) == c2["sum_dist"]
