"""The bench line's contract, checked on the committed default-bench record
(profiles/r02_bench_default.json, written by `python bench.py` on a B200): every key the
driver and the judge read is present with the right type, the roofline / CPU baseline /
end-to-end / clocks objects are complete, and the internal arithmetic holds (value =
transitions / time, frac = achieved / peak)."""

from __future__ import annotations

import json
import os

import pytest

from conftest import ROOT

RECORD = os.path.join(ROOT, "profiles", "r02_bench_default.json")


@pytest.fixture(scope="module")
def line():
    if not os.path.exists(RECORD):
        pytest.skip("no committed bench record")
    with open(RECORD) as f:
        return json.load(f)


def test_required_keys(line):
    for k, t in (("metric", str), ("value", float), ("unit", str), ("n_gpus", int), ("steps", int),
                 ("warmup", int), ("ms_per_step", float), ("higher_is_better", bool), ("scaling", str),
                 ("dtype", str), ("data", str), ("config", dict), ("gpu_launches", int)):
        assert isinstance(line[k], t), k
    assert "vs_baseline" in line
    assert line["warmup"] >= 3 and line["steps"] >= 1
    assert "workload" in line["config"] and "l2" in line["config"]


def test_roofline_cpu_baseline_e2e_clocks(line):
    r = line["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac"):
        assert k in r, k
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    c = line["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("port", "reference") and c["matches_gpu"] is True
    e = line["e2e"]
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in e, k
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    ck = line["clocks"]
    assert ck["sm_mhz"] and ck["sm_max_mhz"] and isinstance(ck["reasons"], list)
    assert not {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"} & set(ck["reasons"])


def test_value_is_transitions_over_time_and_parity_green(line):
    ws = line["walk_stats"]
    t = line["ms_per_step"] * line["steps"] / 1e3
    assert abs(ws["transitions"] / t - line["value"]) / line["value"] < 1e-6
    p = line["parity"]
    assert p["c1_reference_digest"] and p["c2_starts_digest"] and all(p["c2_batches"])


def test_steps12_and_next_rows(line):
    s = line["steps12"]
    assert s["k2_enumerate"]["parity_first_4_rows_vs_oracle"] and s["k3_prune"]["parity_sample_vs_oracle"]
    assert s["k3_prune"]["roofline"]["frac"] > 0
    n = line["next_rows"]
    assert n["edge_sort"]["ascending"] and n["edge_sort"]["stable"]
    assert n["parity_2p20_sort_cut_cycles_vs_restatement"]
