"""Every kernel control-flow mode on the checked library build (-DLC_CHECKS=1, built by
__graft_entry__.build() into paper_1210_6411_b200/_lib/checked/): device-side bounds and
invariant checks on the parked-lane pool, the walk's item indices, the prune's
shared-memory ring and global spill ring, and the sort's staging and scatter positions
trap on violation, failing the call.  (compute-sanitizer cannot be used on this GPU pool:
it is closed there.)  Each mode also checks its results against the C restatement."""

from __future__ import annotations

import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

TARGET = os.path.join(ROOT, "tests", "_kernel_modes.py")
CHECKED = os.path.join(ROOT, "paper_1210_6411_b200", "_lib", "checked", "liblfsr_b200.so")
MODES = ["walk_warp", "walk_lane", "walk_park", "walk_park_device", "prune", "prune_v2", "prune_spill", "enumerate",
         "sort"]


@pytest.mark.parametrize("mode", MODES)
def test_checked_build_runs_clean(gpu, mode):
    assert os.path.exists(CHECKED), "checked build missing: run __graft_entry__.build()"
    env = dict(os.environ, LFSR_LIB=CHECKED)
    if mode == "prune_spill":
        env["LFSR_PRUNE_SPILL"] = "2"  # v2's spill ring overflowed: exercises drop-and-climb
        env["LFSR_PRUNE_V1"] = "2"
    if mode == "prune_v2":  # DFS on the v2 kernel (the default DFS kernel is v3)
        env["LFSR_PRUNE_V1"] = "2"
    out = subprocess.run([sys.executable, TARGET, mode], env=env, cwd=ROOT, capture_output=True, text=True,
                         timeout=900)
    log = out.stdout + out.stderr
    assert out.returncode == 0 and f"{mode}: ok" in log, log[-4000:]
    assert "LC_CHECK failed" not in log
