"""The C ABI as a standalone library: examples/walk_c1.c -- a C program with no Python
and no torch -- is compiled against include/lfsr_b200.h, linked with the in-tree
liblfsr_b200.so, and run; its walk of the reference sampler's first config-1 starts must
equal the C restatement of the reference (oracle/lfsr_oracle.c) on the same starts."""

from __future__ import annotations

import os
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_host_walk_matches_restatement(gpu, tmp_path):
    from oracle import port

    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    lib_dir = os.path.join(ROOT, "paper_1210_6411_b200", "_lib")
    exe = str(tmp_path / "walk_c1")
    subprocess.run([gcc, "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "examples", "walk_c1.c"), "-L", lib_dir, "-llfsr_b200",
                    f"-Wl,-rpath,{lib_dir}", "-o", exe], check=True)
    n = 2048
    out = subprocess.run([exe, str(n)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    got = out.stdout.split()
    starts = port.random_candidates(port.A51, 0x2AAA00, 0, n)
    dst, dist = port.walk(port.A51, 0x2AAA00, starts, stride=11_170_000)
    dst, dist = dst[:, 0].astype(np.uint64), dist[:, 0].astype(np.uint64)
    h = 1469598103934665603
    for d, w in zip(dst.tolist(), dist.tolist()):
        h = ((h ^ d) * 1099511628211) & (2**64 - 1)
        h = ((h ^ w) * 1099511628211) & (2**64 - 1)
    assert got == [str(n), str(int(dist.sum())), str(int(dist.min())), str(int(dist.max())), f"{h:016x}"]
