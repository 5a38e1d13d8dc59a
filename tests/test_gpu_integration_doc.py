"""The minimal ctypes binding printed in INTEGRATION.md §2 (what a maintainer would add
next to the reference) runs as written and returns the package's results."""

from __future__ import annotations

import os
import re

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_integration_stub_runs(gpu, lc, specs, params):
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    stub = next(b for b in re.findall(r"```python\n(.*?)```", text, re.S) if "lc_ctx_create" in b)
    ns: dict = {"StrideError": lc.StrideError}
    cwd = os.getcwd()
    os.chdir(ROOT)  # the stub loads the library by its repo-relative path
    try:
        exec(compile(stub, "INTEGRATION.md", "exec"), ns)
    finally:
        os.chdir(cwd)
    cands = list(lc.enumerate_candidates(specs["mini567"], params["mini567"]))
    got = ns["forward_to_candidate"](cands, params["mini567"], specs["mini567"])
    assert got == lc.forward_to_candidate(cands, params["mini567"], specs["mini567"])
