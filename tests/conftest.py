"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything else runs on
CPU (the oracle vs the reference's golden vectors, host logic, ABI exports, gloo)."""

from __future__ import annotations

import json
import os
import random
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
    # a fresh checkout: compile the library (and the C oracle) once before collecting,
    # exactly as __graft_entry__.build() does; nvcc cross-compiles without a GPU
    if not os.environ.get("LFSR_LIB") and not os.path.exists(
            os.path.join(ROOT, "paper_1210_6411_b200", "_lib", "liblfsr_b200.so")):
        import __graft_entry__

        __graft_entry__.build()


def golden_npz(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def has_golden(name):
    return os.path.exists(os.path.join(GOLDEN, name))


def random_states(spec, n, seed):
    """The reference tests' sampler (pkg/tests/conftest.py:43-46)."""
    from paper_1210_6411_b200.cipher import unrank_state

    rng = random.Random(seed)
    total = spec.valid_state_count
    return [unrank_state(rng.randrange(total), spec) for _ in range(n)]


@pytest.fixture(scope="session")
def lc():
    import paper_1210_6411_b200 as pkg

    return pkg


@pytest.fixture(scope="session")
def specs(lc):
    return {"a51": lc.A51, "mini567": lc.MINI567, "mini789": lc.MINI789}


@pytest.fixture(scope="session")
def params(lc, specs):
    return {k: lc.CandidateParams.from_spec(s, lc.default_fixed_r3(s)) for k, s in specs.items()}


@pytest.fixture(scope="session")
def gpu():
    """GPU tests fail (not skip) without a device: a silent skip would hide a missing
    native path on the GPU box.  CPU runs deselect them with -m "not gpu"."""
    from paper_1210_6411_b200 import _native

    if _native.device_count() == 0:
        pytest.fail("no CUDA device visible to liblfsr_b200")
    return _native.context()
