"""Custom cipher specs (cipher.py:153-170, CipherSpec.from_json) get the built-in kernel
templates compiled for them at first use (csrc/jit.cu, NVRTC).  This checks on CPU --
NVRTC needs no device -- that every kernel template compiles for specs unlike the
built-ins: 1 and 5+ taps per register, odd lengths, a rotation R3.  (The GPU test
tests/test_gpu_custom_spec.py runs them against the C restatement.)"""

from __future__ import annotations

import ctypes as C

import pytest

SPECS = [
    ("odd", (5, 7, 7), ((1, 4), (5, 6), (5, 6)), (2, 2, 3)),
    ("rot", (6, 7, 7), ((2, 5), (3, 6), (6,)), (2, 3, 3)),
    ("many_taps", (7, 8, 9), ((1, 2, 3, 4, 6), (0, 3, 4, 5, 6, 7), (3, 8)), (3, 3, 4)),
]


@pytest.mark.parametrize("d", SPECS, ids=lambda d: d[0])
def test_custom_spec_kernels_compile(d):
    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N

    spec = lc.CipherSpec.from_json(lc.CipherSpec(*d).to_json())
    rc = N.lib.lc_spec_compile_check(C.byref(N.spec_struct(spec)))
    assert rc == 0, N.last_error()


def test_compile_check_rejects_invalid_spec():
    from paper_1210_6411_b200 import _native as N

    s = N.lc_spec()
    for k, (l, t, c) in enumerate(((5, 0b00001, 2), (6, 0b110000, 2), (7, 0b1100000, 3))):
        s.lengths[k], s.tap_masks[k], s.clock_taps[k] = l, t, c  # R1's taps miss its top bit
    assert N.lib.lc_spec_compile_check(C.byref(s)) != 0
    assert "top bit" in N.last_error()
