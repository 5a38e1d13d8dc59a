"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the C restatement (lfsr_oracle.c).

Functions take a spec-like object (``.lengths``, ``.taps``, ``.clock_taps``) and
numpy ``uint64`` arrays; they mirror the reference semantics they cite.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_build", "liboracle.so")

OK, STRIDE_ERROR, VALUE_ERROR, ARG_ERROR = 0, 1, 2, 3


class OracleError(RuntimeError):
    pass


class OracleStrideError(OracleError):
    """Reference would raise bitslice.StrideError (bitslice.py:316-322)."""


class OracleValueError(OracleError):
    """Reference would raise ValueError from min() of an empty sequence (bitslice.py:317)."""


class SpecConst:
    """Spec-like constants (``.lengths``, ``.taps``, ``.clock_taps``) of a built-in cipher,
    so callers that must not import the product package (bench.py's reference arm) can
    name one: A5/1 is cipher.py:173-178."""

    def __init__(self, lengths, taps, clock_taps):
        self.lengths, self.taps, self.clock_taps = tuple(lengths), tuple(taps), tuple(clock_taps)
        self.reg_masks = tuple((1 << l) - 1 for l in self.lengths)
        self.offsets = (0, self.lengths[0], self.lengths[0] + self.lengths[1])


A51 = SpecConst((19, 22, 23), ((13, 16, 17, 18), (20, 21), (7, 20, 21, 22)), (8, 10, 10))


def random_candidates(spec, fixed_r3: int, seed: int, n: int) -> np.ndarray:
    """``random_candidate(random.Random(seed), ...)`` x n (pipeline.py:301-310): rejection
    over (randrange(1, m1+1), randrange(1, m2+1)) with R3 fixed, drawn from Python's own
    generator and tested with the C restatement of is_candidate (cipher.py:420-428)."""
    import random

    rng = random.Random(seed)
    m1, m2, _ = spec.reg_masks
    o2, o3 = spec.offsets[1], spec.offsets[2]
    packed = int(fixed_r3) << o3
    lib, s = load(), spec_struct(spec)
    out = np.empty(int(n), dtype=np.uint64)
    for i in range(int(n)):
        while True:
            x = rng.randrange(1, m1 + 1) | (rng.randrange(1, m2 + 1) << o2) | packed
            if lib.orc_is_candidate(C.byref(s), int(fixed_r3), x):
                out[i] = x
                break
    return out


class _Spec(C.Structure):
    _fields_ = [("len", C.c_int * 3), ("tap", C.c_uint64 * 3), ("ct", C.c_int * 3)]


def spec_struct(spec) -> _Spec:
    s = _Spec()
    for k in range(3):
        s.len[k] = int(spec.lengths[k])
        m = 0
        for t in spec.taps[k]:
            m |= 1 << int(t)
        s.tap[k] = m
        s.ct[k] = int(spec.clock_taps[k])
    return s


_lib = None
_u64p = C.POINTER(C.c_uint64)


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB):
        build()
    lib = C.CDLL(LIB)
    sp = C.POINTER(_Spec)
    lib.orc_clock_forward.argtypes = [sp, C.c_uint64]
    lib.orc_clock_forward.restype = C.c_uint64
    lib.orc_predecessors.argtypes = [sp, C.c_uint64, _u64p]
    lib.orc_predecessors.restype = C.c_int
    lib.orc_is_candidate.argtypes = [sp, C.c_uint64, C.c_uint64]
    lib.orc_is_candidate.restype = C.c_int
    lib.orc_table_index.argtypes = [sp, C.c_uint64]
    lib.orc_table_index.restype = C.c_int
    lib.orc_table_entry.argtypes = [C.c_int, C.POINTER(C.c_int)]
    lib.orc_table_entry.restype = C.c_int
    lib.orc_enumerate.argtypes = [sp, C.c_uint64, C.c_uint64, C.c_uint64, _u64p, C.c_uint64]
    lib.orc_enumerate.restype = C.c_uint64
    lib.orc_clock_n.argtypes = [sp, _u64p, C.c_uint64, C.c_uint64, _u64p]
    lib.orc_clock_n.restype = None
    lib.orc_clock_sliced.argtypes = [sp, _u64p, C.c_uint64, C.c_uint64, _u64p]
    lib.orc_clock_sliced.restype = None
    lib.orc_prune.argtypes = [sp, C.c_uint64, C.c_int, C.c_uint64, _u64p, C.c_uint64,
                              C.POINTER(C.c_uint8), _u64p]
    lib.orc_prune.restype = C.c_int
    lib.orc_probe_segment.argtypes = [sp, C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _u64p,
                                      C.POINTER(C.c_int), _u64p, C.c_uint64]
    lib.orc_probe_segment.restype = C.c_uint64
    lib.orc_walk.argtypes = [sp, C.c_uint64, _u64p, C.c_uint64, C.c_uint64, C.c_uint32,
                             C.c_uint64, C.c_int, _u64p, _u64p, C.POINTER(C.c_int64)]
    lib.orc_walk.restype = C.c_int
    _lib = lib
    return lib


def _arr(x) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(x, dtype=np.uint64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


def clock_forward(spec, x: int) -> int:
    return int(load().orc_clock_forward(C.byref(spec_struct(spec)), int(x)))


def clock_n(spec, xs, t: int) -> np.ndarray:
    xs = _arr(xs)
    out = np.empty_like(xs)
    load().orc_clock_n(C.byref(spec_struct(spec)), _p(xs), xs.size, int(t), _p(out))
    return out


def clock_sliced(spec, xs, t: int) -> np.ndarray:
    xs = _arr(xs)
    out = np.empty_like(xs)
    load().orc_clock_sliced(C.byref(spec_struct(spec)), _p(xs), xs.size, int(t), _p(out))
    return out


def predecessors(spec, x: int) -> list[int]:
    out = np.zeros(4, dtype=np.uint64)
    n = load().orc_predecessors(C.byref(spec_struct(spec)), int(x), _p(out))
    return [int(v) for v in out[:n]]


def table_index(spec, x: int) -> int:
    return int(load().orc_table_index(C.byref(spec_struct(spec)), int(x)))


def table_entries() -> list[tuple[int, ...]]:
    out = (C.c_int * 4)()
    res = []
    for i in range(64):
        n = load().orc_table_entry(i, out)
        res.append(tuple(out[k] for k in range(n)))
    return res


def is_candidate(spec, fixed_r3: int, x: int) -> bool:
    return bool(load().orc_is_candidate(C.byref(spec_struct(spec)), int(fixed_r3), int(x)))


def enumerate_rows(spec, fixed_r3: int, r2_lo: int, r2_hi: int) -> np.ndarray:
    lib = load()
    s = spec_struct(spec)
    n = lib.orc_enumerate(C.byref(s), int(fixed_r3), int(r2_lo), int(r2_hi), None, 0)
    out = np.empty(n, dtype=np.uint64)
    lib.orc_enumerate(C.byref(s), int(fixed_r3), int(r2_lo), int(r2_hi), _p(out), n)
    return out


def prune(spec, fixed_r3: int, mode: str, limit: int, cands):
    """Per-candidate (removed, work) as in pipeline._prune_chunk (pipeline.py:163-178)."""
    cands = _arr(cands)
    removed = np.zeros(cands.size, dtype=np.uint8)
    work = np.zeros(cands.size, dtype=np.uint64)
    load().orc_prune(C.byref(spec_struct(spec)), int(fixed_r3), 0 if mode == "dfs" else 1,
                     int(limit), _p(cands), cands.size,
                     removed.ctypes.data_as(C.POINTER(C.c_uint8)), _p(work))
    return removed, work


def probe_segment(spec, fixed_r3: int, root: int, depth_cap=None, node_cap=None, levels=4096):
    nodes = C.c_uint64()
    cens = C.c_int()
    lc = np.zeros(levels, dtype=np.uint64)
    depth = load().orc_probe_segment(C.byref(spec_struct(spec)), int(fixed_r3), int(root),
                                     -1 if depth_cap is None else int(depth_cap),
                                     -1 if node_cap is None else int(node_cap),
                                     C.byref(nodes), C.byref(cens), _p(lc), levels)
    return int(depth), int(nodes.value), bool(cens.value), lc[: int(depth) + 1].tolist()


def walk(spec, fixed_r3: int, starts, *, stride: int = 1, legs: int = 1, max_clocks=None,
         width: int = 0):
    """bitslice._run_walks restated (bitslice.py:259-323).

    Returns (dst, dist) arrays of shape [n, legs].  Raises OracleStrideError /
    OracleValueError where the reference raises StrideError / ValueError.
    """
    from fractions import Fraction

    if stride < 1 or legs < 1:
        raise ValueError("stride must be >= 1 / legs must be >= 1")
    if max_clocks is None:
        l3 = spec.lengths[2]
        max_clocks = 16 * int(Fraction(4 * ((1 << l3) - 1), 3)) + 64
    starts = _arr(starts)
    n = starts.size
    dst = np.zeros((n, legs), dtype=np.uint64)
    dist = np.zeros((n, legs), dtype=np.uint64)
    bad = C.c_int64(-1)
    rc = load().orc_walk(C.byref(spec_struct(spec)), int(fixed_r3), _p(starts), n, int(stride),
                         int(legs), int(max_clocks), int(width), _p(dst), _p(dist), C.byref(bad))
    if rc == STRIDE_ERROR:
        raise OracleStrideError(f"wave {bad.value}: walk cap {max_clocks} exceeded")
    if rc == VALUE_ERROR:
        raise OracleValueError(f"wave {bad.value}: min() iterable argument is empty")
    if rc == ARG_ERROR:
        raise ValueError("bad walk arguments")
    return dst, dist
