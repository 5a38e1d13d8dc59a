"""Array front end of the C ABI: numpy ``uint64`` in, numpy out, GPU in between.

These are the fast paths behind the reference-shaped API (``bitslice``, ``pipeline``,
``cipher`` batch forms).  Every function here launches CUDA kernels; none has a host
implementation.
"""

from __future__ import annotations

import ctypes as C
from fractions import Fraction

import numpy as np

from . import _native as N


class StrideError(RuntimeError):
    """A walk exceeded its clock cap: wrong fixed R3 / stride configuration
    (bitslice.py:49-50)."""


class UnsupportedSpecError(NotImplementedError):
    """No compiled kernel for this cipher instance (built-ins only; no CPU fallback)."""


def _raise(err: N.NativeError, max_clocks=None):
    if err.code == N.LC_ERR_CAP or err.code == N.LC_ERR_INVALID_STATE:
        raise StrideError("no candidate within %s clocks; check the fixed R3 / stride configuration"
                          % (max_clocks,)) from err
    if err.code == N.LC_ERR_ARG:
        raise ValueError(str(err)) from err
    if err.code == N.LC_ERR_UNSUPPORTED:
        raise UnsupportedSpecError(str(err)) from err
    raise err


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def default_max_clocks(spec) -> int:
    """bitslice.py:273-274: 16 * int(L) + 64 with L = (4/3)(2^l3 - 1)."""
    return 16 * int(Fraction(4 * ((1 << spec.lengths[2]) - 1), 3)) + 64


def default_histogram(spec):
    """(hist_lo, shift, bins): 1-clock bins over L +- 2^15 for A5/1, [0, 2^12) for minis."""
    if spec.lengths[2] >= 20:
        center = int(Fraction(4 * ((1 << spec.lengths[2]) - 1), 3))
        return center - (1 << 15), 0, 1 << 16
    return 0, 0, 1 << 12


class WalkResult:
    """Walk output: dest/dist arrays [n, legs] plus the GPU statistics block."""

    def __init__(self, dst, dist, stats):
        self.dst = dst
        self.dist = dist
        self.stats = stats

    @property
    def edges(self) -> int:
        return int(self.stats[N.ST_EDGES])

    @property
    def transitions(self) -> int:
        return int(self.stats[N.ST_TRANSITIONS])

    @property
    def histogram(self) -> np.ndarray:
        return self.stats[N.ST_HEADER:]


def walk(starts, params, spec, *, stride: int = 1, legs: int = 1, max_clocks=None, refill: int = 0,
         histogram=None, device=None) -> WalkResult:
    """GPU chain walk (replaces bitslice._run_walks, bitslice.py:259-323)."""
    if stride < 1:
        raise ValueError("stride must be >= 1")
    if legs < 1:
        raise ValueError("legs must be >= 1")
    if max_clocks is None:
        max_clocks = default_max_clocks(spec)
    max_clocks = min(int(max_clocks), (1 << 64) - 1)
    lo, shift, bins = histogram or default_histogram(spec)
    s = _u64(starts)
    n = s.size
    dst = np.zeros((n, legs), dtype=np.uint64)
    dist = np.zeros((n, legs), dtype=np.uint64)
    stats = np.zeros(N.ST_HEADER + bins + 2, dtype=np.uint64)
    ctx = N.context(device)
    rc = N.lib.lc_walk(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3, N.u64p(s), n,
                       int(stride), max_clocks, int(legs), int(refill), N.u64p(dst), N.u64p(dist),
                       int(lo), int(shift), int(bins), N.u64p(stats))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()), max_clocks)
    return WalkResult(dst, dist, stats)


def clock(states, spec, t: int) -> np.ndarray:
    """Every state advanced t clocks by the bitsliced GPU stepper."""
    if t < 0:
        raise ValueError("clock count must be >= 0")
    s = _u64(states)
    out = np.empty_like(s)
    ctx = N.context()
    rc = N.lib.lc_clock(ctx.handle, C.byref(N.spec_struct(spec)), N.u64p(s), s.size, int(t), N.u64p(out))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return out


def is_candidate(states, params, spec) -> np.ndarray:
    s = _u64(states)
    out = np.zeros(s.size, dtype=np.uint8)
    ctx = N.context()
    rc = N.lib.lc_is_candidate(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3, N.u64p(s), s.size,
                               N.u8p(out))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return out.astype(bool).reshape(np.shape(states))


def predecessors(states, spec):
    s = _u64(states)
    out = np.zeros((s.size, 4), dtype=np.uint64)
    cnt = np.zeros(s.size, dtype=np.uint8)
    ctx = N.context()
    rc = N.lib.lc_predecessors(ctx.handle, C.byref(N.spec_struct(spec)), N.u64p(s), s.size, N.u64p(out),
                               N.u8p(cnt))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return out, cnt


def enumerate_rows(spec, params, r2_lo: int, r2_hi: int) -> np.ndarray:
    """All special nodes with R2 in [r2_lo, r2_hi), ascending (GPU closed-form writer, K2)."""
    m1 = spec.reg_masks[0]
    cap = max(1, (r2_hi - r2_lo) * m1 // 2 + 1024)
    ctx = N.context()
    while True:
        out = np.empty(cap, dtype=np.uint64)
        count = C.c_uint64(0)
        rc = N.lib.lc_enumerate(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3, int(r2_lo),
                                int(r2_hi), N.u64p(out), cap, C.byref(count))
        if rc == N.LC_ERR_OVERFLOW:
            cap = int(count.value)
            continue
        if rc != N.LC_OK:
            _raise(N.NativeError(rc, N.last_error()))
        return out[: int(count.value)]


def prune(cands, spec, params, mode: str, limit: int, device=None):
    """Per-candidate (removed, work) of the step-2 prune (GPU reverse DFS)."""
    c = _u64(cands)
    removed = np.zeros(c.size, dtype=np.uint8)
    work = np.zeros(c.size, dtype=np.uint64)
    ctx = N.context(device)
    rc = N.lib.lc_prune(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3, 0 if mode == "dfs" else 1,
                        int(limit), N.u64p(c), c.size, N.u8p(removed), N.u64p(work))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return removed.astype(bool), work


def random_candidates(spec, params, seed: int, n: int) -> np.ndarray:
    """K0: the first n special nodes of the seeded counter-based trial stream."""
    out = np.empty(n, dtype=np.uint64)
    used = C.c_uint64(0)
    ctx = N.context()
    rc = N.lib.lc_random_candidates(ctx.handle, C.byref(N.spec_struct(spec)), params.fixed_r3,
                                    int(seed) & ((1 << 64) - 1), int(n), N.u64p(out), C.byref(used))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return out


def first_missing(sorted_set, queries) -> int:
    s = _u64(sorted_set)
    q = _u64(queries)
    res = C.c_uint64(0)
    ctx = N.context()
    rc = N.lib.lc_first_missing(ctx.handle, N.u64p(s), s.size, N.u64p(q), q.size, C.byref(res))
    if rc != N.LC_OK:
        _raise(N.NativeError(rc, N.last_error()))
    return int(res.value)
