"""ctypes binding of the C ABI in ``include/lfsr_b200.h`` (``_lib/liblfsr_b200.so``).

There is no CPU fallback: if the library is missing the import fails, and if no CUDA
device is visible the first call that needs one raises ``RuntimeError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFSR_LIB") or os.path.join(_HERE, "_lib", "liblfsr_b200.so")  # override: A/B builds

LC_OK = 0
LC_ERR_ARG = -1
LC_ERR_CUDA = -2
LC_ERR_UNSUPPORTED = -3
LC_ERR_CAP = -4
LC_ERR_INVALID_STATE = -5
LC_ERR_OVERFLOW = -6
LC_ERR_UNSORTED = -7
LC_ERR_NOT_CLOSED = -8
LC_ERR_NOT_PERMUTATION = -9

# LC_ST_* (include/lfsr_b200.h)
ST_EDGES, ST_TRANSITIONS, ST_MIN, ST_MAX, ST_SQ_LO, ST_SQ_HI = 0, 1, 2, 3, 4, 5
ST_ERROR, ST_ERROR_INDEX, ST_HIST_LO, ST_HIST_SHIFT, ST_HIST_BINS = 6, 7, 8, 9, 10
ST_HEADER = 16


class lc_spec(C.Structure):
    _fields_ = [("lengths", C.c_int32 * 3), ("tap_masks", C.c_uint64 * 3), ("clock_taps", C.c_int32 * 3)]


class NativeError(RuntimeError):
    def __init__(self, code: int, message: str):
        super().__init__(message)
        self.code = code


_u64p = C.POINTER(C.c_uint64)
_u8p = C.POINTER(C.c_uint8)
_vp = C.c_void_p

_SIGNATURES = {
    "lc_abi_version": ([], C.c_int),
    "lc_last_error": ([], C.c_char_p),
    "lc_device_count": ([C.POINTER(C.c_int)], C.c_int),
    "lc_spec_compile_check": ([C.POINTER(lc_spec)], C.c_int),
    "lc_ctx_create": ([C.c_int, C.POINTER(C.c_void_p)], C.c_int),
    "lc_ctx_destroy": ([_vp], C.c_int),
    "lc_ctx_sm_count": ([_vp, C.POINTER(C.c_int)], C.c_int),
    "lc_ctx_synchronize": ([_vp], C.c_int),
    "lc_lop3_peak": ([_vp, C.POINTER(C.c_double), C.POINTER(C.c_double)], C.c_int),
    "lc_host_alloc": ([C.c_uint64, C.POINTER(C.c_void_p)], C.c_int),
    "lc_host_free": ([_vp], C.c_int),
    "lc_launch_count": ([], C.c_uint64),
    "lc_launch_count_reset": ([], None),
    "lc_walk": ([_vp, C.POINTER(lc_spec), C.c_uint64, _u64p, C.c_uint64, C.c_uint64, C.c_uint64,
                 C.c_uint32, C.c_uint32, _u64p, _u64p, C.c_uint64, C.c_uint32, C.c_uint32, _u64p], C.c_int),
    "lc_walk_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, _vp, C.c_uint64, C.c_uint64, C.c_uint64,
                        C.c_uint32, C.c_uint32, _vp, _vp, C.c_uint64, C.c_uint32, C.c_uint32, _vp, _vp],
                       C.c_int),
    "lc_clock": ([_vp, C.POINTER(lc_spec), _u64p, C.c_uint64, C.c_uint64, _u64p], C.c_int),
    "lc_is_candidate": ([_vp, C.POINTER(lc_spec), C.c_uint64, _u64p, C.c_uint64, _u8p], C.c_int),
    "lc_predecessors": ([_vp, C.POINTER(lc_spec), _u64p, C.c_uint64, _u64p, _u8p], C.c_int),
    "lc_enumerate": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_uint64, C.c_uint64, _u64p, C.c_uint64,
                      _u64p], C.c_int),
    "lc_enumerate_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_uint64, C.c_uint64, _vp, C.c_uint64,
                             _vp, _vp], C.c_int),
    "lc_prune": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_int32, C.c_uint64, _u64p, C.c_uint64, _u8p,
                  _u64p], C.c_int),
    "lc_prune_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_int32, C.c_uint64, _vp, C.c_uint64, _vp, _vp,
                         _vp], C.c_int),
    "lc_random_candidates": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p],
                             C.c_int),
    "lc_reference_candidates": ([C.POINTER(lc_spec), C.c_uint64, C.c_uint64, C.c_uint64, _u64p, _u64p],
                                C.c_int),
    "lc_reference_candidates_multi": ([C.POINTER(lc_spec), C.c_uint64, _u64p, C.c_uint32, C.c_uint64, _u64p,
                                       C.c_uint32], C.c_int),
    "lc_random_candidates_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_uint64, C.c_uint64, _vp, _vp],
                                    C.c_int),
    "lc_first_missing": ([_vp, _u64p, C.c_uint64, _u64p, C.c_uint64, _u64p], C.c_int),
    "lc_sort_edges": ([_vp, C.c_uint64, _u64p, _u64p, _u64p, _u64p, _u64p], C.c_int),
    "lc_sort_edges_device": ([_vp, C.c_uint64, C.POINTER(_vp), C.POINTER(_vp), _vp], C.c_int),
    "lc_pack_records_device": ([_vp, C.c_uint64, _vp, _vp, _vp, _vp, _vp, _vp, _vp], C.c_int),
    "lc_cut_leaves": ([_vp, C.c_uint64, _u64p, _u64p, _u64p, _u64p, _u64p, C.c_uint32, _u64p, C.c_uint32,
                       C.POINTER(C.c_uint32), _u64p], C.c_int),
    "lc_cut_leaves_device": ([_vp, C.c_uint64, _vp, _vp, _vp, _vp, _vp, C.c_uint32, _u64p, C.c_uint32,
                              C.POINTER(C.c_uint32), _u64p, _vp], C.c_int),
    "lc_cut_shard_create": ([_vp, C.c_uint64, _vp, _vp, _vp, _vp, _vp, C.c_uint32, _u64p, _u64p, _vp,
                             C.POINTER(C.c_void_p), _u64p], C.c_int),
    "lc_cut_shard_emit": ([_vp, C.c_int, _vp, _u64p, _u64p], C.c_int),
    "lc_cut_shard_apply": ([_vp, C.c_int, _vp, C.c_uint64], C.c_int),
    "lc_cut_shard_finish": ([_vp, _u64p], C.c_int),
    "lc_cut_shard_destroy": ([_vp], C.c_int),
    "lc_bf_build_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, C.c_int, C.c_uint64, _vp, _vp, _vp, _vp, _vp],
                           C.c_int),
    "lc_bf_edges_device": ([_vp, C.c_uint64, _vp, _vp, _vp, C.c_uint64, _vp, _vp, _vp], C.c_int),
    "lc_bf_segments_device": ([_vp, C.c_uint64, _vp, _vp, _vp, _vp, C.c_uint64, _vp, _vp, _u64p, C.c_uint32,
                               C.POINTER(C.c_uint32), _vp], C.c_int),
    "lc_bf_cycle_order_device": ([_vp, C.c_uint64, _vp, _vp, _vp, _vp], C.c_int),
    "lc_probe_segments": ([_vp, C.POINTER(lc_spec), C.c_uint64, _u64p, C.c_uint64, C.c_int64, C.c_int64, _u64p, _u64p,
                           C.POINTER(C.c_uint8), _u64p, C.c_uint32], C.c_int),
    "lc_bf_candidates_device": ([_vp, C.c_uint64, _vp, _vp, _u64p, _vp], C.c_int),
    "lc_bf_summary_device": ([_vp, C.c_uint64, _vp, _vp, _vp, C.c_uint64, _vp, _vp, _vp, _vp], C.c_int),
    "lc_bf_cycles_device": ([_vp, C.POINTER(lc_spec), C.c_uint64, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                             _u64p, _u64p, _vp], C.c_int),
    "lc_count_cycles": ([_vp, C.c_uint64, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p, _u64p],
                        C.c_int),
}

EXPORTED = tuple(_SIGNATURES)


def _load() -> C.CDLL:
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"CUDA library {LIB_PATH} is not built; run `python paper_1210_6411_b200/build.py` "
            "(or __graft_entry__.build()).  There is no CPU fallback.")
    lib = C.CDLL(LIB_PATH)
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if lib.lc_abi_version() != 1:
        raise ImportError("liblfsr_b200 ABI version mismatch")
    return lib


lib = _load()


def last_error() -> str:
    msg = lib.lc_last_error()
    return msg.decode() if msg else ""


def check(rc: int) -> None:
    if rc != LC_OK:
        raise NativeError(rc, last_error())


def u64p(a: np.ndarray):
    return a.ctypes.data_as(_u64p)


def u8p(a: np.ndarray):
    return a.ctypes.data_as(_u8p)


def spec_struct(spec) -> lc_spec:
    s = lc_spec()
    for k in range(3):
        s.lengths[k] = int(spec.lengths[k])
        s.tap_masks[k] = int(spec.tap_masks[k])
        s.clock_taps[k] = int(spec.clock_taps[k])
    return s


class Context:
    """One native context per (device, host thread)."""

    def __init__(self, device: int):
        h = C.c_void_p()
        check(lib.lc_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = int(device)
        sms = C.c_int()
        check(lib.lc_ctx_sm_count(h, C.byref(sms)))
        self.sm_count = sms.value

    def __del__(self):
        try:
            if self.handle:
                lib.lc_ctx_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


_tls = threading.local()
_default_device = int(os.environ.get("LFSR_DEVICE", os.environ.get("LOCAL_RANK", "0")))


def set_device(device: int) -> None:
    global _default_device
    _default_device = int(device)


def context(device: int | None = None) -> Context:
    dev = _default_device if device is None else int(device)
    cache = getattr(_tls, "ctx", None)
    if cache is None:
        cache = _tls.ctx = {}
    ctx = cache.get(dev)
    if ctx is None:
        ctx = cache[dev] = Context(dev)
    return ctx


def device_count() -> int:
    n = C.c_int(0)
    rc = lib.lc_device_count(C.byref(n))
    return n.value if rc == LC_OK else 0


def lop3_peak(device: int | None = None) -> tuple:
    """(measured LOP3 results/s, SM MHz during the measurement) of the device."""
    ctx = context(device)
    ops, mhz = C.c_double(), C.c_double()
    check(lib.lc_lop3_peak(ctx.handle, C.byref(ops), C.byref(mhz)))
    return ops.value, mhz.value


def launch_count() -> int:
    return int(lib.lc_launch_count())


def launch_count_reset() -> None:
    lib.lc_launch_count_reset()
