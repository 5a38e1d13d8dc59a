"""Small launches of every control-flow mode of the walk (K1), the prune (K3), the
enumeration (K2) and the edge sort, run by tests/test_gpu_checked.py against the checked
library build (-DLC_CHECKS=1: device-side bounds and invariant checks that trap).  Each
mode also checks its results against the C restatement, so a run that finishes is a
correct run.

    LFSR_LIB=.../checked/liblfsr_b200.so python tests/_kernel_modes.py MODE
    MODE: walk_warp | walk_lane | walk_park | walk_park_device | prune | prune_v2 | prune_spill | enumerate | sort
"""

from __future__ import annotations

import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def random_valid(spec, n, seed):
    rng = np.random.default_rng(seed)
    regs = [rng.integers(1, m + 1, size=n, dtype=np.uint64) for m in spec.reg_masks]
    return regs[0] | (regs[1] << np.uint64(spec.offsets[1])) | (regs[2] << np.uint64(spec.offsets[2]))


def main(mode: str) -> None:
    import paper_1210_6411_b200 as lc
    from oracle import port

    m567 = lc.CandidateParams.from_spec(lc.MINI567, 0x22)
    m789 = lc.CandidateParams.from_spec(lc.MINI789, 0xAA)
    if mode == "walk_warp":  # whole-warp refill: special-node starts, one hop
        cands = lc.enumerate_candidates_array(lc.MINI567, m567)
        res = lc.walk_arrays(cands, m567, lc.MINI567, stride=1, refill=1024)
        d, w = port.walk(lc.MINI567, 0x22, cands, stride=1)
        assert (res.dst == d).all() and (res.dist == w).all()
    elif mode == "walk_lane":  # lane refill, several hops from random states
        s = random_valid(lc.MINI789, 5000, 1)
        res = lc.walk_arrays(s, m789, lc.MINI789, stride=1, legs=3, refill=1)
        d, w = port.walk(lc.MINI789, 0xAA, s, stride=1, legs=3)
        assert (res.dst == d).all() and (res.dist == w).all()
    elif mode in ("walk_park", "walk_park_device"):  # above the parking threshold
        import torch

        from paper_1210_6411_b200 import _native as N

        ctx = N.context()
        n = 4 * ctx.sm_count * 1024 + 4096
        s = random_valid(lc.MINI567, n, 2)
        want = lc.walk_arrays(s, m567, lc.MINI567, stride=1, legs=2)
        ref_d, ref_w = port.walk(lc.MINI567, 0x22, s[:20000], stride=1, legs=2)
        assert (want.dst[:20000] == ref_d).all() and (want.dist[:20000] == ref_w).all()
        if mode == "walk_park_device":
            dev = torch.device("cuda", ctx.device)
            st = torch.cuda.Stream(dev)
            ts = torch.from_numpy(s.view(np.int64)).to(dev)
            dst = torch.empty(2 * n, dtype=torch.int64, device=dev)
            dist = torch.empty(2 * n, dtype=torch.int64, device=dev)
            stats = torch.zeros(N.ST_HEADER + 2, dtype=torch.int64, device=dev)
            torch.cuda.synchronize()
            N.check(N.lib.lc_walk_device(ctx.handle, C.byref(N.spec_struct(lc.MINI567)), 0x22,
                                         C.c_void_p(ts.data_ptr()), n, 1, 16 * 169 + 64, 2, 0,
                                         C.c_void_p(dst.data_ptr()), C.c_void_p(dist.data_ptr()), 0, 0, 0,
                                         C.c_void_p(stats.data_ptr()), C.c_void_p(st.cuda_stream)))
            torch.cuda.synchronize()
            assert (dst.cpu().numpy().view(np.uint64) == want.dst.reshape(-1)).all()
    elif mode in ("prune", "prune_v2", "prune_spill"):  # K3, dfs and bfs; prune_spill: tiny ring spill
        cands = lc.enumerate_candidates_array(lc.MINI789, m789)
        for how, limit in (("dfs", 40), ("dfs", 400), ("bfs", 300)):
            rem, work = _prune(lc, cands, how, limit, m789)
            o_rem, o_work = port.prune(lc.MINI789, 0xAA, how, limit, cands)
            assert (rem == o_rem).all() and (work == o_work).all(), (how, limit)
        a51 = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
        c = lc.enumerate_candidates_array(lc.A51, a51, r2_lo=0x2AAA, r2_hi=0x2AAA + 1)[:2048]
        rem, work = _prune(lc, c, "dfs", 3000, a51, spec=lc.A51)
        o_rem, o_work = port.prune(lc.A51, 0x2AAA00, "dfs", 3000, c)
        assert (rem == o_rem).all() and (work == o_work).all()
    elif mode == "sort":
        rng = np.random.default_rng(4)
        for n, dups in ((4097, True), (300_000, True), (300_000, False)):
            src = rng.integers(0, 1 << 63, size=n, dtype=np.uint64)
            if dups:  # duplicates: the sort must be stable (and at 300k one group outgrows
                src[::7] = src[0]  # the MSD route's shared-memory sort: the LSD fallback)
            dst = np.arange(n, dtype=np.uint64)
            s, d, _ = lc.sort_edge_arrays(src, dst, dst.copy())
            order = np.argsort(src, kind="stable")
            assert (s == src[order]).all() and (d == dst[order]).all()
    elif mode == "enumerate":
        a51 = lc.CandidateParams.from_spec(lc.A51, 0x2AAA00)
        got = lc.enumerate_candidates_array(lc.A51, a51, r2_lo=0x2AAA, r2_hi=0x2AAA + 2)
        assert (got == port.enumerate_rows(lc.A51, 0x2AAA00, 0x2AAA, 0x2AAA + 2)).all()
    else:
        raise SystemExit(f"unknown mode {mode}")
    print(f"{mode}: ok")


def _prune(lc, cands, how, limit, params, spec=None):
    from paper_1210_6411_b200 import _native as N

    spec = spec or lc.MINI789
    cands = np.ascontiguousarray(cands, dtype=np.uint64)
    rem = np.zeros(cands.size, dtype=np.uint8)
    work = np.zeros(cands.size, dtype=np.uint64)
    N.check(N.lib.lc_prune(N.context().handle, C.byref(N.spec_struct(spec)), params.fixed_r3, 0 if how == "dfs" else 1,
                           limit, N.u64p(cands), cands.size, N.u8p(rem), N.u64p(work)))
    return rem, work


if __name__ == "__main__":
    main(sys.argv[1])
