"""Asynchronous calls on one context from different streams: the
context serialises its users on the device, so two lc_walk_device calls queued back to
back on two streams -- each needing the context's lane-parking pools and queues -- give
exactly the results of two sequential calls."""

from __future__ import annotations

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_two_streams_share_one_context():
    import torch

    import paper_1210_6411_b200 as lc
    from paper_1210_6411_b200 import _native as N

    spec = lc.MINI789
    params = lc.CandidateParams.from_spec(spec, 0xAA)
    ctx = N.context()
    sspec = N.spec_struct(spec)
    dev = torch.device("cuda", ctx.device)
    rng = np.random.default_rng(5)
    n = 1 << 21  # above the parking threshold: the queued resume rounds use the pools
    regs = [rng.integers(1, m + 1, size=n, dtype=np.uint64) for m in spec.reg_masks]
    host = regs[0] | (regs[1] << np.uint64(spec.offsets[1])) | (regs[2] << np.uint64(spec.offsets[2]))
    words = N.ST_HEADER + 2
    cap = 16 * int(lc.minimum_cycle_length(spec)) + 64

    def launch(starts, dst, dist, stats, stream):
        N.check(N.lib.lc_walk_device(ctx.handle, C.byref(sspec), params.fixed_r3, C.c_void_p(starts.data_ptr()),
                                     starts.numel(), 1, cap, 2, 0, C.c_void_p(dst.data_ptr()),
                                     C.c_void_p(dist.data_ptr()), 0, 0, 0, C.c_void_p(stats.data_ptr()),
                                     C.c_void_p(stream.cuda_stream)))

    sets = [torch.from_numpy(host.view(np.int64)).to(dev), torch.from_numpy(host[::-1].copy().view(np.int64)).to(dev)]
    outs = [[torch.empty(2 * n, dtype=torch.int64, device=dev) for _ in range(2)] for _ in range(2)]
    stats = [torch.zeros(words, dtype=torch.int64, device=dev) for _ in range(2)]
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    for k in range(2):  # no host synchronisation between the two calls
        launch(sets[k], outs[k][0], outs[k][1], stats[k], streams[k])
    torch.cuda.synchronize()
    for k in range(2):
        ref = lc.walk_arrays(sets[k].cpu().numpy().view(np.uint64), params, spec, stride=1, legs=2)
        assert (outs[k][0].cpu().numpy().view(np.uint64) == ref.dst.reshape(-1)).all()
        assert (outs[k][1].cpu().numpy().view(np.uint64) == ref.dist.reshape(-1)).all()
        assert int(stats[k][N.ST_EDGES].item()) == 2 * n and int(stats[k][N.ST_ERROR].item()) == 0
