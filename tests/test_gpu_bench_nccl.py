"""The NCCL data plane of the bench: the statistics all-reduce and the
max-over-ranks timing go through a real NCCL communicator.  This box has one GPU, so the
communicator has one rank (LFSR_BENCH_NCCL=1 under torchrun); on a multi-GPU node the
same calls run with N ranks.  The all-reduced statistics must equal a plain walk of the
same stream, and NCCL must report the communicator (NCCL_DEBUG=INFO)."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

STRIDE = 11_170_000


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_one_rank_nccl_bench(gpu, lc, specs, params):
    from paper_1210_6411_b200 import pipeline as P

    log2 = 15
    env = dict(os.environ, LFSR_BENCH_NCCL="1", NCCL_DEBUG="INFO")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "1", "--steps", "2", "--warmup", "3", "--workload-log2", str(log2), "--batch-log2", str(log2 - 1),
           "--no-cpu", "--no-steps12", "--no-next"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["nccl"] and line["nccl"]["backend"] == "nccl" and line["nccl"]["world_size"] == 1
    assert "NCCL communicator: 1 ranks" in out.stderr
    assert "NCCL INFO" in out.stderr + out.stdout  # the library itself reported in
    starts = P.reference_candidates(specs["a51"], params["a51"], 0, 1 << log2)
    res = lc.walk_arrays(starts, params["a51"], specs["a51"], stride=STRIDE)
    d = res.dist[:, 0].astype(np.int64)
    ws = line["walk_stats"]
    assert ws["edges"] == d.size and ws["transitions"] == int(d.sum())
    assert ws["min"] == int(d.min()) and ws["max"] == int(d.max())
    assert line["e2e"]["dst_equal_to_device_path"] is True
