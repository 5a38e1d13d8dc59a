"""The multi-rank bench path with the kernel walking: two ranks share
cuda:0 over gloo (LFSR_BENCH_SHARE_GPU=1 -- this run has one GPU; NCCL replaces gloo on
a multi-GPU node and nothing else changes), each walks its own seeded reference-sampler
stream, and the statistics block is all-reduced.  The global statistics in rank 0's JSON
line must equal a single-process walk over the concatenated shards, and per-rank setup
must not grow with the rank (every rank generates only its own stream)."""

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


def test_two_rank_bench_equals_concatenated_walk(gpu, lc, specs, params):
    from paper_1210_6411_b200 import pipeline as P

    log2 = 15
    env = dict(os.environ, LFSR_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--workload-log2", str(log2), "--batch-log2", str(log2 - 1),
           "--no-e2e", "--no-cpu", "--no-steps12"]
    out = subprocess.run(cmd, env=env, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = json.loads([ln for ln in out.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["gpu_launches"] > 0
    # the same shards walked in one process: rank r's stream is seed r
    starts = np.concatenate([P.reference_candidates(specs["a51"], params["a51"], r, 1 << log2) for r in range(2)])
    res = lc.walk_arrays(starts, params["a51"], specs["a51"], stride=STRIDE)
    d = res.dist[:, 0].astype(np.int64)
    ws = line["walk_stats"]
    assert ws["edges"] == d.size and ws["transitions"] == int(d.sum())
    assert ws["min"] == int(d.min()) and ws["max"] == int(d.max())
    assert abs(ws["mean"] - d.mean()) < 1e-6 and abs(ws["sd"] - d.astype(np.float64).std()) < 1e-3
    assert line["parity"]["walks_hashed"] == 1 << log2
