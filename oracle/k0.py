"""TEST INFRASTRUCTURE ONLY -- numpy restatement of the K0 seeded start-set generator.

K0 (csrc/kernels.cu RandGen) is this repo's own synthetic-input generator (the reference
samples with Python's ``random.Random``, pipeline.py:301-310, which cannot run on a
GPU).  Trial i: h = splitmix64(seed + (i + 1) * 0x9E3779B97F4A7C15);
r1 = 1 + (lo32(h) * m1 >> 32), r2 = 1 + (hi32(h) * m2 >> 32), R3 = fixed; the state is
kept iff it is a special node (checked here with the C oracle's is_candidate).
"""

from __future__ import annotations

import numpy as np

from . import port

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def trials(spec, fixed_r3: int, seed: int, lo: int, hi: int) -> np.ndarray:
    i = np.arange(lo, hi, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = splitmix64(np.uint64(seed) + (i + np.uint64(1)) * _GOLDEN)
    m1, m2 = (1 << spec.lengths[0]) - 1, (1 << spec.lengths[1]) - 1
    r1 = np.uint64(1) + (((h & np.uint64(0xFFFFFFFF)) * np.uint64(m1)) >> np.uint64(32))
    r2 = np.uint64(1) + (((h >> np.uint64(32)) * np.uint64(m2)) >> np.uint64(32))
    return r1 | (r2 << np.uint64(spec.lengths[0])) | np.uint64(fixed_r3 << (spec.lengths[0] + spec.lengths[1]))


def random_candidates(spec, fixed_r3: int, seed: int, n: int) -> np.ndarray:
    out, lo = [], 0
    got = 0
    while got < n:
        xs = trials(spec, fixed_r3, seed, lo, lo + max(4096, 3 * (n - got)))
        keep = np.array([port.is_candidate(spec, fixed_r3, int(x)) for x in xs], dtype=bool)
        out.append(xs[keep])
        got += int(keep.sum())
        lo += xs.size
    return np.concatenate(out)[:n]
