"""Step 3, the chain walk: drop-in for ``lfsrcycles.bitslice`` (reference
``pkg/src/lfsrcycles/bitslice.py``), running on the B200 walk kernel (csrc/walk.cu).

``forward_to_candidate`` / ``candidate_hops`` keep the reference signatures and results
(bit-exact edges; ``width`` is accepted and has no effect on the results -- the GPU
packs 32 lanes per thread and 1024 per warp).  ``transpose`` / ``untranspose`` /
``SlicedBatch`` keep the reference's host data format for callers that use it;
``clock_sliced`` runs on the GPU.
"""

from __future__ import annotations

import random
from dataclasses import dataclass

import numpy as np

from . import _batch
from ._batch import StrideError, UnsupportedSpecError, WalkResult, default_max_clocks  # noqa: F401
from .cipher import (CandidateParams, CipherSpec, PredecessorTable, clock_forward,  # noqa: F401  (re-exported
                     minimum_cycle_length, predecessors, shared_table, unrank_state)  # as the reference's module does)

__all__ = [
    "SlicedBatch", "transpose", "untranspose", "clock_sliced", "forward_to_candidate",
    "candidate_hops", "calibrate_stride", "DEFAULT_STRIDE_A51", "StrideError",
    "walk_arrays",
]

#: Bulk-clock count used by the paper and the reference for the stock A5/1 fixed R3
#: (bitslice.py:43): the first candidate at clock >= this is reported.
DEFAULT_STRIDE_A51 = 11_170_000

#: Register values of unoccupied lanes in a SlicedBatch (bitslice.py:46).
_FILLER_REGS = (1, 1, 1)


@dataclass
class SlicedBatch:
    """Transposed batch: ``words[i]`` holds bit i of every lane (bitslice.py:53-63)."""

    words: list
    lane_count: int
    width: int

    @property
    def nbits(self) -> int:
        return len(self.words)


def _lanes_to_words(lanes: np.ndarray, nbits: int, width: int) -> list:
    bits = (lanes[:, None] >> np.arange(nbits, dtype=np.uint64)[None, :]) & np.uint64(1)  # [width, nbits]
    packed = np.packbits(bits.astype(np.uint8).T, axis=1, bitorder="little")  # [nbits, width/8]
    return [int.from_bytes(row.tobytes(), "little") for row in packed]


def _words_to_lanes(words: list, nbits: int, width: int) -> np.ndarray:
    nbytes = (width + 7) // 8
    mat = np.frombuffer(b"".join(int(w).to_bytes(nbytes, "little") for w in words), dtype=np.uint8)
    bits = np.unpackbits(mat.reshape(nbits, nbytes), axis=1, bitorder="little")[:, :width]
    return (bits.T.astype(np.uint64) << np.arange(nbits, dtype=np.uint64)[None, :]).sum(axis=1, dtype=np.uint64)


def transpose(states, spec: CipherSpec, width: int = 64) -> SlicedBatch:
    """Slice up to ``width`` states; unoccupied lanes get the filler state (1,1,1)."""
    states = list(states)
    if len(states) > width:
        raise ValueError(f"batch of {len(states)} exceeds lane width {width}")
    lanes = np.full(width, spec.pack(*_FILLER_REGS), dtype=np.uint64)
    if states:
        lanes[: len(states)] = np.asarray(states, dtype=np.uint64)
    return SlicedBatch(_lanes_to_words(lanes, spec.total_bits, width), len(states), width)


def untranspose(batch: SlicedBatch) -> list:
    lanes = _words_to_lanes(batch.words, batch.nbits, batch.width)
    return [int(v) for v in lanes[: batch.lane_count]]


def clock_sliced(batch: SlicedBatch, spec: CipherSpec, t: int) -> SlicedBatch:
    """Every lane (filler lanes included) advanced t clocks -- on the GPU."""
    if t < 0:
        raise ValueError("clock count must be >= 0")
    lanes = _words_to_lanes(batch.words, batch.nbits, batch.width)
    out = _batch.clock(lanes, spec, t)
    return SlicedBatch(_lanes_to_words(out, spec.total_bits, batch.width), batch.lane_count, batch.width)


def walk_arrays(starts, params: CandidateParams, spec: CipherSpec, *, stride: int = 1, legs: int = 1,
                max_clocks: int | None = None, refill: int = 0, histogram=None) -> WalkResult:
    """Array fast path: ``uint64`` starts -> dest/dist arrays ``[n, legs]`` + statistics."""
    return _batch.walk(starts, params, spec, stride=stride, legs=legs, max_clocks=max_clocks,
                       refill=refill, histogram=histogram)


def forward_to_candidate(batch, params: CandidateParams, spec: CipherSpec,
                         table: PredecessorTable | None = None, stride: int = 1, *,
                         width: int | None = None, max_clocks: int | None = None) -> list:
    """First candidate at clock >= max(stride, 1) from each state, with its distance
    (bitslice.py:326-342).  Raises StrideError when a walk passes the clock cap."""
    res = _batch.walk(batch, params, spec, stride=stride, legs=1, max_clocks=max_clocks)
    return list(zip(res.dst[:, 0].tolist(), res.dist[:, 0].tolist()))


def candidate_hops(starts, params: CandidateParams, spec: CipherSpec,
                   table: PredecessorTable | None = None, *, legs: int = 2,
                   width: int | None = None, max_clocks: int | None = None) -> list:
    """Per start, ``legs`` consecutive (candidate, distance) hops (bitslice.py:345-354)."""
    res = _batch.walk(starts, params, spec, stride=1, legs=legs, max_clocks=max_clocks)
    d, w = res.dst.tolist(), res.dist.tolist()
    return [list(zip(dr, wr)) for dr, wr in zip(d, w)]


def calibrate_stride(spec: CipherSpec, params: CandidateParams, table: PredecessorTable | None = None, *,
                     samples: int = 10_000, seed: int = 0, margin: float = 0.01) -> int:
    """Sampled bulk stride (bitslice.py:357-376): the stock A5/1 constant, otherwise the
    shortest second-leg hop over seeded random starts, less ``margin``.  Like the
    reference this is a sampled bound; the GPU walk itself never needs a stride (it
    skips the provably candidate-free window instead)."""
    if (spec.name, params.fixed_r3) == ("a51", 0x2AAA00):
        return DEFAULT_STRIDE_A51
    rng = random.Random(seed)
    total = spec.valid_state_count
    starts = [unrank_state(rng.randrange(total), spec) for _ in range(samples)]
    res = _batch.walk(starts, params, spec, stride=1, legs=2)
    shortest = int(res.dist[:, 1].min())
    return max(1, int(shortest * (1.0 - margin)))
