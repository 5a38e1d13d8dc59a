"""Sampling statistics of §6 of the paper.

The reference package declares this module (``lfsrcycles/__init__.py:26``) but does not
ship it; its contract is SPEC.md:361-428.  Everything heavy runs on the GPU: segment
distances are two-hop chain walks (the walk kernel with ``legs=2``), segment shapes are
batched reverse level sweeps (``probe_segments``: one GPU predecessor + predicate pass per
level for all sampled segments at once).

* ``random_mapping_expectations(n)`` -- Flajolet-Odlyzko random-mapping expectations
  (the paper's Table "Comparison of the expected values").
* ``sample_segment_distances`` -- distance between consecutive candidates from seeded
  uniform random states (first hop discarded), mean / sd / histogram.
* ``sample_segment_shapes`` -- depth CDF and nodes-per-level curve of sampled segments.
* ``deviation_report`` -- log10(observed / expected) per property, like the paper's table.
"""

from __future__ import annotations

import math
import random
from dataclasses import dataclass, field

import numpy as np

from . import _batch
from .cipher import CandidateParams, CipherSpec, unrank_state
from .pipeline import probe_segments, random_candidate

__all__ = ["ExpectationTable", "SampleStats", "AnalysisReport", "random_mapping_expectations",
           "sample_segment_distances", "sample_segment_shapes", "deviation_report"]


@dataclass(frozen=True)
class ExpectationTable:
    """Random-mapping expectations for n nodes."""

    n: int
    components: float
    largest_cycle: float
    largest_component: float
    max_segment_depth: float
    leaf_fraction: float
    cycle_nodes: float
    nodes_per_level: float


@dataclass
class SampleStats:
    sample_size: int
    seed: int
    distance_mean: float | None = None
    distance_std: float | None = None
    distance_histogram: dict = field(default_factory=dict)
    depth_cdf: list = field(default_factory=list)          # (quantile, depth)
    nodes_per_level: list = field(default_factory=list)    # unconditioned mean nodes at each depth
    nodes_per_level_conditioned: list = field(default_factory=list)  # over segments reaching the depth
    censored: int = 0


@dataclass
class AnalysisReport:
    """Observed whole-graph properties (from the pipeline's outputs or the oracle)."""

    n: int
    components: float | None = None
    largest_cycle: float | None = None
    largest_component: float | None = None
    max_segment_depth: float | None = None
    leaf_fraction: float | None = None
    cycle_nodes: float | None = None
    nodes_per_level: float | None = None


def random_mapping_expectations(n: int) -> ExpectationTable:
    """[Flajolet1990] expectations (natural logarithm)."""
    if n < 2:
        raise ValueError("n must be >= 2")
    return ExpectationTable(n=n, components=0.5 * math.log(n), largest_cycle=0.78248 * math.sqrt(n),
                            largest_component=0.75782 * n, max_segment_depth=0.6 * math.sqrt(n),
                            leaf_fraction=math.exp(-1.0), cycle_nodes=math.sqrt(math.pi * n / 2.0),
                            nodes_per_level=1.0)


def sample_segment_distances(spec: CipherSpec, params: CandidateParams, sample_size: int, seed: int, *,
                             states=None) -> SampleStats:
    """Seeded uniform valid states (mixed-radix unranking, rejection free), each walked two
    candidate hops on the GPU; the second hop is a candidate-to-candidate distance
    (SPEC.md:376-386).  ``states`` overrides the sampler (e.g. the whole population)."""
    if states is None:
        if sample_size < 2:
            raise ValueError("sample_size must be >= 2")
        rng = random.Random(seed)
        total = spec.valid_state_count
        states = [unrank_state(rng.randrange(total), spec) for _ in range(sample_size)]
    res = _batch.walk(states, params, spec, stride=1, legs=2)
    d = res.dist[:, 1].astype(np.float64)
    vals, counts = np.unique(res.dist[:, 1], return_counts=True)
    return SampleStats(sample_size=len(states), seed=seed, distance_mean=float(d.mean()),
                       distance_std=float(d.std()),
                       distance_histogram={int(v): int(c) for v, c in zip(vals, counts)})


def sample_segment_shapes(spec: CipherSpec, params: CandidateParams, sample_size: int, seed: int, *,
                          depth_cap: int | None = None, node_cap: int | None = None, roots=None,
                          quantiles=(0.5, 0.9, 0.99, 0.999)) -> SampleStats:
    """Reverse-traverse seeded random candidates' segments (GPU level sweeps, one pass per
    level for all samples) -> depth CDF and nodes-per-level curves.
    Capped sweeps count as censored observations."""
    if roots is None:
        if sample_size < 2:
            raise ValueError("sample_size must be >= 2")
        rng = random.Random(seed)
        roots = [random_candidate(rng, spec, params) for _ in range(sample_size)]
    levels: list = []
    depth, nodes, censored = probe_segments(roots, spec, params, depth_cap=depth_cap, node_cap=node_cap,
                                            level_counts=levels)
    k = len(roots)
    srt = np.sort(depth)
    cdf = [(q, int(srt[min(k - 1, int(math.ceil(q * k)) - 1)])) for q in quantiles]
    reach = np.array([(depth >= lv).sum() for lv in range(len(levels))], dtype=np.float64)
    uncond = [c / k for c in levels]
    cond = [c / r if r else 0.0 for c, r in zip(levels, reach)]
    return SampleStats(sample_size=k, seed=seed, depth_cdf=cdf, nodes_per_level=uncond,
                       nodes_per_level_conditioned=cond, censored=int(censored.sum()))


def deviation_report(observed: AnalysisReport, expected: ExpectationTable) -> list:
    """Rows (property, observed, expected, log10(observed / expected)) -- the paper's
    'deviation' column."""
    if observed.n != expected.n:
        raise ValueError("observed and expected node counts differ")
    rows = []
    for name in ("components", "largest_cycle", "largest_component", "max_segment_depth", "leaf_fraction",
                 "cycle_nodes", "nodes_per_level"):
        o, e = getattr(observed, name), getattr(expected, name)
        if o is None:
            continue
        rows.append((name, o, e, math.log10(o / e) if o > 0 and e > 0 else float("nan")))
    return rows
