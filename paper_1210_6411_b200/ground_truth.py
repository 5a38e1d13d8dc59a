"""Exhaustive ground truth for desk-scale cipher instances, on the GPU: drop-in for the
reference's ``lfsrcycles.oracle`` (``brute_force_analysis``, ``GroundTruth``,
``CycleInfo``; oracle.py:19-283), SURVEY.md §8(f) rank 4.

The full successor map over the rank-encoded valid states, its in-degrees, the special
nodes, every state's cycle (pointer doubling), the candidate-graph edges, the segment
sweep and the per-cycle order are computed by the kernels in csrc/bruteforce.cu
(``lc_bf_*``); torch tensors hold the arrays in HBM and do the small glue (unique,
bincount, searchsorted).  Results equal the reference's field by field (tests compare
summaries, cycles, histograms and digests of every array with fixtures the reference
produced).  Like the reference, the reverse direction comes from inverting the forward
map, not from the predecessor table, so it is an independent check of steps 1-5.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .cipher import CandidateParams, CipherSpec

__all__ = ["GroundTruth", "CycleInfo", "brute_force_analysis"]

_MAX_NODES = 1 << 31


@dataclass
class CycleInfo:
    """One cycle of the state graph (oracle.py:25-32)."""

    ranks: np.ndarray          # on-cycle states in walk order, from the smallest rank
    leader: int                # minimum packed state on the cycle
    clock_length: int          # number of states on the cycle
    candidate_count: int       # candidates among them
    component_size: int        # states in the surrounding component


@dataclass
class GroundTruth:
    """oracle.py:35-101."""

    spec: CipherSpec
    params: CandidateParams
    node_count: int
    succ: np.ndarray
    pred_count_hist: np.ndarray
    leaf_count: int
    cycles: list
    cand_ranks: np.ndarray
    edge_src: np.ndarray
    edge_dst: np.ndarray
    edge_dist: np.ndarray
    seg_depth: np.ndarray
    seg_size: np.ndarray
    level_counts: np.ndarray
    _packed_cache: dict = field(default_factory=dict, repr=False)

    def packed_of_ranks(self, ranks) -> np.ndarray:
        m1, m2, m3 = self.spec.reg_masks
        _, o2, o3 = self.spec.offsets
        r = np.asarray(ranks, dtype=np.int64)
        r3 = r % m3 + 1
        r2 = (r // m3) % m2 + 1
        r1 = r // m3 // m2 + 1
        return (r1 | (r2 << o2) | (r3 << o3)).astype(np.uint64)

    @property
    def component_count(self) -> int:
        return len(self.cycles)

    @property
    def on_cycle_states(self) -> int:
        return sum(c.clock_length for c in self.cycles)

    def cycle_multiset(self) -> list:
        """Sorted (candidate hop count, clock length) per cycle."""
        return sorted((c.candidate_count, c.clock_length) for c in self.cycles)

    def candidate_edge_map(self) -> dict:
        """Packed source -> (packed destination, distance)."""
        src, dst = self.packed_of_ranks(self.edge_src), self.packed_of_ranks(self.edge_dst)
        return {int(s): (int(d), int(w)) for s, d, w in zip(src, dst, self.edge_dist)}

    def summary(self) -> dict:
        sizes = sorted(c.clock_length for c in self.cycles)
        return {
            "node_count": self.node_count,
            "leaf_count": self.leaf_count,
            "leaf_fraction": self.leaf_count / self.node_count,
            "component_count": self.component_count,
            "cycle_count": len(self.cycles),
            "on_cycle_states": self.on_cycle_states,
            "largest_cycle": sizes[-1] if sizes else 0,
            "largest_component": max((c.component_size for c in self.cycles), default=0),
            "candidate_count": int(self.cand_ranks.size),
            "max_segment_depth": int(self.seg_depth.max(initial=0)),
            "mean_segment_depth": float(self.seg_depth.mean()) if self.seg_depth.size else math.nan,
        }


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t.numel() else None


def brute_force_analysis(spec: CipherSpec, params: CandidateParams, *, clock_all: bool = False,
                         device: int | None = None) -> GroundTruth:
    """Full functional-graph analysis of one instance (oracle.py:141-283).  clock_all
    replaces the majority rule with "advance all three registers" (a bijection)."""
    import torch

    n = spec.valid_state_count
    if n > _MAX_NODES:
        raise ValueError(f"instance too large for exhaustive analysis ({n} > {_MAX_NODES} states)")
    ctx = N.context(device)
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    sspec = N.spec_struct(spec)
    i64 = dict(dtype=torch.int64, device=dev)

    succ = torch.empty(n, **i64)
    indeg = torch.empty(n, dtype=torch.int32, device=dev)
    is_cand = torch.empty(n, dtype=torch.uint8, device=dev)
    g = torch.empty(n, **i64)
    N.check(N.lib.lc_bf_build_device(ctx.handle, C.byref(sspec), params.fixed_r3, int(bool(clock_all)), n,
                                     _ptr(succ), _ptr(indeg), _ptr(is_cand), _ptr(g), stream))
    cand = torch.empty(n, **i64)
    mh = C.c_uint64(0)
    N.check(N.lib.lc_bf_candidates_device(ctx.handle, n, _ptr(is_cand), _ptr(cand), C.byref(mh), stream))
    m = int(mh.value)
    cand = cand[:m]  # ascending ranks

    # candidate-graph edges
    edge_dst, edge_dist = torch.empty(m, **i64), torch.empty(m, **i64)
    N.check(N.lib.lc_bf_edges_device(ctx.handle, n, _ptr(succ), _ptr(is_cand), _ptr(cand), m, _ptr(edge_dst),
                                     _ptr(edge_dist), stream))

    # segment sweep
    root, depth = torch.empty(n, **i64), torch.empty(n, dtype=torch.int32, device=dev)
    cap = 1 << 20
    levels = np.zeros(cap, dtype=np.uint64)
    nlev = C.c_uint32(0)
    N.check(N.lib.lc_bf_segments_device(ctx.handle, n, _ptr(succ), _ptr(indeg), _ptr(is_cand), _ptr(cand), m,
                                        _ptr(root), _ptr(depth), N.u64p(levels), cap, C.byref(nlev), stream))
    pred_hist = torch.empty(5, **i64)
    seg_depth, seg_size = torch.empty(m, **i64), torch.empty(m, **i64)
    N.check(N.lib.lc_bf_summary_device(ctx.handle, n, _ptr(indeg), _ptr(root), _ptr(depth), m, _ptr(pred_hist),
                                       _ptr(seg_depth), _ptr(seg_size), stream))
    if not clock_all and int(seg_size.sum().item()) != n:
        raise AssertionError("segment sweep missed states; graph is inconsistent")

    # cycles (on-cycle states = the image of f^(2^k)), each ordered from its smallest rank
    # in walk order, with leader, candidates on it and component size
    bufs = [torch.empty(n, **i64) for _ in range(6)]
    order, offset, length, leader, cand_on, comp_sizes = bufs
    n_on, n_cyc = C.c_uint64(0), C.c_uint64(0)
    N.check(N.lib.lc_bf_cycles_device(ctx.handle, C.byref(sspec), n, _ptr(succ), _ptr(g), _ptr(is_cand),
                                      *[_ptr(t) for t in bufs], C.byref(n_on), C.byref(n_cyc), stream))
    k_cyc = int(n_cyc.value)
    order = order[: int(n_on.value)]
    offset, length, leader, cand_on, comp_sizes = (t[:k_cyc] for t in (offset, length, leader, cand_on, comp_sizes))

    h = lambda t: t.cpu().numpy()  # noqa: E731
    order_h, length_h, offset_h = h(order), h(length), h(offset)
    leader_h, cand_on_h, comp_h = h(leader), h(cand_on), h(comp_sizes)
    cand_h = h(cand)
    cycles = [CycleInfo(ranks=order_h[offset_h[k]:offset_h[k] + length_h[k]], leader=int(leader_h[k]),
                        clock_length=int(length_h[k]), candidate_count=int(cand_on_h[k]),
                        component_size=int(comp_h[k])) for k in range(k_cyc)]
    return GroundTruth(spec=spec, params=params, node_count=n, succ=h(succ), pred_count_hist=h(pred_hist),
                       leaf_count=int(pred_hist[0]), cycles=cycles, cand_ranks=cand_h, edge_src=cand_h,
                       edge_dst=h(edge_dst), edge_dist=h(edge_dist), seg_depth=h(seg_depth), seg_size=h(seg_size),
                       level_counts=levels[: int(nlev.value)].astype(np.int64))
