"""TEST INFRASTRUCTURE ONLY -- numpy restatement of steps 4-5 of the reference.

``cut_leaves`` restates one or more passes of reduce.cut_leaves_pass (reduce.py:118-186):
a record whose source is no record's destination is a leaf; leaves are dropped and fold
(subtree_size + 1, subtree_depth + 1) into their destination (sizes add, depths max);
survivors keep source order.  ``count_cycles`` restates reduce.count_cycles
(reduce.py:226-266).  Pinned against tests/golden/reduce.json (tests/test_oracle.py).
"""

from __future__ import annotations

import numpy as np


def cut_leaves(src, dst, dist, size, depth, max_passes: int = 0):
    src, dst, dist = (np.asarray(a, dtype=np.uint64).copy() for a in (src, dst, dist))
    size, depth = (np.asarray(a, dtype=np.uint64).copy() for a in (size, depth))
    if np.any(src[1:] <= src[:-1]):
        raise ValueError("sources must be strictly ascending")
    passes = []
    while True:
        n = src.size
        pos = np.searchsorted(src, dst)
        found = (pos < n) & (src[np.minimum(pos, n - 1)] == dst) if n else np.zeros(0, bool)
        has_pred = np.zeros(n, dtype=bool)
        has_pred[pos[found]] = True
        leaf = ~has_pred
        if np.any(leaf & ~found):
            raise ValueError("aggregate has no surviving record; input was not closed")
        tgt = pos[leaf]
        np.add.at(size, tgt, size[leaf] + np.uint64(1))
        np.maximum.at(depth, tgt, depth[leaf] + np.uint64(1))
        keep = has_pred
        src, dst, dist, size, depth = src[keep], dst[keep], dist[keep], size[keep], depth[keep]
        passes.append((int(leaf.sum()), int(keep.sum()), int(size.sum(dtype=np.uint64))))
        if leaf.sum() == 0 or (max_passes and len(passes) >= max_passes):
            break
    return src, dst, dist, size, depth, passes


def count_cycles(src, dst, dist, size):
    order = np.argsort(src, kind="stable")
    src, dst, dist, size = (np.asarray(a, dtype=np.uint64)[order] for a in (src, dst, dist, size))
    n = src.size
    if np.any(src[1:] == src[:-1]):
        raise ValueError("duplicate source")
    pos = np.searchsorted(src, dst)
    if np.any(pos >= n) or np.any(src[np.minimum(pos, n - 1)] != dst):
        raise ValueError("destination is not a source")
    if np.any(np.bincount(pos, minlength=n) != 1):
        raise ValueError("not a permutation")
    seen = np.zeros(n, dtype=bool)
    out = []
    for s in range(n):
        if seen[s]:
            continue
        cur, hops, clocks, tree, lead = s, 0, 0, 0, s
        while not seen[cur]:
            seen[cur] = True
            hops += 1
            clocks += int(dist[cur])
            tree += int(size[cur])
            lead = min(lead, cur)
            cur = int(pos[cur])
        out.append((int(src[lead]), hops, clocks, tree))
    return sorted(out)
