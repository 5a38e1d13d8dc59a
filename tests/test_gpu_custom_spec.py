"""Custom cipher specs (cipher.py:153-170, CipherSpec.from_json): the same kernels,
compiled for the spec at first use (csrc/jit.cu, NVRTC), against the C restatement of
the reference on every hot-path operation -- the walk (one and several legs, strides,
the cap), the special-node predicate, predecessors, the stepper, the step-1 enumeration
and the step-2 prune.  One spec has a maximal-period R3; the other's R3 is a rotation
(period 7 through F, so walks from states off F's cycle must end in StrideError)."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ODD = ("odd", (5, 7, 7), ((1, 4), (5, 6), (5, 6)), (2, 2, 3))
ROT = ("rot", (6, 7, 7), ((2, 5), (3, 6), (6,)), (2, 3, 3))
MANY = ("many_taps", (7, 8, 9), ((1, 2, 3, 4, 6), (0, 3, 4, 5, 6, 7), (3, 8)), (3, 3, 4))  # 5- and 6-tap folds


def _spec(lc, d):
    return lc.CipherSpec.from_json(lc.CipherSpec(*d).to_json())


def _random_valid(spec, n, seed):
    rng = np.random.default_rng(seed)
    regs = [rng.integers(1, m + 1, size=n, dtype=np.uint64) for m in spec.reg_masks]
    return regs[0] | (regs[1] << np.uint64(spec.offsets[1])) | (regs[2] << np.uint64(spec.offsets[2]))


@pytest.mark.parametrize("d", [ODD, ROT, MANY], ids=lambda d: d[0])
def test_custom_spec_matches_restatement(gpu, lc, d):
    from oracle import port
    from paper_1210_6411_b200 import _batch

    spec = _spec(lc, d)
    F = lc.default_fixed_r3(spec)
    p = lc.CandidateParams.from_spec(spec, F)
    # step 1: every candidate of the plane, ascending
    cands = lc.enumerate_candidates_array(spec, p)
    want = port.enumerate_rows(spec, F, 1, spec.reg_masks[1] + 1)
    assert cands.size > 0 and (cands == want).all()
    # predicate, predecessors, stepper on random valid states
    xs = _random_valid(spec, 4000, 1)
    assert lc.is_candidate(xs, p, spec).tolist() == [port.is_candidate(spec, F, int(x)) for x in xs]
    out, cnt = _batch.predecessors(xs[:500], spec)
    for i, x in enumerate(xs[:500]):
        assert sorted(out[i, :cnt[i]].tolist()) == sorted(port.predecessors(spec, int(x)))
    assert (_batch.clock(xs, spec, 37) == port.clock_n(spec, xs, 37)).all()
    # step 3: every candidate to its next special node, one and two legs, two strides
    for stride, legs in ((1, 1), (1, 2), (9, 1)):
        res = lc.walk_arrays(cands, p, spec, stride=stride, legs=legs)
        dst, dist = port.walk(spec, F, cands, stride=stride, legs=legs)
        assert (res.dst == dst).all() and (res.dist == dist).all(), (stride, legs)
    # step 2: the prune, both modes
    for mode, limit in (("dfs", 12), ("dfs", 60), ("bfs", 40)):
        removed, work = _batch.prune(cands, spec, p, mode, limit)
        o_removed, o_work = port.prune(spec, F, mode, limit, cands)
        assert (removed == o_removed).all() and (work == o_work).all(), (mode, limit)


def test_custom_spec_walk_outcomes_from_random_states(gpu, lc):
    from oracle import port

    for d in (ODD, ROT):
        spec = _spec(lc, d)
        F = lc.default_fixed_r3(spec)
        p = lc.CandidateParams.from_spec(spec, F)
        xs = _random_valid(spec, 3000, 2)
        try:
            want = port.walk(spec, F, xs, stride=1, legs=2)
        except port.OracleStrideError:
            want = None
        if want is None:  # some start can never reach F (ROT): both raise StrideError
            with pytest.raises(lc.StrideError):
                lc.walk_arrays(xs, p, spec, stride=1, legs=2)
            # and the starts on F's cycle still walk exactly
            r3 = (xs >> np.uint64(spec.offsets[2])) & np.uint64(spec.reg_masks[2])
            cyc = {F}
            r = F
            while True:
                r = lc.step_register(r, spec.lengths[2], spec.tap_masks[2])
                if r == F:
                    break
                cyc.add(r)
            ok = xs[np.isin(r3, np.array(sorted(cyc), dtype=np.uint64))]
            xs = ok
            want = port.walk(spec, F, xs, stride=1, legs=2)
        res = lc.walk_arrays(xs, p, spec, stride=1, legs=2)
        assert (res.dst == want[0]).all() and (res.dist == want[1]).all(), d[0]
