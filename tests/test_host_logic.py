"""CPU tests of host-side bookkeeping: vectorised schedule/plan builders
against the reference-semantics oracle, and the tile planner."""

import numpy as np
import pytest

from oracle import restated as O
from paper_2412_16481_b200 import attention as A
from paper_2412_16481_b200.backbone import split_table
from paper_2412_16481_b200.pooling import TILE_CAP


@pytest.mark.parametrize("nb,W,stride,shift,rounds", [
    (8, 4, 1, 0, 1), (8, 4, 1, 2, 2), (8, 2, 2, 0, 1), (8, 4, 4, 1, 3), (7, 3, 2, 1, 4),
    (296, 2, 1, 1, 2), (40, 2, 1, 1, 2), (13, 5, 3, 4, 6), (1, 1, 1, 0, 1), (1281, 4, 1, 3, 3),
    (100, 7, 5, 6, 3)])
def test_round_members_equals_build_schedule(nb, W, stride, shift, rounds):
    ref = O.build_schedule(nb, W, stride, shift, rounds)
    for t in range(rounds):
        M = A.round_members(nb, W, stride, shift, t)
        got = sorted(tuple(int(b) for b in row if b >= 0) for row in M)
        got = [g for g in got if g]
        exp = sorted(tuple(int(b) for b in sc) for sc in ref[t])
        assert got == exp
        sched = A.build_schedule(nb, W, stride, shift, rounds)
        assert [s.tolist() for s in sched.rounds[t]] == [s.tolist() for s in ref[t]]


def _plan_ref(starts, lens, scopes):
    """Literal per-scope segment merge (the semantics plan_arrays vectorises)."""
    out = []
    for sc in scopes:
        segs, v, last = [], 0, None
        for b in sc:
            a, ln = int(starts[b]), int(lens[b])
            if ln <= 0:
                continue
            if last is not None and a == last:
                segs[-1][2] += ln
            else:
                segs.append([a, v, ln])
            last = a + ln
            v += ln
        out.append((segs, v))
    return out


@pytest.mark.parametrize("seed", range(6))
def test_plan_arrays_matches_literal_merge(seed):
    r = np.random.default_rng(seed)
    K, S = int(r.integers(2, 300)), 64
    counts = r.integers(0, S + 1, size=K + 1)
    counts[K] = int(r.integers(0, 500))
    base = O.exclusive_scan(counts)
    starts, lens = split_table(counts, base, K, S)
    np.testing.assert_array_equal(starts, O.bucket_table(counts, base, K, S)[0])
    np.testing.assert_array_equal(lens, O.bucket_table(counts, base, K, S)[1])
    nb = len(starts)
    W = int(r.integers(1, min(6, nb) + 1))
    stride = int(r.integers(1, 4))
    M = A.round_members(nb, W, stride, int(r.integers(0, W)), 1)
    P = A.plan_arrays(starts, lens, M)
    ref = _plan_ref(starts, lens, [row[row >= 0] for row in M])
    for s, (segs, m) in enumerate(ref):
        assert P["scope_len"][s] == m
        a, b = P["scope_seg"][s], P["scope_seg"][s + 1]
        assert [[int(x), int(y)] for x, y in zip(P["seg_start"][a:b], P["seg_vstart"][a:b])] == \
            [[x, y] for x, y, _ in segs]
    # every query tile of every non-empty scope appears once, longest scope first
    w = P["work"]
    assert len(w) == sum(-(-m // A.BLOCK_M) for _, m in ref)
    lens_in_order = P["scope_len"][w[:, 0]]
    assert (np.diff(lens_in_order) <= 0).all()


def test_tile_plan_cap_and_targets():
    import torch
    from paper_2412_16481_b200.pooling import TilePlan  # noqa: F401  (device upload needs CUDA)
    counts = np.array([0, 1500, 3, 1024, 2049])
    reps = -(-counts // TILE_CAP)
    assert reps.tolist() == [0, 2, 1, 1, 3]
