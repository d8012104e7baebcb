"""Measured decode profile -> ProfileTable -> estimate_plateau.

The restated plateau rule is checked against the reference's own known
answers (`pkg/tests/test_balancer.py:48-78`, restated here so they run on any
box) and, in this container, against the reference function itself on random
tables."""
import random

import pytest

from paper_2510_19225_b200.domain import ProfileEntry, ProfileTable
from paper_2510_19225_b200.profile import (ProfileNotReadyError, estimate_plateau,
                                           measured_profile_table)


def table(points, calibration=0.0):
    return ProfileTable([ProfileEntry(b, t) for b, t in points], calibration)


def test_known_answers():
    assert estimate_plateau(table([(8, 800.0), (16, 1500.0), (32, 2000.0), (64, 2060.0)]),
                            512.0, epsilon=0.05) == 32
    assert estimate_plateau(table([(4, 400.0), (8, 800.0), (16, 1600.0)]), 512.0) == 16
    with pytest.raises(ProfileNotReadyError, match="profile not ready"):
        estimate_plateau(table([(8, 800.0), (8, 820.0)]), 512.0)
    factor = lambda c: 1.0 / (1.0 + 5e-4 * c)
    assert estimate_plateau(table([(8, 800.0), (16, 1500.0), (32, 2000.0), (64, 2060.0)], 400.0),
                            2000.0, context_factor=factor) == 32


def test_measured_table_from_bursts():
    pts = [(1, 10, 0.1, 100.0), (4, 10, 0.1, 300.0), (4, 30, 0.3, 300.0), (2, 0, 0.0, 50.0)]
    t = measured_profile_table(pts)
    assert [(e.batch_size, round(e.decode_throughput, 6)) for e in t.entries] == [(1, 100.0),
                                                                               (4, 400.0)]
    assert t.context_calibration == pytest.approx((100 * 10 + 300 * 40) / 50)


def test_plateau_matches_reference(spotrl):
    from spotrl.balancer import estimate_plateau as ref_plateau
    from spotrl.domain import ProfileEntry as RE, ProfileTable as RT
    rng = random.Random(0)
    for _ in range(300):
        n = rng.randint(1, 8)
        pts = [(rng.choice([1, 2, 4, 8, 16, 32, 64, 128, 256, 512]), rng.uniform(0, 5e4))
               for _ in range(n)]
        cal = rng.choice([0.0, 300.0, 900.0])
        ctx = rng.uniform(100, 2000)
        eps = rng.choice([0.01, 0.05, 0.2])
        f = rng.choice([None, lambda c: 1.0 / (1.0 + 5e-4 * c)])
        ours = theirs = None
        try:
            ours = estimate_plateau(table(pts, cal), ctx, epsilon=eps, context_factor=f)
        except ProfileNotReadyError:
            ours = "not ready"
        try:
            theirs = ref_plateau(RT([RE(b, t) for b, t in pts], cal), ctx, epsilon=eps,
                                 context_factor=f)
        except Exception as e:   # the reference's ProfileNotReadyError
            assert "not ready" in str(e)
            theirs = "not ready"
        assert ours == theirs, (pts, cal, ctx, eps)
