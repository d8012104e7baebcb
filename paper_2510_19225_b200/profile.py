"""Measured decode profile -> the reference's ProfileTable and plateau rule.

SURVEY.md §8 a8: the reference models decode speed (`instance_throughput`,
`pkg/src/spotrl/sim/models.py:39-48`) and captures a batch-size ->
throughput table online from that model (`_refresh_rate` +
`_finalize_profile`, `pkg/src/spotrl/sim/engine.py:786-802,928-939`).  Here
the table comes from the B200 instances themselves: device time per
constant-batch burst of decode steps (CUDA events, `rlb_decode_profile`),
so the reference's own `estimate_plateau` (`pkg/src/spotrl/balancer.py:95-126`)
and therefore the executing-request branch of its `lb_tick` see real hardware
numbers.
"""
from __future__ import annotations

from typing import Iterable

from spotrl.domain import ProfileEntry, ProfileTable


def measured_profile_table(points: Iterable[tuple[int, int, float, float]]) -> ProfileTable:
    """points: (batch_size, decode steps, device seconds, mean context) from
    one or more instances' `decode_profile()`.  Throughput per batch size is
    time-weighted over all observations: b * sum(steps) / sum(seconds)."""
    acc: dict[int, list[float]] = {}
    ctx_w = ctx_n = 0.0
    for b, steps, seconds, ctx in points:
        if steps <= 0 or seconds <= 0:
            continue
        a = acc.setdefault(int(b), [0.0, 0.0])
        a[0] += steps
        a[1] += seconds
        ctx_w += ctx * steps
        ctx_n += steps
    entries = [ProfileEntry(b, b * s / t) for b, (s, t) in sorted(acc.items())]
    return ProfileTable(entries=entries, context_calibration=ctx_w / ctx_n if ctx_n else 0.0)
