"""Measured decode profile -> the reference's ProfileTable and plateau rule.

SURVEY.md §8 a8: the reference models decode speed (`instance_throughput`,
`pkg/src/spotrl/sim/models.py:39-48`) and captures a batch-size ->
throughput table online from that model (`_refresh_rate` +
`_finalize_profile`, `pkg/src/spotrl/sim/engine.py:786-802,928-939`).  Here
the table comes from the B200 instances themselves: device time per
constant-batch burst of decode steps (CUDA events, `rlb_decode_profile`),
so `estimate_plateau` (`pkg/src/spotrl/balancer.py:95-126`) -- restated below
with the same contract -- and therefore the executing-request branch of the
rebalancer see real hardware numbers.
"""
from __future__ import annotations

from typing import Callable, Iterable

from .domain import ProfileEntry, ProfileTable


class ProfileNotReadyError(RuntimeError):
    """Fewer than two distinct batch sizes observed (`balancer.py:96-116`)."""


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


def estimate_plateau(profile: ProfileTable, current_mean_context: float, *, epsilon: float = 0.05,
                     context_factor: Callable[[float], float] | None = None) -> int:
    """Smallest batch size after which the next observed batch size adds less
    than `epsilon` relative throughput; the largest batch if the curve keeps
    rising.  Points are first rescaled from the capture context to
    `current_mean_context` with `context_factor` (when both are usable), and
    repeated batch sizes are averaged."""
    if profile.distinct_batch_sizes() < 2:
        raise ProfileNotReadyError("profile not ready")
    ratio = 1.0
    if context_factor is not None and profile.context_calibration > 0:
        base = context_factor(profile.context_calibration)
        if base > 0:
            ratio = context_factor(current_mean_context) / base
    points: dict[int, list[float]] = {}
    for e in profile.entries:
        points.setdefault(e.batch_size, []).append(e.decode_throughput * ratio)
    curve = [(b, sum(v) / len(v)) for b, v in sorted(points.items())]
    for i in range(len(curve) - 1):
        b, here = curve[i]
        nxt = curve[i + 1][1]
        if here > 0 and (nxt - here) / here < epsilon:
            return b
    return curve[-1][0]
