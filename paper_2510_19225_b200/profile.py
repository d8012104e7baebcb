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


def calibrate_profile(instance, batch_sizes: Iterable[int], *, prompt_len: int = 256,
                      steps: int = 32, seed: int = 0) -> ProfileTable:
    """Measure the batch-size -> decode-throughput curve of an idle instance
    at one context: for each batch size b, b throwaway requests (seeded
    synthetic prompts of `prompt_len` ids) decode `steps` tokens together and
    the device time of their constant-batch bursts is taken from
    `decode_profile()`.  Every point shares the context, so the reference's
    plateau rule compares like with like -- an online capture during a
    long-tail step (the reference's `profile_prev`, `sim/engine.py:928-939`)
    sees small batches only late, at long contexts, which bends the curve.
    The instance must hold weights and no requests; it is left idle."""
    import random
    rng = random.Random(seed)
    vocab = instance.shape.vocab
    cap = getattr(instance, "max_seq_len", None)
    if cap is not None and prompt_len + steps + 1 > cap:
        raise ValueError(f"calibration needs {prompt_len + steps + 1} positions, "
                         f"the instance holds {cap}")
    points = []
    for b in sorted(set(int(x) for x in batch_sizes)):
        if b <= 0:
            continue
        instance.decode_profile(reset=True)
        for i in range(b):
            instance.generate(f"__calib{b}_{i}", [rng.randrange(vocab) for _ in range(prompt_len)],
                              target_len=steps + 1)
        instance.run_to_completion(steps)
        points.extend(p for p in instance.decode_profile(reset=True) if p[0] == b)
    return measured_profile_table(points)
